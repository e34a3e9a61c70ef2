// tg_build.cu — device builders for the reference's sparse ternary formats,
// bit-exact in every index array:
//   Tcsc                    tcsc.py:71-92         (blocked with one block, B = K)
//   BlockedTcsc             variants.py:146-178
//   InterleavedBlockedTcsc  variants.py:312-376   (+ symmetric 4-column groups)
//
// Pipeline (count -> scan -> fill):
//   1. planes     W (int8, row-major) -> P[w][n], Q[w][n]: 32-row bit masks of
//                 the +1 / -1 entries of column n (also validates W, dense.py:45-49)
//   2. colprefix  exclusive popcount prefix of P, Q down each column
//                 (pref(row, n) = #(+1 in column n above `row`) in O(1))
//   3. cells      per (block, column) cell: p, q counts (variants.py:338 sub = W[lo:hi])
//   4. lengths +  exclusive int64 scan over cells (TCSC/blocked) or over the
//      scan       3 segments of each cell (interleaved-blocked, variants.py:343-350)
//   5. fill       one thread per (32-row word, column): every set bit knows its
//                 rank t inside its cell from the prefixes, hence its output slot:
//                 rows ascending per cell (np.nonzero order, tcsc.py:81-85); for the
//                 interleaved stream the t-th positive goes to s0+2g*(t/g)+(t%g) if
//                 t < r else s1+(t-r), the t-th negative to s0+2g*(t/g)+g+(t%g) if
//                 t < r else s2+(t-r), r = g*floor(min(p,q)/g) (variants.py:53-65);
//                 symmetric dummies (index K) fill [s0+2r, s1) (variants.py:361-376).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <climits>

#include "tg_internal.h"

namespace tg {

namespace {

struct Layout {
  int64_t K, N, B, KW, nb, ncell, nseg;
  size_t off_P, off_Q, off_cpP, off_cpQ, off_cellP, off_cellQ, off_scanP, off_scanQ, off_chunk, off_misc, total;
};

constexpr int SCAN_CHUNK = 1024;

Layout make_layout(int64_t K, int64_t N, int64_t B) {
  Layout L{};
  L.K = K;
  L.N = N;
  L.B = B;
  L.KW = ceil_div(K, 32);
  L.nb = ceil_div(K, B);
  L.ncell = L.nb * N;
  L.nseg = 3 * L.ncell;  // interleaved-blocked scans segments; TCSC/blocked scan cells
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o += (bytes + 255) / 256 * 256;
    return r;
  };
  L.off_P = take(size_t(L.KW) * N * 4);
  L.off_Q = take(size_t(L.KW) * N * 4);
  L.off_cpP = take(size_t(L.KW + 1) * N * 4);
  L.off_cpQ = take(size_t(L.KW + 1) * N * 4);
  L.off_cellP = take(size_t(L.ncell) * 4);
  L.off_cellQ = take(size_t(L.ncell) * 4);
  L.off_scanP = take(size_t(L.nseg + 1) * 8);   // cells (pos) or segments (interleaved)
  L.off_scanQ = take(size_t(L.ncell + 1) * 8);  // cells (neg)
  L.off_chunk = take(size_t(ceil_div(L.nseg + 1, SCAN_CHUNK) + 1) * 8);
  L.off_misc = take(64);  // [0] bad index (u64), [1] header: kind, g, sym
  L.total = o;
  return L;
}

template <typename T>
T* at(void* ws, size_t off) {
  return reinterpret_cast<T*>(static_cast<uint8_t*>(ws) + off);
}
template <typename T>
const T* at(const void* ws, size_t off) {
  return reinterpret_cast<const T*>(static_cast<const uint8_t*>(ws) + off);
}

// ------------------------------------------------------------------ kernels
__global__ void planes_kernel(const int8_t* __restrict__ W, int64_t K, int64_t N, int64_t ldw,
                              uint32_t* __restrict__ P, uint32_t* __restrict__ Q, int64_t KW,
                              unsigned long long* __restrict__ bad_idx) {
  const int64_t total = KW * N;
  for (int64_t id = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; id < total; id += int64_t(gridDim.x) * blockDim.x) {
    const int64_t w = id / N, n = id % N;
    uint32_t p = 0, q = 0;
    const int64_t k0 = w * 32;
    const int jmax = int(K - k0 < 32 ? K - k0 : 32);
    for (int j = 0; j < jmax; ++j) {
      const int v = W[(k0 + j) * ldw + n];
      p |= uint32_t(v == 1) << j;
      q |= uint32_t(v == -1) << j;
      if (v < -1 || v > 1) atomicMin(bad_idx, (unsigned long long)((k0 + j) * N + n));
    }
    P[id] = p;
    Q[id] = q;
  }
}

// Exclusive popcount prefix down each column: cp[w][n] = sum_{w' < w} popc(P[w'][n]).
__global__ void colprefix_kernel(const uint32_t* __restrict__ P, const uint32_t* __restrict__ Q, int64_t KW,
                                 int64_t N, int32_t* __restrict__ cpP, int32_t* __restrict__ cpQ) {
  const int64_t n = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (n >= N) return;
  int32_t a = 0, b = 0;
  for (int64_t w = 0; w < KW; ++w) {
    cpP[w * N + n] = a;
    cpQ[w * N + n] = b;
    a += __popc(P[w * N + n]);
    b += __popc(Q[w * N + n]);
  }
  cpP[KW * N + n] = a;
  cpQ[KW * N + n] = b;
}

// #(bits set in column n above `row`), row in [0, K].
__device__ __forceinline__ int32_t pref(const uint32_t* __restrict__ P, const int32_t* __restrict__ cp, int64_t N,
                                        int64_t KW, int64_t row, int64_t n) {
  const int64_t w = row >> 5;
  const int r = int(row & 31);
  if (w >= KW) return cp[KW * N + n];
  int32_t v = cp[w * N + n];
  if (r) v += __popc(P[w * N + n] & ((1u << r) - 1u));
  return v;
}

__global__ void cells_kernel(const uint32_t* __restrict__ P, const uint32_t* __restrict__ Q,
                             const int32_t* __restrict__ cpP, const int32_t* __restrict__ cpQ, int64_t K, int64_t N,
                             int64_t B, int64_t KW, int64_t ncell, int32_t* __restrict__ cellP,
                             int32_t* __restrict__ cellQ) {
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < ncell; c += int64_t(gridDim.x) * blockDim.x) {
    const int64_t blk = c / N, n = c % N;
    const int64_t lo = blk * B, hi = min(lo + B, K);
    cellP[c] = pref(P, cpP, N, KW, hi, n) - pref(P, cpP, N, KW, lo, n);
    cellQ[c] = pref(Q, cpQ, N, KW, hi, n) - pref(Q, cpQ, N, KW, lo, n);
  }
}

__device__ __forceinline__ int32_t interleaved_r(int32_t p, int32_t q, int g) {
  const int32_t m = p < q ? p : q;
  return g * (m / g);
}

// Segment lengths of the interleaved-blocked stream, 3 per cell (variants.py:343-350).
__global__ void ib_lengths_kernel(const int32_t* __restrict__ cellP, const int32_t* __restrict__ cellQ, int64_t N,
                                  int64_t ncell, int g, int sym, int64_t* __restrict__ len) {
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < ncell; c += int64_t(gridDim.x) * blockDim.x) {
    const int32_t p = cellP[c], q = cellQ[c];
    const int32_t r = interleaved_r(p, q, g);
    int64_t inter = 2 * int64_t(r);
    if (sym) {
      const int64_t n = c % N, c0 = c - (n & 3);
      for (int j = 0; j < 4; ++j) {
        const int64_t o = 2 * int64_t(interleaved_r(cellP[c0 + j], cellQ[c0 + j], g));
        inter = o > inter ? o : inter;
      }
    }
    len[3 * c] = inter;
    len[3 * c + 1] = p - r;
    len[3 * c + 2] = q - r;
  }
}

__global__ void copy_lengths_kernel(const int32_t* __restrict__ cell, int64_t n, int64_t* __restrict__ len) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    len[i] = cell[i];
}

// In-place exclusive scan of len[0, n) (int64), len[n] = total.  Three phases.
__global__ void scan_chunk_sums(const int64_t* __restrict__ len, int64_t n, int64_t* __restrict__ chunk) {
  __shared__ int64_t red[32];
  const int64_t base = int64_t(blockIdx.x) * SCAN_CHUNK;
  int64_t s = 0;
  for (int i = threadIdx.x; i < SCAN_CHUNK; i += blockDim.x)
    if (base + i < n) s += len[base + i];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
    chunk[blockIdx.x] = t;
  }
}

__global__ void scan_chunk_prefix(int64_t* __restrict__ chunk, int64_t nchunks) {
  // single block; sequential per thread over a contiguous range, then a block scan
  __shared__ int64_t part[1024];
  const int64_t per = (nchunks + blockDim.x - 1) / blockDim.x;
  const int64_t a = threadIdx.x * per, b = min(a + per, nchunks);
  int64_t s = 0;
  for (int64_t i = a; i < b; ++i) s += chunk[i];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int t = 0; t < int(blockDim.x); ++t) {
      const int64_t v = part[t];
      part[t] = run;
      run += v;
    }
    chunk[nchunks] = run;
  }
  __syncthreads();
  s = part[threadIdx.x];
  for (int64_t i = a; i < b; ++i) {
    const int64_t v = chunk[i];
    chunk[i] = s;
    s += v;
  }
}

__global__ void scan_apply(int64_t* __restrict__ len, int64_t n, const int64_t* __restrict__ chunk, int64_t nchunks) {
  __shared__ int64_t vals[SCAN_CHUNK];
  const int64_t base = int64_t(blockIdx.x) * SCAN_CHUNK;
  for (int i = threadIdx.x; i < SCAN_CHUNK; i += blockDim.x) vals[i] = (base + i < n) ? len[base + i] : 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = chunk[blockIdx.x];
    for (int i = 0; i < SCAN_CHUNK; ++i) {
      const int64_t v = vals[i];
      vals[i] = run;
      run += v;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < SCAN_CHUNK; i += blockDim.x)
    if (base + i < n) len[base + i] = vals[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) len[n] = chunk[nchunks];
}

// Offsets tables -------------------------------------------------------------
// TCSC / blocked: col_start[blk][n] = scan[blk*N + n], col_start[blk][N] = scan[(blk+1)*N].
__global__ void blocked_offsets_kernel(const int64_t* __restrict__ scan, int64_t N, int64_t nb,
                                       int32_t* __restrict__ cs) {
  const int64_t total = nb * (N + 1);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t blk = i / (N + 1), n = i % (N + 1);
    cs[i] = int32_t(scan[blk * N + n]);
  }
}

__global__ void ib_offsets_kernel(const int64_t* __restrict__ scan, int64_t nseg, int32_t* __restrict__ ptr) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i <= nseg; i += int64_t(gridDim.x) * blockDim.x)
    ptr[i] = int32_t(scan[i]);
}

// Fill row indices of TCSC / blocked (one sign at a time).
__global__ void fill_csc_kernel(const uint32_t* __restrict__ P, const int32_t* __restrict__ cp,
                                const int64_t* __restrict__ start, int64_t K, int64_t N, int64_t B, int64_t KW,
                                int32_t* __restrict__ rows) {
  const int64_t total = KW * N;
  for (int64_t id = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; id < total; id += int64_t(gridDim.x) * blockDim.x) {
    const int64_t w = id / N, n = id % N;
    uint32_t bits = P[id];
    if (!bits) continue;
    const int32_t base = cp[id];
    int32_t seen = 0;
    int64_t cur_blk = -1, cell_base = 0;
    while (bits) {
      const int j = __ffs(bits) - 1;
      bits &= bits - 1;
      const int64_t k = w * 32 + j;
      const int64_t blk = k / B;
      if (blk != cur_blk) {
        cur_blk = blk;
        cell_base = start[blk * N + n] - pref(P, cp, N, KW, blk * B, n);
      }
      rows[cell_base + base + seen] = int32_t(k);
      ++seen;
    }
  }
}

// Fill the interleaved-blocked stream (both signs), variants.py:53-65.
__global__ void fill_ib_kernel(const uint32_t* __restrict__ P, const uint32_t* __restrict__ Q,
                               const int32_t* __restrict__ cpP, const int32_t* __restrict__ cpQ,
                               const int32_t* __restrict__ cellP, const int32_t* __restrict__ cellQ,
                               const int64_t* __restrict__ seg, int64_t K, int64_t N, int64_t B, int64_t KW, int g,
                               int32_t* __restrict__ ai) {
  const int64_t total = KW * N;
  for (int64_t id = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; id < total; id += int64_t(gridDim.x) * blockDim.x) {
    const int64_t w = id / N, n = id % N;
#pragma unroll 1
    for (int sign = 0; sign < 2; ++sign) {
      const uint32_t* PP = sign ? Q : P;
      const int32_t* cp = sign ? cpQ : cpP;
      uint32_t bits = PP[id];
      const int32_t base = cp[id];
      int32_t seen = 0;
      int64_t cur_blk = -1, cell_first = 0, s0 = 0, srem = 0;
      int32_t r = 0;
      while (bits) {
        const int j = __ffs(bits) - 1;
        bits &= bits - 1;
        const int64_t k = w * 32 + j;
        const int64_t blk = k / B;
        if (blk != cur_blk) {
          cur_blk = blk;
          const int64_t c = blk * N + n;
          cell_first = pref(PP, cp, N, KW, blk * B, n);
          r = interleaved_r(cellP[c], cellQ[c], g);
          s0 = seg[3 * c];
          srem = seg[3 * c + 1 + sign];
        }
        const int64_t t = int64_t(base) + seen - cell_first;
        int64_t dest;
        if (t < r) dest = s0 + 2 * g * (t / g) + (sign ? g : 0) + (t % g);
        else dest = srem + (t - r);
        ai[dest] = int32_t(k);
        ++seen;
      }
    }
  }
}

// Symmetric padding: [s0 + 2r, s1) <- K in every cell.
__global__ void fill_dummies_kernel(const int32_t* __restrict__ cellP, const int32_t* __restrict__ cellQ,
                                    const int64_t* __restrict__ seg, int64_t ncell, int g, int64_t K,
                                    int32_t* __restrict__ ai) {
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < ncell; c += int64_t(gridDim.x) * blockDim.x) {
    const int32_t r = interleaved_r(cellP[c], cellQ[c], g);
    for (int64_t i = seg[3 * c] + 2 * int64_t(r); i < seg[3 * c + 1]; ++i) ai[i] = int32_t(K);
  }
}

// ---- SymmetricInterleavedTcsc (variants.py:540-631): one stream per column,
// pairs per 4-column group = the group's max(max(p, q)) rounded up to lcm(4, g).
__device__ __forceinline__ int64_t sym_quantum(int g) {
  int a = 4, b = g;
  while (b) {
    const int t = a % b;
    a = b;
    b = t;
  }
  return int64_t(4 / a) * g;
}

__global__ void sym_lengths_kernel(const int32_t* __restrict__ cellP, const int32_t* __restrict__ cellQ, int64_t N,
                                   int g, int64_t* __restrict__ len) {
  for (int64_t n = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; n < N; n += int64_t(gridDim.x) * blockDim.x) {
    const int64_t n0 = n & ~int64_t(3);
    int64_t need = 0;
    for (int j = 0; j < 4; ++j) {
      const int64_t m = max(cellP[n0 + j], cellQ[n0 + j]);
      need = m > need ? m : need;
    }
    const int64_t q = sym_quantum(g);
    len[n] = need ? 2 * ((need + q - 1) / q * q) : 0;
  }
}

__global__ void fill_value_kernel(int32_t* __restrict__ a, int64_t n, int32_t v) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    a[i] = v;
}

// t-th positive of column n -> s0 + 2g (t / g) + (t % g); t-th negative -> ... + g.
__global__ void fill_sym_kernel(const uint32_t* __restrict__ P, const uint32_t* __restrict__ Q,
                                const int32_t* __restrict__ cpP, const int32_t* __restrict__ cpQ,
                                const int64_t* __restrict__ start, int64_t N, int64_t KW, int g,
                                int32_t* __restrict__ idx) {
  const int64_t total = KW * N;
  for (int64_t id = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; id < total; id += int64_t(gridDim.x) * blockDim.x) {
    const int64_t w = id / N, n = id % N;
    const int64_t s0 = start[n];
#pragma unroll 1
    for (int sign = 0; sign < 2; ++sign) {
      uint32_t bits = (sign ? Q : P)[id];
      int64_t t = (sign ? cpQ : cpP)[id];  // rank of the first set bit in its column
      while (bits) {
        const int j = __ffs(bits) - 1;
        bits &= bits - 1;
        idx[s0 + 2 * g * (t / g) + (sign ? g : 0) + (t % g)] = int32_t(w * 32 + j);
        ++t;
      }
    }
  }
}

// ---- CompressedTcsc (variants.py:451-532): codes[n][gi] = sum_i (w(5gi+i, n) + 1) 3^i.
// Thread per (gi, n), n fastest so the reads of W rows coalesce.
__global__ void compress_kernel(const int8_t* __restrict__ W, int64_t K, int64_t N, int64_t ldw, int64_t G,
                                uint8_t* __restrict__ codes, unsigned long long* __restrict__ bad) {
  const int64_t total = G * N;
  for (int64_t id = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; id < total; id += int64_t(gridDim.x) * blockDim.x) {
    const int64_t gi = id / N, n = id % N;
    int code = 0, p3 = 1;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const int64_t k = 5 * gi + i;
      int v = 0;
      if (k < K) {
        v = W[k * ldw + n];
        if (v < -1 || v > 1) {
          atomicMin(bad, (unsigned long long)(k * N + n));
          v = 0;
        }
      }
      code += (v + 1) * p3;
      p3 *= 3;
    }
    codes[n * G + gi] = uint8_t(code);
  }
}

__global__ void codes_check_kernel(const uint8_t* __restrict__ codes, int64_t n, tg_device_flags* __restrict__ flags) {
  bool badc = false;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    badc |= codes[i] >= 243;
  if (__any_sync(0xffffffffu, badc) && (threadIdx.x & 31) == 0) atomicOr(&flags->corrupt, 4);
}

unsigned grid_for(int64_t work, int threads = 256) {
  const int64_t b = (work + threads - 1) / threads;
  return unsigned(std::max<int64_t>(1, std::min<int64_t>(b, 148 * 64)));
}

int run_scan(int64_t* len, int64_t n, int64_t* chunk, cudaStream_t st) {
  const int64_t nchunks = ceil_div(n, SCAN_CHUNK);
  if (nchunks > 0) scan_chunk_sums<<<unsigned(nchunks), 256, 0, st>>>(len, n, chunk);
  scan_chunk_prefix<<<1, 1024, 0, st>>>(chunk, nchunks);
  if (nchunks > 0) {
    scan_apply<<<unsigned(nchunks), 256, 0, st>>>(len, n, chunk, nchunks);
  } else {
    // n == 0: write the zero total
    cudaMemsetAsync(len, 0, sizeof(int64_t), st);
  }
  return check_launch("scan");
}

struct Header {
  int32_t kind, g, sym, pad;
};

}  // namespace

}  // namespace tg

using namespace tg;

extern "C" {

size_t tg_build_workspace_bytes(int64_t K, int64_t N, int64_t B) {
  if (K < 1 || N < 1 || B < 1) return 0;
  return make_layout(K, N, B).total;
}

int tg_build_count(const int8_t* W, int64_t K, int64_t N, int64_t ldw, int kind, int64_t B, int g, int symmetric,
                   void* ws, size_t ws_bytes, tg_sizes* sizes, void* stream) {
  if (K < 1 || N < 1) return set_error(TG_ERR_PARAM, "ternary matrix must be 2-D and non-empty");
  if (B < 1) return set_error(TG_ERR_PARAM, "block size must be >= 1");
  if (ldw < N) return set_error(TG_ERR_PARAM, "ldw must be >= N");
  if (!W || !ws || !sizes) return set_error(TG_ERR_PARAM, "null pointer");
  if (kind != TG_FMT_TCSC && kind != TG_FMT_BLOCKED && kind != TG_FMT_INTERLEAVED_BLOCKED &&
      kind != TG_FMT_SYMMETRIC)
    return set_error(TG_ERR_PARAM, "unknown format kind");
  if (kind == TG_FMT_SYMMETRIC && (g < 1 || N % 4 != 0))
    return set_error(TG_ERR_PARAM, g < 1 ? "group size must be >= 1" : "N must be divisible by 4");
  if (kind == TG_FMT_INTERLEAVED_BLOCKED && g < 1) return set_error(TG_ERR_PARAM, "group size must be >= 1");
  if (kind == TG_FMT_INTERLEAVED_BLOCKED && symmetric && N % 4 != 0)
    return set_error(TG_ERR_PARAM, "symmetric groups need N divisible by 4");
  if (kind == TG_FMT_TCSC || kind == TG_FMT_SYMMETRIC) B = K;
  if (K >= INT32_MAX) return set_error(TG_ERR_OVERFLOW, "K does not fit int32 row indices");
  const Layout Lo = make_layout(K, N, B);
  if (ws_bytes < Lo.total) return set_error(TG_ERR_PARAM, "build workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);

  uint32_t* P = at<uint32_t>(ws, Lo.off_P);
  uint32_t* Q = at<uint32_t>(ws, Lo.off_Q);
  int32_t* cpP = at<int32_t>(ws, Lo.off_cpP);
  int32_t* cpQ = at<int32_t>(ws, Lo.off_cpQ);
  int32_t* cellP = at<int32_t>(ws, Lo.off_cellP);
  int32_t* cellQ = at<int32_t>(ws, Lo.off_cellQ);
  int64_t* scanP = at<int64_t>(ws, Lo.off_scanP);
  int64_t* scanQ = at<int64_t>(ws, Lo.off_scanQ);
  int64_t* chunk = at<int64_t>(ws, Lo.off_chunk);
  unsigned long long* bad = at<unsigned long long>(ws, Lo.off_misc);
  Header* hdr = at<Header>(ws, Lo.off_misc + 8);

  cudaError_t e = cudaMemsetAsync(bad, 0xFF, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaMemsetAsync");
  planes_kernel<<<grid_for(Lo.KW * N), 256, 0, st>>>(W, K, N, ldw, P, Q, Lo.KW, bad);
  colprefix_kernel<<<unsigned(ceil_div(N, 128)), 128, 0, st>>>(P, Q, Lo.KW, N, cpP, cpQ);
  cells_kernel<<<grid_for(Lo.ncell), 256, 0, st>>>(P, Q, cpP, cpQ, K, N, B, Lo.KW, Lo.ncell, cellP, cellQ);
  int rc = check_launch("tg_build_count");
  if (rc != TG_OK) return rc;
  if (kind == TG_FMT_INTERLEAVED_BLOCKED) {
    ib_lengths_kernel<<<grid_for(Lo.ncell), 256, 0, st>>>(cellP, cellQ, N, Lo.ncell, g, symmetric, scanP);
    rc = run_scan(scanP, Lo.nseg, chunk, st);
  } else if (kind == TG_FMT_SYMMETRIC) {
    sym_lengths_kernel<<<grid_for(N), 256, 0, st>>>(cellP, cellQ, N, g, scanP);
    rc = run_scan(scanP, N, chunk, st);
  } else {
    copy_lengths_kernel<<<grid_for(Lo.ncell), 256, 0, st>>>(cellP, Lo.ncell, scanP);
    copy_lengths_kernel<<<grid_for(Lo.ncell), 256, 0, st>>>(cellQ, Lo.ncell, scanQ);
    rc = run_scan(scanP, Lo.ncell, chunk, st);
    if (rc == TG_OK) rc = run_scan(scanQ, Lo.ncell, chunk, st);
  }
  if (rc != TG_OK) return rc;
  Header h{kind, g, symmetric, 0};
  e = cudaMemcpyAsync(hdr, &h, sizeof(h), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaMemcpyAsync(header)");

  unsigned long long bad_h = 0;
  int64_t totP = 0, totQ = 0;
  e = cudaMemcpyAsync(&bad_h, bad, sizeof(bad_h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(&totP,
                        scanP + (kind == TG_FMT_INTERLEAVED_BLOCKED ? Lo.nseg : kind == TG_FMT_SYMMETRIC ? N : Lo.ncell),
                        sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && kind != TG_FMT_INTERLEAVED_BLOCKED && kind != TG_FMT_SYMMETRIC)
    e = cudaMemcpyAsync(&totQ, scanQ + Lo.ncell, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return set_cuda_error(e, "tg_build_count");
  if (bad_h != ~0ull) {
    const int64_t k = int64_t(bad_h) / N, n = int64_t(bad_h) % N;
    int8_t v = 0;
    cudaMemcpy(&v, W + k * ldw + n, 1, cudaMemcpyDeviceToHost);
    char msg[160];
    snprintf(msg, sizeof msg, "entry (%lld, %lld) = %d is not in {-1, 0, +1}", (long long)k, (long long)n, int(v));
    return set_error(TG_ERR_PARAM, msg);
  }
  if (totP > INT32_MAX || totQ > INT32_MAX) return set_error(TG_ERR_OVERFLOW, "index arrays exceed int32 offsets");
  sizes->num_blocks = Lo.nb;
  if (kind == TG_FMT_INTERLEAVED_BLOCKED) {
    sizes->nnz_pos = sizes->nnz_neg = 0;
    sizes->n_indices = totP;
    sizes->offsets_len = Lo.nseg + 1;
  } else if (kind == TG_FMT_SYMMETRIC) {
    sizes->nnz_pos = sizes->nnz_neg = 0;
    sizes->n_indices = totP;
    sizes->offsets_len = N + 1;
  } else {
    sizes->nnz_pos = totP;
    sizes->nnz_neg = totQ;
    sizes->n_indices = totP + totQ;
    sizes->offsets_len = Lo.nb * (N + 1);
  }
  return TG_OK;
}

static int fill_csc_common(const void* ws, int64_t K, int64_t N, int64_t B, int32_t* csp, int32_t* rip, int32_t* csn,
                           int32_t* rin, cudaStream_t st) {
  const Layout Lo = make_layout(K, N, B);
  const uint32_t* P = at<uint32_t>(ws, Lo.off_P);
  const uint32_t* Q = at<uint32_t>(ws, Lo.off_Q);
  const int32_t* cpP = at<int32_t>(ws, Lo.off_cpP);
  const int32_t* cpQ = at<int32_t>(ws, Lo.off_cpQ);
  const int64_t* scanP = at<int64_t>(ws, Lo.off_scanP);
  const int64_t* scanQ = at<int64_t>(ws, Lo.off_scanQ);
  blocked_offsets_kernel<<<grid_for(Lo.nb * (N + 1)), 256, 0, st>>>(scanP, N, Lo.nb, csp);
  blocked_offsets_kernel<<<grid_for(Lo.nb * (N + 1)), 256, 0, st>>>(scanQ, N, Lo.nb, csn);
  fill_csc_kernel<<<grid_for(Lo.KW * N), 256, 0, st>>>(P, cpP, scanP, K, N, B, Lo.KW, rip);
  fill_csc_kernel<<<grid_for(Lo.KW * N), 256, 0, st>>>(Q, cpQ, scanQ, K, N, B, Lo.KW, rin);
  return check_launch("tg_build_fill");
}

int tg_build_fill_tcsc(const void* ws, int64_t K, int64_t N, int32_t* csp, int32_t* rip, int32_t* csn, int32_t* rin,
                       void* stream) {
  if (K < 1 || N < 1 || !ws || !csp || !csn) return set_error(TG_ERR_PARAM, "bad arguments");
  return fill_csc_common(ws, K, N, K, csp, rip, csn, rin, static_cast<cudaStream_t>(stream));
}

int tg_build_fill_blocked(const void* ws, int64_t K, int64_t N, int64_t B, int32_t* csp, int32_t* rip, int32_t* csn,
                          int32_t* rin, void* stream) {
  if (K < 1 || N < 1 || B < 1 || !ws || !csp || !csn) return set_error(TG_ERR_PARAM, "bad arguments");
  return fill_csc_common(ws, K, N, B, csp, rip, csn, rin, static_cast<cudaStream_t>(stream));
}

int tg_build_fill_interleaved_blocked(const void* ws, int64_t K, int64_t N, int64_t B, int g, int symmetric,
                                      int32_t* ai, int32_t* ptr, void* stream) {
  if (K < 1 || N < 1 || B < 1 || g < 1 || !ws || !ptr) return set_error(TG_ERR_PARAM, "bad arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Layout Lo = make_layout(K, N, B);
  const uint32_t* P = at<uint32_t>(ws, Lo.off_P);
  const uint32_t* Q = at<uint32_t>(ws, Lo.off_Q);
  const int32_t* cpP = at<int32_t>(ws, Lo.off_cpP);
  const int32_t* cpQ = at<int32_t>(ws, Lo.off_cpQ);
  const int32_t* cellP = at<int32_t>(ws, Lo.off_cellP);
  const int32_t* cellQ = at<int32_t>(ws, Lo.off_cellQ);
  const int64_t* seg = at<int64_t>(ws, Lo.off_scanP);
  ib_offsets_kernel<<<grid_for(Lo.nseg + 1), 256, 0, st>>>(seg, Lo.nseg, ptr);
  fill_ib_kernel<<<grid_for(Lo.KW * N), 256, 0, st>>>(P, Q, cpP, cpQ, cellP, cellQ, seg, K, N, B, Lo.KW, g, ai);
  if (symmetric) fill_dummies_kernel<<<grid_for(Lo.ncell), 256, 0, st>>>(cellP, cellQ, seg, Lo.ncell, g, K, ai);
  return check_launch("tg_build_fill_interleaved_blocked");
}

int tg_build_fill_symmetric(const void* ws, int64_t K, int64_t N, int g, int32_t* indices, int32_t* col_ptr,
                            int64_t n_indices, void* stream) {
  if (K < 1 || N < 1 || g < 1 || N % 4 != 0 || !ws || !col_ptr || n_indices < 0)
    return set_error(TG_ERR_PARAM, "bad arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Layout Lo = make_layout(K, N, K);
  const uint32_t* P = at<uint32_t>(ws, Lo.off_P);
  const uint32_t* Q = at<uint32_t>(ws, Lo.off_Q);
  const int32_t* cpP = at<int32_t>(ws, Lo.off_cpP);
  const int32_t* cpQ = at<int32_t>(ws, Lo.off_cpQ);
  const int64_t* start = at<int64_t>(ws, Lo.off_scanP);
  ib_offsets_kernel<<<grid_for(N + 1), 256, 0, st>>>(start, N, col_ptr);
  if (n_indices > 0) {
    if (!indices) return set_error(TG_ERR_PARAM, "null indices");
    fill_value_kernel<<<grid_for(n_indices), 256, 0, st>>>(indices, n_indices, int32_t(K));  // dummies
    fill_sym_kernel<<<grid_for(Lo.KW * N), 256, 0, st>>>(P, Q, cpP, cpQ, start, N, Lo.KW, g, indices);
  }
  return check_launch("tg_build_fill_symmetric");
}

int tg_build_compressed(const int8_t* W, int64_t K, int64_t N, int64_t ldw, uint8_t* codes, void* stream) {
  if (K < 1 || N < 1) return set_error(TG_ERR_PARAM, "ternary matrix must be 2-D and non-empty");
  if (ldw < N) return set_error(TG_ERR_PARAM, "ldw must be >= N");
  if (!W || !codes) return set_error(TG_ERR_PARAM, "null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t G = ceil_div(K, 5);
  unsigned long long* bad = nullptr;
  cudaError_t e = cudaMallocAsync(&bad, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaMallocAsync");
  cudaMemsetAsync(bad, 0xFF, sizeof(unsigned long long), st);
  compress_kernel<<<grid_for(G * N), 256, 0, st>>>(W, K, N, ldw, G, codes, bad);
  unsigned long long bad_h = ~0ull;
  e = cudaMemcpyAsync(&bad_h, bad, sizeof(bad_h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaFreeAsync(bad, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return set_cuda_error(e, "tg_build_compressed");
  if (bad_h != ~0ull) {
    const int64_t k = int64_t(bad_h) / N, n = int64_t(bad_h) % N;
    int8_t v = 0;
    cudaMemcpy(&v, W + k * ldw + n, 1, cudaMemcpyDeviceToHost);
    char msg[160];
    snprintf(msg, sizeof msg, "entry (%lld, %lld) = %d is not in {-1, 0, +1}", (long long)k, (long long)n, int(v));
    return set_error(TG_ERR_PARAM, msg);
  }
  return TG_OK;
}

int tg_codes_check(const uint8_t* codes, int64_t count, tg_device_flags* flags, void* stream) {
  if (count < 0 || (count && (!codes || !flags))) return set_error(TG_ERR_PARAM, "bad arguments");
  if (count == 0) return TG_OK;
  codes_check_kernel<<<grid_for(count), 256, 0, static_cast<cudaStream_t>(stream)>>>(codes, count, flags);
  return check_launch("tg_codes_check");
}

}  // extern "C"
