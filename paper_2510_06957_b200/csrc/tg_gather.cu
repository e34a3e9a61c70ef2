// tg_gather.cu — CUDA-core gather-add path over the reference's own index
// streams (no re-encoding).  Each output element Y[m, n] is accumulated by one
// thread lane in exactly the reference kernel's fp32 operation order, so the
// result is bit-identical to the reference for any finite input:
//
//   VAR_BASE      kernels/scalar.py:109-132  acc=0; acc+=x (pos); acc-=x (neg); out=b+acc
//   VAR_UNROLLED  kernels/scalar.py:156-257  uf accumulator banks; bank u takes stream
//                 positions start+u, start+u+uf, ...; the tail of each sign goes to
//                 bank 0; tot = ((0 + bank0) + bank1) + ...; out = b + tot
//   VAR_BLOCKED   kernels/scalar.py:286-367  out=b; per block: rows m < floor(M/mr)*mr use the
//                 banked sum (out += tot), the leftover rows acc=0; +pos; -neg; out+=acc
//   VAR_IB        kernels/scalar.py:397-485  out=b; per block: acc=0; runs of g (+,-); +rem; -rem; out+=acc
//   VAR_OPTIMAL   kernels/simd.py:282-420    out=b; per block: acc over the interleaved segment
//                 (sign = parity of t//g); out+=acc; out+=x (pos rem); out-=x (neg rem)
//   then PReLU y = (y > 0) ? y : alpha*y in fp32 (simd.py:410-417).
//
// Layout: X is first transposed into row-group tiles Xt[M_pad/128][K+1][128]
// (row K = the dummy slot of PaddedInput, simd.py:40-75), so one warp-wide
// float4 load fetches X[m, k] for 128 consecutive rows m (lanes = rows, one warp
// = one column n) and a K window of one row group is one contiguous byte range.
//
// Two kernels walk the streams:
//   tg_gather_staged_kernel (BASE, IB, OPTIMAL: the BASELINE variants).  A CTA owns
//     128 rows x up to 64 columns.  K windows of its X rows (192 k x 512 B) are
//     brought into shared memory by TMA bulk copies (double-buffered, mbarrier
//     completion) while each warp walks its columns' streams: 128 stream indices
//     per coalesced 128-bit-per-lane load, broadcast by shuffle, one conflict-free
//     LDS.128 per index (the lanes read 512 consecutive bytes), four fp32 adds per
//     lane.  A stream segment is ascending in k, so a column simply pauses at the
//     end of the staged window and resumes in the next one: the per-output order
//     of the reference is untouched.  Indices outside the window (the dummy index
//     K, the short remainder segments, any unsorted stream) are read from the
//     transposed copy in L2.  Bound: one 512 B shared-memory wavefront group per
//     128 adds = 32 adds/clk/SM, a quarter of the fp32-add peak.
//   tg_gather_kernel (every variant): the same walk with every operand from L1/L2.
// Outputs are staged in shared memory and written row-wise.
#include <cuda_runtime.h>
#include <climits>
#include <cstdint>
#include <cstdlib>

#include "tg_internal.h"
#include "tg_ptx.cuh"
#include "tg_walk.cuh"

namespace tg {

constexpr int G_WARPS = 8;    // columns per CTA
constexpr int G_ROWS = 128;   // rows per CTA (4 per lane)

size_t gather_ws_bytes(int64_t M, int64_t K) {
  return size_t(K + 1) * size_t(round_up(M, G_ROWS)) * sizeof(float) + 256;
}

// X (M x ldx) -> Xt[M_pad/128][K+1][128], zero padded; columns k < Kx are read from X (Kx = K + 1
// for a padded input: the dummy index K reads X[:, K] as the reference kernels do).
__global__ void tg_transpose_kernel(const float* __restrict__ X, int64_t M, int64_t K, int64_t Kx, int64_t ldx,
                                    float* __restrict__ Xt, int64_t M_pad, tg_device_flags* flags) {
  __shared__ float tile[32][33];
  const int64_t k0 = int64_t(blockIdx.x) * 32, m0 = int64_t(blockIdx.y) * 32;
  bool bad = false;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t m = m0 + r, k = k0 + threadIdx.x;
    float v = 0.f;
    if (m < M && k < Kx) {
      v = X[m * ldx + k];
      bad |= !isfinite(v);
    }
    tile[r][threadIdx.x] = v;
  }
  if (flags && bad) atomicOr(&flags->bad_input, 4);
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t k = k0 + r, m = m0 + threadIdx.x;
    if (k <= K && m < M_pad) Xt[((m / G_ROWS) * (K + 1) + k) * G_ROWS + (m % G_ROWS)] = tile[threadIdx.x][r];
  }
}

template <int VAR>
__global__ void __launch_bounds__(G_WARPS * 32)
    tg_gather_kernel(const float* __restrict__ Xt, int64_t K, int64_t M, GatherArgs a,
                     const float* __restrict__ bias, float* __restrict__ Y, int64_t ldy, int use_alpha, float alpha,
                     tg_device_flags* __restrict__ flags) {
  __shared__ float stage[G_ROWS][G_WARPS + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t N = a.N;
  const int64_t n = int64_t(blockIdx.x) * G_WARPS + warp;
  const int64_t mrow = int64_t(blockIdx.y) * G_ROWS + lane * 4;
  float4 out = make_float4(0.f, 0.f, 0.f, 0.f);
  if (n < N) {
    const float b = bias ? __ldg(bias + n) : 0.f;
    unsigned banked = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) banked |= unsigned(mrow + r < a.m_full) << r;
    out = column_value<VAR>(a, n, b, SrcXt{Xt + int64_t(blockIdx.y) * (K + 1) * G_ROWS + lane * 4, G_ROWS}, banked);
  }
  // epilogue: PReLU, flags, row-wise store through shared memory
  float v[4] = {out.x, out.y, out.z, out.w};
  bool bad = false;
  unsigned long long npos = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const bool live = n < N && mrow + r < M;
    if (use_alpha && !(v[r] > 0.f)) {
      if (live) ++npos;
      v[r] = alpha * v[r];
    }
    if (live) bad |= !isfinite(v[r]);
    stage[lane * 4 + r][warp] = v[r];
  }
  if (flags) {
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&flags->nonfinite_output, 1);
    for (int o = 16; o; o >>= 1) npos += __shfl_xor_sync(0xffffffffu, npos, o);
    if (lane == 0 && npos) atomicAdd(reinterpret_cast<unsigned long long*>(&flags->nonpositive_outputs), npos);
  }
  __syncthreads();
  const int64_t nbase = int64_t(blockIdx.x) * G_WARPS;
  for (int e = threadIdx.x; e < G_ROWS * G_WARPS; e += blockDim.x) {
    const int r = e / G_WARPS, c = e % G_WARPS;
    const int64_t m = int64_t(blockIdx.y) * G_ROWS + r, nn = nbase + c;
    if (m < M && nn < N) Y[m * ldy + nn] = stage[r][c];
  }
}


// ------------------------------------------------------------------ staged kernel
constexpr int S_WARPS = 32;                      // warps per CTA
constexpr int S_CPW = 2;                         // columns per warp (at most)
constexpr int S_CMAX = S_WARPS * S_CPW;          // columns per CTA (at most)
constexpr int S_WK = 192;                        // k per staged window: 192 x 512 B = 96 KB
constexpr int S_STAGE_FLOATS = S_WK * G_ROWS;
constexpr size_t S_SMEM = 2 * size_t(S_STAGE_FLOATS) * sizeof(float);  // two stages, 192 KB
static_assert(size_t(G_ROWS) * (S_CMAX + 1) * sizeof(float) <= S_SMEM, "the Y tile reuses the window memory");

struct Window {
  const float4* base;  // this lane's float4 column of the staged stage: element d is X[rows of the lane, k0 + d]
  int32_t k0;          // first staged k
  uint32_t nk;         // staged k count
  int32_t k1;          // the column pauses at the first stream index >= k1 (INT32_MAX in a sweep's last window)
};

// acc +- x as fma(x, +-1, acc): x * (+-1) is exact, so the single rounding is that of the
// reference's add / subtract, bit for bit -- and the sign is data, not a branch (the switch over
// the four sign phases of a group took 45% of the kernel's stall samples).
__device__ __forceinline__ void fma4(float4& acc, const float4 x, const float m) {
  acc.x = __fmaf_rn(x.x, m, acc.x);
  acc.y = __fmaf_rn(x.y, m, acc.y);
  acc.z = __fmaf_rn(x.z, m, acc.z);
  acc.w = __fmaf_rn(x.w, m, acc.w);
}

// Sign of stream position t (relative to the segment start): GM 0 = one sign for the whole
// segment (TCSC pos / neg streams), GM 2 = alternating runs of 2 (the default g), GM 1 = runs of g.
template <int GM>
__device__ __forceinline__ bool is_neg(int32_t t, int g, bool neg0) {
  if (GM == 0) return neg0;
  if (GM == 2) return ((t >> 1) & 1) != 0;
  return ((t / g) & 1) != 0;
}

// Walk positions [i, e) of the stream `ai` into acc, strictly in stream order, until the
// first index >= w.k1; returns the position reached (e when the segment is finished).
// 128 stream positions per coalesced load (one int4 per lane), broadcast by shuffle.
// `ai` must be 16-byte aligned (positions are loaded in aligned groups of four).
template <int GM>
__device__ __forceinline__ int32_t walk_staged(float4& acc, const int32_t* __restrict__ ai, int32_t i, const int32_t e,
                                               const int32_t s0, const int g, const bool neg0, const Window& w,
                                               const SrcXt& glob, const int lane) {
  while (i < e) {
    const int32_t base = i & ~127;
    const int32_t p = base + 4 * lane;
    int4 mine = make_int4(0, 0, 0, 0);
    if (p < e) mine = __ldg(reinterpret_cast<const int4*>(ai + p));
    const int32_t jend = min(e, base + 128);
    for (int32_t q = (i - base) >> 2; base + 4 * q < jend; ++q) {
      int32_t kk[4];
      kk[0] = __shfl_sync(0xffffffffu, mine.x, q);
      kk[1] = __shfl_sync(0xffffffffu, mine.y, q);
      kk[2] = __shfl_sync(0xffffffffu, mine.z, q);
      kk[3] = __shfl_sync(0xffffffffu, mine.w, q);
      const int32_t pq = base + 4 * q;
      const int32_t c0 = i - pq, c1 = jend - pq;  // live components: max(c0, 0) <= c < min(c1, 4)
      const uint32_t d0 = uint32_t(kk[0] - w.k0), d1 = uint32_t(kk[1] - w.k0);
      const uint32_t d2 = uint32_t(kk[2] - w.k0), d3 = uint32_t(kk[3] - w.k0);
      if (c0 <= 0 && c1 >= 4 && GM != 1 && d0 < w.nk && d1 < w.nk && d2 < w.nk && d3 < w.nk) {
        // four staged operands: the lanes read 512 consecutive bytes per index (no bank conflicts)
        const float4 x0 = w.base[d0 * (G_ROWS / 4)], x1 = w.base[d1 * (G_ROWS / 4)];
        const float4 x2 = w.base[d2 * (G_ROWS / 4)], x3 = w.base[d3 * (G_ROWS / 4)];
        if (GM == 0) {
          const float m = neg0 ? -1.f : 1.f;
          fma4(acc, x0, m);
          fma4(acc, x1, m);
          fma4(acc, x2, m);
          fma4(acc, x3, m);
        } else {  // runs of two from the segment start: the sign of position t is bit 1 of t - s0
          const uint32_t ph = uint32_t(pq - s0);
          fma4(acc, x0, (ph & 2u) ? -1.f : 1.f);
          fma4(acc, x1, ((ph + 1u) & 2u) ? -1.f : 1.f);
          fma4(acc, x2, ((ph + 2u) & 2u) ? -1.f : 1.f);
          fma4(acc, x3, ((ph + 3u) & 2u) ? -1.f : 1.f);
        }
        continue;
      }
      // Mixed group (a window edge, a segment end, an operand outside the window): no branch
      // per component.  The first live component at or beyond k1 stops the group (the column
      // pauses there); every component before it loads through ONE generic pointer -- the
      // staged element or the transposed copy in L2 -- and its four FFMAs are predicated.
      int cstop = c1 < 4 ? c1 : 4;
#pragma unroll
      for (int c = 3; c >= 0; --c)
        if (c >= c0 && c < c1 && kk[c] >= w.k1) cstop = c;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const bool live = c >= c0 && c < cstop;
        const int32_t k = live ? kk[c] : w.k0;  // (dead components read a valid staged element)
        const uint32_t d = uint32_t(k - w.k0);
        const float4* src = d < w.nk ? w.base + d * (G_ROWS / 4)
                                     : reinterpret_cast<const float4*>(glob.xt + int64_t(k) * glob.ld);
        const float4 x = *src;
        if (live) fma4(acc, x, is_neg<GM>(pq + c - s0, g, neg0) ? -1.f : 1.f);
      }
      if (cstop < c1 && cstop < 4) return pq + cstop;  // paused: the next window (or sweep end) resumes here
    }
    i = jend;
  }
  return e;
}

template <int VAR>
__global__ void __launch_bounds__(S_WARPS * 32, 1)
    tg_gather_staged_kernel(const float* __restrict__ Xt, int64_t K, int64_t M, GatherArgs a, int C, int nw_full,
                            int nw_total, int64_t Bk, const float* __restrict__ bias, float* __restrict__ Y,
                            int64_t ldy, int use_alpha, float alpha, tg_device_flags* __restrict__ flags) {
  extern __shared__ __align__(128) float swin[];
  __shared__ uint64_t full[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t N = a.N;
  const int64_t nbase = int64_t(blockIdx.x) * C;
  const float* xt_rg = Xt + int64_t(blockIdx.y) * (K + 1) * G_ROWS;  // this row group's [K+1][128] tile
  const SrcXt glob{xt_rg + lane * 4, G_ROWS};
  const int nsweep = VAR == VAR_BASE ? 2 : int(a.nblocks);

  // window wi of the flattened (sweep, window) sequence -> stage wi & 1 (issued by one thread)
  auto issue = [&](int wi) {
    const int sweep = wi / nw_full, wn = wi - sweep * nw_full;
    const int64_t lo = VAR == VAR_BASE ? 0 : int64_t(sweep) * Bk;
    const int64_t hi = VAR == VAR_BASE ? K : min(K, lo + Bk);
    const int64_t k0 = lo + int64_t(wn) * S_WK;
    const uint32_t nk = uint32_t(min(int64_t(S_WK), hi - k0));
    float* dst = swin + (wi & 1) * S_STAGE_FLOATS;
    const float* src = xt_rg + k0 * G_ROWS;
    mbar_arrive_expect_tx(&full[wi & 1], nk * uint32_t(G_ROWS * sizeof(float)));
    for (uint32_t off = 0; off < nk; off += 32) {  // 16 KB pieces
      const uint32_t n = min(32u, nk - off);
      bulk_load(dst + off * G_ROWS, src + off * G_ROWS, n * uint32_t(G_ROWS * sizeof(float)), &full[wi & 1]);
    }
  };
  if (threadIdx.x == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    issue(0);
    if (nw_total > 1) issue(1);
  }

  int64_t ncol[S_CPW];
  bool valid[S_CPW];
  float bv[S_CPW];
  float4 out[S_CPW], acc[S_CPW];
  int32_t pi[S_CPW], pe[S_CPW], ps0[S_CPW];
#pragma unroll
  for (int j = 0; j < S_CPW; ++j) {
    ncol[j] = nbase + warp + S_WARPS * j;
    valid[j] = warp + S_WARPS * j < C && ncol[j] < N;
    bv[j] = (valid[j] && bias) ? __ldg(bias + ncol[j]) : 0.f;
    out[j] = splat_<float4>(bv[j]);
    acc[j] = zero_<float4>();
    pi[j] = pe[j] = ps0[j] = 0;
  }

  int wi = 0;
  for (int sweep = 0; sweep < nsweep; ++sweep) {
    const int32_t* ai = (VAR == VAR_BASE && sweep == 1) ? a.i1 : a.i0;
#pragma unroll
    for (int j = 0; j < S_CPW; ++j) {
      if (!valid[j]) continue;
      if (VAR == VAR_BASE) {
        const int32_t* cp = sweep ? a.p1 : a.p0;
        pi[j] = __ldg(cp + ncol[j]);
        pe[j] = __ldg(cp + ncol[j] + 1);
      } else {
        const int64_t cell = int64_t(sweep) * N + ncol[j];
        pi[j] = __ldg(a.p0 + 3 * cell);
        pe[j] = __ldg(a.p0 + 3 * cell + 1);
        acc[j] = zero_<float4>();
      }
      ps0[j] = pi[j];
    }
    const int64_t lo = VAR == VAR_BASE ? 0 : int64_t(sweep) * Bk;
    const int64_t hi = VAR == VAR_BASE ? K : min(K, lo + Bk);
    const int nw = sweep == nsweep - 1 ? nw_total - sweep * nw_full : nw_full;
    for (int wn = 0; wn < nw; ++wn, ++wi) {
      mbar_wait(&full[wi & 1], uint32_t(wi >> 1) & 1u);
      Window w;
      w.base = reinterpret_cast<const float4*>(swin + (wi & 1) * S_STAGE_FLOATS) + lane;
      w.k0 = int32_t(lo + int64_t(wn) * S_WK);
      w.nk = uint32_t(min(int64_t(S_WK), hi - w.k0));
      w.k1 = wn == nw - 1 ? INT32_MAX : w.k0 + S_WK;
#pragma unroll
      for (int j = 0; j < S_CPW; ++j) {
        if (pi[j] >= pe[j]) continue;
        if (VAR == VAR_BASE) pi[j] = walk_staged<0>(acc[j], ai, pi[j], pe[j], ps0[j], 1, sweep == 1, w, glob, lane);
        else if (a.g == 2) pi[j] = walk_staged<2>(acc[j], ai, pi[j], pe[j], ps0[j], 2, false, w, glob, lane);
        else pi[j] = walk_staged<1>(acc[j], ai, pi[j], pe[j], ps0[j], a.g, false, w, glob, lane);
      }
      __syncthreads();  // every warp is done with this stage: refill it with the window after next
      if (threadIdx.x == 0 && wi + 2 < nw_total) issue(wi + 2);
    }
    // the rest of the sweep's per-output order (short segments: operands from L2)
#pragma unroll
    for (int j = 0; j < S_CPW; ++j) {
      if (!valid[j]) continue;
      if (VAR == VAR_BASE) {
        if (sweep == 1) out[j] = badd_(bv[j], acc[j]);
      } else {
        const int64_t cell = int64_t(sweep) * N + ncol[j];
        const int32_t s1 = __ldg(a.p0 + 3 * cell + 1), s2 = __ldg(a.p0 + 3 * cell + 2);
        const int32_t s3 = __ldg(a.p0 + 3 * cell + 3);
        if (VAR == VAR_IB) {
          walk<false>(acc[j], a.i0, s1, s2, glob);
          walk<true>(acc[j], a.i0, s2, s3, glob);
          add_(out[j], acc[j]);
        } else {
          add_(out[j], acc[j]);
          walk<false>(out[j], a.i0, s1, s2, glob);
          walk<true>(out[j], a.i0, s2, s3, glob);
        }
      }
    }
  }

  // epilogue: PReLU, flags, row-wise store through shared memory (the window memory is idle now)
  float* stage = swin;
  const int ldst = C + 1;
  bool bad = false;
  unsigned long long npos = 0;
#pragma unroll
  for (int j = 0; j < S_CPW; ++j) {
    if (warp + S_WARPS * j >= C) continue;
    float v[4] = {out[j].x, out[j].y, out[j].z, out[j].w};
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const bool live = valid[j] && int64_t(blockIdx.y) * G_ROWS + lane * 4 + r < M;
      if (use_alpha && !(v[r] > 0.f)) {
        if (live) ++npos;
        v[r] = alpha * v[r];
      }
      if (live) bad |= !isfinite(v[r]);
      stage[(lane * 4 + r) * ldst + warp + S_WARPS * j] = v[r];
    }
  }
  if (flags) {
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&flags->nonfinite_output, 1);
    for (int o = 16; o; o >>= 1) npos += __shfl_xor_sync(0xffffffffu, npos, o);
    if (lane == 0 && npos) atomicAdd(reinterpret_cast<unsigned long long*>(&flags->nonpositive_outputs), npos);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < G_ROWS * C; e += blockDim.x) {
    const int r = e / C, c = e % C;
    const int64_t m = int64_t(blockIdx.y) * G_ROWS + r, nn = nbase + c;
    if (m < M && nn < N) Y[m * ldy + nn] = stage[r * ldst + c];
  }
}

// Columns per CTA: as few waves of CTAs over the SMs as possible, then as few columns
// per CTA (cost ~ waves x columns: a CTA's time is its columns' stream length).
static int staged_columns(int64_t N, int64_t row_groups, int sms) {
  int best = 1;
  int64_t best_cost = INT64_MAX;
  const int cmin = int(std::min<int64_t>(N, 16));
  for (int c = int(std::min<int64_t>(N, S_CMAX)); c >= cmin; --c) {
    const int64_t units = ceil_div(N, c) * row_groups;
    const int64_t cost = ceil_div(units, sms) * c;
    if (cost < best_cost) {
      best_cost = cost;
      best = c;
    }
  }
  return best;
}

static bool staged_enabled() {
  const char* e = std::getenv("TG_GATHER_STAGED");  // 0 forces the L2 walk (A/B runs, tests)
  return !(e && e[0] == '0');
}

template <int VAR>
static int launch_staged(const float* Xt, int64_t M, int64_t M_pad, int64_t K, const GatherArgs& ga, const float* bias,
                         float* Y, int64_t ldy, int use_alpha, float alpha, tg_device_flags* flags, cudaStream_t st) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaFuncSetAttribute(tg_gather_staged_kernel<VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(S_SMEM));  // per device context; cheap next to the walk
  if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(tg_gather_staged_kernel)");
  const int64_t row_groups = M_pad / G_ROWS;
  const int C = staged_columns(ga.N, row_groups, std::max(sms, 1));
  const int nsweep = VAR == VAR_BASE ? 2 : int(ga.nblocks);
  const int64_t Bk = (VAR != VAR_BASE && ga.nblocks > 1 && ga.B > 0) ? ga.B : K;
  const int nw_full = int(ceil_div(std::min(Bk, K), S_WK));
  const int nw_total = VAR == VAR_BASE ? 2 * nw_full
                                       : (nsweep - 1) * nw_full + int(ceil_div(K - int64_t(nsweep - 1) * Bk, S_WK));
  dim3 grid(unsigned(ceil_div(ga.N, C)), unsigned(row_groups));
  tg_gather_staged_kernel<VAR><<<grid, S_WARPS * 32, S_SMEM, st>>>(Xt, K, M, ga, C, nw_full, nw_total, Bk, bias, Y,
                                                                   ldy, use_alpha, alpha, flags);
  return check_launch("tg_gather_staged_kernel");
}

int run_transpose(const float* X, int64_t M, int64_t K, int64_t Kx, int64_t ldx, float* Xt, int64_t M_pad,
                  tg_device_flags* flags, cudaStream_t st) {
  dim3 grid(unsigned(ceil_div(K + 1, 32)), unsigned(ceil_div(M_pad, 32)));
  tg_transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(X, M, K, Kx, ldx, Xt, M_pad, flags);
  return check_launch("tg_transpose_kernel");
}

int run_gather_args(int variant, const float* X, int64_t M, int64_t K, int64_t ldx, const GatherArgs& ga,
                    const float* bias, float* Y, int64_t ldy, int use_alpha, float alpha, void* ws,
                    tg_device_flags* flags, cudaStream_t st) {
  const int64_t M_pad = round_up(M, G_ROWS);
  float* Xt = static_cast<float*>(ws);
  // the PaddedInput variants (simd.py:40-75) read their dummy slot X[:, K] like the reference
  const bool padded = variant == VAR_OPTIMAL || variant == VAR_VERTICAL || variant == VAR_HORIZONTAL;
  int rc = run_transpose(X, M, K, (padded && ldx > K) ? K + 1 : K, ldx, Xt, M_pad, flags, st);
  if (rc != TG_OK) return rc;
  // the BASELINE variants walk shared-memory windows of X; their index arrays are read in
  // aligned groups of four positions
  const bool aligned = (reinterpret_cast<uintptr_t>(ga.i0) & 15u) == 0 &&
                       (variant != VAR_BASE || (reinterpret_cast<uintptr_t>(ga.i1) & 15u) == 0);
  if (aligned && ga.g >= 1 && staged_enabled()) {
    if (variant == VAR_BASE)
      return launch_staged<VAR_BASE>(Xt, M, M_pad, K, ga, bias, Y, ldy, use_alpha, alpha, flags, st);
    if (variant == VAR_IB)
      return launch_staged<VAR_IB>(Xt, M, M_pad, K, ga, bias, Y, ldy, use_alpha, alpha, flags, st);
    if (variant == VAR_OPTIMAL)
      return launch_staged<VAR_OPTIMAL>(Xt, M, M_pad, K, ga, bias, Y, ldy, use_alpha, alpha, flags, st);
  }
  dim3 grid(unsigned(ceil_div(ga.N, G_WARPS)), unsigned(M_pad / G_ROWS));
#define TG_GATHER_LAUNCH(V) \
  tg_gather_kernel<V><<<grid, G_WARPS * 32, 0, st>>>(Xt, K, M, ga, bias, Y, ldy, use_alpha, alpha, flags)
  switch (variant) {
    case VAR_BASE: TG_GATHER_LAUNCH(VAR_BASE); break;
    case VAR_UNROLLED: TG_GATHER_LAUNCH(VAR_UNROLLED); break;
    case VAR_BLOCKED: TG_GATHER_LAUNCH(VAR_BLOCKED); break;
    case VAR_IB: TG_GATHER_LAUNCH(VAR_IB); break;
    case VAR_VERTICAL: TG_GATHER_LAUNCH(VAR_VERTICAL); break;
    case VAR_HORIZONTAL: TG_GATHER_LAUNCH(VAR_HORIZONTAL); break;
    case VAR_COMPRESSED: TG_GATHER_LAUNCH(VAR_COMPRESSED); break;
    default: TG_GATHER_LAUNCH(VAR_OPTIMAL); break;
  }
#undef TG_GATHER_LAUNCH
  return check_launch("tg_gather_kernel");
}

int run_gather(int variant, const float* X, int64_t M, int64_t K, int64_t ldx, const int32_t* p0, const int32_t* i0,
               const int32_t* p1, const int32_t* i1, int64_t nblocks, int g, int uf, int64_t m_full, int64_t N,
               const float* bias, float* Y, int64_t ldy, int use_alpha, float alpha, void* ws,
               tg_device_flags* flags, cudaStream_t st, int64_t B) {
  GatherArgs ga{p0, i0, p1, i1, N, nblocks, m_full, g, uf, nullptr, 0, B};
  return run_gather_args(variant, X, M, K, ldx, ga, bias, Y, ldy, use_alpha, alpha, ws, flags, st);
}

}  // namespace tg
