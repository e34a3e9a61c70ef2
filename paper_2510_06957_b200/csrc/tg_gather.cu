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
// Layout: X is first transposed into Xt[K+1][M_pad] (row K = 0, the dummy slot
// of PaddedInput, simd.py:40-75), so one warp-wide float4 load fetches X[m, k]
// for 128 consecutive rows m: lanes = rows, one warp = one column n, the index
// stream is read warp-uniformly (broadcast) from L1/L2.  Outputs are staged in
// shared memory and written row-wise.
#include <cuda_runtime.h>
#include <cstdint>

#include "tg_internal.h"

namespace tg {

enum { VAR_BASE = 0, VAR_BLOCKED = 1, VAR_IB = 2, VAR_OPTIMAL = 3, VAR_UNROLLED = 4 };

constexpr int G_WARPS = 8;    // columns per CTA
constexpr int G_ROWS = 128;   // rows per CTA (4 per lane)

size_t gather_ws_bytes(int64_t M, int64_t K) {
  return size_t(K + 1) * size_t(round_up(M, G_ROWS)) * sizeof(float) + 256;
}

// X (M x ldx) -> Xt ((K+1) x M_pad), zero padded.
__global__ void tg_transpose_kernel(const float* __restrict__ X, int64_t M, int64_t K, int64_t ldx,
                                    float* __restrict__ Xt, int64_t M_pad, tg_device_flags* flags) {
  __shared__ float tile[32][33];
  const int64_t k0 = int64_t(blockIdx.x) * 32, m0 = int64_t(blockIdx.y) * 32;
  bool bad = false;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t m = m0 + r, k = k0 + threadIdx.x;
    float v = 0.f;
    if (m < M && k < K) {
      v = X[m * ldx + k];
      bad |= !isfinite(v);
    }
    tile[r][threadIdx.x] = v;
  }
  if (flags && bad) atomicOr(&flags->bad_input, 4);
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t k = k0 + r, m = m0 + threadIdx.x;
    if (k <= K && m < M_pad) Xt[k * M_pad + m] = tile[threadIdx.x][r];
  }
}

__device__ __forceinline__ float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void add_(float4& a, const float4 b) {
  a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
}
__device__ __forceinline__ void sub_(float4& a, const float4 b) {
  a.x -= b.x; a.y -= b.y; a.z -= b.z; a.w -= b.w;
}
__device__ __forceinline__ void add_(float& a, const float b) { a += b; }
__device__ __forceinline__ void sub_(float& a, const float b) { a -= b; }
template <typename V> __device__ __forceinline__ V zero_();
template <> __device__ __forceinline__ float zero_<float>() { return 0.f; }
template <> __device__ __forceinline__ float4 zero_<float4>() { return make_float4(0.f, 0.f, 0.f, 0.f); }
template <typename V> __device__ __forceinline__ V splat_(float b);
template <> __device__ __forceinline__ float splat_<float>(float b) { return b; }
template <> __device__ __forceinline__ float4 splat_<float4>(float b) { return make_float4(b, b, b, b); }
// b + acc (scalar.py:127 `bias[n] + acc`), component-wise
__device__ __forceinline__ float badd_(float b, float a) { return b + a; }
__device__ __forceinline__ float4 badd_(float b, float4 a) { return make_float4(b + a.x, b + a.y, b + a.z, b + a.w); }

// Operand sources: the value X[., k] for a stream index k.
struct SrcXt {  // 4 consecutive rows from the transposed copy Xt[K+1][M_pad]
  using V = float4;
  const float* xt;
  int64_t ld;
  __device__ __forceinline__ float4 operator()(int32_t k) const { return ld4(xt + int64_t(k) * ld); }
};
struct SrcRow {  // one row of X in place (ldx = K or K+1)
  using V = float;
  const float* x;
  __device__ __forceinline__ float operator()(int32_t k) const { return __ldg(x + k); }
};

// Walk [a, b) of an index stream adding (NEG=false) or subtracting into acc,
// strictly in stream order.
template <bool NEG, typename S>
__device__ __forceinline__ void walk(typename S::V& acc, const int32_t* __restrict__ idx, int32_t a, int32_t b,
                                     const S& src) {
  int32_t i = a;
  for (; i + 4 <= b; i += 4) {
    const int32_t k0 = __ldg(idx + i), k1 = __ldg(idx + i + 1), k2 = __ldg(idx + i + 2), k3 = __ldg(idx + i + 3);
    const typename S::V v0 = src(k0), v1 = src(k1), v2 = src(k2), v3 = src(k3);
    if (NEG) { sub_(acc, v0); sub_(acc, v1); sub_(acc, v2); sub_(acc, v3); }
    else { add_(acc, v0); add_(acc, v1); add_(acc, v2); add_(acc, v3); }
  }
  for (; i < b; ++i) {
    const typename S::V v = src(__ldg(idx + i));
    if (NEG) sub_(acc, v); else add_(acc, v);
  }
}

// Interleaved segment [s0, s1): alternating runs of g, positives first.
template <typename S>
__device__ __forceinline__ void walk_interleaved(typename S::V& acc, const int32_t* __restrict__ ai, int32_t s0,
                                                 int32_t s1, int g, const S& src) {
  for (int32_t i = s0; i < s1; i += 2 * g) {
    walk<false>(acc, ai, i, min(i + g, s1), src);
    walk<true>(acc, ai, min(i + g, s1), min(i + 2 * g, s1), src);
  }
}

// Banked sum of one (pos, neg) cell, kernels/scalar.py:167-206: every bank is an
// independent sequential accumulation, so the banks are evaluated one after the
// other and folded into tot in bank order -- two live accumulators for any uf.
template <typename S>
__device__ __forceinline__ typename S::V banked_sum(const int32_t* __restrict__ rp, int32_t ap, int32_t bp,
                                                    const int32_t* __restrict__ rn, int32_t an, int32_t bn, int uf,
                                                    const S& src) {
  using V = typename S::V;
  V tot = zero_<V>();
  const int32_t fp = ap + (bp - ap) / uf * uf, fn = an + (bn - an) / uf * uf;
  for (int u = 0; u < uf; ++u) {
    V bank = zero_<V>();
    for (int32_t i = ap + u; i < fp; i += uf) add_(bank, src(__ldg(rp + i)));
    if (u == 0) walk<false>(bank, rp, fp, bp, src);
    for (int32_t i = an + u; i < fn; i += uf) sub_(bank, src(__ldg(rn + i)));
    if (u == 0) walk<true>(bank, rn, fn, bn, src);
    add_(tot, bank);
  }
  return tot;
}

struct GatherArgs {
  const int32_t* p0;  // col_start_pos (TCSC / blocked) or col_segment_ptr (interleaved)
  const int32_t* i0;  // row_index_pos or all_indices
  const int32_t* p1;  // col_start_neg
  const int32_t* i1;  // row_index_neg
  int64_t N, nblocks, m_full;
  int g, uf;
};

// Y[m, n] before the activation, in the reference's operation order for VAR.
// `banked_rows` (blocked only): bit r set if component r belongs to a row < m_full.
template <int VAR, typename S>
__device__ __forceinline__ typename S::V column_value(const GatherArgs& a, int64_t n, float b, const S& src,
                                                      unsigned banked_rows) {
  using V = typename S::V;
  if (VAR == VAR_BASE) {
    V acc = zero_<V>();
    walk<false>(acc, a.i0, __ldg(a.p0 + n), __ldg(a.p0 + n + 1), src);
    walk<true>(acc, a.i1, __ldg(a.p1 + n), __ldg(a.p1 + n + 1), src);
    return badd_(b, acc);
  } else if (VAR == VAR_UNROLLED) {
    const V tot = banked_sum(a.i0, __ldg(a.p0 + n), __ldg(a.p0 + n + 1), a.i1, __ldg(a.p1 + n), __ldg(a.p1 + n + 1),
                             a.uf, src);
    return badd_(b, tot);
  } else if (VAR == VAR_BLOCKED) {
    V out = splat_<V>(b);
    for (int64_t blk = 0; blk < a.nblocks; ++blk) {
      const int32_t* cp = a.p0 + blk * (a.N + 1);
      const int32_t* cn = a.p1 + blk * (a.N + 1);
      const int32_t ap = __ldg(cp + n), bp = __ldg(cp + n + 1), an = __ldg(cn + n), bn = __ldg(cn + n + 1);
      V tot = zero_<V>(), acc = zero_<V>();
      if (banked_rows) tot = banked_sum(a.i0, ap, bp, a.i1, an, bn, a.uf, src);
      if (banked_rows != (sizeof(V) == 4 ? 1u : 15u)) {
        walk<false>(acc, a.i0, ap, bp, src);
        walk<true>(acc, a.i1, an, bn, src);
      }
      if constexpr (sizeof(V) == 4) {
        out += (banked_rows & 1u) ? tot : acc;
      } else {
        out.x += (banked_rows & 1u) ? tot.x : acc.x;
        out.y += (banked_rows & 2u) ? tot.y : acc.y;
        out.z += (banked_rows & 4u) ? tot.z : acc.z;
        out.w += (banked_rows & 8u) ? tot.w : acc.w;
      }
    }
    return out;
  } else {
    V out = splat_<V>(b);
    for (int64_t blk = 0; blk < a.nblocks; ++blk) {
      const int64_t cell = blk * a.N + n;
      const int32_t s0 = __ldg(a.p0 + 3 * cell), s1 = __ldg(a.p0 + 3 * cell + 1);
      const int32_t s2 = __ldg(a.p0 + 3 * cell + 2), s3 = __ldg(a.p0 + 3 * cell + 3);
      V acc = zero_<V>();
      walk_interleaved(acc, a.i0, s0, s1, a.g, src);
      if (VAR == VAR_IB) {
        walk<false>(acc, a.i0, s1, s2, src);
        walk<true>(acc, a.i0, s2, s3, src);
        add_(out, acc);
      } else {
        add_(out, acc);
        walk<false>(out, a.i0, s1, s2, src);
        walk<true>(out, a.i0, s2, s3, src);
      }
    }
    return out;
  }
}

template <int VAR>
__global__ void __launch_bounds__(G_WARPS * 32)
    tg_gather_kernel(const float* __restrict__ Xt, int64_t M_pad, int64_t M, GatherArgs a,
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
    out = column_value<VAR>(a, n, b, SrcXt{Xt + mrow, M_pad}, banked);
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

// Recompute the rows listed by the X split (rows whose dynamic range is too wide
// for the 22-bit fixed-point limbs) with the exact-order walk, one thread per
// (listed row, column).  rows[0] = count, rows[1..] = row ids.  The MMA epilogue
// skipped the PReLU count for these rows; it is taken here.
template <int VAR>
__global__ void __launch_bounds__(256)
    tg_fixup_kernel(const float* __restrict__ X, int64_t ldx, int64_t M, const int32_t* __restrict__ rows,
                    GatherArgs a, const float* __restrict__ bias, float* __restrict__ Y, int64_t ldy, int use_alpha,
                    float alpha, tg_device_flags* __restrict__ flags) {
  const int32_t count = __ldg(rows);
  const int64_t n = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int32_t i = blockIdx.y; i < count; i += gridDim.y) {
    const int64_t m = __ldg(rows + 1 + i);
    if (n >= a.N || m >= M) continue;
    const float b = bias ? __ldg(bias + n) : 0.f;
    float y = column_value<VAR>(a, n, b, SrcRow{X + m * ldx}, m < a.m_full ? 1u : 0u);
    if (use_alpha && !(y > 0.f)) {
      if (flags) atomicAdd(reinterpret_cast<unsigned long long*>(&flags->nonpositive_outputs), 1ull);
      y = alpha * y;
    }
    Y[m * ldy + n] = y;
    if (flags && !isfinite(y)) atomicOr(&flags->nonfinite_output, 1);
  }
}

int run_transpose(const float* X, int64_t M, int64_t K, int64_t ldx, float* Xt, int64_t M_pad,
                  tg_device_flags* flags, cudaStream_t st) {
  dim3 grid(unsigned(ceil_div(K + 1, 32)), unsigned(ceil_div(M_pad, 32)));
  tg_transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(X, M, K, ldx, Xt, M_pad, flags);
  return check_launch("tg_transpose_kernel");
}

int run_gather(int variant, const float* X, int64_t M, int64_t K, int64_t ldx, const int32_t* p0, const int32_t* i0,
               const int32_t* p1, const int32_t* i1, int64_t nblocks, int g, int uf, int64_t m_full, int64_t N,
               const float* bias, float* Y, int64_t ldy, int use_alpha, float alpha, void* ws,
               tg_device_flags* flags, cudaStream_t st) {
  const int64_t M_pad = round_up(M, G_ROWS);
  float* Xt = static_cast<float*>(ws);
  int rc = run_transpose(X, M, K, ldx, Xt, M_pad, flags, st);
  if (rc != TG_OK) return rc;
  dim3 grid(unsigned(ceil_div(N, G_WARPS)), unsigned(M_pad / G_ROWS));
  GatherArgs ga{p0, i0, p1, i1, N, nblocks, m_full, g, uf};
#define TG_GATHER_LAUNCH(V) \
  tg_gather_kernel<V><<<grid, G_WARPS * 32, 0, st>>>(Xt, M_pad, M, ga, bias, Y, ldy, use_alpha, alpha, flags)
  switch (variant) {
    case VAR_BASE: TG_GATHER_LAUNCH(VAR_BASE); break;
    case VAR_UNROLLED: TG_GATHER_LAUNCH(VAR_UNROLLED); break;
    case VAR_BLOCKED: TG_GATHER_LAUNCH(VAR_BLOCKED); break;
    case VAR_IB: TG_GATHER_LAUNCH(VAR_IB); break;
    default: TG_GATHER_LAUNCH(VAR_OPTIMAL); break;
  }
#undef TG_GATHER_LAUNCH
  return check_launch("tg_gather_kernel");
}

}  // namespace tg

namespace tg {

int run_fixup(int variant, const float* X, int64_t M, int64_t ldx, const int32_t* rows, const int32_t* p0,
              const int32_t* i0, const int32_t* p1, const int32_t* i1, int64_t nblocks, int g, int uf, int64_t m_full,
              int64_t N, const float* bias, float* Y, int64_t ldy, int use_alpha, float alpha, tg_device_flags* flags,
              cudaStream_t st) {
  GatherArgs ga{p0, i0, p1, i1, N, nblocks, m_full, g, uf};
  dim3 grid(unsigned(ceil_div(N, 256)), unsigned(std::min<int64_t>(M, 32)));
#define TG_FIXUP_LAUNCH(V) \
  tg_fixup_kernel<V><<<grid, 256, 0, st>>>(X, ldx, M, rows, ga, bias, Y, ldy, use_alpha, alpha, flags)
  switch (variant) {
    case VAR_BASE: TG_FIXUP_LAUNCH(VAR_BASE); break;
    case VAR_UNROLLED: TG_FIXUP_LAUNCH(VAR_UNROLLED); break;
    case VAR_BLOCKED: TG_FIXUP_LAUNCH(VAR_BLOCKED); break;
    case VAR_IB: TG_FIXUP_LAUNCH(VAR_IB); break;
    default: TG_FIXUP_LAUNCH(VAR_OPTIMAL); break;
  }
#undef TG_FIXUP_LAUNCH
  return check_launch("tg_fixup_kernel");
}

}  // namespace tg
