// tg_mma.cu — dense-decode tensor-core path for Y = X W + b (+PReLU).
//
// Semantics: same result contract as the reference kernels
//   gemm_base                /root/reference/pkg/src/terngemm/kernels/scalar.py:109-148
//   gemm_vectorized_optimal  /root/reference/pkg/src/terngemm/kernels/simd.py:282-449
// i.e. Y[m,n] = b[n] + sum_{k: W[k,n]=+1} X[m,k] - sum_{k: W[k,n]=-1} X[m,k],
// then y <- (y > 0 ? y : alpha*y) in fp32 when PReLU is on (simd.py:410-417).
//
// Realisation (B200-native):
//   1. tg_xsplit_*_kernel: each X row is scaled by a power of two 2^s so that
//      max|x| < 2^22, rounded to an integer v, and v is split into three
//      balanced signed base-256 digits (int8 "limbs").  Exact for integer X.
//      Rows whose nonzeros span a wide dynamic range are marked "wide".
//   2. tg_mma_kernel: persistent, warp-specialised, one CTA per SM.  A work
//      unit is (128 output columns) x (MT output rows) x (a K range):
//        warp 0     TMA: the three limb tiles of X (SWIZZLE_128B), multicast
//                   across a cluster of 1/2/4 CTAs sharing the rows
//        warp 6     bulk copies of the packed 2-bit ternary W tiles (own ring)
//        warps 2-5  decode the packed tile into int8 {-1,0,+1} W^T rows and
//                   write them straight into TMEM (tcgen05.st)
//        warp 1     one lane issues tcgen05.mma.kind::i8, A = W^T from TMEM,
//                   B = [limb0; limb1; limb2] from smem (N = 3*MT), into one of
//                   two int32 TMEM accumulators (the epilogue of a unit
//                   overlaps the MMAs of the next).  Integer accumulation is
//                   exact and order-independent, so K may be split across CTAs.
//        warps 7-14 epilogue: tcgen05.ld the three limb sums, recombine them with
//                   three fp32 FMAs (exact for integer X), add the bias, PReLU,
//                   st.shared into the Y tile, one TMA store per unit.  Split-K
//                   units write per-limb int32 partials; the last unit of a tile
//                   sums them and takes the same epilogue.  Rows marked "wide"
//                   are then recomputed in the reference's exact operation
//                   order (tg_walk.cuh).
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "tg_ptx.cuh"
#include "tg_internal.h"
#include "tg_walk.cuh"

namespace tg {

// ------------------------------------------------------------------ trace (debug builds only)
#ifdef TG_TRACE
// [cta slot][event][iteration]: clock64 stamps of CTA 0 and CTA 1, first 512 pipeline iterations
__device__ unsigned long long g_tg_trace[2][8][512];
#define TG_STAMP(ev, it)                                                           \
  do {                                                                             \
    if (blockIdx.x < 2 && (it) < 512) g_tg_trace[blockIdx.x][ev][it] = clock64(); \
  } while (0)
// global-time (ns) milestones of the whole step: [ev][0] = min over CTAs, [ev][1] = max
__device__ unsigned long long g_tg_gt[16][2];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TG_GT(ev)                                           \
  do {                                                      \
    const unsigned long long _t = gtime();                  \
    atomicMin(&g_tg_gt[ev][0], _t);                         \
    atomicMax(&g_tg_gt[ev][1], _t);                         \
  } while (0)
#else
#define TG_STAMP(ev, it) \
  do {                   \
  } while (0)
#define TG_GT(ev) \
  do {            \
  } while (0)
#endif

// ------------------------------------------------------------------ X split
// One CTA per (padded) row.  limbs: [3][M_pad][K_pad] int8, rscale: [M_pad] f64.
//
// Row m is scaled by 2^s, s = 22 - e with amax < 2^e, so |x 2^s| < 2^22; the
// rounded integer v splits into balanced base-256 digits v = d0 2^16 + d1 2^8 + d2.
// The grid step 2^(e-22) is relative to the row maximum, so a row whose nonzero
// entries span a wide dynamic range gets its rscale stored negated: the MMA
// epilogue then recomputes the row in the exact reference order (and takes its
// PReLU count there).  Wide means amax > kWideRatio * rms of its nonzeros, or
// fewer than 1/kWideFrac of its nonzeros within kWideRatio of amax.  The second
// rule catches a few outliers in a short row (one entry 5000x the rest in K = 128
// passes the rms test, yet leaves the other entries 9 bits on the grid: an output
// that does not see the outlier then misses the 1e-5 bar; tests/test_gpu_fuzz.py).
constexpr float kWideRatio = 16.f;
constexpr int kWideFrac = 4;
// The epilogue applies 2^-s and 2^(24-s) as normal floats: |s| <= 100 keeps both
// (and every partial product) far inside the fp32 range.  Rows outside take the
// exact-order path.
constexpr int kMaxScaleExp = 100;
// Split-K arrival counters (one per (row block, column block) tile) live right after
// the row scales.  The X split zeroes them, so the tile GEMM needs no memset node
// between the two kernels (that node costs ~6 us and the programmatic overlap);
// the last-arriving unit of a tile resets its counter for replays.  Split-K is only
// used while the tiles fit (split_layout).
constexpr int kSplitCounters = 4096;
__device__ __forceinline__ void zero_split_counters(double* rscale, int64_t M_pad) {
  int32_t* c = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(rscale) + ((M_pad * 8 + 255) / 256) * 256);
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < kSplitCounters) c[i] = 0;
}
// Outlier entries of a row (LLM-style activations: a few channels tens to hundreds of times
// the rest).  A row whose amax is more than kWideRatio x the rms of its nonzeros would leave
// the bulk of its entries only a few bits on the 22-bit grid.  Instead of sending the whole
// row down the exact-order walk, the X split takes the few large entries out of the limbs:
// entries beyond kOutlierCut x the scale of the rest (its rms, or 1.25 x its mean |x| when
// that is smaller) are listed as (k, x) pairs (at most kOutlierCap per row, in ascending k),
// the limbs carry the rest at the rest's own scale, and the GEMM epilogue adds sum_k (+-x) of
// the listed entries, W[k, n] read from the row-major 2-bit plane behind the tiles (exact fp32
// adds, a fixed order).  Rows that stay wide after kOutlierRounds rounds keep the exact walk.
constexpr int kOutlierCap = 128;  // (1 KB of list per row)
constexpr float kOutlierCut = 8.f;
constexpr int kOutlierRounds = 4;
// Tail of the prepare workspace, relative to the row scales: split-K counters, the per-row
// outlier counts, the outlier lists.
struct PrepTail {
  int64_t counters, ocount, olist, end;
};
__host__ __device__ inline PrepTail prep_tail(int64_t M_pad) {
  PrepTail t;
  t.counters = ((M_pad * 8 + 255) / 256) * 256;
  t.ocount = t.counters + int64_t(kSplitCounters) * 4;
  t.olist = t.ocount + ((M_pad * 4 + 255) / 256) * 256;
  t.end = t.olist + M_pad * int64_t(kOutlierCap) * 8;
  return t;
}
__device__ __forceinline__ int32_t* outlier_counts(double* rscale, int64_t M_pad) {
  return reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(rscale) + prep_tail(M_pad).ocount);
}
__device__ __forceinline__ int2* outlier_list(double* rscale, int64_t M_pad) {
  return reinterpret_cast<int2*>(reinterpret_cast<uint8_t*>(rscale) + prep_tail(M_pad).olist);
}
constexpr int64_t XS_SMEM_MAX_K = 16384;  // rows up to 64 KB are staged in shared memory

// max that propagates NaN (fmaxf drops it), so a NaN anywhere in a row makes
// its amax non-finite and the row is reported like an inf (dense.py:77).
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

template <int XS_THREADS>
__device__ __forceinline__ float block_max(float v, float* red) {
  for (int o = 16; o; o >>= 1) v = fmax_nan(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  v = red[0];
#pragma unroll
  for (int i = 1; i < XS_THREADS / 32; ++i) v = fmax_nan(v, red[i]);
  return v;
}
template <int XS_THREADS>
__device__ __forceinline__ float block_sum(float v, float* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  v = 0.f;
#pragma unroll
  for (int i = 0; i < XS_THREADS / 32; ++i) v += red[i];
  return v;
}

__device__ __forceinline__ uint32_t limb_digits(int v, uint32_t& p1, uint32_t& p2, int j) {
  const int d2 = ((v + 128) & 255) - 128;
  const int v1 = (v - d2) >> 8;
  const int d1 = ((v1 + 128) & 255) - 128;
  const int d0 = (v1 - d1) >> 8;
  p1 |= (uint32_t(d1) & 255u) << (8 * j);
  p2 |= (uint32_t(d2) & 255u) << (8 * j);
  return (uint32_t(d0) & 255u) << (8 * j);
}

// SMEM: the row is loaded once into dynamic shared memory (K_pad floats);
// otherwise every pass re-reads it from global memory (L2-resident).
template <bool SMEM, int XS_THREADS>
__global__ void __launch_bounds__(XS_THREADS) tg_xsplit_kernel(const float* __restrict__ X, int64_t M, int64_t K,
                                                               int64_t ldx, int8_t* __restrict__ limbs,
                                                               double* __restrict__ rscale,
                                                               int64_t M_pad,
                                                               int64_t K_pad, tg_device_flags* __restrict__ flags) {
  extern __shared__ float srow[];
  __shared__ float red[XS_THREADS / 32];
  grid_dep_launch();  // the MMA kernel may start its prologue (it waits before reading our output)
  zero_split_counters(rscale, M_pad);
  const int64_t m = blockIdx.x;
  const float* grow = X + m * ldx;
  const bool in = m < M;
  // pass 1: stage the row, amax
  float amax = 0.f;
  if (in) {
    if (SMEM) {
      const bool vec = ((ldx & 3) == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
      if (vec) {
        const int64_t K4 = K >> 2;
        for (int64_t i = threadIdx.x; i < K4; i += XS_THREADS) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(grow) + i);
          reinterpret_cast<float4*>(srow)[i] = v;
          amax = fmax_nan(amax, fmax_nan(fmax_nan(fabsf(v.x), fabsf(v.y)), fmax_nan(fabsf(v.z), fabsf(v.w))));
        }
        for (int64_t k = (K4 << 2) + threadIdx.x; k < K; k += XS_THREADS) {
          const float v = __ldg(grow + k);
          srow[k] = v;
          amax = fmax_nan(amax, fabsf(v));
        }
      } else {
        for (int64_t k = threadIdx.x; k < K; k += XS_THREADS) {
          const float v = __ldg(grow + k);
          srow[k] = v;
          amax = fmax_nan(amax, fabsf(v));
        }
      }
    } else {
      for (int64_t k = threadIdx.x; k < K; k += XS_THREADS) amax = fmax_nan(amax, fabsf(__ldg(grow + k)));
    }
  }
  amax = block_max<XS_THREADS>(amax, red);  // (also orders the smem stores before pass 2)
  const bool finite = amax <= 3.402823466e38f;  // false for inf / nan
  const bool live = in && amax > 0.f && finite;
  int s = 0;
  if (live) {
    int e;
    frexpf(amax, &e);  // amax < 2^e
    s = 22 - e;        // |x * 2^s| < 2^22
  } else if (in && !finite && threadIdx.x == 0 && flags) {
    atomicOr(&flags->bad_input, 4);
  }
  // pass 2: limbs (16 consecutive k per thread-iteration) + dynamic range statistics.
  // x * 2^s as two exact power-of-two multiplies (2^s alone may exceed the float range).
  const int s_a = s > 126 ? 126 : (s < -126 ? -126 : s);
  const float sc_a = __int_as_float((127 + s_a) << 23), sc_b = __int_as_float((127 + s - s_a) << 23);
  const float inv = live ? 1.f / amax : 0.f;
  float s2 = 0.f, nzf = 0.f, bigf = 0.f;
  int8_t* l0 = limbs + m * K_pad;
  int8_t* l1 = limbs + (M_pad + m) * K_pad;
  int8_t* l2 = limbs + (2 * M_pad + m) * K_pad;
  constexpr int WORDS = XS_THREADS >= 1024 ? 1 : 4;  // 4-byte words of each limb per thread-iteration
  constexpr int VEC = 4 * WORDS;
  for (int64_t k0 = int64_t(threadIdx.x) * VEC; k0 < K_pad; k0 += int64_t(XS_THREADS) * VEC) {
    uint32_t q0[WORDS], q1[WORDS], q2[WORDS];
#pragma unroll
    for (int w = 0; w < WORDS; ++w) {
      uint32_t p0 = 0, p1 = 0, p2 = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t k = k0 + 4 * w + j;
        int v = 0;
        if (live && k < K) {
          const float x = SMEM ? srow[k] : __ldg(grow + k);
          v = __float2int_rn((x * sc_a) * sc_b);
          const float t = x * inv;
          s2 += t * t;
          nzf += (x != 0.f) ? 1.f : 0.f;
          bigf += (fabsf(t) * kWideRatio >= 1.f) ? 1.f : 0.f;
        }
        p0 |= limb_digits(v, p1, p2, j);
      }
      q0[w] = p0;
      q1[w] = p1;
      q2[w] = p2;
    }
    if constexpr (WORDS == 4) {
      *reinterpret_cast<uint4*>(l0 + k0) = make_uint4(q0[0], q0[1], q0[2], q0[3]);
      *reinterpret_cast<uint4*>(l1 + k0) = make_uint4(q1[0], q1[1], q1[2], q1[3]);
      *reinterpret_cast<uint4*>(l2 + k0) = make_uint4(q2[0], q2[1], q2[2], q2[3]);
    } else {
      *reinterpret_cast<uint32_t*>(l0 + k0) = q0[0];
      *reinterpret_cast<uint32_t*>(l1 + k0) = q1[0];
      *reinterpret_cast<uint32_t*>(l2 + k0) = q2[0];
    }
  }
  s2 = block_sum<XS_THREADS>(s2, red);
  nzf = block_sum<XS_THREADS>(nzf, red);
  bigf = block_sum<XS_THREADS>(bigf, red);
  if (threadIdx.x == 0) {
    // amax / rms(nonzeros) > kWideRatio, few entries near amax, or a scale outside the
    // epilogue's fp32 range
    const bool is_wide = live && (nzf > kWideRatio * kWideRatio * s2 || bigf * kWideFrac < nzf ||
                                  s > kMaxScaleExp || s < -kMaxScaleExp);
    const double sc = live ? ldexp(1.0, -s) : 0.0;
    rscale[m] = is_wide ? -sc : sc;
    outlier_counts(rscale, M_pad)[m] = 0;  // (long rows: no outlier extraction, wide rows take the exact walk)
  }
}

// Register-resident variant: thread t owns EPT consecutive k of the row, so the
// row is read once, reduced once (amax, sum x^2 in fp64, nonzero count) and
// converted from registers.  Digits: with |v| < 2^22, u = v + 0x808080 lies in
// [0, 2^24) and byte i of u, minus 128, is the i-th balanced base-256 digit of v
// (the same digits as limb_digits); as int8 that is byte ^ 0x80.
// CTAs per SM the register allocation must allow (the row lives in EPT registers): the split
// is a streaming kernel and wants bytes in flight.  Three 256-thread CTAs of the 32-per-thread
// variant per SM (80 registers, 4 bytes of spills) instead of two (98): cfg5's split 0.139 ->
// 0.120 ms.
constexpr int xs_min_blocks(int threads, int ept) {
  if (threads >= 512) return ept <= 16 ? 2 : 1;  // (two wide CTAs per SM, as the few-row launch plan assumes)
  const int b = 65536 / (threads * (20 + 2 * ept));
  return b < 1 ? 1 : (b > 4 ? 4 : b);
}
template <int THREADS, int EPT>
__global__ void __launch_bounds__(THREADS, xs_min_blocks(THREADS, EPT)) tg_xsplit_reg_kernel(const float* __restrict__ X, int64_t M, int64_t K,
                                                                int64_t ldx, int8_t* __restrict__ limbs,
                                                                double* __restrict__ rscale, int64_t M_pad,
                                                                int64_t K_pad, tg_device_flags* __restrict__ flags) {
  static_assert(EPT % 4 == 0, "EPT");
  constexpr int NW = THREADS / 32;
  __shared__ float red_f[NW];
  __shared__ double red_d[NW];
  __shared__ int red_i[NW];
  __shared__ int red_j[NW];
  __shared__ float red_g[NW];
  __shared__ int red_k[NW];
  grid_dep_launch();  // the MMA kernel may start its prologue (it waits before reading our output)
  zero_split_counters(rscale, M_pad);
  if (threadIdx.x == 0) TG_GT(0);
  const int64_t m = blockIdx.x;
  const float* grow = X + m * ldx;
  const int64_t k0 = int64_t(threadIdx.x) * EPT;
  float x[EPT];
  const bool in = m < M;
  if (in && k0 + EPT <= K && ((reinterpret_cast<uintptr_t>(grow + k0) & 15) == 0)) {
#pragma unroll
    for (int j = 0; j < EPT; j += 4) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(grow + k0 + j));
      x[j] = v.x; x[j + 1] = v.y; x[j + 2] = v.z; x[j + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < EPT; ++j) x[j] = (in && k0 + j < K) ? __ldg(grow + k0 + j) : 0.f;
  }
  const int w = threadIdx.x >> 5;
  // block-wide (max, sum, sum, sum, sum, sum) of (float, float, double, int, int, int); every thread
  // gets the result; red_j keeps the per-warp partials of j2 until the next call
  auto reduce6 = [&](float& a, float& g, double& d, int& i, int& j2, int& k3) {
    for (int o = 16; o; o >>= 1) {
      a = fmax_nan(a, __shfl_xor_sync(0xffffffffu, a, o));
      g += __shfl_xor_sync(0xffffffffu, g, o);
      d += __shfl_xor_sync(0xffffffffu, d, o);
      i += __shfl_xor_sync(0xffffffffu, i, o);
      j2 += __shfl_xor_sync(0xffffffffu, j2, o);
      k3 += __shfl_xor_sync(0xffffffffu, k3, o);
    }
    __syncthreads();  // (the previous round's readers are done with the arrays)
    if ((threadIdx.x & 31) == 0) {
      red_f[w] = a;
      red_g[w] = g;
      red_d[w] = d;
      red_i[w] = i;
      red_j[w] = j2;
      red_k[w] = k3;
    }
    __syncthreads();
    a = red_f[0];
    g = red_g[0];
    d = red_d[0];
    i = red_i[0];
    j2 = red_j[0];
    k3 = red_k[0];
#pragma unroll
    for (int q = 1; q < NW; ++q) {
      a = fmax_nan(a, red_f[q]);
      g += red_g[q];
      d += red_d[q];
      i += red_i[q];
      j2 += red_j[q];
      k3 += red_k[q];
    }
  };
  float amax = 0.f, s1 = 0.f;  // (s1 = sum |x| may overflow to inf for huge rows: the cut then falls back to the rms)
  double s2 = 0.0;
  int nz = 0;
#pragma unroll
  for (int j = 0; j < EPT; ++j) {
    amax = fmax_nan(amax, fabsf(x[j]));
    s1 += fabsf(x[j]);
    s2 = fma(double(x[j]), double(x[j]), s2);
    nz += x[j] != 0.f;
  }
  for (int o = 16; o; o >>= 1) {
    amax = fmax_nan(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    nz += __shfl_xor_sync(0xffffffffu, nz, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red_f[w] = amax;
    red_g[w] = s1;
    red_d[w] = s2;
    red_i[w] = nz;
  }
  __syncthreads();
  amax = red_f[0];
  s1 = red_g[0];
  s2 = red_d[0];
  nz = red_i[0];
#pragma unroll
  for (int i = 1; i < NW; ++i) {
    amax = fmax_nan(amax, red_f[i]);
    s1 += red_g[i];
    s2 += red_d[i];
    nz += red_i[i];
  }
  const bool finite = amax <= 3.402823466e38f;  // false for inf / nan
  const bool live = in && amax > 0.f && finite;
  if (in && !finite && threadIdx.x == 0 && flags) atomicOr(&flags->bad_input, 4);

  // block-wide sum of an int; every thread gets the result
  auto reduce_int = [&](int v) {
    v = __reduce_add_sync(0xffffffffu, v);
    __syncthreads();  // (the previous round's readers are done with the array)
    if ((threadIdx.x & 31) == 0) red_i[w] = v;
    __syncthreads();
    v = red_i[0];
#pragma unroll
    for (int q = 1; q < NW; ++q) v += red_i[q];
    return v;
  };
  // The two "wide" rules: amax / rms(nonzeros) > kWideRatio (nz amax^2 > kWideRatio^2 sum x^2),
  // or fewer than 1 / kWideFrac of the nonzeros within kWideRatio of amax.
  const double wide2 = double(kWideRatio) * double(kWideRatio);
  int big = 0;
#pragma unroll
  for (int j = 0; j < EPT; ++j) big += (fabsf(x[j]) * kWideRatio >= amax && x[j] != 0.f) ? 1 : 0;
  big = reduce_int(big);
  bool wide = live && (double(nz) * double(amax) * double(amax) > wide2 * s2 || big * kWideFrac < nz);

  // Outlier extraction (every branch below is block-uniform): a wide row sheds the entries
  // beyond kOutlierCut x rms(rest), round by round, until the rest passes both rules.
  static_assert(EPT <= 32, "the outlier mask is one word per thread");
  uint32_t omask = 0;  // bit j: x[j] is listed instead of entering the limbs
  int n_out = 0;
  if (wide) {
    float amax_r = amax;
    double s2_r = s2;
    int nz_r = nz;
    bool ok = false;
    // The cut is kOutlierCut x the scale of the rest: its rms, or 1.25 x its mean |x| (the
    // ratio of the two for a normal bulk) when that is smaller -- a few huge entries inflate the
    // rms far more than the mean, so the mean-based cut usually clears the row in one round.
    float s1_r = s1;  // sum |x| over the current rest
#pragma unroll 1
    for (int round = 0; round < kOutlierRounds; ++round) {
      const float cut = kOutlierCut * fminf(float(sqrt(s2_r / double(nz_r))), 1.25f * s1_r / float(nz_r));
      float am = 0.f, ssf = 0.f, s1f = 0.f;  // (a thread's <= 32 terms in fp32, scaled by the cut: no overflow)
      const float icut = 1.f / cut;
      int cnt = 0, near = 0;  // near: nonzeros of the rest within kWideRatio of the CUT (a lower bound of
                              // the second rule's count, which is relative to the rest's amax <= cut)
#pragma unroll
      for (int j = 0; j < EPT; ++j) {
        const float a = fabsf(x[j]);
        if (a > cut) {
          omask |= 1u << j;
        } else if (!((omask >> j) & 1u)) {
          am = fmaxf(am, a);
          const float t = a * icut;
          ssf = fmaf(t, t, ssf);
          s1f += t;
          cnt += a != 0.f;
          near += t * kWideRatio >= 1.f;
        }
      }
      double ss = double(ssf) * double(cut) * double(cut);
      int no = __popc(omask);
      reduce6(am, s1f, ss, cnt, no, near);
      amax_r = am;
      s1_r = s1f * cut;
      s2_r = ss;
      nz_r = cnt;
      n_out = no;
      if (n_out > kOutlierCap || nz_r == 0) break;
      if (double(nz_r) * double(amax_r) * double(amax_r) > wide2 * s2_r) continue;  // still wide: next round
      if (near * kWideFrac >= nz_r) {  // the second rule holds already by the lower bound
        ok = true;
        break;
      }
      int big_r = 0;
#pragma unroll
      for (int j = 0; j < EPT; ++j)
        big_r += (!((omask >> j) & 1u) && x[j] != 0.f && fabsf(x[j]) * kWideRatio >= amax_r) ? 1 : 0;
      big_r = reduce_int(big_r);
      if (big_r * kWideFrac >= nz_r) {  // the rest passes both rules
        ok = true;
        break;
      }
    }
    if (ok) {
      // the rest's scale must stay inside the epilogue's range: else the row keeps all its
      // entries in the limbs and takes the exact walk (or, without an exact-order format, the
      // fp64 recombination of the limb sums, which knows nothing of listed entries)
      int e_r;
      frexpf(amax_r, &e_r);
      const int s_r = 22 - e_r;
      ok = s_r <= kMaxScaleExp && s_r >= -kMaxScaleExp;
    }
    if (ok) {
      // list the outliers in ascending k: exclusive prefix of the per-thread counts (the
      // per-warp totals are the partials the last reduce6 left in red_j)
      const int mine = __popc(omask);
      int incl = mine;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if ((threadIdx.x & 31) >= o) incl += t;
      }
      int pos = incl - mine;
      for (int q = 0; q < w; ++q) pos += red_j[q];
      int2* lst = outlier_list(rscale, M_pad) + m * kOutlierCap;
#pragma unroll
      for (int j = 0; j < EPT; ++j) {
        if ((omask >> j) & 1u) {
          lst[pos++] = make_int2(int(k0) + j, __float_as_int(x[j]));
          x[j] = 0.f;  // the limbs see the rest only
        }
      }
      amax = amax_r;
      wide = false;
    } else {
      n_out = 0;
    }
  }
  int s = 0;
  if (live) {
    int e;
    frexpf(amax, &e);  // amax < 2^e
    s = 22 - e;        // |x * 2^s| < 2^22
  }
  if (threadIdx.x == 0) {
    // (a scale outside the epilogue's fp32 range also sends the row to the exact walk)
    const bool is_wide = wide || (live && (s > kMaxScaleExp || s < -kMaxScaleExp));
    const double sc = live ? ldexp(1.0, -s) : 0.0;
    rscale[m] = is_wide ? -sc : sc;
    outlier_counts(rscale, M_pad)[m] = is_wide ? 0 : n_out;
  }
  if (k0 < K_pad) {
    // x * 2^s as two exact power-of-two multiplies (2^s alone may exceed the float range)
    const int s_a = s > 126 ? 126 : (s < -126 ? -126 : s);
    const float sc_a = __int_as_float((127 + s_a) << 23), sc_b = __int_as_float((127 + s - s_a) << 23);
    uint32_t w0[EPT / 4], w1[EPT / 4], w2[EPT / 4];
#pragma unroll
    for (int j = 0; j < EPT; j += 4) {
      uint32_t u[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) u[i] = uint32_t((live ? __float2int_rn((x[j + i] * sc_a) * sc_b) : 0) + 0x808080);
      const uint32_t lo01 = __byte_perm(u[0], u[1], 0x5140);  // b0(u0) b0(u1) b1(u0) b1(u1)
      const uint32_t lo23 = __byte_perm(u[2], u[3], 0x5140);
      const uint32_t hi01 = __byte_perm(u[0], u[1], 0x7362);  // b2(u0) b2(u1) b3 b3
      const uint32_t hi23 = __byte_perm(u[2], u[3], 0x7362);
      w2[j / 4] = __byte_perm(lo01, lo23, 0x5410) ^ 0x80808080u;  // byte 0 of each u: low digit
      w1[j / 4] = __byte_perm(lo01, lo23, 0x7632) ^ 0x80808080u;  // byte 1: middle digit
      w0[j / 4] = __byte_perm(hi01, hi23, 0x5410) ^ 0x80808080u;  // byte 2: high digit
    }
    int8_t* l0 = limbs + m * K_pad + k0;
    int8_t* l1 = limbs + (M_pad + m) * K_pad + k0;
    int8_t* l2 = limbs + (2 * M_pad + m) * K_pad + k0;
    if constexpr (EPT % 16 == 0) {
#pragma unroll
      for (int j = 0; j < EPT / 4; j += 4) {
        reinterpret_cast<uint4*>(l0)[j / 4] = make_uint4(w0[j], w0[j + 1], w0[j + 2], w0[j + 3]);
        reinterpret_cast<uint4*>(l1)[j / 4] = make_uint4(w1[j], w1[j + 1], w1[j + 2], w1[j + 3]);
        reinterpret_cast<uint4*>(l2)[j / 4] = make_uint4(w2[j], w2[j + 1], w2[j + 2], w2[j + 3]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < EPT / 4; ++j) {
        reinterpret_cast<uint32_t*>(l0)[j] = w0[j];
        reinterpret_cast<uint32_t*>(l1)[j] = w1[j];
        reinterpret_cast<uint32_t*>(l2)[j] = w2[j];
      }
    }
  }
  if (threadIdx.x == 0) TG_GT(1);
}

// ------------------------------------------------------------------ decode
// Ternary tile word -> four int8x4 words (16 consecutive k of one column).
// Word layout (see tg_internal.h): byte i, bit 2q = nonzero, bit 2q+1 = sign,
// for entry k = 16c + 4q + i.
__device__ __forceinline__ uint4 decode_word(uint32_t w) {
  uint4 o;
  uint32_t x;
  x = w;
  o.x = (x & 0x01010101u) + (x & 0x02020202u) * 0x7Fu;
  x = w >> 2;
  o.y = (x & 0x01010101u) + (x & 0x02020202u) * 0x7Fu;
  x = w >> 4;
  o.z = (x & 0x01010101u) + (x & 0x02020202u) * 0x7Fu;
  x = w >> 6;
  o.w = (x & 0x01010101u) + (x & 0x02020202u) * 0x7Fu;
  return o;
}

// ------------------------------------------------------------------ MMA
struct MmaParams {
  const uint32_t* tiles;   // [KC][N_pad][8] packed ternary words
  const uint32_t* wrows;   // [KC * 128][N_pad / 16] the same codes row-major, 16 columns per word (outlier terms)
  const double* rscale;    // [M_pad], < 0 marks a wide row
  const float* bias;       // [N] or null
  float* Y;
  int64_t ldy;
  int M, N, K, KC, KS, M_pad, N_pad, MB, NB, splits;  // KC 128-k chunks, KS = ceil(KC/2) stages
  int NBG;                 // column-block groups: one group of CS blocks per cluster unit
  int units;               // cluster units = MB * NBG * splits
  int use_alpha;
  float alpha;
  int32_t* part;           // split-K limb partials [splits][3][M_pad][N_pad] (splits > 1)
  int32_t* counters;       // [MB * NB] arrival counters, zero between launches
  tg_device_flags* flags;
  int fix_var;             // < 0: no exact-order fix-up of wide rows
  int64_t m_full;          // blocked: rows < m_full take the banked order
  GatherArgs fix;
  const float* X;          // original X (fix-up reads it in place)
  int64_t ldx;
  int tma_y;               // 1: Y tiles leave through smem + TMA store (ymap), 0: direct stores
  // peer scatter (tg_gemm_tiles_run_scatter): every finished tile also goes to
  // ypeers[q] + col_off + m * ldy + n for q != rank; sig_local == null: off
  float* const* ypeers;
  uint32_t* const* speers;
  uint32_t* sig_local;
  int world, rank;
  int64_t col_off;
  // host streaming: every finished tile is also stored straight into the caller's pinned
  // host Y (device-mapped), so no copy-engine D2H follows the GEMM; null: off
  float* yh;
  int64_t ldyh;
  // outlier entries the X split kept out of the limbs: counts [M_pad], lists [M_pad][kOutlierCap] of (k, x bits)
  const int32_t* ocount;
  const int2* olist;
};

// One Y row segment to every other rank's full Y (plain st.global over NVLink).
__device__ __forceinline__ void peer_store(const MmaParams& p, int64_t off, float y) {
#pragma unroll 1
  for (int q = 0; q < p.world; ++q)
    if (q != p.rank) p.ypeers[q][off] = y;
}

// Tile configuration.  A pipeline stage covers 256 k (two 128-k chunks: 8
// MMAs of K = 32 and ONE tcgen05.commit -- a commit costs about as much as an
// MMA, so 4-MMA stages ran at ~55% of the issue rate: a round-1 probe; csrc/tg_peak.cu is its kept form).
// TMEM (512 columns x 128 lanes x 32 bit) holds ACC_BUFS accumulators of NMMA
// int32 columns plus two 64-column slots of the decoded W^T tile (128 lanes x
// 256 int8): the expanded ternary tile never touches shared memory, which
// carries only the X limbs and the packed W.
template <int MT>
struct MmaCfg {
  static constexpr int BN = 128;                 // output columns per unit (= MMA M)
  static constexpr int BK = 128;                 // k per chunk (bytes, int8; one 128-byte swizzle atom)
  static constexpr int CH = 2;                   // chunks per stage
  static constexpr int NMMA = 3 * MT;            // MMA N: three limbs of MT rows
  static constexpr int B_CHUNK = NMMA * BK;      // X limbs of one chunk
  static constexpr int B_BYTES = CH * B_CHUNK;
  static constexpr int P_CHUNK = BN * 32;        // packed 2-bit W of one chunk (128 k x 128 n)
  static constexpr int P_BYTES = CH * P_CHUNK;
#ifndef TG_SMEM_BUDGET
#define TG_SMEM_BUDGET 226000
#endif
  // packed-W ring: released by the decoders as soon as they read it
  // (deep for small MT: a decode-like GEMM streams W from HBM and needs many bytes in flight)
  static constexpr int P_STAGES = MT <= 16 ? 12 : MT <= 32 ? 8 : 4;
  // Y tile of one unit, written by the epilogue and stored with one TMA bulk-tensor store
  // (none at MT = 80: the X ring needs the room; that tile size stores Y directly)
  static constexpr int Y_BYTES = MT >= 80 ? 0 : MT * BN * 4;
  // X-limb ring: released by the MMA commit
  static constexpr int STAGES_RAW = (TG_SMEM_BUDGET - 3072 - P_STAGES * P_BYTES - Y_BYTES) / B_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int ACC_COLS = (NMMA + 31) / 32 * 32;
  static constexpr int A_COLS = CH * 32;         // TMEM columns of one decoded stage
  static constexpr int ACC_BUFS = (2 * ACC_COLS + 2 * A_COLS <= 512) ? 2 : 1;
  // decoded W^T slots: as many as TMEM holds next to the accumulators (at most 4, and no
  // more than the X stages their release rides on), so the decoders can run stages ahead
  static constexpr int A_SLOTS_ROOM = (512 - ACC_BUFS * ACC_COLS) / A_COLS;
  static constexpr int A_SLOTS_MAX = A_SLOTS_ROOM < 4 ? A_SLOTS_ROOM : 4;
  static constexpr int A_SLOTS = A_SLOTS_MAX < STAGES ? A_SLOTS_MAX : STAGES;
  static constexpr int A_BASE = ACC_BUFS * ACC_COLS;  // first TMEM column of the A ring
  static constexpr int TMEM_COLS = 512;
  static constexpr int SMEM =
      STAGES * B_BYTES + P_STAGES * P_BYTES + Y_BYTES + 1024 /*align*/ + 2048 /*barriers, scales*/;
  static constexpr int EPI_WARP0 = 7;            // warps: 0 X producer, 1 MMA, 2-5 decoders, 6 W producer
  // two per TMEM lane quarter, splitting the 16-row chunks; one per quarter at MT <= 32 (one or two
  // chunks): 480 threads instead of 608 leave 128 registers per thread, and the small-tile
  // kernel no longer spills (a spilled register costs a DRAM round trip after an L2 flush)
  static constexpr int EPI_WARPS = MT <= 32 ? 4 : 8;
  static constexpr int EPI_HALVES = EPI_WARPS / 4;
  // Small MT: N <= 96 MMAs take ~60 cycles each, faster than one decoder group expands a
  // stage (~700 cycles, mostly latency), so a second group (warps 15-18) takes every other
  // stage.
  static constexpr int DEC_GROUPS = MT <= 32 ? 2 : 1;
  static constexpr int DEC2_WARP0 = EPI_WARP0 + EPI_WARPS;
  static constexpr int THREADS = 32 * (EPI_WARP0 + EPI_WARPS + 4 * (DEC_GROUPS - 1));
  static_assert(MT % 16 == 0 && NMMA <= 256, "bad MT");
  static_assert(STAGES >= A_SLOTS, "slot release rides on the stage barrier: needs STAGES >= A_SLOTS");
  static_assert(STAGES >= 3 || MT < 64, "the X ring needs 3 stages at MT = 64");
  static_assert(A_BASE + A_SLOTS * A_COLS <= 512, "TMEM budget");
};

// Cluster unit u -> this CTA's column block nb (may be >= NB: a "ghost" block that
// only helps its cluster load the shared X tile), row block mb and stage range.
template <int CS>
__device__ __forceinline__ void unit_coords(const MmaParams& p, int u, int crank, int& nb, int& mb, int& ks0, int& ks1,
                                            int& split) {
  nb = (u % p.NBG) * CS + crank;
  const int rest = u / p.NBG;
  split = rest % p.splits;
  mb = rest / p.splits;
  ks0 = int((int64_t(split) * p.KS) / p.splits);
  ks1 = int((int64_t(split + 1) * p.KS) / p.splits);
}

// Finish 16 consecutive rows of one output column:
//   y = fp32(S0 2^(16-s) + S1 2^(8-s) + S2 2^-s + b) with three FMAs on the exact
//   float limb sums (|S_l| < 2^24), PReLU, and write y into the smem Y tile (or
//   straight to Y).  No FP64 and no 64-bit conversions on this path (each costs
//   ~13 issue cycles per warp on B200, a round-1 probe).  For integer-valued
//   X the low limbs are zero and every step is exact.  The per-row scales
//   {2^-s, 2^(8-s), 2^(16-s), 2^(24-s)} are staged in shared memory; rows whose
//   scale leaves the float range are "wide" and recomputed exactly afterwards
//   (or, without an exact-order format, here in full-range fp64).
struct EmitCtx {
  uint32_t sc_addr;  // smem address of the float scale of row m_first
  float bf;
  uint32_t wide_bits;
  uint32_t out_bits;  // rows (of the 16) with listed outlier entries
  const float* corr;  // their summed outlier terms (16 floats, 0 for the other rows)
  int m_first;
  int nlive;   // rows of this chunk inside Y (counting, fp64 fall-back)
  int nvalid;  // rows to store (16 into the smem tile: the TMA store clips rows >= M)
  bool n_ok;
  bool to_smem;      // true: st.shared into the Y tile at ysmem (row stride 512 bytes)
  uint32_t ysmem;
  float* ydst;       // false: Y (row stride ldy)
  int64_t ystride;
  int64_t yoff;      // element offset of ydst in this rank's full Y (peer scatter)
  int n;             // output column (host Y copy of direct stores)
};

// Row scales of 16 consecutive rows.  Full form: {2^-s, 2^(8-s), 2^(16-s), 2^(24-s)} per row
// (one ld.shared.v4 each).  Compact form (the small-tile kernels, MT <= 32, whose register
// budget is 104): 2^-s only; 2^(8-s) and 2^(16-s) are exact power-of-two multiples of it for
// every row whose scale is in range (the others are "wide" and recomputed).  Measured: the
// full form is ~4% faster at MT = 64, the compact one avoids spills at MT <= 32 (cfg4 -2 us).
__device__ __forceinline__ void load_scales(uint32_t addr, float4 (&sc)[16]) {
#pragma unroll
  for (int j = 0; j < 16; ++j)
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(sc[j].x), "=f"(sc[j].y), "=f"(sc[j].z), "=f"(sc[j].w)
                 : "r"(addr + 16u * j));
}
// (2^-s of 16 consecutive rows from either form: `stride` bytes between rows)
__device__ __forceinline__ void load_scales(uint32_t addr, float (&sc)[16], uint32_t stride) {
#pragma unroll
  for (int j = 0; j < 16; ++j) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(sc[j]) : "r"(addr + stride * j));
}
__device__ __forceinline__ void load_scales(uint32_t addr, float (&sc)[16]) {
#pragma unroll
  for (int j = 0; j < 16; j += 4)
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(sc[j]), "=f"(sc[j + 1]), "=f"(sc[j + 2]), "=f"(sc[j + 3])
                 : "r"(addr + 4u * j));
}

// tail shared by both emitters: PReLU, PReLU count, finiteness, the rare fp64 rows, store
__device__ __forceinline__ void emit_tail(float (&v)[16], const uint32_t* r0, const uint32_t* r1, const uint32_t* r2,
                                          const EmitCtx& e, const MmaParams& p, unsigned long long& npos,
                                          bool& bad) {
  const bool fix = p.fix_var >= 0;
  if (!fix && e.wide_bits) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (((e.wide_bits >> j) & 1u) && j < e.nlive) {
        const long long t = (static_cast<long long>(static_cast<int>(r0[j])) << 16) +
                            (static_cast<long long>(static_cast<int>(r1[j])) << 8) +
                            static_cast<long long>(static_cast<int>(r2[j]));
        v[j] = static_cast<float>(fma(static_cast<double>(t), fabs(__ldg(p.rscale + e.m_first + j)), double(e.bf)));
      }
    }
  }
  float mx = 0.f;
  if (p.use_alpha) {
    const float alpha = p.alpha;
    // the reference's `mults`: #(y <= 0) with PReLU; wide rows are counted by the fix-up
    if (e.nlive >= 16 && !(fix && e.wide_bits)) {
      unsigned cnt = 0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const bool neg = !(v[j] > 0.f);
        cnt += neg;
        v[j] = neg ? alpha * v[j] : v[j];
        mx = fmax_nan(mx, fabsf(v[j]));
      }
      if (e.n_ok) npos += cnt;
    } else {
      uint32_t negbits = 0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const bool neg = !(v[j] > 0.f);
        negbits |= uint32_t(neg) << j;
        v[j] = neg ? alpha * v[j] : v[j];
        mx = fmax_nan(mx, fabsf(v[j]));
      }
      const uint32_t live = e.nlive > 0 ? (e.nlive >= 16 ? 0xFFFFu : (1u << e.nlive) - 1u) : 0u;
      if (e.n_ok) npos += __popc(negbits & live & ~(fix ? e.wide_bits : 0u));
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) mx = fmax_nan(mx, fabsf(v[j]));  // padded rows / columns are exactly b or 0
  }
  if (!e.n_ok) return;
  bad |= !(mx <= 3.402823466e38f);
  if (e.to_smem) {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(e.ysmem + 512u * uint32_t(j)), "f"(v[j]) : "memory");
    return;
  }
  if (e.nvalid >= 16) {
#pragma unroll
    for (int j = 0; j < 16; ++j) e.ydst[int64_t(j) * e.ystride] = v[j];
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j < e.nvalid) e.ydst[int64_t(j) * e.ystride] = v[j];
  }
  if (p.yh) {
    float* d = p.yh + int64_t(e.m_first) * p.ldyh + e.n;
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j < e.nvalid) d[int64_t(j) * p.ldyh] = v[j];
  }
  if (p.sig_local) {
#pragma unroll 1
    for (int q = 0; q < p.world; ++q) {
      if (q == p.rank) continue;
      float* d = p.ypeers[q] + e.yoff;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < e.nvalid) d[int64_t(j) * e.ystride] = v[j];
    }
  }
}

// A finished smem Y tile (MT x 128, row pitch 512 B) to every other rank:
// each warp stores whole 512-byte row segments with 16-byte stores.
template <int MT>
__device__ __forceinline__ void peer_copy_tile(const MmaParams& p, const float* ytile, int m0, int n0, int et,
                                               int nthreads) {
  const int rows = min(MT, p.M - m0), cols = min(128, p.N - n0);
#pragma unroll 1
  for (int i = et; i < rows * 32; i += nthreads) {
    const int r = i >> 5, c = (i & 31) * 4;
    if (c >= cols) continue;
    const float4 v = *reinterpret_cast<const float4*>(ytile + r * 128 + c);
    const int64_t off = p.col_off + int64_t(m0 + r) * p.ldy + n0 + c;
#pragma unroll 1
    for (int q = 0; q < p.world; ++q) {
      if (q == p.rank) continue;
      float* d = p.ypeers[q] + off;
      if (c + 4 <= cols) {
        *reinterpret_cast<float4*>(d) = v;
      } else {
        d[0] = v.x;
        if (c + 1 < cols) d[1] = v.y;
        if (c + 2 < cols) d[2] = v.z;
      }
    }
  }
}

// A finished smem Y tile to the pinned host Y (16-byte stores over PCIe).
template <int MT>
__device__ __forceinline__ void host_copy_tile(const MmaParams& p, const float* ytile, int m0, int n0, int et,
                                               int nthreads) {
  const int rows = min(MT, p.M - m0), cols = min(128, p.N - n0);
#pragma unroll 1
  for (int i = et; i < rows * 32; i += nthreads) {
    const int r = i >> 5, c = (i & 31) * 4;
    if (c >= cols) continue;
    const float4 v = *reinterpret_cast<const float4*>(ytile + r * 128 + c);
    float* d = p.yh + int64_t(m0 + r) * p.ldyh + n0 + c;
    if (c + 4 <= cols) {
      *reinterpret_cast<float4*>(d) = v;
    } else {
      d[0] = v.x;
      if (c + 1 < cols) d[1] = v.y;
      if (c + 2 < cols) d[2] = v.z;
    }
  }
}

// Outlier terms of 16 consecutive rows for this lane's column n: corr[r] = sum over row
// (m_first + r)'s listed entries of W[k, n] * x, in list order (ascending k: a fixed order).
// The whole warp cooperates, in two memory round trips per pass of 16 entries of every row:
//   1. lanes l and l + 16 load entry 16 pass + l % 16 of each of the 16 lists (slots beyond a
//      row's count hold stale pairs and are masked), with the 16 counts;
//   2. each loads, for each of those entries, ITS half-warp's word of the row-major 2-bit plane
//      behind the tiles (16 columns per word: W[k, .] for the warp's 32 columns is two words);
// then entry i of every row is broadcast from lane i (to lanes 0-15) and lane i + 16 (to lanes
// 16-31) by shuffle -- a rolled loop over i, the rows unrolled, two shuffles per (row, entry) --
// and each lane adds its column's term.  Branch-free: bit 1 of a code flips the sign of x, bit
// 0 selects x or 0.  (One lane per column walking its rows' lists paid ~0.5 us of L2 latency
// per entry; a fully unrolled (entry, row) nest was 150 KB of code, fetch-bound.)
__device__ __noinline__ void outlier_chunk(const MmaParams& p, int m_first, int n, float* corr) {
  static_assert(kOutlierCap % 16 == 0, "passes of 16 entries");
  const int lane = int(threadIdx.x) & 31;
  const int hi = lane >> 4, lo = lane & 15;
  const uint32_t* wword = p.wrows + (n >> 4);  // this lane's word of a plane row (n >> 4 = warp base + hi)
  const int64_t kstride = p.N_pad >> 4;        // row pitch of the plane in words
  const int sh = 2 * (n & 15);
  const int cnt_l = __ldg(p.ocount + m_first + lo);  // lanes j and j + 16 hold row j's count
  int maxcnt = cnt_l;
  for (int o = 8; o; o >>= 1) maxcnt = max(maxcnt, __shfl_xor_sync(0xffffffffu, maxcnt, o));
  float acc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = 0.f;
#pragma unroll 1
  for (int pass = 0; 16 * pass < maxcnt; ++pass) {
    const int ei = 16 * pass + lo;  // the entry this lane holds, of every row
    const int2* lst = p.olist + int64_t(m_first) * kOutlierCap + ei;
    int2 e[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) e[j] = __ldg(lst + j * kOutlierCap);
    uint32_t wv[16];
    float xv[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const bool live = ei < __shfl_sync(0xffffffffu, cnt_l, j);
      xv[j] = live ? __int_as_float(e[j].y) : 0.f;  // (x = 0, codes 0: adds 0)
      wv[j] = live ? __ldg(wword + int64_t(e[j].x) * kstride) : 0u;
    }
    const int iend = min(16, maxcnt - 16 * pass);
#pragma unroll 1
    for (int i = 0; i < iend; ++i) {
      const int src = i + 16 * hi;  // the lane of my half-warp that holds entry i
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float x = __shfl_sync(0xffffffffu, xv[j], src);
        const uint32_t code = __shfl_sync(0xffffffffu, wv[j], src) >> sh;
        const float xs = __int_as_float(__float_as_int(x) ^ int((code & 2u) << 30));
        acc[j] += (code & 1u) ? xs : 0.f;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) corr[j] = acc[j];
}

// from the three limb sums of a finished accumulator (TMEM)
template <bool COMPACT>
__device__ __forceinline__ void emit16_limbs(const uint32_t (&r0)[16], const uint32_t (&r1)[16],
                                             const uint32_t (&r2)[16], const EmitCtx& e, const MmaParams& p,
                                             unsigned long long& npos, bool& bad) {
  float v[16];
  if (e.out_bits && e.n_ok) {
    // rows with listed outliers: y = limbs + (b + the row's outlier terms); the terms were
    // summed while the unit's MMAs ran and wait in local memory (e.corr)
    float sc[16];
    load_scales(e.sc_addr, sc, COMPACT ? 4u : 16u);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float s0 = sc[j], s1 = s0 * 256.f, s2 = s0 * 65536.f;
      v[j] = __fmaf_rn(float(int(r0[j])), s2,
                       __fmaf_rn(float(int(r1[j])), s1, __fmaf_rn(float(int(r2[j])), s0, e.bf + e.corr[j])));
    }
  } else if constexpr (COMPACT) {
    float sc[16];
    load_scales(e.sc_addr, sc);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float s0 = sc[j], s1 = s0 * 256.f, s2 = s0 * 65536.f;
      v[j] = __fmaf_rn(float(int(r0[j])), s2,
                       __fmaf_rn(float(int(r1[j])), s1, __fmaf_rn(float(int(r2[j])), s0, e.bf)));
    }
  } else {
    float4 sc[16];
    load_scales(e.sc_addr, sc);
#pragma unroll
    for (int j = 0; j < 16; ++j)
      v[j] = __fmaf_rn(float(int(r0[j])), sc[j].z,
                       __fmaf_rn(float(int(r1[j])), sc[j].y, __fmaf_rn(float(int(r2[j])), sc[j].x, e.bf)));
  }
  emit_tail(v, r0, r1, r2, e, p, npos, bad);
}


template <int MT, int CS>
__global__ void __launch_bounds__(MmaCfg<MT>::THREADS, 1)
    tg_mma_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap ymap,
                  const __grid_constant__ MmaParams p) {
  using C = MmaCfg<MT>;
  static_assert(CS == 1 || CS == 2 || CS == 4, "cluster size");
  static_assert(MT / CS >= 8, "multicast slices must be whole 8-row swizzle atoms");
  constexpr int SL = MT / CS;                       // X-limb rows this CTA loads and multicasts
  constexpr uint16_t CMASK = uint16_t((1u << CS) - 1u);
  constexpr int S = C::STAGES;
  constexpr int AS = C::A_SLOTS;
  constexpr int NACC = C::ACC_BUFS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int SP = C::P_STAGES;
  uint8_t* sB = smem;                       // S x B_BYTES (multiples of 1024)
  uint8_t* sP = sB + S * C::B_BYTES;        // SP x P_BYTES
  float* ytile = reinterpret_cast<float*>(sP + SP * C::P_BYTES);  // [MT][BN] fp32 (1024-aligned)
  uint64_t* full_raw = reinterpret_cast<uint64_t*>(sP + SP * C::P_BYTES + C::Y_BYTES);  // [S] X limbs landed
  uint64_t* empty = full_raw + S;           // [S]  MMAs of the stage done (all cluster CTAs)
  uint64_t* p_full = empty + S;             // [SP] packed W landed
  uint64_t* p_empty = p_full + SP;          // [SP] decoders done reading it
  uint64_t* a_full = p_empty + SP;          // [AS] decoded W^T slot written
  uint64_t* tfull = a_full + AS;            // [2]
  uint64_t* tempty = tfull + 2;             // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int32_t* last_flag = reinterpret_cast<int32_t*>(tmem_slot + 1);
  // [80] row scales of the current unit (float or float4 each, 16-byte aligned), then [4] wide-row masks
  double* rs_s = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(tmem_slot + 2) + 15) & ~uintptr_t(15));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int crank = CS > 1 ? int(cluster_ctarank()) : 0;
  const int cid = int(blockIdx.x) / CS, ncl = int(gridDim.x) / CS;
  if (threadIdx.x == 0) TG_STAMP(7, 0);
  if (threadIdx.x == 0) TG_GT(2);

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_raw[s], 1);
      mbar_init(&empty[s], CS);  // every CTA of the cluster must be done with the shared X stage
    }
    for (int s = 0; s < SP; ++s) {
      mbar_init(&p_full[s], 1);
      mbar_init(&p_empty[s], 4);
    }
    for (int s = 0; s < AS; ++s) mbar_init(&a_full[s], 4);
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], C::EPI_WARPS);
    }
    fence_mbar_init();
    *reinterpret_cast<unsigned long long*>(rs_s + 162) = 0ull;  // the CTA's PReLU count (epilogue)
    tma_prefetch_desc(&xmap);
    if (p.tma_y) tma_prefetch_desc(&ymap);
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  if (CS > 1) cluster_sync_all();  // peers multicast into our smem / arrive on our barriers
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) TG_STAMP(7, 1);
  // Programmatic dependent launch: everything above overlapped the X split.  Only
  // the X producer (limbs) and the epilogue (row scales) read its output and wait
  // for it; the W producer and the decoders start on the packed tiles at once.
  if (warp == 0 || (warp >= C::EPI_WARP0 && warp < C::DEC2_WARP0)) grid_dep_wait();
  if (threadIdx.x == 0) TG_GT(3);

  if (warp == 0) {
    // ---------------- producer of the X limbs (TMA 2D, multicast to the cluster).  The
    // whole warp runs the loop and an elected lane issues (see the MMA issuer: an
    // `if (lane == 0)` block costs a waterfall loop around every TMA instruction).
    uint32_t it = 0;
    for (int u = cid; u < p.units; u += ncl) {
      int nb, mb, ks0, ks1, split;
      unit_coords<CS>(p, u, crank, nb, mb, ks0, ks1, split);
      const int m0 = mb * MT;
      for (int ks = ks0; ks < ks1; ++ks, ++it) {
        const int s = int(it % S);
        const uint32_t r = it / S;
        const int nch = (2 * ks + 1 < p.KC) ? 2 : 1;
        mbar_wait(&empty[s], (r & 1) ^ 1);
        if (elect_one()) {
          TG_STAMP(0, it);
          mbar_arrive_expect_tx(&full_raw[s], uint32_t(nch * C::B_CHUNK));
          for (int c = 0; c < nch; ++c) {
            const int kc = 2 * ks + c;
            uint8_t* dst = sB + s * C::B_BYTES + c * C::B_CHUNK;
#pragma unroll
            for (int l = 0; l < 3; ++l) {
              uint8_t* d = dst + (l * MT + crank * SL) * C::BK;
              const int row = l * p.M_pad + m0 + crank * SL;
              if (CS == 1) tma_load_2d(d, &xmap, &full_raw[s], kc * C::BK, row);
              else tma_load_2d_mc(d, &xmap, &full_raw[s], kc * C::BK, row, CMASK);
            }
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 6) {
    // ---------------- producer of the packed W tiles (own ring, runs ahead of the X ring)
    uint32_t it = 0;
    for (int u = cid; u < p.units; u += ncl) {
      int nb, mb, ks0, ks1, split;
      unit_coords<CS>(p, u, crank, nb, mb, ks0, ks1, split);
      const int nsrc = nb < p.NB ? nb * C::BN : (p.NB - 1) * C::BN;  // ghost blocks decode a valid tile
      for (int ks = ks0; ks < ks1; ++ks, ++it) {
        const int sp = int(it % SP);
        const uint32_t rp = it / SP;
        const int nch = (2 * ks + 1 < p.KC) ? 2 : 1;
        mbar_wait(&p_empty[sp], (rp & 1) ^ 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&p_full[sp], uint32_t(nch * C::P_CHUNK));
          for (int c = 0; c < nch; ++c)
            bulk_load(sP + sp * C::P_BYTES + c * C::P_CHUNK, p.tiles + (size_t(2 * ks + c) * p.N_pad + nsrc) * 8,
                      C::P_CHUNK, &p_full[sp]);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: A = decoded W^T from TMEM, B = X limbs from smem.
    // One commit per stage (to the stage's `empty` barrier, in every cluster CTA);
    // the decoders derive the release of the A slot from the same barrier.  The whole
    // warp runs the loop and one elected lane issues: inside an elect.sync block ptxas
    // moves the operands to uniform registers directly, where an `if (lane == 0)` block
    // got a waterfall loop (ELECT + R2UR.BROADCAST + branch) around every tcgen05.mma,
    // ~70 cycles each -- the issue floor of small-N stages.
    {
      constexpr uint32_t idesc = idesc_i8(128, C::NMMA);
      // The CTA owns all 512 TMEM columns, so its allocation starts at address 0 (checked):
      // compile-time operand addresses.
      constexpr uint32_t tmem_base = 0;
      static_assert(C::TMEM_COLS == 512, "the MMA issuer assumes the whole TMEM");
      if (*tmem_slot != 0u) __trap();
      uint32_t it = 0, lu = 0;
      for (int u = cid; u < p.units; u += ncl, ++lu) {
        int nb, mb, ks0, ks1, split;
        unit_coords<CS>(p, u, crank, nb, mb, ks0, ks1, split);
        const uint32_t acc = lu % NACC, use = lu / NACC;
        mbar_wait(&tempty[acc], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t dtm = tmem_base + acc * C::ACC_COLS;
        for (int ks = ks0; ks < ks1; ++ks, ++it) {
          const int s = int(it % S);
          const int a = int(it % AS);
          const uint32_t ra = it / AS;
          const int nch = (2 * ks + 1 < p.KC) ? 2 : 1;
          // a_full implies full_raw: the decoders arrive on a_full only after they
          // observed this stage's bytes land, and the MMA reads the X limbs through
          // the same async proxy that wrote them.
          if (lane == 0) TG_STAMP(1, it);
          mbar_wait(&a_full[a], ra & 1);
          if (lane == 0) TG_STAMP(2, it);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t db = smem_desc_k_sw128(smem_u32(sB + s * C::B_BYTES));
            const uint32_t ta = tmem_base + uint32_t(C::A_BASE + a * C::A_COLS);
            for (int c = 0; c < nch; ++c) {
#pragma unroll
              for (int kk = 0; kk < C::BK / 32; ++kk) {
                // K step of 32 int8: +8 TMEM columns for A, +32 bytes (= +2 in the >>4 field) for B
                mma_i8_tmem_a(dtm, ta + uint32_t(c * 32 + kk * 8),
                              db + uint64_t((c * C::B_CHUNK) >> 4) + uint64_t(kk * 2), idesc,
                              (ks != ks0 || c != 0 || kk != 0) ? 1u : 0u);
              }
            }
            if (CS == 1) mma_commit(&empty[s]);
            else mma_commit_mc(&empty[s], CMASK);
            TG_STAMP(3, it);
            if (it == 0) TG_GT(4);
          }
          __syncwarp();
        }
        if (elect_one()) mma_commit(&tfull[acc]);
        __syncwarp();
      }
      if (lane == 0) TG_GT(5);
    }
  } else if (warp < 6 || warp >= C::DEC2_WARP0) {
    // ---------------- decoders (warps 2..5, and 15..18 for the odd stages when
    // DEC_GROUPS = 2): packed smem -> decoded W^T rows in TMEM.
    // Warp w may only access TMEM lanes 32*(w%4)..+31; lane = W^T row = output column.
    const int q = warp & 3;
    const uint32_t grp = warp < 6 ? 0u : 1u;
    const uint32_t row = uint32_t(q * 32 + lane);
    const uint32_t lane_addr = uint32_t(q * 32) << 16;
    uint32_t it = 0;
    for (int u = cid; u < p.units; u += ncl) {
      int nb, mb, ks0, ks1, split;
      unit_coords<CS>(p, u, crank, nb, mb, ks0, ks1, split);
      for (int ks = ks0; ks < ks1; ++ks, ++it) {
        if (it % C::DEC_GROUPS != grp) continue;  // the other group's stage
        const int s = int(it % S);
        const uint32_t r = it / S;
        const int a = int(it % AS);
        const int nch = (2 * ks + 1 < p.KC) ? 2 : 1;
        const int sp = int(it % SP);
        mbar_wait(&p_full[sp], (it / SP) & 1);
        if (q == 0 && lane == 0) TG_STAMP(4, it);
        uint4 w[2][2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (c < nch) {
            // (two 16-byte loads at a 32-byte lane stride: a 2-way bank conflict.  Swapping the
            // halves on lanes 4-7 of every phase removes it but costs selects on the decoders'
            // critical path: cfg4 +1.7 us, cfg2 neutral, profiles/r02_v3/ab_halfswap.txt)
            const uint32_t src = smem_u32(sP + sp * C::P_BYTES + c * C::P_CHUNK) + row * 32u;
            w[c][0] = lds128(src);
            w[c][1] = lds128(src + 16u);
          }
        }
        // slot a was last read by the MMAs of iteration it - AS, released with stage
        // (it - AS) % S (at most one phase behind: STAGES >= A_SLOTS)
        if (it >= uint32_t(AS)) {
          const uint32_t prev = it - AS;
          mbar_wait(&empty[prev % S], (prev / S) & 1);
        }
        if (q == 0 && lane == 0) TG_STAMP(5, it);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (c < nch) {
            uint32_t v[32];
            const uint32_t pw[8] = {w[c][0].x, w[c][0].y, w[c][0].z, w[c][0].w,
                                    w[c][1].x, w[c][1].y, w[c][1].z, w[c][1].w};
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint4 o = decode_word(pw[j]);
              v[4 * j + 0] = o.x;
              v[4 * j + 1] = o.y;
              v[4 * j + 2] = o.z;
              v[4 * j + 3] = o.w;
            }
            tmem_st32(tmem_base + lane_addr + uint32_t(C::A_BASE + a * C::A_COLS + c * 32), v);
          }
        }
        // The packed tile goes back to the W producer only here, after the tcgen05.st that
        // consumed the decoded words: every lane's ld.shared has then delivered its data.
        // Released right after the loads were ISSUED (round 1), the arrive could overtake loads
        // still in flight when the load/store pipe was busy (the epilogue's outlier lookups),
        // the producer refilled the slot, and single lanes decoded the next tile's bytes: wrong
        // W^T rows for a stage, non-deterministically (8192 x 8192 x 1024 with outlier rows,
        // profiles/r02_v3/README.md).  An early release behind a true data dependence on the
        // loads (the arrive address XORed with dep ^ own-lane-shuffle(dep)) is also correct but
        // puts a shuffle on the decoders' critical path: cfg3 +5.5 us, cfg4 +1.8 us
        // (profiles/r02_v3/ab_release.txt).
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_empty[sp]);
        tmem_st_wait();
        // the MMA waits only on a_full: make it imply that this stage's X limbs landed too
        mbar_wait(&full_raw[s], r & 1);
        if (q == 0 && lane == 0) TG_STAMP(6, it);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[a]);
      }
    }
  } else {
    // ---------------- epilogue (warps 7..14): warp w owns TMEM lane quarter w%4
    // (32 output columns) and the 16-row chunks of parity `half`.  The unit's Y
    // tile is assembled in shared memory and leaves with one TMA store.
    constexpr int ET = 32 * C::EPI_WARPS;
    const int q = warp & 3;
    const int et = threadIdx.x - 32 * C::EPI_WARP0;  // 0..ET-1
    const int half = (warp - C::EPI_WARP0) >> 2;
    const uint32_t rs_addr = smem_u32(rs_s);
    constexpr bool COMPACT = C::DEC_GROUPS > 1;     // (the small-tile kernels: see load_scales)
    float* sc_s = reinterpret_cast<float*>(rs_s);  // [80] row scales of the unit (x4 when !COMPACT)
    uint32_t* wmask = reinterpret_cast<uint32_t*>(rs_s + 160);  // [4] wide-row bits of the unit (after 80 float4)
    uint32_t* omask = reinterpret_cast<uint32_t*>(rs_s + 163);  // [4] rows with listed outliers (after the PReLU count)
    bool any_bad = false;
    unsigned long long npos = 0;
    uint32_t lu = 0;
    for (int u = cid; u < p.units; u += ncl, ++lu) {
      int nb, mb, ks0, ks1, split;
      unit_coords<CS>(p, u, crank, nb, mb, ks0, ks1, split);
      const bool ghost = nb >= p.NB;
      const int n0 = nb * C::BN, m0 = mb * MT;
      const uint32_t acc = lu % NACC, use = lu / NACC;
      const int c = q * 32 + lane;  // column inside the tile
      const int n = n0 + c;
      const bool n_ok = n < p.N;
      const float bf = (n_ok && p.bias) ? __ldg(p.bias + n) : 0.f;
      // previous unit: its TMA store must have read the Y tile, everyone done with the scales
      if (et < 32 && p.tma_y && elect_one()) bulk_wait_group_read0();  // (the storing lane)
      named_bar_sync(1, ET);
      {  // stage the unit's row scales (and which rows are "wide") in shared memory
        const double rs = et < MT ? __ldcg(p.rscale + m0 + et) : 0.0;
        if (et < MT) {
          const double a = fabs(rs);
          if (COMPACT) sc_s[et] = float(a);
          else reinterpret_cast<float4*>(sc_s)[et] =
              make_float4(float(a), float(a * 256.0), float(a * 65536.0), float(a * 16777216.0));
        }
        const uint32_t wbits = __ballot_sync(0xffffffffu, rs < 0.0);
        const uint32_t obits = __ballot_sync(0xffffffffu, et < MT && __ldcg(p.ocount + m0 + et) > 0);
        if (lane == 0 && (et >> 5) < 4) {
          wmask[et >> 5] = wbits;
          omask[et >> 5] = obits;
        }
      }
      named_bar_sync(1, ET);
      // Outlier terms of this thread's rows (the X split listed the entries it kept out of the
      // limbs): summed here, while the unit's MMAs run, so the lookups hide behind them.
      constexpr int MSTEP = 16 * C::EPI_HALVES;  // rows between two chunks of one warp
      constexpr int MSHIFT = C::EPI_HALVES == 2 ? 5 : 4;
      float corr[16 * ((MT + MSTEP - 1) / MSTEP)];
      auto fill_corr = [&]() {
        if (ghost) return;  // (warp-uniform; padded columns n < N_pad read valid words)
#pragma unroll 1
        for (int mm = 16 * half; mm < MT; mm += MSTEP) {
          const uint32_t bits = (omask[mm >> 5] >> (mm & 31)) & 0xFFFFu;
          if (bits) outlier_chunk(p, m0 + mm, n, corr + (mm >> MSHIFT) * 16);  // (warp-uniform)
        }
      };
      if (et == 0 && lu == 0) TG_GT(8);
      if (p.splits == 1) fill_corr();
      if (et == 0 && lu == 0) TG_GT(9);
      mbar_wait(&tfull[acc], use & 1);
      if (et == 0 && lu == 0) TG_GT(10);
      if (et == 0) TG_STAMP(7, 2 + 2 * lu);
      tc_fence_after();
      const uint32_t tbase = tmem_base + acc * C::ACC_COLS + (uint32_t(q * 32) << 16);
      bool final_writer = p.splits == 1;
      auto ctx = [&](int mm) {
        EmitCtx e;
        e.sc_addr = rs_addr + (COMPACT ? 4u : 16u) * uint32_t(mm);
        e.bf = bf;
        e.wide_bits = (wmask[mm >> 5] >> (mm & 31)) & 0xFFFFu;
        e.out_bits = (omask[mm >> 5] >> (mm & 31)) & 0xFFFFu;
        e.corr = corr + (mm >> MSHIFT) * 16;
        e.m_first = m0 + mm;
        e.nlive = min(16, p.M - (m0 + mm));
        e.nvalid = e.nlive;
        e.n_ok = n_ok;
        static_assert(C::BN * 4 == 512, "Y tile row pitch");
        e.to_smem = p.tma_y != 0;  // the TMA store clips rows >= M
        e.ysmem = smem_u32(ytile) + uint32_t(mm * C::BN + c) * 4u;
        e.ydst = p.Y + int64_t(m0 + mm) * p.ldy + n;
        e.ystride = p.ldy;
        e.yoff = p.col_off + int64_t(m0 + mm) * p.ldy + n;
        e.n = n;
        return e;
      };
#pragma unroll 1
      for (int mm = 16 * half; mm < MT; mm += MSTEP) {
        if (et == 0 && lu == 0) TG_STAMP(7, 200 + mm / 16);
        uint32_t r0[16], r1[16], r2[16];
#ifdef TG_EPI_NOLDTM
#pragma unroll
        for (int j = 0; j < 16; ++j) r0[j] = r1[j] = r2[j] = uint32_t(j + mm + et);
#else
        tmem_ld16(tbase + mm, r0);
        tmem_ld16(tbase + MT + mm, r1);
        tmem_ld16(tbase + 2 * MT + mm, r2);
        tmem_ld_wait();
#endif
        // The accumulator goes back to the MMA warp as soon as this warp's LAST chunk is in
        // registers, before that chunk is emitted (with a single accumulator, MT = 80, the MMAs
        // of the next unit wait for this; with two it only matters when the epilogue is the
        // slower side).
        if (mm + MSTEP >= MT) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        if (et == 0 && lu == 0) TG_STAMP(7, 220 + mm / 16);
        if (p.splits == 1) {
          emit16_limbs<COMPACT>(r0, r1, r2, ctx(mm), p, npos, any_bad);
          if (et == 0 && lu == 0) TG_STAMP(7, 240 + mm / 16);
        } else if (!ghost) {
          // per-limb partials: the reduced sums take exactly the unsplit epilogue, so a
          // row's bits do not depend on whether its GEMM was split
          const int64_t plane = int64_t(p.M_pad) * p.N_pad;
          int32_t* dst = p.part + 3 * int64_t(split) * plane + int64_t(m0 + mm) * p.N_pad + n;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            dst[int64_t(j) * p.N_pad] = int32_t(r0[j]);
            dst[plane + int64_t(j) * p.N_pad] = int32_t(r1[j]);
            dst[2 * plane + int64_t(j) * p.N_pad] = int32_t(r2[j]);
          }
        }
      }
      if (et == 0 && lu == 0) TG_STAMP(7, 120);

      if (p.splits > 1 && !ghost) {
        // last-arriving unit of this (mb, nb) tile reduces the limb partials
        __threadfence();
        named_bar_sync(1, ET);
        if (et == 0) {
          const int old = atomicAdd(p.counters + (mb * p.NB + nb), 1);
          const int last = old == p.splits - 1;
          if (last) p.counters[mb * p.NB + nb] = 0;  // reset for the next launch
          *last_flag = last;
        }
        named_bar_sync(1, ET);
        final_writer = *last_flag != 0;
        if (final_writer) {
          __threadfence();
          fill_corr();
#pragma unroll 1
          for (int j0 = 16 * half; j0 < MT; j0 += MSTEP) {
            // 16 independent rows per batch so the L2 reads of the partials overlap;
            // int32 sums stay exact (|S_l| < 128 K < 2^31)
            const int64_t plane = int64_t(p.M_pad) * p.N_pad;
            uint32_t t0[16], t1[16], t2[16];
            const int32_t* src = p.part + int64_t(m0 + j0) * p.N_pad + n;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              t0[j] = uint32_t(__ldcg(src + int64_t(j) * p.N_pad));
              t1[j] = uint32_t(__ldcg(src + plane + int64_t(j) * p.N_pad));
              t2[j] = uint32_t(__ldcg(src + 2 * plane + int64_t(j) * p.N_pad));
            }
#pragma unroll 1
            for (int sp = 1; sp < p.splits; ++sp) {
              const int32_t* s2 = src + 3 * int64_t(sp) * plane;
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                t0[j] += uint32_t(__ldcg(s2 + int64_t(j) * p.N_pad));
                t1[j] += uint32_t(__ldcg(s2 + plane + int64_t(j) * p.N_pad));
                t2[j] += uint32_t(__ldcg(s2 + 2 * plane + int64_t(j) * p.N_pad));
              }
            }
            emit16_limbs<COMPACT>(t0, t1, t2, ctx(j0), p, npos, any_bad);
          }
        }
        named_bar_sync(1, ET);  // last_flag is reused by the next unit
      }
      if (et == 0 && lu == 0) TG_STAMP(7, 121);
      // exact-order recomputation of wide rows in this tile (usually none)
      if (final_writer && p.fix_var >= 0 && n_ok) {
#pragma unroll 1
        for (int w = 0; w < (MT + 31) / 32; ++w) {
          uint32_t bits = wmask[w];
          while (bits) {
            const int j = 32 * w + (__ffs(bits) - 1);
            bits &= bits - 1;
            const int m = m0 + j;
            if (m >= p.M || ((j >> 4) & (C::EPI_HALVES - 1)) != half) continue;
            float y = column_value_row(p.fix_var, p.fix, n, bf, p.X + int64_t(m) * p.ldx, p.K, m < p.m_full);
            if (p.use_alpha && !(y > 0.f)) {
              y = p.alpha * y;
              ++npos;
            }
            any_bad |= !isfinite(y);
            if (p.tma_y) {
              ytile[j * C::BN + c] = y;
            } else {
              p.Y[int64_t(m) * p.ldy + n] = y;
              if (p.yh) p.yh[int64_t(m) * p.ldyh + n] = y;
              if (p.sig_local) peer_store(p, p.col_off + int64_t(m) * p.ldy + n, y);
            }
          }
        }
      }
      if (p.tma_y && final_writer && !ghost) {
        fence_proxy_async_smem();  // our st.shared -> visible to the TMA (async proxy)
        named_bar_sync(1, ET);
        if (et < 32 && elect_one()) {  // (the same lane commits, and later waits for, the bulk group)
          tma_store_2d(&ymap, ytile, n0, m0);
          bulk_commit_group();
        }
        if (p.sig_local) peer_copy_tile<MT>(p, ytile, m0, n0, et, ET);  // overlaps the local TMA store
        if (p.yh) host_copy_tile<MT>(p, ytile, m0, n0, et, ET);
      }
    }
    if (p.sig_local) {
      // the last CTA to finish tells every rank that this rank's shard is in place: its own
      // Y (TMA store) must be complete too, not only read out of shared memory
      if (et < 32 && p.tma_y && elect_one()) bulk_wait_group0();  // (the storing lane)
      __threadfence_system();  // this thread's peer stores before the CTA's arrival
      named_bar_sync(1, ET);
      if (et == 0) {
        const unsigned old = atomicAdd(p.sig_local + TG_PEER_DONE_WORD, 1u);
        if (old == gridDim.x - 1) {
          p.sig_local[TG_PEER_DONE_WORD] = 0u;  // every CTA has arrived: reset for the next launch
          __threadfence_system();
#pragma unroll 1
          for (int q = 0; q < p.world; ++q)
            asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(p.speers[q] + p.rank) : "memory");
        }
      }
    }
    if (et == 0) TG_STAMP(7, 301);
    if (et == 0) TG_STAMP(7, 3 + 2 * (lu - 1));
    if (et == 0) TG_GT(6);
    if (p.flags) {
      // one global atomic per CTA: ~1000 same-address atomics from every warp of the grid
      // serialise in L2 for microseconds at the end of the kernel
      if (__any_sync(0xffffffffu, any_bad) && lane == 0) atomicOr(&p.flags->nonfinite_output, 1);
      for (int o = 16; o; o >>= 1) npos += __shfl_xor_sync(0xffffffffu, npos, o);
      unsigned long long* npos_s = reinterpret_cast<unsigned long long*>(rs_s + 162);
      if (lane == 0 && npos) atomicAdd(npos_s, npos);
      named_bar_sync(1, ET);
      if (et == 0 && *npos_s) atomicAdd(reinterpret_cast<unsigned long long*>(&p.flags->nonpositive_outputs), *npos_s);
    }
    // The smem Y tile must have been read by the TMA store before the CTA exits (waited for
    // here, after the status words so the two overlap); the global writes complete with the
    // grid, as in CUTLASS's store tail.
    if (et < 32 && p.tma_y && elect_one()) bulk_wait_group_read0();  // (the storing lane)
  }
  if (threadIdx.x == 32 * C::EPI_WARP0) TG_STAMP(7, 302);
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) TG_STAMP(7, 303);
  if (CS > 1) cluster_sync_relaxed();  // no CTA leaves while peers may still multicast to it
  if (threadIdx.x == 0) TG_STAMP(7, 304);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
  if (threadIdx.x == 0) TG_STAMP(7, 500);
  if (threadIdx.x == 0) TG_GT(7);
}

// ------------------------------------------------------------------ pack
// Dense int8 W (K x N, leading dimension ldw) -> ternary tiles.
__global__ void tg_pack_tiles_dense_kernel(const int8_t* __restrict__ W, int64_t K, int64_t N, int64_t ldw,
                                           uint32_t* __restrict__ tiles, int64_t KC, int64_t N_pad,
                                           tg_device_flags* __restrict__ flags) {
  const int64_t total = KC * 8 * N_pad;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t n = idx % N_pad;
    const int64_t rest = idx / N_pad;
    const int c = int(rest % 8);
    const int64_t kc = rest / 8;
    uint32_t word = 0;
    if (n < N) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int64_t k = kc * 128 + c * 16 + j;
        if (k < K) {
          const int v = W[k * ldw + n];
          const int bit = 8 * (j & 3) + 2 * (j >> 2);
          if (v == 1) word |= 1u << bit;
          else if (v == -1) word |= 3u << bit;
          else if (v != 0 && flags) atomicOr(&flags->bad_input, 1);
        }
      }
    }
    tiles[(kc * N_pad + n) * 8 + c] = word;
  }
}

// Scatter one sparse entry (row k, column n, sign) into the tile array.
// Sets flags->corrupt bit0 on a duplicate (row, col) of the same sign and bit1
// on a cell claimed by both signs (tcsc.py:105-113).
__device__ __forceinline__ void tile_set(uint32_t* tiles, int64_t N_pad, int64_t k, int64_t n, bool neg,
                                         tg_device_flags* flags) {
  const int64_t kc = k >> 7;
  const int c = int((k >> 4) & 7);
  const int j = int(k & 15);
  const int bit = 8 * (j & 3) + 2 * (j >> 2);
  const uint32_t old = atomicOr(tiles + (kc * N_pad + n) * 8 + c, (neg ? 3u : 1u) << bit);
  if (flags && ((old >> bit) & 1u)) {
    const bool old_neg = ((old >> (bit + 1)) & 1u) != 0;
    atomicOr(&flags->corrupt, old_neg == neg ? 1 : 2);
  }
}

// TCSC-style (col_start, row_index) list for one sign -> tiles.  One warp per column.
__global__ void tg_pack_tiles_csc_kernel(const int32_t* __restrict__ col_start, const int32_t* __restrict__ rows,
                                         int64_t ncols, int64_t col_stride_blocks, int64_t nblocks, bool neg,
                                         uint32_t* __restrict__ tiles, int64_t N_pad, int64_t K,
                                         tg_device_flags* __restrict__ flags) {
  const int64_t warp_id = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp_id >= ncols * nblocks) return;
  const int64_t blk = warp_id / ncols;
  const int64_t n = warp_id % ncols;
  const int32_t* cs = col_start + blk * col_stride_blocks;
  const int32_t a = cs[n], b = cs[n + 1];
  for (int32_t i = a + lane; i < b; i += 32) {
    const int32_t k = rows[i];
    if (k < 0 || k >= K) {
      if (flags) atomicOr(&flags->bad_input, 2);
      continue;
    }
    tile_set(tiles, N_pad, k, n, neg, flags);
  }
}

// Interleaved-blocked stream -> tiles.  One warp per cell (blk, n).
__global__ void tg_pack_tiles_ib_kernel(const int32_t* __restrict__ ai, const int32_t* __restrict__ ptr,
                                        int64_t N, int64_t nblocks, int g, int64_t K,
                                        uint32_t* __restrict__ tiles, int64_t N_pad, tg_device_flags* __restrict__ flags) {
  const int64_t cell = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (cell >= N * nblocks) return;
  const int64_t n = cell % N;
  const int32_t s0 = ptr[3 * cell], s1 = ptr[3 * cell + 1], s2 = ptr[3 * cell + 2], s3 = ptr[3 * cell + 3];
  for (int32_t i = s0 + lane; i < s3; i += 32) {
    const int32_t k = ai[i];
    if (k == K) continue;  // symmetric dummy
    if (k < 0 || k > K) {
      if (flags) atomicOr(&flags->bad_input, 2);
      continue;
    }
    bool neg;
    if (i < s1) neg = (((i - s0) / g) & 1) != 0;
    else neg = i >= s2;
    tile_set(tiles, N_pad, k, n, neg, flags);
  }
}

// Symmetric interleaved stream -> tiles.  One warp per column; the sign of
// stream position t is the run parity (t / g) & 1 (variants.py:622-631).
__global__ void tg_pack_tiles_sym_kernel(const int32_t* __restrict__ idx, const int32_t* __restrict__ ptr,
                                         int64_t N, int g, int64_t K, uint32_t* __restrict__ tiles, int64_t N_pad,
                                         tg_device_flags* __restrict__ flags) {
  const int64_t n = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (n >= N) return;
  const int32_t s = ptr[n], e = ptr[n + 1];
  for (int32_t i = s + lane; i < e; i += 32) {
    const int32_t k = idx[i];
    if (k == K) continue;  // dummy
    if (k < 0 || k > K) {
      if (flags) atomicOr(&flags->bad_input, 2);
      continue;
    }
    tile_set(tiles, N_pad, k, n, (((i - s) / g) & 1) != 0, flags);
  }
}

// Compressed codes (N x G, 5 base-3 digits per byte, low digit first) -> tiles.
// One thread per tile word (16 consecutive k of one column).
__global__ void tg_pack_tiles_codes_kernel(const uint8_t* __restrict__ codes, int64_t K, int64_t N, int64_t G,
                                           uint32_t* __restrict__ tiles, int64_t KC, int64_t N_pad) {
  const int64_t total = KC * 8 * N_pad;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t n = idx % N_pad;
    const int64_t rest = idx / N_pad;
    const int c = int(rest % 8);
    const int64_t kc = rest / 8;
    uint32_t word = 0;
    if (n < N) {
      int64_t gi = -1;
      int code = 121;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int64_t k = kc * 128 + c * 16 + j;
        if (k < K) {
          if (k / 5 != gi) {
            gi = k / 5;
            code = codes[n * G + gi];
          }
          int d = code;
          for (int t = int(k - 5 * gi); t > 0; --t) d /= 3;
          d %= 3;  // 0: -1, 1: 0, 2: +1
          const int bit = 8 * (j & 3) + 2 * (j >> 2);
          if (d == 2) word |= 1u << bit;
          else if (d == 0) word |= 3u << bit;
        }
      }
    }
    tiles[(kc * N_pad + n) * 8 + c] = word;
  }
}

// ------------------------------------------------------------------ host launchers
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// Per-device caches: kernel attributes (cudaFuncSetAttribute) and occupancy apply per device
// context, so every cache below is keyed by the current device (up to 64 devices).
static int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev & 63;
}

// true once per (flag set, device): the caller then applies its per-device setup
static bool first_on_device(std::atomic<uint64_t>& done) {
  const uint64_t bit = uint64_t(1) << current_device();
  return (done.fetch_or(bit) & bit) == 0;
}

static int num_sms() {
  static std::atomic<int> cache[64];
  const int d = current_device();
  int n = cache[d].load(std::memory_order_relaxed);
  if (n == 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || n <= 0) n = 148;
    cache[d].store(n, std::memory_order_relaxed);
  }
  return n;
}

int mma_pick_mt(int64_t M) {
  if (const char* env = getenv("TG_MMA_MT")) {
    const int v = atoi(env);
    if (v == 16 || v == 32 || v == 48 || v == 64 || v == 80) return v;
  }
  if (M <= 16) return 16;
  if (M <= 32) return 32;
  if (M <= 48) return 48;
  // MT = 80 (MMA N = 240) hides the per-stage commit inside the longer MMAs (round-1 probe:
  // 131 cycles per 128x240x32 MMA with a commit every 8, at the issue-rate peak) but has room for
  // one TMEM accumulator only, so its epilogue is not overlapped: worth it for tall X (many units
  // per CTA) whose padding to 80 rows is small.
  if (M >= 2048 && round_up(M, 80) * 100 <= round_up(M, 64) * 102) return 80;
  return 64;  // N = 192: two TMEM accumulators + a 2-slot A ring fill the 512 columns
}

// K splits per (column group, row block) tile: minimise rounds x (stages + overhead)
// over a persistent grid of `slots` clusters.  Integer accumulation makes any split exact.
static int pick_splits(int64_t base_units, int64_t KC, int slots) {
  int best = 1;
  int64_t best_cost = INT64_MAX;
  const int64_t smax = std::min<int64_t>(KC, 16);
  for (int64_t s = 1; s <= smax; ++s) {
    const int64_t rounds = ceil_div(base_units * s, slots);
    // a split unit pays its partial stores and the last arrival's reduction: measured on
    // B200 at about 6 stages' worth (cfg2 / cfg4 with 2-4 splits: +4.5 to +13 us)
    const int64_t cost = rounds * (ceil_div(KC, s) + (s > 1 ? 6 : 0));
    if (cost < best_cost) {
      best_cost = cost;
      best = int(s);
    }
  }
  return best;
}

// Cluster size: the X-limb tile of a row block is multicast to CS CTAs that
// work on CS adjacent column blocks, cutting the L2->SM traffic (the bound of
// the 1-CTA kernel) by CS.  Slices must be whole 8-row swizzle atoms.
static int pick_cluster(int64_t mt, int64_t NB) {
  int cs = mt >= 64 ? 4 : mt >= 32 ? (mt == 48 ? 2 : 4) : 1;
  if (const char* env = getenv("TG_MMA_CLUSTER")) {
    const int v = atoi(env);
    if (v == 1 || v == 2 || v == 4) cs = v;
  }
  while (cs > 1 && (mt / cs < 8 || (mt / cs) % 8 != 0)) cs /= 2;
  while (cs > 1 && NB < cs) cs /= 2;
  return cs;
}

template <int MT, int CS>
static int max_clusters() {
  static std::atomic<int> cache[64];
  const int d = current_device();
  int n = cache[d].load(std::memory_order_relaxed);
  if (n == 0) {
    using C = MmaCfg<MT>;
    cudaFuncSetAttribute(tg_mma_kernel<MT, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (CS > 1) cudaFuncSetAttribute(tg_mma_kernel<MT, CS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(CS * 256));
    cfg.blockDim = dim3(C::THREADS);
    cfg.dynamicSmemBytes = C::SMEM;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, tg_mma_kernel<MT, CS>, &cfg) != cudaSuccess || c <= 0) {
      cudaGetLastError();
      c = num_sms() / CS;
    }
    n = c;
    cache[d].store(n, std::memory_order_relaxed);
  }
  return n;
}

static int max_clusters_for(int64_t mt, int cs) {
  switch (mt * 10 + cs) {
    case 161: return max_clusters<16, 1>();
    case 162: return max_clusters<16, 2>();
    case 321: return max_clusters<32, 1>();
    case 322: return max_clusters<32, 2>();
    case 324: return max_clusters<32, 4>();
    case 481: return max_clusters<48, 1>();
    case 482: return max_clusters<48, 2>();
    case 641: return max_clusters<64, 1>();
    case 642: return max_clusters<64, 2>();
    case 801: return max_clusters<80, 1>();
    case 802: return max_clusters<80, 2>();
    default: return max_clusters<64, 4>();
  }
}

struct SplitLayout {
  int64_t mt, M_pad, K_pad, N_pad, KC, MB, NB, NBG;
  int splits, cs, clusters;
  size_t off_rscale, off_counters, off_ocount, off_olist, off_part, total_prepare, total;
};

// `share` > 1: this GEMM runs beside share - 1 others (host streaming's row chunks on
// their own streams) and takes 1/share of the co-resident clusters, so the chunks'
// GEMMs run side by side on disjoint SMs instead of one after another.
static SplitLayout split_layout(int64_t M, int64_t K, int64_t N, int share = 1) {
  SplitLayout L;
  L.mt = mma_pick_mt(M);
  L.M_pad = round_up(M, L.mt);
  L.K_pad = round_up(K, 128);
  L.KC = L.K_pad / 128;
  L.MB = L.M_pad / L.mt;
  L.N_pad = N > 0 ? round_up(N, 128) : 0;
  L.NB = L.N_pad / 128;
  L.cs = N > 0 ? pick_cluster(L.mt, L.NB) : 1;
  L.NBG = ceil_div(L.NB, L.cs);
  L.clusters = N > 0 ? std::max(1, max_clusters_for(L.mt, L.cs) / std::max(1, share)) : 1;
  L.splits = N > 0 ? pick_splits(L.MB * L.NBG, ceil_div(L.KC, 2), L.clusters) : 1;
  if (const char* env = getenv("TG_MMA_SPLITS"))  // experiments only
    if (N > 0) L.splits = int(std::max<int64_t>(1, std::min<int64_t>(atoi(env), ceil_div(L.KC, 2))));
  if (L.MB * L.NB > kSplitCounters) L.splits = 1;  // the split zeroes kSplitCounters counters
  L.off_rscale = size_t(round_up(3 * L.M_pad * L.K_pad, 256));
  const PrepTail pt = prep_tail(L.M_pad);
  L.off_counters = L.off_rscale + size_t(pt.counters);
  L.off_ocount = L.off_rscale + size_t(pt.ocount);
  L.off_olist = L.off_rscale + size_t(pt.olist);
  L.total_prepare = size_t(round_up(int64_t(L.off_rscale) + pt.end, 256));
  L.off_part = L.total_prepare;
  L.total = L.splits > 1 ? L.off_part + size_t(L.splits) * 3 * size_t(L.M_pad) * size_t(L.N_pad) * 4
                         : L.total_prepare;
  return L;
}

size_t xsplit_bytes(int64_t M, int64_t K) { return split_layout(M, K, 0).total_prepare; }
// true when the X split reads each row once (register- or smem-resident kernels); the
// multi-pass fall-back for longer rows reads a row twice, which over PCIe (X read in place
// from host memory) would double the transfer
bool xsplit_single_read(int64_t K) { return split_layout(1, K, 0).K_pad <= 1024 * 32 || K <= XS_SMEM_MAX_K; }
size_t mma_ws_bytes(int64_t M, int64_t K, int64_t N, int share) { return split_layout(M, K, N, share).total; }

// rows left to the exact walk / rows with listed outliers / listed entries of a prepared workspace
int xsplit_row_stats(const void* ws, int64_t M, int64_t K, int64_t* stats, cudaStream_t st) {
  const SplitLayout L = split_layout(M, K, 0);
  const uint8_t* base = static_cast<const uint8_t*>(ws);
  double* rs = static_cast<double*>(malloc(size_t(M) * sizeof(double)));
  int32_t* oc = static_cast<int32_t*>(malloc(size_t(M) * sizeof(int32_t)));
  if (!rs || !oc) {
    free(rs);
    free(oc);
    return set_error(TG_ERR_PARAM, "out of host memory");
  }
  cudaError_t e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = cudaMemcpy(rs, base + L.off_rscale, size_t(M) * sizeof(double), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(oc, base + L.off_ocount, size_t(M) * sizeof(int32_t), cudaMemcpyDeviceToHost);
  stats[0] = stats[1] = stats[2] = 0;
  if (e == cudaSuccess) {
    for (int64_t m = 0; m < M; ++m) {
      stats[0] += rs[m] < 0.0;
      stats[1] += oc[m] > 0;
      stats[2] += oc[m];
    }
  }
  free(rs);
  free(oc);
  return e == cudaSuccess ? TG_OK : set_cuda_error(e, "xsplit_row_stats");
}

int run_xsplit(const float* X, int64_t M, int64_t K, int64_t ldx, void* ws, size_t ws_bytes, tg_device_flags* flags,
               cudaStream_t st) {
  const SplitLayout L = split_layout(M, K, 0);
  if (ws_bytes < L.total_prepare) return set_error(TG_ERR_PARAM, "workspace too small for X split");
  uint8_t* base = static_cast<uint8_t*>(ws);
  int8_t* limbs = reinterpret_cast<int8_t*>(base);
  double* rscale = reinterpret_cast<double*>(base + L.off_rscale);
  cudaError_t e = cudaSuccess;
  // register-resident kernel: one pass over the row when K_pad <= THREADS * EPT
  const unsigned grid = unsigned(L.M_pad);
#define TG_XS_REG(T, E)                                                                                       \
  if (L.K_pad <= int64_t(T) * (E)) {                                                                           \
    tg_xsplit_reg_kernel<T, E><<<grid, T, 0, st>>>(X, M, K, ldx, limbs, rscale, L.M_pad, L.K_pad, flags);  \
    return check_launch("tg_xsplit_reg_kernel");                                                               \
  }
  if (L.M_pad <= 4 * num_sms()) {  // few rows: wide CTAs (two per SM) so the whole GPU has loads in flight
    TG_XS_REG(512, 4)
    TG_XS_REG(512, 8)
    TG_XS_REG(512, 16)
  } else {
    TG_XS_REG(256, 16)
    TG_XS_REG(256, 32)
    TG_XS_REG(512, 32)
  }
  TG_XS_REG(1024, 32)
#undef TG_XS_REG
  if (K <= XS_SMEM_MAX_K) {
    const size_t smem = size_t(round_up(K, 4)) * sizeof(float);
    static std::atomic<uint64_t> attr_done{0};
    if (first_on_device(attr_done)) {
      e = cudaFuncSetAttribute(tg_xsplit_kernel<true, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(XS_SMEM_MAX_K * sizeof(float)));
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(tg_xsplit_kernel<true, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(XS_SMEM_MAX_K * sizeof(float)));
      if (e != cudaSuccess) {
        attr_done.fetch_and(~(uint64_t(1) << current_device()));
        return set_cuda_error(e, "cudaFuncSetAttribute(tg_xsplit_kernel)");
      }
    }
    // few rows: more threads per row so the whole GPU has loads in flight
    if (L.M_pad <= 4 * num_sms())
      tg_xsplit_kernel<true, 1024><<<unsigned(L.M_pad), 1024, smem, st>>>(X, M, K, ldx, limbs, rscale,
                                                                          L.M_pad, L.K_pad, flags);
    else
      tg_xsplit_kernel<true, 256><<<unsigned(L.M_pad), 256, smem, st>>>(X, M, K, ldx, limbs, rscale, L.M_pad,
                                                                        L.K_pad, flags);
  } else {
    tg_xsplit_kernel<false, 256><<<unsigned(L.M_pad), 256, 0, st>>>(X, M, K, ldx, limbs, rscale, L.M_pad,
                                                                     L.K_pad, flags);
  }
  return check_launch("tg_xsplit_kernel");
}

template <int MT, int CS>
static int launch_mma(const CUtensorMap& map, const CUtensorMap& ymap, const MmaParams& p, int grid,
                      cudaStream_t st) {
  using C = MmaCfg<MT>;
  static std::atomic<uint64_t> attr_done{0};
  if (first_on_device(attr_done)) {
    cudaError_t e =
        cudaFuncSetAttribute(tg_mma_kernel<MT, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) {
      attr_done.fetch_and(~(uint64_t(1) << current_device()));
      return set_cuda_error(e, "cudaFuncSetAttribute(tg_mma_kernel)");
    }
  }
  MmaParams pp = p;
  if (C::Y_BYTES == 0) pp.tma_y = 0;  // no smem Y tile at this tile size
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap our prologue with the X split
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = CS;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = CS > 1 ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, tg_mma_kernel<MT, CS>, map, ymap, pp);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaLaunchKernelEx(tg_mma_kernel)");
  return check_launch("tg_mma_kernel");
}

int run_mma(const float* X, int64_t M, int64_t K, int64_t ldx, const uint32_t* tiles, int64_t N, const float* bias,
            float* Y, int64_t ldy, int use_alpha, float alpha, const MmaFixup* fix, void* ws, size_t ws_bytes,
            tg_device_flags* flags, cudaStream_t st, const tg_peer_scatter* sc, int share, float* yh,
            int64_t ldyh) {
  const SplitLayout L = split_layout(M, K, N, share);
  if (ws_bytes < L.total) return set_error(TG_ERR_PARAM, "workspace too small for the tensor-core path");
  uint8_t* base = static_cast<uint8_t*>(ws);
  int8_t* limbs = reinterpret_cast<int8_t*>(base);

  auto enc = get_encode();
  if (!enc) return set_error(TG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap map;
  cuuint64_t gdim[2] = {cuuint64_t(L.K_pad), cuuint64_t(3 * L.M_pad)};
  cuuint64_t gstride[1] = {cuuint64_t(L.K_pad)};
  cuuint32_t box[2] = {128u, cuuint32_t(L.mt / L.cs)};  // each cluster CTA loads (and multicasts) one slice
  cuuint32_t estride[2] = {1u, 1u};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, limbs, gdim, gstride, box, estride,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(TG_ERR_CUDA, "cuTensorMapEncodeTiled failed");

  // Y leaves through a TMA store when its layout allows it (16-byte aligned base and row pitch)
  CUtensorMap ymap;
  memset(&ymap, 0, sizeof(ymap));
  int tma_y = 0;
  // (the peer copy of a scattered tile reuses that alignment: 16-byte stores need col_off % 4 == 0)
  if ((reinterpret_cast<uintptr_t>(Y) & 15) == 0 && (ldy * 4) % 16 == 0 && !getenv("TG_MMA_DIRECT_Y") &&
      !(sc && sc->col_off % 4 != 0)) {
    cuuint64_t ydim[2] = {cuuint64_t(N), cuuint64_t(M)};
    cuuint64_t ystride[1] = {cuuint64_t(ldy) * 4};
    cuuint32_t ybox[2] = {128u, cuuint32_t(L.mt)};
    cuuint32_t yes[2] = {1u, 1u};
    if (enc(&ymap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, Y, ydim, ystride, ybox, yes, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
      tma_y = 1;
  }
  MmaParams p{};
  p.tma_y = tma_y;
  p.tiles = tiles;
  p.wrows = tiles + size_t(L.KC) * size_t(L.N_pad) * 8;
  p.rscale = reinterpret_cast<const double*>(base + L.off_rscale);
  p.bias = bias;
  p.Y = Y;
  p.ldy = ldy;
  p.M = int(M);
  p.N = int(N);
  p.K = int(K);
  p.KC = int(L.KC);
  p.KS = int(ceil_div(L.KC, 2));
  p.M_pad = int(L.M_pad);
  p.N_pad = int(L.N_pad);
  p.MB = int(L.MB);
  p.NB = int(L.NB);
  p.NBG = int(L.NBG);
  p.splits = L.splits;
  p.units = int(L.MB * L.NBG * L.splits);
  p.use_alpha = use_alpha;
  p.alpha = alpha;
  p.flags = flags;
  p.fix_var = -1;
  if (fix) {
    p.fix_var = fix->var;
    p.m_full = fix->m_full;
    p.fix = fix->args;
    p.X = X;
    p.ldx = ldx;
  }
  p.yh = yh;
  p.ldyh = ldyh;
  p.ocount = reinterpret_cast<const int32_t*>(base + L.off_ocount);
  p.olist = reinterpret_cast<const int2*>(base + L.off_olist);
  if (sc) {
    p.ypeers = sc->y_peers;
    p.speers = sc->sig_peers;
    p.sig_local = sc->sig_local;
    p.world = sc->world;
    p.rank = sc->rank;
    p.col_off = sc->col_off;
  }
  if (L.splits > 1) {  // (the counters were zeroed by the X split of this call)
    p.counters = reinterpret_cast<int32_t*>(base + L.off_counters);
    p.part = reinterpret_cast<int32_t*>(base + L.off_part);
  }
  const int grid = int(std::min<int64_t>(p.units, L.clusters)) * L.cs;
  switch (L.mt * 10 + L.cs) {
    case 161: return launch_mma<16, 1>(map, ymap, p, grid, st);
    case 162: return launch_mma<16, 2>(map, ymap, p, grid, st);
    case 321: return launch_mma<32, 1>(map, ymap, p, grid, st);
    case 322: return launch_mma<32, 2>(map, ymap, p, grid, st);
    case 324: return launch_mma<32, 4>(map, ymap, p, grid, st);
    case 481: return launch_mma<48, 1>(map, ymap, p, grid, st);
    case 482: return launch_mma<48, 2>(map, ymap, p, grid, st);
    case 641: return launch_mma<64, 1>(map, ymap, p, grid, st);
    case 642: return launch_mma<64, 2>(map, ymap, p, grid, st);
    case 801: return launch_mma<80, 1>(map, ymap, p, grid, st);
    case 802: return launch_mma<80, 2>(map, ymap, p, grid, st);
    default: return launch_mma<64, 4>(map, ymap, p, grid, st);
  }
}

int run_pack_dense(const int8_t* W, int64_t K, int64_t N, int64_t ldw, uint32_t* tiles, tg_device_flags* flags,
                   cudaStream_t st) {
  const int64_t KC = round_up(K, 128) / 128;
  const int64_t N_pad = round_up(N, 128);
  const int64_t total = KC * 8 * N_pad;
  const unsigned blocks = unsigned(std::min<int64_t>((total + 255) / 256, 148 * 16));
  tg_pack_tiles_dense_kernel<<<blocks, 256, 0, st>>>(W, K, N, ldw, tiles, KC, N_pad, flags);
  return check_launch("tg_pack_tiles_dense_kernel");
}

int run_pack_csc(const int32_t* col_start, const int32_t* rows, int64_t N, int64_t nblocks, bool neg,
                 uint32_t* tiles, int64_t K, tg_device_flags* flags, cudaStream_t st) {
  const int64_t N_pad = round_up(N, 128);
  const int64_t warps = N * nblocks;
  if (warps == 0) return TG_OK;
  tg_pack_tiles_csc_kernel<<<unsigned((warps * 32 + 255) / 256), 256, 0, st>>>(col_start, rows, N, N + 1, nblocks,
                                                                                 neg, tiles, N_pad, K, flags);
  return check_launch("tg_pack_tiles_csc_kernel");
}

int run_pack_ib(const int32_t* ai, const int32_t* ptr, int64_t N, int64_t nblocks, int g, int64_t K,
                uint32_t* tiles, tg_device_flags* flags, cudaStream_t st) {
  const int64_t N_pad = round_up(N, 128);
  const int64_t warps = N * nblocks;
  if (warps == 0) return TG_OK;
  tg_pack_tiles_ib_kernel<<<unsigned((warps * 32 + 255) / 256), 256, 0, st>>>(ai, ptr, N, nblocks, g, K, tiles,
                                                                                N_pad, flags);
  return check_launch("tg_pack_tiles_ib_kernel");
}

}  // namespace tg

namespace tg {

// Tiles -> the row-major 2-bit plane stored right behind them: rows[k][N_pad / 16], column n of
// row k at bits 2 (n % 16) of word n / 16 (1: +1, 3: -1, 0: zero).  One thread per output word.
__global__ void tg_rows_plane_kernel(const uint32_t* __restrict__ tiles, int64_t KC, int64_t N_pad,
                                     uint32_t* __restrict__ rows) {
  const int64_t wpr = N_pad >> 4;
  const int64_t total = KC * 128 * wpr;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = idx / wpr, j16 = idx % wpr;
    const int64_t kc = k >> 7;
    const int c = int((k >> 4) & 7), j = int(k & 15);
    const int bit = 8 * (j & 3) + 2 * (j >> 2);
    uint32_t out = 0;
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const uint32_t w = __ldg(tiles + (kc * N_pad + j16 * 16 + t) * 8 + c);
      out |= ((w >> bit) & 3u) << (2 * t);
    }
    rows[idx] = out;
  }
}

int run_rows_plane(uint32_t* tiles, int64_t K, int64_t N, cudaStream_t st) {
  const int64_t KC = round_up(K, 128) / 128;
  const int64_t N_pad = round_up(N, 128);
  const int64_t total = KC * 128 * (N_pad >> 4);
  const unsigned blocks = unsigned(std::min<int64_t>((total + 255) / 256, 148 * 32));
  tg_rows_plane_kernel<<<blocks, 256, 0, st>>>(tiles, KC, N_pad, tiles + KC * N_pad * 8);
  return check_launch("tg_rows_plane_kernel");
}

// Tiles -> dense int8 W (K x N, ld = N).  One thread per (k, n).
__global__ void tg_unpack_dense_kernel(const uint32_t* __restrict__ tiles, int64_t K, int64_t N, int64_t N_pad,
                                       int8_t* __restrict__ W) {
  const int64_t total = K * N;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = idx / N, n = idx % N;
    const uint32_t w = __ldg(tiles + ((k >> 7) * N_pad + n) * 8 + ((k >> 4) & 7));
    const int j = int(k & 15);
    const int bit = 8 * (j & 3) + 2 * (j >> 2);
    const uint32_t v = (w >> bit) & 3u;
    W[idx] = v == 1u ? int8_t(1) : v == 3u ? int8_t(-1) : int8_t(0);
  }
}

int run_unpack_dense(const uint32_t* tiles, int64_t K, int64_t N, int8_t* W, cudaStream_t st) {
  const int64_t total = K * N;
  const unsigned blocks = unsigned(std::min<int64_t>((total + 255) / 256, 148 * 32));
  tg_unpack_dense_kernel<<<blocks, 256, 0, st>>>(tiles, K, N, round_up(N, 128), W);
  return check_launch("tg_unpack_dense_kernel");
}

}  // namespace tg

#ifdef TG_TRACE
extern "C" int tg_debug_trace(unsigned long long* host_out) {
  return cudaMemcpyFromSymbol(host_out, tg::g_tg_trace, sizeof(tg::g_tg_trace)) == cudaSuccess ? 0 : 3;
}
extern "C" int tg_debug_gt(unsigned long long* host_out, int reset) {
  if (reset) {
    unsigned long long init[16][2];
    for (int i = 0; i < 16; ++i) {
      init[i][0] = ~0ull;
      init[i][1] = 0;
    }
    return cudaMemcpyToSymbol(tg::g_tg_gt, init, sizeof(init)) == cudaSuccess ? 0 : 3;
  }
  return cudaMemcpyFromSymbol(host_out, tg::g_tg_gt, sizeof(tg::g_tg_gt)) == cudaSuccess ? 0 : 3;
}
#endif

namespace tg {

int run_pack_sym(const int32_t* idx, const int32_t* ptr, int64_t N, int g, int64_t K, uint32_t* tiles,
                 tg_device_flags* flags, cudaStream_t st) {
  if (N == 0) return TG_OK;
  tg_pack_tiles_sym_kernel<<<unsigned((N * 32 + 255) / 256), 256, 0, st>>>(idx, ptr, N, g, K, tiles,
                                                                             round_up(N, 128), flags);
  return check_launch("tg_pack_tiles_sym_kernel");
}

int run_pack_codes(const uint8_t* codes, int64_t K, int64_t N, uint32_t* tiles, cudaStream_t st) {
  const int64_t KC = round_up(K, 128) / 128;
  const int64_t N_pad = round_up(N, 128);
  const int64_t total = KC * 8 * N_pad;
  const unsigned blocks = unsigned(std::min<int64_t>((total + 255) / 256, 148 * 16));
  tg_pack_tiles_codes_kernel<<<blocks, 256, 0, st>>>(codes, K, N, ceil_div(K, 5), tiles, KC, N_pad);
  return check_launch("tg_pack_tiles_codes_kernel");
}

}  // namespace tg
