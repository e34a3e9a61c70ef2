// tg_mma.cu — dense-decode tensor-core path for Y = X W + b (+PReLU).
//
// Semantics: same result contract as the reference kernels
//   gemm_base                /root/reference/pkg/src/terngemm/kernels/scalar.py:109-148
//   gemm_vectorized_optimal  /root/reference/pkg/src/terngemm/kernels/simd.py:282-449
// i.e. Y[m,n] = b[n] + sum_{k: W[k,n]=+1} X[m,k] - sum_{k: W[k,n]=-1} X[m,k],
// then y <- (y > 0 ? y : alpha*y) in fp32 when PReLU is on (simd.py:410-417).
//
// Realisation (B200-native):
//   1. tg_xsplit_kernel: each X row is scaled by a power of two 2^s so that
//      max|x| < 2^22, rounded to an integer v, and v is split into three
//      balanced signed base-256 digits (int8 "limbs").  Exact for integer X.
//   2. tg_mma_kernel (warp specialised, one CTA per 128 n x MT m tile):
//        warp 0   TMA: the three limb tiles of X -> smem (SWIZZLE_128B)
//        warps 2-5 decode the 2-bit ternary tiles of W into int8 {-1,0,+1}
//                 K-major SW128 smem tiles (the "expanded ternary tile")
//        warp 1   one elected lane issues tcgen05.mma.kind::i8 with
//                 A = W^T tile (M=128 rows = output columns n),
//                 B = [limb0; limb1; limb2] (N = 3*MT rows = output rows m)
//                 into an int32 accumulator in TMEM.  Integer accumulation is
//                 exact, so the result does not depend on summation order.
//        warps 2-5 epilogue: tcgen05.ld the three limb sums, recombine
//                 exactly in int64, scale by 2^-s in fp64, add the bias,
//                 round once to fp32, PReLU, coalesced store of Y.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>

#include "tg_ptx.cuh"
#include "tg_internal.h"

namespace tg {

// ------------------------------------------------------------------ X split
// One CTA per (padded) row.  limbs: [3][M_pad][K_pad] int8, rscale: [M_pad] f64,
// wide: [1 + M_pad] int32 (count, then row ids).
//
// Row m is scaled by 2^s, s = 22 - e with amax < 2^e, so |x 2^s| < 2^22; the
// rounded integer v splits into balanced base-256 digits v = d0 2^16 + d1 2^8 + d2.
// The grid step 2^(e-22) is relative to the row maximum, so a row whose nonzero
// entries span a wide dynamic range (amax > kWideRatio * rms of its nonzeros)
// is listed in `wide` and later recomputed by the exact-order fix-up kernel;
// its rscale is stored negated so the MMA epilogue leaves its PReLU count alone.
constexpr float kWideRatio = 16.f;

__global__ void __launch_bounds__(256) tg_xsplit_kernel(const float* __restrict__ X, int64_t M, int64_t K,
                                                        int64_t ldx, int8_t* __restrict__ limbs,
                                                        double* __restrict__ rscale, int32_t* __restrict__ wide,
                                                        int64_t M_pad, int64_t K_pad,
                                                        tg_device_flags* __restrict__ flags) {
  const int64_t m = blockIdx.x;
  const float* row = X + m * ldx;
  __shared__ float red[8];
  __shared__ float red2[8];
  __shared__ int redn[8];
  float amax = 0.f;
  if (m < M) {
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) amax = fmaxf(amax, fabsf(row[k]));
  }
  for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
  __syncthreads();
  amax = red[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) amax = fmaxf(amax, red[i]);
  const bool finite = amax <= 3.402823466e38f;  // false for inf / nan
  int s = 0;
  if (m < M && amax > 0.f) {
    if (!finite) {
      if (threadIdx.x == 0 && flags) atomicOr(&flags->bad_input, 4);
    } else {
      int e;
      frexpf(amax, &e);  // amax < 2^e
      s = 22 - e;        // |x * 2^s| < 2^22
    }
  }
  // dynamic range of the nonzero entries: sum (x / amax)^2 and their count
  bool is_wide = false;
  if (m < M && amax > 0.f && finite) {
    const float inv = 1.f / amax;
    float s2 = 0.f;
    int nz = 0;
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
      const float t = row[k] * inv;
      s2 += t * t;
      nz += t != 0.f;
    }
    for (int o = 16; o; o >>= 1) {
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      nz += __shfl_xor_sync(0xffffffffu, nz, o);
    }
    if ((threadIdx.x & 31) == 0) {
      red2[threadIdx.x >> 5] = s2;
      redn[threadIdx.x >> 5] = nz;
    }
    __syncthreads();
    s2 = 0.f;
    nz = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      s2 += red2[i];
      nz += redn[i];
    }
    is_wide = float(nz) > kWideRatio * kWideRatio * s2;  // amax / rms(nonzeros) > kWideRatio
  }
  if (threadIdx.x == 0) {
    const double sc = (m < M && amax > 0.f && finite) ? ldexp(1.0, -s) : 0.0;
    rscale[m] = is_wide ? -sc : sc;
    if (is_wide && wide) {
      const int slot = atomicAdd(wide, 1);
      wide[1 + slot] = int32_t(m);
    }
  }
  int8_t* l0 = limbs + m * K_pad;
  int8_t* l1 = limbs + (M_pad + m) * K_pad;
  int8_t* l2 = limbs + (2 * M_pad + m) * K_pad;
  const bool live = m < M && amax > 0.f && finite;
  for (int64_t k0 = int64_t(threadIdx.x) * 4; k0 < K_pad; k0 += int64_t(blockDim.x) * 4) {
    uint32_t p0 = 0, p1 = 0, p2 = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t k = k0 + j;
      int v = 0;
      if (live && k < K) v = __float2int_rn(ldexpf(row[k], s));
      const int d2 = ((v + 128) & 255) - 128;
      const int v1 = (v - d2) >> 8;
      const int d1 = ((v1 + 128) & 255) - 128;
      const int d0 = (v1 - d1) >> 8;
      p0 |= (uint32_t(d0) & 255u) << (8 * j);
      p1 |= (uint32_t(d1) & 255u) << (8 * j);
      p2 |= (uint32_t(d2) & 255u) << (8 * j);
    }
    *reinterpret_cast<uint32_t*>(l0 + k0) = p0;
    *reinterpret_cast<uint32_t*>(l1 + k0) = p1;
    *reinterpret_cast<uint32_t*>(l2 + k0) = p2;
  }
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
template <int MT, int STAGES>
struct MmaCfg {
  static constexpr int BN = 128;                 // output columns per CTA (= MMA M)
  static constexpr int BK = 128;                 // k per stage (bytes, int8)
  static constexpr int NMMA = 3 * MT;            // MMA N: three limbs of MT rows
  static constexpr int A_BYTES = BN * BK;        // decoded W^T stage
  static constexpr int B_BYTES = NMMA * BK;      // X limb stage
  static constexpr int TMEM_COLS = NMMA <= 32 ? 32 : NMMA <= 64 ? 64 : NMMA <= 128 ? 128 : 256;
  static constexpr int SMEM = STAGES * (A_BYTES + B_BYTES) + 1024 /*align*/ + 256 /*barriers*/;
  static_assert(MT % 16 == 0 && NMMA <= 256, "bad MT");
};

template <int MT, int STAGES>
__global__ void __launch_bounds__(192, 1)
    tg_mma_kernel(const __grid_constant__ CUtensorMap xmap, const uint32_t* __restrict__ tiles,
                  const double* __restrict__ rscale, const float* __restrict__ bias, float* __restrict__ Y,
                  int64_t ldy, int M, int N, int KC, int M_pad, int N_pad, int use_alpha, float alpha,
                  tg_device_flags* __restrict__ flags) {
  using C = MmaCfg<MT, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint64_t* full_a = reinterpret_cast<uint64_t*>(sB + STAGES * C::B_BYTES);
  uint64_t* full_b = full_a + STAGES;
  uint64_t* empty = full_b + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * C::BN;
  const int m0 = blockIdx.y * MT;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_a[s], 4);
      mbar_init(&full_b[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_mbar_init();
    tma_prefetch_desc(&xmap);
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer: X limbs
    if (lane == 0) {
      for (int kc = 0; kc < KC; ++kc) {
        const int s = kc % STAGES;
        const uint32_t round = kc / STAGES;
        mbar_wait(&empty[s], (round & 1) ^ 1);
        mbar_arrive_expect_tx(&full_b[s], C::B_BYTES);
        uint8_t* dst = sB + s * C::B_BYTES;
#pragma unroll
        for (int l = 0; l < 3; ++l)
          tma_load_2d(dst + l * MT * C::BK, &xmap, &full_b[s], kc * C::BK, l * M_pad + m0);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_i8(128, C::NMMA);
      for (int kc = 0; kc < KC; ++kc) {
        const int s = kc % STAGES;
        const uint32_t round = kc / STAGES;
        mbar_wait(&full_a[s], round & 1);
        mbar_wait(&full_b[s], round & 1);
        tc_fence_after();
        const uint64_t da = smem_desc_k_sw128(smem_u32(sA + s * C::A_BYTES));
        const uint64_t db = smem_desc_k_sw128(smem_u32(sB + s * C::B_BYTES));
#pragma unroll
        for (int kk = 0; kk < C::BK / 32; ++kk) {
          // +32 bytes along K inside the 128-byte swizzle atom = +2 in the (>>4) address field
          mma_i8(tmem_base, da + uint64_t(kk * 2), db + uint64_t(kk * 2), idesc, (kc | kk) != 0);
        }
        mma_commit(&empty[s]);
      }
      mma_commit(tmem_full);
    }
  } else {
    // ---------------- decoders (warps 2..5), then epilogue
    const int t = threadIdx.x - 64;  // 0..127 = row of the W^T tile
    const uint4* src = reinterpret_cast<const uint4*>(tiles) + (size_t(n0 + t) * 2);
    const size_t kc_stride = size_t(N_pad) * 2;  // uint4 per kc
    uint4 c0 = __ldg(src), c1 = __ldg(src + 1);
    const uint32_t row_off = uint32_t(t) * 128u;
    const uint32_t sw = uint32_t(t) & 7u;
    for (int kc = 0; kc < KC; ++kc) {
      const int s = kc % STAGES;
      const uint32_t round = kc / STAGES;
      uint4 n0v = make_uint4(0, 0, 0, 0), n1v = make_uint4(0, 0, 0, 0);
      if (kc + 1 < KC) {
        n0v = __ldg(src + (kc + 1) * kc_stride);
        n1v = __ldg(src + (kc + 1) * kc_stride + 1);
      }
      mbar_wait(&empty[s], (round & 1) ^ 1);
      uint8_t* a = sA + s * C::A_BYTES + row_off;
      const uint32_t w[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        *reinterpret_cast<uint4*>(a + ((uint32_t(c) ^ sw) << 4)) = decode_word(w[c]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_a[s]);
      c0 = n0v;
      c1 = n1v;
    }

    // ---------------- epilogue
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int n = n0 + q * 32 + lane;
    const bool n_ok = n < N;
    const double bn = (n_ok && bias) ? double(bias[n]) : 0.0;
    bool any_bad = false;
    unsigned long long npos = 0;
    const uint32_t tbase = tmem_base + (uint32_t(q * 32) << 16);
#pragma unroll 1
    for (int mm = 0; mm < MT; mm += 16) {
      uint32_t r0[16], r1[16], r2[16];
      tmem_ld16(tbase + mm, r0);
      tmem_ld16(tbase + MT + mm, r1);
      tmem_ld16(tbase + 2 * MT + mm, r2);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int m = m0 + mm + j;
        if (m < M && n_ok) {
          const long long tot = (static_cast<long long>(static_cast<int>(r0[j])) << 16) +
                                (static_cast<long long>(static_cast<int>(r1[j])) << 8) +
                                static_cast<long long>(static_cast<int>(r2[j]));
          const double rs = __ldg(rscale + m);  // < 0: wide row, the fix-up kernel owns its count
          const double v = static_cast<double>(tot) * fabs(rs) + bn;
          float y = static_cast<float>(v);
          if (use_alpha && !(y > 0.f)) {
            y = alpha * y;
            npos += rs >= 0.0;
          }
          any_bad |= !isfinite(y);
          Y[int64_t(m) * ldy + n] = y;
        }
      }
    }
    if (flags) {
      if (__any_sync(0xffffffffu, any_bad) && lane == 0) atomicOr(&flags->nonfinite_output, 1);
      for (int o = 16; o; o >>= 1) npos += __shfl_xor_sync(0xffffffffu, npos, o);
      if (lane == 0 && npos)
        atomicAdd(reinterpret_cast<unsigned long long*>(&flags->nonpositive_outputs), npos);
    }
    tc_fence_before();
  }
  __syncwarp();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
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

template <int MT, int STAGES>
static int launch_mma(const CUtensorMap& map, const uint32_t* tiles, const double* rscale, const float* bias,
                      float* Y, int64_t ldy, int64_t M, int64_t N, int64_t KC, int64_t M_pad, int64_t N_pad,
                      int use_alpha, float alpha, tg_device_flags* flags, cudaStream_t st) {
  using C = MmaCfg<MT, STAGES>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(tg_mma_kernel<MT, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(tg_mma_kernel)");
    attr_set = true;
  }
  dim3 grid(unsigned(N_pad / C::BN), unsigned(M_pad / MT));
  tg_mma_kernel<MT, STAGES><<<grid, 192, C::SMEM, st>>>(map, tiles, rscale, bias, Y, ldy, int(M), int(N),
                                                         int(KC), int(M_pad), int(N_pad), use_alpha, alpha,
                                                         flags);
  return check_launch("tg_mma_kernel");
}

int mma_pick_mt(int64_t M) {
  if (M <= 16) return 16;
  if (M <= 32) return 32;
  return 64;
}

struct SplitLayout {
  int64_t mt, M_pad, K_pad;
  size_t off_rscale, off_wide, total;
};

static SplitLayout split_layout(int64_t M, int64_t K) {
  SplitLayout L;
  L.mt = mma_pick_mt(M);
  L.M_pad = round_up(M, L.mt);
  L.K_pad = round_up(K, 128);
  L.off_rscale = size_t(round_up(3 * L.M_pad * L.K_pad, 256));
  L.off_wide = L.off_rscale + size_t(round_up(L.M_pad * int64_t(sizeof(double)), 256));
  L.total = L.off_wide + size_t(round_up((L.M_pad + 1) * 4, 256));
  return L;
}

size_t xsplit_bytes(int64_t M, int64_t K) { return split_layout(M, K).total; }

const int32_t* wide_rows(void* ws, int64_t M, int64_t K) {
  return reinterpret_cast<const int32_t*>(static_cast<uint8_t*>(ws) + split_layout(M, K).off_wide);
}

int run_xsplit(const float* X, int64_t M, int64_t K, int64_t ldx, void* ws, size_t ws_bytes, tg_device_flags* flags,
               cudaStream_t st) {
  const SplitLayout L = split_layout(M, K);
  if (ws_bytes < L.total) return set_error(TG_ERR_PARAM, "workspace too small for X split");
  uint8_t* base = static_cast<uint8_t*>(ws);
  int8_t* limbs = reinterpret_cast<int8_t*>(base);
  double* rscale = reinterpret_cast<double*>(base + L.off_rscale);
  int32_t* wide = reinterpret_cast<int32_t*>(base + L.off_wide);
  cudaError_t e = cudaMemsetAsync(wide, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaMemsetAsync(wide rows)");
  tg_xsplit_kernel<<<unsigned(L.M_pad), 256, 0, st>>>(X, M, K, ldx, limbs, rscale, wide, L.M_pad, L.K_pad, flags);
  return check_launch("tg_xsplit_kernel");
}

int run_mma(int64_t M, int64_t K, const uint32_t* tiles, int64_t N, const float* bias, float* Y, int64_t ldy,
            int use_alpha, float alpha, void* ws, tg_device_flags* flags, cudaStream_t st) {
  const SplitLayout L = split_layout(M, K);
  const int64_t mt = L.mt, M_pad = L.M_pad, K_pad = L.K_pad;
  const int64_t N_pad = round_up(N, 128);
  const int64_t KC = K_pad / 128;
  int8_t* limbs = static_cast<int8_t*>(ws);
  double* rscale = reinterpret_cast<double*>(static_cast<uint8_t*>(ws) + L.off_rscale);

  auto enc = get_encode();
  if (!enc) return set_error(TG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap map;
  cuuint64_t gdim[2] = {cuuint64_t(K_pad), cuuint64_t(3 * M_pad)};
  cuuint64_t gstride[1] = {cuuint64_t(K_pad)};
  cuuint32_t box[2] = {128u, cuuint32_t(mt)};
  cuuint32_t estride[2] = {1u, 1u};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, limbs, gdim, gstride, box, estride,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(TG_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  switch (mt) {
    case 16:
      return launch_mma<16, 6>(map, tiles, rscale, bias, Y, ldy, M, N, KC, M_pad, N_pad, use_alpha, alpha,
                               flags, st);
    case 32:
      return launch_mma<32, 5>(map, tiles, rscale, bias, Y, ldy, M, N, KC, M_pad, N_pad, use_alpha, alpha,
                               flags, st);
    default:
      return launch_mma<64, 4>(map, tiles, rscale, bias, Y, ldy, M, N, KC, M_pad, N_pad, use_alpha, alpha,
                               flags, st);
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
