// tg_peak.cu — measured int8 tcgen05.mma rate of this GPU, the denominator of the tensor
// roofline that bench.py reports for tg_mma_kernel (which runs kind::i8 MMAs).
//
// One persistent CTA per SM; one elected thread issues back-to-back
// `tcgen05.mma.cta_group::1.kind::i8` of M=128 x N x K=32 into one TMEM accumulator (A from
// shared memory or from TMEM, B from shared memory, SWIZZLE_128B K-major), the K offset cycling
// through a 128-byte swizzle atom, one commit every 16 MMAs and at most two commits in flight.
// Operands are pseudo-random bytes (zeros draw less power, so they clock higher than real
// data under the power cap).  The host times the launches with CUDA events;
// ops = grid * iters * 16 * 2 * 128 * N * 32.  Not on any product path.
#include <cuda_runtime.h>

#include "tg_internal.h"
#include "tg_ptx.cuh"

namespace tg {
namespace {

constexpr int kPeakSmemA = 128 * 128;  // 128 rows x 128 k bytes
constexpr int kPeakSmemB = 256 * 128;  // up to 256 rows x 128 k bytes

template <int N, bool kATmem>
__global__ void __launch_bounds__(128, 1) tg_peak_i8_kernel(int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x / 32;
  // pseudo-random int8 operands: the tensor pipe's power (and so the clock under the 1 kW cap)
  // depends on operand switching, so zeros would measure an unreachable rate
  auto rnd = [](uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
  };
  for (int i = threadIdx.x; i < (kPeakSmemA + kPeakSmemB) / 16; i += blockDim.x) {
    const uint32_t s0 = (blockIdx.x * 65536u + i) * 4u;
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(rnd(s0), rnd(s0 + 1), rnd(s0 + 2), rnd(s0 + 3));
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(&tmem_slot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_slot;
  if (kATmem && warp < 4) {
    // A operand columns [256, 288): 4 x (K = 32 int8 per lane as 8 x b32), pseudo-random.
    uint32_t z[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) z[i] = (threadIdx.x * 2654435761u) ^ (i * 0x9e3779b9u) ^ (blockIdx.x << 20);
    tmem_st32(tbase + ((warp * 32u) << 16) + 256u, z);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    const uint32_t leader = elect_one();
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + kPeakSmemA);
    constexpr uint32_t idesc = idesc_i8(128, N);
    uint32_t phase[2] = {0, 0};
    int commits = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t koff = (j & 3) * 32;
        const uint64_t db = smem_desc_k_sw128(sb + koff);
        const uint32_t acc = (it | j) ? 1u : 0u;
        if constexpr (kATmem) {
          mma_i8_tmem_a_warp(tbase, tbase + 256u + (j & 3) * 8u, db, idesc, acc, leader);
        } else {
          const uint64_t da = smem_desc_k_sw128(sa + koff);
          asm volatile(
              "{\n\t.reg .pred p, l;\n\t"
              "setp.ne.b32 p, %4, 0;\n\t"
              "setp.ne.b32 l, %5, 0;\n\t"
              "@l tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase),
              "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(leader)
              : "memory");
        }
      }
      const int s = commits & 1;
      if (commits >= 2) {  // keep at most two commit groups in flight
        mbar_wait(&bar[s], phase[s]);
        phase[s] ^= 1;
      }
      mma_commit_warp(&bar[s], leader);
      ++commits;
    }
    for (int c = commits > 2 ? commits - 2 : 0; c < commits; ++c) {
      const int s = c & 1;
      mbar_wait(&bar[s], phase[s]);
      phase[s] ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

template <int N, bool kATmem>
int launch_peak(int grid, int iters, cudaStream_t st) {
  auto k = tg_peak_i8_kernel<N, kATmem>;
  const int smem = kPeakSmemA + kPeakSmemB + 1024;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return set_cuda_error(e, "tg_probe_i8_mma_rate: smem attribute");
  k<<<grid, 128, smem, st>>>(iters);
  return check_launch("tg_probe_i8_mma_rate");
}

int launch_peak_n(int n, int a_tmem, int grid, int iters, cudaStream_t st) {
  if (a_tmem) {
    switch (n) {
      case 64: return launch_peak<64, true>(grid, iters, st);
      case 128: return launch_peak<128, true>(grid, iters, st);
      case 192: return launch_peak<192, true>(grid, iters, st);
      case 256: return launch_peak<256, true>(grid, iters, st);
    }
  } else {
    switch (n) {
      case 64: return launch_peak<64, false>(grid, iters, st);
      case 128: return launch_peak<128, false>(grid, iters, st);
      case 192: return launch_peak<192, false>(grid, iters, st);
      case 256: return launch_peak<256, false>(grid, iters, st);
    }
  }
  return set_error(TG_ERR_PARAM, "tg_probe_i8_mma_rate: n must be 64, 128, 192 or 256");
}

}  // namespace
}  // namespace tg

extern "C" int tg_probe_i8_mma_rate(int n, int a_in_tmem, int iters, int repeats, double* ops_per_s,
                                    double* seconds) {
  using namespace tg;
  if (!ops_per_s || iters <= 0 || repeats <= 0) return set_error(TG_ERR_PARAM, "tg_probe_i8_mma_rate: bad argument");
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return set_cuda_error(e, "tg_probe_i8_mma_rate: device query");
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if ((e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaEventCreate(&e0)) != cudaSuccess || (e = cudaEventCreate(&e1)) != cudaSuccess)
    return set_cuda_error(e, "tg_probe_i8_mma_rate: stream/event");
  int rc = launch_peak_n(n, a_in_tmem, sms, iters / 8 > 0 ? iters / 8 : 1, st);  // warm-up
  if (rc == 0) {
    cudaEventRecord(e0, st);
    for (int r = 0; r < repeats && rc == 0; ++r) rc = launch_peak_n(n, a_in_tmem, sms, iters, st);
    cudaEventRecord(e1, st);
  }
  if (rc == 0) {
    e = cudaEventSynchronize(e1);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
    if (e != cudaSuccess) {
      rc = set_cuda_error(e, "tg_probe_i8_mma_rate: timing");
    } else {
      const double ops = double(sms) * double(iters) * 16.0 * 2.0 * 128.0 * double(n) * 32.0 * double(repeats);
      *ops_per_s = ops / (double(ms) * 1e-3);
      if (seconds) *seconds = double(ms) * 1e-3;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(st);
  return rc;
}
