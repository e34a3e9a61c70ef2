// tg_peer.cu — completion wait of the fused column-shard scatter
// (tg_gemm_tiles_run_scatter, include/terngemm_b200.h "peer scatter").
//
// The producing GEMM kernel (tg_mma.cu) stores each finished Y tile into
// every rank's full Y over NVLink and, after its last CTA, adds 1 to word
// `rank` of every rank's signal header.  This kernel is the consumer side:
// stream-ordered, one warp, it waits until every source rank's counter in the
// local header has reached the next epoch, so any kernel queued after it on
// the same stream reads the complete Y from local HBM.  It replaces the
// north star's assembly all-gather (partition.py gather_columns).
#include <cuda_runtime.h>

#include "tg_internal.h"

namespace tg {

__global__ void __launch_bounds__(32) tg_peer_wait_kernel(uint32_t* sig, int world) {
  const int t = threadIdx.x;
  const uint32_t target = sig[TG_PEER_EPOCH_WORD] + 1u;  // only this kernel writes the epoch word
  bool ok = true;
  if (t < world) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(sig + t) : "memory");
      if (int(v - target) >= 0) break;
      unsigned long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (t1 - t0 > 10000000000ull) {  // ~10 s: a rank never arrived -- give up rather than hang the GPU
        ok = false;
        break;
      }
      __nanosleep(256);
    }
  }
  ok = __all_sync(0xffffffffu, ok);
  if (t == 0) {
    if (!ok) sig[TG_PEER_TIMEOUT_WORD] = 1u;
    sig[TG_PEER_EPOCH_WORD] = target;
  }
  __threadfence_system();
}

int run_peer_wait(uint32_t* sig, int world, cudaStream_t st) {
  tg_peer_wait_kernel<<<1, 32, 0, st>>>(sig, world);
  return check_launch("tg_peer_wait_kernel");
}

}  // namespace tg
