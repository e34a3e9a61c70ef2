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
#include "tg_walk.cuh"

namespace tg {

constexpr int G_WARPS = 8;    // columns per CTA
constexpr int G_ROWS = 128;   // rows per CTA (4 per lane)

size_t gather_ws_bytes(int64_t M, int64_t K) {
  return size_t(K + 1) * size_t(round_up(M, G_ROWS)) * sizeof(float) + 256;
}

// X (M x ldx) -> Xt ((K+1) x M_pad), zero padded; columns k < Kx are read from X (Kx = K + 1
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
    if (k <= K && m < M_pad) Xt[k * M_pad + m] = tile[threadIdx.x][r];
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
  dim3 grid(unsigned(ceil_div(ga.N, G_WARPS)), unsigned(M_pad / G_ROWS));
#define TG_GATHER_LAUNCH(V) \
  tg_gather_kernel<V><<<grid, G_WARPS * 32, 0, st>>>(Xt, M_pad, M, ga, bias, Y, ldy, use_alpha, alpha, flags)
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
               tg_device_flags* flags, cudaStream_t st) {
  GatherArgs ga{p0, i0, p1, i1, N, nblocks, m_full, g, uf, nullptr, 0};
  return run_gather_args(variant, X, M, K, ldx, ga, bias, Y, ldy, use_alpha, alpha, ws, flags, st);
}

}  // namespace tg
