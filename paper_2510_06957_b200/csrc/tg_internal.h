// tg_internal.h — shared host-side helpers of the terngemm_b200 library.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>
#include <algorithm>

#include "../../include/terngemm_b200.h"

namespace tg {

int set_error(int code, const char* msg);
int set_cuda_error(cudaError_t e, const char* where);
int check_launch(const char* where);

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline int64_t ceil_div(int64_t x, int64_t m) { return (x + m - 1) / m; }

// tg_mma.cu
struct GatherArgs;  // tg_walk.cuh
int mma_pick_mt(int64_t M);
size_t xsplit_bytes(int64_t M, int64_t K);
bool xsplit_single_read(int64_t K);
int xsplit_row_stats(const void* ws, int64_t M, int64_t K, int64_t* stats, cudaStream_t st);
size_t mma_ws_bytes(int64_t M, int64_t K, int64_t N, int share = 1);
int run_xsplit(const float* X, int64_t M, int64_t K, int64_t ldx, void* ws, size_t ws_bytes, tg_device_flags* flags,
               cudaStream_t st);
int run_pack_dense(const int8_t* W, int64_t K, int64_t N, int64_t ldw, uint32_t* tiles, tg_device_flags* flags,
                   cudaStream_t st);
int run_pack_csc(const int32_t* col_start, const int32_t* rows, int64_t N, int64_t nblocks, bool neg,
                 uint32_t* tiles, int64_t K, tg_device_flags* flags, cudaStream_t st);
int run_pack_ib(const int32_t* ai, const int32_t* ptr, int64_t N, int64_t nblocks, int g, int64_t K,
                uint32_t* tiles, tg_device_flags* flags, cudaStream_t st);

// tg_peer.cu
int run_peer_wait(uint32_t* sig, int world, cudaStream_t st);

int run_unpack_dense(const uint32_t* tiles, int64_t K, int64_t N, int8_t* W, cudaStream_t st);
int run_rows_plane(uint32_t* tiles, int64_t K, int64_t N, cudaStream_t st);

// tg_gather.cu
enum { GATHER_BASE = 0, GATHER_BLOCKED = 1, GATHER_IB = 2, GATHER_OPTIMAL = 3, GATHER_UNROLLED = 4 };
size_t gather_ws_bytes(int64_t M, int64_t K);
int run_gather(int variant, const float* X, int64_t M, int64_t K, int64_t ldx, const int32_t* p0, const int32_t* i0,
               const int32_t* p1, const int32_t* i1, int64_t nblocks, int g, int uf, int64_t m_full, int64_t N,
               const float* bias, float* Y, int64_t ldy, int use_alpha, float alpha, void* ws,
               tg_device_flags* flags, cudaStream_t st, int64_t B = 0);


}  // namespace tg

#include "tg_walk.cuh"

namespace tg {
// Exact-order recomputation of wide rows inside the tensor-core epilogue.
struct MmaFixup {
  int var;          // VAR_* of tg_walk.cuh
  int64_t m_full;   // blocked: rows below take the banked order
  GatherArgs args;
};
int run_gather_args(int variant, const float* X, int64_t M, int64_t K, int64_t ldx, const GatherArgs& ga,
                    const float* bias, float* Y, int64_t ldy, int use_alpha, float alpha, void* ws,
                    tg_device_flags* flags, cudaStream_t st);
int run_pack_sym(const int32_t* idx, const int32_t* ptr, int64_t N, int g, int64_t K, uint32_t* tiles,
                 tg_device_flags* flags, cudaStream_t st);
int run_pack_codes(const uint8_t* codes, int64_t K, int64_t N, uint32_t* tiles, cudaStream_t st);
int run_mma(const float* X, int64_t M, int64_t K, int64_t ldx, const uint32_t* tiles, int64_t N, const float* bias,
            float* Y, int64_t ldy, int use_alpha, float alpha, const MmaFixup* fix, void* ws, size_t ws_bytes,
            tg_device_flags* flags, cudaStream_t st, const tg_peer_scatter* sc = nullptr, int share = 1,
            float* yh = nullptr, int64_t ldyh = 0);
}  // namespace tg
