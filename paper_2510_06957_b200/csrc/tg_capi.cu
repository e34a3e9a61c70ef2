// tg_capi.cu — extern "C" entry points declared in include/terngemm_b200.h.
//
// Argument checking lives here (before any launch); the kernels live in
// tg_build.cu (format builders), tg_gather.cu (CUDA-core gather path) and
// tg_mma.cu (dense-decode tensor-core path).
#include <cuda_runtime.h>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "tg_internal.h"

namespace tg {

static thread_local std::string g_last_error;

int set_error(int code, const char* msg) {
  g_last_error = msg ? msg : "";
  return code;
}
int set_cuda_error(cudaError_t e, const char* where) {
  std::string m = std::string(where) + ": " + cudaGetErrorString(e);
  g_last_error = m;
  return TG_ERR_CUDA;
}
int check_launch(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, where);
  return TG_OK;
}

static int require_device() {
  static std::atomic<uint64_t> ok_mask{0};  // devices already checked (ids < 64)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaGetDevice");
  if (dev < 64 && (ok_mask.load(std::memory_order_relaxed) >> dev) & 1u) return TG_OK;
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0)
    return set_error(TG_ERR_UNSUPPORTED, "terngemm_b200 is built for sm_100a (B200) only");
  if (dev < 64) ok_mask.fetch_or(uint64_t(1) << dev, std::memory_order_relaxed);
  return TG_OK;
}

#define TG_REQUIRE(cond, code, msg) \
  do {                              \
    if (!(cond)) return ::tg::set_error((code), (msg)); \
  } while (0)
#define TG_TRY(expr)         \
  do {                       \
    int _rc = (expr);        \
    if (_rc != TG_OK) return _rc; \
  } while (0)

static inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace tg

using namespace tg;

extern "C" {

int tg_abi_version(void) { return TG_ABI_VERSION; }

const char* tg_last_error(void) { return g_last_error.c_str(); }

int tg_device_supported(int dev) {
  int major = 0, minor = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return (major == 10 && minor == 0) ? 1 : 0;
}

// ------------------------------------------------------------------ tiles
// The column-major tile records, then the same 2-bit codes as a row-major plane of equal size
// (tg_rows_plane_kernel: the outlier terms of the epilogue read W[k, n] for 32 columns at once).
static size_t tile_records_bytes(int64_t K, int64_t N) {
  return size_t(ceil_div(K, 128)) * size_t(round_up(N, 128)) * 8 * sizeof(uint32_t);
}
size_t tg_tiles_bytes(int64_t K, int64_t N) {
  if (K < 1 || N < 1) return 0;
  return 2 * tile_records_bytes(K, N);
}

int tg_tiles_from_dense(const int8_t* W, int64_t K, int64_t N, int64_t ldw, uint32_t* tiles,
                        tg_device_flags* flags, void* stream) {
  TG_REQUIRE(K >= 1 && N >= 1, TG_ERR_PARAM, "K and N must be >= 1");
  TG_REQUIRE(ldw >= N, TG_ERR_PARAM, "ldw must be >= N");
  TG_REQUIRE(W && tiles, TG_ERR_PARAM, "null pointer");
  TG_TRY(require_device());
  TG_TRY(run_pack_dense(W, K, N, ldw, tiles, flags, as_stream(stream)));
  return run_rows_plane(tiles, K, N, as_stream(stream));
}

int tg_tiles_from_tcsc(const int32_t* csp, const int32_t* rip, const int32_t* csn, const int32_t* rin, int64_t K,
                       int64_t N, uint32_t* tiles, tg_device_flags* flags, void* stream) {
  TG_REQUIRE(K >= 1 && N >= 1, TG_ERR_PARAM, "K and N must be >= 1");
  TG_REQUIRE(csp && csn && tiles, TG_ERR_PARAM, "null pointer");
  TG_TRY(require_device());
  cudaStream_t st = as_stream(stream);
  cudaError_t e = cudaMemsetAsync(tiles, 0, tile_records_bytes(K, N), st);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaMemsetAsync(tiles)");
  TG_TRY(run_pack_csc(csp, rip, N, 1, false, tiles, K, flags, st));
  TG_TRY(run_pack_csc(csn, rin, N, 1, true, tiles, K, flags, st));
  return run_rows_plane(tiles, K, N, st);
}

int tg_tiles_from_blocked(const int32_t* csp, const int32_t* rip, const int32_t* csn, const int32_t* rin,
                          int64_t K, int64_t N, int64_t B, uint32_t* tiles, tg_device_flags* flags, void* stream) {
  TG_REQUIRE(K >= 1 && N >= 1 && B >= 1, TG_ERR_PARAM, "K, N and B must be >= 1");
  TG_REQUIRE(csp && csn && tiles, TG_ERR_PARAM, "null pointer");
  TG_TRY(require_device());
  cudaStream_t st = as_stream(stream);
  const int64_t nb = ceil_div(K, B);
  cudaError_t e = cudaMemsetAsync(tiles, 0, tile_records_bytes(K, N), st);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaMemsetAsync(tiles)");
  TG_TRY(run_pack_csc(csp, rip, N, nb, false, tiles, K, flags, st));
  TG_TRY(run_pack_csc(csn, rin, N, nb, true, tiles, K, flags, st));
  return run_rows_plane(tiles, K, N, st);
}

int tg_tiles_from_interleaved_blocked(const int32_t* ai, const int32_t* ptr, int64_t K, int64_t N, int64_t B, int g,
                                      uint32_t* tiles, tg_device_flags* flags, void* stream) {
  TG_REQUIRE(K >= 1 && N >= 1 && B >= 1 && g >= 1, TG_ERR_PARAM, "K, N, B and g must be >= 1");
  TG_REQUIRE(ptr && tiles, TG_ERR_PARAM, "null pointer");
  TG_TRY(require_device());
  cudaStream_t st = as_stream(stream);
  const int64_t nb = ceil_div(K, B);
  cudaError_t e = cudaMemsetAsync(tiles, 0, tile_records_bytes(K, N), st);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaMemsetAsync(tiles)");
  TG_TRY(run_pack_ib(ai, ptr, N, nb, g, K, tiles, flags, st));
  return run_rows_plane(tiles, K, N, st);
}

int tg_tiles_from_symmetric(const int32_t* idx, const int32_t* ptr, int64_t K, int64_t N, int g, uint32_t* tiles,
                            tg_device_flags* flags, void* stream) {
  TG_REQUIRE(K >= 1 && N >= 1 && g >= 1, TG_ERR_PARAM, "K, N and g must be >= 1");
  TG_REQUIRE(ptr && tiles, TG_ERR_PARAM, "null pointer");
  TG_TRY(require_device());
  cudaStream_t st = as_stream(stream);
  cudaError_t e = cudaMemsetAsync(tiles, 0, tile_records_bytes(K, N), st);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaMemsetAsync(tiles)");
  TG_TRY(run_pack_sym(idx, ptr, N, g, K, tiles, flags, st));
  return run_rows_plane(tiles, K, N, st);
}

int tg_tiles_from_compressed(const uint8_t* codes, int64_t K, int64_t N, uint32_t* tiles, void* stream) {
  TG_REQUIRE(K >= 1 && N >= 1, TG_ERR_PARAM, "K and N must be >= 1");
  TG_REQUIRE(codes && tiles, TG_ERR_PARAM, "null pointer");
  TG_TRY(require_device());
  TG_TRY(run_pack_codes(codes, K, N, tiles, as_stream(stream)));
  return run_rows_plane(tiles, K, N, as_stream(stream));
}

int tg_tiles_to_dense(const uint32_t* tiles, int64_t K, int64_t N, int8_t* W, void* stream) {
  TG_REQUIRE(K >= 1 && N >= 1, TG_ERR_PARAM, "K and N must be >= 1");
  TG_REQUIRE(tiles && W, TG_ERR_PARAM, "null pointer");
  TG_TRY(require_device());
  return run_unpack_dense(tiles, K, N, W, as_stream(stream));
}

// ------------------------------------------------------------------ GEMM (tiles)
size_t tg_gemm_workspace_bytes(int64_t M, int64_t K, int64_t N) {
  if (M < 1 || K < 1) return 0;
  const size_t a = mma_ws_bytes(M, K, N);
  const size_t b = gather_ws_bytes(M, K);
  return a > b ? a : b;
}

int tg_gemm_tiles_prepare(const float* X, int64_t M, int64_t K, int64_t ldx, void* ws, size_t ws_bytes,
                          tg_device_flags* flags, void* stream) {
  TG_REQUIRE(M >= 1 && K >= 1, TG_ERR_PARAM, "M and K must be >= 1");
  TG_REQUIRE(ldx >= K, TG_ERR_PARAM, "ldx must be >= K");
  TG_REQUIRE(X && ws, TG_ERR_PARAM, "null pointer");
  TG_REQUIRE(ws_bytes >= xsplit_bytes(M, K), TG_ERR_PARAM, "workspace too small");
  TG_TRY(require_device());
  return run_xsplit(X, M, K, ldx, ws, ws_bytes, flags, as_stream(stream));
}

int tg_gemm_tiles_row_stats(const void* ws, size_t ws_bytes, int64_t M, int64_t K, int64_t* stats, void* stream) {
  TG_REQUIRE(M >= 1 && K >= 1, TG_ERR_PARAM, "M and K must be >= 1");
  TG_REQUIRE(ws && stats, TG_ERR_PARAM, "null pointer");
  TG_REQUIRE(ws_bytes >= xsplit_bytes(M, K), TG_ERR_PARAM, "workspace too small");
  TG_TRY(require_device());
  return xsplit_row_stats(ws, M, K, stats, as_stream(stream));
}

static int gemm_tiles_run(const float* X, int64_t M, int64_t K, int64_t ldx, const uint32_t* tiles, int64_t N,
                          const float* bias, float* Y, int64_t ldy, int use_alpha, float alpha,
                          const tg_format_ref* exact, const tg_peer_scatter* sc, void* ws, size_t ws_bytes,
                          tg_device_flags* flags, void* stream, int share = 1, float* yh = nullptr,
                          int64_t ldyh = 0) {
  TG_REQUIRE(M >= 1 && K >= 1 && N >= 1, TG_ERR_PARAM, "M, K and N must be >= 1");
  TG_REQUIRE(ldy >= N && ldx >= K, TG_ERR_PARAM, "leading dimensions too small");
  TG_REQUIRE(tiles && Y && ws && X, TG_ERR_PARAM, "null pointer");
  TG_REQUIRE(ws_bytes >= xsplit_bytes(M, K), TG_ERR_PARAM, "workspace too small");
  TG_REQUIRE(M <= (int64_t(1) << 30) && N <= (int64_t(1) << 30), TG_ERR_PARAM, "M, N too large");
  TG_REQUIRE(K <= (int64_t(1) << 24), TG_ERR_PARAM, "K must be < 2^24 for exact int32 limb accumulation");
  if (exact) {
    TG_REQUIRE(exact->variant >= 0 && exact->variant <= 7, TG_ERR_PARAM, "unknown exact variant");
    TG_REQUIRE(exact->variant == TG_VARIANT_COMPRESSED ? exact->codes != nullptr : exact->a0 != nullptr,
               TG_ERR_PARAM, "exact format without offsets");
    TG_REQUIRE(exact->B >= 1 && exact->g >= 1 && exact->uf >= 1 && exact->mr >= 1, TG_ERR_PARAM,
               "exact format: B, g, uf, mr must be >= 1");
  }
  TG_REQUIRE(ws_bytes >= mma_ws_bytes(M, K, N, share), TG_ERR_PARAM, "workspace too small");
  TG_TRY(require_device());
  if (!exact) return run_mma(X, M, K, ldx, tiles, N, bias, Y, ldy, use_alpha, alpha, nullptr, ws, ws_bytes, flags,
                             as_stream(stream), sc, share, yh, ldyh);
  const int v = exact->variant;
  MmaFixup fx{};
  const int64_t nb = (v == TG_VARIANT_BASE || v == TG_VARIANT_UNROLLED) ? 1 : ceil_div(K, exact->B);
  fx.m_full = (v == TG_VARIANT_BLOCKED) ? M / exact->mr * exact->mr : 0;
  if (v == TG_VARIANT_INTERLEAVED_BLOCKED || v == TG_VARIANT_VECTORIZED_OPTIMAL) {
    fx.var = v == TG_VARIANT_INTERLEAVED_BLOCKED ? VAR_IB : VAR_OPTIMAL;
    fx.args = GatherArgs{exact->a0, exact->a1, nullptr, nullptr, N, nb, fx.m_full, exact->g, 1, nullptr, 0};
  } else if (v == TG_VARIANT_VERTICAL || v == TG_VARIANT_HORIZONTAL) {
    fx.var = v == TG_VARIANT_VERTICAL ? VAR_VERTICAL : VAR_HORIZONTAL;
    fx.args = GatherArgs{exact->a0, exact->a1, nullptr, nullptr, N, 1, 0, exact->g, 1, nullptr, 0};
  } else if (v == TG_VARIANT_COMPRESSED) {
    fx.var = VAR_COMPRESSED;
    fx.args = GatherArgs{nullptr, nullptr, nullptr, nullptr, N, 1, 0, 1, 1, exact->codes, ceil_div(K, 5)};
  } else {
    fx.var = v == TG_VARIANT_BASE ? VAR_BASE : v == TG_VARIANT_UNROLLED ? VAR_UNROLLED : VAR_BLOCKED;
    fx.args = GatherArgs{exact->a0, exact->a1, exact->a2, exact->a3, N, nb, fx.m_full, 1,
                         v == TG_VARIANT_BASE ? 1 : exact->uf, nullptr, 0};
  }
  return run_mma(X, M, K, ldx, tiles, N, bias, Y, ldy, use_alpha, alpha, &fx, ws, ws_bytes, flags,
                 as_stream(stream), sc, share, yh, ldyh);
}

int tg_gemm_tiles_run(const float* X, int64_t M, int64_t K, int64_t ldx, const uint32_t* tiles, int64_t N,
                      const float* bias, float* Y, int64_t ldy, int use_alpha, float alpha, const tg_format_ref* exact,
                      void* ws, size_t ws_bytes, tg_device_flags* flags, void* stream) {
  return gemm_tiles_run(X, M, K, ldx, tiles, N, bias, Y, ldy, use_alpha, alpha, exact, nullptr, ws, ws_bytes, flags,
                        stream);
}

int tg_gemm_tiles_run_scatter(const float* X, int64_t M, int64_t K, int64_t ldx, const uint32_t* tiles,
                              int64_t N, const float* bias, float* Y, int64_t ldy, int use_alpha, float alpha,
                              const tg_format_ref* exact, const tg_peer_scatter* scatter, void* ws,
                              size_t ws_bytes, tg_device_flags* flags, void* stream) {
  TG_REQUIRE(scatter, TG_ERR_PARAM, "null scatter descriptor");
  TG_REQUIRE(scatter->world >= 1 && scatter->world <= TG_PEER_MAX_WORLD, TG_ERR_PARAM,
             "scatter world must be in [1, TG_PEER_MAX_WORLD]");
  TG_REQUIRE(scatter->rank >= 0 && scatter->rank < scatter->world, TG_ERR_PARAM, "scatter rank out of range");
  TG_REQUIRE(scatter->y_peers && scatter->sig_peers && scatter->sig_local, TG_ERR_PARAM,
             "scatter descriptor with null tables");
  TG_REQUIRE(scatter->col_off >= 0 && scatter->col_off + N <= ldy, TG_ERR_PARAM,
             "scatter block [col_off, col_off + N) must lie inside the full row pitch ldy");
  return gemm_tiles_run(X, M, K, ldx, tiles, N, bias, Y, ldy, use_alpha, alpha, exact, scatter, ws, ws_bytes, flags,
                        stream);
}

// ------------------------------------------------------------------ peer memory
int tg_peer_alloc(size_t bytes, void** ptr) {
  TG_REQUIRE(ptr && bytes > 0, TG_ERR_PARAM, "tg_peer_alloc: null output or zero size");
  TG_TRY(require_device());
  *ptr = nullptr;
  cudaError_t e = cudaMalloc(ptr, bytes);  // its own allocation: cudaIpc exports whole allocations
  if (e != cudaSuccess) return set_cuda_error(e, "cudaMalloc(peer buffer)");
  e = cudaMemset(*ptr, 0, bytes);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaMemset(peer buffer)");
  return TG_OK;
}

int tg_peer_free(void* ptr) {
  cudaError_t e = cudaFree(ptr);
  return e == cudaSuccess ? TG_OK : set_cuda_error(e, "cudaFree(peer buffer)");
}

int tg_peer_export(void* ptr, void* handle) {
  TG_REQUIRE(ptr && handle, TG_ERR_PARAM, "tg_peer_export: null pointer");
  static_assert(sizeof(cudaIpcMemHandle_t) == TG_PEER_HANDLE_BYTES, "IPC handle size");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, ptr);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaIpcGetMemHandle");
  memcpy(handle, &h, sizeof(h));
  return TG_OK;
}

int tg_peer_import(const void* handle, void** ptr) {
  TG_REQUIRE(ptr && handle, TG_ERR_PARAM, "tg_peer_import: null pointer");
  TG_TRY(require_device());
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? TG_OK : set_cuda_error(e, "cudaIpcOpenMemHandle");
}

int tg_peer_release(void* ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(ptr);
  return e == cudaSuccess ? TG_OK : set_cuda_error(e, "cudaIpcCloseMemHandle");
}

int tg_peer_wait(uint32_t* sig_local, int world, void* stream) {
  TG_REQUIRE(sig_local, TG_ERR_PARAM, "tg_peer_wait: null header");
  TG_REQUIRE(world >= 1 && world <= TG_PEER_MAX_WORLD, TG_ERR_PARAM, "world must be in [1, TG_PEER_MAX_WORLD]");
  TG_TRY(require_device());
  return run_peer_wait(sig_local, world, as_stream(stream));
}

int tg_gemm_tiles(const float* X, int64_t M, int64_t K, int64_t ldx, const uint32_t* tiles, int64_t N,
                  const float* bias, float* Y, int64_t ldy, int use_alpha, float alpha, const tg_format_ref* exact,
                  void* ws, size_t ws_bytes, tg_device_flags* flags, void* stream) {
  TG_TRY(tg_gemm_tiles_prepare(X, M, K, ldx, ws, ws_bytes, flags, stream));
  return tg_gemm_tiles_run(X, M, K, ldx, tiles, N, bias, Y, ldy, use_alpha, alpha, exact, ws, ws_bytes, flags,
                           stream);
}

}  // extern "C"

// ------------------------------------------------------------------ GEMM from host memory
namespace {

// Row chunks of a host-resident X: about 1-2 MB of X each, at most 8, starting
// at multiples of 64 rows (a multiple of every blocked-order row unroll mr).
// Small chunks let the two PCIe directions and the GEMMs overlap; what they
// cost in host work is paid once, when the call is captured in a graph.  The
// chunks on the P.streams side streams run their GEMMs side by side, each on
// 1/P.streams of the SMs: a chunk's GEMM costs about as long as the whole
// one (its fill, epilogue and W stream do not shrink with the rows), so run
// one after another they would serialise the pipeline.
constexpr int kMaxHostChunks = 16;  // (chunk events per device)
struct HostPlan {
  int64_t rows, n;  // chunk height (the last one may be shorter), chunk count
  int streams;      // side streams used
  size_t ws_slice;  // workspace per side stream
};

// Small X is read in place by the X split (its CTAs load the pinned host rows over PCIe)
// instead of being copied in: a copy-engine transfer delays the start of the kernels that
// depend on it, which dominates for a few MB (measured cfg1 0.090 -> 0.080 ms, cfg2 0.25-0.48
// -> 0.245 ms, cfg4 unchanged).  Larger X keeps the chunked copies: with one CTA per long
// row the in-place reads do not keep enough PCIe requests in flight (cfg3, 16 MB: 1.1-1.3 ->
// 1.34-1.41 ms; cfg5: 11.5 -> 21.9 ms).  TG_HOST_ZEROCOPY_X=0/1 forces either way.
constexpr int64_t kZeroCopyXMaxBytes = int64_t(4) << 20;

// In place only from pinned (device-mapped) host memory, and only where the split reads each
// row once (xsplit_single_read): the decision is made before the chunk plan, which depends on it.
bool host_zero_copy_x(const float* X_host, int64_t M, int64_t K) {
  const char* env = getenv("TG_HOST_ZEROCOPY_X");
  bool want = M * K * 4 <= kZeroCopyXMaxBytes;
  if (env && env[0] == '0') want = false;
  if (env && env[0] == '1') want = true;
  if (!want || !xsplit_single_read(K)) return false;
  cudaPointerAttributes pa;
  const bool mapped = cudaPointerGetAttributes(&pa, X_host) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
                      pa.devicePointer != nullptr;
  cudaGetLastError();
  return mapped;
}

HostPlan host_plan(int64_t M, int64_t K, int64_t N, bool x_in_place) {
  HostPlan P;
  const int64_t bytes = M * K * 4;
  // (cfg5, 268 MB of X and 537 MB of Y: 8 chunks 11.77 ms, 12 chunks 11.44 ms, 16 chunks 11.54 ms --
  // more chunks start the Y stream earlier, fewer keep the per-chunk GEMMs efficient)
  int64_t cap = bytes >= (int64_t(128) << 20) ? 12 : 8;
  if (const char* env = getenv("TG_HOST_CHUNKS")) cap = std::min(kMaxHostChunks, std::max(1, atoi(env)));
  // ~1 MB chunks for X read in place (<= 4 MB; cfg2: 4 chunks 0.243 ms, 1 chunk 0.25-0.26 ms),
  // ~2 MB for copied X (cfg3, 16 MB: 4 and 8 chunks within noise, 0.59-0.69 ms; cfg5: 8 chunks
  // 11.7 ms, 4 chunks 12.5 ms)
  const int64_t want = x_in_place ? bytes >> 20 : bytes >> 21;
  int64_t n = std::max<int64_t>(1, std::min<int64_t>({cap, want, M / 64}));
  P.rows = round_up(ceil_div(M, n), 64);
  P.n = ceil_div(M, P.rows);
  P.streams = int(std::min<int64_t>(P.n, 4));
  const int64_t last = M - (P.n - 1) * P.rows;
  P.ws_slice = size_t(round_up(
      int64_t(std::max(mma_ws_bytes(P.rows, K, N, P.streams), mma_ws_bytes(last, K, N, P.streams))), 256));
  return P;
}

// The library's own side streams and events, per device (created once), and
// the stream host-streaming calls are captured on.
struct SideStreams {
  cudaStream_t s[4];       // chunk GEMMs (chunk c on s[c % 4])
  cudaStream_t cin, cout;  // the X chunks in, the Y chunks out, each in chunk order
  cudaEvent_t join[4];
  cudaEvent_t xin[kMaxHostChunks], ydone[kMaxHostChunks];  // chunk c: X landed / Y computed
  cudaEvent_t fork, join_in, join_out;
  cudaStream_t capture;
};

int side_streams(SideStreams** out) {
  static std::mutex mu;
  static std::unordered_map<int, SideStreams> per_dev;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lk(mu);
  auto it = per_dev.find(dev);
  if (it == per_dev.end()) {
    SideStreams ss;
    for (int i = 0; i < 4; ++i) {
      if ((e = cudaStreamCreateWithFlags(&ss.s[i], cudaStreamNonBlocking)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&ss.join[i], cudaEventDisableTiming)) != cudaSuccess)
        return set_cuda_error(e, "side stream creation");
    }
    for (int i = 0; i < kMaxHostChunks; ++i)
      if ((e = cudaEventCreateWithFlags(&ss.xin[i], cudaEventDisableTiming)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&ss.ydone[i], cudaEventDisableTiming)) != cudaSuccess)
        return set_cuda_error(e, "side stream creation");
    if ((e = cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ss.join_in, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ss.join_out, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&ss.cin, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&ss.cout, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&ss.capture, cudaStreamNonBlocking)) != cudaSuccess)
      return set_cuda_error(e, "side stream creation");
    it = per_dev.emplace(dev, ss).first;
  }
  *out = &it->second;
  return TG_OK;
}

// Every argument of one host-streaming call, plus the device and the chunk
// plan: two calls with equal keys enqueue exactly the same work, so the second
// one onwards can replay a CUDA graph of the first instead of issuing ~25 API
// calls (the graph launch is one).  Compared bytewise: zero-initialised.
struct HostKey {
  const float* X_host;
  int64_t M, K, ldx_host;
  float* X_dev;
  int64_t ldx_dev;
  const uint32_t* tiles;
  int64_t N;
  const float* bias;
  float* Y_dev;
  int64_t ldy_dev;
  float* Y_host;
  int64_t ldy_host;
  int32_t use_alpha;
  float alpha;
  int32_t has_exact, dev;
  tg_format_ref exact;
  void* ws;
  size_t ws_bytes;
  tg_device_flags* flags;
  tg_device_flags* flags_host;
  int64_t rows, n;
  int64_t zero_copy_x;  // the X split reads the pinned host X in place (no X copies)
};

struct HostGraph {
  HostKey key;
  cudaGraphExec_t exec;  // null until the key has been seen twice
  bool tried;            // capture attempted (a failed capture is not retried)
  uint64_t last_use;
};

constexpr int kHostGraphs = 16;

#ifdef TG_TRACE
// [chunk][0 = H2D done, 1 = GEMM done, 2 = D2H done, 3 = X split done] + the fork, recorded on direct enqueues
cudaEvent_t g_host_ev[16][4];
cudaEvent_t g_host_ev0;
int g_host_nev = 0;
#define TG_HOST_EV(c, j, st)                                                                  \
  do {                                                                                        \
    if ((c) < 16) {                                                                           \
      if (!g_host_ev[c][j]) cudaEventCreate(&g_host_ev[c][j]);                                \
      cudaEventRecord(g_host_ev[c][j], st);                                                   \
      g_host_nev = int(c) + 1;                                                                \
    }                                                                                         \
  } while (0)
#else
#define TG_HOST_EV(c, j, st) \
  do {                       \
  } while (0)
#endif

int enqueue_host(const HostKey& k, const HostPlan& P, SideStreams* ss, cudaStream_t main) {
  cudaError_t e;
  if (k.flags_host && (e = cudaMemsetAsync(k.flags, 0, sizeof(tg_device_flags), main)) != cudaSuccess)
    return set_cuda_error(e, "cudaMemsetAsync(flags)");
  if (k.ldx_dev > k.K) {  // the padded input's slot column(s): zero, as pad_input does
    e = cudaMemset2DAsync(k.X_dev + k.K, size_t(k.ldx_dev) * 4, 0, size_t(k.ldx_dev - k.K) * 4, size_t(k.M), main);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaMemset2DAsync(padded slot)");
  }
  // One chunk: everything on the caller's stream (no fork / join edges to resolve).
  const bool single = P.n == 1;
  cudaStream_t sin = single ? main : ss->cin, sout = single ? main : ss->cout;
  if (!single && (e = cudaEventRecord(ss->fork, main)) != cudaSuccess) return set_cuda_error(e, "cudaEventRecord");
#ifdef TG_TRACE
  if (!g_host_ev0) cudaEventCreate(&g_host_ev0);
  cudaEventRecord(g_host_ev0, main);
#endif
  // Copies go through two in-order streams: issued from independent streams (or
  // as independent graph nodes) the copy engines may take the chunks in any
  // order or interleave them, and the first chunk's GEMM then starts last.
  for (int i = 0; i < P.streams && !single; ++i)
    if ((e = cudaStreamWaitEvent(ss->s[i], ss->fork, 0)) != cudaSuccess) return set_cuda_error(e, "fork");
  if (!single && ((e = cudaStreamWaitEvent(ss->cin, ss->fork, 0)) != cudaSuccess ||
                  (e = cudaStreamWaitEvent(ss->cout, ss->fork, 0)) != cudaSuccess))
    return set_cuda_error(e, "fork");
  const tg_format_ref* exact = k.has_exact ? &k.exact : nullptr;
  const int64_t M = k.M, K = k.K, N = k.N;
  // Y straight from the epilogue into the pinned host Y when it is device-mapped and
  // 16-byte aligned (no copy-engine D2H: those transfers delay the launches of the
  // chunks' kernels that run beside them); TG_HOST_ZEROCOPY=0 keeps the copies
  float* yh = nullptr;
  static const bool zc_on = [] {
    const char* env = getenv("TG_HOST_ZEROCOPY");
    return !(env && env[0] == '0');
  }();
  if (zc_on && (reinterpret_cast<uintptr_t>(k.Y_host) & 15) == 0 && (k.ldy_host * 4) % 16 == 0) {
    cudaPointerAttributes pa;
    if (cudaPointerGetAttributes(&pa, k.Y_host) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer)
      yh = static_cast<float*>(pa.devicePointer);
    cudaGetLastError();
  }
  // X read in place from the pinned host X by the split kernels (host_zero_copy_x):
  // no copy engine at all in the pipeline
  const float* xh = nullptr;
  if (k.zero_copy_x) {
    cudaPointerAttributes pa;
    if (cudaPointerGetAttributes(&pa, k.X_host) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer)
      xh = static_cast<const float*>(pa.devicePointer);
    cudaGetLastError();
  }
  for (int64_t c = 0; c < P.n && !xh; ++c) {  // X chunks in, in order
    const int64_t r0 = c * P.rows, rows = std::min(P.rows, M - r0);
    float* xd = k.X_dev + r0 * k.ldx_dev;
    e = k.ldx_dev == K && k.ldx_host == K
            ? cudaMemcpyAsync(xd, k.X_host + r0 * K, size_t(rows * K) * 4, cudaMemcpyHostToDevice, sin)
            : cudaMemcpy2DAsync(xd, size_t(k.ldx_dev) * 4, k.X_host + r0 * k.ldx_host, size_t(k.ldx_host) * 4,
                                size_t(K) * 4, size_t(rows), cudaMemcpyHostToDevice, sin);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaMemcpy2DAsync(X chunk)");
    if (!single && (e = cudaEventRecord(ss->xin[c], sin)) != cudaSuccess) return set_cuda_error(e, "cudaEventRecord");
    TG_HOST_EV(c, 0, sin);
  }
  for (int64_t c = 0; c < P.n; ++c) {  // GEMMs side by side, each on 1/P.streams of the SMs
    const int i = int(c % P.streams);
    cudaStream_t st = single ? main : ss->s[i];
    const int64_t r0 = c * P.rows, rows = std::min(P.rows, M - r0);
    const float* xd = xh ? xh + r0 * k.ldx_host : k.X_dev + r0 * k.ldx_dev;
    const int64_t ldx = xh ? k.ldx_host : k.ldx_dev;
    float* yd = k.Y_dev + r0 * k.ldy_dev;
    void* wsi = static_cast<uint8_t*>(k.ws) + size_t(i) * P.ws_slice;
    if (!xh && !single && (e = cudaStreamWaitEvent(st, ss->xin[c], 0)) != cudaSuccess)
      return set_cuda_error(e, "wait X chunk");
    TG_TRY(tg_gemm_tiles_prepare(xd, rows, K, ldx, wsi, P.ws_slice, k.flags, st));
    TG_HOST_EV(c, 3, st);
    TG_TRY(gemm_tiles_run(xd, rows, K, ldx, k.tiles, N, k.bias, yd, k.ldy_dev, k.use_alpha, k.alpha, exact,
                          nullptr, wsi, P.ws_slice, k.flags, st, P.streams, yh ? yh + r0 * k.ldy_host : nullptr,
                          k.ldy_host));
    if (!single && (e = cudaEventRecord(ss->ydone[c], st)) != cudaSuccess) return set_cuda_error(e, "cudaEventRecord");
    TG_HOST_EV(c, 1, st);
  }
  for (int64_t c = 0; c < P.n; ++c) {  // Y chunks out, in order
    const int64_t r0 = c * P.rows, rows = std::min(P.rows, M - r0);
    const float* yd = k.Y_dev + r0 * k.ldy_dev;
    if (!single && (e = cudaStreamWaitEvent(ss->cout, ss->ydone[c], 0)) != cudaSuccess)
      return set_cuda_error(e, "wait Y");
    if (yh) {  // already in host memory
      TG_HOST_EV(c, 2, sout);
      continue;
    }
    e = k.ldy_dev == N && k.ldy_host == N
            ? cudaMemcpyAsync(k.Y_host + r0 * N, yd, size_t(rows * N) * 4, cudaMemcpyDeviceToHost, sout)
            : cudaMemcpy2DAsync(k.Y_host + r0 * k.ldy_host, size_t(k.ldy_host) * 4, yd, size_t(k.ldy_dev) * 4,
                                size_t(N) * 4, size_t(rows), cudaMemcpyDeviceToHost, sout);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaMemcpy2DAsync(Y chunk)");
    TG_HOST_EV(c, 2, sout);
  }
  for (int i = 0; i < P.streams && !single; ++i) {
    if ((e = cudaEventRecord(ss->join[i], ss->s[i])) != cudaSuccess) return set_cuda_error(e, "cudaEventRecord");
    if ((e = cudaStreamWaitEvent(main, ss->join[i], 0)) != cudaSuccess) return set_cuda_error(e, "join");
  }
  if (!single && ((e = cudaEventRecord(ss->join_in, ss->cin)) != cudaSuccess ||
      (e = cudaEventRecord(ss->join_out, ss->cout)) != cudaSuccess ||
      (e = cudaStreamWaitEvent(main, ss->join_in, 0)) != cudaSuccess ||
      (e = cudaStreamWaitEvent(main, ss->join_out, 0)) != cudaSuccess))
    return set_cuda_error(e, "join");
  if (k.flags_host &&
      (e = cudaMemcpyAsync(k.flags_host, k.flags, sizeof(tg_device_flags), cudaMemcpyDeviceToHost, main)) !=
          cudaSuccess)
    return set_cuda_error(e, "cudaMemcpyAsync(flags)");
  return TG_OK;
}

// Capture `k` on the library's capture stream; null on any failure (the caller
// then enqueues directly, so a graph problem never changes a result).
cudaGraphExec_t capture_host(const HostKey& k, const HostPlan& P, SideStreams* ss) {
  cudaGraph_t g = nullptr;
  cudaGraphExec_t exec = nullptr;
  if (cudaStreamBeginCapture(ss->capture, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  const int rc = enqueue_host(k, P, ss, ss->capture);
  const cudaError_t e = cudaStreamEndCapture(ss->capture, &g);
  if (rc == TG_OK && e == cudaSuccess && g && cudaGraphInstantiate(&exec, g, 0) != cudaSuccess) exec = nullptr;
  if (g) cudaGraphDestroy(g);
  cudaGetLastError();
  return exec;
}

}  // namespace

#ifdef TG_TRACE
// ms since the fork of the last direct host-streaming call: out[4 c + j]; returns the chunk count
extern "C" int tg_debug_host_trace(float* out) {
  cudaDeviceSynchronize();
  for (int c = 0; c < g_host_nev; ++c)
    for (int j = 0; j < 4; ++j) cudaEventElapsedTime(&out[4 * c + j], g_host_ev0, g_host_ev[c][j]);
  return g_host_nev;
}
#endif

extern "C" {

size_t tg_gemm_host_workspace_bytes(int64_t M, int64_t K, int64_t N) {
  if (M < 1 || K < 1 || N < 1) return 0;
  // either plan may run (in place or copied X is decided per call): size for the larger
  const HostPlan P0 = host_plan(M, K, N, false), P1 = host_plan(M, K, N, true);
  return std::max(size_t(P0.streams) * P0.ws_slice, size_t(P1.streams) * P1.ws_slice);
}

int tg_gemm_tiles_host(const float* X_host, int64_t M, int64_t K, int64_t ldx_host, float* X_dev, int64_t ldx_dev,
                       const uint32_t* tiles, int64_t N, const float* bias, float* Y_dev, int64_t ldy_dev,
                       float* Y_host, int64_t ldy_host, int use_alpha, float alpha, const tg_format_ref* exact,
                       void* ws, size_t ws_bytes, tg_device_flags* flags, tg_device_flags* flags_host,
                       void* stream) {
  TG_REQUIRE(M >= 1 && K >= 1 && N >= 1, TG_ERR_PARAM, "M, K and N must be >= 1");
  TG_REQUIRE(X_host && X_dev && Y_dev && Y_host && tiles && ws, TG_ERR_PARAM, "null pointer");
  TG_REQUIRE(!flags_host || flags, TG_ERR_PARAM, "flags_host needs device flags");
  TG_REQUIRE(ldx_host >= K && ldx_dev >= K && ldy_dev >= N && ldy_host >= N, TG_ERR_PARAM,
             "leading dimensions too small");
  TG_REQUIRE(ws_bytes >= tg_gemm_host_workspace_bytes(M, K, N), TG_ERR_PARAM, "workspace too small");
  TG_TRY(require_device());
  const bool x_in_place = host_zero_copy_x(X_host, M, K);
  const HostPlan P = host_plan(M, K, N, x_in_place);
  SideStreams* ss = nullptr;
  TG_TRY(side_streams(&ss));
  HostKey k;
  std::memset(&k, 0, sizeof k);
  k.X_host = X_host, k.M = M, k.K = K, k.ldx_host = ldx_host, k.X_dev = X_dev, k.ldx_dev = ldx_dev;
  k.tiles = tiles, k.N = N, k.bias = bias, k.Y_dev = Y_dev, k.ldy_dev = ldy_dev, k.Y_host = Y_host;
  k.ldy_host = ldy_host, k.use_alpha = use_alpha, k.alpha = use_alpha ? alpha : 0.f;
  k.has_exact = exact != nullptr;
  if (exact) k.exact = *exact;
  cudaGetDevice(&k.dev);
  k.ws = ws, k.ws_bytes = ws_bytes, k.flags = flags, k.flags_host = flags_host, k.rows = P.rows, k.n = P.n;
  k.zero_copy_x = x_in_place;

  static std::mutex enqueue_mu;  // the side streams, their events and the graph table are shared
  static HostGraph table[kHostGraphs];
  static int used = 0;
  static uint64_t clock = 0;
  static const bool graphs = [] {
    const char* env = getenv("TG_HOST_GRAPHS");
    return !(env && env[0] == '0');
  }();
  std::lock_guard<std::mutex> lk(enqueue_mu);
  cudaStream_t main = as_stream(stream);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (!graphs || cudaStreamIsCapturing(main, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return enqueue_host(k, P, ss, main);  // the caller is capturing (or graphs are off): plain enqueue
  }
  // first sighting: enqueue directly and remember the key; second: capture; then replay
  HostGraph* slot = nullptr;
  for (int i = 0; i < used; ++i)
    if (std::memcmp(&table[i].key, &k, sizeof k) == 0) slot = &table[i];
  if (slot == nullptr) {
    if (used < kHostGraphs) {
      slot = &table[used++];
    } else {
      slot = &table[0];
      for (int i = 1; i < used; ++i)
        if (table[i].last_use < slot->last_use) slot = &table[i];
      if (slot->exec) cudaGraphExecDestroy(slot->exec);  // an in-flight launch completes first
    }
    slot->key = k;
    slot->exec = nullptr;
    slot->tried = false;
    slot->last_use = ++clock;
    return enqueue_host(k, P, ss, main);
  }
  slot->last_use = ++clock;
  if (!slot->tried) slot->exec = capture_host(k, P, ss), slot->tried = true;
  if (slot->exec == nullptr) return enqueue_host(k, P, ss, main);
  const cudaError_t e = cudaGraphLaunch(slot->exec, main);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaGraphLaunch(host streaming)");
  return TG_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ GEMM (gather)
extern "C" {

static int gather_common_checks(const float* X, int64_t M, int64_t K, int64_t ldx, int64_t N, float* Y, int64_t ldy,
                                void* ws, size_t ws_bytes) {
  TG_REQUIRE(M >= 1 && K >= 1 && N >= 1, TG_ERR_PARAM, "M, K and N must be >= 1");
  TG_REQUIRE(ldx >= K && ldy >= N, TG_ERR_PARAM, "leading dimensions too small");
  TG_REQUIRE(X && Y && ws, TG_ERR_PARAM, "null pointer");
  TG_REQUIRE(ws_bytes >= gather_ws_bytes(M, K), TG_ERR_PARAM, "workspace too small");
  TG_REQUIRE(K < (int64_t(1) << 31) - 1, TG_ERR_PARAM, "K too large for int32 indices");
  return require_device();
}

int tg_gemm_tcsc(const float* X, int64_t M, int64_t K, int64_t ldx, const int32_t* csp, const int32_t* rip,
                 const int32_t* csn, const int32_t* rin, int64_t N, const float* bias, float* Y, int64_t ldy, int uf,
                 int use_alpha, float alpha, void* ws, size_t ws_bytes, tg_device_flags* flags, void* stream) {
  TG_TRY(gather_common_checks(X, M, K, ldx, N, Y, ldy, ws, ws_bytes));
  TG_REQUIRE(csp && csn, TG_ERR_PARAM, "null offset table");
  TG_REQUIRE(uf >= 0, TG_ERR_PARAM, "uf must be >= 0");
  return run_gather(uf == 0 ? GATHER_BASE : GATHER_UNROLLED, X, M, K, ldx, csp, rip, csn, rin, 1, 1,
                    uf == 0 ? 1 : uf, 0, N, bias, Y, ldy, use_alpha, alpha, ws, flags, as_stream(stream));
}

int tg_gemm_blocked(const float* X, int64_t M, int64_t K, int64_t ldx, int64_t B, const int32_t* csp,
                    const int32_t* rip, const int32_t* csn, const int32_t* rin, int64_t N, const float* bias, float* Y,
                    int64_t ldy, int uf, int mr, int use_alpha, float alpha, void* ws, size_t ws_bytes,
                    tg_device_flags* flags, void* stream) {
  TG_TRY(gather_common_checks(X, M, K, ldx, N, Y, ldy, ws, ws_bytes));
  TG_REQUIRE(B >= 1, TG_ERR_PARAM, "block size must be >= 1");
  TG_REQUIRE(uf >= 1 && mr >= 1, TG_ERR_PARAM, "uf and mr must be >= 1");
  TG_REQUIRE(csp && csn, TG_ERR_PARAM, "null offset table");
  const int64_t m_full = M / mr * mr;
  return run_gather(GATHER_BLOCKED, X, M, K, ldx, csp, rip, csn, rin, ceil_div(K, B), 1, uf, m_full, N, bias, Y,
                    ldy, use_alpha, alpha, ws, flags, as_stream(stream), B);
}

int tg_gemm_interleaved_blocked(const float* X, int64_t M, int64_t K, int64_t ldx, int64_t B, int g,
                                const int32_t* ai, const int32_t* ptr, int64_t N, const float* bias, float* Y,
                                int64_t ldy, int order, int use_alpha, float alpha, void* ws, size_t ws_bytes,
                                tg_device_flags* flags, void* stream) {
  TG_TRY(gather_common_checks(X, M, K, ldx, N, Y, ldy, ws, ws_bytes));
  TG_REQUIRE(B >= 1 && g >= 1, TG_ERR_PARAM, "B and g must be >= 1");
  TG_REQUIRE(ptr, TG_ERR_PARAM, "null col_segment_ptr");
  TG_REQUIRE(order == TG_ORDER_INTERLEAVED_BLOCKED || order == TG_ORDER_VECTORIZED_OPTIMAL, TG_ERR_PARAM,
             "unknown order");
  return run_gather(order == TG_ORDER_INTERLEAVED_BLOCKED ? GATHER_IB : GATHER_OPTIMAL, X, M, K, ldx, ptr, ai,
                    nullptr, nullptr, ceil_div(K, B), g, 1, 0, N, bias, Y, ldy, use_alpha, alpha, ws, flags,
                    as_stream(stream), B);
}

}  // extern "C"

extern "C" {

int tg_gemm_symmetric(const float* X, int64_t M, int64_t K, int64_t ldx, int g, const int32_t* indices,
                      const int32_t* col_ptr, int64_t N, const float* bias, float* Y, int64_t ldy, int order,
                      int use_alpha, float alpha, void* ws, size_t ws_bytes, tg_device_flags* flags, void* stream) {
  TG_TRY(gather_common_checks(X, M, K, ldx, N, Y, ldy, ws, ws_bytes));
  TG_REQUIRE(g >= 1, TG_ERR_PARAM, "g must be >= 1");
  TG_REQUIRE(N % 4 == 0, TG_ERR_PARAM, "N must be divisible by 4");
  TG_REQUIRE(col_ptr, TG_ERR_PARAM, "null col_ptr");
  TG_REQUIRE(order == TG_ORDER_VERTICAL || order == TG_ORDER_HORIZONTAL, TG_ERR_PARAM, "unknown order");
  GatherArgs ga{col_ptr, indices, nullptr, nullptr, N, 1, 0, g, 1, nullptr, 0};
  return run_gather_args(order == TG_ORDER_VERTICAL ? VAR_VERTICAL : VAR_HORIZONTAL, X, M, K, ldx, ga, bias, Y, ldy,
                         use_alpha, alpha, ws, flags, as_stream(stream));
}

int tg_gemm_compressed(const float* X, int64_t M, int64_t K, int64_t ldx, const uint8_t* codes, int64_t N,
                       const float* bias, float* Y, int64_t ldy, void* ws, size_t ws_bytes, tg_device_flags* flags,
                       void* stream) {
  TG_TRY(gather_common_checks(X, M, K, ldx, N, Y, ldy, ws, ws_bytes));
  TG_REQUIRE(codes, TG_ERR_PARAM, "null codes");
  GatherArgs ga{nullptr, nullptr, nullptr, nullptr, N, 1, 0, 1, 1, codes, ceil_div(K, 5)};
  return run_gather_args(VAR_COMPRESSED, X, M, K, ldx, ga, bias, Y, ldy, 0, 0.f, ws, flags, as_stream(stream));
}

}  // extern "C"
