/*
 * terngemm_b200.h — C ABI of the B200-native sparse ternary GEMM
 *                   Y = X W + b  (optionally PReLU), W in {-1, 0, +1}^{K x N}.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `terngemm` (/root/reference/pkg/src/terngemm).  Every entry point below names
 * the reference function it replaces (file:line, relative to
 * /root/reference/pkg/src/terngemm).  The reference is Python; the binding a
 * maintainer would add is a ctypes stub (INTEGRATION.md shows it).
 *
 * Conventions
 *   - All array pointers are DEVICE pointers (cudaMalloc / torch CUDA storage),
 *     except `tg_sizes*` / `int64_t*` outputs documented as host.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Calls are stream-ordered and asynchronous unless documented otherwise.
 *   - Index arrays are int32, exactly the reference layouts (tcsc.py:1-14,
 *     variants.py:86-101, variants.py:251-263).  Dense matrices are row-major
 *     with an explicit leading dimension (elements).
 *   - Every function returns a tg_status; the message of the last failure on
 *     the calling thread is available from tg_last_error().  Preconditions are
 *     checked before any launch (dimension mismatches -> TG_ERR_PARAM, the
 *     reference's ParameterError; inconsistent sparse structure ->
 *     TG_ERR_CORRUPT, the reference's CorruptionError).
 *   - There is no CPU fallback: without a usable sm_100a device every compute
 *     entry point fails with TG_ERR_CUDA.
 */
#ifndef TERNGEMM_B200_H
#define TERNGEMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TG_ABI_VERSION 5

typedef enum {
  TG_OK = 0,
  TG_ERR_PARAM = 1,       /* errors.py:4   ParameterError   */
  TG_ERR_CORRUPT = 2,     /* errors.py:8   CorruptionError  */
  TG_ERR_CUDA = 3,        /* CUDA runtime / launch failure   */
  TG_ERR_UNSUPPORTED = 4, /* device is not sm_100            */
  TG_ERR_OVERFLOW = 5     /* an index array would exceed int32 (tcsc.py:24 INDEX_DTYPE) */
} tg_status;

/* Format kinds for the two-phase builder. */
#define TG_FMT_TCSC 0                /* tcsc.py:35 Tcsc                      */
#define TG_FMT_BLOCKED 1             /* variants.py:86 BlockedTcsc           */
#define TG_FMT_INTERLEAVED_BLOCKED 2 /* variants.py:251 InterleavedBlockedTcsc */
#define TG_FMT_SYMMETRIC 3           /* variants.py:540 SymmetricInterleavedTcsc */

/* Orders of the interleaved-blocked gather kernel. */
#define TG_ORDER_INTERLEAVED_BLOCKED 0 /* kernels/scalar.py:397-485 */
#define TG_ORDER_VECTORIZED_OPTIMAL 1  /* kernels/simd.py:282-420   */

/* Device-side status words, written by kernels (optional, may be NULL). */
typedef struct {
  int32_t bad_input;           /* bit0: W entry outside {-1,0,1}; bit1: index out of range; bit2: non-finite X */
  int32_t nonfinite_output;    /* 1 if any produced Y entry is inf/nan (dense.py:77 DenseMatrix check) */
  uint64_t nonpositive_outputs;/* #(y <= 0) before PReLU: the reference's `mults` counter (simd.py:410-417) */
  int32_t corrupt;             /* bit0: duplicate (row, col); bit1: cell in both sign arrays (tcsc.py:95-114);
                                  bit2: a packed code >= 243 (variants.py:505-507, InvalidCodeError) */
  int32_t _pad;
} tg_device_flags;

/* Host-side sizes reported by the builder's count phase. */
typedef struct {
  int64_t nnz_pos;      /* len(row_index_pos)  (TCSC / blocked)              */
  int64_t nnz_neg;      /* len(row_index_neg)  (TCSC / blocked)              */
  int64_t n_indices;    /* len(all_indices)    (interleaved-blocked, incl. dummies) */
  int64_t num_blocks;   /* ceil(K / B)                                         */
  int64_t offsets_len;  /* elements of each offset table                        */
} tg_sizes;

/* ------------------------------------------------------------------ misc */
int tg_abi_version(void);
const char* tg_last_error(void);
/* 1 if device `dev` is a compute-capability 10.0 (sm_100) GPU this library can run on. */
int tg_device_supported(int dev);

/* ------------------------------------------------------------------ format construction
 * Two-phase device builder, bit-exact with the reference builders:
 *   tcsc.py:71-92           tcsc_from_dense(W)
 *   variants.py:146-178     blocked_from_dense(W, B)
 *   variants.py:312-350     interleaved_blocked_from_dense(W, B, g, symmetric_cols)
 * Phase 1 (tg_build_count) validates W (ParameterError for entries outside
 * {-1,0,+1}, dense.py:45-49), counts every (block, column) cell and returns
 * the output sizes; it synchronises `stream`.  Phase 2 (tg_build_fill_*)
 * writes the arrays, stream-ordered.  `ws` must hold
 * tg_build_workspace_bytes(K, N, B) bytes and stay untouched between phases.
 * B is the resolved block size (variants.py:38-42); use B = K for TCSC.     */
size_t tg_build_workspace_bytes(int64_t K, int64_t N, int64_t B);
int tg_build_count(const int8_t* W, int64_t K, int64_t N, int64_t ldw, int kind, int64_t B, int g,
                   int symmetric, void* ws, size_t ws_bytes, tg_sizes* sizes /* host */, void* stream);
int tg_build_fill_tcsc(const void* ws, int64_t K, int64_t N, int32_t* col_start_pos, int32_t* row_index_pos,
                       int32_t* col_start_neg, int32_t* row_index_neg, void* stream);
int tg_build_fill_blocked(const void* ws, int64_t K, int64_t N, int64_t B, int32_t* col_start_pos /* nb x (N+1) */,
                          int32_t* row_index_pos, int32_t* col_start_neg /* nb x (N+1) */, int32_t* row_index_neg,
                          void* stream);
int tg_build_fill_interleaved_blocked(const void* ws, int64_t K, int64_t N, int64_t B, int g, int symmetric,
                                      int32_t* all_indices, int32_t* col_segment_ptr /* 3*nb*N+1 */,
                                      void* stream);
/* variants.py:582-631 symmetric_from_dense(W, g): kind TG_FMT_SYMMETRIC in
 * tg_build_count (B ignored), then this fill; n_indices = sizes.n_indices. */
int tg_build_fill_symmetric(const void* ws, int64_t K, int64_t N, int g, int32_t* indices,
                            int32_t* col_ptr /* N+1 */, int64_t n_indices, void* stream);
/* variants.py:515-521 compressed_from_dense(W): codes is N x ceil(K/5) uint8
 * (column-major packed, 5 base-3 digits per byte).  Validates W; synchronises. */
int tg_build_compressed(const int8_t* W, int64_t K, int64_t N, int64_t ldw, uint8_t* codes, void* stream);
/* Sets flags->corrupt bit2 if any code is >= 243 (CompressedTcsc.__post_init__, variants.py:503-507). */
int tg_codes_check(const uint8_t* codes, int64_t count, tg_device_flags* flags, void* stream);

/* ------------------------------------------------------------------ ternary tiles
 * GPU-native re-encoding of any of the formats above for the dense-decode
 * tensor-core path: 2 bits per (k, n), grouped in 128-row x 1-column tiles.
 * Built from the format's own device arrays (never from a host copy).
 * Duplicate / overlapping entries set flags->corrupt (tcsc.py:105-113).
 * The buffer (tg_tiles_bytes) holds the column-major tile records the decoders
 * stream, then a row-major plane of the same 2-bit codes (16 columns per word)
 * from which the epilogue reads W[k, n] of a row's listed outlier entries.      */
size_t tg_tiles_bytes(int64_t K, int64_t N);
int tg_tiles_from_dense(const int8_t* W, int64_t K, int64_t N, int64_t ldw, uint32_t* tiles,
                        tg_device_flags* flags, void* stream);
int tg_tiles_from_tcsc(const int32_t* col_start_pos, const int32_t* row_index_pos, const int32_t* col_start_neg,
                       const int32_t* row_index_neg, int64_t K, int64_t N, uint32_t* tiles,
                       tg_device_flags* flags, void* stream);
int tg_tiles_from_blocked(const int32_t* col_start_pos, const int32_t* row_index_pos,
                          const int32_t* col_start_neg, const int32_t* row_index_neg, int64_t K, int64_t N,
                          int64_t B, uint32_t* tiles, tg_device_flags* flags, void* stream);
int tg_tiles_from_interleaved_blocked(const int32_t* all_indices, const int32_t* col_segment_ptr, int64_t K,
                                      int64_t N, int64_t B, int g, uint32_t* tiles, tg_device_flags* flags,
                                      void* stream);
int tg_tiles_from_symmetric(const int32_t* indices, const int32_t* col_ptr, int64_t K, int64_t N, int g,
                            uint32_t* tiles, tg_device_flags* flags, void* stream);
int tg_tiles_from_compressed(const uint8_t* codes, int64_t K, int64_t N, uint32_t* tiles, void* stream);
/* Decode tiles back to dense int8 W (K x N, ld = N): tcsc.py:95 tcsc_to_dense. */
int tg_tiles_to_dense(const uint32_t* tiles, int64_t K, int64_t N, int8_t* W, void* stream);

/* ------------------------------------------------------------------ GEMM
 * Workspace for any GEMM entry point below (X copies, limb split). */
size_t tg_gemm_workspace_bytes(int64_t M, int64_t K, int64_t N);

/* Gather path (CUDA cores, fp32 adds in the reference's own order, so the
 * output is bit-identical to the reference kernel for any finite X):
 *   gemm_base            kernels/scalar.py:109-148   (also `unrolled`, scalar.py:156-278)
 *   gemm_blocked         kernels/scalar.py:286-389
 *   gemm_interleaved_blocked / gemm_vectorized_optimal
 *                        kernels/scalar.py:397-511, kernels/simd.py:282-449
 * X is M x K (ldx >= K; an M x (K+1) PaddedInput, simd.py:40-75, passes ldx = K+1).
 * use_alpha/alpha fuse the PReLU epilogue (simd.py:410-417).                     */
/* uf = 0: gemm_base order (scalar.py:116-127); uf >= 1: gemm_unrolled's uf
 * accumulator banks (scalar.py:167-206; uf = 1 equals the base order).     */
int tg_gemm_tcsc(const float* X, int64_t M, int64_t K, int64_t ldx, const int32_t* col_start_pos,
                 const int32_t* row_index_pos, const int32_t* col_start_neg, const int32_t* row_index_neg,
                 int64_t N, const float* bias, float* Y, int64_t ldy, int uf, int use_alpha, float alpha, void* ws,
                 size_t ws_bytes, tg_device_flags* flags, void* stream);
/* uf, mr: gemm_blocked's banks for rows < floor(M/mr)*mr (scalar.py:296-358). */
int tg_gemm_blocked(const float* X, int64_t M, int64_t K, int64_t ldx, int64_t B, const int32_t* col_start_pos,
                    const int32_t* row_index_pos, const int32_t* col_start_neg, const int32_t* row_index_neg,
                    int64_t N, const float* bias, float* Y, int64_t ldy, int uf, int mr, int use_alpha, float alpha,
                    void* ws, size_t ws_bytes, tg_device_flags* flags, void* stream);
int tg_gemm_interleaved_blocked(const float* X, int64_t M, int64_t K, int64_t ldx, int64_t B, int g,
                                const int32_t* all_indices, const int32_t* col_segment_ptr, int64_t N,
                                const float* bias, float* Y, int64_t ldy, int order, int use_alpha, float alpha,
                                void* ws, size_t ws_bytes, tg_device_flags* flags, void* stream);
/* gemm_vertical (order 0, kernels/simd.py:98-188) and gemm_horizontal (order 1,
 * kernels/simd.py:196-274) over a SymmetricInterleavedTcsc; X padded (ldx = K+1). */
#define TG_ORDER_VERTICAL 0
#define TG_ORDER_HORIZONTAL 1
int tg_gemm_symmetric(const float* X, int64_t M, int64_t K, int64_t ldx, int g, const int32_t* indices,
                      const int32_t* col_ptr, int64_t N, const float* bias, float* Y, int64_t ldy, int order,
                      int use_alpha, float alpha, void* ws, size_t ws_bytes, tg_device_flags* flags, void* stream);
/* gemm_compressed, kernels/scalar.py:561-602 (codes N x ceil(K/5)). */
int tg_gemm_compressed(const float* X, int64_t M, int64_t K, int64_t ldx, const uint8_t* codes, int64_t N,
                       const float* bias, float* Y, int64_t ldy, void* ws, size_t ws_bytes, tg_device_flags* flags,
                       void* stream);

/* Reference kernel whose fp32 operation order a gather walk reproduces. */
#define TG_VARIANT_BASE 0               /* kernels/scalar.py:109-148 */
#define TG_VARIANT_BLOCKED 1            /* kernels/scalar.py:286-389 */
#define TG_VARIANT_INTERLEAVED_BLOCKED 2 /* kernels/scalar.py:397-511 */
#define TG_VARIANT_VECTORIZED_OPTIMAL 3 /* kernels/simd.py:282-449  */
#define TG_VARIANT_UNROLLED 4           /* kernels/scalar.py:156-278 */
#define TG_VARIANT_VERTICAL 5           /* kernels/simd.py:98-188    */
#define TG_VARIANT_HORIZONTAL 6         /* kernels/simd.py:196-274   */
#define TG_VARIANT_COMPRESSED 7         /* kernels/scalar.py:561-602 */

/* The format a tensor-core call was derived from, for the exact-order fix-up
 * of rows the fixed-point limbs cannot carry (see tg_gemm_tiles).
 *   BASE / UNROLLED: a0..a3 = col_start_pos, row_index_pos, col_start_neg, row_index_neg
 *   BLOCKED:         same four arrays of the blocked format, plus B
 *   INTERLEAVED_BLOCKED / VECTORIZED_OPTIMAL: a0 = col_segment_ptr, a1 = all_indices, B, g
 *   VERTICAL / HORIZONTAL: a0 = col_ptr, a1 = indices, g
 *   COMPRESSED:      codes */
typedef struct {
  int32_t variant;
  int32_t g;
  int32_t uf;
  int32_t mr;
  int64_t B;
  const int32_t* a0;
  const int32_t* a1;
  const int32_t* a2;
  const int32_t* a3;
  const uint8_t* codes;
} tg_format_ref;

/* Dense-decode tensor-core path.
 *   tg_gemm_tiles_prepare: every X row is scaled by a power of two so that
 *     max|x| < 2^22, rounded, and split into three exact int8 limbs (one launch).
 *   tg_gemm_tiles_run: tcgen05.mma.kind::i8 of the decoded ternary tiles against
 *     the limbs with exact int32 accumulation in TMEM; the epilogue recombines the
 *     limbs exactly, scales in fp64, adds the bias, rounds once to fp32 and
 *     applies PReLU.  Rows whose nonzero entries span more than a 16x
 *     max/rms dynamic range first shed their few large entries (at most 128 per
 *     row, e.g. LLM outlier channels): prepare lists them as (k, x) pairs, the limbs
 *     carry the rest at the rest's own scale, and the epilogue adds the listed
 *     terms from the packed tile words in fp32.  Rows that stay wide after that
 *     are recomputed in the reference's exact order from `exact` (inside the
 *     epilogue); with exact == NULL they keep the limb result.
 * Bit-exact with the reference for integer-valued X; otherwise the only
 * rounding is X's 22-bit per-row grid and one final rounding (~1e-7 normwise).
 * The tiles hold only real nonzeros: the symmetric formats' dummy indices
 * (index K) are dropped, which equals the reference only while a padded
 * input's slot X[:, K] is zero (the PaddedInput invariant, simd.py:40-70).
 * The gather entry points read the slot as the reference does.
 * tg_gemm_tiles = prepare + run.                                               */
int tg_gemm_tiles_prepare(const float* X, int64_t M, int64_t K, int64_t ldx, void* ws, size_t ws_bytes,
                          tg_device_flags* flags, void* stream);
/* Diagnostics of a prepared workspace (synchronises `stream`): stats[0] = rows left to the
 * exact-order walk, stats[1] = rows with listed outlier entries, stats[2] = listed entries. */
int tg_gemm_tiles_row_stats(const void* ws, size_t ws_bytes, int64_t M, int64_t K, int64_t* stats, void* stream);
int tg_gemm_tiles_run(const float* X, int64_t M, int64_t K, int64_t ldx, const uint32_t* tiles, int64_t N,
                      const float* bias, float* Y, int64_t ldy, int use_alpha, float alpha, const tg_format_ref* exact,
                      void* ws, size_t ws_bytes, tg_device_flags* flags, void* stream);
int tg_gemm_tiles(const float* X, int64_t M, int64_t K, int64_t ldx, const uint32_t* tiles, int64_t N,
                  const float* bias, float* Y, int64_t ldy, int use_alpha, float alpha, const tg_format_ref* exact,
                  void* ws, size_t ws_bytes, tg_device_flags* flags, void* stream);

/* Host-resident X and Y: the reference's own calling convention (numpy in,
 * numpy out, dense.py:67-90).  X rows are streamed in chunks of about 1-2 MB;
 * each chunk's host->device copy (2-D, into the device staging X_dev of row
 * pitch ldx_dev, whose columns K..ldx_dev-1 are zeroed: the padded input's
 * slot, simd.py:72-75), X split + tile GEMM, and device->host copy of its Y
 * rows (also left in Y_dev) are queued on one of the library's side streams,
 * so the two PCIe directions and the GEMMs overlap.  Stream-ordered with
 * respect to `stream` (forks from it and joins back).  Host buffers should be
 * pinned for the copies to be asynchronous.  Rows are independent and the
 * epilogue does not depend on the chunking: Y is bit-identical to
 * tg_gemm_tiles on the whole X.
 * When Y_host is pinned (device-mapped) and 16-byte aligned with a 16-byte row
 * pitch, the GEMM epilogue stores Y straight into it over PCIe and no D2H copy
 * is queued (TG_HOST_ZEROCOPY=0 restores the copies); Y_dev receives Y either way.
 * When X_host is pinned (device-mapped) and X is at most 4 MB, the X split
 * reads it in place over PCIe and no H2D copy is queued (X_dev is then not
 * written; TG_HOST_ZEROCOPY_X=0 / 1 forces the copies / the in-place read).
 * With flags_host != NULL the call owns the status words: it zeroes `flags`
 * first and copies them to flags_host (pinned) after the last chunk, so one
 * synchronisation of `stream` delivers Y and its status together.
 * A call whose arguments (every pointer and size) repeat an earlier call's is
 * replayed from a CUDA graph of that call: one launch instead of ~25 API calls
 * (TG_HOST_GRAPHS=0 disables it; a caller that is capturing `stream` itself
 * gets the plain enqueue).                                                     */
size_t tg_gemm_host_workspace_bytes(int64_t M, int64_t K, int64_t N);
int tg_gemm_tiles_host(const float* X_host, int64_t M, int64_t K, int64_t ldx_host, float* X_dev, int64_t ldx_dev,
                       const uint32_t* tiles, int64_t N, const float* bias, float* Y_dev, int64_t ldy_dev,
                       float* Y_host, int64_t ldy_host, int use_alpha, float alpha, const tg_format_ref* exact,
                       void* ws, size_t ws_bytes, tg_device_flags* flags, tg_device_flags* flags_host,
                       void* stream);

/* ---------------------------------------------------------------- peer scatter
 * Column-sharded GEMM whose epilogue writes every finished Y tile straight
 * into the full-width Y of every rank over NVLink (peer-mapped memory), so
 * the shard result never takes a separate all-gather (the north star's "one
 * NCCL all-gather" assembly, partition.py, fused into the producing kernel).
 *
 * Peer memory: each rank allocates one buffer with tg_peer_alloc (a 256-byte
 * signal header followed by its Y slots), exports it with tg_peer_export,
 * exchanges the 64-byte handles out of band (e.g. torch.distributed
 * all_gather_object) and maps the others with tg_peer_import.
 *
 * Signal header (uint32 words): [0, world) arrival counters, one per source
 * rank; TG_PEER_DONE_WORD: this rank's CTA completion counter;
 * TG_PEER_EPOCH_WORD: the epoch the last tg_peer_wait consumed.
 *
 * tg_gemm_tiles_run_scatter = tg_gemm_tiles_run with Y = this rank's block
 * (its columns col_off.. of its own full Y, row pitch ldy); every finished
 * tile is additionally stored at the same offset into y_peers[q] for q !=
 * rank; after the last tile of the grid the kernel adds 1 to word `rank` of
 * every rank's header (system-scope release).  tg_peer_wait (stream-ordered,
 * one tiny launch) returns once every rank's counter in this rank's header
 * has reached the next epoch: all shards of this step are then in local HBM.
 * With two Y slots used alternately, a rank cannot overwrite a peer's slot
 * before that peer has passed its previous wait.            */
#define TG_PEER_HEADER_BYTES 256
#define TG_PEER_MAX_WORLD 32
#define TG_PEER_DONE_WORD 32
#define TG_PEER_EPOCH_WORD 33
#define TG_PEER_TIMEOUT_WORD 34 /* set to 1 by a tg_peer_wait that gave up after ~10 s */
#define TG_PEER_HANDLE_BYTES 64

typedef struct {
  float* const* y_peers;      /* device array [world]: Y slot base (column 0, row 0) of every rank */
  uint32_t* const* sig_peers; /* device array [world]: signal header of every rank */
  uint32_t* sig_local;        /* this rank's header (== sig_peers[rank]) */
  int32_t world;
  int32_t rank;
  int64_t col_off;            /* first column of this rank's block in the full Y */
} tg_peer_scatter;

int tg_peer_alloc(size_t bytes, void** ptr);               /* zeroed, cudaIpc-exportable */
int tg_peer_free(void* ptr);
int tg_peer_export(void* ptr, void* handle /* TG_PEER_HANDLE_BYTES */);
int tg_peer_import(const void* handle, void** ptr);        /* maps a peer's buffer */
int tg_peer_release(void* ptr);                             /* unmaps an imported buffer */
int tg_peer_wait(uint32_t* sig_local, int world, void* stream);
int tg_gemm_tiles_run_scatter(const float* X, int64_t M, int64_t K, int64_t ldx, const uint32_t* tiles,
                              int64_t N, const float* bias, float* Y, int64_t ldy, int use_alpha, float alpha,
                              const tg_format_ref* exact, const tg_peer_scatter* scatter, void* ws,
                              size_t ws_bytes, tg_device_flags* flags, void* stream);

/* ------------------------------------------------------------------ measurement probe
 * Not on the GEMM path: the measured int8 tcgen05.mma rate of the current device, the
 * denominator of bench.py's tensor roofline (tg_mma_kernel issues kind::i8 MMAs).  One
 * persistent CTA per SM issues back-to-back M=128 x n x K=32 MMAs (A in smem or, with
 * a_in_tmem, in TMEM as tg_mma_kernel does); `repeats` launches of `iters` x 16 MMAs per SM
 * are timed with CUDA events.  n in {64, 128, 192, 256}.  Synchronous.                      */
int tg_probe_i8_mma_rate(int n, int a_in_tmem, int iters, int repeats, double* ops_per_s /* host */,
                         double* seconds /* host, may be NULL */);

#ifdef __cplusplus
}
#endif
#endif /* TERNGEMM_B200_H */
