// tg_build.cu — placeholder (builder kernels land in the next step)
#include "tg_internal.h"
extern "C" {
size_t tg_build_workspace_bytes(int64_t, int64_t, int64_t) { return 0; }
int tg_build_count(const int8_t*, int64_t, int64_t, int64_t, int, int64_t, int, int, void*, size_t, tg_sizes*, void*) { return TG_ERR_UNSUPPORTED; }
int tg_build_fill_tcsc(const void*, int64_t, int64_t, int32_t*, int32_t*, int32_t*, int32_t*, void*) { return TG_ERR_UNSUPPORTED; }
int tg_build_fill_blocked(const void*, int64_t, int64_t, int64_t, int32_t*, int32_t*, int32_t*, int32_t*, void*) { return TG_ERR_UNSUPPORTED; }
int tg_build_fill_interleaved_blocked(const void*, int64_t, int64_t, int64_t, int, int, int32_t*, int32_t*, void*) { return TG_ERR_UNSUPPORTED; }
}
