// tg_walk.cuh — exact-order evaluation of one output column over the
// reference's own index streams.  Shared by the CUDA-core gather kernels
// (tg_gather.cu) and the wide-row fix-up inside the tensor-core epilogue
// (tg_mma.cu).  Every function reproduces the fp32 operation order of the
// reference kernel it names, so results are bit-identical to it:
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
//   VAR_VERTICAL  kernels/simd.py:98-188     p, q = run sums of the symmetric stream by run parity
//                 (t//g)&1; out = (b + p) - q
//   VAR_HORIZONTAL kernels/simd.py:196-274   a[t%4] +/-= x (sign (t//g)&1); out = b + ((a0+a1)+(a2+a3))
//   VAR_COMPRESSED kernels/scalar.py:561-602 codes in order, base-3 digits low first (2: +x, 0: -x);
//                 out = b + acc
#pragma once
#include <cstdint>

namespace tg {

enum {
  VAR_BASE = 0,
  VAR_BLOCKED = 1,
  VAR_IB = 2,
  VAR_OPTIMAL = 3,
  VAR_UNROLLED = 4,
  VAR_VERTICAL = 5,
  VAR_HORIZONTAL = 6,
  VAR_COMPRESSED = 7
};

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

// Eight rows of one column (the shared-memory slab kernel's register tile).
struct F8 {
  float4 a, b;
};
__device__ __forceinline__ void add_(F8& x, const F8 y) { add_(x.a, y.a); add_(x.b, y.b); }
__device__ __forceinline__ void sub_(F8& x, const F8 y) { sub_(x.a, y.a); sub_(x.b, y.b); }
template <> __device__ __forceinline__ F8 zero_<F8>() { return F8{zero_<float4>(), zero_<float4>()}; }
template <> __device__ __forceinline__ F8 splat_<F8>(float b) { return F8{splat_<float4>(b), splat_<float4>(b)}; }
__device__ __forceinline__ F8 badd_(float b, F8 a) { return F8{badd_(b, a.a), badd_(b, a.b)}; }

// out += (row r banked ? tot : acc), per component (blocked kernel, scalar.py:350-358)
__device__ __forceinline__ void add_sel_(float& o, float t, float a, unsigned bk) { o += (bk & 1u) ? t : a; }
__device__ __forceinline__ void add_sel_(float4& o, const float4 t, const float4 a, unsigned bk) {
  o.x += (bk & 1u) ? t.x : a.x;
  o.y += (bk & 2u) ? t.y : a.y;
  o.z += (bk & 4u) ? t.z : a.z;
  o.w += (bk & 8u) ? t.w : a.w;
}
__device__ __forceinline__ void add_sel_(F8& o, const F8 t, const F8 a, unsigned bk) {
  add_sel_(o.a, t.a, a.a, bk);
  add_sel_(o.b, t.b, a.b, bk >> 4);
}
template <typename V> __device__ __forceinline__ constexpr unsigned lanes_all_() { return (1u << (sizeof(V) / 4)) - 1u; }

// Operand sources: the value X[., k] for a stream index k.
struct SrcXt {  // 4 consecutive rows from the transposed copy Xt[K+1][M_pad]
  using V = float4;
  const float* xt;
  int64_t ld;
  __device__ __forceinline__ float4 operator()(int32_t k) const { return ld4(xt + int64_t(k) * ld); }
};
struct SrcRow {  // one row of X in place; the padded slot k = K reads as the exact zero it holds
  using V = float;  // (simd.py:72-75), so the row needs no slot column (a contiguous [M, K] X works)
  const float* x;
  int32_t K;
  __device__ __forceinline__ float operator()(int32_t k) const { return k < K ? __ldg(x + k) : 0.f; }
};
// Walk [a, b) of an index stream adding (NEG=false) or subtracting into acc,
// strictly in stream order.
template <bool NEG, typename S>
__device__ __forceinline__ void walk(typename S::V& acc, const int32_t* __restrict__ idx, int32_t a, int32_t b,
                                     const S& src) {
  int32_t i = a;
  // head up to a 16-byte boundary, then 128-bit index loads
  for (; i < b && (reinterpret_cast<uintptr_t>(idx + i) & 15u); ++i) {
    const typename S::V v = src(__ldg(idx + i));
    if (NEG) sub_(acc, v); else add_(acc, v);
  }
  for (; i + 4 <= b; i += 4) {
    const int4 k = __ldg(reinterpret_cast<const int4*>(idx + i));
    const typename S::V v0 = src(k.x), v1 = src(k.y), v2 = src(k.z), v3 = src(k.w);
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
  const int32_t* p0;  // col_start_pos (TCSC / blocked), col_segment_ptr (interleaved) or col_ptr (symmetric)
  const int32_t* i0;  // row_index_pos, all_indices or indices (symmetric)
  const int32_t* p1;  // col_start_neg
  const int32_t* i1;  // row_index_neg
  int64_t N, nblocks, m_full;
  int g, uf;
  const uint8_t* codes;  // compressed: N x G packed base-3 codes
  int64_t G;
  int64_t B = 0;  // block size in k (blocked / interleaved formats); 0 = one block over all of K
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
  } else if (VAR == VAR_VERTICAL) {
    const int32_t s = __ldg(a.p0 + n), len = __ldg(a.p0 + n + 1) - s;
    V p = zero_<V>(), q = zero_<V>();
    for (int32_t t = 0; t < len; ++t) {
      const V v = src(__ldg(a.i0 + s + t));
      if (((t / a.g) & 1) == 0) add_(p, v);
      else add_(q, v);
    }
    V out = badd_(b, p);
    sub_(out, q);
    return out;
  } else if (VAR == VAR_HORIZONTAL) {
    const int32_t s = __ldg(a.p0 + n), e = __ldg(a.p0 + n + 1);
    V a0 = zero_<V>(), a1 = zero_<V>(), a2 = zero_<V>(), a3 = zero_<V>();
    for (int32_t w = s; w < e; w += 4) {
      const int32_t t = w - s;
      const V v0 = src(__ldg(a.i0 + w)), v1 = src(__ldg(a.i0 + w + 1));
      const V v2 = src(__ldg(a.i0 + w + 2)), v3 = src(__ldg(a.i0 + w + 3));
      if (((t / a.g) & 1) == 0) add_(a0, v0); else sub_(a0, v0);
      if ((((t + 1) / a.g) & 1) == 0) add_(a1, v1); else sub_(a1, v1);
      if ((((t + 2) / a.g) & 1) == 0) add_(a2, v2); else sub_(a2, v2);
      if ((((t + 3) / a.g) & 1) == 0) add_(a3, v3); else sub_(a3, v3);
    }
    add_(a0, a1);
    add_(a2, a3);
    add_(a0, a2);
    return badd_(b, a0);
  } else if (VAR == VAR_COMPRESSED) {
    V acc = zero_<V>();
    const uint8_t* c = a.codes + n * a.G;
    for (int64_t gi = 0; gi < a.G; ++gi) {
      int code = __ldg(c + gi);
      if (code == 121) continue;  // five zero digits: no operation (as the reference, which skips zeros)
#pragma unroll
      for (int t = 0; t < 5; ++t) {
        const int d = code % 3;
        code /= 3;
        if (d == 2) add_(acc, src(int32_t(5 * gi + t)));
        else if (d == 0) sub_(acc, src(int32_t(5 * gi + t)));
      }
    }
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
      if (banked_rows != lanes_all_<V>()) {
        walk<false>(acc, a.i0, ap, bp, src);
        walk<true>(acc, a.i1, an, bn, src);
      }
      add_sel_(out, tot, acc, banked_rows);
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

// Runtime dispatch of the one-row (SrcRow) evaluation, for the fix-up paths.  Out of line: the
// eight inlined walks are ~38 K SASS lines, which otherwise sit in the middle of the tensor-core
// kernel between its warp roles' hot loops (the fix-up is the rare, slow path anyway).
static __device__ __noinline__ float column_value_row(int var, const GatherArgs& a, int64_t n, float b, const float* xrow,
                                                  int32_t K, bool banked) {
  const SrcRow src{xrow, K};
  const unsigned br = banked ? 1u : 0u;
  switch (var) {
    case VAR_BASE: return column_value<VAR_BASE>(a, n, b, src, br);
    case VAR_UNROLLED: return column_value<VAR_UNROLLED>(a, n, b, src, br);
    case VAR_BLOCKED: return column_value<VAR_BLOCKED>(a, n, b, src, br);
    case VAR_IB: return column_value<VAR_IB>(a, n, b, src, br);
    case VAR_VERTICAL: return column_value<VAR_VERTICAL>(a, n, b, src, br);
    case VAR_HORIZONTAL: return column_value<VAR_HORIZONTAL>(a, n, b, src, br);
    case VAR_COMPRESSED: return column_value<VAR_COMPRESSED>(a, n, b, src, br);
    default: return column_value<VAR_OPTIMAL>(a, n, b, src, br);
  }
}

}  // namespace tg
