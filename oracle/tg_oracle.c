/*
 * tg_oracle.c — CPU restatement of the reference's hot path.  TEST
 * INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py, never by the product
 * package (which has no CPU path at all).
 *
 * Each function restates one reference routine (paths relative to
 * /root/reference/pkg/src/terngemm) and keeps its per-output fp32 operation
 * order, so results are bit-identical to the reference's numba kernels for any
 * finite input (checked against the tests/golden fixtures, generated from the
 * reference itself by tests/golden/make_golden.py).  Compiled with
 * -ffp-contract=off and without -ffast-math so every `+=`/`-=` is one IEEE
 * binary32 rounding, exactly as numba emits them.
 *
 * Kernels take an optional [n_lo, n_hi) column range so the harness can run
 * disjoint column ranges on several threads; output elements are independent,
 * so the result does not depend on the split.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int32_t i32;
typedef int64_t i64;

/* ------------------------------------------------------------------ formats */

/* tcsc.py:71-92 tcsc_from_dense: per sign, rows of each column in ascending
 * order, column by column; col_start = [0, cumsum(counts)].  Pass NULL index
 * arrays to obtain only the offsets (sizes) first. */
void tgo_tcsc_from_dense(const int8_t* W, i64 K, i64 N, i32* csp, i32* rip, i32* csn, i32* rin) {
  i64 p = 0, q = 0;
  csp[0] = 0;
  csn[0] = 0;
  for (i64 n = 0; n < N; ++n) {
    for (i64 k = 0; k < K; ++k) {
      const int8_t v = W[k * N + n];
      if (v == 1) {
        if (rip) rip[p] = (i32)k;
        ++p;
      } else if (v == -1) {
        if (rin) rin[q] = (i32)k;
        ++q;
      }
    }
    csp[n + 1] = (i32)p;
    csn[n + 1] = (i32)q;
  }
}

/* variants.py:146-178 blocked_from_dense: blocks of B rows; within a block the
 * TCSC of the sub-matrix with GLOBAL row indices; offset tables (nb, N+1)
 * whose row blk starts at the running total of earlier blocks. */
void tgo_blocked_from_dense(const int8_t* W, i64 K, i64 N, i64 B, i32* csp, i32* rip, i32* csn, i32* rin) {
  const i64 nb = (K + B - 1) / B;
  i64 p = 0, q = 0;
  for (i64 blk = 0; blk < nb; ++blk) {
    const i64 lo = blk * B, hi = (lo + B < K) ? lo + B : K;
    i32* cp = csp + blk * (N + 1);
    i32* cn = csn + blk * (N + 1);
    cp[0] = (i32)p;
    cn[0] = (i32)q;
    for (i64 n = 0; n < N; ++n) {
      for (i64 k = lo; k < hi; ++k) {
        const int8_t v = W[k * N + n];
        if (v == 1) {
          if (rip) rip[p] = (i32)k;
          ++p;
        } else if (v == -1) {
          if (rin) rin[q] = (i32)k;
          ++q;
        }
      }
      cp[n + 1] = (i32)p;
      cn[n + 1] = (i32)q;
    }
  }
}

/* variants.py:312-376 interleaved_blocked_from_dense.  Per cell (blk, n):
 * p positives and q negatives (ascending rows); r = g*floor(min(p,q)/g);
 * segment 0 = r of each sign as alternating runs of g (positives first),
 * then (symmetric) dummy index K up to the 4-column group's longest segment 0;
 * segment 1 = remaining positives; segment 2 = remaining negatives.
 * ptr has 3*nb*N+1 entries.  Returns len(all_indices); pass ai = NULL to size. */
i64 tgo_interleaved_blocked_from_dense(const int8_t* W, i64 K, i64 N, i64 B, int g, int sym, i32* ai, i32* ptr) {
  const i64 nb = (K + B - 1) / B;
  i32* pos = (i32*)malloc(sizeof(i32) * (size_t)(B > 0 ? B : 1));
  i32* neg = (i32*)malloc(sizeof(i32) * (size_t)(B > 0 ? B : 1));
  i64* seg0 = (i64*)malloc(sizeof(i64) * (size_t)N);
  i64 off = 0;
  ptr[0] = 0;
  for (i64 blk = 0; blk < nb; ++blk) {
    const i64 lo = blk * B, hi = (lo + B < K) ? lo + B : K;
    /* first pass: interleaved lengths for symmetric padding */
    for (i64 n = 0; n < N; ++n) {
      i64 p = 0, q = 0;
      for (i64 k = lo; k < hi; ++k) {
        const int8_t v = W[k * N + n];
        p += (v == 1);
        q += (v == -1);
      }
      const i64 m = p < q ? p : q;
      seg0[n] = 2 * (g * (m / g));
    }
    if (sym) {
      for (i64 n0 = 0; n0 < N; n0 += 4) {
        i64 t = 0;
        for (int c = 0; c < 4; ++c) t = seg0[n0 + c] > t ? seg0[n0 + c] : t;
        for (int c = 0; c < 4; ++c) seg0[n0 + c] = t;
      }
    }
    for (i64 n = 0; n < N; ++n) {
      i64 p = 0, q = 0;
      for (i64 k = lo; k < hi; ++k) {
        const int8_t v = W[k * N + n];
        if (v == 1) pos[p++] = (i32)k;
        else if (v == -1) neg[q++] = (i32)k;
      }
      const i64 m = p < q ? p : q;
      const i64 r = g * (m / g);
      const i64 cell = blk * N + n;
      /* interleaved runs */
      for (i64 run = 0; run < r / g; ++run) {
        for (int u = 0; u < g; ++u) {
          if (ai) ai[off] = pos[run * g + u];
          ++off;
        }
        for (int u = 0; u < g; ++u) {
          if (ai) ai[off] = neg[run * g + u];
          ++off;
        }
      }
      for (i64 d = 2 * r; d < seg0[n]; ++d) {
        if (ai) ai[off] = (i32)K;
        ++off;
      }
      ptr[3 * cell + 1] = (i32)off;
      for (i64 t = r; t < p; ++t) {
        if (ai) ai[off] = pos[t];
        ++off;
      }
      ptr[3 * cell + 2] = (i32)off;
      for (i64 t = r; t < q; ++t) {
        if (ai) ai[off] = neg[t];
        ++off;
      }
      ptr[3 * cell + 3] = (i32)off;
    }
  }
  free(pos);
  free(neg);
  free(seg0);
  return off;
}

/* variants.py:582-631 symmetric_from_dense.  One stream per column: runs of g
 * positives then g negatives (ascending rows), every stream of a 4-column group
 * holds `pairs` index pairs, pairs = the group's max(max(#pos, #neg)) rounded
 * up to lcm(4, g) (0 for an all-zero group); the deficit is padded with K.
 * col_ptr has N+1 entries.  Returns len(indices); pass idx = NULL to size. */
static i64 lcm4(i64 g) {
  i64 a = 4, b = g;
  while (b) {
    const i64 t = a % b;
    a = b;
    b = t;
  }
  return 4 / a * g;
}
i64 tgo_symmetric_from_dense(const int8_t* W, i64 K, i64 N, int g, i32* idx, i32* col_ptr) {
  const i64 quantum = lcm4(g);
  i32* pos = (i32*)malloc(sizeof(i32) * (size_t)(K > 0 ? K : 1));
  i32* neg = (i32*)malloc(sizeof(i32) * (size_t)(K > 0 ? K : 1));
  i64 off = 0;
  col_ptr[0] = 0;
  for (i64 n0 = 0; n0 < N; n0 += 4) {
    i64 need = 0;
    for (int c = 0; c < 4; ++c) {
      i64 p = 0, q = 0;
      for (i64 k = 0; k < K; ++k) {
        const int8_t v = W[k * N + n0 + c];
        p += (v == 1);
        q += (v == -1);
      }
      const i64 m = p > q ? p : q;
      need = m > need ? m : need;
    }
    const i64 pairs = need ? (need + quantum - 1) / quantum * quantum : 0;
    for (int c = 0; c < 4; ++c) {
      i64 p = 0, q = 0;
      for (i64 k = 0; k < K; ++k) {
        const int8_t v = W[k * N + n0 + c];
        if (v == 1) pos[p++] = (i32)k;
        else if (v == -1) neg[q++] = (i32)k;
      }
      for (i64 run = 0; run < pairs / g; ++run) {
        for (int u = 0; u < g; ++u) {
          const i64 t = run * g + u;
          if (idx) idx[off] = t < p ? pos[t] : (i32)K;
          ++off;
        }
        for (int u = 0; u < g; ++u) {
          const i64 t = run * g + u;
          if (idx) idx[off] = t < q ? neg[t] : (i32)K;
          ++off;
        }
      }
      col_ptr[n0 + c + 1] = (i32)off;
    }
  }
  free(pos);
  free(neg);
  return off;
}

/* variants.py:451-532 compressed_from_dense: codes[n][gi] = sum_i (w(5gi+i, n) + 1) 3^i,
 * columns zero-padded to a multiple of 5. */
void tgo_compressed_from_dense(const int8_t* W, i64 K, i64 N, uint8_t* codes) {
  const i64 G = (K + 4) / 5;
  for (i64 n = 0; n < N; ++n) {
    for (i64 gi = 0; gi < G; ++gi) {
      int code = 0, p3 = 1;
      for (int i = 0; i < 5; ++i) {
        const i64 k = 5 * gi + i;
        const int v = k < K ? W[k * N + n] : 0;
        code += (v + 1) * p3;
        p3 *= 3;
      }
      codes[n * G + gi] = (uint8_t)code;
    }
  }
}

/* ------------------------------------------------------------------ kernels
 * X is M x ldx row-major (ldx = K, or K+1 for a PaddedInput whose slot K is 0),
 * Y is M x N.  Column range [n_lo, n_hi). */

/* kernels/scalar.py:109-132 */
void tgo_gemm_base(const float* X, i64 M, i64 ldx, const i32* csp, const i32* rip, const i32* csn, const i32* rin,
                   const float* bias, i64 N, float* Y, i64 n_lo, i64 n_hi) {
  for (i64 m = 0; m < M; ++m) {
    const float* x = X + m * ldx;
    for (i64 n = n_lo; n < n_hi; ++n) {
      float acc = 0.0f;
      for (i32 i = csp[n]; i < csp[n + 1]; ++i) acc += x[rip[i]];
      for (i32 i = csn[n]; i < csn[n + 1]; ++i) acc -= x[rin[i]];
      Y[m * N + n] = bias[n] + acc;
    }
  }
}

/* One banked dot product, kernels/scalar.py:167-206 (bank[u] takes stream
 * positions start+u (mod uf); the tail of each sign goes to bank 0). */
static float banked(const float* x, const i32* rip, i32 ps, i32 pe, const i32* rin, i32 ns, i32 ne, int uf,
                    float* bank) {
  for (int u = 0; u < uf; ++u) bank[u] = 0.0f;
  i32 i = ps;
  for (; i + uf <= pe; i += uf)
    for (int u = 0; u < uf; ++u) bank[u] += x[rip[i + u]];
  for (; i < pe; ++i) bank[0] += x[rip[i]];
  i = ns;
  for (; i + uf <= ne; i += uf)
    for (int u = 0; u < uf; ++u) bank[u] -= x[rin[i + u]];
  for (; i < ne; ++i) bank[0] -= x[rin[i]];
  float tot = 0.0f;
  for (int u = 0; u < uf; ++u) tot += bank[u];
  return tot;
}

/* kernels/scalar.py:156-257 (mr/nr only tile the loops; every row uses the banks) */
void tgo_gemm_unrolled(const float* X, i64 M, i64 ldx, const i32* csp, const i32* rip, const i32* csn,
                       const i32* rin, const float* bias, i64 N, float* Y, int uf, i64 n_lo, i64 n_hi) {
  float* bank = (float*)malloc(sizeof(float) * (size_t)uf);
  for (i64 n = n_lo; n < n_hi; ++n)
    for (i64 m = 0; m < M; ++m)
      Y[m * N + n] = bias[n] + banked(X + m * ldx, rip, csp[n], csp[n + 1], rin, csn[n], csn[n + 1], uf, bank);
  free(bank);
}

/* kernels/scalar.py:286-367: out = bias; per block, rows < floor(M/mr)*mr add the
 * banked cell sum, leftover rows a plain accumulator. */
void tgo_gemm_blocked(const float* X, i64 M, i64 ldx, i64 nb, const i32* csp, const i32* rip, const i32* csn,
                      const i32* rin, const float* bias, i64 N, float* Y, int uf, int mr, i64 n_lo, i64 n_hi) {
  float* bank = (float*)malloc(sizeof(float) * (size_t)uf);
  const i64 mf = M / mr * mr;
  for (i64 m = 0; m < M; ++m)
    for (i64 n = n_lo; n < n_hi; ++n) Y[m * N + n] = bias[n];
  for (i64 blk = 0; blk < nb; ++blk) {
    const i32* cp = csp + blk * (N + 1);
    const i32* cn = csn + blk * (N + 1);
    for (i64 n = n_lo; n < n_hi; ++n) {
      for (i64 m = 0; m < M; ++m) {
        const float* x = X + m * ldx;
        if (m < mf) {
          Y[m * N + n] += banked(x, rip, cp[n], cp[n + 1], rin, cn[n], cn[n + 1], uf, bank);
        } else {
          float acc = 0.0f;
          for (i32 i = cp[n]; i < cp[n + 1]; ++i) acc += x[rip[i]];
          for (i32 i = cn[n]; i < cn[n + 1]; ++i) acc -= x[rin[i]];
          Y[m * N + n] += acc;
        }
      }
    }
  }
  free(bank);
}

/* kernels/scalar.py:397-485 */
void tgo_gemm_interleaved_blocked(const float* X, i64 M, i64 ldx, const i32* ai, const i32* ptr, i64 nb, int g,
                                  const float* bias, i64 N, float* Y, i64 n_lo, i64 n_hi) {
  for (i64 m = 0; m < M; ++m)
    for (i64 n = n_lo; n < n_hi; ++n) Y[m * N + n] = bias[n];
  for (i64 blk = 0; blk < nb; ++blk) {
    for (i64 n = n_lo; n < n_hi; ++n) {
      const i64 cell = blk * N + n;
      const i32 s0 = ptr[3 * cell], s1 = ptr[3 * cell + 1], s2 = ptr[3 * cell + 2], s3 = ptr[3 * cell + 3];
      for (i64 m = 0; m < M; ++m) {
        const float* x = X + m * ldx;
        float acc = 0.0f;
        for (i32 i = s0; i < s1; i += 2 * g) {
          for (int u = 0; u < g; ++u) acc += x[ai[i + u]];
          for (int u = 0; u < g; ++u) acc -= x[ai[i + g + u]];
        }
        for (i32 i = s1; i < s2; ++i) acc += x[ai[i]];
        for (i32 i = s2; i < s3; ++i) acc -= x[ai[i]];
        Y[m * N + n] += acc;
      }
    }
  }
}

/* kernels/simd.py:282-420 gemm_vectorized_optimal over a symmetric
 * interleaved-blocked stream.  Same loop nest as the reference: 4 columns x 4
 * rows register tile over the common segment, scalar leftover rows, then the
 * excess-sign remainders added straight into Y, PReLU last.  X is the padded
 * input (ldx = K+1, slot K = 0) so dummy indices read 0.  n_lo, n_hi must be
 * multiples of 4. */
void tgo_gemm_vectorized_optimal(const float* Xp, i64 M, i64 ldx, const i32* ai, const i32* ptr, i64 nb, int g,
                                 const float* bias, i64 N, int use_alpha, float alpha, float* Y, i64 n_lo,
                                 i64 n_hi) {
  for (i64 m = 0; m < M; ++m)
    for (i64 n = n_lo; n < n_hi; ++n) Y[m * N + n] = bias[n];
  for (i64 blk = 0; blk < nb; ++blk) {
    for (i64 n0 = n_lo; n0 < n_hi; n0 += 4) {
      const i64 cell = blk * N + n0;
      const i32 sa = ptr[3 * cell], sb = ptr[3 * (cell + 1)], sc = ptr[3 * (cell + 2)], sd = ptr[3 * (cell + 3)];
      const i32 seglen = ptr[3 * cell + 1] - sa;
      i64 m0 = 0;
      for (; m0 + 4 <= M; m0 += 4) {
        float a[4][4];
        memset(a, 0, sizeof a);
        const float* x0 = Xp + m0 * ldx;
        for (i32 t = 0; t < seglen; ++t) {
          const i32 id[4] = {ai[sa + t], ai[sb + t], ai[sc + t], ai[sd + t]};
          if (((t / g) & 1) == 0) {
            for (int c = 0; c < 4; ++c)
              for (int r = 0; r < 4; ++r) a[c][r] += x0[r * ldx + id[c]];
          } else {
            for (int c = 0; c < 4; ++c)
              for (int r = 0; r < 4; ++r) a[c][r] -= x0[r * ldx + id[c]];
          }
        }
        for (int c = 0; c < 4; ++c)
          for (int r = 0; r < 4; ++r) Y[(m0 + r) * N + n0 + c] += a[c][r];
      }
      for (i64 m = m0; m < M; ++m) {
        const float* x = Xp + m * ldx;
        for (int c = 0; c < 4; ++c) {
          const i32 s0 = ptr[3 * (cell + c)], s1 = ptr[3 * (cell + c) + 1];
          float acc = 0.0f;
          for (i32 t = 0; t < s1 - s0; ++t) {
            const float v = x[ai[s0 + t]];
            if (((t / g) & 1) == 0) acc += v;
            else acc -= v;
          }
          Y[m * N + n0 + c] += acc;
        }
      }
      for (int c = 0; c < 4; ++c) {
        const i32 s1 = ptr[3 * (cell + c) + 1], s2 = ptr[3 * (cell + c) + 2], s3 = ptr[3 * (cell + c) + 3];
        for (i64 m = 0; m < M; ++m) {
          const float* x = Xp + m * ldx;
          float* y = Y + m * N + n0 + c;
          for (i32 i = s1; i < s2; ++i) *y += x[ai[i]];
          for (i32 i = s2; i < s3; ++i) *y -= x[ai[i]];
        }
      }
    }
  }
  if (use_alpha) {
    for (i64 m = 0; m < M; ++m)
      for (i64 n = n_lo; n < n_hi; ++n) {
        const float y = Y[m * N + n];
        if (!(y > 0.0f)) Y[m * N + n] = alpha * y;
      }
  }
}

/* kernels/simd.py:98-188 gemm_vertical over a SymmetricInterleavedTcsc: per
 * column, positive-run and negative-run sums (run parity of the stream
 * position t: (t / g) & 1) and y = (b + p) - q, PReLU.  n_lo, n_hi multiples of 4. */
void tgo_gemm_vertical(const float* Xp, i64 M, i64 ldx, const i32* idx, const i32* col_ptr, int g, const float* bias,
                       i64 N, int use_alpha, float alpha, float* Y, i64 n_lo, i64 n_hi) {
  for (i64 m = 0; m < M; ++m) {
    const float* x = Xp + m * ldx;
    for (i64 n = n_lo; n < n_hi; ++n) {
      const i32 s = col_ptr[n], len = col_ptr[n + 1] - col_ptr[n];
      float p = 0.0f, q = 0.0f;
      for (i32 t = 0; t < len; ++t) {
        const float v = x[idx[s + t]];
        if (((t / g) & 1) == 0) p += v;
        else q += v;
      }
      float y = bias[n] + p - q;
      if (use_alpha && !(y > 0.0f)) y = alpha * y;
      Y[m * N + n] = y;
    }
  }
}

/* kernels/simd.py:196-274 gemm_horizontal: four lane accumulators take stream
 * positions t = 0, 1, 2, 3 (mod 4), sign = ((t / g) & 1); y = b + ((a0 + a1) + (a2 + a3)). */
void tgo_gemm_horizontal(const float* Xp, i64 M, i64 ldx, const i32* idx, const i32* col_ptr, int g,
                         const float* bias, i64 N, int use_alpha, float alpha, float* Y, i64 n_lo, i64 n_hi) {
  for (i64 m = 0; m < M; ++m) {
    const float* x = Xp + m * ldx;
    for (i64 n = n_lo; n < n_hi; ++n) {
      const i32 s = col_ptr[n], e = col_ptr[n + 1];
      float a[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      for (i32 w = s; w < e; w += 4) {
        const i32 t = w - s;
        for (int j = 0; j < 4; ++j) {
          const float v = x[idx[w + j]];
          if ((((t + j) / g) & 1) == 0) a[j] += v;
          else a[j] -= v;
        }
      }
      float y = bias[n] + ((a[0] + a[1]) + (a[2] + a[3]));
      if (use_alpha && !(y > 0.0f)) y = alpha * y;
      Y[m * N + n] = y;
    }
  }
}

/* kernels/scalar.py:561-602 gemm_compressed: per column, codes in order, the 5
 * base-3 digits of each code (digit 2 -> +x, 0 -> -x), out = b + acc. */
void tgo_gemm_compressed(const float* X, i64 M, i64 ldx, const uint8_t* codes, i64 G, const float* bias, i64 N,
                         float* Y, i64 n_lo, i64 n_hi) {
  for (i64 m = 0; m < M; ++m) {
    const float* x = X + m * ldx;
    for (i64 n = n_lo; n < n_hi; ++n) {
      float acc = 0.0f;
      for (i64 gi = 0; gi < G; ++gi) {
        int code = codes[n * G + gi];
        for (int t = 0; t < 5; ++t) {
          const int d = code % 3 - 1;
          code /= 3;
          if (d > 0) acc += x[5 * gi + t];
          else if (d < 0) acc -= x[5 * gi + t];
        }
      }
      Y[m * N + n] = bias[n] + acc;
    }
  }
}

/* ------------------------------------------------------------------ threaded driver
 * Runs one of the kernels above over `threads` disjoint column ranges
 * (multiples of 4) with pthreads.  kind: 0 base, 1 unrolled, 2 blocked,
 * 3 interleaved_blocked, 4 vectorized_optimal, 5 vertical (a0 = indices,
 * a1 = col_ptr), 6 horizontal, 7 compressed (a0 = codes, nb = groups per column). */
typedef struct {
  int kind;
  const float* X;
  i64 M, ldx;
  const i32 *a0, *a1, *a2, *a3;
  i64 nb;
  int g, uf, mr;
  const float* bias;
  i64 N;
  int use_alpha;
  float alpha;
  float* Y;
  i64 lo, hi;
} tgo_job;

static void* tgo_worker(void* arg) {
  const tgo_job* j = (const tgo_job*)arg;
  if (j->lo >= j->hi) return NULL;
  switch (j->kind) {
    case 0: tgo_gemm_base(j->X, j->M, j->ldx, j->a0, j->a1, j->a2, j->a3, j->bias, j->N, j->Y, j->lo, j->hi); break;
    case 1:
      tgo_gemm_unrolled(j->X, j->M, j->ldx, j->a0, j->a1, j->a2, j->a3, j->bias, j->N, j->Y, j->uf, j->lo, j->hi);
      break;
    case 2:
      tgo_gemm_blocked(j->X, j->M, j->ldx, j->nb, j->a0, j->a1, j->a2, j->a3, j->bias, j->N, j->Y, j->uf, j->mr,
                       j->lo, j->hi);
      break;
    case 3:
      tgo_gemm_interleaved_blocked(j->X, j->M, j->ldx, j->a0, j->a1, j->nb, j->g, j->bias, j->N, j->Y, j->lo, j->hi);
      break;
    case 5:
      tgo_gemm_vertical(j->X, j->M, j->ldx, j->a0, j->a1, j->g, j->bias, j->N, j->use_alpha, j->alpha, j->Y, j->lo,
                        j->hi);
      break;
    case 6:
      tgo_gemm_horizontal(j->X, j->M, j->ldx, j->a0, j->a1, j->g, j->bias, j->N, j->use_alpha, j->alpha, j->Y,
                          j->lo, j->hi);
      break;
    case 7:
      tgo_gemm_compressed(j->X, j->M, j->ldx, (const uint8_t*)j->a0, j->nb, j->bias, j->N, j->Y, j->lo, j->hi);
      break;
    default:
      tgo_gemm_vectorized_optimal(j->X, j->M, j->ldx, j->a0, j->a1, j->nb, j->g, j->bias, j->N, j->use_alpha,
                                  j->alpha, j->Y, j->lo, j->hi);
      break;
  }
  return NULL;
}

int tgo_run_threaded(int kind, int threads, const float* X, i64 M, i64 ldx, const i32* a0, const i32* a1,
                     const i32* a2, const i32* a3, i64 nb, int g, int uf, int mr, const float* bias, i64 N,
                     int use_alpha, float alpha, float* Y) {
  if (threads < 1) threads = 1;
  const i64 groups = (N + 3) / 4;
  if (threads > groups) threads = (int)groups;
  tgo_job* jobs = (tgo_job*)calloc((size_t)threads, sizeof(tgo_job));
  pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int t = 0; t < threads; ++t) {
    tgo_job* j = &jobs[t];
    j->kind = kind; j->X = X; j->M = M; j->ldx = ldx;
    j->a0 = a0; j->a1 = a1; j->a2 = a2; j->a3 = a3;
    j->nb = nb; j->g = g; j->uf = uf; j->mr = mr;
    j->bias = bias; j->N = N; j->use_alpha = use_alpha; j->alpha = alpha; j->Y = Y;
    j->lo = groups * t / threads * 4;
    j->hi = groups * (t + 1) / threads * 4;
    if (j->hi > N) j->hi = N;
  }
  int rc = 0;
  for (int t = 1; t < threads; ++t)
    if (pthread_create(&tids[t], NULL, tgo_worker, &jobs[t]) != 0) rc = -1;
  tgo_worker(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(tids[t], NULL);
  free(jobs);
  free(tids);
  return rc;
}
