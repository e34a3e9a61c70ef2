"""CPU oracle for the sparse ternary GEMM hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs import this module, and only as the checker (or as
the timed CPU baseline); the product package ``paper_2510_06957_b200`` never
does.

Two layers:
  * ``oracle_gemm`` — numpy fp64 restatement of the reference's dense oracle
    (/root/reference/pkg/src/terngemm/dense.py:192-213).
  * ctypes wrappers of ``tg_oracle.c`` (built by ``make -C oracle``): the
    format builders (tcsc.py:71-92, variants.py:146-178, variants.py:312-376)
    and the five kernels with the reference's per-output fp32 operation order
    (kernels/scalar.py:109-485, kernels/simd.py:282-420).

Pinning: tests/test_oracle_golden.py checks every function here against
tests/golden/*.npz, fixtures written by tests/golden/make_golden.py from the
reference package itself (integer-valued and real-valued inputs, bit-exact).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtg_oracle.so")

KIND_BASE, KIND_UNROLLED, KIND_BLOCKED, KIND_IB, KIND_OPTIMAL = 0, 1, 2, 3, 4
KIND_VERTICAL, KIND_HORIZONTAL, KIND_COMPRESSED = 5, 6, 7

_lib = None


def build() -> str:
    """Compile tg_oracle.c (idempotent)."""
    src = os.path.join(HERE, "tg_oracle.c")
    if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        P, I64, I, F = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float
        L.tgo_tcsc_from_dense.argtypes = [P, I64, I64, P, P, P, P]
        L.tgo_blocked_from_dense.argtypes = [P, I64, I64, I64, P, P, P, P]
        L.tgo_interleaved_blocked_from_dense.argtypes = [P, I64, I64, I64, I, I, P, P]
        L.tgo_interleaved_blocked_from_dense.restype = I64
        L.tgo_symmetric_from_dense.argtypes = [P, I64, I64, I, P, P]
        L.tgo_symmetric_from_dense.restype = I64
        L.tgo_compressed_from_dense.argtypes = [P, I64, I64, P]
        L.tgo_run_threaded.argtypes = [I, I, P, I64, I64, P, P, P, P, I64, I, I, I, P, I64, I, F, P]
        L.tgo_run_threaded.restype = I
        _lib = L
    return _lib


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _w(W) -> np.ndarray:
    v = np.ascontiguousarray(getattr(W, "values", W), dtype=np.int8)
    assert v.ndim == 2
    return v


# ---------------------------------------------------------------- formats


def tcsc_from_dense(W) -> dict:
    w = _w(W)
    K, N = w.shape
    csp = np.zeros(N + 1, np.int32)
    csn = np.zeros(N + 1, np.int32)
    lib().tgo_tcsc_from_dense(_ptr(w), K, N, _ptr(csp), None, _ptr(csn), None)
    rip = np.empty(int(csp[-1]), np.int32)
    rin = np.empty(int(csn[-1]), np.int32)
    lib().tgo_tcsc_from_dense(_ptr(w), K, N, _ptr(csp), _ptr(rip), _ptr(csn), _ptr(rin))
    return dict(K=K, N=N, col_start_pos=csp, row_index_pos=rip, col_start_neg=csn, row_index_neg=rin)


def resolve_block_size(B, K: int) -> int:
    """variants.py:38-42."""
    return min(K, 4096) if B is None else int(B)


def blocked_from_dense(W, B=None) -> dict:
    w = _w(W)
    K, N = w.shape
    B = resolve_block_size(B, K)
    nb = -(-K // B)
    csp = np.zeros((nb, N + 1), np.int32)
    csn = np.zeros((nb, N + 1), np.int32)
    lib().tgo_blocked_from_dense(_ptr(w), K, N, B, _ptr(csp), None, _ptr(csn), None)
    rip = np.empty(int(csp[-1, -1]), np.int32)
    rin = np.empty(int(csn[-1, -1]), np.int32)
    lib().tgo_blocked_from_dense(_ptr(w), K, N, B, _ptr(csp), _ptr(rip), _ptr(csn), _ptr(rin))
    return dict(K=K, N=N, B=B, col_start_pos=csp, row_index_pos=rip, col_start_neg=csn, row_index_neg=rin)


def interleaved_blocked_from_dense(W, B=None, g: int = 2, symmetric_cols: bool = False) -> dict:
    w = _w(W)
    K, N = w.shape
    B = resolve_block_size(B, K)
    nb = -(-K // B)
    ptr = np.zeros(3 * nb * N + 1, np.int32)
    n = lib().tgo_interleaved_blocked_from_dense(_ptr(w), K, N, B, g, int(symmetric_cols), None, _ptr(ptr))
    ai = np.empty(int(n), np.int32)
    lib().tgo_interleaved_blocked_from_dense(_ptr(w), K, N, B, g, int(symmetric_cols), _ptr(ai), _ptr(ptr))
    return dict(K=K, N=N, B=B, g=g, all_indices=ai, col_segment_ptr=ptr, symmetric_groups=bool(symmetric_cols))


def symmetric_from_dense(W, g: int = 2) -> dict:
    """variants.py:582-631."""
    w = _w(W)
    K, N = w.shape
    assert N % 4 == 0
    ptr = np.zeros(N + 1, np.int32)
    n = lib().tgo_symmetric_from_dense(_ptr(w), K, N, g, None, _ptr(ptr))
    idx = np.empty(int(n), np.int32)
    lib().tgo_symmetric_from_dense(_ptr(w), K, N, g, _ptr(idx), _ptr(ptr))
    return dict(K=K, N=N, g=g, indices=idx, col_ptr=ptr)


def compressed_from_dense(W) -> dict:
    """variants.py:515-521."""
    w = _w(W)
    K, N = w.shape
    codes = np.empty((N, (K + 4) // 5), np.uint8)
    lib().tgo_compressed_from_dense(_ptr(w), K, N, _ptr(codes))
    return dict(K=K, N=N, codes=codes)


# ---------------------------------------------------------------- inputs


def pad_input(X) -> np.ndarray:
    """simd.py:72-75: M x (K+1) copy whose slot K is 0."""
    x = np.ascontiguousarray(getattr(X, "values", X), dtype=np.float32)
    xp = np.zeros((x.shape[0], x.shape[1] + 1), np.float32)
    xp[:, :-1] = x
    return xp


def oracle_gemm(X, W, b, alpha=None) -> np.ndarray:
    """dense.py:192-213: fp64 X @ W + b, PReLU in fp64, one cast to fp32."""
    x = np.asarray(getattr(X, "values", X), dtype=np.float64)
    w = np.asarray(getattr(W, "values", W), dtype=np.float64)
    bb = np.asarray(getattr(b, "values", b), dtype=np.float64)
    y = x @ w + bb
    if alpha is not None:
        y = np.where(y > 0, y, float(alpha) * y)
    return y.astype(np.float32)


# ---------------------------------------------------------------- kernels


def _run(kind, X, fmt_arrays, N, bias, threads=1, nb=1, g=1, uf=1, mr=1, alpha=None) -> np.ndarray:
    x = np.ascontiguousarray(X, dtype=np.float32)
    M, ldx = x.shape
    b = np.ascontiguousarray(bias, dtype=np.float32)
    arrs = [None if a is None else np.ascontiguousarray(a, dtype=np.int32) for a in fmt_arrays]
    arrs += [None] * (4 - len(arrs))
    y = np.empty((M, N), np.float32)
    rc = lib().tgo_run_threaded(
        kind, int(threads), _ptr(x), M, ldx, *[_ptr(a) for a in arrs], nb, g, uf, mr, _ptr(b), N,
        int(alpha is not None), float(alpha or 0.0), _ptr(y),
    )
    if rc != 0:
        raise RuntimeError("tgo_run_threaded failed")
    return y


def gemm_base(X, t: dict, b, threads=1):
    """kernels/scalar.py:109-148."""
    return _run(KIND_BASE, X, [t["col_start_pos"], t["row_index_pos"], t["col_start_neg"], t["row_index_neg"]],
                t["N"], b, threads)


def gemm_unrolled(X, t: dict, b, uf=12, threads=1):
    """kernels/scalar.py:156-278 (mr, nr do not change any output bit)."""
    return _run(KIND_UNROLLED, X, [t["col_start_pos"], t["row_index_pos"], t["col_start_neg"], t["row_index_neg"]],
                t["N"], b, threads, uf=uf)


def gemm_blocked(X, t: dict, b, uf=12, mr=4, threads=1):
    """kernels/scalar.py:286-389."""
    nb = t["col_start_pos"].shape[0]
    return _run(KIND_BLOCKED, X, [t["col_start_pos"], t["row_index_pos"], t["col_start_neg"], t["row_index_neg"]],
                t["N"], b, threads, nb=nb, uf=uf, mr=mr)


def gemm_interleaved_blocked(X, t: dict, b, threads=1):
    """kernels/scalar.py:397-511."""
    nb = -(-t["K"] // t["B"])
    return _run(KIND_IB, X, [t["all_indices"], t["col_segment_ptr"]], t["N"], b, threads, nb=nb, g=t["g"])


def gemm_vectorized_optimal(Xp, t: dict, b, alpha=None, threads=1):
    """kernels/simd.py:282-449; Xp is the padded M x (K+1) input."""
    nb = -(-t["K"] // t["B"])
    return _run(KIND_OPTIMAL, Xp, [t["all_indices"], t["col_segment_ptr"]], t["N"], b, threads, nb=nb, g=t["g"],
                alpha=alpha)


def gemm_vertical(Xp, t: dict, b, alpha=None, threads=1):
    """kernels/simd.py:98-188; Xp is the padded M x (K+1) input."""
    return _run(KIND_VERTICAL, Xp, [t["indices"], t["col_ptr"]], t["N"], b, threads, g=t["g"], alpha=alpha)


def gemm_horizontal(Xp, t: dict, b, alpha=None, threads=1):
    """kernels/simd.py:196-274."""
    return _run(KIND_HORIZONTAL, Xp, [t["indices"], t["col_ptr"]], t["N"], b, threads, g=t["g"], alpha=alpha)


def gemm_compressed(X, t: dict, b, threads=1):
    """kernels/scalar.py:561-602."""
    codes = np.ascontiguousarray(t["codes"], dtype=np.uint8)
    x = np.ascontiguousarray(X, dtype=np.float32)
    M, ldx = x.shape
    bb = np.ascontiguousarray(b, dtype=np.float32)
    y = np.empty((M, t["N"]), np.float32)
    rc = lib().tgo_run_threaded(KIND_COMPRESSED, int(threads), _ptr(x), M, ldx, _ptr(codes), None, None, None,
                                codes.shape[1], 1, 1, 1, _ptr(bb), t["N"], 0, 0.0, _ptr(y))
    if rc != 0:
        raise RuntimeError("tgo_run_threaded failed")
    return y


# ---------------------------------------------------------------- parity predicates


def normwise_error(y, ref) -> float:
    """max|Y - ref| / max|ref| (SURVEY.md section 8(c) predicate (ii))."""
    y = np.asarray(y, np.float64)
    r = np.asarray(ref, np.float64)
    den = np.abs(r).max() if r.size else 0.0
    return float(np.abs(y - r).max() / den) if den > 0 else float(np.abs(y - r).max() if r.size else 0.0)


def scaled_error(y, X, W, b, alpha=None) -> float:
    """max_mn |Y - Y64| / (sum_k |x_mk||w_kn| + |b_n|)  (predicate (iii)); PReLU scales both sides."""
    x = np.abs(np.asarray(getattr(X, "values", X), np.float64))
    w = np.abs(np.asarray(getattr(W, "values", W), np.float64))
    bb = np.abs(np.asarray(getattr(b, "values", b), np.float64))
    scale = x @ w + bb
    if alpha is not None:
        scale = scale * max(1.0, abs(float(alpha)))
    ref = oracle_gemm(X, W, b, alpha).astype(np.float64)
    err = np.abs(np.asarray(y, np.float64) - ref)
    with np.errstate(divide="ignore", invalid="ignore"):
        q = np.where(scale > 0, err / scale, np.where(err > 0, np.inf, 0.0))
    return float(q.max()) if q.size else 0.0
