"""Invalid arguments raise the reference's exception classes (kernels/scalar.py:79-101,
simd.py:78-90, 438-439, kernels/__init__.py:211-230, dense.py:32-111, variants.py:451-521,
tcsc.py:35-68).  The checks run on the host before any device work, so this is a CPU test;
it compares against the reference package imported read-only from /root/reference when it
is mounted (skipped otherwise)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

import paper_2510_06957_b200 as tg
from oracle import oracle as orc

REF = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def rtg():
    if not os.path.isdir(REF):
        pytest.skip("reference package not mounted")
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    try:
        import terngemm
    except Exception as exc:  # noqa: BLE001
        pytest.skip(f"reference not importable: {exc}")
    return terngemm


def _formats(pkg, W, ours: bool):
    """(tcsc, ib, ib_sym) of W in package `pkg` (ours from the oracle's arrays: no device here)."""
    K, N = W.shape
    if not ours:
        w = pkg.TernaryDense(W)
        return (pkg.tcsc_from_dense(w), pkg.interleaved_blocked_from_dense(w, None, 2),
                pkg.interleaved_blocked_from_dense(w, None, 2, symmetric_cols=True))
    t = orc.tcsc_from_dense(W)
    ib = orc.interleaved_blocked_from_dense(W, None, 2, False)
    ibs = orc.interleaved_blocked_from_dense(W, None, 2, True)
    return (tg.Tcsc(K, N, t["col_start_pos"], t["row_index_pos"], t["col_start_neg"], t["row_index_neg"]),
            tg.InterleavedBlockedTcsc(K, N, ib["B"], 2, ib["all_indices"], ib["col_segment_ptr"]),
            tg.InterleavedBlockedTcsc(K, N, ibs["B"], 2, ibs["all_indices"], ibs["col_segment_ptr"], True))


def _cases(pkg, ours):
    rng = np.random.default_rng(0)
    K, N, M = 12, 8, 3
    W = rng.integers(-1, 2, size=(K, N)).astype(np.int8)
    X = rng.standard_normal((M, K)).astype(np.float32)
    b = np.zeros(N, np.float32)
    t, ib, ibs = _formats(pkg, W, ours)
    Xbad = rng.standard_normal((M, K + 1)).astype(np.float32)
    Xp = np.hstack([X, np.zeros((M, 1), np.float32)])        # padded inputs built directly:
    Xpbad = np.hstack([Xbad, np.zeros((M, 1), np.float32)])  # pad_input itself needs the device here
    Xinf = X.copy()
    Xinf[1, 2] = np.inf
    W2 = W.copy()
    W2[3, 4] = 2
    return {
        "x_cols": lambda: pkg.gemm_base(pkg.DenseMatrix(Xbad), t, pkg.BiasVector(b)),
        "bias_len": lambda: pkg.gemm_base(pkg.DenseMatrix(X), t, pkg.BiasVector(np.zeros(N + 1, np.float32))),
        "unrolled_x_cols": lambda: pkg.gemm_unrolled(pkg.DenseMatrix(Xbad), t, pkg.BiasVector(b)),
        "ib_symmetric_into_scalar": lambda: pkg.gemm_interleaved_blocked(pkg.DenseMatrix(X), ibs, pkg.BiasVector(b)),
        "optimal_needs_symmetric": lambda: pkg.gemm_vectorized_optimal(pkg.PaddedInput(Xp), ib, pkg.BiasVector(b)),
        "optimal_nan_alpha": lambda: pkg.gemm_vectorized_optimal(pkg.PaddedInput(Xp), ibs, pkg.BiasVector(b),
                                                                  float("nan")),
        "optimal_k_mismatch": lambda: pkg.gemm_vectorized_optimal(pkg.PaddedInput(Xpbad), ibs, pkg.BiasVector(b)),
        "cfg_uf0": lambda: pkg.GemmConfig(uf=0),
        "cfg_mr3": lambda: pkg.GemmConfig(mr=3),
        "cfg_nan_alpha": lambda: pkg.GemmConfig(alpha=float("inf")),
        "ternary_value_2": lambda: pkg.TernaryDense(W2),
        "ternary_1d": lambda: pkg.TernaryDense(W[0]),
        "dense_inf": lambda: pkg.DenseMatrix(Xinf),
        "bias_2d": lambda: pkg.BiasVector(np.zeros((2, 2), np.float32)),
        "padded_slot_nonzero": lambda: pkg.PaddedInput(np.ones((2, 3), np.float32)),
        "alpha_on_scalar_tag": lambda: pkg.run_variant("base", pkg.DenseMatrix(X), pkg.TernaryDense(W),
                                                       pkg.BiasVector(b), pkg.GemmConfig(alpha=0.25)),
        "compress5_bad": lambda: pkg.compress5([0, 1, 2, 0, 0]),
        "compress5_len": lambda: pkg.compress5([0, 1]),
        "decompress5_bad": lambda: pkg.decompress5(243),
        "compressed_bad_code": lambda: pkg.CompressedTcsc(5, 1, np.array([[250]], np.uint8)),
        "tcsc_bad_len": lambda: pkg.Tcsc(K, N, np.zeros(N, np.int32), np.zeros(0, np.int32),
                                         np.zeros(N + 1, np.int32), np.zeros(0, np.int32)),
        "tcsc_zero_k": lambda: pkg.Tcsc(0, N, np.zeros(N + 1, np.int32), np.zeros(0, np.int32),
                                        np.zeros(N + 1, np.int32), np.zeros(0, np.int32)),
        "ib_bad_ptr": lambda: pkg.InterleavedBlockedTcsc(K, N, 4, 2, np.zeros(0, np.int32), np.zeros(3, np.int32)),
        "ib_sym_n": lambda: pkg.InterleavedBlockedTcsc(K, 6, 12, 2, np.zeros(0, np.int32), np.zeros(19, np.int32),
                                                       True),
        "blocked_b0": lambda: pkg.BlockedTcsc(K, N, 0, np.zeros((1, N + 1), np.int32), np.zeros(0, np.int32),
                                              np.zeros((1, N + 1), np.int32), np.zeros(0, np.int32)),
    }


def _outcome(fn):
    try:
        fn()
    except Exception as exc:  # noqa: BLE001
        return type(exc).__name__
    return "ok"


def test_invalid_arguments_raise_the_reference_exceptions(rtg):
    theirs, mine = _cases(rtg, False), _cases(tg, True)
    mismatches = {}
    for name in theirs:
        r, o = _outcome(theirs[name]), _outcome(mine[name])
        if r != o:
            mismatches[name] = (r, o)
    assert not mismatches, mismatches
