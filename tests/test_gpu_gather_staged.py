"""The shared-memory-staged gather kernel (tg_gather_staged_kernel) against the oracle.

The kernel walks each column's index stream in K windows of X staged in shared
memory by TMA bulk copies; a column pauses at the window end and resumes in the
next window, so the per-output fp32 operation order of the reference kernels
(kernels/scalar.py:109-148, 397-511; kernels/simd.py:282-449) is unchanged.
Bar: Y bit-identical to the C restatement of the reference kernels (pinned to
the reference's own outputs, tests/test_oracle_golden.py) on real-valued X, and
bit-identical to the L2 walk (TG_GATHER_STAGED=0) of the same library.

Shapes cross several windows (192 k each), several K blocks, several row groups
(128 rows) and column groups (up to 64 columns), with every group size g, dummy
indices (symmetric formats) and very sparse / dense W.
"""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tg():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2510_06957_b200 as m

    return m


def _inputs(seed, M, K, N, density):
    rng = np.random.default_rng(seed)
    u = rng.random((K, N))
    W = np.where(u < density / 2, 1, np.where(u < density, -1, 0)).astype(np.int8)
    X = (rng.standard_normal((M, K)) * np.exp(rng.uniform(-2, 2, size=(M, 1)))).astype(np.float32)
    b = rng.standard_normal(N).astype(np.float32)
    return W, X, b


def _both_modes(fn):
    """fn() with the staged kernel (default) and with the L2 walk."""
    old = os.environ.get("TG_GATHER_STAGED")
    try:
        os.environ.pop("TG_GATHER_STAGED", None)
        staged = fn()
        os.environ["TG_GATHER_STAGED"] = "0"
        plain = fn()
    finally:
        if old is None:
            os.environ.pop("TG_GATHER_STAGED", None)
        else:
            os.environ["TG_GATHER_STAGED"] = old
    return staged, plain


CASES = [
    # (M, K, N, density, B, g)
    (1, 1, 4, 1.0, None, 2),           # one entry
    (5, 191, 8, 0.5, None, 2),         # one short window
    (130, 193, 68, 0.5, None, 2),      # two windows, two row groups, two columns per warp
    (257, 1000, 132, 0.5, 256, 2),     # four K blocks, block boundaries inside windows' ranges
    (64, 1000, 40, 0.5, 333, 3),       # g = 3 (general run length), ragged blocks
    (40, 2000, 24, 0.5, None, 1),      # g = 1
    (33, 4500, 64, 0.06, 4096, 2),     # sparse: a handful of indices per window
    (20, 700, 16, 1.0, None, 2),       # dense +-1
    (16, 900, 12, 0.5, 1, 2),          # B = 1: one window per block
    (300, 5000, 200, 0.3, 4096, 2),    # two blocks of 4096 / 904, three row groups
]


@pytest.mark.parametrize("M,K,N,density,B,g", CASES)
def test_staged_gather_bit_exact(tg, M, K, N, density, B, g):
    from oracle import oracle as orc

    W, X, b = _inputs(M * 7919 + K * 31 + N, M, K, N, density)
    Wd = tg.TernaryDense(torch.from_numpy(W).cuda())
    Xd = torch.from_numpy(X).cuda()
    G = "gather"
    # base (two sweeps: the positive stream, then the negative one)
    t, r = tg.tcsc_from_dense(Wd), orc.tcsc_from_dense(W)
    ys, yp = _both_modes(lambda: tg.gemm_base(Xd, t, b, method=G).values)
    ref = orc.gemm_base(X, r, b)
    assert np.array_equal(ys, ref) and np.array_equal(yp, ref)
    # interleaved_blocked
    ib, ri = tg.interleaved_blocked_from_dense(Wd, B, g), orc.interleaved_blocked_from_dense(W, B, g)
    ys, yp = _both_modes(lambda: tg.gemm_interleaved_blocked(Xd, ib, b, method=G).values)
    ref = orc.gemm_interleaved_blocked(X, ri, b)
    assert np.array_equal(ys, ref) and np.array_equal(yp, ref)
    # vectorized_optimal (symmetric groups: dummy indices K read the padded slot), with PReLU
    ibs, ris = tg.interleaved_blocked_from_dense(Wd, B, g, True), orc.interleaved_blocked_from_dense(W, B, g, True)
    Xp = tg.pad_input(Xd)
    (ys, cs), (yp, cp) = _both_modes(lambda: tg.gemm_vectorized_optimal(Xp, ibs, b, 0.25, method=G, counted=True))
    ref = orc.gemm_vectorized_optimal(orc.pad_input(X), ris, b, 0.25)
    assert np.array_equal(ys.values, ref) and np.array_equal(yp.values, ref)
    assert cs == cp


def test_staged_gather_full_cfg2_slice(tg):
    """cfg2 at full K and N (21 windows, 148 CTAs of 56 columns): 128 seeded rows against the oracle."""
    from oracle import oracle as orc
    from paper_2510_06957_b200.workloads import make_inputs

    W, X, b = make_inputs("cfg2")
    X = np.ascontiguousarray(X[:128])
    Wd = tg.TernaryDense(torch.from_numpy(W).cuda())
    fmt = tg.interleaved_blocked_from_dense(Wd, None, 2, True)
    y = tg.gemm_vectorized_optimal(tg.pad_input(torch.from_numpy(X).cuda()), fmt, b, 0.25, method="gather").values
    ref = orc.gemm_vectorized_optimal(orc.pad_input(X), orc.interleaved_blocked_from_dense(W, None, 2, True), b, 0.25)
    assert np.array_equal(y, ref)


@pytest.mark.parametrize("p_pos,p_neg", [(0.45, 0.05), (0.05, 0.45), (0.3, 0.2)])
def test_staged_gather_sign_imbalance_drift(tg, p_pos, p_neg):
    """Unequal +1 / -1 densities: the two subsequences of the interleaved segment drift apart
    linearly in k, so most operands of the slower one lie outside the staged window and take
    the L2 path; long remainder segments follow.  Still bit-identical."""
    from oracle import oracle as orc

    rng = np.random.default_rng(int(p_pos * 100) * 7 + 3)
    M, K, N = 200, 3000, 124
    u = rng.random((K, N))
    W = np.where(u < p_pos, 1, np.where(u < p_pos + p_neg, -1, 0)).astype(np.int8)
    X = rng.standard_normal((M, K)).astype(np.float32)
    b = rng.standard_normal(N).astype(np.float32)
    Wd, Xd = tg.TernaryDense(torch.from_numpy(W).cuda()), torch.from_numpy(X).cuda()
    for B in (None, 1024, 700):
        ibs, ris = tg.interleaved_blocked_from_dense(Wd, B, 2, True), orc.interleaved_blocked_from_dense(W, B, 2, True)
        ys, yp = _both_modes(lambda: tg.gemm_vectorized_optimal(tg.pad_input(Xd), ibs, b, 0.25, method="gather").values)
        ref = orc.gemm_vectorized_optimal(orc.pad_input(X), ris, b, 0.25)
        assert np.array_equal(ys, ref) and np.array_equal(yp, ref), B
        ib, ri = tg.interleaved_blocked_from_dense(Wd, B, 2), orc.interleaved_blocked_from_dense(W, B, 2)
        ys = tg.gemm_interleaved_blocked(Xd, ib, b, method="gather").values
        assert np.array_equal(ys, orc.gemm_interleaved_blocked(X, ri, b)), B
