"""GPU parity of the tensor-core path on heavy-tailed activations.

LLM-style X has a few channels tens to hundreds of times larger than the rest.  Such a row
is "wide" for the 22-bit limb grid; the X split now lists its few large entries, the limbs
carry the rest at the rest's own scale, and the epilogue adds the listed terms (tg_mma.cu,
kOutlierCap).  Bars as in test_gpu_parity.py: normwise and |terms|-scaled
error <= 1e-5 against the fp64 oracle (the reference's dense.py:192-213), integer-valued X
bit-exact with the reference-order kernels (kernels/scalar.py:397-511), and rows that cannot
shed their outliers still bit-identical with the reference order.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import oracle as orc

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def tg():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2510_06957_b200 as m

    return m


def _w(rng, K, N, p=0.6):
    u = rng.random((K, N))
    return np.where(u < p / 2, 1, np.where(u < p, -1, 0)).astype(np.int8)


def _stats(tg, X, fmt, b):
    from paper_2510_06957_b200 import kernels as kn

    r = kn.GemmRunner("interleaved_blocked", torch.from_numpy(X).cuda(), fmt, torch.from_numpy(b).cuda(),
                      method="mma")
    return r.row_stats()


def _gemm(tg, X, W, b, alpha=None, method="mma", counted=False, device=False):
    """interleaved_blocked (no activation) or vectorized_optimal (PReLU) through the public API."""
    if alpha is None:
        Xin = tg.DenseMatrix(torch.from_numpy(X).cuda()) if device else X
        return tg.gemm_interleaved_blocked(Xin, tg.interleaved_blocked_from_dense(W), b, counted=counted, method=method)
    t = tg.interleaved_blocked_from_dense(W, None, 2, True)
    Xp = tg.pad_input(tg.DenseMatrix(torch.from_numpy(X).cuda()) if device else X)
    return tg.gemm_vectorized_optimal(Xp, t, b, alpha, counted=counted, method=method)


def _bars(y, X, W, b, alpha=None):
    ref = orc.oracle_gemm(X, W, b, alpha)
    return orc.normwise_error(y, ref), orc.scaled_error(y, X, W, b, alpha)


@pytest.mark.parametrize("M,K,N,scale,nch", [(16, 4096, 1024, 100.0, 8), (256, 4096, 512, 100.0, 8),
                                             (33, 1000, 200, 1000.0, 3), (16, 4096, 256, 30.0, 24)])
def test_outlier_channels_stay_on_tensor_cores(tg, M, K, N, scale, nch):
    """N(0,1) activations with `nch` channels at `scale` x: no row takes the exact walk, every
    row sheds a few entries, and both parity bars hold (with and without PReLU)."""
    rng = np.random.default_rng(M + K + N)
    W = _w(rng, K, N)
    X = rng.standard_normal((M, K)).astype(np.float32)
    ch = rng.choice(K, nch, replace=False)
    X[:, ch] *= np.float32(scale)
    b = rng.standard_normal(N).astype(np.float32)
    t = tg.interleaved_blocked_from_dense(W)
    st = _stats(tg, X, t, b)
    assert st["exact_rows"] == 0, st
    assert st["outlier_rows"] == M and 0 < st["outlier_entries"] <= 128 * M, st
    for alpha in (None, 0.25):
        y = _gemm(tg, X, W, b, alpha).values
        nw, sc = _bars(y, X, W, b, alpha)
        assert nw <= TOL and sc <= TOL, (alpha, nw, sc)


def test_integer_outliers_bit_exact_with_reference_order(tg):
    """Integer-valued X (the reference's own regime, dense.py:17-19) with large integer
    outliers: limbs, int32 accumulation and the listed fp32 adds are all exact, so the
    tensor-core result equals the reference-order gather bit for bit, OpCount included."""
    rng = np.random.default_rng(11)
    M, K, N = 70, 1000, 200
    W = _w(rng, K, N, 0.5)
    X = rng.integers(-8, 9, size=(M, K)).astype(np.float32)
    for m in range(M):
        idx = rng.choice(K, 5, replace=False)
        X[m, idx] = rng.integers(1000, 4000, size=5) * rng.choice([-1, 1], 5)
    b = rng.integers(-4, 5, size=N).astype(np.float32)
    t = tg.interleaved_blocked_from_dense(W)
    st = _stats(tg, X, t, b)
    assert st["exact_rows"] == 0 and st["outlier_rows"] == M and st["outlier_entries"] == 5 * M, st
    y_m, ops_m = _gemm(tg, X, W, b, 0.25, "mma", counted=True)
    y_g, ops_g = _gemm(tg, X, W, b, 0.25, "gather", counted=True)
    assert np.array_equal(y_m.values, y_g.values)
    assert ops_m.mults == ops_g.mults and ops_m.adds == ops_g.adds
    ref = orc.gemm_vectorized_optimal(orc.pad_input(X), orc.interleaved_blocked_from_dense(W, None, 2, True), b, 0.25)
    assert np.array_equal(y_m.values, ref)
    y_p = _gemm(tg, X, W, b, None, "mma").values
    assert np.array_equal(y_p, orc.gemm_interleaved_blocked(X, orc.interleaved_blocked_from_dense(W, None, 2, False), b))


def test_rows_that_cannot_shed_keep_the_exact_walk(tg):
    """More large entries than the list holds, or a scale outside the epilogue's range: the
    row is recomputed in the reference's exact order (bit-identical), as before."""
    rng = np.random.default_rng(12)
    M, K, N = 20, 2048, 96
    W = _w(rng, K, N, 0.5)
    X = rng.standard_normal((M, K)).astype(np.float32)
    X[2, rng.choice(K, 400, replace=False)] *= np.float32(1000.0)  # more than the list's 128 entries
    X[5, :] *= np.float32(1e-30)
    X[5, 9] = 3e-20  # the rest's scale 2^s has s > 100
    X[9, 100] = 7e5  # one entry: shed
    b = rng.standard_normal(N).astype(np.float32)
    t = tg.interleaved_blocked_from_dense(W, None, 2, True)
    st = _stats(tg, X, t, b)
    assert st["exact_rows"] == 2 and st["outlier_rows"] == 1 and st["outlier_entries"] == 1, st
    ref_t = orc.interleaved_blocked_from_dense(W, None, 2, True)
    ref = orc.gemm_vectorized_optimal(orc.pad_input(X), ref_t, b, 0.25)
    y = tg.gemm_vectorized_optimal(tg.pad_input(X), t, b, 0.25, method="mma").values
    for r in (2, 5):
        assert np.array_equal(y[r], ref[r]), r
    nw, sc = _bars(y, X, W, b, 0.25)
    assert nw <= TOL and sc <= TOL, (nw, sc)


def test_outlier_rows_do_not_depend_on_the_batch(tg):
    """A row's bits are a function of the row alone: computed alone (MT = 16 kernel), inside a
    tall batch (MT = 64), device-resident or streamed from host memory."""
    rng = np.random.default_rng(13)
    M, K, N = 130, 1536, 384
    W = _w(rng, K, N)
    X = rng.standard_normal((M, K)).astype(np.float32)
    X[:, rng.choice(K, 6, replace=False)] *= np.float32(250.0)
    b = rng.standard_normal(N).astype(np.float32)
    y_dev = _gemm(tg, X, W, b, 0.25, device=True).values
    y_host = _gemm(tg, X, W, b, 0.25).values  # host X: streamed in row chunks
    assert np.array_equal(y_dev, y_host)
    for r in (0, 64, 129):
        y1 = _gemm(tg, X[r:r + 1].copy(), W, b, 0.25).values
        assert np.array_equal(y1[0], y_dev[r]), r
    nw, sc = _bars(y_dev, X, W, b, 0.25)
    assert nw <= TOL and sc <= TOL, (nw, sc)


def test_outliers_with_split_k(tg):
    """Few column blocks and a long K: the GEMM splits K; the last-arriving unit adds the
    listed terms once."""
    rng = np.random.default_rng(14)
    M, K, N = 16, 16384, 128
    W = _w(rng, K, N)
    X = rng.standard_normal((M, K)).astype(np.float32)
    X[:, rng.choice(K, 8, replace=False)] *= np.float32(100.0)
    b = rng.standard_normal(N).astype(np.float32)
    y = tg.gemm_base(X, tg.tcsc_from_dense(W), b, method="mma").values
    nw, sc = _bars(y, X, W, b)
    assert nw <= TOL and sc <= TOL, (nw, sc)


@pytest.mark.parametrize("seed", range(6))
def test_heavy_tailed_rows_fuzz(tg, seed):
    """Random mixtures of magnitudes (student-t tails, scattered spikes, per-row scales)."""
    rng = np.random.default_rng(100 + seed)
    M, K, N = int(rng.integers(1, 90)), int(rng.integers(300, 3000)), int(rng.integers(40, 300))
    W = _w(rng, K, N, float(rng.uniform(0.3, 0.9)))
    X = rng.standard_t(df=float(rng.uniform(1.2, 3.0)), size=(M, K)).astype(np.float32)
    X *= np.exp(rng.uniform(-20, 20, size=(M, 1))).astype(np.float32)
    spikes = rng.random((M, K)) < 2e-3
    X[spikes] *= np.float32(rng.uniform(50, 5000))
    b = rng.standard_normal(N).astype(np.float32)
    t = tg.tcsc_from_dense(W)
    y = tg.gemm_base(X, t, b, method="mma").values
    nw, sc = _bars(y, X, W, b)
    assert nw <= TOL and sc <= TOL, (seed, nw, sc)


@pytest.mark.parametrize("tag", ["base", "unrolled", "blocked", "interleaved_blocked", "compressed", "vertical",
                                 "horizontal", "vectorized_optimal"])
def test_every_registry_variant_with_outlier_rows(tg, tag):
    """Every registry tag (kernels/__init__.py:98-198) on the tensor-core path with outlier
    channels, a row that cannot shed (exact walk of that variant's own order) and plain rows."""
    rng = np.random.default_rng(sum(map(ord, tag)))
    M, K, N = 37, 1300, 96
    W = _w(rng, K, N)
    X = rng.standard_normal((M, K)).astype(np.float32)
    X[:30, rng.choice(K, 5, replace=False)] *= np.float32(200.0)      # rows 0-29: five outlier channels
    X[31, :] *= np.float32(1e-33)                                      # row 31 cannot shed: the rest's scale
    X[31, 7] = np.float32(3e-20)                                       # is outside the epilogue's range
    b = rng.standard_normal(N).astype(np.float32)
    spec = tg.get_variant(tag)
    alpha = 0.25 if spec.supports_alpha else None
    cfg = tg.GemmConfig(method="mma", alpha=alpha, b=512)
    y = tg.run_variant(tag, X, W, b, cfg).values
    nw, sc = _bars(y, X, W, b, alpha)
    assert nw <= TOL and sc <= TOL, (tag, nw, sc)
    # the row on the exact walk is bit-identical with the variant's gather path
    y_g = tg.run_variant(tag, X, W, b, tg.GemmConfig(method="gather", alpha=alpha, b=512)).values
    assert np.array_equal(y[31], y_g[31]), tag
    # integer-valued twin: bit-exact everywhere (outlier rows included)
    Xi = rng.integers(-6, 7, size=(M, K)).astype(np.float32)
    Xi[:30, rng.choice(K, 5, replace=False)] *= np.float32(300.0)
    bi = rng.integers(-3, 4, size=N).astype(np.float32)
    yi = tg.run_variant(tag, Xi, W, bi, cfg).values
    yg = tg.run_variant(tag, Xi, W, bi, tg.GemmConfig(method="gather", alpha=alpha, b=512)).values
    assert np.array_equal(yi, yg), tag


def test_outlier_rows_without_an_exact_format(tg):
    """tg_gemm_tiles with exact == NULL (no reference-order format to walk): shed rows still get
    their listed terms, and a row whose rest is out of the epilogue's scale range keeps all
    its entries in the limbs (the fp64 recombination then sees the whole row)."""
    import ctypes

    from paper_2510_06957_b200 import _native as nat

    rng = np.random.default_rng(77)
    M, K, N = 24, 1024, 128
    W = _w(rng, K, N, 0.5)
    X = rng.standard_normal((M, K)).astype(np.float32)
    X[:, rng.choice(K, 4, replace=False)] *= np.float32(300.0)   # every row sheds four entries
    X[7, :] *= np.float32(1e-33)                                 # the rest of row 7: scale 2^s with s > 100
    X[7, 3] = np.float32(2e-20)
    b = rng.standard_normal(N).astype(np.float32)
    t = tg.tcsc_from_dense(torch.from_numpy(W).cuda())
    tiles = t.tiles()
    dX, db = torch.from_numpy(X).cuda(), torch.from_numpy(b).cuda()
    y = torch.empty((M, N), dtype=torch.float32, device="cuda")
    L = nat.load()
    ws = torch.empty(L.tg_gemm_workspace_bytes(M, K, N), dtype=torch.uint8, device="cuda")
    flags = torch.zeros(6, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    P = lambda v: ctypes.c_void_p(v.data_ptr())
    nat.call("tg_gemm_tiles", P(dX), M, K, K, P(tiles), N, P(db), P(y), N, 0, 0.0, None, P(ws), ws.numel(),
             P(flags), st)
    torch.cuda.synchronize()
    nw, sc = _bars(y.cpu().numpy(), X, W, b)
    assert nw <= TOL and sc <= TOL, (nw, sc)
