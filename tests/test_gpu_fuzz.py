"""Seeded randomized sweep of the tensor-core path: random shapes (M, K, N), densities
and variants, integer-valued X (the limbs and the int32 accumulation are exact, so Y
must equal the reference-order gather path bit for bit), device-resident and
host-streamed inputs.  Catches tile / cluster / split-K / decoder-group / chunking
corner cases that the hand-picked shapes of test_gpu_paths.py may miss."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

CASES = int(__import__("os").environ.get("TG_FUZZ_CASES", "60"))


@pytest.fixture(scope="module")
def tg():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2510_06957_b200 as m

    return m


def _case(i):
    rng = np.random.default_rng(1000 + i)
    M = int(rng.choice([1, 3, 16, 17, 31, 48, 64, 65, 100, 129, 200, 257, 513]))
    K = int(rng.choice([1, 5, 127, 128, 129, 300, 512, 1000, 2048, 4100]))
    N = int(4 * rng.integers(1, 200))
    dens = float(rng.choice([0.02, 0.1, 0.5, 0.9]))
    u = rng.random((K, N))
    W = np.where(u < dens / 2, 1, np.where(u < dens, -1, 0)).astype(np.int8)
    X = rng.integers(-8, 9, size=(M, K)).astype(np.float32)
    b = rng.integers(-8, 9, size=N).astype(np.float32)
    variant = str(rng.choice(["base", "blocked", "interleaved_blocked", "vectorized_optimal", "horizontal"]))
    alpha = 0.25 if variant in ("vectorized_optimal", "horizontal") and rng.random() < 0.7 else None
    return M, K, N, W, X, b, variant, alpha


@pytest.mark.parametrize("i", range(CASES))
def test_fuzz_mma_equals_reference_order(tg, i):
    M, K, N, W, X, b, variant, alpha = _case(i)
    Wd = torch.from_numpy(W).cuda()
    cfg = tg.GemmConfig(alpha=alpha, b=max(1, K // 2) if variant == "blocked" else None)
    spec = tg.get_variant(variant)
    fmt = spec.build(tg.TernaryDense(Wd), cfg)
    outs, counts = {}, {}
    for method in ("gather", "mma"):
        c = tg.GemmConfig(alpha=alpha, method=method, b=cfg.b)
        xd = spec.prepare(tg.DenseMatrix(torch.from_numpy(X).cuda()))
        y, ops = spec.run(xd, fmt, tg.BiasVector(b), c, True)
        outs[method], counts[method] = y.values.copy(), ops
    assert np.array_equal(outs["mma"], outs["gather"]), (M, K, N, variant, alpha)
    assert counts["mma"] == counts["gather"], (M, K, N, variant, alpha, counts)  # adds and PReLU mults
    # the public call on host memory (streamed when large enough) gives the same bits
    c = tg.GemmConfig(alpha=alpha, method="mma", b=cfg.b)
    xh = spec.prepare(tg.DenseMatrix(torch.from_numpy(X).pin_memory()))
    y = spec.run(xh, fmt, tg.BiasVector(b), c, False).values
    assert np.array_equal(y, outs["gather"]), (M, K, N, variant, alpha, "host")


@pytest.mark.parametrize("i", range(CASES))
def test_fuzz_mma_real_x_within_tolerance(tg, i):
    """Real-valued X (some rows with a wide dynamic range): the tensor-core path stays
    within the 1e-5 normwise bar of the fp64 oracle (TOL as in test_gpu_parity.py)."""
    TOL = 1e-5
    M, K, N, W, _, b, variant, alpha = _case(i)
    rng = np.random.default_rng(5000 + i)
    X = rng.standard_normal((M, K)).astype(np.float32)
    if M > 2 and K > 2:
        X[M // 2, K // 3] *= 1e4  # a wide row: exact-order fix-up
    b = b + rng.standard_normal(N).astype(np.float32)
    Wd = torch.from_numpy(W).cuda()
    c = tg.GemmConfig(alpha=alpha, method="mma", b=max(1, K // 2) if variant == "blocked" else None)
    spec = tg.get_variant(variant)
    fmt = spec.build(tg.TernaryDense(Wd), c)
    y = spec.run(spec.prepare(tg.DenseMatrix(torch.from_numpy(X).cuda())), fmt, tg.BiasVector(b), c, False).values
    ref = torch.from_numpy(X).cuda().double() @ Wd.double() + torch.from_numpy(b).cuda().double()
    if alpha is not None:
        ref = torch.where(ref > 0, ref, alpha * ref)
    ref = ref.cpu().numpy()
    den = np.abs(ref).max()
    err = np.abs(y.astype(np.float64) - ref).max() / den if den > 0 else np.abs(y).max()
    assert err <= TOL, (M, K, N, variant, alpha, err)


@pytest.mark.parametrize("i", range(CASES))
def test_fuzz_auto_adversarial_rows(tg, i):
    """Rows built to stress a per-row fixed-point grid (bimodal magnitudes, a few large
    outliers, log-uniform magnitudes over e^+-8, tiny or huge rows) with sparse and dense W.
    Under method="auto" every output must meet both bars of SURVEY 8(c): normwise <= 1e-5
    and |terms|-scaled elementwise <= 1e-5 (outputs with few terms take the exact gather)."""
    TOL = 1e-5
    rng = np.random.default_rng(9000 + i)
    M = int(rng.choice([8, 33, 64, 130]))
    K = int(rng.choice([64, 128, 256, 1024, 4096]))
    N = int(4 * rng.integers(1, 64))
    dens = float(rng.choice([0.02, 0.05, 0.2, 0.5]))
    u = rng.random((K, N))
    W = np.where(u < dens / 2, 1, np.where(u < dens, -1, 0)).astype(np.int8)
    X = rng.standard_normal((M, K)).astype(np.float32)
    pat = i % 4
    if pat == 0:
        X = np.where(rng.random((M, K)) < 0.5, X * 1e4, X).astype(np.float32)
    elif pat == 1:
        for m in range(M):
            X[m, rng.choice(K, size=int(rng.integers(2, 4)), replace=False)] *= 3e3
    elif pat == 2:
        X = (X * np.exp(rng.uniform(-8, 8, size=(M, K)))).astype(np.float32)
    else:
        X *= np.float32(rng.choice([1e-30, 1e-12, 1e12, 1e30]))
    b = rng.standard_normal(N).astype(np.float32) * np.float32(np.abs(X).mean())
    Wd = torch.from_numpy(W).cuda()
    fmt = tg.interleaved_blocked_from_dense(Wd, None, 2, True)
    y = tg.gemm_vectorized_optimal(tg.pad_input(torch.from_numpy(X).cuda()), fmt, b, 0.25).values
    Xd, Wdd, bd = torch.from_numpy(X).double(), torch.from_numpy(W).double(), torch.from_numpy(b).double()
    ref = Xd @ Wdd + bd
    terms = (Xd.abs() @ Wdd.abs() + bd.abs()).numpy()
    ref = torch.where(ref > 0, ref, 0.25 * ref).numpy()
    err = np.abs(y.astype(np.float64) - ref)
    assert err.max() <= TOL * max(np.abs(ref).max(), 1e-300), (i, pat, M, K, N, dens)
    assert (err <= TOL * terms).all(), (i, pat, M, K, N, dens, (err / np.maximum(terms, 1e-300)).max())


@pytest.mark.parametrize("i", range(CASES))
def test_fuzz_device_builders_match_oracle(tg, i):
    """Device builders against the C oracle (itself pinned to the reference) for random
    shapes, block sizes, group sizes and sign balances: every index array bit for bit."""
    from oracle import oracle as orc

    rng = np.random.default_rng(7000 + i)
    K = int(rng.integers(1, 700))
    N = int(4 * rng.integers(1, 80)) if rng.random() < 0.7 else int(rng.integers(1, 300))
    p_pos, p_neg = float(rng.random() * 0.6), float(rng.random() * 0.6)
    u = rng.random((K, N))
    W = np.where(u < p_pos, 1, np.where(u < min(1.0, p_pos + p_neg), -1, 0)).astype(np.int8)
    Wd = tg.TernaryDense(torch.from_numpy(W).cuda())
    B = int(rng.choice([1, 3, 16, 128, 4096])) if rng.random() < 0.8 else None
    g = int(rng.integers(1, 5))

    t, r = tg.tcsc_from_dense(Wd), orc.tcsc_from_dense(W)
    for k in ("col_start_pos", "row_index_pos", "col_start_neg", "row_index_neg"):
        assert np.array_equal(getattr(t, k), r[k]), ("tcsc", k)
    bl, rb = tg.blocked_from_dense(Wd, B), orc.blocked_from_dense(W, B)
    for k in ("col_start_pos", "row_index_pos", "col_start_neg", "row_index_neg"):
        assert np.array_equal(getattr(bl, k), rb[k]), ("blocked", k)
    sym_ok = N % 4 == 0
    for sym in ((False, True) if sym_ok else (False,)):
        ib, ri = tg.interleaved_blocked_from_dense(Wd, B, g, symmetric_cols=sym), \
            orc.interleaved_blocked_from_dense(W, B, g, sym)
        assert np.array_equal(ib.all_indices, ri["all_indices"]), ("ib", sym, K, N, B, g)
        assert np.array_equal(ib.col_segment_ptr, ri["col_segment_ptr"]), ("ib ptr", sym)
    if sym_ok:
        sy, rs = tg.symmetric_from_dense(Wd, g), orc.symmetric_from_dense(W, g)
        assert np.array_equal(sy.indices, rs["indices"]) and np.array_equal(sy.col_ptr, rs["col_ptr"])
    cp, rc = tg.compressed_from_dense(Wd), orc.compressed_from_dense(W)
    assert np.array_equal(cp.codes, rc["codes"])
    # every format decodes back to W on the device
    for f in (t, bl, cp):
        assert np.array_equal(f.to_dense().values, W)


@pytest.mark.parametrize("i", range(CASES))
def test_fuzz_gather_bit_exact_with_reference_kernels(tg, i):
    """The gather path against the C restatement of every reference kernel (pinned bit for
    bit to the reference's own outputs) on real-valued X: identical fp32 bits, for random
    shapes, block sizes, group sizes, unroll factors and row unrolls."""
    from oracle import oracle as orc

    rng = np.random.default_rng(11000 + i)
    M = int(rng.integers(1, 70))
    K = int(rng.integers(1, 600))
    N = int(4 * rng.integers(1, 40))
    u = rng.random((K, N))
    d = float(rng.random())
    W = np.where(u < d / 2, 1, np.where(u < d, -1, 0)).astype(np.int8)
    X = (rng.standard_normal((M, K)) * np.exp(rng.uniform(-3, 3, size=(M, 1)))).astype(np.float32)
    b = rng.standard_normal(N).astype(np.float32)
    Wd = tg.TernaryDense(torch.from_numpy(W).cuda())
    Xd = torch.from_numpy(X).cuda()
    B = int(rng.choice([1, 7, 64, 4096]))
    g = int(rng.integers(1, 4))
    uf = int(rng.integers(1, 9))
    mr = int(rng.choice([1, 2, 4]))
    alpha = 0.25 if rng.random() < 0.5 else None
    G = "gather"
    t, r = tg.tcsc_from_dense(Wd), orc.tcsc_from_dense(W)
    assert np.array_equal(tg.gemm_base(Xd, t, b, method=G).values, orc.gemm_base(X, r, b))
    assert np.array_equal(tg.gemm_unrolled(Xd, t, b, tg.GemmConfig(uf=uf), method=G).values,
                          orc.gemm_unrolled(X, r, b, uf=uf))
    bl, rb = tg.blocked_from_dense(Wd, B), orc.blocked_from_dense(W, B)
    assert np.array_equal(tg.gemm_blocked(Xd, bl, b, tg.GemmConfig(uf=uf, mr=mr), method=G).values,
                          orc.gemm_blocked(X, rb, b, uf=uf, mr=mr))
    ib, ri = tg.interleaved_blocked_from_dense(Wd, B, g), orc.interleaved_blocked_from_dense(W, B, g)
    assert np.array_equal(tg.gemm_interleaved_blocked(Xd, ib, b, method=G).values,
                          orc.gemm_interleaved_blocked(X, ri, b))
    ibs, ris = tg.interleaved_blocked_from_dense(Wd, B, g, True), orc.interleaved_blocked_from_dense(W, B, g, True)
    Xp = orc.pad_input(X)
    assert np.array_equal(tg.gemm_vectorized_optimal(tg.pad_input(Xd), ibs, b, alpha, method=G).values,
                          orc.gemm_vectorized_optimal(Xp, ris, b, alpha))
    sy, rs = tg.symmetric_from_dense(Wd, g), orc.symmetric_from_dense(W, g)
    assert np.array_equal(tg.gemm_vertical(tg.pad_input(Xd), sy, b, alpha, method=G).values,
                          orc.gemm_vertical(Xp, rs, b, alpha))
    assert np.array_equal(tg.gemm_horizontal(tg.pad_input(Xd), sy, b, alpha, method=G).values,
                          orc.gemm_horizontal(Xp, rs, b, alpha))
    cp, rc = tg.compressed_from_dense(Wd), orc.compressed_from_dense(W)
    assert np.array_equal(tg.gemm_compressed(Xd, cp, b, method=G).values, orc.gemm_compressed(X, rc, b))
