"""Tensor-core path: every code path of the persistent tcgen05 kernel against
an fp64 reference on the device.

The shapes pick each branch on purpose:
* MT = 16 / 32 / 48 / 64 (M <= 16, <= 32, <= 48, larger), padded rows;
* an odd number of 128-k chunks (a half-filled last 256-k stage), K = 1;
* cluster sizes 1 / 2 / 4 with ghost column blocks (NB not a multiple of CS);
* split-K with the last-arriving reduction (few tiles, long K);
* N not a multiple of 4 (direct Y stores instead of the TMA store);
* the three X-split kernels (register-resident, smem-staged K > 16384,
  global multi-pass K > 32768).

Integer-valued X must be bit-exact (exact limbs, exact integer accumulation);
real X within the 1e-5 normwise / |terms|-scaled bars.
"""

from __future__ import annotations


import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def tg():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2510_06957_b200 as m

    return m


def _ref(X, W, b, alpha=None):
    y = X.double() @ W.double() + b.double()
    if alpha is not None:
        y = torch.where(y > 0, y, alpha * y)
    return y


CASES = [
    # (M, K, N)
    (1, 1, 4),
    (10, 100, 130),       # MT 16, one chunk, N % 4 != 0 -> direct stores
    (30, 384, 520),       # MT 32, 3 chunks (odd), NB = 5 -> ghost blocks with CS = 4
    (40, 257, 256),       # MT 48
    (100, 1000, 384),     # MT 64, padded rows, NB = 3
    (64, 8192, 128),      # one tile, long K -> split-K
    (16, 4096, 1024),     # decode-like, split-K
    (300, 640, 1000),     # NB = 8, N % 128 != 0
    (24, 20000, 64),      # K > 16384: split staged without shared memory
    (8, 40000, 32),       # K > 32768: multi-pass split
]


@pytest.mark.parametrize("M,K,N", CASES)
def test_tensor_core_paths(tg, M, K, N):
    g = torch.Generator(device="cuda").manual_seed(M * 7919 + K * 31 + N)
    W = torch.randint(-1, 2, (K, N), device="cuda", generator=g, dtype=torch.int8)
    Xi = torch.randint(-8, 9, (M, K), device="cuda", generator=g).float()
    bi = torch.randint(-8, 9, (N,), device="cuda", generator=g).float()
    t = tg.tcsc_from_dense(tg.TernaryDense(W))
    y = tg.gemm_base(Xi, t, bi, method="mma").device_values
    assert torch.equal(y.double(), _ref(Xi, W, bi)), (M, K, N)
    Xr = torch.randn((M, K), device="cuda", generator=g)
    br = torch.randn((N,), device="cuda", generator=g)
    y = tg.gemm_base(Xr, t, br, method="mma").device_values.double()
    ref = _ref(Xr, W, br)
    nw = float((y - ref).abs().max() / ref.abs().max().clamp_min(1e-30))
    scale = Xr.abs().double() @ W.abs().double() + br.abs().double()
    sc = float(((y - ref).abs() / scale.clamp_min(1e-30)).max())
    assert nw <= TOL and sc <= TOL, (M, K, N, nw, sc)


def test_cluster_sizes_agree(tg, monkeypatch):
    """The X-limb multicast (cluster of 1, 2 or 4 CTAs) must not change a single bit."""
    from paper_2510_06957_b200.workloads import make_inputs

    W, X, b = make_inputs("cfg2", M=90)
    W, b = np.ascontiguousarray(W[:, :1164]), b[:1164]  # NB = 10: ghost blocks for CS = 4
    t = tg.interleaved_blocked_from_dense(torch.from_numpy(W).cuda(), None, 2, True)
    Xp = tg.pad_input(torch.from_numpy(X).cuda())
    ys = []
    for cs in ("1", "2", "4"):
        monkeypatch.setenv("TG_MMA_CLUSTER", cs)  # read whenever a launch is planned
        ys.append(tg.gemm_vectorized_optimal(Xp, t, b, 0.25, method="mma").device_values.clone())
    assert torch.equal(ys[0], ys[1]) and torch.equal(ys[0], ys[2])


def test_wide_rows_without_exact_format_use_fp64(tg):
    """tg_gemm_tiles with exact == NULL: rows outside the fp32 scale range take the
    fp64 epilogue branch (no exact-order fix-up available) and stay accurate."""
    import ctypes

    from paper_2510_06957_b200 import _native as nat

    M, K, N = 20, 300, 64
    g = torch.Generator(device="cuda").manual_seed(5)
    W = torch.randint(-1, 2, (K, N), device="cuda", generator=g, dtype=torch.int8)
    X = torch.randn((M, K), device="cuda", generator=g)
    X[3] *= 1e-35   # 2^-s far below the float range
    X[7] *= 1e35    # and far above
    b = torch.zeros(N, device="cuda")
    t = tg.tcsc_from_dense(tg.TernaryDense(W))
    tiles = t.tiles()
    y = torch.empty((M, N), device="cuda")
    L = nat.load()
    ws = torch.empty(L.tg_gemm_workspace_bytes(M, K, N), dtype=torch.uint8, device="cuda")
    nat.call("tg_gemm_tiles", ctypes.c_void_p(X.data_ptr()), M, K, K, ctypes.c_void_p(tiles.data_ptr()), N,
             ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(y.data_ptr()), N, 0, 0.0, None,
             ctypes.c_void_p(ws.data_ptr()), ws.numel(), None, torch.cuda.current_stream().cuda_stream)
    ref = _ref(X, W, b)
    for m in range(M):
        den = ref[m].abs().max()
        err = float((y[m].double() - ref[m]).abs().max() / den) if den > 0 else float(y[m].abs().max())
        assert err <= TOL, (m, err)


@pytest.mark.parametrize("bad", [float("inf"), float("-inf"), float("nan")])
def test_nonfinite_input_is_reported(tg, bad):
    """A non-finite X entry (the reference rejects it when constructing DenseMatrix,
    dense.py:77) is flagged by the tensor-core split and raised on first host access."""
    from paper_2510_06957_b200.errors import ParameterError

    M, K, N = 20, 256, 128
    W = torch.randint(-1, 2, (K, N), device="cuda", dtype=torch.int8)
    X = torch.randn((M, K), device="cuda")
    X[5, 7] = bad
    t = tg.tcsc_from_dense(tg.TernaryDense(W))
    with pytest.raises(ParameterError):
        tg.gemm_base(X, t, torch.zeros(N, device="cuda"), method="mma").values


@pytest.mark.parametrize("xmode", [None, "0", "1"])
@pytest.mark.parametrize("method", ["mma", "gather"])
def test_host_input_is_streamed_bit_exact(tg, method, xmode, monkeypatch):
    """Host X (pinned tensor, numpy) goes through the row-chunked H2D / GEMM / D2H
    pipeline (or, for small pinned X, is read in place by the X split; xmode forces
    copies "0" / in-place "1"); every entry point must give the bits of the
    device-resident call."""
    from paper_2510_06957_b200 import _native as nat

    if xmode is not None:
        monkeypatch.setenv("TG_HOST_ZEROCOPY_X", xmode)  # read by every host call

    M, K, N = 700, 1024, 320   # 2.9 MB of X: several chunks, a ragged last one
    rng = np.random.default_rng(3)
    W = rng.integers(-1, 2, size=(K, N)).astype(np.int8)
    X = rng.standard_normal((M, K)).astype(np.float32)
    X[5, 3] = 4e4  # a wide row in the middle of a chunk
    b = rng.standard_normal(N).astype(np.float32)
    assert nat.load().tg_gemm_host_workspace_bytes(M, K + 1, N) > nat.load().tg_gemm_workspace_bytes(192, K + 1, N)
    Wd = torch.from_numpy(W).cuda()
    Xd = torch.from_numpy(X).cuda()
    Xpin = torch.from_numpy(X).pin_memory()
    cfg = tg.GemmConfig(uf=2, mr=2, alpha=0.25)
    t = tg.tcsc_from_dense(tg.TernaryDense(Wd))
    bl = tg.blocked_from_dense(tg.TernaryDense(Wd), 256)
    ib = tg.interleaved_blocked_from_dense(Wd, 256, 2, False)
    ibs = tg.interleaved_blocked_from_dense(Wd, 256, 2, True)
    calls = [
        lambda x: tg.gemm_base(x, t, b, method=method),
        lambda x: tg.gemm_unrolled(x, t, b, cfg, method=method),
        lambda x: tg.gemm_blocked(x, bl, b, cfg, method=method),
        lambda x: tg.gemm_interleaved_blocked(x, ib, b, method=method),
        lambda x: tg.gemm_vectorized_optimal(tg.pad_input(x), ibs, b, 0.25, method=method),
    ]
    for i, call in enumerate(calls):
        ref = call(Xd).values
        for x in (Xpin, X):
            y = call(x)
            assert np.array_equal(y.values, ref), (i, type(x))
            assert torch.equal(y.device_values.cpu(), torch.from_numpy(ref))


def test_host_streaming_graph_replay(tg):
    """Repeated host-streamed calls replay the library's CUDA graph of the first
    (same pointers): new X contents in the same pinned buffer, results kept
    alive (new Y pointers: a fresh capture), counted mode, a side stream, and a
    non-finite X in a replay must all behave exactly like the direct enqueue."""
    from paper_2510_06957_b200.errors import ParameterError

    M, K, N = 512, 1024, 512
    rng = np.random.default_rng(11)
    W = rng.integers(-1, 2, size=(K, N)).astype(np.int8)
    b = rng.standard_normal(N).astype(np.float32)
    Wd = torch.from_numpy(W).cuda()
    ibs = tg.interleaved_blocked_from_dense(Wd, None, 2, True)
    Xpin = torch.empty((M, K)).pin_memory()
    kept = []
    for it in range(6):
        X = rng.standard_normal((M, K)).astype(np.float32)
        Xpin.copy_(torch.from_numpy(X))
        yr, ops_ref = tg.gemm_vectorized_optimal(tg.pad_input(torch.from_numpy(X).cuda()), ibs, b, 0.25,
                                                 counted=True)
        ref = yr.values.copy()
        y, ops = tg.gemm_vectorized_optimal(tg.pad_input(Xpin), ibs, b, 0.25, counted=True)
        assert np.array_equal(y.values, ref), it
        assert ops == ops_ref, (it, ops, ops_ref)
        if it % 2:
            kept.append(y)  # Y stays alive: the next call gets another device Y
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        y2 = tg.gemm_vectorized_optimal(tg.pad_input(Xpin), ibs, b, 0.25).values
    assert np.array_equal(y2, ref)
    Xpin[100, 3] = float("nan")
    with pytest.raises(ParameterError):
        tg.gemm_vectorized_optimal(tg.pad_input(Xpin), ibs, b, 0.25).values
    Xpin[100, 3] = 0.0
    assert np.isfinite(tg.gemm_vectorized_optimal(tg.pad_input(Xpin), ibs, b, 0.25).values).all()


@pytest.mark.parametrize("xmode", [None, "1"])
@pytest.mark.parametrize("chunks", ["8", "3", "1"])
def test_host_streaming_multi_chunk(tg, chunks, xmode, monkeypatch):
    """X large enough for several row chunks (ragged last one): in-order copy streams
    (or the chunks' X splits reading the pinned X in place, xmode "1"), side-by-side
    chunk GEMMs on SM shares, graph replay of the whole pipeline; every chunking gives
    the device-resident call's bits (wide rows included)."""
    monkeypatch.setenv("TG_HOST_CHUNKS", chunks)
    if xmode is not None:
        monkeypatch.setenv("TG_HOST_ZEROCOPY_X", xmode)
    M, K, N = 2100, 2048, 640   # 17 MB of X: 8 chunks -> 7 of 320 rows (the last 180); 3 -> 704 rows
    rng = np.random.default_rng(21)
    W = rng.integers(-1, 2, size=(K, N)).astype(np.int8)
    X = rng.standard_normal((M, K)).astype(np.float32)
    # wide rows on both sides of the chunk boundaries of either plan (320- and 704-row chunks),
    # inside a chunk, and the first and last rows
    for r in (0, 319, 320, 703, 704, 1300, 1407, 1408, 2099):
        X[r, 9] = 3e4
    b = rng.standard_normal(N).astype(np.float32)
    Wd = torch.from_numpy(W).cuda()
    ibs = tg.interleaved_blocked_from_dense(Wd, None, 2, True)
    ref = tg.gemm_vectorized_optimal(tg.pad_input(torch.from_numpy(X).cuda()), ibs, b, 0.25).values.copy()
    Xpin = torch.from_numpy(X).pin_memory()
    for it in range(3):  # first call direct, second captured, third replayed
        y = tg.gemm_vectorized_optimal(tg.pad_input(Xpin), ibs, b, 0.25)
        assert np.array_equal(y.values, ref), (chunks, it)
    t = tg.tcsc_from_dense(tg.TernaryDense(Wd))
    ref_b = tg.gemm_base(torch.from_numpy(X).cuda(), t, b).values.copy()
    assert np.array_equal(tg.gemm_base(X, t, b).values, ref_b)  # pageable numpy X


@pytest.mark.parametrize("xmode", ["0", "1"])
@pytest.mark.parametrize("zerocopy_pitch", [False, True])
def test_host_streaming_c_abi_pitched(tg, zerocopy_pitch, xmode, monkeypatch):
    """tg_gemm_tiles_host through the C ABI with pitched buffers: host X of pitch K+1
    (2-D copies), a padded device staging X (ldx_dev > K: its slot columns are zeroed),
    a device Y of pitch N+3, and a host Y whose pitch either rules out the zero-copy
    store (N+1: 2-D D2H copies) or allows it (N+4).  Y and the status words must equal the
    device-resident call.  xmode: X copied in ("0") or read in place by the split ("1",
    a host pitch of K+1 floats: unaligned rows)."""
    import ctypes

    from paper_2510_06957_b200 import _native as nat

    monkeypatch.setenv("TG_HOST_ZEROCOPY_X", xmode)
    M, K, N = 600, 1536, 256
    rng = np.random.default_rng(33)
    W = rng.integers(-1, 2, size=(K, N)).astype(np.int8)
    X = rng.standard_normal((M, K)).astype(np.float32)
    b = rng.standard_normal(N).astype(np.float32)
    Wd = torch.from_numpy(W).cuda()
    t = tg.tcsc_from_dense(tg.TernaryDense(Wd))
    ref = tg.gemm_base(torch.from_numpy(X).cuda(), t, b).values
    L = nat.load()
    hx = torch.zeros((M, K + 1)).pin_memory()
    hx[:, :K] = torch.from_numpy(X)
    xd = torch.full((M, K + 5), 7.0, device="cuda")       # slot columns must be zeroed by the call
    yd = torch.empty((M, N + 3), device="cuda")
    ldyh = N + 4 if zerocopy_pitch else N + 1
    yh = torch.full((M, ldyh), -1.0).pin_memory()
    fl = torch.zeros(6, dtype=torch.int32, device="cuda")
    fh = torch.full((6,), 99, dtype=torch.int32).pin_memory()
    ws = torch.empty(L.tg_gemm_host_workspace_bytes(M, K, N), dtype=torch.uint8, device="cuda")
    bd = torch.from_numpy(b).cuda()
    r = tg.kernels.GemmRunner("base", xd, t, bd, method="mma")
    for _ in range(3):  # direct, captured, replayed
        nat.call("tg_gemm_tiles_host", ctypes.c_void_p(hx.data_ptr()), M, K, K + 1, ctypes.c_void_p(xd.data_ptr()),
                 K + 5, ctypes.c_void_p(t.tiles().data_ptr()), N, ctypes.c_void_p(bd.data_ptr()),
                 ctypes.c_void_p(yd.data_ptr()), N + 3, ctypes.c_void_p(yh.data_ptr()), ldyh, 0, 0.0,
                 ctypes.byref(r.exact), ctypes.c_void_p(ws.data_ptr()), ws.numel(), ctypes.c_void_p(fl.data_ptr()),
                 ctypes.c_void_p(fh.data_ptr()), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert np.array_equal(yh.numpy()[:, :N], ref)
        assert torch.equal(yd[:, :N].cpu(), torch.from_numpy(ref))
        assert bool((xd[:, K:] == 0).all())
        assert int(fh[0]) == 0 and int(fh[1]) == 0


def test_host_streaming_more_than_eight_chunks(tg, monkeypatch):
    """26 MB of X with TG_HOST_CHUNKS=16: 12 row chunks (the plan very large X takes by
    default, tg_capi.cu host_plan) through the 4 side streams and 16 chunk events; the result
    equals the device-resident call bit for bit, replayed from the library's graph too."""
    monkeypatch.setenv("TG_HOST_CHUNKS", "16")
    rng = np.random.default_rng(33)
    M, K, N = 3200, 2048, 256
    W = rng.integers(-1, 2, size=(K, N)).astype(np.int8)
    X = rng.standard_normal((M, K)).astype(np.float32)
    X[::257, 11] = 4e4  # a few rows shed an outlier entry
    b = rng.standard_normal(N).astype(np.float32)
    ib = tg.interleaved_blocked_from_dense(torch.from_numpy(W).cuda())
    ref = tg.gemm_interleaved_blocked(tg.DenseMatrix(torch.from_numpy(X).cuda()), ib, b, method="mma").values.copy()
    Xpin = torch.from_numpy(X).pin_memory()
    for _ in range(3):  # direct, captured, replayed
        y = tg.gemm_interleaved_blocked(Xpin, ib, b, method="mma").values
        assert np.array_equal(y, ref)
