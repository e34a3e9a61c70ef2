"""Fused shard assembly (peer scatter) on one GPU.

``PeerYBuffers.loopback`` gives every "rank" its own full-width Y buffer on
the one device of this box, with the same peer tables, kernel epilogue and
arrival counters a multi-GPU job uses (NVLink peers become local pointers).
All shard GEMMs are launched before any wait, so no kernel ever waits on a
kernel that has not been queued ahead of it.

Bar: every rank's assembled Y equals the unsharded tensor-core GEMM bit for
bit (output columns are independent and the X limb split is per row), over
both epilogue store paths (smem tile + TMA store + 16-byte peer stores, and
direct stores when a shard offset is not 4-aligned or at MT = 80), split-K,
PReLU and the exact-order wide-row fix-up; over several steps (slot
alternation, counter and epoch reuse); and the wait gives up instead of
hanging when a rank never arrives.
"""

from __future__ import annotations

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


def _setup(tg, M, K, N, seed, wide=False, integer=False):
    g = torch.Generator(device="cuda").manual_seed(seed)
    W = torch.randint(-1, 2, (K, N), device="cuda", generator=g, dtype=torch.int8)
    if integer:
        X = torch.randint(-8, 9, (M, K), device="cuda", generator=g).float()
    else:
        X = torch.randn((M, K), device="cuda", generator=g)
    if wide:
        X[1, 0] = 3e4  # one huge entry: the row leaves the limb range -> exact-order fix-up
        X[2] *= 1e-30
    b = torch.randint(-8, 9, (N,), device="cuda", generator=g).float() if integer else \
        torch.randn((N,), device="cuda", generator=g)
    return W, X, b


def _runner(tg, W, X, b, alpha, cols=None, **kw):
    from paper_2510_06957_b200.kernels import GemmRunner

    Wc = W if cols is None else W[:, cols].contiguous()
    bc = b if cols is None else b[cols].contiguous()
    t = tg.tcsc_from_dense(tg.TernaryDense(Wc))
    return GemmRunner("base", X, t, bc, method="mma", alpha=alpha, **kw)


def _full(tg, W, X, b, alpha):
    r = _runner(tg, W, X, b, alpha)
    r.launch()
    return r.y.clone()


CASES = [
    # (M, K, N, world, alpha, wide)
    (10, 300, 256, 2, None, False),     # MT 16, TMA tile path, 4-aligned offsets
    (40, 1000, 1000, 3, 0.25, False),   # ragged shards: offsets 334, 667 -> direct stores + peer stores
    (64, 8192, 512, 2, None, False),    # split-K
    (33, 600, 130, 4, 0.1, True),       # wide rows (fix-up), N % 4 != 0
    (2080, 256, 384, 2, None, False),   # MT = 80: direct stores only
]


@pytest.mark.parametrize("M,K,N,world,alpha,wide", CASES)
def test_loopback_scatter_matches_unsharded(tg, M, K, N, world, alpha, wide):
    from paper_2510_06957_b200.peer import PeerYBuffers, ScatterGemm

    W, X, b = _setup(tg, M, K, N, seed=M * 131 + N + world, wide=wide)
    ref = _full(tg, W, X, b, alpha)
    views = PeerYBuffers.loopback(M, N, world)
    gems = [ScatterGemm(lambda out, scatter, v=v: _runner(tg, W, X, b, alpha, cols=v.shard.slice(), out=out,
                                                          scatter=scatter), v) for v in views]
    try:
        for step in range(3):
            slot = gems[0].slot
            for v in views:
                v.y(slot).fill_(float("nan"))
            torch.cuda.synchronize()
            for gm in gems:  # every rank's GEMM first ...
                gm.runners[gm.slot].launch()
            for gm in gems:  # ... then every rank's wait
                gm.bufs.wait()
                gm.n += 1
            torch.cuda.synchronize()
            for v in views:
                assert torch.equal(v.y(slot), ref), (step, v.rank)
                assert not v.timed_out()
                hdr = v.header.cpu().numpy().view(np.uint32)
                assert list(hdr[:world]) == [step + 1] * world
                assert hdr[32] == 0 and hdr[33] == step + 1  # CTA counter reset, epoch advanced
    finally:
        views[0].close()


def test_world1_scatter_equals_plain_call(tg):
    """A single rank (no process group): the scatter path writes only its own Y."""
    from paper_2510_06957_b200.peer import PeerYBuffers, ScatterGemm

    M, K, N = 100, 2000, 700
    W, X, b = _setup(tg, M, K, N, seed=7, integer=True)
    ref = _full(tg, W, X, b, 0.5)
    bufs = PeerYBuffers(M, N)
    gm = ScatterGemm(lambda out, scatter: _runner(tg, W, X, b, 0.5, out=out, scatter=scatter), bufs)
    try:
        for _ in range(4):
            y = gm.step()
            torch.cuda.synchronize()
            assert torch.equal(y, ref)
        # integer X: bit-exact against fp64 too
        exact = X.double() @ W.double() + b.double()
        exact = torch.where(exact > 0, exact, 0.5 * exact).float()
        assert torch.equal(ref, exact)
    finally:
        bufs.close()


def test_scatter_graph_replay(tg):
    """Captured GEMM + wait replays: counters live in device memory, so replays stay in step."""
    from paper_2510_06957_b200.peer import PeerYBuffers, ScatterGemm

    M, K, N = 48, 512, 384
    W, X, b = _setup(tg, M, K, N, seed=11)
    ref = _full(tg, W, X, b, None)
    bufs = PeerYBuffers(M, N, slots=1)
    gm = ScatterGemm(lambda out, scatter: _runner(tg, W, X, b, None, out=out, scatter=scatter), bufs)
    try:
        r = gm.runners[0]
        r.pin_workspace()
        gm.step()
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                r.launch()
                bufs.wait()
        torch.cuda.current_stream().wait_stream(s)
        for _ in range(5):
            bufs.y(0).zero_()
            g.replay()
        torch.cuda.synchronize()
        assert torch.equal(bufs.y(0), ref)
        hdr = bufs.header.cpu().numpy().view(np.uint32)
        assert hdr[0] == 6 and hdr[33] == 6 and not bufs.timed_out()
    finally:
        bufs.close()


def test_wait_gives_up_when_a_rank_never_arrives(tg):
    """Rank 1 never runs its GEMM: rank 0's wait must time out (~10 s), not hang the GPU."""
    from paper_2510_06957_b200.peer import PeerYBuffers, ScatterGemm

    M, K, N = 16, 128, 256
    W, X, b = _setup(tg, M, K, N, seed=3)
    views = PeerYBuffers.loopback(M, N, 2)
    try:
        gm = ScatterGemm(lambda out, scatter: _runner(tg, W, X, b, None, cols=views[0].shard.slice(), out=out,
                                                      scatter=scatter), views[0])
        res = gm.result()
        torch.cuda.synchronize()
        assert views[0].timed_out()
        with pytest.raises(RuntimeError, match="timed out"):
            res.values  # the result path reports the incomplete assembly
        hdr = views[1].header.cpu().numpy().view(np.uint32)
        assert hdr[0] == 1  # rank 0 still delivered its arrival to rank 1
    finally:
        views[0].close()


def test_scatter_rejects_bad_descriptors(tg):
    from paper_2510_06957_b200 import _native as nat
    from paper_2510_06957_b200.errors import ParameterError
    from paper_2510_06957_b200.peer import PeerYBuffers

    M, K, N = 8, 64, 64
    W, X, b = _setup(tg, M, K, N, seed=1)
    bufs = PeerYBuffers(M, N)
    try:
        r = _runner(tg, W, X, b, None, out=bufs.block(0), scatter=bufs.descriptor(0))
        d = nat.TgPeerScatter.from_buffer_copy(bufs.descriptor(0))
        d.col_off = 10  # block would run past the row pitch
        r.scatter = d
        with pytest.raises(ParameterError):
            r.launch()
        d.col_off, d.rank = 0, 1  # rank >= world
        with pytest.raises(ParameterError):
            r.launch()
        with pytest.raises(ParameterError):
            _runner(tg, W, X, b, None, out=torch.empty((M, N + 1), device="cuda"))
    finally:
        bufs.close()


FUZZ = 30


@pytest.mark.parametrize("i", range(FUZZ))
def test_loopback_scatter_fuzz(tg, i):
    """Random shapes, world sizes, shard offsets (aligned or not), PReLU and wide rows:
    every loopback rank's assembled Y equals the unsharded GEMM bit for bit, two steps."""
    from paper_2510_06957_b200.peer import PeerYBuffers, ScatterGemm

    rng = np.random.default_rng(20000 + i)
    world = int(rng.integers(1, 5))
    M = int(rng.integers(1, 260))
    K = int(rng.integers(1, 2500))
    N = int(rng.integers(world, 1400))
    alpha = 0.25 if rng.random() < 0.5 else None
    wide = bool(rng.random() < 0.3) and M >= 3 and K >= 2
    W, X, b = _setup(tg, M, K, N, seed=30000 + i, wide=wide)
    ref = _full(tg, W, X, b, alpha)
    views = PeerYBuffers.loopback(M, N, world)
    gems = [ScatterGemm(lambda out, scatter, v=v: _runner(tg, W, X, b, alpha, cols=v.shard.slice(), out=out,
                                                          scatter=scatter), v) for v in views]
    try:
        for step in range(2):
            slot = gems[0].slot
            for v in views:
                v.y(slot).fill_(float("nan"))
            torch.cuda.synchronize()
            for gm in gems:
                gm.runners[gm.slot].launch()
            for gm in gems:
                gm.bufs.wait()
                gm.n += 1
            torch.cuda.synchronize()
            for v in views:
                assert torch.equal(v.y(slot), ref), (i, step, v.rank, M, K, N, world)
                assert not v.timed_out()
    finally:
        views[0].close()
