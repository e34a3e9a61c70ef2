"""Multi-rank partitioner on CPU: world_size-2 gloo process groups.

The GPU run of this path (bench.py under torchrun) uses NCCL and the CUDA
kernels; here each rank computes its shard with the C oracle (the checker),
and the assembled Y must equal the unsharded oracle output bit for bit:
output columns are independent (kernels/scalar.py:116-127) and 4-aligned
shards keep symmetric groups intact (variants.py:361-376).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc
from paper_2510_06957_b200.partition import ShardedGemm, column_shards, row_shards, split


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_split_shapes():
    assert [(s.start, s.stop) for s in split(10, 3)] == [(0, 4), (4, 7), (7, 10)]
    sh = column_shards(11008, 8, symmetric=True)
    assert all(s.width == 1376 for s in sh)
    sh = column_shards(4100, 8, symmetric=True)
    assert sum(s.width for s in sh) == 4100 and all(s.width % 4 == 0 for s in sh)
    assert max(s.width for s in sh) - min(s.width for s in sh) <= 4
    sh = column_shards(10, 4, symmetric=True)  # 2 groups + tail of 2 over 4 ranks
    assert [s.width for s in sh] == [4, 4, 0, 2]
    assert [s.width for s in row_shards(5, 2)] == [3, 2]
    assert split(0, 3)[0].width == 0


def _worker(rank, world, port, mode, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(7)
        M, K, N = case
        W = rng.integers(-1, 2, size=(K, N)).astype(np.int8)
        X = rng.standard_normal((M, K)).astype(np.float32)
        b = rng.standard_normal(N).astype(np.float32)
        part = ShardedGemm(M, N, mode, symmetric=(N % 4 == 0))

        def compute(sh):
            if mode == "columns":
                Ws, bs, Xs = W[:, sh.slice()], b[sh.slice()], X
            else:
                Ws, bs, Xs = W, b, X[sh.slice()]
            if Ws.shape[1] == 0 or Xs.shape[0] == 0:
                return torch.zeros((Xs.shape[0], Ws.shape[1]), dtype=torch.float32)
            if N % 4 == 0 and Ws.shape[1] % 4 == 0:
                t = orc.interleaved_blocked_from_dense(Ws, 64, 2, True)
                y = orc.gemm_vectorized_optimal(orc.pad_input(Xs), t, bs, 0.25)
            else:
                t = orc.interleaved_blocked_from_dense(Ws, 64, 2, False)
                y = orc.gemm_interleaved_blocked(Xs, t, bs)
            return torch.from_numpy(y)

        y = part.run(compute).numpy()
        if N % 4 == 0:
            ref = orc.gemm_vectorized_optimal(orc.pad_input(X), orc.interleaved_blocked_from_dense(W, 64, 2, True),
                                              b, 0.25)
        else:
            ref = orc.gemm_interleaved_blocked(X, orc.interleaved_blocked_from_dense(W, 64, 2, False), b)
        q.put((rank, bool(np.array_equal(y, ref)), y.shape))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["columns", "rows"])
@pytest.mark.parametrize("case", [(12, 200, 64), (7, 130, 30)])
def test_two_rank_assembly_equals_unsharded(mode, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = sorted(q.get(timeout=10) for _ in procs)
    for p in procs:
        assert p.exitcode == 0
    for rank, ok, shape in results:
        assert ok, (rank, mode, case)
        assert shape == (case[0], case[2])
