"""The fused shard assembly across PROCESSES: real cudaIpc export / import.

tests/test_gpu_peer.py runs the peer-store epilogue with every "rank" inside
one process (loopback pointers).  Here two (and three) processes share cuda:0,
each with its own CUDA context, so every peer pointer is a cudaIpc mapping
obtained through tg_peer_export / tg_peer_import, exactly as ranks on separate
GPUs obtain theirs; only the transport under the mapping (local HBM instead of
NVLink) differs.  See tests/_peer_ipc_worker.py for the protocol and why no
kernel waits on another process's kernel.
"""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_peer_scatter_over_cuda_ipc(world):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(HERE, "_peer_ipc_worker.py")]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    # (the ranks share one stdout: two records may land on one line)
    dec = json.JSONDecoder()
    recs = [dec.raw_decode(chunk.lstrip())[0] for chunk in p.stdout.split("PEER_IPC ")[1:]]
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    assert sorted(r["rank"] for r in recs) == list(range(world)), p.stdout[-2000:]
    for rec in recs:
        assert rec["world"] == world
        assert rec["cases"] and all(c["ok"] for c in rec["cases"]), rec
