"""Worker of tests/test_gpu_peer_ipc.py: one of WORLD_SIZE processes sharing cuda:0.

Each process is a rank with its own CUDA context.  The ranks exchange real
cudaIpc handles (tg_peer_export / tg_peer_import through PeerYBuffers over a
gloo group), run their column shard of the GEMM with the fused peer-store
epilogue into every rank's Y, and check the assembled Y bit for bit against the
unsharded GEMM computed locally.

No kernel ever waits on a kernel of another process that has not finished: each
step synchronises the device and passes a host barrier between the shard GEMMs
and the arrival wait, so the wait finds every arrival already posted (two
contexts on one GPU are time-sliced; a spinning wait would only burn a slice,
but the test does not rely on that).
"""

from __future__ import annotations

import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def main() -> None:
    import paper_2510_06957_b200 as tg
    from paper_2510_06957_b200.kernels import GemmRunner
    from paper_2510_06957_b200.peer import PeerYBuffers, ScatterGemm

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    out = {"rank": rank, "world": world, "cases": []}
    # (M, K, N, alpha, symmetric, variant)
    cases = [(48, 640, 512, 0.25, True, "vectorized_optimal"),   # smem tile + TMA store + 16-byte peer stores
             (33, 900, 250, None, False, "base"),                # shard offset 125: direct stores to the peers
             (16, 4096, 1376 * 2, 0.25, True, "vectorized_optimal")]  # cfg4's 8-GPU shard width, two of them
    for ci, (M, K, N, alpha, sym, variant) in enumerate(cases):
        g = torch.Generator(device="cuda").manual_seed(1000 + ci)  # the same inputs on every rank
        W = torch.randint(-1, 2, (K, N), device="cuda", generator=g, dtype=torch.int8)
        X = torch.randn((M, K), device="cuda", generator=g)
        b = torch.randn((N,), device="cuda", generator=g)
        spec = tg.get_variant(variant)
        cfgk = tg.GemmConfig(method="mma", alpha=alpha)
        xin = tg.pad_input(X).device_values if sym else X

        def fmt_of(Wc):
            return spec.build(tg.TernaryDense(Wc.contiguous()), cfgk)

        full = GemmRunner(variant, xin, fmt_of(W), b, method="mma", alpha=alpha)
        full.launch()
        ref = full.y.clone()

        bufs = PeerYBuffers(M, N, symmetric=sym)
        assert bufs.world == world and len(bufs._imported) == world - 1  # real cudaIpc mappings
        cols = bufs.shard.slice()
        fmt = fmt_of(W[:, cols])
        bs = b[cols].contiguous()
        sg = ScatterGemm(lambda out, scatter: GemmRunner(variant, xin, fmt, bs, method="mma", alpha=alpha,
                                                         out=out, scatter=scatter), bufs)
        ok = True
        for step in range(4):  # both slots twice: counters, epoch and slot reuse
            s = sg.slot
            bufs.y(s).fill_(float("nan"))
            torch.cuda.synchronize()
            dist.barrier()                 # every rank's slot is poisoned before anyone stores
            sg.runners[s].launch()         # shard GEMM: own block by TMA, the peers' by NVLink/IPC stores
            torch.cuda.synchronize()
            dist.barrier()                 # every rank's GEMM (and its arrival signal) has completed
            bufs.wait()
            sg.n += 1
            torch.cuda.synchronize()
            ok = ok and bool(torch.equal(bufs.y(s), ref)) and not bufs.timed_out()
            hdr = bufs.header.cpu()
            ok = ok and [int(v) for v in hdr[:world]] == [step + 1] * world
            dist.barrier()                 # nobody starts the next step while a peer still reads
        out["cases"].append({"case": ci, "ok": ok, "shard": [bufs.shard.start, bufs.shard.stop]})
        bufs.close()
    dist.barrier()
    dist.destroy_process_group()
    print("PEER_IPC " + json.dumps(out), flush=True)
    if not all(c["ok"] for c in out["cases"]):
        raise SystemExit(1)


if __name__ == "__main__":
    main()
