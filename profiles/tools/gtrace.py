#!/usr/bin/env python
"""Timeline of one step (X split + tile GEMM) from the kernels' own %globaltimer stamps.

Needs the instrumented build (developer use only, never loaded by the package by default):

    make -C paper_2510_06957_b200 libterngemm_b200_trace.so
    TG_LIB_PATH=$PWD/paper_2510_06957_b200/libterngemm_b200_trace.so \
        python profiles/tools/gtrace.py --config cfg4 [--reps 20] [--x-outliers 8@100]

Per milestone it prints min / max over the CTAs in microseconds from the first split CTA's
start, the median over `reps` graph replays, each after a 256 MB L2 flush.  Milestones
(TG_GT in csrc/tg_mma.cu): 0 split CTA start, 1 split row done, 2 GEMM CTA start, 3
griddepcontrol.wait returned, 4 first MMA stage committed, 5 last MMA issued, 6 epilogue
done, 7 CTA exit, 8-10 (first unit of each CTA) the epilogue's outlier-term lookups and the
moment its accumulator is ready.  Not a bench number: the stamps cost a few hundred ns.
"""
from __future__ import annotations

import argparse
import ctypes
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

NAMES = ["split CTA start", "split row done", "GEMM CTA start", "dep wait returned", "first MMA commit",
         "last MMA issued", "epilogue done", "CTA exit", "outlier terms: start", "outlier terms: done",
         "accumulator ready"]


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--x-outliers", default=None)
    args = ap.parse_args()
    import bench
    import paper_2510_06957_b200 as tg
    from paper_2510_06957_b200 import _native as nat
    from paper_2510_06957_b200.kernels import GemmRunner
    from paper_2510_06957_b200.workloads import WORKLOADS

    lib = nat.load()
    if not hasattr(lib, "tg_debug_gt"):
        raise SystemExit("load the TG_TRACE build through TG_LIB_PATH (see the docstring)")
    lib.tg_debug_gt.argtypes = [ctypes.c_void_p, ctypes.c_int]
    wl = WORKLOADS[args.config]
    W, X, b = bench.bench_inputs(args.config, args.x_outliers)
    dev = torch.device("cuda", 0)
    sym = wl.variant == "vectorized_optimal"
    fmt = tg.get_variant(wl.variant).build(tg.TernaryDense(torch.from_numpy(W).to(dev)), tg.GemmConfig(alpha=wl.alpha))
    dX = torch.from_numpy(X).to(dev)
    xin = tg.pad_input(dX).device_values if sym else dX
    r = GemmRunner(wl.variant, xin, fmt, torch.from_numpy(b).to(dev), method="mma", alpha=wl.alpha)
    r.pin_workspace()
    g = r.capture()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    out = (ctypes.c_ulonglong * 32)()
    rows = []
    for _ in range(args.reps + 3):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        lib.tg_debug_gt(None, 1)
        g.replay()
        torch.cuda.synchronize()
        lib.tg_debug_gt(out, 0)
        v = np.array(out[:], dtype=np.uint64).reshape(16, 2)[:len(NAMES)].astype(np.int64)
        rows.append((v - v[0, 0]) / 1e3)
    rows = np.array(rows[3:])
    print(f"{args.config} x_outliers={args.x_outliers}: median over {args.reps} replays, us from the first split CTA")
    for i, n in enumerate(NAMES):
        print(f"  {i} {n:20s} first {statistics.median(rows[:, i, 0]):7.2f}   last {statistics.median(rows[:, i, 1]):7.2f}")


if __name__ == "__main__":
    main()
