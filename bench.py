#!/usr/bin/env python
"""Benchmark of the B200 sparse ternary GEMM hot path  Y = X W + b (+PReLU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--method auto|mma|gather]
    python bench.py --impl reference ...      # the reference's CPU path (oracle port) on the host cores

One "step" is one evaluation of the GEMM over the config's synthetic inputs
(BASELINE.json configs; recipe in paper_2510_06957_b200/workloads.py).  The
sparse format is built once on the device before timing (the reference
builds it once too: bench.py:164 ``spec.build``).

Timed quantities (rank 0 prints ONE JSON line):
  value        effective GOP/s = (M*nnz + M*N) / step time, inputs resident in
               HBM; the L2 (126 MB) is flushed before every step outside the
               events; with N > 1 ranks the step includes the NCCL all-gather
               that assembles Y, and the time is the max over ranks.
  e2e          the same metric through the public API (gemm_* on a pinned
               host X, result read back to the host every step).
  roofline     the north star's roofline (fp32-add peak vs compulsory HBM
               bytes) for the dominant kernel, timed with CUDA
               events on its own stream; ``tensor`` adds the dense-decode
               kernel's int8 tensor-pipe rate.
  cpu_baseline the reference's CPU path restated in C (oracle/, bit-exact
               with the reference kernels) on the host cores, bounded sample.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import shutil
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2510_06957_b200.workloads import (  # noqa: E402
    WORKLOADS,
    algorithmic_bytes,
    cfg5_oracle_rows,
    make_inputs,
    ops,
)

FADD_PER_CLK_PER_SM = 128  # fp32 FADD lanes per SM per clock (4 SMSP x 32)
NOMINAL_HBM_GBS = 8000.0  # the north star's 8 TB/s


def peaks() -> dict:
    p = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
    except OSError:
        pass
    return {
        "hbm_gbs": float(p.get("hbm_gbs", 6650.0)),
        "bf16_tflops": float(p.get("bf16_tflops", 1590.0)),
        "sm_max_mhz": float(p.get("sm_max_mhz", 1965.0)),
        "source": "measured (MEASURED_PEAKS.json)" if p else "fallback (B200_PROFILING.md)",
    }


# ---------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
        self.gpu = gpu_index
        if shutil.which("nvidia-smi"):
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)

    def stop(self) -> dict | None:
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], 0.0, set()
        for row in csv.reader(io.StringIO(out)):
            if len(row) < 9:
                continue
            row = [c.strip() for c in row]
            try:
                sm.append(float(row[1]))
                mx = max(mx, float(row[2]))
            except ValueError:
                continue
            for name, v in zip(self.REASONS, row[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- distributed


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def max_over_ranks(x: float, world: int, device) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------- CPU reference (oracle port)


def _cpu_setup(cfg: str, rows: np.ndarray | None):
    """Inputs and reference-built format for the CPU path of config ``cfg``."""
    from oracle import oracle as orc

    wl = WORKLOADS[cfg]
    W, X, b = make_inputs(cfg)
    if rows is not None:
        X = X[rows]
    if wl.variant == "vectorized_optimal":
        fmt = orc.interleaved_blocked_from_dense(W, None, 2, True)
        Xs = orc.pad_input(X)
        run = lambda xs, th: orc.gemm_vectorized_optimal(xs, fmt, b, wl.alpha, threads=th)  # noqa: E731
    elif wl.variant == "interleaved_blocked":
        fmt = orc.interleaved_blocked_from_dense(W, None, 2, False)
        Xs = X
        run = lambda xs, th: orc.gemm_interleaved_blocked(xs, fmt, b, threads=th)  # noqa: E731
    else:
        fmt = orc.tcsc_from_dense(W)
        Xs = X
        run = lambda xs, th: orc.gemm_base(xs, fmt, b, threads=th)  # noqa: E731
    nnz = int(np.count_nonzero(W))
    return Xs, run, nnz, wl


def cpu_time(cfg: str, threads: int, budget_s: float = 8.0, reps: int = 3):
    """Time the reference CPU path on a bounded row sample: (GOP/s, sample description, seconds/rep)."""
    rows = cfg5_oracle_rows() if cfg == "cfg5" else None
    Xs, run, nnz, wl = _cpu_setup(cfg, rows)
    M = Xs.shape[0]
    t0 = time.perf_counter()
    run(Xs[: min(M, 16)], threads)  # probe on 16 rows
    per_row = (time.perf_counter() - t0) / min(M, 16)
    m = int(max(1, min(M, budget_s / max(reps + 1, 1) / max(per_row, 1e-9))))
    xs = Xs[:m]
    run(xs, threads)  # warm-up (run_point: bench.py:171-173)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter_ns()
        run(xs, threads)
        ts.append((time.perf_counter_ns() - t0) / 1e9)
    t = statistics.median(ts)
    gops = ops(m, wl.N, nnz) / t / 1e9
    what = "seeded 256-row slice" if rows is not None else "rows"
    sample = f"{m} of {M} {what} x full K={wl.K}, N={wl.N} ({wl.variant}, {threads} threads, median of {reps})"
    return gops, sample, t, m


def run_reference(args) -> None:
    """--impl reference: the reference's CPU path on the box's host cores."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = args.config
    cores = len(os.sched_getaffinity(0))
    wl = WORKLOADS[cfg]
    rows = cfg5_oracle_rows() if cfg == "cfg5" else None
    Xs, run, nnz, _ = _cpu_setup(cfg, rows)
    M = Xs.shape[0]
    # size each step to <= ~1.5 s so --steps K --warmup W stays within minutes
    t0 = time.perf_counter()
    run(Xs[: min(M, 8)], cores)
    per_row = (time.perf_counter() - t0) / min(M, 8)
    m = int(max(1, min(M, 1.5 / max(per_row, 1e-9))))
    xs = Xs[:m]
    for _ in range(args.warmup):
        run(xs, cores)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter_ns()
        run(xs, cores)
        ts.append((time.perf_counter_ns() - t0) / 1e9)
    step = sum(ts) / len(ts)
    value = ops(m, wl.N, nnz) / step / 1e9
    sample = f"{m} of {M} rows x full K={wl.K}, N={wl.N} per step ({wl.variant})"
    line = {
        "impl": "reference", "metric": "effective_gops", "value": round(value, 4), "unit": "GOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step * 1e3, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (BASELINE.json recipe, seeded)",
        "config": {"workload": cfg, "M": wl.M, "K": wl.K, "N": wl.N, "p_nonzero": wl.p_pos + wl.p_neg,
                   "alpha": wl.alpha, "variant": wl.variant, "sample_rows": m},
        "cpu_baseline": {"value": round(value, 4), "unit": "GOP/s", "cores": cores, "kind": "port",
                         "sample": sample + "; C restatement of the reference numba kernel (oracle/tg_oracle.c), "
                                            "bit-exact with it, N-column threads"},
        "e2e": {"value": round(value, 4), "unit": "GOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    import paper_2510_06957_b200 as tg
    from paper_2510_06957_b200 import _native as nat
    from paper_2510_06957_b200.kernels import GemmRunner, choose_method
    from paper_2510_06957_b200.partition import ShardedGemm

    rank, world, local = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (there is no CPU path; use --impl reference for the CPU arm)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    nat.load()

    cfg = args.config
    wl = WORKLOADS[cfg]
    W, X, b = make_inputs(cfg)
    M, K, N = wl.M, wl.K, wl.N
    sym = wl.variant == "vectorized_optimal"
    part = ShardedGemm(M, N, "columns", symmetric=sym)
    sh = part.shard
    nnz_total = int(np.count_nonzero(W))

    # ---- build the device format for this rank's columns (untimed, once)
    dW = torch.from_numpy(np.ascontiguousarray(W[:, sh.slice()])).to(dev)
    db = torch.from_numpy(b[sh.slice()].copy()).to(dev)
    dX = torch.from_numpy(X).to(dev)
    cfgk = tg.GemmConfig(method=args.method, alpha=wl.alpha)
    spec = tg.get_variant(wl.variant)
    fmt = spec.build(tg.TernaryDense(dW), cfgk)
    nnz_local = int(np.count_nonzero(W[:, sh.slice()]))
    xin = tg.pad_input(dX).device_values if sym else dX
    method = choose_method(args.method, K, sh.width, nnz_local)
    kind = wl.variant
    runner = GemmRunner(kind, xin, fmt, db, method=method, alpha=wl.alpha)
    runner.pin_workspace()
    y_full = torch.empty((M, N), dtype=torch.float32, device=dev) if world > 1 else None

    # ---- verify before timing (bench.py:167-169): device fp64 oracle_gemm, normwise <= 1e-5
    runner.launch()
    y_loc = runner.y
    ref = (dX.double() @ dW.double() + db.double())
    if wl.alpha is not None:
        ref = torch.where(ref > 0, ref, wl.alpha * ref)
    nw = float((y_loc.double() - ref).abs().max() / ref.abs().max().clamp_min(1e-300))
    if not nw <= 1e-5:
        raise SystemExit(f"refusing to time a wrong kernel: normwise error {nw:.3e} > 1e-5")
    del ref

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2
    stream = torch.cuda.current_stream()

    # ---- shard assembly (N > 1): the fused peer-store epilogue by default, NCCL on request
    assembly = "none" if world == 1 else args.assembly
    asm_note = None
    # (agreed over ranks: every rank must take the same assembly)
    if assembly == "peer" and max_over_ranks(0.0 if method == "mma" else 1.0, world, dev) != 0.0:
        assembly, asm_note = "nccl", "gather method has no fused epilogue; NCCL all-gather"
    sg = bufs = None
    if assembly == "peer":
        from paper_2510_06957_b200.peer import PeerYBuffers, ScatterGemm

        # set-up failures (e.g. no cudaIpc between these processes) are agreed over the ranks
        # and fall back to the NCCL all-gather instead of ending the run
        why = None
        try:
            bufs = PeerYBuffers(M, N, symmetric=sym)
            assert bufs.shard == sh, (bufs.shard, sh)
            sg = ScatterGemm(lambda out, scatter: GemmRunner(kind, xin, fmt, db, method=method, alpha=wl.alpha,
                                                             out=out, scatter=scatter), bufs)
            for r in sg.runners:
                r.pin_workspace()
        except Exception as exc:  # noqa: BLE001 (reported in the JSON line)
            why = f"{type(exc).__name__}: {exc}"
            sg = None
        if max_over_ranks(0.0 if why is None else 1.0, world, dev) != 0.0:
            assembly = "nccl"
            asm_note = f"peer buffers unavailable on some rank ({why or 'another rank'}); NCCL all-gather"
            sg = bufs = None  # (left mapped: closing needs every rank)
        else:
            # validate once: the kernel-assembled Y equals the NCCL-assembled Y bit for bit, on every slot
            y_nccl = part.assemble(runner.y, y_full).clone()
            ok = True
            for _ in range(2 * bufs.slots):
                yf = sg.step()
                torch.cuda.synchronize()
                ok = ok and bool(torch.equal(yf, y_nccl)) and not bufs.timed_out()
            if max_over_ranks(0.0 if ok else 1.0, world, dev) != 0.0:
                assembly, asm_note = "nccl", "peer scatter failed validation on some rank; fell back to NCCL all-gather"
                sg = None
            del y_nccl

    def capture(fn):
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                fn()
        torch.cuda.current_stream().wait_stream(s)
        return g

    graphs = None
    if not args.no_graph:
        if sg is not None:  # one graph per Y slot: shard GEMM with the peer scatter + arrival wait
            graphs = [capture(lambda r=r: (r.launch(), bufs.wait())) for r in sg.runners]
        else:
            graphs = [runner.capture()]
    graph = graphs[0] if graphs else None

    def step():
        if sg is not None:  # slots strictly alternate (ScatterGemm's counter), graph or not
            if graphs is not None:
                graphs[sg.slot].replay()
                sg.n += 1
            else:
                sg.step()
            return
        if graph is not None:
            graph.replay()
        else:
            runner.launch(stage="prepare")
            runner.launch(stage="run")
        if world > 1:
            part.assemble(runner.y, y_full)

    for _ in range(max(args.warmup, 3)):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # ---- headline: K whole steps, each preceded by an L2 flush.  One event pair
    # around all K (flush + step) and one around K flushes alone: per-step event
    # pairs would add their own ~6 us each on this box (measured), so
    # t_step = (t[flush + step] - t[flush]) / K.
    clocks = ClockSampler(local)
    t_clk0 = time.perf_counter()
    e_all = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e_all[0].record(stream)
    for i in range(args.steps):
        flush.zero_()
        step()
    e_all[1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e_all[2].record(stream)
    for i in range(args.steps):
        flush.zero_()
    e_all[3].record(stream)
    torch.cuda.synchronize()
    # keep the GPU loaded until the clock sampler has ~1 s of samples (untimed); the
    # iteration count is agreed over ranks (every rank must run the same steps)
    per_it = max(e_all[0].elapsed_time(e_all[1]) / max(args.steps, 1), 1e-3) * 1e-3
    n_more = int(max(0.0, 1.2 - (time.perf_counter() - t_clk0)) / per_it) + 1
    n_more = int(max_over_ranks(float(min(n_more, 200000)), world, dev))
    for i in range(n_more):
        flush.zero_()
        step()
        if i % 64 == 63:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    clk = clocks.stop()
    t_with = e_all[0].elapsed_time(e_all[1])
    t_flush = e_all[2].elapsed_time(e_all[3])
    t_step = (t_with - t_flush) / args.steps  # ms

    # ---- breakdown (same loop-difference method, direct launches):
    #   prepare = K x (flush + X split) - K x flush;  run = K x (flush + split + GEMM) - K x (flush + split)
    n_bd = max(args.steps, 20)  # enough repetitions for the differences to be above timer noise

    def loop_ms(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(n_bd):
            flush.zero_()
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    t_f = loop_ms(lambda: None)
    t_fp = loop_ms(lambda: runner.launch(stage="prepare"))
    t_fpr = loop_ms(lambda: (runner.launch(stage="prepare"), runner.launch(stage="run")))
    t_prep = max(t_fp - t_f, 0.0) / n_bd
    t_run = max(t_fpr - t_fp, 1e-6) / n_bd
    t_comm = 0.0
    if sg is not None:  # the peer scatter + arrival wait over the plain shard GEMM
        t_fpra = loop_ms(lambda: sg.step())
        t_comm = max(t_fpra - t_fpr, 0.0) / n_bd
    elif world > 1:
        t_fpra = loop_ms(lambda: (runner.launch(stage="prepare"), runner.launch(stage="run"),
                                  part.assemble(runner.y, y_full)))
        t_comm = max(t_fpra - t_fpr, 0.0) / n_bd
    t_step_max = max_over_ranks(t_step, world, dev)

    total_ops = ops(M, N, nnz_total)
    value = total_ops / (t_step_max * 1e-3) / 1e9

    # ---- e2e through the public API: pinned host X -> device, GEMM, Y back to the host
    Xh = torch.from_numpy(X).pin_memory()
    tb = tg.BiasVector(db)

    h2d_bytes = int(world * M * K * 4)
    if sg is not None:
        # the fused path's public surface is ScatterGemm: X (pinned) -> the runners' X buffer,
        # one step, the assembled Y back to the host on rank 0
        Xh_in = torch.zeros(tuple(xin.shape), dtype=torch.float32).pin_memory()
        Xh_in[:, :K] = torch.from_numpy(X)
        h2d_bytes = int(world * Xh_in.numel() * 4)

    def api_call():
        if sg is not None:
            xin.copy_(Xh_in, non_blocking=True)
            y = sg.step()
            return tg.DenseMatrix(y).values if rank == 0 else None
        if sym:
            y = tg.gemm_vectorized_optimal(tg.pad_input(Xh), fmt, tb, wl.alpha, method=method)
        elif kind == "interleaved_blocked":
            y = tg.gemm_interleaved_blocked(Xh, fmt, tb, method=method)
        elif kind == "blocked":
            y = tg.gemm_blocked(Xh, fmt, tb, method=method)
        else:
            y = tg.gemm_base(Xh, fmt, tb, method=method)
        if world == 1:
            return y.values  # the reference's contract: a host numpy array (pinned D2H + status check)
        yd = part.assemble(y.check().device_values, y_full)
        return tg.DenseMatrix(yd).values if rank == 0 else None

    if not args.no_e2e:
        # (the first calls capture the library's graph of the call and fill its buffer
        # pools; the PCIe path also takes a few dozen calls to settle: samples drift down
        # ~20% over the first 20)
        for _ in range(max(args.warmup, 30)):
            api_call()
    torch.cuda.synchronize()
    e2e_steps = max(3, min(args.steps, 20)) if not args.no_e2e else 0
    t_e2e = []
    for _ in range(e2e_steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        api_call()
        e1.record(stream)
        e1.synchronize()
        t_e2e.append(e0.elapsed_time(e1))
    if t_e2e and os.environ.get("BENCH_E2E_SAMPLES"):
        print("e2e samples (ms):", " ".join(f"{t:.4f}" for t in t_e2e), file=sys.stderr)
    t_e2e_ms = max_over_ranks(sum(t_e2e) / len(t_e2e), world, dev) if t_e2e else float("nan")
    e2e_value = total_ops / (t_e2e_ms * 1e-3) / 1e9 if t_e2e else None

    if rank != 0:
        if world > 1:
            dist.barrier()
            if bufs is not None:
                torch.cuda.synchronize()
                bufs.close()
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (per-GPU shard)
    pk = peaks()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    p_add = sms * FADD_PER_CLK_PER_SM * pk["sm_max_mhz"] * 1e6 / 1e12  # T adds/s
    w_loc = sh.width
    ops_loc = ops(M, w_loc, nnz_local)
    bytes_loc = algorithmic_bytes(M, K, w_loc, nnz_local)
    t_kernel = max(t_run if method == "mma" else t_prep + t_run, 1e-6)
    kern_name = "tg_mma_kernel" if method == "mma" else "tg_gather_kernel"
    t_add = ops_loc / (p_add * 1e12)
    t_hbm = bytes_loc / (NOMINAL_HBM_GBS * 1e9)
    bound = "hbm" if t_hbm > t_add else "fp32_add"
    achieved_tops = ops_loc / (t_kernel * 1e-3) / 1e12
    achieved_gbs = bytes_loc / (t_kernel * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(f"{cfg}:{method}")
    except (OSError, ValueError):
        pass
    roof = {
        "bound": bound,
        "kernel": kern_name,
        "achieved": round(achieved_tops if bound == "fp32_add" else achieved_gbs, 3),
        "peak": round(p_add if bound == "fp32_add" else pk["hbm_gbs"], 3),
        "unit": "TFLOP/s" if bound == "fp32_add" else "GB/s",
        "frac": round((t_add if bound == "fp32_add" else bytes_loc / (pk["hbm_gbs"] * 1e9)) / (t_kernel * 1e-3), 4),
        "traffic": traffic,
        "kernel_ms": round(t_kernel, 5),
        "algorithmic_ops_per_launch": ops_loc,
        "algorithmic_bytes_per_launch": bytes_loc,
        "peak_source": (f"fp32 FADD peak = {sms} SMs x {FADD_PER_CLK_PER_SM}/clk x {pk['sm_max_mhz']:.0f} MHz "
                        f"(sm_max_mhz of {pk['source']}); HBM {pk['hbm_gbs']} GB/s {pk['source']}"),
        "north_star_frac": round(max(t_add, t_hbm) / (t_kernel * 1e-3), 4),
        "hbm": {"achieved_gbs": round(achieved_gbs, 2), "peak_gbs": pk["hbm_gbs"],
                "frac": round(achieved_gbs / pk["hbm_gbs"], 4)},
    }
    if method == "mma":
        M_pad = -(-M // 16) * 16
        tens = 2 * 3 * M * K * w_loc  # int8 ops of the three limb GEMMs at the unpadded shape
        peak_i8 = 2 * pk["bf16_tflops"]
        roof["tensor"] = {"achieved": round(tens / (t_run * 1e-3) / 1e12, 2), "peak": round(peak_i8, 1),
                          "unit": "TOP/s int8",
                          "frac": round(tens / (t_run * 1e-3) / 1e12 / peak_i8, 4),
                          "peak_source": "2 x measured bf16 dense (kind::i8 issues at twice kind::f16 on B200)",
                          "m_pad": M_pad}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cores = len(os.sched_getaffinity(0))
        g_all, sample, _, _ = cpu_time(cfg, cores, budget_s=10.0)
        g_one, sample1, _, _ = cpu_time(cfg, 1, budget_s=6.0, reps=1)
        cpu = {"value": round(g_all, 4), "unit": "GOP/s", "cores": cores, "kind": "port", "sample": sample,
               "one_core": {"value": round(g_one, 4), "sample": sample1},
               "what": "oracle/tg_oracle.c: C restatement of the reference numba kernel, bit-exact with it"}

    launches_per_step = 2  # mma: X split + tile MMA; gather: transpose + gather
    if sg is not None:
        launches_per_step = 3  # + the arrival wait
    line = {
        "metric": "effective_gops", "value": round(value, 3), "unit": "GOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t_step_max, 5), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (BASELINE.json recipe, seeded; no dataset)",
        "config": {"workload": cfg, "M": M, "K": K, "N": N, "p_nonzero": wl.p_pos + wl.p_neg, "nnz": nnz_total,
                   "alpha": wl.alpha, "variant": wl.variant, "method": method,
                   "parallelism": f"N-sharded x{world}" + (
                       "" if world == 1 else " + fused peer-store epilogue over NVLink" if assembly == "peer"
                       else " + NCCL all-gather"),
                   "l2": "flushed (256 MB write) before every timed step; step time = (K x (flush+step) - K x flush) / K",
                   "launch": "CUDA graph replay per step" if graph is not None else "direct launches"},
        "breakdown_ms": {"prepare": round(t_prep, 5), "run": round(t_run, 5), "assemble": round(t_comm, 5),
                         "note": "loop differences over K steps with direct launches; run = GEMM kernel after the "
                                 "split; assemble = extra time of the shard assembly (NCCL all-gather, or the fused "
                                 "peer stores + arrival wait)"},
        "assembly": {"kind": assembly, "note": asm_note},
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": {"value": round(e2e_value, 3) if e2e_value else None, "unit": "GOP/s", "ms_per_step": round(t_e2e_ms, 4),
                "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": int(M * N * 4),
                "path": (f"ScatterGemm.step on pinned host X (H2D into the shard runners' X), rank 0 reads the "
                         f"assembled Y" if sg is not None else
                         f"public API gemm_* on pinned host X ({'pad_input + ' if sym else ''}{kind}), Y.values")},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk,
        "parity": {"normwise_vs_fp64": nw},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        if bufs is not None:
            torch.cuda.synchronize()
            bufs.close()
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--method", default="auto", choices=("auto", "mma", "gather"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the public-API end-to-end leg (profiling runs)")
    ap.add_argument("--no-graph", action="store_true", help="issue the step's kernels one by one instead of a CUDA graph")
    ap.add_argument("--assembly", default="peer", choices=("peer", "nccl"),
                    help="N > 1: assemble Y in the GEMM epilogue over NVLink peer memory (default) or NCCL all-gather")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
