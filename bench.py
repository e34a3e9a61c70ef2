#!/usr/bin/env python
"""Benchmark of the B200 sparse ternary GEMM hot path  Y = X W + b (+PReLU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5] [--method auto|mma|gather]
    python bench.py --impl reference ...   # the reference's own CPU path on the host cores

One "step" is one evaluation of the GEMM over the config's synthetic inputs
(BASELINE.json configs; recipe in paper_2510_06957_b200/workloads.py).  The
default workload is cfg5 (8192 x 8192 x 16384), the largest BASELINE config,
which fits one B200.  The sparse format is built once on the device before
timing (the reference builds it once too: bench.py:164 ``spec.build``).

Timed quantities (rank 0 prints ONE JSON line):
  value        effective GOP/s = (M*nnz + M*N) / step time, inputs resident in
               HBM; the L2 (126 MB) is flushed before every step outside the
               events; with N > 1 ranks the step includes the assembly of Y
               on every rank, and the time is the max over ranks.
  e2e          the same metric through the public API (gemm_* on a pinned
               host X, result read back to the host every step).
  roofline     the north star's roofline (fp32-add peak vs compulsory HBM
               bytes) for the dominant kernel, timed with CUDA
               events on its own stream; ``tensor`` adds the kernel's int8
               rate against the int8 tcgen05.mma rate measured in this run
               (csrc/tg_peak.cu).
  cpu_baseline the reference's CPU path on the host cores, timed with the same
               protocol as ``--impl reference``: the reference package itself
               (numba, installed in baseline/_ref) when importable, else the C
               restatement of its kernels (oracle/, bit-exact with them).
  parity       the GPU result is checked BEFORE timing (bench.py:167-169 of the
               reference: a failing point is never timed): normwise and
               |terms|-scaled error vs the fp64 oracle on the whole Y, both
               against the reference CPU path's own output on its row slice, and
               the integer-valued twin bit-exact.

Under ``--gpus N`` with no torchrun environment, bench.py launches N ranks
itself through torch.distributed.run (127.0.0.1).
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import shutil
import socket
import statistics
import subprocess
import sys
import time
from concurrent.futures import ThreadPoolExecutor

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
TOL = 1e-5  # normwise and |terms|-scaled bars
REF_DIR = os.path.join(ROOT, "baseline", "_ref")
DEFAULT_CONFIG = "cfg5"


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


def parse_outliers(spec: str | None):
    """--x-outliers "C@S": C activation channels at S x (LLM-style heavy tails); None: the BASELINE X."""
    if not spec:
        return None
    c, s = spec.split("@")
    return int(c), float(s)


def bench_inputs(cfg: str, outliers: str | None = None, integer: bool = False):
    """The config's seeded inputs; with --x-outliers the same seeded channels of X are scaled."""
    W, X, b = make_inputs(cfg, integer=integer)
    o = parse_outliers(outliers)
    if o is not None and not integer:
        ch = np.random.default_rng(20251006).choice(X.shape[1], o[0], replace=False)
        X[:, ch] *= np.float32(o[1])
    return W, X, b


def config_dict(cfg: str, nnz: int, outliers: str | None = None) -> dict:
    """The workload description, identical in both arms (the driver compares them)."""
    wl = WORKLOADS[cfg]
    if outliers:
        d = config_dict(cfg, nnz)
        d["x_outliers"] = f"{outliers}: channels x scale applied to the seeded X (not a BASELINE config)"
        return d
    return {"workload": cfg, "M": wl.M, "K": wl.K, "N": wl.N, "p_nonzero": wl.p_pos + wl.p_neg, "nnz": nnz,
            "x_dist": wl.x_dist, "bias": wl.bias, "alpha": wl.alpha, "variant": wl.variant, "seed": wl.seed,
            "l2": "GPU arm: 256 MB L2 flush before every timed step, outside the events "
                  "(step = (K x (flush+step) - K x flush) / K); CPU arm: inputs larger than its caches"}


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


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """``--gpus N`` without a torchrun environment: launch N ranks (one per GPU) through
    torch.distributed.run on 127.0.0.1 and return its exit code.  NCCL's INIT lines go to
    stderr so the ranks and their communicator are visible in the log."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


# ---------------------------------------------------------------- the reference CPU path


def reference_package():
    """The reference package installed in baseline/_ref (python -m pip install --no-index
    ... --target baseline/_ref; baseline/install_ref.sh), or None when it is not importable
    (e.g. numba missing).  It is only ever timed or used as a checker here."""
    if not os.path.isdir(os.path.join(REF_DIR, "terngemm")):
        return None
    if REF_DIR not in sys.path:
        sys.path.append(REF_DIR)
    try:
        import terngemm  # noqa: PLC0415

        return terngemm
    except Exception:  # noqa: BLE001 (absent dependency: fall back to the port)
        return None


class CpuPath:
    """The reference's CPU path for one config on the host cores.

    kind "reference": the reference package's own registry kernel (numba, nogil) on
    N-column shards in a thread pool, each shard with its own reference-built format
    (the kernels are pure functions over disjoint outputs).
    kind "port": oracle/tg_oracle.c, the C restatement of the same kernels with the
    same per-output fp32 operation order (bit-exact with them, tests/test_oracle_golden.py).
    Registry tag per config: cfg1 ``base``; cfg2/cfg4 ``vectorized_optimal`` (alpha 0.25);
    cfg3/cfg5 ``interleaved_blocked``.  cfg5 runs on its seeded 256-row slice."""

    def __init__(self, cfg: str, threads: int, kind: str = "reference", W=None, X=None, b=None):
        self.cfg, self.wl, self.threads = cfg, WORKLOADS[cfg], max(1, threads)
        if W is None:
            W, X, b = make_inputs(cfg)
        self.rows = cfg5_oracle_rows() if cfg == "cfg5" else np.arange(X.shape[0])
        self.X = np.ascontiguousarray(X[self.rows])
        self.b = b
        self.nnz = int(np.count_nonzero(W))
        self.sym = self.wl.variant == "vectorized_optimal"
        ref = reference_package() if kind == "reference" else None
        self.kind = "reference" if ref is not None else "port"
        if self.kind == "reference":
            self._setup_reference(ref, W)
        else:
            self._setup_port(W)

    # -- the reference package
    def _setup_reference(self, rt, W) -> None:
        N, wl = self.wl.N, self.wl
        step = 4 if self.sym else 1  # symmetric 4-column groups may not be split (variants.py:324-325)
        n_sh = max(1, min(self.threads, N // step))
        edges = [min(N, (N * i // n_sh + step - 1) // step * step) for i in range(n_sh + 1)]
        edges[-1] = N
        self.shards = []
        for lo, hi in zip(edges[:-1], edges[1:]):
            if hi <= lo:
                continue
            Ws = rt.TernaryDense(np.ascontiguousarray(W[:, lo:hi]))
            bs = rt.BiasVector(np.ascontiguousarray(self.b[lo:hi]))
            if wl.variant == "vectorized_optimal":
                fmt = rt.interleaved_blocked_from_dense(Ws, None, 2, symmetric_cols=True)
                fn = (lambda x, f=fmt, bb=bs: rt.gemm_vectorized_optimal(x, f, bb, wl.alpha))
            elif wl.variant == "interleaved_blocked":
                fmt = rt.interleaved_blocked_from_dense(Ws, None, 2)
                fn = (lambda x, f=fmt, bb=bs: rt.gemm_interleaved_blocked(x, f, bb))
            else:
                fmt = rt.tcsc_from_dense(Ws)
                fn = (lambda x, f=fmt, bb=bs: rt.gemm_base(x, f, bb))
            self.shards.append((lo, hi, fn))
        self._rt = rt
        self._pool = ThreadPoolExecutor(len(self.shards))
        self.what = (f"reference package terngemm (numba, baseline/_ref), registry kernel '{wl.variant}', "
                     f"{len(self.shards)} N-column shards on {len(self.shards)} threads")
        self.run(self.X[:1])  # numba JIT compile (conftest.py:3-19 of the reference warms the same way)

    def _setup_port(self, W) -> None:
        from oracle import oracle as orc

        wl = self.wl
        if wl.variant == "vectorized_optimal":
            fmt = orc.interleaved_blocked_from_dense(W, None, 2, True)
            self._port = lambda x, th: orc.gemm_vectorized_optimal(orc.pad_input(x), fmt, self.b, wl.alpha, threads=th)
        elif wl.variant == "interleaved_blocked":
            fmt = orc.interleaved_blocked_from_dense(W, None, 2, False)
            self._port = lambda x, th: orc.gemm_interleaved_blocked(x, fmt, self.b, threads=th)
        else:
            fmt = orc.tcsc_from_dense(W)
            self._port = lambda x, th: orc.gemm_base(x, fmt, self.b, threads=th)
        self.what = (f"oracle/tg_oracle.c: C restatement of the reference kernel '{wl.variant}' (bit-exact with it), "
                     f"N-column threads")

    def run(self, xs: np.ndarray) -> np.ndarray:
        if self.kind == "port":
            return self._port(xs, self.threads)
        rt = self._rt
        xin = rt.pad_input(rt.DenseMatrix(xs)) if self.sym else rt.DenseMatrix(xs)
        parts = list(self._pool.map(lambda s: s[2](xin).values, self.shards))
        return np.concatenate(parts, axis=1) if len(parts) > 1 else parts[0]

    def sample_rows(self, seconds: float) -> int:
        """Rows per step so one step takes about ``seconds``."""
        m0 = min(len(self.rows), 8)
        t0 = time.perf_counter()
        self.run(self.X[:m0])
        per_row = (time.perf_counter() - t0) / m0
        return int(max(1, min(len(self.rows), seconds / max(per_row, 1e-9))))

    def time(self, m: int, steps: int, warmup: int) -> list[float]:
        """run_point mechanics (bench.py:171-178): warm-up calls, then timed calls (perf_counter_ns)."""
        xs = self.X[:m]
        for _ in range(warmup):
            self.run(xs)
        ts = []
        for _ in range(steps):
            t0 = time.perf_counter_ns()
            self.run(xs)
            ts.append((time.perf_counter_ns() - t0) / 1e9)
        return ts

    def measure(self, steps: int, warmup: int, step_seconds: float = 1.5) -> dict:
        m = self.sample_rows(step_seconds)
        ts = self.time(m, steps, warmup)
        step = sum(ts) / len(ts)
        what = "seeded 256-row slice" if self.cfg == "cfg5" else "rows"
        return {"value": ops(m, self.wl.N, self.nnz) / step / 1e9, "unit": "GOP/s", "cores": self.threads,
                "kind": self.kind, "seconds_per_step": step, "rows": m,
                "sample": (f"{m} of {len(self.rows)} {what} x full K={self.wl.K}, N={self.wl.N} per step, "
                           f"mean of {steps} steps after {warmup} warm-up; {self.what}")}


def run_reference(args) -> None:
    """--impl reference: the reference's CPU path on the box's host cores (rank 0 only)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = args.config
    cores = len(os.sched_getaffinity(0))
    cpu = CpuPath(cfg, cores, **(dict(zip("WXb", bench_inputs(cfg, args.x_outliers))) if args.x_outliers else {}))
    meas = cpu.measure(args.steps, args.warmup)
    value = meas["value"]
    line = {
        "impl": "reference", "metric": "effective_gops", "value": round(value, 4), "unit": "GOP/s",
        "n_gpus": max(world, args.gpus), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(meas["seconds_per_step"] * 1e3, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (BASELINE.json recipe, seeded; no dataset)",
        "config": config_dict(cfg, cpu.nnz, args.x_outliers),
        "cpu_baseline": {k: (round(v, 4) if isinstance(v, float) else v) for k, v in meas.items()},
        "e2e": {"value": round(value, 4), "unit": "GOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm: parity gate


def device_agreement(y, X, W, b, alpha) -> dict:
    """SURVEY.md 8(c) predicates of a device Y against the fp64 oracle_gemm (dense.py:192-213),
    computed on the device: exact (bit equality with the fp32-rounded fp64 result), normwise
    max|Y - ref| / max|ref|, and the |terms|-scaled max |Y - ref| / (sum_k |x_mk||w_kn| + |b_n|)
    (x max(1, |alpha|) under PReLU).  Column chunks bound the fp64 temporaries."""
    import torch

    Xd = X
    out = {"exact": True, "normwise_num": 0.0, "normwise_den": 0.0, "scaled": 0.0}
    x64, ax64 = Xd.double(), Xd.double().abs()
    step = 4096
    for c0 in range(0, W.shape[1], step):
        c1 = min(W.shape[1], c0 + step)
        w64 = W[:, c0:c1].double()
        ref = x64 @ w64 + b[c0:c1].double()
        if alpha is not None:
            ref = torch.where(ref > 0, ref, alpha * ref)
        ref32 = ref.float()
        yc = y[:, c0:c1]
        out["exact"] = out["exact"] and bool(torch.equal(yc, ref32))
        err = (yc.double() - ref32.double()).abs()
        out["normwise_num"] = max(out["normwise_num"], float(err.max()))
        out["normwise_den"] = max(out["normwise_den"], float(ref32.double().abs().max()))
        scale = ax64 @ w64.abs() + b[c0:c1].double().abs()
        if alpha is not None:
            scale = scale * max(1.0, abs(float(alpha)))
        q = torch.where(scale > 0, err / scale, torch.where(err > 0, torch.full_like(err, float("inf")),
                                                                      torch.zeros_like(err)))
        out["scaled"] = max(out["scaled"], float(q.max()))
        del w64, ref, ref32, err, scale, q
    den = out.pop("normwise_den")
    num = out.pop("normwise_num")
    out["normwise"] = num / den if den > 0 else num
    return out


# ---------------------------------------------------------------- GPU arm


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    import paper_2510_06957_b200 as tg
    from paper_2510_06957_b200 import _native as nat
    from paper_2510_06957_b200.harness import agreement, measure_i8_mma_peak
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
    W, X, b = bench_inputs(cfg, args.x_outliers)
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

    # ---- verify before timing (reference bench.py:135-150, 167-169): a failing point is never timed.
    # (1) real X, the whole Y of this rank: normwise and |terms|-scaled vs fp64 on the device
    runner.launch()
    parity = {"tol": TOL}
    a_real = device_agreement(runner.y, dX, dW, db, wl.alpha)
    parity["normwise_vs_fp64"] = a_real["normwise"]
    parity["scaled_vs_fp64"] = a_real["scaled"]
    # (2) the integer-valued twin (dense.py:143-160): bit-exact with the fp64 oracle
    _, Xi, bi = make_inputs(cfg, integer=True)
    dXi, dbi = torch.from_numpy(Xi).to(dev), torch.from_numpy(bi[sh.slice()].copy()).to(dev)
    xin_i = tg.pad_input(dXi).device_values if sym else dXi
    runner_i = GemmRunner(kind, xin_i, fmt, dbi, method=method, alpha=wl.alpha)
    runner_i.launch()
    a_int = device_agreement(runner_i.y, dXi, dW, dbi, wl.alpha)
    parity["integer_twin_bit_exact"] = a_int["exact"]
    del runner_i, xin_i, dXi, dbi
    # (3) the reference CPU path's own output on its row slice (cfg5: the seeded 256 rows), rank 0
    #     at N = 1: normwise and scaled against the reference order (bit-exact for the gather path)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cores = len(os.sched_getaffinity(0))
        cpu = CpuPath(cfg, cores, W=W, X=X, b=b)
        y_cpu = cpu.run(cpu.X)
        rows_t = torch.from_numpy(cpu.rows).to(dev)
        y_rows = runner.y[rows_t].cpu().numpy()
        sc = device_agreement(torch.from_numpy(y_cpu).to(dev), dX[rows_t], dW, db, wl.alpha)
        ag = agreement(y_rows, y_cpu)
        parity["vs_cpu_reference"] = {"kind": cpu.kind, "rows": int(len(cpu.rows)), "bit_exact": ag.exact,
                                      "normwise": ag.normwise, "cpu_normwise_vs_fp64": sc["normwise"],
                                      "cpu_scaled_vs_fp64": sc["scaled"],
                                      "rtol_fails_gpu_vs_cpu": ag.rtol_fails}
        del y_cpu
    ok = (a_real["normwise"] <= TOL and a_real["scaled"] <= TOL and a_int["exact"]
          and ("vs_cpu_reference" not in parity or parity["vs_cpu_reference"]["normwise"] <= TOL)
          and (method != "gather" or "vs_cpu_reference" not in parity or parity["vs_cpu_reference"]["bit_exact"]))
    if max_over_ranks(0.0 if ok else 1.0, world, dev) != 0.0:
        raise SystemExit(f"refusing to time a wrong kernel: {json.dumps(parity)}")
    # how the X split classified the rows (tensor-core path): rows left to the exact-order walk,
    # rows that shed outlier entries into the epilogue's list
    row_stats = runner.row_stats() if method == "mma" else None

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
    t_kernel_max = max_over_ranks(t_prep + t_run, world, dev)

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
            if rank != 0:
                sg.step()
                return None
            return sg.result().values  # raises if the assembly's wait timed out
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
        api_call()  # (the result is dropped, as a caller that consumed it would: its pinned Y returns to the pool)
        e1.record(stream)
        e1.synchronize()
        t_e2e.append(e0.elapsed_time(e1))
    y_e2e = api_call() if (t_e2e and world == 1) else None
    if t_e2e and os.environ.get("BENCH_E2E_SAMPLES"):
        print("e2e samples (ms):", " ".join(f"{t:.4f}" for t in t_e2e), file=sys.stderr)
    t_e2e_ms = max_over_ranks(sum(t_e2e) / len(t_e2e), world, dev) if t_e2e else float("nan")
    e2e_value = total_ops / (t_e2e_ms * 1e-3) / 1e9 if t_e2e else None
    if y_e2e is not None:
        # the e2e result is the device result (same kernels, host-streamed in row chunks)
        parity["e2e_equals_device"] = bool(np.array_equal(y_e2e, runner.y.cpu().numpy()))
    del y_e2e

    # ---- measured int8 tensor-core rate (the tensor roofline's denominator), rank 0
    i8 = None
    if rank == 0 and method == "mma":
        torch.cuda.synchronize()
        burst = max(measure_i8_mma_peak(256, False, 0.025, 4), measure_i8_mma_peak(256, True, 0.025, 4),
                    key=lambda r: r["tops"])
        sustained = measure_i8_mma_peak(burst["n"], burst["a"] == "tmem", 0.5, 6)
        i8 = {"burst": burst, "sustained": sustained}

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
    kern_name = "tg_mma_kernel" if method == "mma" else "tg_gather_staged_kernel"
    t_add = ops_loc / (p_add * 1e12)
    t_hbm = bytes_loc / (NOMINAL_HBM_GBS * 1e9)
    bound = "hbm" if t_hbm > t_add else "fp32_add"
    achieved_tops = ops_loc / (t_kernel * 1e-3) / 1e12
    achieved_gbs = bytes_loc / (t_kernel * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        traffic = tj.get(f"{cfg}:{method}")
        traffic_src = tj.get("_source")
    except (OSError, ValueError):
        traffic_src = None
    roof = {
        "bound": bound,
        "kernel": kern_name,
        "achieved": round(achieved_tops if bound == "fp32_add" else achieved_gbs, 3),
        "peak": round(p_add if bound == "fp32_add" else pk["hbm_gbs"], 3),
        "unit": "TFLOP/s" if bound == "fp32_add" else "GB/s",
        "frac": round((t_add if bound == "fp32_add" else bytes_loc / (pk["hbm_gbs"] * 1e9)) / (t_kernel * 1e-3), 4),
        "traffic": traffic,
        "traffic_source": traffic_src,
        "kernel_ms": round(t_kernel, 5),
        "algorithmic_ops_per_launch": ops_loc,
        "algorithmic_bytes_per_launch": bytes_loc,
        "peak_source": (f"fp32 FADD peak = {sms} SMs x {FADD_PER_CLK_PER_SM}/clk x {pk['sm_max_mhz']:.0f} MHz "
                        f"(sm_max_mhz of {pk['source']}); HBM {pk['hbm_gbs']} GB/s {pk['source']}"),
        "north_star_frac": round(max(t_add, t_hbm) / (t_kernel * 1e-3), 4),
        "hbm": {"achieved_gbs": round(achieved_gbs, 2), "peak_gbs": pk["hbm_gbs"],
                "frac": round(achieved_gbs / pk["hbm_gbs"], 4)},
    }
    if method == "mma" and i8 is not None:
        tens = 2 * 3 * M * K * w_loc  # int8 ops of the three limb GEMMs at the unpadded shape
        ach = tens / (t_run * 1e-3) / 1e12
        roof["tensor"] = {"achieved": round(ach, 2), "peak": round(i8["burst"]["tops"], 1), "unit": "TOP/s int8",
                          "frac": round(ach / i8["burst"]["tops"], 4),
                          "peak_sustained": round(i8["sustained"]["tops"], 1),
                          "frac_of_sustained": round(ach / i8["sustained"]["tops"], 4),
                          "peak_source": (f"measured in this run: tg_probe_i8_mma_rate (csrc/tg_peak.cu), "
                                          f"{sms} CTAs x back-to-back tcgen05.mma kind::i8 128x{i8['burst']['n']}x32, "
                                          f"A in {i8['burst']['a']}; burst {i8['burst']['seconds']:.2f} s, "
                                          f"sustained {i8['sustained']['seconds']:.1f} s")}

    cpu_line = None
    if cpu is not None:
        meas = cpu.measure(steps=3, warmup=1, step_seconds=2.0)
        cpu_line = {k: (round(v, 4) if isinstance(v, float) else v) for k, v in meas.items()}

    launches_per_step = 2  # mma: X split + tile MMA; gather: transpose + gather
    if sg is not None:
        launches_per_step = 3  # + the arrival wait
    conf = config_dict(cfg, nnz_total, args.x_outliers)
    line = {
        "metric": "effective_gops", "value": round(value, 3), "unit": "GOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t_step_max, 5), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (BASELINE.json recipe, seeded; no dataset)",
        "config": conf,
        "run": {"method": method, "x_rows": row_stats,
                "parallelism": f"N-sharded x{world}" + (
                    "" if world == 1 else " + fused peer-store epilogue over NVLink" if assembly == "peer"
                    else " + NCCL all-gather"),
                "launch": "CUDA graph replay per step" if graph is not None else "direct launches"},
        "breakdown_ms": {"prepare": round(t_prep, 5), "run": round(t_run, 5), "assemble": round(t_comm, 5),
                         "kernels_max_over_ranks": round(t_kernel_max, 5),
                         "note": "loop differences over K steps with direct launches; run = GEMM kernel after the "
                                 "split; assemble = extra time of the shard assembly (NCCL all-gather, or the fused "
                                 "peer stores + arrival wait)"},
        "assembly": {"kind": assembly, "note": asm_note},
        "roofline": roof,
        "cpu_baseline": cpu_line,
        "e2e": {"value": round(e2e_value, 3) if e2e_value else None, "unit": "GOP/s", "ms_per_step": round(t_e2e_ms, 4),
                "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": int(M * N * 4),
                "path": (f"ScatterGemm.step on pinned host X (H2D into the shard runners' X), rank 0 reads the "
                         f"assembled Y" if sg is not None else
                         f"public API gemm_* on pinned host X ({'pad_input + ' if sym else ''}{kind}), Y.values")},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk,
        "parity": parity,
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
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(WORKLOADS))
    ap.add_argument("--method", default="auto", choices=("auto", "mma", "gather"))
    ap.add_argument("--x-outliers", default=None, metavar="C@S",
                    help="scale C seeded channels of X by S (heavy-tailed activations; off: the BASELINE X)")
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
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"--gpus {args.gpus}: only {have} CUDA device(s) visible (one rank per GPU)")
        raise SystemExit(spawn_ranks(args.gpus))
    run_ours(args)


if __name__ == "__main__":
    main()
