"""Cost model and parity predicates of the reference harness (reference: bench.py:53-73
flop_count / operational_intensity; bench.py:135-150 _verify's comparison), plus the measured
int8 tensor-core rate the roofline uses.  The verify-then-time gate itself (a failing point is
refused, bench.py:167-169) lives in the repo's bench.py, on the device.

The grid search, presets and CSV plumbing of the reference harness tune CPU
unroll factors and are out of scope.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .errors import ParameterError

VERIFY_RTOL = 1e-5  # reference bench.py:49 (its elementwise check is reported, the gate is normwise / |terms|-scaled)


def flop_count(M: int, K: int, N: int, nnz: int) -> int:
    """bench.py:53-61: M*N bias adds + one add per (row, nonzero)."""
    if M < 1 or K < 1 or N < 1:
        raise ParameterError(f"dimensions must be >= 1, got M={M} K={K} N={N}")
    if not 0 <= nnz <= K * N:
        raise ParameterError(f"nnz = {nnz} outside [0, K*N = {K * N}]")
    return M * N + M * nnz


def operational_intensity(M: int, K: int, N: int, nnz: int, format_bytes: int) -> float:
    """bench.py:64-73: flops / (format bytes + 4MK + 4MN + 4N)."""
    if format_bytes < 0:
        raise ParameterError(f"format_bytes must be >= 0, got {format_bytes}")
    return flop_count(M, K, N, nnz) / (format_bytes + 4 * M * K + 4 * M * N + 4 * N)


@dataclass(frozen=True)
class Agreement:
    exact: bool
    normwise: float
    scaled: float
    rtol_fails: int  # the reference's own elementwise rtol=1e-5, atol=0 check (reported, not gated)


def agreement(y: np.ndarray, ref: np.ndarray, scale: np.ndarray | None = None) -> Agreement:
    """Parity predicates of SURVEY.md 8(c): bit-exact / normwise / |terms|-scaled."""
    y64 = np.asarray(y, np.float64)
    r64 = np.asarray(ref, np.float64)
    err = np.abs(y64 - r64)
    den = np.abs(r64).max() if r64.size else 0.0
    normwise = float(err.max() / den) if den > 0 else float(err.max() if err.size else 0.0)
    if scale is None:
        scaled = float("nan")
    else:
        with np.errstate(divide="ignore", invalid="ignore"):
            q = np.where(scale > 0, err / scale, np.where(err > 0, np.inf, 0.0))
        scaled = float(q.max()) if q.size else 0.0
    fails = int((~np.isclose(y64, r64, rtol=VERIFY_RTOL, atol=0.0)).sum())
    return Agreement(bool(np.array_equal(np.asarray(y), np.asarray(ref))), normwise, scaled, fails)


def measure_i8_mma_peak(n: int = 256, a_in_tmem: bool = False, seconds: float = 0.05,
                        repeats: int = 4) -> dict:
    """Measured int8 tcgen05.mma rate of the current device (``tg_probe_i8_mma_rate``,
    csrc/tg_peak.cu): one persistent CTA per SM issuing back-to-back M=128 x n x K=32
    kind::i8 MMAs.  ``seconds`` sizes each launch; ``repeats`` launches are timed
    back to back with CUDA events (a ~0.2 s run gives the burst rate, a few seconds the
    rate under the power cap).  Returns {"tops", "seconds", "n", "a"}."""
    from . import _native

    lib = _native.load()
    ops, sec = ctypes.c_double(), ctypes.c_double()
    # calibrate the per-launch iteration count on a short run (~16 MMAs per iteration)
    iters = 2000
    _native.check(lib.tg_probe_i8_mma_rate(n, int(a_in_tmem), iters, 1, ctypes.byref(ops), ctypes.byref(sec)),
                  "tg_probe_i8_mma_rate")
    iters = max(1, int(iters * seconds / max(sec.value, 1e-6)))
    _native.check(lib.tg_probe_i8_mma_rate(n, int(a_in_tmem), iters, repeats, ctypes.byref(ops),
                                           ctypes.byref(sec)), "tg_probe_i8_mma_rate")
    return {"tops": ops.value / 1e12, "seconds": sec.value, "n": n, "a": "tmem" if a_in_tmem else "smem"}
