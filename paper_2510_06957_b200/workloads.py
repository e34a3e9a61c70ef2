"""Seeded synthetic inputs for the BASELINE.json configurations.

The reference's own generators (dense.py:114-181) draw exact per-column
densities and integer-valued X; BASELINE.json's configs instead specify i.i.d.
nonzero positions and real-valued X / b.  This module implements the recipe
of SURVEY.md section 8(d) so that the GPU path, the CPU oracle and the golden
fixtures all see the same arrays:

  rng = np.random.default_rng(seed); draw order W, X, b
  u = rng.random((K, N), float32); W = +1 if u < p+, -1 if p+ <= u < p+ + p-, else 0
  X = (rng.random((M, K), float64) * 2 - 1).astype(float32)      (uniform[-1, 1))
      or rng.standard_normal((M, K), float32)                     (N(0, 1))
  b = rng.standard_normal(N, float32) or zeros

The integer-regime twin (``integer=True``) keeps W and draws integer X and b
in [-8, 8] (dense.py:143-160, 176-181), for which every kernel is bit-exact.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    M: int
    K: int
    N: int
    p_pos: float
    p_neg: float
    x_dist: str  # "uniform" | "normal"
    bias: str  # "normal" | "zeros"
    alpha: float | None
    seed: int
    variant: str  # reference registry tag whose path the config exercises
    description: str


def _cfg3(s: Fraction) -> Workload:
    return Workload(f"cfg3_s{s.numerator}_{s.denominator}", 512, 8192, 8192, float(s) / 2, float(s) / 2, "normal",
                    "normal", None, 3, "interleaved_blocked", f"sparsity sweep s={s}")


WORKLOADS: dict[str, Workload] = {
    "cfg1": Workload("cfg1", 64, 512, 512, 0.25, 0.25, "uniform", "normal", None, 1, "base",
                     "BaseTCSC, no activation (CPU-runnable)"),
    "cfg2": Workload("cfg2", 256, 4096, 4096, 0.25, 0.25, "uniform", "normal", 0.25, 2, "vectorized_optimal",
                     "blocked/interleaved TCSC + fused PReLU(0.25)"),
    "cfg4": Workload("cfg4", 16, 4096, 11008, 0.30, 0.30, "normal", "zeros", 0.25, 4, "vectorized_optimal",
                     "ternary-LLM FFN projection, decode-like M=16"),
    "cfg5": Workload("cfg5", 8192, 8192, 16384, 0.25, 0.25, "uniform", "normal", None, 5, "interleaved_blocked",
                     "large multi-GPU GEMM (N-sharded)"),
}
for _s in (Fraction(1, 16), Fraction(1, 8), Fraction(1, 4), Fraction(1, 2)):
    WORKLOADS[_cfg3(_s).name] = _cfg3(_s)
WORKLOADS["cfg3"] = WORKLOADS["cfg3_s1_2"]

CFG5_SLICE_SEED = 5000


def cfg5_oracle_rows(M: int = 8192, n: int = 256) -> np.ndarray:
    """The seeded 256-row slice of cfg5 the CPU oracle is checked and timed on."""
    return np.sort(np.random.default_rng(CFG5_SLICE_SEED).choice(M, n, replace=False))


def make_w(wl: Workload, rng: np.random.Generator) -> np.ndarray:
    u = rng.random((wl.K, wl.N), dtype=np.float32)
    w = np.zeros((wl.K, wl.N), dtype=np.int8)
    w[u < wl.p_pos] = 1
    w[(u >= wl.p_pos) & (u < wl.p_pos + wl.p_neg)] = -1
    return w


def make_inputs(name: str, integer: bool = False, M: int | None = None):
    """Return (W int8 KxN, X float32 MxK, b float32 N) for a BASELINE config.

    ``M`` overrides the row count (X is drawn for the override, so it is a
    different stream; used only for scaled-down smoke cases)."""
    wl = WORKLOADS[name]
    rng = np.random.default_rng(wl.seed)
    W = make_w(wl, rng)
    m = wl.M if M is None else M
    if integer:
        X = rng.integers(-8, 9, size=(m, wl.K)).astype(np.float32)
        b = rng.integers(-8, 9, size=wl.N).astype(np.float32)
        return W, X, b
    if wl.x_dist == "uniform":
        X = (rng.random((m, wl.K), dtype=np.float64) * 2.0 - 1.0).astype(np.float32)
    else:
        X = rng.standard_normal((m, wl.K), dtype=np.float32)
    b = rng.standard_normal(wl.N, dtype=np.float32) if wl.bias == "normal" else np.zeros(wl.N, np.float32)
    return W, X, b


def ops(M: int, N: int, nnz: int) -> int:
    """Algorithmic ops of one evaluation: M*nnz add/subs + M*N bias adds (bench.py:53-61)."""
    return M * N + M * nnz


def tcsc_bytes(K: int, N: int, nnz: int) -> int:
    """tcsc.py:186-190: two N+1 offset arrays + nnz int32 indices."""
    return 4 * (2 * (N + 1) + nnz)


def algorithmic_bytes(M: int, K: int, N: int, nnz: int) -> int:
    """Compulsory bytes with the reference's TCSC accounting (bench.py:64-73)."""
    return tcsc_bytes(K, N, nnz) + 4 * M * K + 4 * M * N + 4 * N
