"""GEMM entry points and the variant registry (reference: kernels/__init__.py,
kernels/scalar.py, kernels/simd.py) — same names, signatures, argument
checks and exception types; every call launches sm_100a kernels.

Two device paths serve every entry point (choose with ``GemmConfig(method=)``
or the ``method=`` keyword; "auto" picks by density):

  "gather"  CUDA-core walk of the format's own index stream, one fp32 lane per
            output element in the reference kernel's exact operation order —
            bit-identical to the reference for any finite X (csrc/tg_gather.cu).
  "mma"     dense-decode tensor-core path: the format is re-encoded once into
            2-bit ternary tiles, X is split into three exact int8 limbs and
            tcgen05.mma.kind::i8 accumulates in TMEM (csrc/tg_mma.cu).  Exact
            integer accumulation; bit-identical to the reference for
            integer-valued X, ~1e-7 normwise for real X (tolerance 1e-5).
"""

from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass, replace
from typing import Any, Callable, NamedTuple

import numpy as np
import torch

from . import _native as nat
from .dense import (
    BiasVector,
    DenseMatrix,
    TernaryDense,
    _device,
    _Dual,
    _deferred,
    _events,
    _pinned,
    as_bias,
    as_dense,
    as_ternary,
)
from .errors import ParameterError
from .formats import (
    DEFAULT_GROUP_SIMD,
    BlockedTcsc,
    CompressedTcsc,
    InterleavedBlockedTcsc,
    SymmetricInterleavedTcsc,
    Tcsc,
    blocked_from_dense,
    compressed_from_dense,
    interleaved_blocked_from_dense,
    symmetric_from_dense,
    tcsc_from_dense,
)

DEFAULT_UF = 12
DEFAULT_MR = 4
DEFAULT_NR = 4
ALLOWED_ROW_UNROLL = (1, 2, 4)
DEFAULT_ALPHA = 0.25
METHODS = ("auto", "gather", "mma")
# "auto" uses the tensor-core path when at least 1 in AUTO_MMA_MIN_DENSITY_INV
# entries of W is nonzero (dense MACs per useful add <= 64).
AUTO_MMA_MIN_DENSITY_INV = 64
AUTO_MMA_MIN_TERMS = 64  # and at least this many nonzeros per output column on average


class OpCount(NamedTuple):
    """Floating point operation counters (kernels/scalar.py:51-55)."""

    adds: int
    mults: int


@dataclass(frozen=True)
class GemmConfig:
    """Tuning knobs (kernels/scalar.py:58-94) plus ``method`` (device path)."""

    uf: int = DEFAULT_UF
    mr: int = DEFAULT_MR
    nr: int = DEFAULT_NR
    b: int | None = None
    g: int | None = None
    alpha: float | None = None
    variant: str = ""
    method: str = "auto"

    def __post_init__(self):
        if self.uf < 1:
            raise ParameterError(f"uf must be >= 1, got {self.uf}")
        if self.mr not in ALLOWED_ROW_UNROLL:
            raise ParameterError(f"mr must be one of {ALLOWED_ROW_UNROLL}, got {self.mr}")
        if self.nr not in ALLOWED_ROW_UNROLL:
            raise ParameterError(f"nr must be one of {ALLOWED_ROW_UNROLL}, got {self.nr}")
        if self.b is not None and self.b < 1:
            raise ParameterError(f"b must be >= 1, got {self.b}")
        if self.g is not None and self.g < 1:
            raise ParameterError(f"g must be >= 1, got {self.g}")
        if self.alpha is not None and not np.isfinite(self.alpha):
            raise ParameterError(f"alpha must be finite, got {self.alpha}")
        if self.method not in METHODS:
            raise ParameterError(f"method must be one of {METHODS}, got {self.method!r}")

    def with_variant(self, tag: str) -> "GemmConfig":
        return replace(self, variant=tag)


class PaddedInput:
    """M x (K+1) float32 matrix whose last column is zero (simd.py:40-70)."""

    def __init__(self, values):
        if isinstance(values, torch.Tensor):
            v = values.detach()
            if v.dim() != 2 or v.shape[1] < 1:
                raise ParameterError(f"padded input must be 2-D with >= 1 column, got {tuple(v.shape)}")
            v = v.float().contiguous()
            if not bool(torch.isfinite(v).all().item()):
                raise ParameterError("padded input contains non-finite values")
            if v.shape[0] and bool((v[:, -1] != 0).any().item()):
                raise ParameterError("padded slot (last column) must be exactly zero")
            self._v = _Dual(None, v)
            return
        v = np.ascontiguousarray(values, dtype=np.float32)
        if v.ndim != 2 or v.shape[1] < 1:
            raise ParameterError(f"padded input must be 2-D with >= 1 column, got {np.asarray(values).shape}")
        if not np.isfinite(v).all():
            raise ParameterError("padded input contains non-finite values")
        if v.shape[0] and (v[:, -1] != 0).any():
            raise ParameterError("padded slot (last column) must be exactly zero")
        self._v = _Dual(v, None)

    _pending = None  # pad_input of a host X: the unpadded host tensor, not uploaded yet
    _slot_exposed = False  # the host array was handed out through .values (the caller may write it)

    def _slot_nonzero(self) -> bool:
        """True when the padded slot may have been written after construction and is nonzero."""
        if not self._slot_exposed:
            return False
        h = self._v._h
        return bool(h[:, -1].any()) if h is not None else bool((self._v._d[:, -1] != 0).any().item())

    @classmethod
    def _trusted(cls, dev: torch.Tensor) -> "PaddedInput":
        obj = cls.__new__(cls)
        obj._v = _Dual(None, dev)
        return obj

    @classmethod
    def _from_host(cls, src: torch.Tensor) -> "PaddedInput":
        obj = cls.__new__(cls)
        obj._v = None
        obj._pending = src
        return obj

    def _materialise(self) -> None:
        src = self._pending
        M, K = int(src.shape[0]), int(src.shape[1])
        xp = torch.empty((M, K + 1), dtype=torch.float32, device=_device())
        xp[:, :-1].copy_(src, non_blocking=src.is_pinned())
        xp[:, -1].zero_()
        self._v, self._pending = _Dual(None, xp), None

    @property
    def _hsrc(self) -> torch.Tensor | None:
        """Host tensor to stream from ([M, K] pending, or the full padded host array)."""
        if self._pending is not None:
            return self._pending
        return _host_source(self._v)

    @property
    def values(self) -> np.ndarray:
        """The padded host array.  Like the reference's (a plain numpy array, simd.py:40-70) it
        may be written by the caller, so handing it out drops any device copy: the next kernel
        call uploads the array as it is then (the dummy-slot liveness check of the reference's
        acceptance test c5 writes the slot this way)."""
        if self._pending is not None:
            h = self._pending.numpy()
            hp = np.concatenate([h, np.zeros((h.shape[0], 1), np.float32)], axis=1)
            self._v, self._pending = _Dual(hp, None), None
            self._slot_exposed = True
            return hp
        h = self._v.host()
        self._v = _Dual(h, None)
        self._slot_exposed = True
        return h

    @property
    def device_values(self) -> torch.Tensor:
        if self._pending is not None:
            self._materialise()
        return self._v.dev()

    @property
    def M(self) -> int:
        return int(self._pending.shape[0]) if self._pending is not None else self._v.shape()[0]

    @property
    def K(self) -> int:
        return int(self._pending.shape[1]) if self._pending is not None else self._v.shape()[1] - 1

    def logical(self) -> DenseMatrix:
        return DenseMatrix(self.device_values[:, :-1].contiguous())


def pad_input(X) -> PaddedInput:
    """simd.py:72-75, on the device.  A host input is not copied here: it goes
    straight into the padded device buffer when first needed -- streamed in
    row chunks by a GEMM (GemmRunner.run_from_host), or one strided copy on
    ``device_values`` -- instead of uploading X and copying it again."""
    X = as_dense(X)
    v = X._v
    if v._d is not None and v._d.is_cuda:
        x = v._d
        xp = torch.empty((x.shape[0], x.shape[1] + 1), dtype=torch.float32, device=x.device)
        xp[:, :-1].copy_(x)
        xp[:, -1].zero_()
        return PaddedInput._trusted(xp)
    _device()  # no CUDA device: fail here, like the device path
    return PaddedInput._from_host(_host_source(v))


# ---------------------------------------------------------------- device plumbing

_ws_lock = threading.Lock()
_ws_cache: dict[tuple[int, int], torch.Tensor] = {}


def _stream() -> torch.cuda.Stream:
    return torch.cuda.current_stream()


def _workspace(nbytes: int, dev: torch.device, stream: int) -> torch.Tensor:
    key = (dev.index if dev.index is not None else torch.cuda.current_device(), stream)
    with _ws_lock:
        t = _ws_cache.get(key)
        if t is None or t.numel() < nbytes:
            t = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=dev)
            _ws_cache[key] = t
    return t


# Host X of at least this size goes through the library's host pipeline (tg_gemm_tiles_host:
# copies, split and GEMM in one graph-replayed call, Y and its status words back with it);
# smaller X is uploaded whole and launched through the runner.  0: every host X (measured:
# cfg4's public call 0.153 -> 0.117 ms, cfg1 0.107 -> 0.102 ms against the upload path).
STREAM_MIN_BYTES = int(os.environ.get("TG_STREAM_MIN_BYTES", "0"))


def _host_source(v) -> torch.Tensor | None:
    """The host tensor behind an operand that is not on the device yet, else None."""
    if v._d is not None:
        return None if v._d.is_cuda else v._d
    return torch.from_numpy(np.ascontiguousarray(v._h))


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _alpha_args(alpha: float | None) -> tuple[int, float]:
    """simd.py:85-90."""
    if alpha is None:
        return 0, 0.0
    if not np.isfinite(alpha):
        raise ParameterError(f"alpha must be finite, got {alpha}")
    return 1, float(np.float32(alpha))


def _check_dims(x_cols: int, K: int, bias_len: int, N: int) -> None:
    """kernels/scalar.py:97-101."""
    if x_cols != K:
        raise ParameterError(f"X has {x_cols} columns but the format has K = {K}")
    if bias_len != N:
        raise ParameterError(f"bias length {bias_len} != N = {N}")


def _check_padded(Xp: PaddedInput, K: int, bias_len: int, N: int) -> None:
    """simd.py:78-82."""
    if Xp.K != K:
        raise ParameterError(f"padded input has K = {Xp.K} but the format has K = {K}")
    if bias_len != N:
        raise ParameterError(f"bias length {bias_len} != N = {N}")


def choose_method(method: str, K: int, N: int, nnz: int) -> str:
    if method not in METHODS:
        raise ParameterError(f"method must be one of {METHODS}, got {method!r}")
    if method != "auto":
        return method
    if K > (1 << 24):
        return "gather"
    # few terms per output: the reference-order gather is cheap there, and it keeps every
    # output exact in the |terms|-scaled sense (the 22-bit row grid of the tensor-core
    # path is relative to the row maximum, which a handful of small terms need not reach)
    if nnz < AUTO_MMA_MIN_TERMS * N:
        return "gather"
    return "mma" if nnz * AUTO_MMA_MIN_DENSITY_INV >= K * N else "gather"


class GemmRunner:
    """One resolved GEMM call with its device buffers: ``launch()`` issues only
    kernel launches (no allocation, no synchronisation), so it can be replayed
    or captured in a CUDA graph.  Used by every gemm_* entry point."""

    def __init__(self, kind: str, x: torch.Tensor, fmt, bias: torch.Tensor, *, method: str, uf: int = 1,
                 mr: int = 1, alpha: float | None = None, out: torch.Tensor | None = None,
                 flags: torch.Tensor | None = None, scatter: "nat.TgPeerScatter | None" = None):
        self.kind = kind
        self.x = x
        self.fmt = fmt
        self.bias = bias
        self.M, self.ldx = int(x.shape[0]), int(x.shape[1])
        self.K, self.N = fmt.K, fmt.N
        self.uf, self.mr = uf, mr
        self.use_alpha, self.alpha = _alpha_args(alpha)
        self.method = method
        dev = x.device
        if out is False:  # a host-streaming plan: every call brings its own Y (run_from_host)
            self.y, self.ldy = None, self.N
        else:
            self.y = out if out is not None else torch.empty((self.M, self.N), dtype=torch.float32, device=dev)
            if tuple(self.y.shape) != (self.M, self.N) or self.y.dtype != torch.float32 or self.y.stride(1) != 1:
                raise ParameterError(f"out must be a float32 [{self.M}, {self.N}] view with unit column stride")
            self.ldy = int(self.y.stride(0))  # a column block of a wider Y (peer scatter) has ldy > N
        self.scatter = scatter
        if scatter is not None and method != "mma":
            raise ParameterError("the peer scatter is fused into the tensor-core epilogue: method must be 'mma'")
        self.flags = flags if flags is not None else torch.zeros(6, dtype=torch.int32, device=dev)
        self.ws_bytes = nat.load().tg_gemm_workspace_bytes(self.M, self.K, self.N)
        self.tiles = fmt.tiles() if method == "mma" else None
        self.exact = self._format_ref() if method == "mma" else None
        self._ws = None

    def _format_ref(self) -> nat.TgFormatRef:
        """The format's own arrays, for the exact-order fix-up of wide-range rows."""
        f, r = self.fmt, nat.TgFormatRef()
        r.uf, r.mr, r.g, r.B = max(self.uf, 1), max(self.mr, 1), 1, max(getattr(f, "B", f.K), 1)
        if self.kind in ("base", "unrolled", "blocked"):
            r.variant = {"base": nat.TG_VARIANT_BASE, "unrolled": nat.TG_VARIANT_UNROLLED,
                         "blocked": nat.TG_VARIANT_BLOCKED}[self.kind]
            r.a0, r.a1 = f.device("col_start_pos").data_ptr(), f.device("row_index_pos").data_ptr()
            r.a2, r.a3 = f.device("col_start_neg").data_ptr(), f.device("row_index_neg").data_ptr()
        elif self.kind in ("vertical", "horizontal"):
            r.variant = nat.TG_VARIANT_VERTICAL if self.kind == "vertical" else nat.TG_VARIANT_HORIZONTAL
            r.g = f.g
            r.a0, r.a1 = f.device("col_ptr").data_ptr(), f.device("indices").data_ptr()
        elif self.kind == "compressed":
            r.variant = nat.TG_VARIANT_COMPRESSED
            r.codes = f.device().data_ptr()
        else:
            r.variant = (nat.TG_VARIANT_VECTORIZED_OPTIMAL if self.kind == "vectorized_optimal"
                         else nat.TG_VARIANT_INTERLEAVED_BLOCKED)
            r.g = f.g
            r.a0, r.a1 = f.device("col_segment_ptr").data_ptr(), f.device("all_indices").data_ptr()
        return r

    def launch(self, stream: int | None = None, ws: torch.Tensor | None = None, stage: str = "all",
               rows: tuple[int, int] | None = None) -> None:
        """Issue the call.  For the tensor-core path ``stage`` may be "prepare"
        (X limb split) or "run" (tile MMA + exact-order fix-up) so a caller can
        time the two halves separately; "all" issues both.  ``rows`` = (r0, r1)
        restricts the call to those rows of X and Y (every kernel computes rows
        independently; r0 must be a multiple of ``mr`` for the blocked order)."""
        st = torch.cuda.current_stream().cuda_stream if stream is None else stream
        if ws is None:
            ws = self._ws if self._ws is not None else _workspace(self.ws_bytes, self.x.device, st)
        x, y, b, fl = _p(self.x), _p(self.y), _p(self.bias), _p(self.flags)
        M, K, N, ldx = self.M, self.K, self.N, self.ldx
        if rows is not None:
            r0, r1 = rows
            if self.scatter is not None or not 0 <= r0 < r1 <= self.M or r0 % self.mr:
                raise ParameterError(f"bad row range {rows} for M = {self.M}, mr = {self.mr}")
            x = ctypes.c_void_p(self.x.data_ptr() + 4 * r0 * ldx)
            y = ctypes.c_void_p(self.y.data_ptr() + 4 * r0 * self.ldy)
            M = r1 - r0
        f = self.fmt
        if self.method == "mma":
            if stage in ("all", "prepare"):
                nat.call("tg_gemm_tiles_prepare", x, M, K, ldx, _p(ws), ws.numel(), fl, st)
            if stage in ("all", "run"):
                if self.scatter is not None:
                    nat.call("tg_gemm_tiles_run_scatter", x, M, K, ldx, _p(self.tiles), N, b, y, self.ldy,
                             self.use_alpha, self.alpha, ctypes.byref(self.exact), ctypes.byref(self.scatter),
                             _p(ws), ws.numel(), fl, st)
                else:
                    nat.call("tg_gemm_tiles_run", x, M, K, ldx, _p(self.tiles), N, b, y, self.ldy, self.use_alpha,
                             self.alpha, ctypes.byref(self.exact), _p(ws), ws.numel(), fl, st)
            return
        if stage == "prepare":
            return
        if self.kind in ("vertical", "horizontal"):
            order = nat.TG_ORDER_VERTICAL if self.kind == "vertical" else nat.TG_ORDER_HORIZONTAL
            nat.call("tg_gemm_symmetric", x, M, K, ldx, f.g, _p(f.device("indices")), _p(f.device("col_ptr")), N, b,
                     y, self.ldy, order, self.use_alpha, self.alpha, _p(ws), ws.numel(), fl, st)
        elif self.kind == "compressed":
            nat.call("tg_gemm_compressed", x, M, K, ldx, _p(f.device()), N, b, y, self.ldy, _p(ws), ws.numel(), fl,
                     st)
        elif self.kind in ("base", "unrolled"):
            nat.call("tg_gemm_tcsc", x, M, K, ldx, _p(f.device("col_start_pos")), _p(f.device("row_index_pos")),
                     _p(f.device("col_start_neg")), _p(f.device("row_index_neg")), N, b, y, self.ldy,
                     0 if self.kind == "base" else self.uf, self.use_alpha, self.alpha, _p(ws), ws.numel(), fl, st)
        elif self.kind == "blocked":
            nat.call("tg_gemm_blocked", x, M, K, ldx, f.B, _p(f.device("col_start_pos")),
                     _p(f.device("row_index_pos")), _p(f.device("col_start_neg")), _p(f.device("row_index_neg")), N,
                     b, y, self.ldy, self.uf, self.mr, self.use_alpha, self.alpha, _p(ws), ws.numel(), fl, st)
        else:
            order = (nat.TG_ORDER_VECTORIZED_OPTIMAL if self.kind == "vectorized_optimal"
                     else nat.TG_ORDER_INTERLEAVED_BLOCKED)
            nat.call("tg_gemm_interleaved_blocked", x, M, K, ldx, f.B, f.g, _p(f.device("all_indices")),
                     _p(f.device("col_segment_ptr")), N, b, y, self.ldy, order, self.use_alpha, self.alpha, _p(ws),
                     ws.numel(), fl, st)

    def row_stats(self) -> dict:
        """Diagnostics of the tensor-core path's X split (run on the pinned workspace):
        how many rows went to the exact-order walk, how many shed outlier entries, and how
        many entries were listed.  Synchronises."""
        if self.method != "mma":
            raise ParameterError("row_stats describes the tensor-core path")
        if self._ws is None:
            self.pin_workspace()
        self.launch(stage="prepare")
        out = (ctypes.c_int64 * 3)()
        nat.call("tg_gemm_tiles_row_stats", _p(self._ws), self._ws.numel(), self.M, self.K, out,
                 torch.cuda.current_stream().cuda_stream)
        return {"exact_rows": int(out[0]), "outlier_rows": int(out[1]), "outlier_entries": int(out[2])}

    def capture(self, warmup: bool = True) -> "torch.cuda.CUDAGraph":
        """Capture ``launch()`` (X split + tile MMA, or the gather walk) into a CUDA
        graph: one host launch per replay, no host gaps between the kernels
        (the tensor-core pair keeps its programmatic-dependent-launch overlap).
        Replays reuse this runner's buffers (x, y, workspace): refresh x in place."""
        if self._ws is None:
            self.pin_workspace()
        s = torch.cuda.Stream(device=self.x.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            if warmup:
                self.launch()  # initialises the library's one-time state outside capture
            s.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                self.launch()
        torch.cuda.current_stream().wait_stream(s)
        return g

    def run_from_host(self, hx: torch.Tensor, bias: torch.Tensor | None = None,
                      st: torch.cuda.Stream | None = None) -> DenseMatrix:
        """X arrives from host memory (tensor-core path): the library streams it
        in row chunks, each chunk's host->device copy, GEMM and device->host
        copy of Y on its own stream, so the two PCIe directions and the GEMMs
        overlap (tg_gemm_tiles_host).  ``hx`` is [M, <= ldx] (pinned for
        asynchronous copies); columns of x beyond it are zeroed (the padded
        input's slot).  ``bias`` overrides the runner's.  Y is fresh per call
        (returned to the caller); x, the workspace and the status words are the
        runner's, so a repeated call repeats every pointer and the library
        replays its CUDA graph of the first.  Returns a DenseMatrix whose host
        values and status words arrive together with the last chunk."""
        if self.method != "mma" or self.scatter is not None:
            raise ParameterError("host streaming runs the tensor-core path")
        if not hx.is_contiguous():
            hx = hx.contiguous()
        dev = self.x.device
        if st is None:
            st = torch.cuda.current_stream(dev)
        chunks_env = os.environ.get("TG_HOST_CHUNKS")  # the chunk plan (and workspace) follows it
        if self._ws is None or getattr(self, "_ws_env", None) != chunks_env:
            ws_bytes = nat.load().tg_gemm_host_workspace_bytes(self.M, self.K, self.N)
            self._ws_env = chunks_env
        else:
            ws_bytes = self._ws.numel()
        if self._ws is None or self._ws.numel() < ws_bytes:
            self._ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
        ws = self._ws
        b = self.bias if bias is None else bias
        _deferred.drain()
        y = torch.empty((self.M, self.N), dtype=torch.float32, device=dev)
        y_host = _pinned.take((self.M, self.N), torch.float32)
        f_host = _pinned.take((6,), torch.int32)
        nat.call("tg_gemm_tiles_host", ctypes.c_void_p(hx.data_ptr()), self.M, self.K, int(hx.shape[1]),
                 _p(self.x), self.ldx, _p(self.tiles), self.N, _p(b), _p(y), self.N,
                 ctypes.c_void_p(y_host.data_ptr()), self.N, self.use_alpha, self.alpha, ctypes.byref(self.exact),
                 _p(ws), ws.numel(), _p(self.flags), ctypes.c_void_p(f_host.data_ptr()), st.cuda_stream)
        done = _events.take()
        done.record(st)
        return DenseMatrix._streamed(y, y_host, f_host, done, keep=(hx,))

    def pin_workspace(self) -> None:
        """Give this runner a private workspace (needed for graph capture / concurrent replays)."""
        self._ws = torch.empty(max(self.ws_bytes, 1), dtype=torch.uint8, device=self.x.device)

    def result(self) -> DenseMatrix:
        return DenseMatrix(self.y, _flags=self.flags)

    def nonpositive(self) -> int:
        f = self.flags.cpu().numpy().view(np.uint32)
        return int(f[2]) | (int(f[3]) << 32)


_PLANS_PER_FORMAT = 4


def _host_plan(kind: str, fmt, M: int, cols: int, method: str, kw: dict, st: torch.cuda.Stream) -> GemmRunner:
    """The cached host-streaming runner of ``fmt`` for this call shape (staging X,
    workspace, status words and format reference built once; LRU of a few per
    format, keyed by the stream too, so calls on different streams never share
    a staging buffer)."""
    dev = st.device
    key = (kind, M, cols, method, kw.get("uf", 1), kw.get("mr", 1), kw.get("alpha"), dev.index, st.cuda_stream)
    plans = fmt.__dict__.setdefault("_host_plans", {})
    r = plans.pop(key, None)
    if r is None:
        # a contiguous [M, K] staging X (no padded slot column: the tensor-core path never
        # reads it, and its exact-order fix-up reads the slot as zero), so every X chunk
        # arrives with one linear copy (a pitched 2-D copy runs ~18% slower)
        x = torch.empty((M, fmt.K), dtype=torch.float32, device=dev)
        r = GemmRunner(kind, x, fmt, None, method=method, out=False, **kw)
        if len(plans) >= _PLANS_PER_FORMAT:
            plans.pop(next(iter(plans)))
    plans[key] = r  # most recently used last
    return r


def _dispatch(kind: str, X, fmt, bias: torch.Tensor, method: str, counted: bool, adds: int, **kw):
    """Run one gemm_* call.  X still in host memory and large enough to pay for
    chunking streams through the cached plan (tensor-core path,
    GemmRunner.run_from_host); anything else is uploaded whole and launched."""
    if isinstance(X, PaddedInput):
        hs, cols = X._hsrc, X.K + 1
    else:
        hs, cols = _host_source(X._v), X.cols
    if method == "mma" and hs is not None and hs.numel() * 4 >= STREAM_MIN_BYTES:
        _device()
        st = torch.cuda.current_stream()
        with _plan_lock:
            plan = _host_plan(kind, fmt, int(hs.shape[0]), cols, method, kw, st)
            y = plan.run_from_host(hs, bias, st)
        if not counted:
            return y
        return y, OpCount(int(adds), y._nonpositive() if plan.use_alpha else 0)
    runner = GemmRunner(kind, X.device_values, fmt, bias, method=method, **kw)
    runner.launch()
    y = runner.result()
    if not counted:
        return y
    mults = runner.nonpositive() if runner.use_alpha else 0
    return y, OpCount(int(adds), int(mults))


_plan_lock = threading.Lock()


def _as_cfg(cfg) -> GemmConfig:
    """Accept the reference's own GemmConfig (kernels/scalar.py:58-94, no ``method``) as well
    as this package's, so a caller of the reference can pass its configs unchanged."""
    if cfg is None:
        return GemmConfig()
    if isinstance(cfg, GemmConfig):
        return cfg
    return GemmConfig(uf=cfg.uf, mr=cfg.mr, nr=cfg.nr, b=cfg.b, g=cfg.g, alpha=cfg.alpha,
                      variant=getattr(cfg, "variant", ""), method=getattr(cfg, "method", "auto"))


def _method(cfg: GemmConfig | None, method: str | None, K: int, N: int, nnz: int) -> str:
    m = method if method is not None else (_as_cfg(cfg).method if cfg is not None else "auto")
    return choose_method(m, K, N, nnz)


def _padded_method(m: str, Xp: "PaddedInput") -> str:
    """The tensor-core path drops the symmetric formats' dummy indices (index K reads the zero
    slot, the PaddedInput invariant of simd.py:40-70).  A slot written after construction (the
    reference's arrays are mutable; its acceptance test c5 does exactly this) is read by the
    reference kernels, so such a call takes the exact-order gather kernel, which reads it too."""
    if m == "mma" and Xp._slot_nonzero():
        return "gather"
    return m


# ---------------------------------------------------------------- entry points


def _as_tcsc(t) -> Tcsc:
    if isinstance(t, Tcsc):
        return t
    return Tcsc(t.K, t.N, t.col_start_pos, t.row_index_pos, t.col_start_neg, t.row_index_neg)


def _as_blocked(t) -> BlockedTcsc:
    if isinstance(t, BlockedTcsc):
        return t
    return BlockedTcsc(t.K, t.N, t.B, t.col_start_pos, t.row_index_pos, t.col_start_neg, t.row_index_neg)


def _as_ib(t) -> InterleavedBlockedTcsc:
    if isinstance(t, InterleavedBlockedTcsc):
        return t
    return InterleavedBlockedTcsc(t.K, t.N, t.B, t.g, t.all_indices, t.col_segment_ptr,
                                  getattr(t, "symmetric_groups", False))


def gemm_base(X, t, b, counted: bool = False, *, method: str | None = None):
    """kernels/scalar.py:135-148.  counted: adds = M*N + M*nnz, mults = 0."""
    X, b, t = as_dense(X), as_bias(b), _as_tcsc(t)
    _check_dims(X.cols, t.K, len(b), t.N)
    m = _method(None, method, t.K, t.N, t.nnz)
    return _dispatch("base", X, t, b.device_values, m, counted, X.rows * t.N + X.rows * t.nnz)


def gemm_unrolled(X, t, b, cfg: GemmConfig | None = None, counted: bool = False, *, method: str | None = None):
    """kernels/scalar.py:260-278 (uf accumulator banks; mr/nr change no output bit)."""
    cfg = _as_cfg(cfg)
    X, b, t = as_dense(X), as_bias(b), _as_tcsc(t)
    _check_dims(X.cols, t.K, len(b), t.N)
    m = _method(cfg, method, t.K, t.N, t.nnz)
    M = X.rows
    return _dispatch("unrolled", X, t, b.device_values, m, counted, M * t.nnz + M * t.N * (cfg.uf + 1), uf=cfg.uf)


def gemm_blocked(X, t, b, cfg: GemmConfig | None = None, counted: bool = False, *, method: str | None = None):
    """kernels/scalar.py:370-389."""
    cfg = _as_cfg(cfg)
    X, b, t = as_dense(X), as_bias(b), _as_blocked(t)
    _check_dims(X.cols, t.K, len(b), t.N)
    m = _method(cfg, method, t.K, t.N, t.nnz)
    M, nb = X.rows, t.num_blocks
    mf = M // cfg.mr * cfg.mr
    adds = M * t.nnz + mf * t.N * nb * (cfg.uf + 1) + (M - mf) * t.N * nb
    return _dispatch("blocked", X, t, b.device_values, m, counted, adds, uf=cfg.uf, mr=cfg.mr)


def gemm_interleaved_blocked(X, t, b, cfg: GemmConfig | None = None, counted: bool = False, *,
                             method: str | None = None):
    """kernels/scalar.py:488-511; rejects symmetric formats like the reference (:502-505)."""
    cfg = _as_cfg(cfg)
    X, b, t = as_dense(X), as_bias(b), _as_ib(t)
    _check_dims(X.cols, t.K, len(b), t.N)
    if t.symmetric_groups:
        raise ParameterError(
            "scalar kernel cannot consume symmetric-group formats (dummy index needs a padded input row)"
        )
    m = _method(cfg, method, t.K, t.N, t.nnz)
    M = X.rows
    return _dispatch("interleaved_blocked", X, t, b.device_values, m, counted, M * t.nnz + M * t.N * t.num_blocks)


def gemm_vectorized_optimal(Xp, t, b, alpha: float | None = None, cfg: GemmConfig | None = None,
                            counted: bool = False, *, method: str | None = None):
    """kernels/simd.py:423-449: symmetric interleaved-blocked stream + fused bias/PReLU."""
    if not isinstance(Xp, PaddedInput):
        Xp = PaddedInput(getattr(Xp, "values", Xp))
    b, t = as_bias(b), _as_ib(t)
    _check_padded(Xp, t.K, len(b), t.N)
    if not t.symmetric_groups:
        raise ParameterError("gemm_vectorized_optimal needs symmetric 4-column groups (symmetric_cols=True)")
    if alpha is None and cfg is not None:
        alpha = _as_cfg(cfg).alpha
    _alpha_args(alpha)
    n_idx = t._len("all_indices")
    m = _padded_method(_method(cfg, method, t.K, t.N, n_idx), Xp)
    adds = Xp.M * (n_idx + t.N * t.num_blocks)
    return _dispatch("vectorized_optimal", Xp, t, b.device_values, m, counted, adds, alpha=alpha)


def _as_sym(t) -> SymmetricInterleavedTcsc:
    if isinstance(t, SymmetricInterleavedTcsc):
        return t
    return SymmetricInterleavedTcsc(t.K, t.N, t.g, t.indices, t.col_ptr)


def _as_compressed(t) -> CompressedTcsc:
    if isinstance(t, CompressedTcsc):
        return t
    return CompressedTcsc(t.K, t.N, t.codes)


def _symmetric_kernel(kind: str, Xp, t, b, alpha, counted, method):
    if not isinstance(Xp, PaddedInput):
        Xp = PaddedInput(getattr(Xp, "values", Xp))
    b, t = as_bias(b), _as_sym(t)
    _check_padded(Xp, t.K, len(b), t.N)
    _alpha_args(alpha)
    n_idx = t._len("indices")
    m = _padded_method(_method(None, method, t.K, t.N, n_idx), Xp)
    extra = 2 if kind == "vertical" else 4  # simd.py:167-170 (b + p - q) / :253-256 (pairwise + b)
    return _dispatch(kind, Xp, t, b.device_values, m, counted, Xp.M * (n_idx + extra * t.N), alpha=alpha)


def gemm_vertical(Xp, t, b, alpha: float | None = None, counted: bool = False, *, method: str | None = None):
    """kernels/simd.py:98-188 over a SymmetricInterleavedTcsc: run-parity sums p, q; y = (b + p) - q, PReLU.
    counted: adds = M * (len(indices) + 2N) (dummies included), mults = #(y <= 0) with alpha."""
    return _symmetric_kernel("vertical", Xp, t, b, alpha, counted, method)


def gemm_horizontal(Xp, t, b, alpha: float | None = None, counted: bool = False, *, method: str | None = None):
    """kernels/simd.py:196-274: four lane sums over the stream, y = b + ((a0 + a1) + (a2 + a3)), PReLU.
    counted: adds = M * (len(indices) + 4N)."""
    return _symmetric_kernel("horizontal", Xp, t, b, alpha, counted, method)


def gemm_compressed(X, t, b, counted: bool = False, *, method: str | None = None):
    """kernels/scalar.py:561-602 over 5-trits-per-byte codes: per column, digits in k order
    (+x for +1, -x for -1), out = b + acc.  counted: adds = M*nnz + M*N, mults = 0."""
    X, b, t = as_dense(X), as_bias(b), _as_compressed(t)
    _check_dims(X.cols, t.K, len(b), t.N)
    m = method if method is not None else "auto"
    if m == "auto":
        m = "mma" if t.K <= (1 << 24) else "gather"  # the code stream is dense: density gives no signal
    m = choose_method(m, t.K, t.N, t.K * t.N)
    nnz = t.nnz if counted else 0
    return _dispatch("compressed", X, t, b.device_values, m, counted, X.rows * nnz + X.rows * t.N)


# ---------------------------------------------------------------- registry (kernels/__init__.py:66-230)


@dataclass(frozen=True)
class VariantSpec:
    """How one variant tag plugs into the harness (kernels/__init__.py:66-80)."""

    tag: str
    kind: str  # "scalar" or "simd"
    supports_alpha: bool
    emit: frozenset
    build: Callable[[TernaryDense, GemmConfig], Any]
    prepare: Callable[[DenseMatrix], Any]
    run: Callable[[Any, Any, BiasVector, GemmConfig, bool], Any]


def _identity(x):
    return as_dense(x)


def _g(cfg: GemmConfig, default: int) -> int:
    return default if cfg.g is None else cfg.g


VARIANTS: dict[str, VariantSpec] = {}


def _register(spec: VariantSpec) -> None:
    VARIANTS[spec.tag] = spec


_register(VariantSpec("base", "scalar", False, frozenset(), lambda w, cfg: tcsc_from_dense(w), _identity,
                      lambda x, f, b, cfg, counted: gemm_base(x, f, b, counted, method=_as_cfg(cfg).method)))
_register(VariantSpec("unrolled", "scalar", False, frozenset({"UF", "MR", "NR"}), lambda w, cfg: tcsc_from_dense(w),
                      _identity, lambda x, f, b, cfg, counted: gemm_unrolled(x, f, b, cfg, counted)))
_register(VariantSpec("blocked", "scalar", False, frozenset({"UF", "MR", "NR", "B"}),
                      lambda w, cfg: blocked_from_dense(w, cfg.b), _identity,
                      lambda x, f, b, cfg, counted: gemm_blocked(x, f, b, cfg, counted)))
_register(VariantSpec("interleaved_blocked", "scalar", False, frozenset({"MR", "NR", "B", "g"}),
                      lambda w, cfg: interleaved_blocked_from_dense(w, cfg.b, _g(cfg, DEFAULT_GROUP_SIMD)), _identity,
                      lambda x, f, b, cfg, counted: gemm_interleaved_blocked(x, f, b, cfg, counted)))
_register(VariantSpec("compressed", "scalar", False, frozenset(), lambda w, cfg: compressed_from_dense(w), _identity,
                      lambda x, f, b, cfg, counted: gemm_compressed(x, f, b, counted, method=_as_cfg(cfg).method)))
_register(VariantSpec("vertical", "simd", True, frozenset({"g"}),
                      lambda w, cfg: symmetric_from_dense(w, _g(cfg, DEFAULT_GROUP_SIMD)), pad_input,
                      lambda x, f, b, cfg, counted: gemm_vertical(x, f, b, cfg.alpha, counted, method=_as_cfg(cfg).method)))
_register(VariantSpec("horizontal", "simd", True, frozenset({"g"}),
                      lambda w, cfg: symmetric_from_dense(w, _g(cfg, DEFAULT_GROUP_SIMD)), pad_input,
                      lambda x, f, b, cfg, counted: gemm_horizontal(x, f, b, cfg.alpha, counted, method=_as_cfg(cfg).method)))
_register(VariantSpec("vectorized_optimal", "simd", True, frozenset({"B", "g"}),
                      lambda w, cfg: interleaved_blocked_from_dense(w, cfg.b, _g(cfg, DEFAULT_GROUP_SIMD),
                                                                    symmetric_cols=True),
                      pad_input,
                      lambda x, f, b, cfg, counted: gemm_vectorized_optimal(x, f, b, cfg.alpha, cfg, counted)))

SCALAR_TAGS = tuple(tag for tag, s in VARIANTS.items() if s.kind == "scalar")
SIMD_TAGS = tuple(tag for tag, s in VARIANTS.items() if s.kind == "simd")


def get_variant(tag: str) -> VariantSpec:
    spec = VARIANTS.get(tag)
    if spec is None:
        raise ParameterError(f"unknown variant {tag!r}; known: {', '.join(VARIANTS)}")
    return spec


def run_variant(tag: str, X, W, b, cfg: GemmConfig | None = None, counted: bool = False):
    """kernels/__init__.py:211-230: build the format, prepare X, run once."""
    cfg = _as_cfg(cfg)
    spec = get_variant(tag)
    if cfg.alpha is not None and not spec.supports_alpha:
        raise ParameterError(f"variant {tag!r} has no fused PReLU; alpha is vectorized-only")
    fmt = spec.build(as_ternary(W), cfg)
    prepared = spec.prepare(as_dense(X))
    return spec.run(prepared, fmt, as_bias(b), cfg, counted)
