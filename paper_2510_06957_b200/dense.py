"""Dense operand types of the drop-in API (reference: dense.py:32-111).

Each type wraps either a host numpy array (validated on construction exactly
like the reference) or a CUDA tensor (kept resident in HBM).  ``.values``
always returns a host numpy array — the reference's contract — copying from
the device lazily and once; ``.device_values`` returns the CUDA tensor,
uploading lazily and once.  Kernel outputs are device-resident DenseMatrix
objects whose finiteness check (dense.py:77) is carried by a device flag
written by the kernel epilogue and raised on first host access, so the hot
path never synchronises.
"""

from __future__ import annotations

import threading
from collections import deque
from fractions import Fraction
import weakref

import numpy as np
import torch

from .errors import ParameterError

EXACT_FLOAT32_BOUND = 2**24  # dense.py:17


_cuda_seen = False


def _device() -> torch.device:
    global _cuda_seen
    if not _cuda_seen:  # is_available() costs microseconds per call; a device does not go away
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2510_06957_b200 needs a CUDA (sm_100a) device; there is no CPU path")
        _cuda_seen = True
    return torch.device("cuda", torch.cuda.current_device())


def _is_tensor(v) -> bool:
    return isinstance(v, torch.Tensor)


class _PinnedPool:
    """Pinned host buffers for results, recycled when the numpy array handed out
    is garbage-collected.  A fresh pinned allocation costs ~100 us on this box
    (and can stall the device); a result D2H of a few MB costs less than that."""

    def __init__(self):
        self._free: dict[tuple, list[torch.Tensor]] = {}
        self._lock = threading.Lock()

    def take(self, shape: tuple, dtype: torch.dtype) -> torch.Tensor:
        key = (tuple(int(s) for s in shape), dtype)
        with self._lock:
            lst = self._free.get(key)
            if lst:
                return lst.pop()
        return torch.empty(key[0], dtype=dtype, pin_memory=True)

    def give(self, t: torch.Tensor) -> None:
        with self._lock:
            lst = self._free.setdefault((tuple(t.shape), t.dtype), [])
            if len(lst) < 8:
                lst.append(t)

    def lease(self, t: torch.Tensor) -> np.ndarray:
        """numpy view of ``t``; ``t`` returns to the pool when the view (and every
        view of it) is gone."""
        a = t.numpy()
        weakref.finalize(a, self.give, t)
        return a


_pinned = _PinnedPool()


class _EventPool:
    """Recycled CUDA events for streamed results (creating one costs a few us)."""

    def __init__(self):
        self._free: list[torch.cuda.Event] = []
        self._lock = threading.Lock()

    def take(self) -> torch.cuda.Event:
        with self._lock:
            if self._free:
                return self._free.pop()
        return torch.cuda.Event()

    def give(self, e: torch.cuda.Event) -> None:
        with self._lock:
            if len(self._free) < 16:
                self._free.append(e)


_events = _EventPool()


class _Deferred:
    """Pinned buffers of streamed results that were dropped before they arrived.

    The library reads the host X and writes the pinned Y and status words through raw
    pointers, so torch's caching host allocator records no stream use for them: freed on
    the spot, they could be handed to the next ``pin_memory()`` while the copies (or the
    epilogue's direct stores) are still in flight.  A result's finalizer parks them here
    with the event that marks the end of those transfers; every new streamed call drains
    the entries whose event has completed, returning Y and the status words to the pool."""

    def __init__(self):
        self._q: deque = deque()
        self._lock = threading.Lock()

    def park(self, box: list) -> None:
        if box:  # empty once the result arrived normally
            with self._lock:
                self._q.append(tuple(box))
            box.clear()

    def drain(self) -> None:
        done = []
        with self._lock:
            while self._q and self._q[0][1].query():
                done.append(self._q.popleft())
        for host, ev, flags, _keep in done:
            _pinned.give(host)
            _pinned.give(flags)
            _events.give(ev)


_deferred = _Deferred()


def _to_host(d: torch.Tensor, extra: torch.Tensor | None = None):
    """Device -> host through pinned memory (one stream-ordered async copy, one
    synchronisation); ``extra`` (a small status tensor) rides along and is
    returned too."""
    if not d.is_cuda:
        h = d.numpy()
        return (h, extra.cpu().numpy()) if extra is not None else h
    h = _pinned.take(d.shape, d.dtype)
    h.copy_(d, non_blocking=True)
    he = None
    if extra is not None:
        he = _pinned.take(extra.shape, extra.dtype)
        he.copy_(extra, non_blocking=True)
    torch.cuda.current_stream(d.device).synchronize()
    if extra is None:
        return _pinned.lease(h)
    f = he.numpy().copy()
    _pinned.give(he)
    return _pinned.lease(h), f


def _same_kind(other, cls) -> bool:
    """Equality accepts this package's object or the reference's class of the same name
    (dense.py:63-64 compares by class), so values round-trip between the two packages."""
    return isinstance(other, cls) or (type(other).__name__ == cls.__name__ and hasattr(other, "values"))


class _Dual:
    """Host/device pair with lazy, cached transfers."""

    __slots__ = ("_h", "_d")

    def __init__(self, host: np.ndarray | None, dev: torch.Tensor | None):
        self._h = host
        self._d = dev

    def host(self) -> np.ndarray:
        if self._h is None:
            self._h = _to_host(self._d.detach())
        return self._h

    def dev(self) -> torch.Tensor:
        if self._d is None:
            self._d = torch.from_numpy(np.ascontiguousarray(self._h)).to(_device(), non_blocking=False)
        elif not self._d.is_cuda:
            # host torch tensor: pinned memory uploads asynchronously on the current stream
            src = self._d
            self._d = src.to(_device(), non_blocking=src.is_pinned())
        return self._d

    def shape(self):
        return tuple(self._h.shape) if self._h is not None else tuple(self._d.shape)


class TernaryDense:
    """K x N weight matrix with entries in {-1, 0, +1} (dense.py:32-64).

    Host input is validated here (ParameterError naming the first bad entry);
    a CUDA tensor is validated by the device builder on first use."""

    def __init__(self, values):
        if _is_tensor(values):
            v = values.detach()
            if v.dtype != torch.int8:
                v = v.to(torch.int8)
            if v.dim() != 2 or v.shape[0] < 1 or v.shape[1] < 1:
                raise ParameterError(f"ternary matrix must be 2-D and non-empty, got shape {tuple(values.shape)}")
            self._v = _Dual(None, v.contiguous())
            return
        v = np.ascontiguousarray(values, dtype=np.int8)
        raw = np.asarray(values)
        if v.ndim != 2 or v.shape[0] < 1 or v.shape[1] < 1:
            raise ParameterError(f"ternary matrix must be 2-D and non-empty, got shape {raw.shape}")
        bad = (raw < -1) | (raw > 1) if raw.dtype.kind in "iuf" else (v < -1) | (v > 1)
        if bad.any():
            k, n = np.argwhere(bad)[0]
            raise ParameterError(f"entry ({k}, {n}) = {raw[k, n]} is not in {{-1, 0, +1}}")
        self._v = _Dual(v, None)

    @property
    def values(self) -> np.ndarray:
        return self._v.host()

    @property
    def device_values(self) -> torch.Tensor:
        return self._v.dev()

    @property
    def K(self) -> int:
        return self._v.shape()[0]

    @property
    def N(self) -> int:
        return self._v.shape()[1]

    @property
    def nnz(self) -> int:
        if self._v._h is not None:
            return int(np.count_nonzero(self._v._h))
        return int(torch.count_nonzero(self._v._d).item())

    def __eq__(self, other) -> bool:
        return _same_kind(other, TernaryDense) and np.array_equal(self.values, np.asarray(other.values))

    def __repr__(self) -> str:
        return f"TernaryDense(K={self.K}, N={self.N})"


PEER_TIMEOUT_BIT = 8  # bad_input bit 3: a fused shard assembly gave up waiting for a rank (peer.py)


def _flags_bad(f) -> bool:
    """Kernel status words (tg_device_flags as int32): a non-finite output, or a
    non-finite X entry seen by the tensor-core split (bad_input bit 2; the
    reference rejects such an X when it is constructed, dense.py:77).  A peer
    timeout (bit 3) is raised as its own error first."""
    if int(f[0]) & PEER_TIMEOUT_BIT:
        raise RuntimeError("fused shard assembly timed out: a rank never arrived, Y is incomplete")
    return int(f[1]) != 0 or (int(f[0]) & 4) != 0


class DenseMatrix:
    """Row-major float32 matrix with all entries finite (dense.py:67-90).

    ``flags`` (internal) is the kernel-written device status word of an output;
    its non-finite bit is turned into the reference's ParameterError the first
    time the host looks at the values (or on ``check()``)."""

    _arrival = None  # streamed result: (pinned host Y, pinned host flags, event of their copies)

    def __init__(self, values, _flags: torch.Tensor | None = None):
        self._flags = _flags
        self._checked = _flags is None
        if _is_tensor(values):
            v = values.detach()
            if v.dim() != 2:
                raise ParameterError(f"dense matrix must be 2-D, got shape {tuple(values.shape)}")
            if v.dtype != torch.float32:
                v = v.float()
            self._v = _Dual(None, v.contiguous())
            if _flags is None:
                self._checked = False  # lazily checked with torch.isfinite
            return
        v = np.ascontiguousarray(values, dtype=np.float32)
        if v.ndim != 2:
            raise ParameterError(f"dense matrix must be 2-D, got shape {np.asarray(values).shape}")
        if not np.isfinite(v).all():
            raise ParameterError("dense matrix contains non-finite values")
        self._v = _Dual(v, None)
        self._checked = True

    @classmethod
    def _streamed(cls, dev: torch.Tensor, host: torch.Tensor, host_flags: torch.Tensor,
                  done: torch.cuda.Event, keep: tuple = ()) -> "DenseMatrix":
        """A kernel output whose host copy (and status words) are already on their
        way through pinned memory; ``done`` marks their arrival.  ``keep`` holds host
        inputs the call reads in place (a pinned X) until then."""
        obj = cls.__new__(cls)  # (dev is the library's own contiguous fp32 [M, N] output)
        obj._flags = host_flags
        obj._checked = False
        obj._v = _Dual(None, dev)
        box = [host, done, host_flags, keep]
        obj._arrival = box
        weakref.finalize(obj, _deferred.park, box)  # dropped before arrival: park the buffers
        return obj

    def _arrive(self) -> None:
        box = self._arrival
        host, done = box[0], box[1]
        done.synchronize()
        box.clear()  # arrived: nothing for the finalizer to park
        _events.give(done)
        self._arrival = None
        f = self._flags
        self._flags = f.numpy().copy()  # (host words; the pinned buffer goes back to the pool)
        _pinned.give(f)
        if _flags_bad(self._flags):
            _pinned.give(host)
            raise ParameterError("dense matrix contains non-finite values")
        self._checked = True
        self._v._h = _pinned.lease(host)

    def _nonpositive(self) -> int:
        """#(y <= 0) before PReLU from the streamed status words (simd.py:410-417 mults)."""
        self.check()
        f = np.asarray(self._flags.numpy() if _is_tensor(self._flags) else self._flags).view(np.uint32)
        return int(f[2]) | (int(f[3]) << 32)

    def check(self) -> "DenseMatrix":
        if self._arrival is not None:
            self._arrive()
        if not self._checked:
            if self._flags is not None:
                f = self._flags
                bad = _flags_bad(f if isinstance(f, np.ndarray) else f.cpu().numpy())
            else:
                bad = not bool(torch.isfinite(self._v._d).all().item())
            if bad:
                raise ParameterError("dense matrix contains non-finite values")
            self._checked = True
        return self

    @property
    def values(self) -> np.ndarray:
        if self._arrival is not None:
            self._arrive()
        v = self._v
        if v._h is None and not self._checked and self._flags is not None and v._d is not None and v._d.is_cuda:
            # fetch Y and the kernel's status words with one synchronisation
            h, f = _to_host(v._d.detach(), self._flags)
            if _flags_bad(f):
                raise ParameterError("dense matrix contains non-finite values")
            self._checked = True
            v._h = h
            return h
        self.check()
        return v.host()

    @property
    def device_values(self) -> torch.Tensor:
        return self._v.dev()

    @property
    def rows(self) -> int:
        return self._v.shape()[0]

    @property
    def cols(self) -> int:
        return self._v.shape()[1]

    def __eq__(self, other) -> bool:
        return _same_kind(other, DenseMatrix) and np.array_equal(self.values, np.asarray(other.values))

    def __repr__(self) -> str:
        return f"DenseMatrix({self.rows}x{self.cols})"


class BiasVector:
    """Length-N float32 vector broadcast over the output rows (dense.py:93-111)."""

    def __init__(self, values):
        if _is_tensor(values):
            v = values.detach()
            if v.dim() != 1:
                raise ParameterError(f"bias must be 1-D, got shape {tuple(values.shape)}")
            if v.dtype != torch.float32:
                v = v.float()
            if not bool(torch.isfinite(v).all().item()):
                raise ParameterError("bias contains non-finite values")
            self._v = _Dual(None, v.contiguous())
            return
        v = np.ascontiguousarray(values, dtype=np.float32)
        if v.ndim != 1:
            raise ParameterError(f"bias must be 1-D, got shape {np.asarray(values).shape}")
        if not np.isfinite(v).all():
            raise ParameterError("bias contains non-finite values")
        self._v = _Dual(v, None)

    @property
    def values(self) -> np.ndarray:
        return self._v.host()

    @property
    def device_values(self) -> torch.Tensor:
        return self._v.dev()

    def __len__(self) -> int:
        return self._v.shape()[0]

    def __eq__(self, other) -> bool:
        return _same_kind(other, BiasVector) and np.array_equal(self.values, np.asarray(other.values))


def as_ternary(W) -> TernaryDense:
    if isinstance(W, TernaryDense):
        return W
    if hasattr(W, "values") and not _is_tensor(W) and not isinstance(W, np.ndarray):
        return TernaryDense(W.values)  # e.g. the reference's own TernaryDense
    return TernaryDense(W)


def as_dense(X) -> DenseMatrix:
    if isinstance(X, DenseMatrix):
        return X
    if hasattr(X, "values") and not _is_tensor(X) and not isinstance(X, np.ndarray):
        return DenseMatrix(X.values)  # e.g. the reference's own DenseMatrix
    return DenseMatrix(X)


def as_bias(b) -> BiasVector:
    if isinstance(b, BiasVector):
        return b
    if hasattr(b, "values") and not _is_tensor(b) and not isinstance(b, np.ndarray):
        return BiasVector(b.values)
    return BiasVector(b)


def prelu(v, alpha: float):
    """dense.py:184-189: v if v > 0 else alpha * v (host helper)."""
    if np.isscalar(v):
        return v if v > 0 else type(v)(alpha * v)
    arr = np.asarray(v)
    return np.where(arr > 0, arr, np.float32(alpha) * arr).astype(arr.dtype)


def oracle_gemm(X, W, b, alpha: float | None = None) -> DenseMatrix:
    """dense.py:192-213 semantics: fp64 X @ W + b, PReLU in fp64, one cast to fp32.

    Runs as an fp64 cuBLAS GEMM on the device (a verification utility for
    the harness, not the ternary hot path)."""
    X, W, b = as_dense(X), as_ternary(W), as_bias(b)
    if X.cols != W.K:
        raise ParameterError(f"X has {X.cols} columns but W has {W.K} rows")
    if len(b) != W.N:
        raise ParameterError(f"bias length {len(b)} != N = {W.N}")
    y = X.device_values.double() @ W.device_values.double() + b.device_values.double()
    if alpha is not None:
        y = torch.where(y > 0, y, float(alpha) * y)
    return DenseMatrix(y.float())


# ---------------------------------------------------------------- seeded generators (dense.py:24-181)
# Host-side input generators with the reference's exact recipes, so files and
# `verify` runs made with either package hold the same matrices for a seed.

DEFAULT_INT_RANGE = 8  # dense.py:21


def as_fraction(s) -> Fraction:
    """dense.py:24-29."""
    frac = Fraction(s)
    if not 0 < frac <= 1:
        raise ParameterError(f"sparsity must lie in (0, 1], got {s!r}")
    return frac


def gen_ternary(K: int, N: int, s, seed: int) -> TernaryDense:
    """dense.py:112-140: every column gets exactly round(s*K) nonzeros at
    rng.choice positions, the first ceil(nz/2) of them +1, the rest -1."""
    if K < 1 or N < 1:
        raise ParameterError(f"K and N must be >= 1, got K={K} N={N}")
    nz = round(as_fraction(s) * K)
    if nz > K:
        raise ParameterError(f"round(s*K) = {nz} exceeds K = {K}")
    n_pos = (nz + 1) // 2
    rng = np.random.default_rng(seed)
    w = np.zeros((K, N), dtype=np.int8)
    for n in range(N):
        chosen = rng.choice(K, size=nz, replace=False)
        w[chosen[:n_pos], n] = 1
        w[chosen[n_pos:], n] = -1
    return TernaryDense(w)


def gen_input(M: int, K: int, seed: int, int_range: int = DEFAULT_INT_RANGE) -> DenseMatrix:
    """dense.py:143-162: integers uniform in [-int_range, int_range] (exact fp32 sums)."""
    if M < 1 or K < 1:
        raise ParameterError(f"M and K must be >= 1, got M={M} K={K}")
    if int_range < 1:
        raise ParameterError(f"int_range must be >= 1, got {int_range}")
    if K * int_range >= EXACT_FLOAT32_BOUND:
        raise ParameterError(f"K * int_range = {K * int_range} >= 2**24 would break exact float32 accumulation")
    rng = np.random.default_rng(seed)
    return DenseMatrix(rng.integers(-int_range, int_range + 1, size=(M, K)).astype(np.float32))


def gen_input_uniform(M: int, K: int, seed: int) -> DenseMatrix:
    """dense.py:165-175: uniform [-1, 1) drawn in fp64, cast to fp32."""
    if M < 1 or K < 1:
        raise ParameterError(f"M and K must be >= 1, got M={M} K={K}")
    rng = np.random.default_rng(seed)
    return DenseMatrix((rng.random(size=(M, K), dtype=np.float64) * 2.0 - 1.0).astype(np.float32))


def gen_bias(N: int, seed: int, int_range: int = DEFAULT_INT_RANGE) -> BiasVector:
    """dense.py:178-181."""
    if N < 1:
        raise ParameterError(f"N must be >= 1, got N={N}")
    rng = np.random.default_rng(seed)
    return BiasVector(rng.integers(-int_range, int_range + 1, size=N).astype(np.float32))
