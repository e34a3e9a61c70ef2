"""Sparse ternary formats, resident in HBM (reference: tcsc.py, variants.py).

The three in-scope formats keep the reference's exact array layouts (int32,
same offsets, same index order) so they can be compared bit for bit with the
reference builders and fed to either GPU path:

  Tcsc                    tcsc.py:35-68    built by tcsc_from_dense (tcsc.py:71-92)
  BlockedTcsc             variants.py:86-143   blocked_from_dense (variants.py:146-178)
  InterleavedBlockedTcsc  variants.py:251-309  interleaved_blocked_from_dense (variants.py:312-376)
  SymmetricInterleavedTcsc variants.py:540-580 symmetric_from_dense (variants.py:582-631)
  CompressedTcsc          variants.py:488-512  compressed_from_dense (variants.py:515-521), with the
                          5-trits-per-byte codec compress5 / decompress5 / DECODE_TABLE (variants.py:451-485)

Construction runs the two-phase device builder (csrc/tg_build.cu) through the
C ABI.  Index arrays live on the device; the reference attribute names
(``col_start_pos``, ``all_indices`` ...) return lazily cached host numpy
copies so reference-style callers keep working, ``.device(name)`` returns the
CUDA tensor.  ``tiles()`` derives (once, from the device arrays) the 2-bit
ternary-tile re-encoding consumed by the dense-decode tensor-core path.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native as nat
from .dense import TernaryDense, _device, _Dual, as_ternary
from .errors import CorruptionError, InvalidCodeError, ParameterError

INDEX_DTYPE = np.int32
DEFAULT_BLOCK_SIZE = 4096
DEFAULT_GROUP_SIMD = 2


def resolve_block_size(B: int | None, K: int) -> int:
    """variants.py:38-42."""
    b = min(K, DEFAULT_BLOCK_SIZE) if B is None else B
    if b < 1:
        raise ParameterError(f"block size must be >= 1, got {b}")
    return int(b)


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _p(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _index_array(a, name: str) -> _Dual:
    if isinstance(a, torch.Tensor):
        t = a.detach()
        if t.dim() != 1:
            raise ParameterError(f"{name} must be 1-D")
        return _Dual(None, t.to(torch.int32).contiguous())
    arr = np.ascontiguousarray(a, dtype=INDEX_DTYPE)
    if arr.ndim != 1:
        raise ParameterError(f"{name} must be 1-D")
    return _Dual(arr, None)


def _table(a, name: str, shape) -> _Dual:
    if isinstance(a, torch.Tensor):
        t = a.detach().to(torch.int32).contiguous()
        if tuple(t.shape) != tuple(shape):
            raise ParameterError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
        return _Dual(None, t)
    arr = np.ascontiguousarray(a, dtype=INDEX_DTYPE)
    if arr.shape != tuple(shape):
        raise ParameterError(f"{name} must have shape {tuple(shape)}, got {arr.shape}")
    return _Dual(arr, None)


class _Format:
    """Common machinery: host/device array pairs, lazy tiles."""

    _arrays: tuple[str, ...] = ()

    def __getattr__(self, name):
        arrs = object.__getattribute__(self, "_a")
        if name in arrs:
            return arrs[name].host()
        raise AttributeError(name)

    def device(self, name: str) -> torch.Tensor:
        return self._a[name].dev()

    def _len(self, name: str) -> int:
        lens = self.__dict__.setdefault("_lens", {})  # the arrays never change size
        n = lens.get(name)
        if n is None:
            n = lens[name] = int(np.prod(self._a[name].shape()))
        return n

    def format_bytes(self) -> int:
        return 4 * sum(self._len(n) for n in self._arrays)

    def tiles(self) -> torch.Tensor:
        """2-bit ternary tiles (csrc/tg_mma.cu) derived from this format's device arrays."""
        t = self.__dict__.get("_tiles")
        if t is None:
            L = nat.load()
            nbytes = L.tg_tiles_bytes(self.K, self.N)
            t = torch.empty(nbytes // 4, dtype=torch.int32, device=_device())
            flags = torch.zeros(6, dtype=torch.int32, device=t.device)
            self._pack_tiles(t, flags)
            f = flags.cpu().numpy()
            if f[0] & 2:
                raise CorruptionError(f"{type(self).__name__} contains a row index outside [0, {self.K})")
            if f[4] & 2:
                raise CorruptionError(f"{type(self).__name__}: a cell appears in both sign arrays")
            if f[4] & 1:
                raise CorruptionError(f"{type(self).__name__}: duplicate row index within a column")
            self.__dict__["_tiles"] = t
        return t

    def to_dense(self) -> TernaryDense:
        """Decode on the device (tcsc.py:95-114); duplicates / overlaps raise CorruptionError."""
        t = self.tiles()
        w = torch.empty((self.K, self.N), dtype=torch.int8, device=t.device)
        nat.call("tg_tiles_to_dense", _p(t), self.K, self.N, _p(w), _stream())
        return TernaryDense(w)


class Tcsc(_Format):
    """TCSC of a K x N ternary matrix: two (N+1) offset arrays + two row-index arrays (tcsc.py:35-68)."""

    _arrays = ("col_start_pos", "col_start_neg", "row_index_pos", "row_index_neg")

    def __init__(self, K: int, N: int, col_start_pos, row_index_pos, col_start_neg, row_index_neg):
        if K < 1 or N < 1:
            raise ParameterError(f"K and N must be >= 1, got K={K} N={N}")
        self.__dict__["K"], self.__dict__["N"] = int(K), int(N)
        a = {
            "col_start_pos": _index_array(col_start_pos, "col_start_pos"),
            "row_index_pos": _index_array(row_index_pos, "row_index_pos"),
            "col_start_neg": _index_array(col_start_neg, "col_start_neg"),
            "row_index_neg": _index_array(row_index_neg, "row_index_neg"),
        }
        self.__dict__["_a"] = a
        for name in ("col_start_pos", "col_start_neg"):
            if a[name].shape()[0] != N + 1:
                raise ParameterError(f"{name} must have length N+1 = {N + 1}")

    @property
    def nnz(self) -> int:
        return self._len("row_index_pos") + self._len("row_index_neg")

    def _pack_tiles(self, t, flags):
        nat.call("tg_tiles_from_tcsc", _p(self.device("col_start_pos")), _p(self.device("row_index_pos")),
                 _p(self.device("col_start_neg")), _p(self.device("row_index_neg")), self.K, self.N, _p(t),
                 _p(flags), _stream())


class BlockedTcsc(_Format):
    """TCSC split into row blocks of height B; (nb, N+1) offset tables, global rows (variants.py:86-143)."""

    _arrays = ("col_start_pos", "col_start_neg", "row_index_pos", "row_index_neg")

    def __init__(self, K: int, N: int, B: int, col_start_pos, row_index_pos, col_start_neg, row_index_neg):
        if B < 1:
            raise ParameterError(f"block size must be >= 1, got {B}")
        self.__dict__.update(K=int(K), N=int(N), B=int(B))
        shape = (self.num_blocks, N + 1)
        self.__dict__["_a"] = {
            "col_start_pos": _table(col_start_pos, "col_start_pos", shape),
            "row_index_pos": _index_array(row_index_pos, "row_index_pos"),
            "col_start_neg": _table(col_start_neg, "col_start_neg", shape),
            "row_index_neg": _index_array(row_index_neg, "row_index_neg"),
        }

    @property
    def num_blocks(self) -> int:
        return -(-self.K // self.B)

    @property
    def nnz(self) -> int:
        return self._len("row_index_pos") + self._len("row_index_neg")

    def _pack_tiles(self, t, flags):
        nat.call("tg_tiles_from_blocked", _p(self.device("col_start_pos")), _p(self.device("row_index_pos")),
                 _p(self.device("col_start_neg")), _p(self.device("row_index_neg")), self.K, self.N, self.B, _p(t),
                 _p(flags), _stream())


class InterleavedBlockedTcsc(_Format):
    """One index stream; col_segment_ptr has 3*nb*N+1 entries, cell = blk*N + n (variants.py:251-309)."""

    _arrays = ("all_indices", "col_segment_ptr")

    def __init__(self, K: int, N: int, B: int, g: int, all_indices, col_segment_ptr, symmetric_groups: bool = False):
        if B < 1 or g < 1:
            raise ParameterError(f"need B >= 1 and g >= 1, got B={B} g={g}")
        if symmetric_groups and N % 4 != 0:
            raise ParameterError(f"symmetric groups need N divisible by 4, got N={N}")
        self.__dict__.update(K=int(K), N=int(N), B=int(B), g=int(g), symmetric_groups=bool(symmetric_groups))
        ptr = _index_array(col_segment_ptr, "col_segment_ptr")
        expected = 3 * self.num_blocks * N + 1
        if ptr.shape()[0] != expected:
            raise ParameterError(f"col_segment_ptr must have length {expected}")
        self.__dict__["_a"] = {"all_indices": _index_array(all_indices, "all_indices"), "col_segment_ptr": ptr}

    @property
    def num_blocks(self) -> int:
        return -(-self.K // self.B)

    @property
    def nnz(self) -> int:
        if not self.symmetric_groups:
            return self._len("all_indices")
        return int((self.device("all_indices") != self.K).sum().item())

    def _pack_tiles(self, t, flags):
        nat.call("tg_tiles_from_interleaved_blocked", _p(self.device("all_indices")),
                 _p(self.device("col_segment_ptr")), self.K, self.N, self.B, self.g, _p(t), _p(flags), _stream())


class SymmetricInterleavedTcsc(_Format):
    """One interleaved stream per column, equal lengths inside 4-column groups
    (variants.py:540-580); column n occupies indices[col_ptr[n]:col_ptr[n+1]]."""

    _arrays = ("indices", "col_ptr")

    def __init__(self, K: int, N: int, g: int, indices, col_ptr):
        if N % 4 != 0:
            raise ParameterError(f"N must be divisible by 4, got {N}")
        if g < 1:
            raise ParameterError(f"group size must be >= 1, got {g}")
        self.__dict__.update(K=int(K), N=int(N), g=int(g))
        ptr = _index_array(col_ptr, "col_ptr")
        if ptr.shape()[0] != N + 1:
            raise ParameterError(f"col_ptr must have length N+1 = {N + 1}")
        self.__dict__["_a"] = {"indices": _index_array(indices, "indices"), "col_ptr": ptr}

    def pairs_in_group(self, group: int) -> int:
        n = 4 * group
        p = self.col_ptr
        return (int(p[n + 1]) - int(p[n])) // 2

    @property
    def dummy_count(self) -> int:
        return int((self.device("indices") == self.K).sum().item())

    @property
    def nnz(self) -> int:
        return self._len("indices") - self.dummy_count

    def _pack_tiles(self, t, flags):
        nat.call("tg_tiles_from_symmetric", _p(self.device("indices")), _p(self.device("col_ptr")), self.K, self.N,
                 self.g, _p(t), _p(flags), _stream())


PACK_WIDTH = 5
CODE_COUNT = 3**PACK_WIDTH
_POW3 = np.array([3**i for i in range(PACK_WIDTH)], dtype=np.int64)


def compress5(values) -> int:
    """variants.py:451-462: code = sum((v_i + 1) 3^i), little-endian digits."""
    vals = np.asarray(values, dtype=np.int64)
    if vals.shape != (PACK_WIDTH,):
        raise ParameterError(f"compress5 needs exactly {PACK_WIDTH} values, got shape {vals.shape}")
    if ((vals < -1) | (vals > 1)).any():
        raise ParameterError(f"values must be in {{-1, 0, +1}}, got {values!r}")
    return int(((vals + 1) * _POW3).sum())


def decompress5(code: int) -> tuple[int, ...]:
    """variants.py:465-469."""
    if not 0 <= code < CODE_COUNT:
        raise InvalidCodeError(f"code must be in [0, {CODE_COUNT}), got {code}")
    return tuple(int(code // 3**i % 3) - 1 for i in range(PACK_WIDTH))


def _decode_table() -> np.ndarray:
    codes = np.arange(CODE_COUNT, dtype=np.int64)
    table = ((codes[:, None] // _POW3[None, :]) % 3 - 1).astype(np.int8)
    table.flags.writeable = False
    return table


DECODE_TABLE = _decode_table()  # variants.py:472-481: DECODE_TABLE[code, i] = i-th ternary digit


class CompressedTcsc:
    """Column-major packed bytes, ceil(K/5) codes per column (variants.py:488-512);
    codes >= 243 raise InvalidCodeError like the reference constructor."""

    def __init__(self, K: int, N: int, codes):
        self.K, self.N = int(K), int(N)
        shape = (self.N, -(-self.K // PACK_WIDTH))
        if isinstance(codes, torch.Tensor):
            c = codes.detach().to(torch.uint8).contiguous()
            if tuple(c.shape) != shape:
                raise ParameterError(f"codes must have shape {shape}, got {tuple(c.shape)}")
            if c.is_cuda:
                flags = torch.zeros(6, dtype=torch.int32, device=c.device)
                nat.call("tg_codes_check", _p(c), c.numel(), _p(flags), _stream())
                if int(flags[4].item()) & 4:
                    bad = int(c[c >= CODE_COUNT][0].item())
                    raise InvalidCodeError(f"code {bad} is outside [0, {CODE_COUNT})")
            elif bool((c >= CODE_COUNT).any()):
                raise InvalidCodeError(f"code {int(c[c >= CODE_COUNT][0])} is outside [0, {CODE_COUNT})")
            self._c = _Dual(None, c)
        else:
            arr = np.ascontiguousarray(codes, dtype=np.uint8)
            if arr.shape != shape:
                raise ParameterError(f"codes must have shape {shape}, got {arr.shape}")
            if (arr >= CODE_COUNT).any():
                raise InvalidCodeError(f"code {int(arr[arr >= CODE_COUNT][0])} is outside [0, {CODE_COUNT})")
            self._c = _Dual(arr, None)

    @property
    def codes(self) -> np.ndarray:
        return self._c.host()

    def device(self, name: str = "codes") -> torch.Tensor:
        if name != "codes":
            raise AttributeError(name)
        return self._c.dev()

    @property
    def groups_per_col(self) -> int:
        return -(-self.K // PACK_WIDTH)

    def format_bytes(self) -> int:
        """variants.py:495-498: one byte per code (the decode table is program data)."""
        return self.N * self.groups_per_col

    @property
    def nnz(self) -> int:
        return int(np.count_nonzero(DECODE_TABLE[self.codes].reshape(self.N, -1)[:, : self.K]))

    def tiles(self) -> torch.Tensor:
        t = self.__dict__.get("_tiles")
        if t is None:
            nbytes = nat.load().tg_tiles_bytes(self.K, self.N)
            t = torch.empty(nbytes // 4, dtype=torch.int32, device=_device())
            nat.call("tg_tiles_from_compressed", _p(self.device()), self.K, self.N, _p(t), _stream())
            self.__dict__["_tiles"] = t
        return t

    def to_dense(self) -> TernaryDense:
        """variants.py:500-503, decoded on the device."""
        t = self.tiles()
        w = torch.empty((self.K, self.N), dtype=torch.int8, device=t.device)
        nat.call("tg_tiles_to_dense", _p(t), self.K, self.N, _p(w), _stream())
        return TernaryDense(w)


# ---------------------------------------------------------------- builders


def _build(W: TernaryDense, kind: int, B: int, g: int, sym: bool):
    L = nat.load()
    dW = W.device_values
    K, N = int(dW.shape[0]), int(dW.shape[1])
    dev = dW.device
    ws = torch.empty(L.tg_build_workspace_bytes(K, N, B), dtype=torch.uint8, device=dev)
    sizes = nat.TgSizes()
    nat.call("tg_build_count", _p(dW), K, N, N, kind, B, g, int(sym), _p(ws), ws.numel(), ctypes.byref(sizes),
             _stream())
    return ws, sizes, K, N, dev


def tcsc_from_dense(W) -> Tcsc:
    """tcsc.py:71-92, on the device (count -> scan -> fill)."""
    W = as_ternary(W)
    ws, s, K, N, dev = _build(W, nat.TG_FMT_TCSC, W.K, 1, False)
    csp = torch.empty(N + 1, dtype=torch.int32, device=dev)
    csn = torch.empty(N + 1, dtype=torch.int32, device=dev)
    rip = torch.empty(s.nnz_pos, dtype=torch.int32, device=dev)
    rin = torch.empty(s.nnz_neg, dtype=torch.int32, device=dev)
    nat.call("tg_build_fill_tcsc", _p(ws), K, N, _p(csp), _p(rip), _p(csn), _p(rin), _stream())
    return Tcsc(K, N, csp, rip, csn, rin)


def blocked_from_dense(W, B: int | None = None) -> BlockedTcsc:
    """variants.py:146-178, on the device.  B defaults to min(K, 4096)."""
    W = as_ternary(W)
    b = resolve_block_size(B, W.K)
    ws, s, K, N, dev = _build(W, nat.TG_FMT_BLOCKED, b, 1, False)
    nb = s.num_blocks
    csp = torch.empty((nb, N + 1), dtype=torch.int32, device=dev)
    csn = torch.empty((nb, N + 1), dtype=torch.int32, device=dev)
    rip = torch.empty(s.nnz_pos, dtype=torch.int32, device=dev)
    rin = torch.empty(s.nnz_neg, dtype=torch.int32, device=dev)
    nat.call("tg_build_fill_blocked", _p(ws), K, N, b, _p(csp), _p(rip), _p(csn), _p(rin), _stream())
    return BlockedTcsc(K, N, b, csp, rip, csn, rin)


def interleaved_blocked_from_dense(W, B: int | None = None, g: int = DEFAULT_GROUP_SIMD,
                                   symmetric_cols: bool = False) -> InterleavedBlockedTcsc:
    """variants.py:312-350 (+ _pad_groups, variants.py:361-376), on the device."""
    W = as_ternary(W)
    if symmetric_cols and W.N % 4 != 0:
        raise ParameterError(f"symmetric groups need N divisible by 4, got N={W.N}")
    if g < 1:
        raise ParameterError(f"group size must be >= 1, got {g}")
    b = resolve_block_size(B, W.K)
    ws, s, K, N, dev = _build(W, nat.TG_FMT_INTERLEAVED_BLOCKED, b, g, symmetric_cols)
    ai = torch.empty(s.n_indices, dtype=torch.int32, device=dev)
    ptr = torch.empty(s.offsets_len, dtype=torch.int32, device=dev)
    nat.call("tg_build_fill_interleaved_blocked", _p(ws), K, N, b, g, int(symmetric_cols), _p(ai), _p(ptr),
             _stream())
    return InterleavedBlockedTcsc(K, N, b, g, ai, ptr, symmetric_cols)


def symmetric_from_dense(W, g: int = DEFAULT_GROUP_SIMD) -> SymmetricInterleavedTcsc:
    """variants.py:582-631, on the device (count -> scan -> fill, dummies = K)."""
    W = as_ternary(W)
    if W.N % 4 != 0:
        raise ParameterError(f"N must be divisible by 4, got {W.N}")
    if g < 1:
        raise ParameterError(f"group size must be >= 1, got {g}")
    ws, s, K, N, dev = _build(W, nat.TG_FMT_SYMMETRIC, W.K, g, False)
    idx = torch.empty(s.n_indices, dtype=torch.int32, device=dev)
    ptr = torch.empty(N + 1, dtype=torch.int32, device=dev)
    nat.call("tg_build_fill_symmetric", _p(ws), K, N, g, _p(idx), _p(ptr), s.n_indices, _stream())
    return SymmetricInterleavedTcsc(K, N, g, idx, ptr)


def compressed_from_dense(W) -> CompressedTcsc:
    """variants.py:515-521, on the device (validates W like dense.py:45-49)."""
    W = as_ternary(W)
    dW = W.device_values
    K, N = int(dW.shape[0]), int(dW.shape[1])
    codes = torch.empty((N, -(-K // PACK_WIDTH)), dtype=torch.uint8, device=dW.device)
    nat.call("tg_build_compressed", _p(dW), K, N, N, _p(codes), _stream())
    obj = CompressedTcsc.__new__(CompressedTcsc)
    obj.K, obj.N, obj._c = K, N, _Dual(None, codes)
    return obj


# ---------------------------------------------------------------- utilities


def tcsc_to_dense(t: Tcsc) -> TernaryDense:
    return t.to_dense()


def format_bytes(fmt) -> int:
    """tcsc.py:162-179."""
    method = getattr(fmt, "format_bytes", None)
    if method is None:
        raise ParameterError(f"object of type {type(fmt).__name__} is not a sparse format")
    return method()


def tcsc_bytes_for(K: int, N: int, nnz: int) -> int:
    """tcsc.py:186-190."""
    if K < 1 or N < 1 or nnz < 0 or nnz > K * N:
        raise ParameterError(f"inconsistent dimensions K={K} N={N} nnz={nnz}")
    return 4 * (2 * (N + 1) + nnz)


def validate(t: Tcsc) -> list[str]:
    """Semantic audit with the reference's messages and order (tcsc.py:123-159), computed on the device."""
    problems: list[str] = []
    for name in ("pos", "neg"):
        starts = t.device(f"col_start_{name}").long()
        rows = t.device(f"row_index_{name}").long()
        nrows = rows.numel()
        s0, s_last = int(starts[0].item()), int(starts[-1].item())
        if s0 != 0:
            problems.append(f"col_start_{name}[0] = {s0}, expected 0")
        if s_last != nrows:
            problems.append(f"col_start_{name}[-1] = {s_last}, expected row_index_{name} length {nrows}")
        if bool((starts[1:] < starts[:-1]).any().item()):
            problems.append(f"col_start_{name} is not non-decreasing")
            continue
        lo, hi = max(0, s0), min(nrows, s_last)
        a, b = starts[:-1], starts[1:]
        valid = (a >= lo) & (b <= hi)
        if nrows:
            col_of = torch.repeat_interleave(torch.arange(t.N, device=rows.device),
                                             (b - a).clamp(min=0), output_size=None) if s0 == 0 and s_last == nrows \
                else None
            bad_inc = torch.zeros(t.N, dtype=torch.bool, device=rows.device)
            bad_rng = torch.zeros(t.N, dtype=torch.bool, device=rows.device)
            if col_of is not None:
                same = col_of[1:] == col_of[:-1]
                dec = same & (rows[1:] <= rows[:-1])
                bad_inc.index_fill_(0, col_of[1:][dec], True)
                oor = (rows < 0) | (rows >= t.K)
                bad_rng.index_fill_(0, col_of[oor], True)
            else:
                for n in torch.nonzero(valid).flatten().tolist():
                    col = rows[int(a[n]):int(b[n])]
                    if col.numel() > 1 and bool((col[1:] <= col[:-1]).any()):
                        bad_inc[n] = True
                    if col.numel() and bool(((col < 0) | (col >= t.K)).any()):
                        bad_rng[n] = True
            bad_inc &= valid
            bad_rng &= valid
            for n in torch.nonzero(bad_inc | bad_rng).flatten().tolist():
                if bool(bad_inc[n]):
                    problems.append(f"row_index_{name} not strictly increasing in column {n}")
                if bool(bad_rng[n]):
                    problems.append(f"row_index_{name} out of range [0, {t.K}) in column {n}")
    if not problems:
        keys = []
        for name in ("pos", "neg"):
            starts = t.device(f"col_start_{name}").long()
            rows = t.device(f"row_index_{name}").long()
            cols = torch.repeat_interleave(torch.arange(t.N, device=rows.device), starts[1:] - starts[:-1])
            keys.append(rows * t.N + cols)
        both = keys[0][torch.isin(keys[0], keys[1])]
        if both.numel():
            first = int(both.min().item())
            problems.append(f"cell ({first // t.N}, {first % t.N}) appears in both sign arrays")
    return problems
