"""Fused shard assembly: the GEMM epilogue stores Y straight into every rank's HBM.

The north star assembles a column-sharded Y with one NCCL all-gather after
the shard GEMMs (partition.py ``gather_columns``; the reference itself has no
parallelism).  Here the assembly is folded into the
producing kernel instead: every rank keeps a full-width Y in peer-mapped
memory, and the tensor-core epilogue of each rank writes each finished
128-column tile into all of them over NVLink as soon as the tile is done
(tg_gemm_tiles_run_scatter), overlapping the transfer with the remaining
tiles' MMAs.  The last CTA of each rank's grid then bumps an arrival counter
in every rank's signal header, and a one-warp stream-ordered wait
(tg_peer_wait) releases the consumer once all ranks have arrived.

Buffer of one rank (one cudaMalloc, exported with cudaIpc):

    [ signal header, 256 B ][ Y slot 0: M x N fp32 ][ Y slot 1 ] ...

Header words (uint32): [0, world) arrivals per source rank;
TG_PEER_DONE_WORD: CTA completion counter of this rank's running GEMM;
TG_PEER_EPOCH_WORD: epochs consumed by tg_peer_wait; TG_PEER_TIMEOUT_WORD.

Flow control with two slots: step s writes slot s % 2.  A rank's GEMM of step
s+2 runs (stream order) after its wait of step s+1, which needs every peer's
GEMM of step s+1 to have completed, which in turn ran after that peer's
stream-ordered consumers of slot s % 2.  So no rank overwrites a slot a peer
may still read -- provided every rank consumes step s on the stream before
launching step s+1 (ScatterGemm does exactly that).

``PeerYBuffers.loopback`` builds ``world`` buffers on ONE device in one
process: the same kernels and tables with every "peer" local, which is how
the scatter is verified on a single GPU (tests/test_gpu_peer.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _native as nat
from .dense import PEER_TIMEOUT_BIT, DenseMatrix
from .errors import ParameterError
from .partition import Shard, column_shards

_ALIGN = 256


@dataclass(frozen=True)
class PeerLayout:
    """Byte layout of one rank's peer buffer."""

    M: int
    N: int
    slots: int

    @property
    def slot_bytes(self) -> int:
        return -(-self.M * self.N * 4 // _ALIGN) * _ALIGN

    def slot_offset(self, slot: int) -> int:
        if not 0 <= slot < self.slots:
            raise ParameterError(f"slot {slot} outside [0, {self.slots})")
        return nat.TG_PEER_HEADER_BYTES + slot * self.slot_bytes

    @property
    def total_bytes(self) -> int:
        return nat.TG_PEER_HEADER_BYTES + self.slots * self.slot_bytes


class _DevView:
    """__cuda_array_interface__ over a raw device pointer (no copy, no ownership)."""

    def __init__(self, ptr: int, shape: tuple, typestr: str, strides=None):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": strides}


def _view(ptr: int, shape: tuple, dtype: torch.dtype, device: torch.device) -> torch.Tensor:
    typestr = {torch.float32: "<f4", torch.int32: "<i4"}[dtype]
    with torch.cuda.device(device):
        return torch.as_tensor(_DevView(ptr, shape, typestr), device=device)


def _alloc(nbytes: int) -> int:
    p = ctypes.c_void_p()
    nat.call("tg_peer_alloc", nbytes, ctypes.byref(p))
    return int(p.value)


class PeerYBuffers:
    """Full-width Y slots on every rank, mapped into every other rank.

    ``block(slot)`` is this rank's shard of slot ``slot`` (a strided view of its
    full Y, row pitch N); ``y(slot)`` the full Y; ``descriptor(slot)`` the
    tg_peer_scatter the GEMM takes; ``wait()`` the stream-ordered arrival wait."""

    def __init__(self, M: int, N: int, group=None, slots: int = 2, symmetric: bool = False,
                 device: torch.device | None = None, *, _loopback: tuple | None = None):
        if M < 1 or N < 1:
            raise ParameterError(f"M and N must be >= 1, got {M}, {N}")
        if slots < 1:
            raise ParameterError(f"slots must be >= 1, got {slots}")
        self.M, self.N = M, N
        self._group = group
        self._is_loopback = _loopback is not None
        self.layout = PeerLayout(M, N, slots)
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        if _loopback is not None:
            self.rank, self.world, bases, self._owned, self._imported = _loopback
        else:
            if group is None and not dist.is_initialized():
                self.rank, self.world = 0, 1
            else:
                self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
            if self.world > nat.TG_PEER_MAX_WORLD:
                raise ParameterError(f"world {self.world} > TG_PEER_MAX_WORLD = {nat.TG_PEER_MAX_WORLD}")
            with torch.cuda.device(self.device):
                own = _alloc(self.layout.total_bytes)
                self._owned = [own]
                self._imported = []
                bases = [own] * self.world
                if self.world > 1:
                    h = ctypes.create_string_buffer(nat.TG_PEER_HANDLE_BYTES)
                    nat.call("tg_peer_export", ctypes.c_void_p(own), h)
                    handles: list = [None] * self.world
                    dist.all_gather_object(handles, bytes(h.raw), group=group)
                    for r, hr in enumerate(handles):
                        if r == self.rank:
                            continue
                        p = ctypes.c_void_p()
                        nat.call("tg_peer_import", ctypes.create_string_buffer(hr, nat.TG_PEER_HANDLE_BYTES),
                                 ctypes.byref(p))
                        bases[r] = int(p.value)
                        self._imported.append(bases[r])
        self.bases = list(bases)
        self.shards: list[Shard] = column_shards(N, self.world, symmetric)
        self.shard = self.shards[self.rank]
        dev = self.device
        self._sig_table = torch.tensor(self.bases, dtype=torch.int64, device=dev)
        self._y_tables = [torch.tensor([b + self.layout.slot_offset(s) for b in self.bases], dtype=torch.int64,
                                       device=dev) for s in range(slots)]
        self._desc = []
        for s in range(slots):
            d = nat.TgPeerScatter()
            d.y_peers = self._y_tables[s].data_ptr()
            d.sig_peers = self._sig_table.data_ptr()
            d.sig_local = self.bases[self.rank]
            d.world, d.rank, d.col_off = self.world, self.rank, self.shard.start
            self._desc.append(d)
        self.header = _view(self.bases[self.rank], (nat.TG_PEER_HEADER_BYTES // 4,), torch.int32, dev)
        self._y = [_view(self.bases[self.rank] + self.layout.slot_offset(s), (M, N), torch.float32, dev)
                   for s in range(slots)]

    @classmethod
    def loopback(cls, M: int, N: int, world: int, slots: int = 2, symmetric: bool = False,
                 device: torch.device | None = None) -> list["PeerYBuffers"]:
        """``world`` rank views whose buffers all live on one device of this process."""
        if not 1 <= world <= nat.TG_PEER_MAX_WORLD:
            raise ParameterError(f"world must be in [1, {nat.TG_PEER_MAX_WORLD}], got {world}")
        device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        layout = PeerLayout(M, N, slots)
        with torch.cuda.device(device):
            bases = [_alloc(layout.total_bytes) for _ in range(world)]
        views = [cls(M, N, slots=slots, symmetric=symmetric, device=device,
                     _loopback=(r, world, bases, [], [])) for r in range(world)]
        views[0]._owned = bases  # rank 0's view frees them all
        return views

    @property
    def slots(self) -> int:
        return self.layout.slots

    def y(self, slot: int) -> torch.Tensor:
        return self._y[slot]

    def block(self, slot: int) -> torch.Tensor:
        return self._y[slot][:, self.shard.slice()]

    def descriptor(self, slot: int) -> nat.TgPeerScatter:
        return self._desc[slot]

    def wait(self, stream: int | None = None) -> None:
        st = torch.cuda.current_stream(self.device).cuda_stream if stream is None else stream
        nat.call("tg_peer_wait", ctypes.c_void_p(self.bases[self.rank]), self.world, ctypes.c_void_p(st))

    def timed_out(self) -> bool:
        """True if a wait gave up (a rank never arrived); synchronises."""
        return int(self.header[nat.TG_PEER_TIMEOUT_WORD].item()) != 0

    def close(self) -> None:
        """Unmap the peers' buffers, then (once every rank has unmapped ours) free our own."""
        torch.cuda.synchronize(self.device)
        for p in self._imported:
            nat.call("tg_peer_release", ctypes.c_void_p(p))
        self._imported = []
        if not self._is_loopback and self.world > 1 and dist.is_initialized():
            dist.barrier(group=self._group)
        for p in self._owned:
            nat.call("tg_peer_free", ctypes.c_void_p(p))
        self._owned = []


class ScatterGemm:
    """One rank's share of a column-sharded GEMM whose kernel assembles Y.

    ``runners[s]`` is the tensor-core GemmRunner writing slot s; ``step()``
    launches the shard GEMM of the next slot and the arrival wait, and returns
    the full Y of that slot (valid for kernels queued after it on the stream
    until the step after next)."""

    def __init__(self, make_runner, bufs: PeerYBuffers):
        self.bufs = bufs
        self.runners = [make_runner(out=bufs.block(s), scatter=bufs.descriptor(s)) for s in range(bufs.slots)]
        for r in self.runners:
            if r.method != "mma":
                raise ParameterError("the fused scatter runs in the tensor-core epilogue: method must be 'mma'")
        self.n = 0

    @property
    def slot(self) -> int:
        return self.n % self.bufs.slots

    def step(self, stream: int | None = None) -> torch.Tensor:
        s = self.slot
        self.runners[s].launch(stream)
        self.bufs.wait(stream)
        self.n += 1
        return self.bufs.y(s)

    def result(self) -> DenseMatrix:
        """One step on the current stream, returned as a DenseMatrix whose status words carry
        the runner's (non-finite output) and the wait's timeout word: reading ``.values`` or
        ``check()`` raises if the wait gave up, instead of handing out a partly assembled Y."""
        s = self.slot
        y = self.step()
        flags = self.runners[s].flags.clone()
        timeout = self.bufs.header[nat.TG_PEER_TIMEOUT_WORD]
        flags[0] = flags[0] | (timeout != 0).to(torch.int32) * PEER_TIMEOUT_BIT
        return DenseMatrix(y, _flags=flags)
