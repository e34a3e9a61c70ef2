"""Partitioner: shard one Y = X W + b over the ranks of a process group.

The reference has no parallelism; the north star adds
exactly one: split the work by N column blocks (W and b sharded, X
replicated) or by M row blocks (X sharded, W replicated), compute every shard
on its own GPU with no data-path communication, and assemble Y with a single
NCCL all-gather over NVLink.

  * Output columns are independent (scalar.py:116-127: Y[:, n] reads only
    column n of W), so a column shard's Y equals the same columns of the full
    product bit for bit, provided symmetric 4-column groups are not split
    (variants.py:361-376 pads within a group) -- shard widths are multiples
    of ``align`` (4 for symmetric formats).
  * Row shards are trivially independent; the tensor-core path scales each
    X row on its own, so rows computed alone equal rows computed together.

Per-shard formats are built from ``W[:, cols]`` on each rank (their arrays
are not slices of the global arrays: the cell order is blk*N + n,
variants.py:344).

This module is device-agnostic plumbing over ``torch.distributed`` so that
the assembly is exercised by world_size-2 gloo tests on CPU; the compute
callback is the CUDA path in bench.py / the public API.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch
import torch.distributed as dist

from .errors import ParameterError


@dataclass(frozen=True)
class Shard:
    rank: int
    start: int
    stop: int

    @property
    def width(self) -> int:
        return self.stop - self.start

    def slice(self) -> slice:
        return slice(self.start, self.stop)


def split(extent: int, world: int, align: int = 1) -> list[Shard]:
    """Contiguous shards of [0, extent) whose widths are multiples of ``align``
    (except a non-aligned tail, which goes to the last rank) and differ by at
    most ``align``.  Ranks may receive an empty shard when extent < world*align."""
    if world < 1:
        raise ParameterError(f"world size must be >= 1, got {world}")
    if align < 1:
        raise ParameterError(f"align must be >= 1, got {align}")
    if extent < 0:
        raise ParameterError(f"extent must be >= 0, got {extent}")
    units, tail = divmod(extent, align)
    base, extra = divmod(units, world)
    out, pos = [], 0
    for r in range(world):
        w = (base + (r < extra)) * align
        if r == world - 1:
            w += tail
        out.append(Shard(r, pos, pos + w))
        pos += w
    assert pos == extent
    return out


def column_shards(N: int, world: int, symmetric: bool = False) -> list[Shard]:
    """N-sharding (W[:, cols], b[cols]); 4-aligned for symmetric 4-column groups."""
    return split(N, world, 4 if symmetric else 1)


def row_shards(M: int, world: int) -> list[Shard]:
    """M-sharding (X[rows]); W replicated."""
    return split(M, world, 1)


def _world(group) -> tuple[int, int]:
    if group is None and not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def gather_columns(y_local: torch.Tensor, shards: list[Shard], group=None, out: torch.Tensor | None = None,
                   staging: torch.Tensor | None = None) -> torch.Tensor:
    """Assemble row-major Y [M, N] from per-rank column blocks [M, w_r].

    Equal widths: one ``all_gather_into_tensor`` into a [world, M, w] staging
    buffer, then one permuting copy to [M, N].  Unequal widths fall back to
    ``all_gather`` of padded blocks.  Single rank: returns y_local."""
    rank, world = _world(group)
    if world == 1:
        if out is not None:
            out.copy_(y_local)
            return out
        return y_local
    M = y_local.shape[0]
    N = shards[-1].stop
    wmax = max(s.width for s in shards)
    if y_local.shape[1] != shards[rank].width:
        raise ParameterError(f"rank {rank}: local block has {y_local.shape[1]} columns, shard has "
                             f"{shards[rank].width}")
    if staging is None or staging.shape != (world, M, wmax):
        staging = torch.empty((world, M, wmax), dtype=y_local.dtype, device=y_local.device)
    src = y_local if y_local.shape[1] == wmax else torch.nn.functional.pad(y_local, (0, wmax - y_local.shape[1]))
    src = src.contiguous()
    if hasattr(dist, "all_gather_into_tensor") and (y_local.is_cuda or dist.get_backend(group) != "gloo"):
        dist.all_gather_into_tensor(staging, src, group=group)
    else:
        dist.all_gather(list(staging.unbind(0)), src, group=group)
    if out is None:
        out = torch.empty((M, N), dtype=y_local.dtype, device=y_local.device)
    if all(s.width == wmax for s in shards):
        out.view(M, world, wmax).copy_(staging.permute(1, 0, 2))
    else:
        for s in shards:
            out[:, s.slice()] = staging[s.rank, :, : s.width]
    return out


def gather_rows(y_local: torch.Tensor, shards: list[Shard], group=None, out: torch.Tensor | None = None
                ) -> torch.Tensor:
    """Assemble Y [M, N] from per-rank row blocks; equal heights gather straight into Y."""
    rank, world = _world(group)
    if world == 1:
        return y_local
    N = y_local.shape[1]
    M = shards[-1].stop
    hmax = max(s.width for s in shards)
    equal = all(s.width == hmax for s in shards)
    src = y_local.contiguous()
    if equal:
        if out is None:
            out = torch.empty((M, N), dtype=y_local.dtype, device=y_local.device)
        if y_local.is_cuda or dist.get_backend(group) != "gloo":
            dist.all_gather_into_tensor(out, src, group=group)
        else:
            dist.all_gather(list(out.view(world, hmax, N).unbind(0)), src, group=group)
        return out
    pad = torch.zeros((hmax, N), dtype=y_local.dtype, device=y_local.device)
    pad[: src.shape[0]] = src
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([bufs[s.rank][: s.width] for s in shards], 0)


class ShardedGemm:
    """One rank's share of a partitioned GEMM.

    ``compute(shard) -> Tensor`` produces this rank's block (columns
    ``shard.start:shard.stop`` of Y for mode "columns", rows for "rows");
    ``run()`` computes it and all-gathers the full Y."""

    def __init__(self, M: int, N: int, mode: str = "columns", symmetric: bool = False, group=None):
        if mode not in ("columns", "rows"):
            raise ParameterError(f"mode must be 'columns' or 'rows', got {mode!r}")
        self.M, self.N, self.mode, self.group = M, N, mode, group
        self.rank, self.world = _world(group)
        self.shards = column_shards(N, self.world, symmetric) if mode == "columns" else row_shards(M, self.world)
        self.shard = self.shards[self.rank]
        self._staging = None

    def assemble(self, y_local: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if self.mode == "columns":
            if self.world > 1 and self._staging is None:
                wmax = max(s.width for s in self.shards)
                self._staging = torch.empty((self.world, self.M, wmax), dtype=y_local.dtype, device=y_local.device)
            return gather_columns(y_local, self.shards, self.group, out, self._staging)
        return gather_rows(y_local, self.shards, self.group, out)

    def run(self, compute: Callable[[Shard], torch.Tensor]) -> torch.Tensor:
        return self.assemble(compute(self.shard))
