"""Host-side checks of the fused peer scatter (paper_2510_06957_b200/peer.py).

The multi-GPU path cannot run on the one-GPU box, so its flow control is
checked here as a model: every rank executes, in stream order, for each step
s: GEMM(s) (stores its shard into slot s % S of every rank, one peer at a
time, then bumps every rank's arrival counter), WAIT(s) (until every rank's
counter reached s + 1), CONSUME(s) (reads its own slot s % S).  A random
scheduler interleaves the ranks' next enabled operations; the invariant is
that no store ever lands in a slot whose previous step the owner has not yet
consumed, and that every CONSUME sees all shards of its own step.  With two
slots it must hold on every schedule; with one slot the model must find a
violation (which is why PeerYBuffers defaults to two).
"""

from __future__ import annotations

import random

import pytest

from paper_2510_06957_b200.partition import column_shards
from paper_2510_06957_b200.peer import PeerLayout


def _simulate(world: int, slots: int, steps: int, seed: int) -> str | None:
    rng = random.Random(seed)
    # per rank: program counter over ops, arrival counters, consumed steps, slot contents
    prog = [[op for s in range(steps) for op in (("gemm", s), ("wait", s), ("consume", s))] for _ in range(world)]
    pc = [0] * world
    pending = [None] * world          # peers still to store into for the GEMM in flight
    arrivals = [[0] * world for _ in range(world)]  # arrivals[q][r]: rank r's arrivals at rank q
    consumed = [-1] * world
    content = [[[None] * world for _ in range(slots)] for _ in range(world)]  # content[q][slot][r] = step
    while any(pc[r] < len(prog[r]) for r in range(world)):
        ready = []
        for r in range(world):
            if pc[r] >= len(prog[r]):
                continue
            kind, s = prog[r][pc[r]]
            if kind == "wait" and not all(arrivals[r][q] >= s + 1 for q in range(world)):
                continue
            ready.append(r)
        if not ready:
            return "deadlock"
        r = rng.choice(ready)
        kind, s = prog[r][pc[r]]
        if kind == "gemm":
            if pending[r] is None:
                pending[r] = list(range(world))
                rng.shuffle(pending[r])
            q = pending[r].pop()
            # the owner must have consumed the step that last used this slot
            if consumed[q] < s - slots:
                return f"rank {r} overwrote slot {s % slots} of rank {q} (step {s}) before it consumed step {s - slots}"
            content[q][s % slots][r] = s
            if not pending[r]:
                pending[r] = None
                for q2 in range(world):
                    arrivals[q2][r] += 1
                pc[r] += 1
        elif kind == "wait":
            pc[r] += 1
        else:
            if any(content[r][s % slots][q] != s for q in range(world)):
                return f"rank {r} consumed step {s} with shards {content[r][s % slots]}"
            consumed[r] = s
            pc[r] += 1
    return None


@pytest.mark.parametrize("world", [2, 3, 8])
def test_two_slots_never_overwrite_unconsumed_data(world):
    for seed in range(300):
        assert _simulate(world, 2, 6, seed) is None, seed


def test_one_slot_is_not_enough():
    bad = [_simulate(2, 1, 4, seed) for seed in range(300)]
    assert any(b is not None and "overwrote" in b for b in bad)


def test_peer_layout():
    L = PeerLayout(10, 7, 2)
    assert L.slot_bytes == 512 and L.slot_offset(0) == 256 and L.slot_offset(1) == 768 and L.total_bytes == 1280
    L = PeerLayout(4096, 11008, 2)
    assert L.slot_offset(1) % 256 == 0 and L.total_bytes == 256 + 2 * 4096 * 11008 * 4
    with pytest.raises(Exception):
        L.slot_offset(2)


def test_shard_offsets_allow_vector_peer_stores():
    """Symmetric (4-aligned) shards give 4-aligned column offsets: the smem-tile path with
    16-byte peer stores; other widths fall back to the direct-store path (tested on the GPU)."""
    for N, world in [(11008, 8), (4096, 4), (4100, 8)]:
        offs = [s.start for s in column_shards(N, world, symmetric=True)]
        assert all(o % 4 == 0 for o in offs)
