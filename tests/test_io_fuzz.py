"""Corrupted TGW1 / TGS1 files: random byte flips, truncations and splices of valid files
must be rejected exactly as the reference rejects them (same exception class, same byte
offset for ParseError) or load to the same arrays.  Runs on CPU against the reference
package, imported read-only from /root/reference when it is present (it is not on the GPU
boxes; the test is then skipped)."""

from __future__ import annotations

import io as _io
import os
import sys

import numpy as np
import pytest

import paper_2510_06957_b200 as tg
from paper_2510_06957_b200 import io as tio
from oracle import oracle as orc

REF = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(REF):
        pytest.skip("reference package not mounted")
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    try:
        import terngemm
        from terngemm import io as rio
    except Exception as exc:  # noqa: BLE001
        pytest.skip(f"reference not importable: {exc}")
    return terngemm, rio


def _files(W):
    K, N = W.shape
    out = []
    fh = _io.BytesIO()
    tio.save_dense(tg.TernaryDense(W), fh)
    out.append(fh.getvalue())
    t = orc.tcsc_from_dense(W)
    bl = orc.blocked_from_dense(W, 4)
    ib = orc.interleaved_blocked_from_dense(W, 4, 2, False)
    fmts = [
        tg.Tcsc(K, N, t["col_start_pos"], t["row_index_pos"], t["col_start_neg"], t["row_index_neg"]),
        tg.BlockedTcsc(K, N, 4, bl["col_start_pos"], bl["row_index_pos"], bl["col_start_neg"], bl["row_index_neg"]),
        tg.InterleavedBlockedTcsc(K, N, 4, 2, ib["all_indices"], ib["col_segment_ptr"]),
        tg.CompressedTcsc(K, N, orc.compressed_from_dense(W)["codes"]),
    ]
    if N % 4 == 0:
        sy = orc.symmetric_from_dense(W, 2)
        fmts.append(tg.SymmetricInterleavedTcsc(K, N, 2, sy["indices"], sy["col_ptr"]))
    for f in fmts:
        fh = _io.BytesIO()
        tio.save_sparse(f, fh)
        out.append(fh.getvalue())
    return out


def _outcome(fn, data):
    try:
        obj = fn(data)
    except Exception as exc:  # noqa: BLE001 -- the class is the outcome
        return ("raise", type(exc).__name__, getattr(exc, "offset", None))
    if hasattr(obj, "values") and not hasattr(obj, "_a"):
        return ("ok", np.asarray(obj.values).tobytes())
    arrays = {}
    for name in ("col_start_pos", "row_index_pos", "col_start_neg", "row_index_neg", "all_indices",
                 "col_segment_ptr", "indices", "col_ptr", "codes"):
        try:
            arrays[name] = np.asarray(getattr(obj, name)).tobytes()
        except AttributeError:
            pass
    return ("ok", type(obj).__name__, sorted(arrays.items()))


@pytest.mark.parametrize("seed", range(40))
def test_corrupted_files_behave_like_the_reference(ref, seed):
    _, rio = ref
    rng = np.random.default_rng(seed)
    K, N = int(rng.integers(1, 20)), int(4 * rng.integers(1, 5))
    W = rng.integers(-1, 2, size=(K, N)).astype(np.int8)
    for data in _files(W):
        for _ in range(12):
            d = bytearray(data)
            kind = rng.integers(0, 3)
            if kind == 0:  # flip a few bytes
                for _ in range(int(rng.integers(1, 4))):
                    d[int(rng.integers(0, len(d)))] = int(rng.integers(0, 256))
            elif kind == 1:  # truncate
                d = d[: int(rng.integers(0, len(d)))]
            else:  # append junk
                d += bytes(rng.integers(0, 256, size=int(rng.integers(1, 8)), dtype=np.uint8))
            d = bytes(d)
            mine, theirs = _outcome(tio.load_any, d), _outcome(rio.load_any, d)
            if theirs[0] == "raise" and theirs[1] == "ParseError" and "interleaved" not in str(theirs):
                assert mine[:2] == theirs[:2], (seed, kind, mine, theirs)
                assert mine[2] == theirs[2], (seed, kind, mine, theirs)  # same byte offset
            elif theirs[0] == "ok" and mine[0] == "ok":
                assert mine[-1] == theirs[-1], (seed, kind)
            elif theirs[0] == "raise":
                assert mine[0] == "raise", (seed, kind, mine, theirs)
            else:  # the reference loads it: so must we, unless it is a format outside our scope
                assert mine[0] == "ok" or mine[1] == "ParseError", (seed, kind, mine, theirs)
