"""TGW1 / TGS1 files and the seeded generators against bytes written by the
reference itself (tests/golden/files.npz, made by make_golden.py from
/root/reference io.py / dense.py), plus the reference's own io edge cases
(pkg/tests/test_io.py): truncation at every byte, bad magic, unknown tag,
trailing bytes, non-ternary payload offsets, dispatch.  Runs on CPU: parsing
and serialisation are host logic (the GPU tests check the device landing)."""

from __future__ import annotations

import io as _io
import json
import os

import numpy as np
import pytest
import torch

import paper_2510_06957_b200 as tg
from paper_2510_06957_b200 import cli
from paper_2510_06957_b200 import io as tio
from paper_2510_06957_b200.errors import ParseError
from conftest import GOLDEN, worked_example
from oracle import oracle as orc


@pytest.fixture(scope="module")
def files():
    z = np.load(os.path.join(GOLDEN, "files.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    return z, meta


def _bytes(a) -> bytes:
    return np.asarray(a, dtype=np.uint8).tobytes()


def _dump(fn, obj) -> bytes:
    fh = _io.BytesIO()
    fn(obj, fh)
    return fh.getvalue()


def _host_formats(W: np.ndarray) -> dict:
    """Format objects over the C oracle's builder arrays (bit-exact with the reference builders)."""
    K, N = W.shape
    t = orc.tcsc_from_dense(W)
    bl = orc.blocked_from_dense(W, 8)
    ib = orc.interleaved_blocked_from_dense(W, 8, 2, False)
    out = {
        "tcsc": tg.Tcsc(K, N, t["col_start_pos"], t["row_index_pos"], t["col_start_neg"], t["row_index_neg"]),
        "blocked": tg.BlockedTcsc(K, N, 8, bl["col_start_pos"], bl["row_index_pos"], bl["col_start_neg"],
                                  bl["row_index_neg"]),
        "interleaved_blocked": tg.InterleavedBlockedTcsc(K, N, 8, 2, ib["all_indices"], ib["col_segment_ptr"]),
        "compressed": tg.CompressedTcsc(K, N, orc.compressed_from_dense(W)["codes"]),
    }
    if N % 4 == 0:
        ibs = orc.interleaved_blocked_from_dense(W, 8, 2, True)
        out["interleaved_blocked_sym"] = tg.InterleavedBlockedTcsc(K, N, 8, 2, ibs["all_indices"],
                                                                   ibs["col_segment_ptr"], True)
        sy = orc.symmetric_from_dense(W, 2)
        out["symmetric"] = tg.SymmetricInterleavedTcsc(K, N, 2, sy["indices"], sy["col_ptr"])
    return out


def test_generators_match_the_reference(files):
    z, meta = files
    for i, m in enumerate(meta):
        assert np.array_equal(tg.gen_ternary(m["K"], m["N"], m["s"], m["seed"]).values, z[f"f{i}_W"])
        assert np.array_equal(tg.gen_input(5, m["K"], m["seed"] + 1).values, z[f"f{i}_gen_input"])
        assert np.array_equal(tg.gen_bias(m["N"], m["seed"] + 2).values, z[f"f{i}_gen_bias"])
        assert np.array_equal(tg.gen_input_uniform(3, m["K"], m["seed"]).values, z[f"f{i}_gen_uniform"])


def test_dense_file_bytes_and_load(files):
    z, meta = files
    for i, _ in enumerate(meta):
        W = z[f"f{i}_W"]
        ref = _bytes(z[f"f{i}_dense"])
        assert _dump(tio.save_dense, tg.TernaryDense(W)) == ref
        assert np.array_equal(tio.load_dense(ref).values, W)
        assert isinstance(tio.load_any(ref), tg.TernaryDense)


def test_sparse_files_byte_identical_with_the_reference(files):
    """Saving a format built from the same W writes the reference's bytes; loading the
    reference's file gives the same arrays and saves back to the same bytes."""
    z, meta = files
    for i, m in enumerate(meta):
        W = z[f"f{i}_W"]
        fmts = _host_formats(W)
        assert sorted(fmts) == m["formats"]
        for name, fmt in fmts.items():
            ref = _bytes(z[f"f{i}_{name}"])
            assert _dump(tio.save_sparse, fmt) == ref, (i, name)
            back = tio.load_sparse(ref)
            assert type(back) is type(fmt)
            for attr in ("K", "N", "B", "g", "symmetric_groups"):
                if hasattr(fmt, attr):
                    assert getattr(back, attr) == getattr(fmt, attr), (name, attr)
            assert _dump(tio.save_sparse, back) == ref, (i, name)


def test_unsupported_reference_formats_are_parse_errors(files):
    z, _ = files
    with pytest.raises(ParseError, match="interleaved"):
        tio.load_sparse(_bytes(z["f0_interleaved"]))


def test_worked_example_round_trip():
    W, _, _ = worked_example()
    data = _dump(tio.save_dense, tg.TernaryDense(W))
    assert data[:4] == tio.DENSE_MAGIC
    assert np.array_equal(tio.load_dense(data).values, W)


def test_dense_errors():
    W, _, _ = worked_example()
    data = _dump(tio.save_dense, tg.TernaryDense(W))
    with pytest.raises(ParseError):
        tio.load_dense(data + b"\x00")  # trailing bytes
    with pytest.raises(ParseError):
        tio.load_dense(b"XXXX" + data[4:])
    bad = bytearray(data)
    bad[-1] = 5
    with pytest.raises(ParseError) as err:
        tio.load_dense(bytes(bad))
    assert err.value.offset == len(bad) - 1
    bad = bytearray(data)
    bad[16 + 3] = 0x80  # -128 in the middle of the payload
    with pytest.raises(ParseError) as err:
        tio.load_dense(bytes(bad))
    assert err.value.offset == 19
    for cut in range(len(data)):
        with pytest.raises(ParseError):
            tio.load_dense(data[:cut])


def test_sparse_errors(files):
    z, _ = files
    data = _bytes(z["f1_interleaved_blocked"])
    for cut in range(len(data)):
        with pytest.raises(ParseError):
            tio.load_sparse(data[:cut])
    tagged = bytearray(_bytes(z["f0_tcsc"]))
    tagged[8] = 99
    with pytest.raises(ParseError):
        tio.load_sparse(bytes(tagged))
    with pytest.raises(ParseError):
        tio.load_sparse(_bytes(z["f0_tcsc"]) + b"\x01")
    # a section of the wrong length: the constructor's error becomes ParseError at the end of the file
    W = z["f0_W"]
    t = orc.tcsc_from_dense(W)
    short = tg.Tcsc(W.shape[0], W.shape[1] - 1, t["col_start_pos"][:-1], t["row_index_pos"],
                    t["col_start_neg"][:-1], t["row_index_neg"])
    raw = bytearray(_dump(tio.save_sparse, short))
    raw[16:20] = int(W.shape[1]).to_bytes(4, "little")  # claim N columns
    with pytest.raises(ParseError) as err:
        tio.load_sparse(bytes(raw))
    assert err.value.offset == len(raw)


def test_load_any_dispatch(files):
    z, _ = files
    assert isinstance(tio.load_any(_bytes(z["f0_tcsc"])), tg.Tcsc)
    with pytest.raises(ParseError):
        tio.load_any(b"ZZZZ\x00\x00\x00\x00")
    with pytest.raises(ParseError):
        tio.load_any(b"")


def test_cli_gen_writes_the_reference_file(tmp_path, files):
    z, meta = files
    m = meta[1]
    out = tmp_path / "w.tgw"
    assert cli.main(["gen", "--K", str(m["K"]), "--N", str(m["N"]), "--s", m["s"], "--seed", str(m["seed"]),
                     "--out", str(out)]) == 0
    assert out.read_bytes() == _bytes(z["f1_dense"])


def test_cli_exit_codes(tmp_path):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"nope")
    assert cli.main(["convert", "--in", str(bad), "--to", "tcsc", "--out", str(tmp_path / "o")]) == 3
    assert cli.main(["convert", "--in", str(tmp_path / "missing"), "--to", "tcsc", "--out", str(tmp_path / "o")]) == 3
    assert cli.main(["gen", "--K", "0", "--N", "4", "--s", "1/2", "--out", str(tmp_path / "x")]) == 2


@pytest.mark.skipif(torch.cuda.is_available(), reason="host-side parse path (no device)")
def test_sections_stay_on_host_without_a_device(files):
    z, _ = files
    t = tio.load_sparse(_bytes(z["f0_tcsc"]))
    assert isinstance(t._a["row_index_pos"]._h, np.ndarray)
