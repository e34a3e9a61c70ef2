"""Device landing of TGW1 / TGS1 files and the CLI over the device builders:
loaded sections are CUDA tensors, `to_dense` decodes them on the device, and
`convert` writes exactly the reference's bytes (its builders are bit-exact),
`verify` passes every variant on both GPU paths (integer inputs: bit-exact)."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2510_06957_b200 as tg
    from paper_2510_06957_b200 import cli, io as tio
    from conftest import GOLDEN

    z = np.load(os.path.join(GOLDEN, "files.npz"))
    return tg, cli, tio, z, json.loads(bytes(z["meta"]).decode())


def _b(a) -> bytes:
    return np.asarray(a, dtype=np.uint8).tobytes()


def test_load_lands_on_device(env):
    tg, _, tio, z, meta = env
    for i, m in enumerate(meta):
        W = z[f"f{i}_W"]
        d = tio.load_dense(_b(z[f"f{i}_dense"]))
        assert d.device_values.is_cuda and np.array_equal(d.values, W)
        for name in m["formats"]:
            fmt = tio.load_sparse(_b(z[f"f{i}_{name}"]))
            arrays = fmt._a if hasattr(fmt, "_a") else {"codes": fmt._c}
            for dual in arrays.values():
                assert dual._d is not None and dual._d.is_cuda and dual._h is None, (i, name)
            assert np.array_equal(fmt.to_dense().values, W), (i, name)


def test_device_payload_check_reports_offset(env):
    _, _, tio, z, _ = env
    from paper_2510_06957_b200.errors import ParseError

    data = bytearray(_b(z["f2_dense"]))
    data[16 + 777] = 7
    data[16 + 900] = 0xFE  # -2, later: the first bad byte is reported
    with pytest.raises(ParseError) as err:
        tio.load_dense(bytes(data))
    assert err.value.offset == 16 + 777


def test_corrupt_sparse_file_raises_on_decode(env):
    tg, _, tio, z, _ = env
    from paper_2510_06957_b200.errors import CorruptionError

    fmt = tio.load_sparse(_b(z["f0_tcsc"]))
    csp = fmt.col_start_pos
    n = int(np.flatnonzero(np.diff(csp) >= 2)[0])  # a column with two +1 rows
    rip = fmt.device("row_index_pos")
    rip[int(csp[n]) + 1] = rip[int(csp[n])]  # the same row twice in that column
    with pytest.raises(CorruptionError):
        fmt.to_dense()


def test_cli_convert_writes_reference_bytes(env, tmp_path):
    _, cli, _, z, meta = env
    for i, m in enumerate(meta):
        src = tmp_path / f"w{i}.tgw"
        src.write_bytes(_b(z[f"f{i}_dense"]))
        for name in m["formats"]:
            out = tmp_path / f"{i}_{name}.tgs"
            args = ["convert", "--in", str(src), "--out", str(out)]
            if name == "interleaved_blocked_sym":
                args += ["--to", "interleaved_blocked", "--B", "8", "--g", "2", "--symmetric"]
            elif name in ("blocked", "interleaved_blocked"):
                args += ["--to", name, "--B", "8", "--g", "2"]
            else:
                args += ["--to", name, "--g", "2"]
            assert cli.main(args) == 0
            assert out.read_bytes() == _b(z[f"f{i}_{name}"]), (i, name)
            back = tmp_path / f"{i}_{name}.tgw"
            assert cli.main(["convert", "--in", str(out), "--to", "dense", "--out", str(back)]) == 0
            assert back.read_bytes() == _b(z[f"f{i}_dense"]), (i, name)


@pytest.mark.parametrize("method", ["mma", "gather"])
def test_cli_verify_every_variant(env, method, capsys):
    _, cli, _, _, _ = env
    assert cli.main(["verify", "--M", "9", "--K", "300", "--N", "24", "--method", method]) == 0
    assert cli.main(["verify", "--M", "5", "--K", "130", "--N", "16", "--alpha", "0.25", "--method", method]) == 0
    out = capsys.readouterr().out
    assert "FAIL" not in out and out.count("ok ") >= 8
