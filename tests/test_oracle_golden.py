"""Pin the CPU oracle to the reference: every builder and kernel of
oracle/tg_oracle.c must reproduce the fixtures generated from the reference
package (tests/golden/make_golden.py) bit for bit — formats AND real-valued Y."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import worked_example
from oracle import oracle as orc


def _fmt_keys(golden, prefix):
    return {k.split(".")[-1]: golden[k] for k in golden.npz.files if k.startswith(prefix + ".")}


def test_worked_example_known_answers():
    W, X, b = worked_example()
    t = orc.tcsc_from_dense(W)
    # pkg/tests/test_tcsc.py:15-24
    assert t["col_start_pos"].tolist() == [0, 2, 2]
    assert t["row_index_pos"].tolist() == [0, 3]
    assert t["col_start_neg"].tolist() == [0, 1, 2]
    assert t["row_index_neg"].tolist() == [2, 1]
    # pkg/tests/test_variants.py:18-28 (B = 2)
    bl = orc.blocked_from_dense(W, 2)
    assert bl["row_index_pos"].tolist() == [0, 3]
    assert bl["row_index_neg"].tolist() == [1, 2]
    assert bl["col_start_pos"].tolist() == [[0, 1, 1], [1, 2, 2]]
    assert bl["col_start_neg"].tolist() == [[0, 0, 1], [1, 2, 2]]
    # interleaved, g = 1, one block (pkg/tests/test_variants.py:55-61)
    ib = orc.interleaved_blocked_from_dense(W, 4, 1)
    assert ib["col_segment_ptr"].tolist() == [0, 2, 3, 3, 3, 3, 4]
    assert ib["all_indices"].tolist() == [0, 2, 3, 1]
    ib2 = orc.interleaved_blocked_from_dense(W, 2, 1)
    assert ib2["all_indices"].tolist() == [0, 1, 3, 2]
    assert ib2["col_segment_ptr"].tolist() == [0, 0, 1, 1, 1, 1, 2, 4, 4, 4, 4, 4, 4]
    # every kernel gives [[12, 18]] (pkg/tests/test_kernels_scalar.py:38-42)
    assert orc.gemm_base(X, t, b).tolist() == [[12.0, 18.0]]
    assert orc.gemm_unrolled(X, t, b).tolist() == [[12.0, 18.0]]
    assert orc.gemm_blocked(X, bl, b).tolist() == [[12.0, 18.0]]
    assert orc.gemm_interleaved_blocked(X, ib, b).tolist() == [[12.0, 18.0]]
    assert orc.oracle_gemm(X, W, b).tolist() == [[12.0, 18.0]]
    assert orc.oracle_gemm(X, W, np.array([10.0, -30.0], np.float32), 0.5).tolist() == [[12.0, -16.0]]


def test_symmetric_known_answer():
    W = np.zeros((8, 4), np.int8)
    W[0:2, 0] = 1
    W[2:4, 0] = -1
    W[5, 1] = 1
    s = orc.interleaved_blocked_from_dense(W, 4, 2, True)
    assert s["all_indices"].tolist() == [0, 1, 2, 3, 8, 8, 8, 8, 8, 8, 8, 8, 8, 8, 8, 8, 5]
    assert s["col_segment_ptr"].tolist() == [0, 4, 4, 4, 8, 8, 8, 12, 12, 12, 16, 16, 16, 16, 16, 16, 16, 17, 17,
                                             17, 17, 17, 17, 17, 17]
    assert orc.interleaved_blocked_from_dense(W, 4, 2, False)["all_indices"].tolist() == [0, 1, 2, 3, 5]


def test_formats_match_reference(golden_formats):
    checked = 0
    for entry in golden_formats.index:
        key = entry["key"]
        W = golden_formats[f"{key}.W"]
        t = orc.tcsc_from_dense(W)
        for name, arr in _fmt_keys(golden_formats, f"{key}.tcsc").items():
            assert np.array_equal(t[name], arr), (key, "tcsc", name)
        for f in entry["formats"][1:]:
            ref = _fmt_keys(golden_formats, f"{key}.{f['name']}")
            if f["name"].startswith("sym_"):
                got = orc.symmetric_from_dense(W, f["g"])
                assert (got["indices"].size + got["col_ptr"].size) * 4 == f["bytes"]
                assert int((got["indices"] == W.shape[0]).sum()) == f["dummies"]
                for name, arr in ref.items():
                    assert np.array_equal(got[name], arr), (key, f["name"], name)
                checked += 1
                continue
            if f["name"] == "compressed":
                got = orc.compressed_from_dense(W)
                assert np.array_equal(got["codes"], ref["codes"]), key
                assert got["codes"].size == f["bytes"]
                checked += 1
                continue
            if f["name"].startswith("blocked"):
                got = orc.blocked_from_dense(W, f["B"])
            else:
                got = orc.interleaved_blocked_from_dense(W, f["B"], f["g"], f["sym"])
                assert got["all_indices"].size * 4 + got["col_segment_ptr"].size * 4 == f["bytes"]
            assert got["B"] == f["resolved_B"]
            for name, arr in ref.items():
                assert np.array_equal(got[name], arr), (key, f["name"], name)
            checked += 1
    assert checked > 500


def _check_runs(golden, entry, threads):
    key = entry["key"]
    W, X, b = golden[f"{key}.W"], golden[f"{key}.X"], golden[f"{key}.b"]
    for run in entry["runs"]:
        name = run["name"]
        ref = golden[f"{key}.{name}"]
        if name == "base":
            y = orc.gemm_base(X, orc.tcsc_from_dense(W), b, threads=threads)
        elif name.startswith("unrolled"):
            y = orc.gemm_unrolled(X, orc.tcsc_from_dense(W), b, uf=run["uf"], threads=threads)
        elif name.startswith("blocked"):
            y = orc.gemm_blocked(X, orc.blocked_from_dense(W, run["B"]), b, uf=run["uf"], mr=run["mr"],
                                 threads=threads)
        elif name.startswith("ib"):
            y = orc.gemm_interleaved_blocked(X, orc.interleaved_blocked_from_dense(W, run["B"], run["g"]), b,
                                             threads=threads)
        elif name == "compressed":
            y = orc.gemm_compressed(X, orc.compressed_from_dense(W), b, threads=threads)
        elif name.startswith("vertical") or name.startswith("horizontal"):
            t = orc.symmetric_from_dense(W, run["g"])
            fn = orc.gemm_vertical if name.startswith("vertical") else orc.gemm_horizontal
            y = fn(orc.pad_input(X), t, b, run["alpha"], threads=threads)
        else:
            t = orc.interleaved_blocked_from_dense(W, run["B"], run["g"], True)
            y = orc.gemm_vectorized_optimal(orc.pad_input(X), t, b, run["alpha"], threads=threads)
        # bit-exact, including real-valued X (same fp32 operation order as numba)
        assert y.dtype == np.float32
        assert np.array_equal(y.view(np.uint32), ref.view(np.uint32)), (key, entry["xmode"], name)


@pytest.mark.parametrize("threads", [1, 3])
def test_kernels_match_reference_bitwise(golden_kernels, threads):
    for entry in golden_kernels.index:
        _check_runs(golden_kernels, entry, threads)


def test_oracle_gemm_matches_reference(golden_kernels):
    for entry in golden_kernels.index:
        key = entry["key"]
        W, X, b = golden_kernels[f"{key}.W"], golden_kernels[f"{key}.X"], golden_kernels[f"{key}.b"]
        for alpha in (None, 0.25):
            assert np.array_equal(orc.oracle_gemm(X, W, b, alpha), golden_kernels[f"{key}.oracle_a{alpha}"])


def test_integer_regime_is_exact_everywhere(golden_kernels):
    # dense.py:17-19: integer X, |x| <= 8 and K*8 < 2^24 -> every order is exact
    for entry in golden_kernels.index:
        if entry["xmode"] != "int":
            continue
        key = entry["key"]
        for run in entry["runs"]:
            alpha = run.get("alpha")
            if alpha not in (None, 0.25):
                continue
            ref = golden_kernels[f"{key}.oracle_a{alpha}"]
            assert np.array_equal(golden_kernels[f"{key}.{run['name']}"], ref), (key, run["name"])


def test_compressed_and_symmetric_known_answers():
    W, X, b = worked_example()
    # pkg/tests/test_variants.py:216-224: col0 = [+1, 0, -1, +1] -> 140, col1 = [0, -1, 0, 0] -> 118
    c = orc.compressed_from_dense(W)
    assert c["codes"].shape == (2, 1) and c["codes"].tolist() == [[140], [118]]
    assert orc.gemm_compressed(X, c, b).tolist() == [[12.0, 18.0]]
    # the SURVEY 8x4 matrix, g = 2: group max(max(p, q)) = 2 -> 4 pairs (lcm(4, 2))
    W8 = np.zeros((8, 4), np.int8)
    W8[0:2, 0] = 1
    W8[2:4, 0] = -1
    W8[5, 1] = 1
    s = orc.symmetric_from_dense(W8, 2)
    assert s["col_ptr"].tolist() == [0, 8, 16, 24, 32]
    assert s["indices"][:8].tolist() == [0, 1, 2, 3, 8, 8, 8, 8]
    assert s["indices"][8:16].tolist() == [5, 8, 8, 8, 8, 8, 8, 8]


def test_cfg1_pins(golden_cfg1):
    from paper_2510_06957_b200.workloads import make_inputs

    W, X, b = make_inputs("cfg1")
    t = orc.tcsc_from_dense(W)
    for name in ("col_start_pos", "col_start_neg", "row_index_pos", "row_index_neg"):
        assert np.array_equal(t[name], golden_cfg1[name])
    y = orc.gemm_base(X, t, b, threads=4)
    assert np.array_equal(y, golden_cfg1["Y_base"])
    # SURVEY.md 8(c) regression values
    assert int(t["col_start_pos"][-1]) == 65463 and int(t["col_start_neg"][-1]) == 65700
    assert y[0, :4].tolist() == [4.957159996032715, 6.670194625854492, -2.692211866378784, -11.097043991088867]
    assert orc.normwise_error(y, golden_cfg1["oracle"]) < 1e-5
