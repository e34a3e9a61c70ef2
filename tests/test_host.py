"""Host-side logic that needs no GPU: configuration checks, the registry
contract, the cost model, the workload generator pins and the C-ABI symbol
table of the built library (loaded, no compute calls)."""

from __future__ import annotations

import ctypes
import os
import re
from fractions import Fraction

import numpy as np
import pytest

import paper_2510_06957_b200 as tg
from paper_2510_06957_b200 import _native
from paper_2510_06957_b200.workloads import WORKLOADS, algorithmic_bytes, cfg5_oracle_rows, make_inputs, ops

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_config_validation_matches_reference():
    # kernels/scalar.py:79-91
    for bad in (dict(uf=0), dict(mr=3), dict(nr=8), dict(b=0), dict(g=0), dict(alpha=float("nan")),
                dict(method="cpu")):
        with pytest.raises(tg.ParameterError):
            tg.GemmConfig(**bad)
    cfg = tg.GemmConfig().with_variant("base")
    assert cfg.variant == "base" and cfg.uf == 12 and cfg.mr == 4 and cfg.nr == 4 and cfg.b is None


def test_registry_contract():
    # kernels/__init__.py:66-80, 98-208: the reference's tags (in its order), kinds, emit sets and
    # alpha support; `inverted` (variants.py:384-443) is the one format the paper rejected and is absent
    assert tg.SCALAR_TAGS == ("base", "unrolled", "blocked", "interleaved_blocked", "compressed")
    assert tg.SIMD_TAGS == ("vertical", "horizontal", "vectorized_optimal")
    for tag, spec in tg.VARIANTS.items():
        assert spec.tag == tag
        assert spec.supports_alpha == (spec.kind == "simd")
    assert tg.get_variant("blocked").emit == frozenset({"UF", "MR", "NR", "B"})
    assert tg.get_variant("vertical").emit == frozenset({"g"})
    assert tg.get_variant("compressed").emit == frozenset()
    with pytest.raises(tg.ParameterError):
        tg.get_variant("inverted")


def test_packed_byte_codec():
    # pkg/tests/test_variants.py:179-212
    assert tg.compress5([-1] * 5) == 0
    assert tg.compress5([0] * 5) == 121
    assert tg.compress5([1] * 5) == 242
    assert tg.compress5([1, 0, -1, 0, 1]) == 194
    for code in range(tg.CODE_COUNT):
        assert tg.compress5(tg.decompress5(code)) == code
    for code in (tg.CODE_COUNT, 255, -1):
        with pytest.raises(tg.InvalidCodeError):
            tg.decompress5(code)
    with pytest.raises(tg.ParameterError):
        tg.compress5([0, 0, 0, 2, 0])
    with pytest.raises(tg.ParameterError):
        tg.compress5([0, 0, 0])
    assert tg.DECODE_TABLE.shape == (tg.CODE_COUNT, tg.PACK_WIDTH) and tg.DECODE_TABLE.dtype == np.int8
    assert not tg.DECODE_TABLE.flags.writeable
    for code in (0, 121, 194, 242):
        assert tuple(tg.DECODE_TABLE[code]) == tg.decompress5(code)
    # host-side construction checks of the compressed and symmetric formats
    with pytest.raises(tg.InvalidCodeError):
        tg.CompressedTcsc(4, 1, np.array([[250]], dtype=np.uint8))
    with pytest.raises(tg.ParameterError):
        tg.CompressedTcsc(4, 1, np.array([[1, 2]], dtype=np.uint8))
    c = tg.CompressedTcsc(4, 2, np.array([[140], [118]], dtype=np.uint8))
    assert c.format_bytes() == 2 and c.groups_per_col == 1 and c.nnz == 4
    with pytest.raises(tg.ParameterError):
        tg.SymmetricInterleavedTcsc(4, 3, 2, [], [0, 0, 0, 0])
    s = tg.SymmetricInterleavedTcsc(8, 4, 2, [0, 1, 2, 3, 8, 8, 8, 8], [0, 8, 8, 8, 8])
    assert s.format_bytes() == 4 * (8 + 5) and s.pairs_in_group(0) == 4


def test_cost_model_pins():
    # pkg/tests/test_bench.py:23-27 and 45-56
    assert tg.flop_count(32, 1024, 1024, 1024 * 256) == 8_421_376
    assert tg.flop_count(64, 4096, 4096, 4096 * 2048) == 537_133_056
    assert tg.flop_count(3, 10, 4, 0) == 12
    with pytest.raises(tg.ParameterError):
        tg.flop_count(0, 1, 1, 0)
    with pytest.raises(tg.ParameterError):
        tg.flop_count(1, 2, 2, 5)
    oi = tg.operational_intensity(64, 1024, 1024, 1024 * 512, tg.tcsc_bytes_for(1024, 1024, 1024 * 512))
    assert abs(oi - 12.77) < 0.01
    assert oi == 33_619_968 / 2_633_736
    assert tg.tcsc_bytes_for(4, 2, 4) == 40
    assert tg.tcsc_bytes_for(1024, 1024, 524_288) == 2_105_352
    with pytest.raises(tg.ParameterError):
        tg.tcsc_bytes_for(2, 2, 5)


def test_block_size_resolution():
    assert tg.resolve_block_size(None, 100) == 100
    assert tg.resolve_block_size(None, 10_000) == 4096
    assert tg.resolve_block_size(7, 100) == 7
    with pytest.raises(tg.ParameterError):
        tg.resolve_block_size(0, 5)


def test_workload_recipe_pins():
    # cfg1 generator pin (seed 1)
    import hashlib

    W, X, b = make_inputs("cfg1")
    h = lambda a: hashlib.sha256(a.tobytes()).hexdigest()[:16]  # noqa: E731
    assert (h(W), h(X), h(b)) == ("056a3b1eb0c433eb", "3d06f7c898896916", "3af6b41d0defe22c")
    assert int(np.count_nonzero(W)) == 131163
    assert ops(64, 512, 131163) == 64 * 512 + 64 * 131163
    rows = cfg5_oracle_rows()
    assert rows.shape == (256,) and np.all(np.diff(rows) > 0) and rows.max() < 8192
    assert set(WORKLOADS) >= {"cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "cfg3_s1_16", "cfg3_s1_8", "cfg3_s1_4"}
    assert WORKLOADS["cfg3_s1_16"].p_pos == float(Fraction(1, 32))
    assert algorithmic_bytes(256, 4096, 4096, 8_388_608) == 4 * (2 * 4097 + 8_388_608) + 4 * 256 * 4096 * 2 + 4 * 4096


def test_integer_twin_keeps_w():
    W, X, b = make_inputs("cfg1")
    Wi, Xi, bi = make_inputs("cfg1", integer=True)
    assert np.array_equal(W, Wi)
    assert np.all(Xi == np.round(Xi)) and np.abs(Xi).max() <= 8


def test_host_types_validate_like_reference():
    with pytest.raises(tg.ParameterError, match=r"entry \(0, 1\) = 2 is not in"):
        tg.TernaryDense(np.array([[0, 2]]))
    with pytest.raises(tg.ParameterError):
        tg.TernaryDense(np.zeros((0, 3)))
    with pytest.raises(tg.ParameterError):
        tg.DenseMatrix(np.array([1.0, 2.0]))
    with pytest.raises(tg.ParameterError):
        tg.BiasVector(np.array([np.inf], np.float32))
    with pytest.raises(tg.ParameterError):
        tg.PaddedInput(np.ones((2, 3), np.float32))
    p = tg.PaddedInput(np.array([[1.0, 2.0, 0.0]], np.float32))
    assert (p.M, p.K) == (1, 2)
    w = tg.TernaryDense(np.array([[1, 0], [0, -1], [-1, 0], [1, 0]]))
    assert (w.K, w.N, w.nnz) == (4, 2, 4)
    assert tg.prelu(np.array([-2.0, 3.0], np.float32), 0.25).tolist() == [-0.5, 3.0]


def test_formats_structural_checks_on_host():
    with pytest.raises(tg.ParameterError):
        tg.Tcsc(4, 2, [0, 1], [0], [0, 0, 0], [])
    with pytest.raises(tg.ParameterError):
        tg.BlockedTcsc(4, 2, 2, np.zeros((1, 3)), [], np.zeros((2, 3)), [])
    with pytest.raises(tg.ParameterError):
        tg.InterleavedBlockedTcsc(4, 2, 4, 2, [], np.zeros(3))
    with pytest.raises(tg.ParameterError):
        tg.InterleavedBlockedTcsc(4, 2, 4, 2, [], np.zeros(7), symmetric_groups=True)
    t = tg.InterleavedBlockedTcsc(4, 2, 4, 1, [0, 2, 3, 1], [0, 2, 3, 3, 3, 3, 4])
    assert t.format_bytes() == 4 * (4 + 7) and t.num_blocks == 1 and t.nnz == 4
    assert tg.format_bytes(t) == 44
    with pytest.raises(tg.ParameterError):
        tg.format_bytes(object())


def _header_functions() -> list[str]:
    src = open(os.path.join(ROOT, "include", "terngemm_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return re.findall(r"^\s*(?:int|size_t|const char\*)\s+(tg_\w+)\s*\(", src, flags=re.M)


def test_c_abi_library_exports_every_declared_symbol():
    names = _header_functions()
    assert len(names) >= 20
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built")
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_native.SIGNATURES), set(names) ^ set(_native.SIGNATURES)
    L = _native.load()
    assert L.tg_abi_version() == 5
    # pure size queries need no device
    assert L.tg_tiles_bytes(4096, 4096) == 2 * 32 * 4096 * 8 * 4  # tile records + the row-major plane
    assert L.tg_build_workspace_bytes(4096, 4096, 4096) > 0
    assert L.tg_gemm_workspace_bytes(256, 4096, 4096) >= 3 * 256 * 4096


def test_compute_entry_points_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        tg.tcsc_from_dense(np.zeros((2, 2), np.int8))


def test_bench_arms_describe_the_same_workload():
    """Both bench arms print config_dict(...) (the driver compares the two lines' `config`), the
    default workload is the largest BASELINE config, and --x-outliers scales the same seeded
    channels in either arm."""
    import bench

    assert bench.DEFAULT_CONFIG == "cfg5"
    a, b = bench.config_dict("cfg5", 123), bench.config_dict("cfg5", 123)
    assert a == b and a["workload"] == "cfg5" and (a["M"], a["K"], a["N"]) == (8192, 8192, 16384)
    assert "x_outliers" not in a
    o = bench.config_dict("cfg4", 7, "8@100")
    assert o["x_outliers"].startswith("8@100") and o["workload"] == "cfg4"
    assert bench.parse_outliers(None) is None and bench.parse_outliers("8@100") == (8, 100.0)
    W0, X0, b0 = bench.bench_inputs("cfg1")
    W1, X1, b1 = bench.bench_inputs("cfg1", "3@50")
    W2, X2, b2 = bench.bench_inputs("cfg1", "3@50")
    assert np.array_equal(W0, W1) and np.array_equal(b0, b1) and np.array_equal(X1, X2)
    ch = np.flatnonzero((X1 != X0).any(axis=0))
    assert len(ch) == 3 and np.array_equal(X1[:, ch], X0[:, ch] * np.float32(50.0))
    # the integer-valued twin (dense.py:143-160) is never scaled: it must stay exact
    _, Xi, _ = bench.bench_inputs("cfg1", "3@50", integer=True)
    assert np.array_equal(Xi, bench.make_inputs("cfg1", integer=True)[1])
