"""The reference's OWN acceptance tests, run with the B200 backends substituted.

The reference package (terngemm) and its test modules are installed into
baseline/_ref by baseline/install_ref.sh (the one offline install; git-ignored,
travels to the GPU box).  This module applies INTEGRATION.md's maintainer patch
-- the existing registry tags keep their names and kinds but get this package's
``build``/``prepare``/``run`` (kernels/__init__.py:66-230) -- and, because the
acceptance tests also call the module-level entry points directly
(``tg.gemm_base(...)``, ``tg.tcsc_from_dense(...)``), rebinds those names on the
reference module to this package's functions.  The reference's own assertions
then run unchanged: c1/c2 bit-exact against ITS fp64 ``oracle_gemm`` (integer X,
pkg/tests/test_acceptance.py:39-118), c3 format round trips (:121-163), c4 the
cost model (:166-205), c5 symmetric invariants and dummy-slot liveness
(:208-266), c6 the operation counters (:269-292).  c7 is a CPU timing
observation of the reference (never asserted) and is not run.

Out-of-scope names (the Interleaved and Inverted formats, the generators, the
fp64 oracle) stay the reference's.  Skipped, with the reason, when baseline/_ref
is absent or not importable.
"""

from __future__ import annotations

import dataclasses
import importlib.util
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF_DIR, "_reference_tests", "test_acceptance.py")

pytestmark = pytest.mark.gpu

# module-level names rebound on the reference module (in scope: SURVEY.md 8(a), 8(f))
SUBSTITUTED = (
    "tcsc_from_dense", "blocked_from_dense", "interleaved_blocked_from_dense",
    "symmetric_from_dense", "compressed_from_dense", "pad_input", "gemm_base", "gemm_unrolled",
    "gemm_blocked", "gemm_interleaved_blocked", "gemm_compressed", "gemm_vertical", "gemm_horizontal",
    "gemm_vectorized_optimal", "flop_count", "operational_intensity", "compress5", "decompress5",
    "InvalidCodeError",
)
# registry tags whose build/prepare/run are substituted
PATCHED_TAGS = ("base", "unrolled", "blocked", "interleaved_blocked", "compressed", "vertical", "horizontal",
                "vectorized_optimal")


@pytest.fixture(scope="module")
def acceptance():
    if not os.path.exists(REF_TESTS):
        pytest.skip("reference not installed in baseline/_ref (run baseline/install_ref.sh)")
    if REF_DIR not in sys.path:
        sys.path.append(REF_DIR)
    try:
        import terngemm as ref
        import terngemm.kernels as ref_kernels
    except Exception as exc:  # noqa: BLE001
        pytest.skip(f"reference package not importable here: {exc}")
    import paper_2510_06957_b200 as b200

    saved_names = {n: getattr(ref, n) for n in SUBSTITUTED if hasattr(ref, n)}
    saved_specs = {t: ref_kernels.VARIANTS[t] for t in PATCHED_TAGS}
    # the maintainer patch of INTEGRATION.md: same tags, B200 build/prepare/run
    for tag in PATCHED_TAGS:
        ref_kernels.VARIANTS[tag] = dataclasses.replace(
            ref_kernels.VARIANTS[tag], build=b200.VARIANTS[tag].build, prepare=b200.VARIANTS[tag].prepare,
            run=b200.VARIANTS[tag].run)
    for n in saved_names:
        setattr(ref, n, getattr(b200, n))
    spec = importlib.util.spec_from_file_location("_ref_test_acceptance", REF_TESTS)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    try:
        yield mod
    finally:
        for n, v in saved_names.items():
            setattr(ref, n, v)
        for t, s in saved_specs.items():
            ref_kernels.VARIANTS[t] = s


def test_patch_is_in_effect(acceptance):
    import terngemm as ref
    import terngemm.kernels as ref_kernels

    import paper_2510_06957_b200 as b200

    assert ref.gemm_base is b200.gemm_base
    assert ref_kernels.VARIANTS["vectorized_optimal"].run is b200.VARIANTS["vectorized_optimal"].run
    # tags are substituted, never added (test_cli.py:71-74 counts VARIANTS)
    assert list(ref_kernels.VARIANTS) == ["base", "unrolled", "blocked", "interleaved_blocked", "inverted",
                                          "compressed", "vertical", "horizontal", "vectorized_optimal"]
    w, x, b = (ref.gen_ternary(48, 16, "1/2", 9), ref.gen_input(3, 48, 10), ref.gen_bias(16, 11))
    y = ref.run_variant("vectorized_optimal", x, w, b)
    assert type(y).__module__.startswith("paper_2510_06957_b200")


@pytest.mark.parametrize("name", ["test_c1_scalar_kernels_match_oracle_bitwise",
                                  "test_c2_vectorized_kernels_match_oracle_bitwise",
                                  "test_c3_every_format_round_trips",
                                  "test_c4_cost_model_and_operational_intensity",
                                  "test_c5_symmetric_stream_invariants_and_dummy_sensitivity",
                                  "test_c6_operation_counters_are_exact"])
def test_reference_acceptance(acceptance, name):
    getattr(acceptance, name)()
