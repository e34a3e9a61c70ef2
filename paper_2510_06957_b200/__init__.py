"""B200-native sparse ternary GEMM  Y = X W + b (+ fused PReLU).

Drop-in for the hot path of the reference package ``terngemm``
(/root/reference/pkg/src/terngemm/__init__.py): the same names for the data
types, the three in-scope formats and their builders, the five in-scope
GEMM variants and the variant registry — backed by hand-written sm_100a CUDA
(csrc/) behind the C ABI in include/terngemm_b200.h.  There is no CPU path.
"""

from .dense import (
    BiasVector,
    DenseMatrix,
    TernaryDense,
    as_fraction,
    gen_bias,
    gen_input,
    gen_input_uniform,
    gen_ternary,
    oracle_gemm,
    prelu,
)
from .errors import CorruptionError, InvalidCodeError, ParameterError, ParseError, VerificationError
from .formats import (
    CODE_COUNT,
    DECODE_TABLE,
    PACK_WIDTH,
    BlockedTcsc,
    CompressedTcsc,
    InterleavedBlockedTcsc,
    SymmetricInterleavedTcsc,
    Tcsc,
    blocked_from_dense,
    compress5,
    compressed_from_dense,
    decompress5,
    symmetric_from_dense,
    format_bytes,
    interleaved_blocked_from_dense,
    resolve_block_size,
    tcsc_bytes_for,
    tcsc_from_dense,
    tcsc_to_dense,
    validate,
)
from .harness import flop_count, operational_intensity
from .kernels import (
    DEFAULT_ALPHA,
    SCALAR_TAGS,
    SIMD_TAGS,
    VARIANTS,
    GemmConfig,
    GemmRunner,
    OpCount,
    PaddedInput,
    VariantSpec,
    gemm_base,
    gemm_blocked,
    gemm_compressed,
    gemm_horizontal,
    gemm_interleaved_blocked,
    gemm_unrolled,
    gemm_vectorized_optimal,
    gemm_vertical,
    get_variant,
    pad_input,
    run_variant,
)

from . import io  # noqa: E402  (TGW1 / TGS1 files, io.py)

__version__ = "0.1.0"

__all__ = [
    "CODE_COUNT", "CompressedTcsc", "DECODE_TABLE", "PACK_WIDTH", "SymmetricInterleavedTcsc", "compress5",
    "compressed_from_dense", "decompress5", "gemm_compressed", "gemm_horizontal", "gemm_vertical",
    "symmetric_from_dense",
    "BiasVector", "BlockedTcsc", "CorruptionError", "DEFAULT_ALPHA", "DenseMatrix", "GemmConfig", "GemmRunner",
    "InterleavedBlockedTcsc", "InvalidCodeError", "OpCount", "PaddedInput", "ParameterError", "ParseError",
    "SCALAR_TAGS", "SIMD_TAGS", "Tcsc", "TernaryDense", "VARIANTS", "VariantSpec", "VerificationError",
    "blocked_from_dense", "flop_count", "format_bytes", "gemm_base", "gemm_blocked", "gemm_interleaved_blocked",
    "gemm_unrolled", "gemm_vectorized_optimal", "get_variant", "interleaved_blocked_from_dense",
    "operational_intensity", "oracle_gemm", "pad_input", "prelu", "resolve_block_size", "run_variant",
    "tcsc_bytes_for", "tcsc_from_dense", "tcsc_to_dense", "validate", "__version__",
    "as_fraction", "gen_bias", "gen_input", "gen_input_uniform", "gen_ternary", "io",
]
