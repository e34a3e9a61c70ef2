"""B200-native sparse ternary GEMM (placeholder init)."""
