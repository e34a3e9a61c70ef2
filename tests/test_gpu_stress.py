"""GPU stress: many units per CTA, long K and busy epilogues together.

The packed-W ring of the tensor-core kernel (csrc/tg_mma.cu, decoder warps) used to release a
slot right after ISSUING its shared-memory loads; with the load/store pipe busy (outlier rows
make the epilogue warps look up W codes while the next unit's tiles are decoded) the release
overtook loads still in flight, the producer refilled the slot, and single columns of a tile
came out wrong, differently on every run.  Needs several units per CTA and K >= 8192 to show;
no BASELINE config had both plus outlier rows.  Checked here: exact (integer-valued X, the
reference's regime dense.py:17-19) against an fp64 product, and bit-identical over repeats.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tg():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2510_06957_b200 as m

    return m


@pytest.mark.parametrize("M,K,N", [(8192, 8192, 1024), (1024, 8192, 8192)])
def test_many_units_long_k_with_outlier_rows_is_exact_and_repeatable(tg, M, K, N):
    rng = np.random.default_rng(M + N)
    u = rng.random((K, N))
    W = np.where(u < 0.25, 1, np.where(u < 0.5, -1, 0)).astype(np.int8)
    X = rng.integers(-8, 9, size=(M, K)).astype(np.float32)
    ch = rng.choice(K, 8, replace=False)
    X[:, ch] = rng.integers(1000, 4000, size=(M, 8)).astype(np.float32)  # every row sheds 8 entries
    b = rng.integers(-4, 5, size=N).astype(np.float32)
    t = tg.interleaved_blocked_from_dense(W)
    dX = torch.from_numpy(X).cuda()
    ref = (dX.double() @ torch.from_numpy(W).cuda().double() + torch.from_numpy(b).cuda().double()).float()
    first = None
    for rep in range(6):
        y = tg.gemm_interleaved_blocked(tg.DenseMatrix(dX), t, b, method="mma").device_values
        assert torch.equal(y, ref), (rep, int((y != ref).sum()))
        first = y.clone() if first is None else first
        assert torch.equal(y, first), rep
