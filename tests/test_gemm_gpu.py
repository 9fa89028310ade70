"""FP64 DMMA GEMM (tgb_dgemm) against numpy, all transpose combinations and
ragged sizes (the dense building block of the reduction/TEI rows)."""
import ctypes as C

import numpy as np
import pytest

from paper_1504_06289_b200 import lib
from paper_1504_06289_b200._lib import check

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ta", [0, 1])
@pytest.mark.parametrize("tb", [0, 1])
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (17, 9, 5), (64, 64, 16), (130, 70, 33), (257, 129, 1000)])
def test_dgemm_vs_numpy(ctx, ta, tb, M, N, K):
    import torch

    rng = np.random.default_rng(M * 1000 + N * 10 + K)
    A = rng.standard_normal((K, M) if ta else (M, K))
    B = rng.standard_normal((N, K) if tb else (K, N))
    C0 = rng.standard_normal((M, N))
    dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()  # column-major storage
    dB = torch.from_numpy(np.ascontiguousarray(B.T)).cuda()
    dC = torch.from_numpy(np.ascontiguousarray(C0.T)).cuda()
    lda, ldb = A.shape[0], B.shape[0]
    check(lib().tgb_dgemm(ctx.handle, ta, tb, M, N, K, 0.5, dA.data_ptr(), lda, dB.data_ptr(), ldb, -2.0,
                          dC.data_ptr(), M))
    ctx.synchronize()
    got = dC.cpu().numpy().T
    ref = 0.5 * ((A.T if ta else A) @ (B.T if tb else B)) - 2.0 * C0
    assert np.abs(got - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max()) * np.sqrt(K)


def test_fp64_peak_probe(ctx):
    """tgb_probe_fp64_peak: the FP64 roofline denominator bench.py takes in the same run (DFMA chains
    on every SM); a B200 sustains 30-38 TFLOP/s."""
    tf = ctx.probe_fp64_peak()
    assert 20.0 < tf < 45.0, tf
