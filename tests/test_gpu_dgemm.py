"""The batched FP64 tensor-core GEMM of the SAI setup (ldgmg_dgemm_nt_batched,
csrc/dgemm_batched.cu: mma.sync m8n8k4 DMMA) against a PyTorch float64
reference of the same product.  Floating point: the summation order differs
from the reference's, so the bar is a tolerance relative to sum |a||b|."""
import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def run(ctx, M, N, K, batch, lda, ldb, ldd, alpha, beta, seed):
    from paper_2412_12506_b200 import _lib as L
    g = torch.Generator().manual_seed(seed)
    sA, sB, sD = M * lda + 3, N * ldb + 5, N * ldd + 1  # odd strides: unaligned operands
    A = torch.rand(batch * sA, generator=g, dtype=torch.float64) * 2 - 1
    B = torch.rand(batch * sB, generator=g, dtype=torch.float64) * 2 - 1
    D = torch.rand(batch * sD, generator=g, dtype=torch.float64) * 2 - 1
    want = D.clone()
    absb = torch.zeros_like(D)
    for b in range(batch):
        Ab = A[b * sA:b * sA + M * lda].view(M, lda)[:, :K]
        Bb = B[b * sB:b * sB + N * ldb].view(N, ldb)[:, :K]
        Db = want[b * sD:b * sD + N * ldd].view(N, ldd)[:, :M]  # D^T view (column-major D)
        Db.copy_(alpha * (Bb @ Ab.T) + beta * Db)
        absb[b * sD:b * sD + N * ldd].view(N, ldd)[:, :M].copy_(abs(alpha) * (Bb.abs() @ Ab.abs().T) + abs(beta))
    Ad, Bd, Dd = A.cuda(), B.cuda(), D.cuda()
    L.check(L.lib.ldgmg_dgemm_nt_batched(ctx.h, M, N, K, alpha, Ad.data_ptr(), lda, sA, Bd.data_ptr(), ldb, sB, beta,
                                         Dd.data_ptr(), ldd, sD, batch))
    torch.cuda.synchronize()
    got = Dd.cpu()
    err = (got - want).abs()
    assert torch.all(err <= 1e-13 * (absb + 1.0)), float(err.max())
    # entries outside the M x N window are untouched
    for b in range(batch):
        pad = got[b * sD:b * sD + N * ldd].view(N, ldd)[:, M:]
        assert torch.equal(pad, D[b * sD:b * sD + N * ldd].view(N, ldd)[:, M:])


@pytest.mark.parametrize("M,N,K,batch,alpha,beta", [
    (64, 64, 16, 1, 1.0, 0.0),        # one tile, one K step
    (64, 811, 2700, 3, 1.0, 0.0),     # Y = V^T C at the C5 level-0 shape
    (2700, 811, 64, 2, -1.0, 1.0),    # C -= V Z
    (64, 64, 3348, 2, 1.0, 0.0),      # Gram matrix of a wide panel
    (37, 53, 29, 5, 0.5, -2.0),       # ragged everything
    (8, 8, 0, 2, 1.0, 1.0),           # K = 0: D = beta D
    (129, 1, 77, 1, 1.0, 0.0),
])
def test_dgemm_nt_batched_matches_torch(ctx, M, N, K, batch, alpha, beta):
    run(ctx, M, N, K, batch, K + 1, K + 3, M + 2, alpha, beta, seed=M * 7 + N)
