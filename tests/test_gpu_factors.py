"""GPU diagonal-factor setup (factors.cu: factor_diagonal, smoothers.hpp:464-494,
for every element in one launch) against the reference's Eigen-based factors
(oracle/_ref).

Bitwise: the power-of-two equilibration s.  To tolerance (different
eigensolver, same eigenpairs): eigenvalues within 1e-13 max|lambda|, the
block pseudoinverse V diag(1/lambda, cut) V^T within 1e-11 relative, and
relax sweeps built on the GPU factors within 1e-12 of the reference's.
"""
import numpy as np
import pytest

import paper_2412_12506_b200 as g
from tests import cases as K
from tests.test_gpu_kernels import SYSTEMS, dev, host, level_system, rand

pytestmark = pytest.mark.gpu


def _pinv_blocks(V, lam, bs, tol=1e-12):
    V = V.reshape(-1, bs, bs)  # [e, k, i] = V(i, k): eigenvector k
    lam = lam.reshape(-1, bs)
    out = np.empty((len(lam), bs, bs))
    for e in range(len(lam)):
        L = lam[e]
        cut = np.abs(L) <= tol * np.max(np.abs(L))
        inv = np.where(cut, 0.0, 1.0 / np.where(cut, 1.0, L))
        Ve = V[e].T
        out[e] = (Ve * inv) @ Ve.T
    return out


@pytest.mark.parametrize("name", sorted(SYSTEMS))
def test_gpu_factors_match_reference(ctx, ref, name):
    R, _ = level_system(ref, SYSTEMS[name], "jacobi")
    n, bs, _ = R.shape(0)
    A = g.DeviceBsr(ctx, n, n, bs, bs, *R.matrix(0))
    S = g.Smoother(ctx, A, g.SmootherConfig.jacobi(0.8))  # factors computed on the GPU
    V, lam, s = S.diag_factors()
    Vr, lamr, sr = R.diag_factors(0)
    assert np.array_equal(s, sr)
    lmax = np.max(np.abs(lamr.reshape(n, bs)), axis=1, keepdims=True)
    assert np.all(np.abs(lam.reshape(n, bs) - lamr.reshape(n, bs)) <= 1e-13 * lmax)
    assert np.all(np.diff(lam.reshape(n, bs), axis=1) >= 0)  # ascending, like Eigen
    # orthonormal eigenvectors
    Vb = V.reshape(n, bs, bs)
    err = np.abs(np.einsum("eki,eli->ekl", Vb, Vb) - np.eye(bs)).max()
    assert err <= 1e-13 * bs
    P, Pr = _pinv_blocks(V, lam, bs), _pinv_blocks(Vr, lamr, bs)
    scale = np.abs(Pr).max(axis=(1, 2), keepdims=True)
    assert np.all(np.abs(P - Pr) <= 1e-11 * scale)


@pytest.mark.parametrize("name", ["scalar2d-p3-C1", "scalar3d-p2-C2", "stokes2d-stress-p1", "stokes2d-p3-C4"])
def test_relax_on_gpu_factors(ctx, ref, name):
    R, _ = level_system(ref, SYSTEMS[name], "gs")
    n, bs, _ = R.shape(0)
    A = g.DeviceBsr(ctx, n, n, bs, bs, *R.matrix(0))
    S = g.Smoother(ctx, A, g.SmootherConfig.coloured_gs())
    b, x = rand(n * bs, 3), rand(n * bs, 4)
    xd = dev(x)
    for sweep in (g.SWEEP_FORWARD, g.SWEEP_REVERSE):
        S.apply(dev(b), xd, sweep)
        x = R.smoother_apply(0, b, x, sweep)
        got = host(xd)
        assert np.linalg.norm(got - x) <= 1e-12 * np.linalg.norm(x)


def test_gpu_factors_reject_nonsymmetric_block(ctx):
    bs = 3
    blk = np.arange(1.0, 10.0)  # row-major, not symmetric
    A = g.DeviceBsr(ctx, 1, 1, bs, bs, np.array([0, 1]), np.array([0]), blk)
    with pytest.raises(g.InvalidArgument, match="not symmetric"):
        g.Smoother(ctx, A, g.SmootherConfig.jacobi())


def test_gpu_factors_standalone_vcycle(ctx, ref):
    """Multigrid from the built-in setup (GPU factors on every level) keeps
    the reference residual history to 1e-12 (north_star tolerance)."""
    spec, cfg = K.scalar(16, 2, K.D, degree=2), K.cfg("gs")
    R = ref.RefMultigrid(spec, cfg)
    mg = g.Multigrid(ctx, cfg, g.Problem(spec))
    n, bs, _ = R.shape(0)
    b = rand(n * bs, 5)
    x, xd = np.zeros(n * bs), dev(np.zeros(n * bs))
    bd = dev(b)
    for _ in range(4):
        mg.cycle(xd, bd)
        x = R.cycle(x, b)
        got = host(xd)
        assert np.linalg.norm(got - x) <= 1e-11 * np.linalg.norm(x)
