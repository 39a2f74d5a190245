"""The reference's transfer pins (tests/test_multigrid.cpp:110-142) on the
GPU kernels, at test scale and at the C2 / C5 sizes: interpolation is the
exact adjoint of residual restriction (1e-13), and restricting an
interpolated field multiplies it by the child count 2^d (1e-13 * 2^d).
Both go through the K-stationary kernels on these uniform hierarchies."""
import numpy as np
import pytest

import paper_2412_12506_b200 as g
from tests import cases as K

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CASES = {
    "2d-p2-8": K.scalar(8, 2, K.P, degree=2),
    "3d-p2-4": K.scalar(4, 3, K.P, degree=2),
    "3d-p2-32-C2": K.scalar(32, 3, K.P, degree=2, beta=4.0),
    "2d-p4-256-C3": K.scalar(256, 2, K.D, degree=4, beta=16.0),
    "stokes3d-p2-16-C5": K.stokes(16, 3, K.P, gamma=0.0, degree=2, beta=4.0, beta_p=1 / 16, delta=0.01),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_restriction_adjoint_and_child_count(ctx, name):
    P = g.Problem(CASES[name], min_depth=2)
    nf, bs, _ = P.level_shape(0)
    nc = P.level_shape(1)[0]
    p, o = P.level_transfer(0)
    T = g.Transfer(ctx, nf, nc, p, o, P.dim, P.bs_scalar, P.n_comp, P.injection())
    rng = np.random.default_rng(11)
    xc = torch.as_tensor(rng.uniform(-1, 1, nc * bs)).cuda()
    yf = torch.as_tensor(rng.uniform(-1, 1, nf * bs)).cuda()
    Ix = torch.zeros(nf * bs, dtype=torch.float64, device="cuda")
    T.interpolate_add(xc, Ix)
    Ry = torch.empty(nc * bs, dtype=torch.float64, device="cuda")
    T.restrict(yf, Ry)
    a, b = float(torch.dot(Ix, yf)), float(torch.dot(xc, Ry))
    assert abs(a - b) <= 1e-13 * max(abs(a), abs(b)), (name, a, b)
    RIx = torch.empty_like(Ry)
    T.restrict(Ix, RIx)
    scale = float(1 << P.dim)
    err = float((RIx - scale * xc).abs().max())
    assert err <= 1e-13 * scale, (name, err)
