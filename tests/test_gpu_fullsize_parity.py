"""Full-size parity of the PRODUCT route (the product's own setup: device
assembly, GPU diagonal factors, GPU SAI least squares, GPU bottom eig, and
its V-cycle) against the reference's solve at the BASELINE sizes.

The reference histories were produced by the reference itself (oracle/_ref)
with tests/golden/make_histories.py and committed as small fixtures
(tests/golden/histories/*.npz): the stationary solve from x = 0 on the
benchmark right-hand side (Multigrid::cycle, multigrid.hpp:82-85, until
relres <= 1e-10 or the config's cycle budget), ||x||, eight fixed random
projections of x, and for the cheap configs the GMRES eta protocol
(krylov.hpp:293-306).

Bars (floating point; the setups differ from the reference's in the last
bits: SAI least squares by the GPU's blocked QR vs LAPACK dgels, diagonal
and bottom eigenpairs by the GPU eigensolvers):
* converging configs (C1, C2, C3 with the reference-native box interface):
  same cycle count, |h_k - h_k^ref| <= 1e-12 (relres units, i.e. 1e-12 ||b||
  in the residual), ||x|| and the projections within 1e-10 relative;
* configs whose stationary V-cycle DIVERGES in the reference too (the
  curved-interface extension A2: C3 ball, C4 ellipse, C5 sphere): the same
  budget of cycles, every |h_k - h_k^ref| <= tol_rel * h_k with the
  measured-and-recorded tol_rel below -- the iterates grow
  like rho^k, so differences are only meaningful relative to h_k;
* GMRES eta: same iteration count, residuals within 1e-10 relative.
C5 here is at 16^3, the largest size the reference sets up in minutes
(~10 min of one core); 48^3 is not expressible in the reference (extension
A1).  The C5 drop-in route (the reference's own operators uploaded) is
bit-exact at 8^3 with the reference built live."""
import os

import numpy as np
import pytest

import paper_2412_12506_b200 as g
from tests import cases as K

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HIST = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "histories")
CONVERGING = {"C1", "C2", "C3-box-GS", "C3-box-SAI"}
# measured relative history deviation bounds of the diverging configs (A2)
DIVERGING_TOL = {"C3-ball-GS": 1e-9, "C3-ball-SAI": 1e-9, "C4": 1e-9, "C5-16": 1e-9}


def projections(x, k=8, seed=123):
    rng = np.random.default_rng(seed)
    return np.array([float(np.dot(rng.standard_normal(x.size), x)) for _ in range(k)])


@pytest.mark.parametrize("name", ["C1", "C2", "C3-box-GS", "C3-box-SAI", "C3-ball-GS", "C3-ball-SAI", "C4",
                                  "C5-16"])
def test_product_route_matches_reference_history(ctx, name):
    want = np.load(os.path.join(HIST, f"{name}.npz"))
    spec, cfg, normal, budget = K.fullsize_configs()[name]
    P = g.Problem(spec, min_depth=cfg.min_depth, bottom_max_elements=cfg.bottom_max_elements, device_assembly=True)
    mg = g.Multigrid(ctx, cfg, P)
    n, bs = mg.n, mg.bs
    assert (n, bs, P.depth) == (int(want["n"]), int(want["bs"]), int(want["depth"]))
    b = K.baseline_rhs(n, bs, spec.kind, P.dim, P.bs_scalar, P.kernel_constants, P.kernel_pressure, normal=normal,
                       random_rhs=g.random_rhs)
    assert float(np.sum(b)) == float(want["b_sha_sum"])  # the same right-hand side bit for bit
    x, hist, its = mg.solve_host(b, tol=1e-10, maxit=budget)
    h_ref = want["history"]
    assert its == int(want["iterations"]), (name, its, int(want["iterations"]))
    dev = np.abs(hist - h_ref)
    if name in CONVERGING:
        assert dev.max() <= 1e-12, (name, float(dev.max()))
        xn, xr = float(np.linalg.norm(x)), float(want["xnorm"])
        assert abs(xn - xr) <= 1e-10 * xr, (name, xn, xr)
        pr, pw = projections(x), want["proj"]
        assert np.all(np.abs(pr - pw) <= 1e-10 * np.linalg.norm(pw)), (name, np.abs(pr - pw).max())
    else:
        rel = float(np.max(dev / np.maximum(h_ref, 1e-300)))
        assert rel <= DIVERGING_TOL[name], (name, rel)
    if "eta_residuals" in want.files:
        rep = mg.estimate_eta(g._lib.KRYLOV_GMRES, seed=0, tol=1e-12, maxit=60)
        assert rep["iterations"] == int(want["eta_iterations"]), name
        r, rw = rep["residuals"], want["eta_residuals"]
        assert r.shape == rw.shape and np.all(np.abs(r - rw) <= 1e-10 * np.abs(rw)), (name, np.abs(r - rw).max())


def test_c5_dropin_bitwise_8cubed(ctx, ref):
    """C5's physics at 8^3 (unsteady Stokes, sphere, bs 108, balanced SAI1) on
    the drop-in route: the reference's own operators, SAI matrices,
    transfers and bottom eigenpairs uploaded, strict order -> V-cycles and
    apply bit-identical to the reference (setup ~1-2 min of reference CPU)."""
    from tests.test_gpu_vcycle import dropin_mg
    spec, cfg, _, _ = K.fullsize_configs()["C5-16"]
    spec.n = 8
    R = ref.RefMultigrid(spec, cfg)
    n, bs, _ = R.shape(0)
    assert bs == 108 and R.depth == 3
    mg = dropin_mg(ctx, R, cfg)
    mg.set_strict_order(True)
    b = K.baseline_rhs(n, bs, spec.kind, R.dim, R.bs_scalar, R.kernel_constants, R.kernel_pressure,
                       random_rhs=ref.random_rhs)
    x = np.zeros(n * bs)
    xd = torch.as_tensor(x).cuda()
    bd = torch.as_tensor(b).cuda()
    for _ in range(2):
        mg.cycle(xd, bd)
        x = R.cycle(x, b)
        torch.cuda.synchronize()
        assert np.array_equal(xd.cpu().numpy().view(np.int64), x.view(np.int64))
    yd = torch.empty_like(bd)
    mg.apply(bd, yd)
    torch.cuda.synchronize()
    assert np.array_equal(yd.cpu().numpy().view(np.int64), R.apply(b).view(np.int64))
