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
and bottom eigenpairs by the GPU eigensolvers) are per config, set from the
measured deviations (BARS below): the same cycle and GMRES
iteration counts everywhere; for the converging configs the history within
`hist` in relres units (1e-12 = 1e-12 ||b|| in the residual for C1/C2) and
x within `x`; for the configs whose stationary V-cycle DIVERGES in the
reference too (the curved-interface extension A2: C3 ball, C4 ellipse, C5
sphere) every h_k within `hist_rel` * h_k -- the iterates grow like rho^k,
so differences are only meaningful relative to h_k; GMRES residuals within
`eta` * r_0.
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
# Per-config bars, set from the measured deviations (tools/fullsize_parity_report.py,
# profiles/r02/fullsize_parity.jsonl) with ~3x margin:
#   hist: max_k |h_k - h_k^ref| (relres units = ||r|| / ||b||)   [converging]
#   hist_rel: max_k |h_k - h_k^ref| / h_k^ref                     [diverging, A2]
#   x: | ||x|| - ||x_ref|| | / ||x_ref|| and the projections / ||proj_ref||
#   eta: max_k |r_k - r_k^ref| / r_0^ref of the GMRES residuals
BARS = {  # measured (profiles/r02/fullsize_parity.jsonl) -> bar
    "C1": dict(hist=1e-12, x=1e-10, eta=1e-12),            # 4.9e-15, 3.5e-14, 2.3e-14
    "C2": dict(hist=1e-12, x=1e-10, eta=1e-12),            # 7.3e-16, 5.6e-15, 1.7e-14
    "C3-box-GS": dict(hist=3e-9, x=1.5e-8, eta=2e-10),     # 9.2e-10, 4.1e-9, 5.1e-11
    # x: 1.3e-10 with round 2a's QR panel, 3.0e-9 with round 2b's -- the two
    # SAI builds differ from LAPACK's by the same 7e-15 (test_gpu_sai), the 1e4
    # contrast amplifies it: the same bar as the GS smoother's factors get
    "C3-box-SAI": dict(hist=1e-9, x=1.5e-8, eta=5e-9),     # 3.1e-10, 3.0e-9, 1.7e-9
    "C3-ball-GS": dict(hist_rel=1e-10),                    # 2.6e-12 (x 9.6e-13)
    "C3-ball-SAI": dict(hist_rel=1e-10),                   # 1.3e-12 (x 1.5e-12)
    "C4": dict(hist_rel=1e-10),                            # 4.4e-13 (x 1.4e-13)
    "C5-16": dict(hist_rel=1e-10),                         # 1.2e-13 (x 2.5e-13)
}


def projections(x, k=8, seed=123):
    rng = np.random.default_rng(seed)
    return np.array([float(np.dot(rng.standard_normal(x.size), x)) for _ in range(k)])


def measure(ctx, name, want):
    """Product setup + solve at full size; deviations from the reference fixture."""
    spec, cfg, normal, budget = K.fullsize_configs()[name]
    P = g.Problem(spec, min_depth=cfg.min_depth, bottom_max_elements=cfg.bottom_max_elements, device_assembly=True)
    mg = g.Multigrid(ctx, cfg, P)
    n, bs = mg.n, mg.bs
    out = {"shape_ok": (n, bs, P.depth) == (int(want["n"]), int(want["bs"]), int(want["depth"]))}
    b = K.baseline_rhs(n, bs, spec.kind, P.dim, P.bs_scalar, P.kernel_constants, P.kernel_pressure, normal=normal,
                       random_rhs=g.random_rhs)
    out["rhs_identical"] = float(np.sum(b)) == float(want["b_sha_sum"])
    x, hist, its = mg.solve_host(b, tol=1e-10, maxit=budget)
    h_ref = want["history"]
    out.update(iterations=int(its), iterations_ref=int(want["iterations"]))
    if hist.shape == h_ref.shape:
        dev = np.abs(hist - h_ref)
        out["hist"] = float(dev.max())
        out["hist_rel"] = float(np.max(dev / np.maximum(h_ref, 1e-300)))
    xr = float(want["xnorm"])
    out["x"] = max(abs(float(np.linalg.norm(x)) - xr) / xr,
                   float(np.max(np.abs(projections(x) - want["proj"])) / np.linalg.norm(want["proj"])))
    out["final_relres"] = float(hist[-1])
    if "eta_residuals" in want.files:
        rep = mg.estimate_eta(g._lib.KRYLOV_GMRES, seed=0, tol=1e-12, maxit=60)
        rw = want["eta_residuals"]
        out.update(eta_iterations=int(rep["iterations"]), eta_iterations_ref=int(want["eta_iterations"]))
        if rep["residuals"].shape == rw.shape:
            out["eta"] = float(np.max(np.abs(rep["residuals"] - rw)) / rw[0])
    return out


@pytest.mark.parametrize("name", list(BARS))
def test_product_route_matches_reference_history(ctx, name):
    want = np.load(os.path.join(HIST, f"{name}.npz"))
    m = measure(ctx, name, want)
    bar = BARS[name]
    assert m["shape_ok"] and m["rhs_identical"], m
    assert m["iterations"] == m["iterations_ref"], m
    if name in CONVERGING:
        assert m["hist"] <= bar["hist"] and m["x"] <= bar["x"], m
    else:
        assert m["hist_rel"] <= bar["hist_rel"], m
    if "eta" in bar:
        assert m["eta_iterations"] == m["eta_iterations_ref"] and m["eta"] <= bar["eta"], m


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


def test_c5_bottom_pinv_matches_oracle_sym_eig(ctx, ref):
    """The C5 48^3 bottom (3^3 elements x 108 = 2,916 unknowns, the size the
    device eigensolver is used for) -- built here from C5 at 24^3, whose
    hierarchy 24 -> 12 -> 6 -> 3 ends in the same 3^3 bottom -- applied as
    the pseudoinverse (multigrid.hpp:249-253, cutoff 1e-10 max|lambda|) on
    the GPU (cuSOLVER dsyevd eigenpairs) and from the oracle's sym_eig
    (blockla.hpp:318-326, LAPACK dsyevd through the shim) on the same dense
    operator: the same kept spectrum, and the same action to within the
    accuracy two backward-stable eigensolvers can agree on, 64 eps kappa
    with kappa = max|lambda| / min kept |lambda| (this operator: kappa ~ 1e7,
    measured gap 5.2e-9 relative)."""
    spec, cfg, _, _ = K.fullsize_configs()["C5-16"]
    spec.n = 24
    P = g.Problem(spec, min_depth=cfg.min_depth, bottom_max_elements=cfg.bottom_max_elements, any_n=True)
    lb = P.depth - 1
    nb, bs, _ = P.level_shape(lb)
    assert nb == 27 and nb * bs == 2916
    ptr, col, val = P.level_matrix(lb)
    n = nb * bs
    D = np.zeros((n, n))
    for i in range(nb):
        for k in range(ptr[i], ptr[i + 1]):
            D[i * bs:(i + 1) * bs, col[k] * bs:(col[k] + 1) * bs] = val[k * bs * bs:(k + 1) * bs * bs].reshape(bs, bs)
    lam, V = ref.sym_eig(D)
    V = V.reshape(n, n, order="F")
    # GPU: a depth-1 hierarchy on the bottom operator: its v_cycle IS the bottom pseudoinverse
    A = g.DeviceBsr(ctx, nb, nb, bs, bs, ptr, col, val)
    cfg1 = K.cfg("sai", level=1, zeta=0.107, min_depth=1, bottom_max=27)
    mg = g.Multigrid(ctx, cfg1, levels=[A], transfers=[], system_kind=g.SYSTEM_STOKES, dim=3, n_comp=4,
                     bs_scalar=27, kernel_constants=False, kernel_pressure=True)
    b = np.random.default_rng(9).uniform(-1, 1, n)
    xd = torch.zeros(n, dtype=torch.float64, device="cuda")
    mg.vcycle(xd, torch.as_tensor(b).cuda())
    torch.cuda.synchronize()
    got = xd.cpu().numpy()
    cut = 1e-10 * np.max(np.abs(lam))
    inv = np.where(np.abs(lam) > cut, 1.0 / np.where(lam == 0, 1.0, lam), 0.0)
    want = V @ (inv * (V.T @ b))
    kept = np.abs(lam) > cut
    kappa = np.max(np.abs(lam)) / np.min(np.abs(lam[kept]))
    # the GPU keeps the same eigenvalues (its own dsyevd spectrum)
    lam_gpu = np.linalg.eigvalsh(D)
    assert int(np.sum(np.abs(lam_gpu) > 1e-10 * np.max(np.abs(lam_gpu)))) == int(np.sum(kept))
    bar = 64 * np.finfo(float).eps * kappa
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert rel <= bar, (rel, kappa, bar)


@pytest.mark.parametrize("name", ["C1", "C3-ball-GS", "C3-ball-SAI", "C4"])
def test_fullsize_dropin_bitwise(ctx, ref, name):
    """The BASELINE configs at their STATED sizes on the drop-in route (the
    reference's own level operators, diagonal factors / SAI matrices,
    transfers and bottom eigenpairs uploaded, strict order): two V-cycles and
    `apply` bit-identical to the reference's (multigrid.hpp:82-101) on the
    benchmark right-hand side -- C1 64^2 Jacobi, C3 256^2 (ball interface,
    extension A2) with 4-colour GS and with SAI1, C4 128^2 Stokes SAI1.  (C2 at
    32^3: test_gpu_fullsize.py; C5's physics at 8^3: above.)"""
    from tests.test_gpu_vcycle import dropin_mg
    spec, cfg, normal, _ = K.fullsize_configs()[name]
    R = ref.RefMultigrid(spec, cfg)
    n, bs, _ = R.shape(0)
    mg = dropin_mg(ctx, R, cfg)
    mg.set_strict_order(True)
    b = K.baseline_rhs(n, bs, spec.kind, R.dim, R.bs_scalar, R.kernel_constants, R.kernel_pressure, normal=normal,
                       random_rhs=ref.random_rhs)
    x = np.zeros(n * bs)
    xd = torch.as_tensor(x).cuda()
    bd = torch.as_tensor(b).cuda()
    for _ in range(2):
        mg.cycle(xd, bd)
        x = R.cycle(x, b)
        torch.cuda.synchronize()
        assert np.array_equal(xd.cpu().numpy().view(np.int64), x.view(np.int64)), name
    yd = torch.empty_like(bd)
    mg.apply(bd, yd)
    torch.cuda.synchronize()
    assert np.array_equal(yd.cpu().numpy().view(np.int64), R.apply(b).view(np.int64)), name
