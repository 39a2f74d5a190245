"""Pinning the oracle (CPU).

1. The reference's OWN hot-path test binaries (tests/test_{blockla,smoothers,
   multigrid,krylov}.cpp + mesh/basis/ldg_* -- compiled unmodified against
   oracle/shim by `make -C oracle reftests`) pass.  Two assertions fail
   against the reference code itself, not the shim:
   test_smoothers.cpp:570 and test_ldg_scalar.cpp:280.
2. The numpy restatement (oracle/port.py) is BIT-identical to the reference
   on the committed golden fixtures (tests/golden/*.npz, generated from
   oracle/_ref by tests/golden/make_golden.py) and live against oracle/_ref.
"""
import glob
import os
import subprocess

import numpy as np
import pytest

from oracle import port
from tests.conftest import ROOT

REFDIR = os.path.join(ROOT, "oracle", "_ref")
KNOWN_REFERENCE_FAILURES = {
    "test_smoothers": ["a singular Stokes diagonal block is rejected, a scalar one is projected"],
    "test_ldg_scalar": ["donor selection prefers the more viscous side"],
}


@pytest.mark.parametrize("name", ["test_blockla", "test_smoothers", "test_multigrid", "test_krylov",
                                  "test_mesh", "test_basis", "test_ldg_scalar", "test_ldg_stokes"])
def test_reference_suite_passes_on_the_oracle_build(name):
    exe = os.path.join(REFDIR, name)
    if not os.path.exists(exe):
        pytest.skip("reference test binaries not built (make -C oracle reftests)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600).stdout
    failed = [l.split("] ", 1)[1].split(" (")[0] for l in out.splitlines() if l.startswith("[FAIL]")]
    assert sorted(failed) == sorted(KNOWN_REFERENCE_FAILURES.get(name, [])), out[-2000:]
    assert "test cases:" in out


def load(path):
    z = dict(np.load(path))
    depth = int(z["depth"])
    levels = []
    for l in range(depth):
        ptr = z[f"A{l}_ptr"]
        L = {"n": len(ptr) - 1, "bs": int(z["bs_scalar"] * z["n_comp"]),
             "A": (ptr, z[f"A{l}_col"], z[f"A{l}_val"])}
        if f"B{l}_ptr" in z:
            L["B"] = (z[f"B{l}_ptr"], z[f"B{l}_col"], z[f"B{l}_val"])
        if f"F{l}_V" in z:
            L["factors"] = (z[f"F{l}_V"], z[f"F{l}_lam"], z[f"F{l}_s"])
        if f"C{l}" in z:
            L["colour"] = z[f"C{l}"]
        levels.append(L)
    transfers = [(z[f"T{l}_parent"], z[f"T{l}_orth"]) for l in range(depth - 1)]
    from tests import cases as K
    cfg = K.cfg()
    cfg.smoother.kind, cfg.smoother.omega = int(z["smoother"]), float(z["omega"])
    cfg.nu1, cfg.nu2, cfg.pre, cfg.post = int(z["nu1"]), int(z["nu2"]), int(z["pre"]), int(z["post"])
    cfg.bottom_tol = float(z["bottom_tol"])
    bss, nc, dim = int(z["bs_scalar"]), int(z["n_comp"]), int(z["dim"])
    offs = []
    if int(z["kernel_constants"]):
        offs += [c * bss for c in range(1 if nc == 1 else dim)]
    if int(z["kernel_pressure"]):
        offs.append(dim * bss)
    P = port.PortMultigrid(levels, transfers, z["injection"], (z["bottom_V"], z["bottom_lam"]), cfg, bss, nc, offs)
    return z, P


GOLDEN = sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "*.npz")))


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_port_bitwise_on_golden_fixtures(path):
    z, P = load(path)
    L0 = P.levels[0]
    bs = L0["bs"]
    b, x0 = z["b"], z["x0"]
    eq = np.array_equal
    assert eq(port.spmv(*L0["A"], bs, bs, x0), z["want_spmv"])
    assert eq(port.spmv_transpose(*L0["A"], bs, bs, L0["n"], x0), z["want_spmv_t"])
    assert eq(P.smooth(0, b, x0, 0), z["want_smooth_fwd"])
    assert eq(P.smooth(0, b, x0, 1), z["want_smooth_rev"])
    p, o = P.transfers[0]
    assert eq(port.restrict(p, o, P.K, P.bss, P.ncomp, P.levels[1]["n"], x0), z["want_restrict"])
    assert eq(port.interpolate_add(p, o, P.K, P.bss, P.ncomp, z["xc"], x0), z["want_interp"])
    assert eq(P.cycle(x0, b), z["want_cycle"])
    assert eq(P.apply(b), z["want_apply"])


@pytest.mark.parametrize("case", ["periodic-jacobi", "dirichlet-gs-p2", "stokes-sai", "3d-sai", "pgs3-2d", "pgs2-stokes"])
def test_port_bitwise_live_against_reference(ref, case):
    from tests import cases as K
    spec, cfg = {
        "periodic-jacobi": (K.scalar(8, 2, K.P, degree=2), K.cfg("jacobi", omega=0.8)),
        "dirichlet-gs-p2": (K.scalar(8, 2, K.D, degree=2), K.cfg("gs")),
        "stokes-sai": (K.stokes(4, 2, K.P, gamma=1.0, degree=2), K.cfg("sai", level=1, zeta=0.13)),
        "3d-sai": (K.scalar(4, 3, K.P, degree=2), K.cfg("sai", level=1)),
        "pgs3-2d": (K.scalar(8, 2, K.D, degree=1), K.cfg("pgs", partitions=3, nu=2)),
        "pgs2-stokes": (K.stokes(4, 2, K.P, degree=1), K.cfg("pgs", partitions=2, omega=0.7, nu=1,
                                                           pre=1, post=0)),
    }[case]
    R = ref.RefMultigrid(spec, cfg)
    P = port.from_reference(R, cfg)
    n, bs, _ = R.shape(0)
    rng = np.random.default_rng(11)
    b, x = rng.uniform(-1, 1, n * bs), np.zeros(n * bs)
    for _ in range(2):
        x = R.cycle(x, b)
    y = np.zeros(n * bs)
    for _ in range(2):
        y = P.cycle(y, b)
    assert np.array_equal(x, y)
    assert np.array_equal(P.apply(b), R.apply(b))
    assert np.array_equal(port.colour_mesh(*R.matrix(0)[:2]), ref.RefMultigrid(spec, K.cfg("gs")).colours(0)[0])
