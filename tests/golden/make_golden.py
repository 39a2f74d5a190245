"""Generates the golden fixtures from the reference itself (oracle/_ref, the
unmodified reference headers built against oracle/shim).  Run here, where
/root/reference exists:   python tests/golden/make_golden.py
Each fixture is a small .npz: inputs, the reference's outputs, and the level
data the numpy port needs -- so the port (oracle/port.py) can be checked
against the reference even where oracle/_ref is absent."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402
from tests import cases as K  # noqa: E402

FIXTURES = {
    "jacobi_scalar2d_periodic_p2": (K.scalar(4, 2, K.P, degree=2), K.cfg("jacobi", omega=0.7, nu=2)),
    "gs_scalar2d_dirichlet_p1": (K.scalar(4, 2, K.D, degree=1, mu=1.3), K.cfg("gs", nu=2)),
    "sai1_scalar2d_dirichlet_p2": (K.scalar(4, 2, K.D, degree=2), K.cfg("sai", level=1, nu=2)),
    "sai1_stokes2d_stress_p1": (K.stokes(4, 2, K.P, gamma=1.0, degree=1), K.cfg("sai", level=1, zeta=0.13, nu=1)),
    "sai1_scalar3d_periodic_p1": (K.scalar(4, 3, K.P, degree=1), K.cfg("sai", level=1, nu=1)),
}


def main():
    for name, (spec, cfg) in FIXTURES.items():
        R = ref.RefMultigrid(spec, cfg)
        n, bs, _ = R.shape(0)
        rng = np.random.default_rng(7)
        b = rng.uniform(-1, 1, n * bs)
        x0 = rng.uniform(-1, 1, n * bs)
        out = {"depth": R.depth, "dim": R.dim, "n_comp": R.n_comp, "bs_scalar": R.bs_scalar,
               "kernel_constants": R.kernel_constants, "kernel_pressure": R.kernel_pressure,
               "smoother": cfg.smoother.kind, "omega": cfg.smoother.omega, "nu1": cfg.nu1, "nu2": cfg.nu2,
               "pre": cfg.pre, "post": cfg.post, "bottom_tol": cfg.bottom_tol, "b": b, "x0": x0,
               "injection": R.injection()}
        for l in range(R.depth):
            ptr, col, val = R.matrix(l)
            out[f"A{l}_ptr"], out[f"A{l}_col"], out[f"A{l}_val"] = ptr, col, val
            if l + 1 < R.depth:
                out[f"T{l}_parent"], out[f"T{l}_orth"] = R.transfer(l)
                if cfg.smoother.kind == 3:
                    out[f"B{l}_ptr"], out[f"B{l}_col"], out[f"B{l}_val"] = R.sai_matrix(l)
                else:
                    out[f"F{l}_V"], out[f"F{l}_lam"], out[f"F{l}_s"] = R.diag_factors(l)
                    if cfg.smoother.kind == 1:
                        out[f"C{l}"] = R.colours(l)[0]
        out["bottom_V"], out["bottom_lam"] = R.bottom()
        # reference outputs
        out["want_spmv"] = R.spmv(0, x0)
        out["want_spmv_t"] = R.spmv(0, x0, transpose=True)
        out["want_smooth_fwd"] = R.smoother_apply(0, b, x0, 0)
        out["want_smooth_rev"] = R.smoother_apply(0, b, x0, 1)
        out["want_restrict"] = R.restrict(0, x0)
        xc = rng.uniform(-1, 1, R.shape(1)[0] * bs)
        out["xc"] = xc
        out["want_interp"] = R.interpolate_add(0, xc, x0)
        out["want_cycle"] = R.cycle(x0, b)
        out["want_apply"] = R.apply(b)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        print("wrote", name, os.path.getsize(os.path.join(HERE, name + ".npz")), "bytes")


if __name__ == "__main__":
    main()
