"""Full-size golden histories from the reference itself (oracle/_ref).  Run
here, where /root/reference exists (C5 at 16^3 alone needs ~10 min of
reference setup):   python tests/golden/make_histories.py [names...]

Per BASELINE config (tests/cases.fullsize_configs) one small .npz under
tests/golden/histories/: the stationary solve of Multigrid::cycle from x = 0
on the benchmark right-hand side (multigrid.hpp:82-85; stopped at relres <=
1e-10 or after the config's cycle budget), its residual history and count,
||x||_2 and the projections of x on 8 fixed random vectors (default_rng(123)
normals) -- what tests/test_gpu_fullsize_parity.py compares the product's
own setup and V-cycle against.  The GMRES eta protocol (krylov.hpp:293-306)
is added for the configs whose V-cycle is cheap on the CPU."""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402
from tests import cases as K  # noqa: E402

OUT = os.path.join(HERE, "histories")
ETA = {"C1", "C2", "C3-box-GS", "C3-box-SAI"}


def projections(x, k=8, seed=123):
    rng = np.random.default_rng(seed)
    return np.array([float(np.dot(rng.standard_normal(x.size), x)) for _ in range(k)])


def main(names):
    os.makedirs(OUT, exist_ok=True)
    cfgs = K.fullsize_configs()
    for name in names or list(cfgs):
        spec, cfg, normal, budget = cfgs[name]
        t0 = time.time()
        R = ref.RefMultigrid(spec, cfg)
        t_setup = time.time() - t0
        n, bs, _ = R.shape(0)
        b = K.baseline_rhs(n, bs, spec.kind, R.dim, R.bs_scalar, R.kernel_constants, R.kernel_pressure,
                           normal=normal, random_rhs=ref.random_rhs)
        t0 = time.time()
        x, hist, its = R.solve(b, tol=1e-10, maxit=budget)
        t_solve = time.time() - t0
        out = {"name": name, "n": n, "bs": bs, "depth": R.depth, "iterations": its, "history": hist,
               "bnorm": float(np.linalg.norm(b)), "xnorm": float(np.linalg.norm(x)), "proj": projections(x),
               "b_sha_sum": float(np.sum(b)), "budget": budget, "setup_s": t_setup, "solve_s": t_solve}
        if name in ETA:
            e = R.eta(kind=1, seed=0, tol=1e-12, maxit=60)
            out.update({"eta_residuals": e["residuals"], "eta_iterations": e["iterations"], "eta": e["eta"],
                        "eta_rho": e["rho"]})
        np.savez(os.path.join(OUT, f"{name}.npz"), **out)
        print(f"{name}: setup {t_setup:.1f} s, {its} cycles in {t_solve:.1f} s, relres {hist[-1]:.3e}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
