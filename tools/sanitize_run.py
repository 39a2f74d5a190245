"""Memory-safety and determinism target: every kernel family of the product on tiny
problems -- GPU setup (device assembly, diagonal-factor eig, batched SAI
least squares incl. the rank-deficient refit, bottom eig), Jacobi / coloured
GS / processor-block GS / SAI forward + reverse sweeps (B^T as copy or view:
LDGMG_TVIEW=0/1), restriction / prolongation, bottom pseudoinverse, kernel
projection (tree and strict), the graph-captured cycle, the device-loop
solve and GMRES.  Small enough for racecheck (~100x slowdown).

  LDGMG_GUARD_BYTES=4096 python tools/sanitize_run.py   (tests/test_gpu_guards.py)

Every device allocation of the library then carries guard zones that are
checked at the end (out-of-bounds writes), and every case runs its cycles
twice, direct and graph-replayed, and must agree bit for bit (races).
compute-sanitizer itself is closed on the GPU pool this was built on.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_12506_b200 as g  # noqa: E402
from tests import cases as K  # noqa: E402


def run(ctx, spec, cfg, any_n=False, device_assembly=True, strict=False):
    P = g.Problem(spec, min_depth=cfg.min_depth, bottom_max_elements=cfg.bottom_max_elements,
                  device_assembly=device_assembly, any_n=any_n)
    mg = g.Multigrid(ctx, cfg, P)
    mg.set_strict_order(strict)
    n, bs = mg.n, mg.bs
    b = torch.as_tensor(g.random_rhs(n, bs, 1)).cuda()
    x = torch.zeros_like(b)
    mg.cycle(x, b)        # direct launches
    mg.cycles(x, b, 2)    # graph capture + replay
    # determinism (a data race shows up as run-to-run differences): the same
    # cycles from the same start, direct and graph-replayed, bit for bit
    x1, x2 = torch.zeros_like(b), torch.zeros_like(b)
    mg.cycle(x1, b)
    mg.cycle(x1, b)
    mg.cycles(x2, b, 2)
    torch.cuda.synchronize()
    assert torch.equal(x1, x2), "nondeterministic V-cycle"
    y = torch.empty_like(b)
    mg.apply(b, y)
    _, hist, its = mg.solve_host(b.cpu().numpy(), tol=0.0, maxit=2)
    xs = torch.zeros_like(b)
    mg.krylov_solve(b, xs, kind=g._lib.KRYLOV_GMRES, tol=1e-12, maxit=3)
    torch.cuda.synchronize()
    assert torch.isfinite(x).all() and torch.isfinite(y).all()
    return its


def main():
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = g.Context(0, stream=stream)
    ball = dict(phase_shape=g.PHASE_BALL, center=(0.5, 0.5, 0.5), radii=(0.3, 0.3, 0.3), mu_in=1e4, mu_out=1.0)
    sph = dict(phase_shape=g.PHASE_BALL, center=(0.5, 0.5, 0.5), radii=(0.25, 0.25, 0.25), mu_in=1e2, mu_out=1.0)
    cases = [
        ("C1 Jacobi", K.scalar(8, 2, K.P, degree=3, beta=9.0), K.cfg("jacobi", omega=0.7, nu=2), False, False),
        ("C2 SAI1", K.scalar(4, 3, K.P, degree=2, beta=4.0), K.cfg("sai", level=1, nu=2), False, True),
        ("C3 GS", K.scalar(8, 2, K.D, degree=4, beta=16.0, **ball), K.cfg("gs", nu=1), False, False),
        ("C3 PGS", K.scalar(8, 2, K.D, degree=4, beta=16.0, **ball), K.cfg("pgs", nu=1, partitions=2), False, False),
        ("C3 SAI1", K.scalar(8, 2, K.D, degree=4, beta=16.0, **ball), K.cfg("sai", level=1, nu=1), False, False),
        ("C4 SAI1", K.stokes(4, 2, K.P, gamma=0.0, degree=3, beta=9.0, beta_p=1 / 16),
         K.cfg("sai", level=1, zeta=0.099, nu=1), False, False),
        ("C5 SAI1 4^3 (bs 108)", K.stokes(4, 3, K.P, gamma=0.0, degree=2, beta=4.0, beta_p=1 / 16, delta=0.01, **sph),
         K.cfg("sai", level=1, zeta=0.107, nu=1), False, False),
        ("Stokes 3D SAI1 6^3 p=1 (any n)", K.stokes(6, 3, K.P, gamma=0.0, degree=1, beta=1.0, beta_p=1 / 16,
                                                     delta=0.01, **sph),
         K.cfg("sai", level=1, zeta=0.107, nu=1), True, False),
    ]
    for name, spec, cfg, any_n, strict in cases:
        its = run(ctx, spec, cfg, any_n=any_n, strict=strict)
        print(f"{name}: ok ({its} solve iterations)", flush=True)
    g_bad = int(g._lib.lib.ldgmg_debug_guard_check())
    if g_bad >= 0:
        print(f"guard zones: {g_bad} violations, {int(g._lib.lib.ldgmg_debug_guard_live())} live buffers checked",
              flush=True)
        if g_bad:
            sys.exit(3)
    print("sanitize_run: all cases ok", flush=True)


if __name__ == "__main__":
    main()
