"""Shared problem / config builders for the parity tests (mirrors the
reference tests' helpers, e.g. tests/test_multigrid.cpp:17-39)."""
import paper_2412_12506_b200 as g

P, D, N = g.BC_PERIODIC, g.BC_DIRICHLET, g.BC_NEUMANN


def scalar(n, dim, bc=P, degree=1, mu=1.0, beta=-1.0, **kw):
    bcs = bc if isinstance(bc, tuple) else (bc,) * 6
    kw.setdefault("mu_out", mu)
    return g.ProblemSpec(kind=g.SYSTEM_SCALAR, dim=dim, n=n, degree=degree, bc=bcs, beta=beta, **kw)


def stokes(n, dim, bc=P, gamma=0.0, degree=1, beta_p=1.0, delta=0.0, beta=-1.0, **kw):
    bcs = bc if isinstance(bc, tuple) else (bc,) * 6
    return g.ProblemSpec(kind=g.SYSTEM_STOKES, dim=dim, n=n, degree=degree, bc=bcs, gamma=gamma, beta=beta,
                         beta_p=beta_p, delta=delta, **kw)


def cfg(kind="jacobi", omega=0.8, nu=3, level=1, zeta=0.1, pre=g.SWEEP_FORWARD, post=g.SWEEP_REVERSE,
        min_depth=2, bottom_max=64, partitions=4):
    if kind == "jacobi":
        sm = g.SmootherConfig.jacobi(omega)
    elif kind == "gs":
        sm = g.SmootherConfig.coloured_gs()
    elif kind == "pgs":
        sm = g.SmootherConfig.proc_block_gs(partitions, omega)
    else:
        sm = g.SmootherConfig.sai(level, zeta)
    return g.MultigridConfig(smoother=sm, pre=pre, post=post, nu1=nu, nu2=nu, min_depth=min_depth,
                             bottom_max_elements=bottom_max)


# The BASELINE.json configs at test scale (same stencil / block size / BCs /
# phase geometry / smoother, smaller n) -- parity cases, not bench lines.
def baseline_configs(scale=True):
    c1 = (scalar(16 if scale else 64, 2, P, degree=3, beta=9.0), cfg("jacobi", omega=0.7, nu=2))
    c2 = (scalar(8 if scale else 32, 3, P, degree=2, beta=4.0), cfg("sai", level=1))
    ball = dict(phase_shape=g.PHASE_BALL, center=(0.5, 0.5, 0.5), radii=(0.3, 0.3, 0.3), mu_in=1e4, mu_out=1.0)
    c3 = (scalar(16 if scale else 256, 2, D, degree=4, beta=16.0, **ball), cfg("gs"))
    c3s = (scalar(16 if scale else 256, 2, D, degree=4, beta=16.0, **ball), cfg("sai", level=1))
    ell = dict(phase_shape=g.PHASE_ELLIPSE, center=(0.5, 0.5, 0.5), radii=(0.35, 0.2, 0.2), mu_in=1e3, mu_out=1.0)
    c4 = (stokes(8 if scale else 128, 2, P, gamma=0.0, degree=3, beta=9.0, beta_p=1 / 16, **ell),
          cfg("sai", level=1, zeta=0.0990))
    sph = dict(phase_shape=g.PHASE_BALL, center=(0.5, 0.5, 0.5), radii=(0.25, 0.25, 0.25), mu_in=1e2, mu_out=1.0)
    c5 = (stokes(4 if scale else 32, 3, P, gamma=0.0, degree=2, beta=4.0, beta_p=1 / 16, delta=0.01, **sph),
          cfg("sai", level=1, zeta=0.107))
    return {"C1": c1, "C2": c2, "C3-GS": c3, "C3-SAI": c3s, "C4": c4, "C5": c5}


def baseline_rhs(n, bs, kind, dim, bs_scalar, kernel_constants, kernel_pressure, normal=False, seed=0,
                 random_rhs=None):
    """The benchmark right-hand side: the reference's seeded uniform[-1,1]
    draw (random_rhs, krylov.hpp:279-287) -- Box-Muller N(0,1) on consecutive
    uniforms of the same stream for C3 (extension A5) -- with the constant
    mode of every kernel vector removed (krylov.hpp:295-299)."""
    import numpy as np
    v = np.array(random_rhs(n, bs, seed), dtype=np.float64)
    if normal:
        u = (v + 1.0) / 2.0
        u1, u2 = u[0::2], u[1::2]
        z = np.sqrt(-2.0 * np.log(np.maximum(u1, 1e-300)))
        out = np.empty_like(v)
        out[0::2] = z * np.cos(2 * np.pi * u2)
        out[1::2] = z * np.sin(2 * np.pi * u2)
        v = out
    offs = []
    if kernel_constants:
        offs += [c * bs_scalar for c in range(1 if kind == g.SYSTEM_SCALAR else dim)]
    if kernel_pressure:
        offs.append(dim * bs_scalar)
    for off in offs:
        idx = np.arange(n) * bs + off
        v[idx] -= v[idx].mean()
    return v


def fullsize_configs():
    """The BASELINE.json configs at their stated sizes (C5 at 16^3, the
    largest the reference can set up in minutes) + the reference-native box
    interface for C3: (spec, cfg, rhs_is_normal, stationary cycles to run)."""
    ball = dict(phase_shape=g.PHASE_BALL, center=(0.5, 0.5, 0.5), radii=(0.3, 0.3, 0.3), mu_in=1e4, mu_out=1.0)
    box = dict(phase_shape=g.PHASE_BOXES, center=(0.25, 0.25, 0.25), radii=(0.75, 0.75, 0.75), mu_in=1e4, mu_out=1.0)
    ell = dict(phase_shape=g.PHASE_ELLIPSE, center=(0.5, 0.5, 0.5), radii=(0.35, 0.2, 0.2), mu_in=1e3, mu_out=1.0)
    sph = dict(phase_shape=g.PHASE_BALL, center=(0.5, 0.5, 0.5), radii=(0.25, 0.25, 0.25), mu_in=1e2, mu_out=1.0)
    return {
        "C1": (scalar(64, 2, P, degree=3, beta=9.0), cfg("jacobi", omega=0.7, nu=2), False, 40),
        "C2": (scalar(32, 3, P, degree=2, beta=4.0), cfg("sai", level=1), False, 40),
        "C3-ball-GS": (scalar(256, 2, D, degree=4, beta=16.0, **ball), cfg("gs"), True, 12),
        "C3-ball-SAI": (scalar(256, 2, D, degree=4, beta=16.0, **ball), cfg("sai", level=1), True, 12),
        "C3-box-GS": (scalar(256, 2, D, degree=4, beta=16.0, **box), cfg("gs"), True, 40),
        "C3-box-SAI": (scalar(256, 2, D, degree=4, beta=16.0, **box), cfg("sai", level=1), True, 40),
        "C4": (stokes(128, 2, P, gamma=0.0, degree=3, beta=9.0, beta_p=1 / 16, **ell),
               cfg("sai", level=1, zeta=0.0990), False, 12),
        "C5-16": (stokes(16, 3, P, gamma=0.0, degree=2, beta=4.0, beta_p=1 / 16, delta=0.01, **sph),
                  cfg("sai", level=1, zeta=0.107), False, 6),
    }
