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
