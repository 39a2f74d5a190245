"""GPU hot-path kernels against the oracle, BIT-exact.

Each kernel runs through the C ABI on the B200 and is compared with the
compiled reference (oracle/_ref) on the same seeded inputs -- spmv /
spmv_transpose / residual (blockla.hpp:136-176), block Jacobi and coloured
GS sweeps (smoothers.hpp:406-518), the SAI sweep with the reference's B
(smoothers.hpp:437-448), restriction / prolongation (multigrid.hpp:104-149).
The test cases mirror tests/test_blockla.cpp and tests/test_smoothers.cpp.
"""
import numpy as np
import pytest

import paper_2412_12506_b200 as g
from tests import cases as K

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a, np.float64)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def bits_equal(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(a, b)


def rand(n, seed):
    return np.random.default_rng(seed).uniform(-1, 1, n)


def random_bsr(brows, bcols, rbs, cbs, fill, seed, diag=False):
    rng = np.random.default_rng(seed)
    ptr, col, val = [0], [], []
    for i in range(brows):
        for j in range(bcols):
            if rng.random() < fill or (diag and i == j):
                col.append(j)
                val.append(rng.uniform(-1, 1, rbs * cbs))
        ptr.append(len(col))
    return np.array(ptr, np.int32), np.array(col, np.int32), (np.concatenate(val) if val else np.zeros(0))


@pytest.mark.parametrize("shape", [(7, 5, 3, 2, 0.4), (12, 12, 16, 16, 0.3), (9, 11, 27, 25, 0.3),
                                   (5, 5, 48, 48, 0.5), (3, 3, 108, 108, 0.6), (6, 4, 1, 7, 0.5)])
def test_spmv_and_transpose_bitwise(ctx, ref, shape):
    brows, bcols, rbs, cbs, fill = shape
    ptr, col, val = random_bsr(brows, bcols, rbs, cbs, fill, seed=17)
    A = g.DeviceBsr(ctx, brows, bcols, rbs, cbs, ptr, col, val)
    x = rand(bcols * cbs, 1)
    y = torch.empty(brows * rbs, dtype=torch.float64, device="cuda")
    g.spmv(ctx, A, dev(x), y)
    want, mults = ref.bsr_spmv(brows, bcols, rbs, cbs, ptr, col, val, x)
    assert mults == len(col)
    assert bits_equal(host(y), want)
    xt = rand(brows * rbs, 2)
    yt = torch.empty(bcols * cbs, dtype=torch.float64, device="cuda")
    g.spmv_transpose(ctx, A, dev(xt), yt)
    want_t, _ = ref.bsr_spmv(brows, bcols, rbs, cbs, ptr, col, val, xt, transpose=True)
    assert bits_equal(host(yt), want_t)
    # shape errors raise like the reference (blockla.hpp:137)
    with pytest.raises(g.InvalidArgument, match="shape mismatch"):
        g.spmv(ctx, A, dev(rand(bcols * cbs + 1, 3)), y)
    # round trip of the device layout
    p2, c2, v2 = A.download()
    assert np.array_equal(p2, ptr) and np.array_equal(c2, col) and bits_equal(v2, val)


def test_empty_rows_and_empty_matrix(ctx, ref):
    ptr = np.array([0, 0, 2, 2, 3], np.int32)
    col = np.array([0, 3, 1], np.int32)
    val = rand(3 * 4 * 4, 3)
    A = g.DeviceBsr(ctx, 4, 4, 4, 4, ptr, col, val)
    x = rand(16, 4)
    y = torch.full((16,), 7.0, dtype=torch.float64, device="cuda")
    g.spmv(ctx, A, dev(x), y)
    assert bits_equal(host(y), ref.bsr_spmv(4, 4, 4, 4, ptr, col, val, x)[0])
    Z = g.DeviceBsr(ctx, 3, 3, 2, 2, np.zeros(4, np.int32), np.zeros(0, np.int32), np.zeros(0))
    yz = torch.full((6,), 7.0, dtype=torch.float64, device="cuda")
    g.spmv(ctx, Z, dev(np.ones(6)), yz)
    assert bits_equal(host(yz), np.zeros(6))


def level_system(ref, spec, cfgk="jacobi", level=0, **kw):
    cfg = K.cfg(cfgk, **kw)
    R = ref.RefMultigrid(spec, cfg)
    return R, cfg


SYSTEMS = {
    "scalar2d-dirichlet-p1-mu1.3": K.scalar(4, 2, K.D, degree=1, mu=1.3),
    "scalar2d-periodic-p2": K.scalar(8, 2, K.P, degree=2),
    "scalar2d-p3-C1": K.scalar(16, 2, K.P, degree=3, beta=9.0),
    "scalar3d-p2-C2": K.scalar(4, 3, K.P, degree=2, beta=4.0),
    "scalar2d-p4-ball-C3": K.baseline_configs()["C3-GS"][0],
    "stokes2d-stress-p1": K.stokes(4, 2, K.P, gamma=1.0, degree=1),
    "stokes2d-p3-C4": K.baseline_configs()["C4"][0],
}


@pytest.mark.parametrize("name", sorted(SYSTEMS))
def test_residual_bitwise(ctx, ref, name):
    R, _ = level_system(ref, SYSTEMS[name])
    n, bs, _ = R.shape(0)
    A = g.DeviceBsr(ctx, n, n, bs, bs, *R.matrix(0))
    x, b = rand(n * bs, 5), rand(n * bs, 6)
    r = torch.empty(n * bs, dtype=torch.float64, device="cuda")
    g.residual(ctx, A, dev(b), dev(x), r)
    assert bits_equal(host(r), b - R.spmv(0, x))


@pytest.mark.parametrize("name", sorted(SYSTEMS))
@pytest.mark.parametrize("omega", [0.8, 0.6, 0.7])
def test_jacobi_sweeps_bitwise(ctx, ref, name, omega):
    R, _ = level_system(ref, SYSTEMS[name], "jacobi", omega=omega)
    n, bs, _ = R.shape(0)
    A = g.DeviceBsr(ctx, n, n, bs, bs, *R.matrix(0))
    S = g.Smoother(ctx, A, g.SmootherConfig.jacobi(omega), factors=R.diag_factors(0))
    b, x = rand(n * bs, 11), rand(n * bs, 23)
    xd = dev(x)
    want = x
    for _ in range(3):
        S.apply(dev(b), xd, g.SWEEP_FORWARD)
        want = R.smoother_apply(0, b, want, g.SWEEP_FORWARD)
        assert bits_equal(host(xd), want)
    # direction is irrelevant for a snapshot sweep (test_smoothers.cpp:139-143)
    xr = dev(x)
    S.apply(dev(b), xr, g.SWEEP_REVERSE)
    xf = dev(x)
    S.apply(dev(b), xf, g.SWEEP_FORWARD)
    assert bits_equal(host(xr), host(xf))


@pytest.mark.parametrize("name", sorted(SYSTEMS))
def test_coloured_gs_bitwise_and_colouring(ctx, ref, name):
    R, _ = level_system(ref, SYSTEMS[name], "gs")
    n, bs, _ = R.shape(0)
    A = g.DeviceBsr(ctx, n, n, bs, bs, *R.matrix(0))
    S = g.Smoother(ctx, A, g.SmootherConfig.coloured_gs(), factors=R.diag_factors(0))
    colours, nc = R.colours(0)
    assert S.n_colours() == nc
    assert np.array_equal(S.colours(), colours)
    b = rand(n * bs, 77)
    for sweep in (g.SWEEP_FORWARD, g.SWEEP_REVERSE):
        x = rand(n * bs, 78)
        xd = dev(x)
        for _ in range(2):
            S.apply(dev(b), xd, sweep)
            x = R.smoother_apply(0, b, x, sweep)
            assert bits_equal(host(xd), x)


@pytest.mark.parametrize("name", sorted(SYSTEMS))
@pytest.mark.parametrize("P", [1, 3, 4])
def test_proc_block_gs_bitwise(ctx, ref, name, P):
    """Processor-block GS (smoothers.hpp:426-436) run as wavefronts of the
    in-partition dependency DAG: bit-identical to the sequential sweeps."""
    R, cfg = level_system(ref, SYSTEMS[name], "pgs", partitions=P, omega=0.7)
    n, bs, _ = R.shape(0)
    A = g.DeviceBsr(ctx, n, n, bs, bs, *R.matrix(0))
    S = g.Smoother(ctx, A, cfg.smoother, factors=R.diag_factors(0))
    b = rand(n * bs, 31)
    for sweep in (g.SWEEP_FORWARD, g.SWEEP_REVERSE):
        x = rand(n * bs, 32)
        xd = dev(x)
        for _ in range(2):
            S.apply(dev(b), xd, sweep)
            x = R.smoother_apply(0, b, x, sweep)
            assert bits_equal(host(xd), x)


def test_proc_block_gs_rejects_too_many_partitions(ctx, ref):
    R, _ = level_system(ref, SYSTEMS["scalar2d-dirichlet-p1-mu1.3"])
    n, bs, _ = R.shape(0)
    A = g.DeviceBsr(ctx, n, n, bs, bs, *R.matrix(0))
    with pytest.raises(g.InvalidArgument, match="partition count must lie in"):
        g.Smoother(ctx, A, g.SmootherConfig.proc_block_gs(n + 1), factors=R.diag_factors(0))


def test_gs_ignores_damping(ctx, ref):
    R, _ = level_system(ref, SYSTEMS["scalar2d-dirichlet-p1-mu1.3"], "gs")
    n, bs, _ = R.shape(0)
    A = g.DeviceBsr(ctx, n, n, bs, bs, *R.matrix(0))
    cfg = g.SmootherConfig.coloured_gs()
    cfg.omega = 0.37
    S1 = g.Smoother(ctx, A, cfg, factors=R.diag_factors(0))
    S2 = g.Smoother(ctx, A, g.SmootherConfig.coloured_gs(), factors=R.diag_factors(0))
    b, x = rand(n * bs, 9), rand(n * bs, 10)
    x1, x2 = dev(x), dev(x)
    S1.apply(dev(b), x1)
    S2.apply(dev(b), x2)
    assert bits_equal(host(x1), host(x2))


@pytest.mark.parametrize("name", ["scalar2d-dirichlet-p1-mu1.3", "scalar2d-periodic-p2", "scalar3d-p2-C2",
                                  "stokes2d-stress-p1", "stokes2d-p3-C4", "scalar2d-p4-ball-C3"])
def test_sai_sweeps_bitwise_with_reference_B(ctx, ref, name):
    spec = SYSTEMS[name]
    zeta = 0.0990 if "C4" in name else 0.1
    R, _ = level_system(ref, spec, "sai", level=1, zeta=zeta)
    n, bs, _ = R.shape(0)
    A = g.DeviceBsr(ctx, n, n, bs, bs, *R.matrix(0))
    S = g.Smoother(ctx, A, g.SmootherConfig.sai(1, zeta), sai=R.sai_matrix(0))
    b = rand(n * bs, 55)
    for sweep in (g.SWEEP_FORWARD, g.SWEEP_REVERSE):
        x = rand(n * bs, 56)
        xd = dev(x)
        S.apply(dev(b), xd, sweep)
        assert bits_equal(host(xd), R.smoother_apply(0, b, x, sweep))


@pytest.mark.parametrize("name", ["scalar2d-periodic-p2", "scalar2d-p3-C1", "scalar3d-p2-C2", "stokes2d-p3-C4"])
def test_transfers_bitwise(ctx, ref, name):
    R, _ = level_system(ref, SYSTEMS[name])
    nf, bs, _ = R.shape(0)
    nc = R.shape(1)[0]
    p, o = R.transfer(0)
    T = g.Transfer(ctx, nf, nc, p, o, R.dim, R.bs_scalar, R.n_comp, R.injection())
    rf = rand(nf * bs, 12)
    rc = torch.full((nc * bs,), 3.0, dtype=torch.float64, device="cuda")
    T.restrict(dev(rf), rc)
    assert bits_equal(host(rc), R.restrict(0, rf))
    xc, xf = rand(nc * bs, 11), rand(nf * bs, 13)
    xfd = dev(xf)
    T.interpolate_add(dev(xc), xfd)
    assert bits_equal(host(xfd), R.interpolate_add(0, xc, xf))


IRREGULAR_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2412_12506_b200 as g
from oracle import port
ctx = g.Context(0)
# big: one parent with 60 / 80 children of 108-entry blocks -- above the
# per-thread kernel's 48 KB staging, so the per-CTA (<= 64 children) and the
# plain per-entry fallback kernels run
for dim, bss, ncomp, seed, big in [(2, 4, 1, 0, 0), (2, 16, 3, 1, 0), (3, 27, 1, 2, 0), (3, 9, 4, 3, 0),
                                   (2, 25, 1, 4, 0), (3, 27, 4, 5, 60), (3, 27, 4, 6, 80)]:
    rng = np.random.default_rng(seed)
    nc = 37
    cnt = rng.integers(1, 9, nc)
    cnt[5] = big or 11  # more children than one chain batch
    parent = np.repeat(np.arange(nc), cnt)
    rng.shuffle(parent)
    parent = parent.astype(np.int32)
    nf = len(parent)
    orth = rng.integers(-1, 1 << dim, nf).astype(np.int32)
    K = rng.uniform(-1, 1, (1 << dim) * bss * bss)
    BS = bss * ncomp
    T = g.Transfer(ctx, nf, nc, parent, orth, dim, bss, ncomp, K)
    rf = rng.uniform(-1, 1, nf * BS)
    rc = torch.full((nc * BS,), 7.0, dtype=torch.float64, device="cuda")
    T.restrict(torch.as_tensor(rf).cuda(), rc)
    want = port.restrict(parent, orth, K, bss, ncomp, nc, rf)
    got = rc.cpu().numpy()
    assert np.array_equal(got.view(np.int64), want.view(np.int64)), (dim, bss, ncomp, np.abs(got - want).max())
    xc, xf = rng.uniform(-1, 1, nc * BS), rng.uniform(-1, 1, nf * BS)
    xfd = torch.as_tensor(xf).cuda()
    T.interpolate_add(torch.as_tensor(xc).cuda(), xfd)
    want = port.interpolate_add(parent, orth, K, bss, ncomp, xc, xf)
    got = xfd.cpu().numpy()
    assert np.array_equal(got.view(np.int64), want.view(np.int64)), (dim, bss, ncomp, np.abs(got - want).max())
print("ok")
"""


def test_transfers_irregular_bitwise():
    """Restriction / prolongation on irregular parent maps (1..11 children per
    parent in shuffled fine order, orthant -1 copies, Stokes-like ncomp, and
    60 / 80 children of 108-entry blocks for the large-shape fallbacks) are
    bit-identical to the oracle port (multigrid.hpp:104-149 order)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", IRREGULAR_SCRIPT % root], capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]


TVIEW_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2412_12506_b200 as g
from tests import cases as K
case = %r
ctx = g.Context(0)
if case == "scalar3d-p2-16":
    spec, kind, zeta = K.scalar(16, 3, K.P, degree=2, beta=4.0), g.SYSTEM_SCALAR, 0.1
elif case == "scalar2d-p4-64":
    spec, kind, zeta = K.scalar(64, 2, K.D, degree=4, beta=16.0), g.SYSTEM_SCALAR, 0.1
else:
    spec = K.stokes(12, 3, K.P, gamma=0.0, degree=2, beta=4.0, beta_p=1 / 16, delta=0.01)
    kind, zeta = g.SYSTEM_STOKES, 0.107
P = g.Problem(spec, any_n=True)
n, bs, _ = P.level_shape(0)
assert n > 8 * 148
A = P.device_operator(ctx, 0)
S = g.Smoother(ctx, A, g.SmootherConfig.sai(1, zeta), system_kind=kind, n_velocity=P.n_velocity)
Bd = g.DeviceBsr(ctx, n, n, bs, bs, *S.sai_matrix())
rng = np.random.default_rng(7)
b = torch.as_tensor(rng.uniform(-1, 1, n * bs)).cuda()
x = torch.as_tensor(rng.uniform(-1, 1, n * bs)).cuda()
r = torch.empty_like(b)
g.residual(ctx, A, b, x, r)
for sweep, op in ((g.SWEEP_REVERSE, g.spmv_transpose), (g.SWEEP_FORWARD, g.spmv)):
    y = torch.empty_like(b)
    op(ctx, Bd, r, y)
    want = x.cpu().numpy() + y.cpu().numpy()
    got = x.clone()
    S.apply(b, got, sweep)
    got = got.cpu().numpy()
    assert np.array_equal(got.view(np.int64), want.view(np.int64)), (case, sweep, np.abs(got - want).max())
print("ok")
"""


@pytest.mark.parametrize("case", ["scalar3d-p2-16", "scalar2d-p4-64", "stokes3d-p2-12"])
def test_sai_transpose_view_sweeps_bitwise(case):
    """Reverse SAI sweeps read B^T as a VIEW of B's blocks (CSC index +
    permutation, transposed reads in the row pass; forced by LDGMG_TVIEW=1,
    by default only when the explicit copy does not fit): bit-identical to
    x + spmv_transpose(B, b - A x) through the explicit transposed copy
    (blockla.hpp:157-176 order).  Sizes exceed the split-row threshold so the
    streaming kernel runs: bs 27 (odd, 8-byte reads), 25, and 108 (paired
    16-byte reads)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, LDGMG_TVIEW="1")
    out = subprocess.run([sys.executable, "-c", TVIEW_SCRIPT % (root, case)], env=env, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]
