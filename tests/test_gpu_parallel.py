"""The partitioned V-cycle's GPU path (GpuOps over the C ABI, NCCL process
group) at world size 1 equals the single-GPU hierarchy in strict-order mode
bit for bit.  The multi-rank logic is covered on CPU by
tests/test_parallel_gloo.py (2 and 4 ranks, bit-exact)."""
import os
import socket

import numpy as np
import pytest

import paper_2412_12506_b200 as g
from tests import cases as K

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dist1():
    import torch.distributed as dist
    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        yield dist
        dist.destroy_process_group()
    else:
        yield dist


@pytest.mark.parametrize("name,spec,cfg,min_rows", [
    ("sai-3d", K.scalar(8, 3, K.P, degree=2, beta=4.0), K.cfg("sai", level=1), 64),
    ("sai-2d-dirichlet", K.scalar(16, 2, K.D, degree=2), K.cfg("sai", level=1, nu=2), 16),
    ("jacobi-2d", K.scalar(16, 2, K.P, degree=3, beta=9.0), K.cfg("jacobi", omega=0.7, nu=2), 16),
])
def test_partitioned_path_world1_bitwise(ctx, dist1, name, spec, cfg, min_rows):
    from paper_2412_12506_b200 import parallel
    P = g.Problem(spec, min_depth=cfg.min_depth)
    dm = parallel.from_problem(ctx, P, cfg, dist1, min_rows_per_rank=min_rows)
    full = dm._full
    full.set_strict_order(True)
    n, bs = full.n, full.bs
    b = torch.as_tensor(np.random.default_rng(2).uniform(-1, 1, n * bs)).cuda()
    xd = torch.zeros_like(b)
    xf = torch.zeros_like(b)
    for _ in range(2):
        dm.cycle(xd, b)
        full.cycle(xf, b)
    torch.cuda.synchronize()
    assert np.array_equal(xd.cpu().numpy(), xf.cpu().numpy())


SPH = dict(phase_shape=g.PHASE_BALL, center=(0.5, 0.5, 0.5), radii=(0.25, 0.25, 0.25), mu_in=1e2, mu_out=1.0)


@pytest.mark.parametrize("device", [True, False])
@pytest.mark.parametrize("name,spec,cfg,min_rows", [
    ("sai-2d-dirichlet", K.scalar(16, 2, K.D, degree=2), K.cfg("sai", level=1, nu=2), 16),
    ("jacobi-2d", K.scalar(16, 2, K.P, degree=3, beta=9.0), K.cfg("jacobi", omega=0.7, nu=2), 16),
    ("gs-2d", K.scalar(16, 2, K.D, degree=2), K.cfg("gs", nu=2), 16),
    ("pgs-2d", K.scalar(16, 2, K.D, degree=2), K.cfg("pgs", nu=1, partitions=1), 16),
    # C5's physics on a non-power-of-two mesh (extension A1)
    ("sai-stokes3d-anyn", K.stokes(6, 3, K.P, gamma=0.0, degree=1, beta=1.0, beta_p=1 / 16, delta=0.01, **SPH),
     K.cfg("sai", level=1, zeta=0.107, nu=1), 16),
])
def test_distributed_setup_world1_matches_replicated(ctx, dist1, name, spec, cfg, min_rows, device):
    """from_problem_partial (distributed setup: device-assembled operators cut
    by block gathers, or host assembly; GPU SAI / GPU factors on the rank's
    rows; B^T through the transposed view) gives the same cycles as the
    replicated setup, bit for bit."""
    from paper_2412_12506_b200 import parallel
    any_n = spec.n & (spec.n - 1) != 0
    a = parallel.from_problem(ctx, g.Problem(spec, min_depth=cfg.min_depth, any_n=any_n), cfg, dist1,
                              min_rows_per_rank=min_rows)
    b = parallel.from_problem_partial(ctx, spec, cfg, dist1, min_rows_per_rank=min_rows, device=device)
    n, bs = a._full.n, a._full.bs
    rhs = torch.as_tensor(np.random.default_rng(4).uniform(-1, 1, n * bs)).cuda()
    xa, xb = torch.zeros_like(rhs), torch.zeros_like(rhs)
    for _ in range(2):
        a.cycle(xa, rhs)
        b.cycle(xb, rhs)
    torch.cuda.synchronize()
    assert np.array_equal(xa.cpu().numpy(), xb.cpu().numpy())
    da, ba = a.cycle_costs()
    db, bb = b.cycle_costs()
    assert da == db and ba == bb


@pytest.mark.parametrize("kind", [0, 1])
def test_distributed_krylov_world1_matches_single_gpu_strict(ctx, dist1, kind):
    """DistKrylov (P-independent dots) on one rank = the single-GPU strict
    Krylov (both are the reference's sequential order)."""
    from paper_2412_12506_b200 import parallel
    spec, cfg = K.scalar(16, 2, K.D, degree=2), K.cfg("sai", level=1, nu=2)
    dm = parallel.from_problem(ctx, g.Problem(spec, min_depth=cfg.min_depth), cfg, dist1, min_rows_per_rank=16)
    full = dm._full
    full.set_strict_order(True)
    want = full.estimate_eta(kind=kind, seed=3, tol=1e-12, maxit=30)
    got = parallel.DistKrylov(dm).estimate_eta(kind=kind, seed=3, tol=1e-12, maxit=30)
    assert np.array_equal(got["residuals"], want["residuals"])
    assert got["iterations"] == want["iterations"] and got["eta"] == want["eta"]


def test_fast_projection_and_graph_world1(dist1):
    """Fast-mode distributed cycle (device projection over the 256 fixed
    ranges) = single-GPU fast mode bitwise; the captured whole-cycle graph
    validates and replays identically."""
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        _fast_projection_and_graph(g.Context(0, stream=stream), dist1)


def _fast_projection_and_graph(ctx, dist1):
    from paper_2412_12506_b200 import parallel
    spec, cfg = K.scalar(16, 2, K.P, degree=2), K.cfg("sai", level=1, nu=2)
    dm = parallel.from_problem(ctx, g.Problem(spec, min_depth=cfg.min_depth), cfg, dist1, min_rows_per_rank=16)
    full = dm._full
    full.set_strict_order(False)
    n, bs = full.n, full.bs
    b = torch.as_tensor(np.random.default_rng(3).uniform(-1, 1, n * bs)).cuda()
    xs, xd = torch.zeros_like(b), torch.zeros_like(b)
    for _ in range(2):
        full.cycle(xs, b)
        dm.cycle(xd, b, fast=True)
    torch.cuda.synchronize()
    assert np.array_equal(xs.cpu().numpy(), xd.cpu().numpy())
    assert dm.enable_graph(torch.zeros_like(b), b), getattr(dm, "_graph_error", "")
    assert dm.graph_kernels > 0
    xg = torch.zeros_like(b)
    xe = torch.zeros_like(b)
    for _ in range(2):
        dm.cycle(xg, b, fast=True)        # graph replay
        dm._cycle_body(xe, b, True)       # eager
    torch.cuda.synchronize()
    assert np.array_equal(xg.cpu().numpy(), xe.cpu().numpy())


@pytest.mark.parametrize("P", [2, 4])
def test_device_partial_levels_match_global_build(ctx, P):
    """The device-resident distributed setup (device_partial_levels) for
    every rank of a P-rank job, emulated on one GPU (the setup needs no
    communication for SAI): each rank's partial problem is assembled on the
    device (its rows + halo, the other rows empty), its SAI columns solved
    by the masked build on that operator, and its local A and B cut out by
    block gathers -- every block equals the corresponding block of the
    replicated global build (the host-path split of the global B), bit for
    bit."""
    from paper_2412_12506_b200 import parallel
    spec = K.stokes(12, 3, K.P, gamma=0.0, degree=1, beta=1.0, beta_p=1 / 16, delta=0.01, **SPH)
    cfg = K.cfg("sai", level=1, zeta=0.107, nu=1)
    full = g.Problem(spec, min_depth=cfg.min_depth, any_n=True)
    mgf = g.Multigrid(ctx, cfg, full)
    n, bs, _ = full.level_shape(0)
    Ag = full.level_matrix(0)
    Bg = mgf.smoother(0).sai_matrix()
    for rank in range(P):
        prob = g.Problem.partial(spec, P, rank, parallel.sai_halo_hops(spec, cfg.smoother), 8,
                                 min_depth=cfg.min_depth, any_n=True, device_assembly=True)
        levels, _ = parallel.device_partial_levels(ctx, prob, cfg, P, rank, 8, None)
        lv = levels[0]
        pa, pb = lv["plan_A"], lv["plan_B"]
        # A: the rank's rows with the plan's local columns
        lptr, lcol, lval = parallel.local_rows(*Ag, bs, bs, pa)
        A_dev = g.DeviceBsr.adopt(ctx, lv["A_local"].h)
        lv["A_local"].h = None
        p_, c_, v_ = A_dev.download()
        assert np.array_equal(p_, lptr) and np.array_equal(c_, lcol)
        assert np.array_equal(v_.view(np.int64), np.ascontiguousarray(lval).view(np.int64)), rank
        # B: own rows + ghost rows' owned columns (host split of the global build)
        (fptr, fcol, own_val, ghost_val), _ = parallel.split_b_rows(Bg, n, bs, pb)
        B_dev = g.DeviceBsr.adopt(ctx, lv["B_full"].h)
        lv["B_full"].h = None
        p_, c_, v_ = B_dev.download()
        want = np.concatenate([np.ascontiguousarray(own_val), ghost_val])
        assert np.array_equal(p_, fptr) and np.array_equal(c_, fcol)
        assert np.array_equal(v_.view(np.int64), want.view(np.int64)), rank
