"""The partitioned V-cycle's GPU path with P = 2 and 4 ranks on ONE GPU:
every rank is a thread with its own context and stream, and the
torch.distributed calls meet in an in-process mailbox (tests/_fake_dist.py)
-- so the device-resident distributed setup (halo assembly on the device,
masked SAI build, block gathers), the ghost exchange with the
interior/boundary overlap split on every level, B^T through the per-rank
transposed view and processor-block GS across ranks all run on the B200
with P > 1.  Two cycles must equal the single-GPU hierarchy (the same
product setup, strict-order projection) bit for bit on every rank."""
import numpy as np
import pytest

import paper_2412_12506_b200 as g
from tests import cases as K

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SPH = dict(phase_shape=g.PHASE_BALL, center=(0.5, 0.5, 0.5), radii=(0.25, 0.25, 0.25), mu_in=1e2, mu_out=1.0)


def cases(P):
    return {
        "sai-stokes3d-anyn": (K.stokes(12, 3, K.P, gamma=0.0, degree=1, beta=1.0, beta_p=1 / 16, delta=0.01, **SPH),
                              K.cfg("sai", level=1, zeta=0.107, nu=2), 64),
        "sai-scalar3d": (K.scalar(16, 3, K.P, degree=2, beta=4.0), K.cfg("sai", level=1, nu=1), 64),
        "pgs-scalar2d": (K.scalar(32, 2, K.D, degree=2), K.cfg("pgs", nu=1, omega=0.8, partitions=P), 16),
        "jacobi-scalar2d": (K.scalar(32, 2, K.P, degree=3, beta=9.0), K.cfg("jacobi", omega=0.7, nu=2), 16),
    }


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("name", ["sai-stokes3d-anyn", "sai-scalar3d", "pgs-scalar2d", "jacobi-scalar2d"])
def test_partitioned_gpu_path_multirank_bitwise(P, name):
    from paper_2412_12506_b200 import parallel
    from tests._fake_dist import run_ranks
    spec, cfg, min_rows = cases(P)[name]
    any_n = spec.n & (spec.n - 1) != 0
    ctx0 = g.Context(0)
    full = g.Multigrid(ctx0, cfg, g.Problem(spec, min_depth=cfg.min_depth, any_n=any_n, device_assembly=True))
    full.set_strict_order(True)
    n, bs = full.n, full.bs
    b = np.random.default_rng(6).uniform(-1, 1, n * bs)
    xf = torch.zeros(n * bs, dtype=torch.float64, device="cuda")
    bf = torch.as_tensor(b).cuda()
    for _ in range(2):
        full.cycle(xf, bf)
    torch.cuda.synchronize()
    want = xf.cpu().numpy()

    def rank_fn(rank, dist):
        stream = torch.cuda.Stream()
        torch.cuda.set_stream(stream)
        ctx = g.Context(0, stream=stream)
        dm = parallel.from_problem_partial(ctx, spec, cfg, dist, min_rows_per_rank=min_rows, device=True,
                                           overlap_min_rows=1)
        r0, r1 = dm.owned_range()
        b_own = torch.as_tensor(b[r0 * bs:r1 * bs].copy()).cuda()
        x_own = torch.zeros_like(b_own)
        for _ in range(2):
            dm.cycle(x_own, b_own)
        torch.cuda.synchronize()
        return r0, r1, dm.ld, x_own.cpu().numpy()

    outs = run_ranks(P, rank_fn)
    assert sum(o[1] - o[0] for o in outs) == n
    assert min(o[2] for o in outs) >= 1
    for rank, (r0, r1, _, x) in enumerate(outs):
        assert np.array_equal(x.view(np.int64), want[r0 * bs:r1 * bs].view(np.int64)), (name, P, rank)
