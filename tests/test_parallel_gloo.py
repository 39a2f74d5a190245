"""Multi-rank V-cycle on CPU (gloo): the product's partitioned V-cycle
(paper_2412_12506_b200/parallel.py -- partition plans from the C ABI, ghost
exchange, agglomeration, rank-count-independent projection) reproduces the
single-process reference V-cycle BIT for bit, at 2 and 4 ranks.  The local
compute is the oracle port (CPU test double for the GPU kernels, which are
themselves bit-exact against the same port: tests/test_gpu_*.py)."""
import os
import socket

import numpy as np
import pytest

from tests.conftest import ROOT


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("case,partial,world", [
    ("sai-scalar2d-periodic", False, 2), ("sai-scalar2d-periodic", False, 4),
    ("sai-scalar2d-dirichlet-p2", False, 2), ("jacobi-scalar2d-periodic", False, 4),
    ("sai-stokes2d-stress", False, 2), ("sai-scalar3d-periodic", False, 4),
    # distributed setup (each rank assembles its rows + halo, solves its SAI columns)
    ("sai-scalar2d-periodic", True, 4), ("sai-scalar2d-dirichlet-p2", True, 2), ("sai-stokes2d-stress", True, 4),
    # coloured GS: one exchange per colour phase; colouring from the ranks' rows
    ("gs-scalar2d-dirichlet-p2", False, 2), ("gs-scalar2d-dirichlet-p2", True, 4), ("gs-stokes2d-stress", True, 2),
    ("jacobi-scalar2d-periodic", True, 2),
    # processor-block GS across ranks (one partition per rank, frozen ghosts)
    ("pgs-scalar2d-dirichlet-p2", False, 2), ("pgs-scalar2d-dirichlet-p2", True, 4),
    ("pgs-stokes2d-stress", False, 4),
    # non-power-of-two 3D unsteady Stokes (C5's physics, extension A1)
    ("sai-stokes3d-unsteady-n12", False, 2), ("sai-stokes3d-unsteady-n12", True, 4)])
def test_partitioned_vcycle_matches_reference(ref, tmp_path, case, partial, world):
    """Every pass of a level with >= 1 owned rows is split into interior rows
    (run while the ghost layer is in flight) and boundary rows: the split
    is exercised everywhere and must not change a bit."""
    import torch.multiprocessing as mp
    from tests import _dist_worker

    mp.start_processes(_dist_worker.worker, args=(world, free_port(), case, str(tmp_path), partial), nprocs=world,
                       join=True, start_method="spawn")
    spec, cfg, _ = _dist_worker.case_spec(case, world)
    if spec.n & (spec.n - 1):
        truth, prob = _dist_worker.any_n_truth(spec, cfg)
        n, bs = prob.level_shape(0)[:2]
        cycle = lambda x, b: truth.cycle(x, b)  # noqa: E731
    else:
        R = ref.RefMultigrid(spec, cfg)
        n, bs, _ = R.shape(0)
        cycle = R.cycle
    b = np.random.default_rng(5).uniform(-1, 1, n * bs)
    x = np.zeros(n * bs)
    for _ in range(2):
        x = cycle(x, b)
    lds = set()
    for rank in range(world):
        z = np.load(tmp_path / f"rank{rank}.npz")
        r0, r1 = int(z["r0"]), int(z["r1"])
        lds.add(int(z["ld"]))
        assert np.array_equal(z["x"], x[r0 * bs:r1 * bs]), f"rank {rank}"
    assert min(lds) >= 1  # at least one partitioned level


def test_partition_plan_invariants():
    """Ghost / send lists are mutually consistent across ranks (CPU, C ABI)."""
    import paper_2412_12506_b200 as g
    from paper_2412_12506_b200.parallel import partition_level
    from tests import cases as K
    P = g.Problem(K.stokes(8, 2, K.P, gamma=1.0, degree=1), min_depth=1)
    ptr, col, _ = P.level_matrix(0)
    N = P.level_shape(0)[0]
    for world in (1, 2, 3, 4, 8):
        plans = [partition_level(ptr, col, N, world, r) for r in range(world)]
        assert sum(p.n_own for p in plans) == N
        for r, p in enumerate(plans):
            for q in range(world):
                # what r receives from q is exactly what q sends to r, in order
                want = p.ghost_gid[p.recv_off[q]:p.recv_off[q + 1]]
                got = plans[q].send_idx[plans[q].send_off[r]:plans[q].send_off[r + 1]] + plans[q].r0
                assert np.array_equal(want, got)
            # local columns address owned rows first, ghosts after
            assert p.local_col.max(initial=0) < p.n_own + p.n_ghost
    with pytest.raises(g.InvalidArgument):
        partition_level(ptr, col, N, N + 1, 0)


@pytest.mark.parametrize("case,kind,world", [("sai-scalar2d-periodic", 1, 4), ("sai-scalar2d-dirichlet-p2", 1, 2),
                                             ("jacobi-scalar2d-periodic", 0, 2), ("sai-stokes2d-stress", 1, 2),
                                             ("sai-scalar2d-dirichlet-p2", 0, 4)])
def test_distributed_krylov_matches_reference(ref, tmp_path, case, kind, world):
    """estimate_eta (GMRES / PCG with the partitioned V-cycle as
    preconditioner, P-independent dots) reproduces the reference's residual
    history, rho and eta bit for bit on every rank."""
    import torch.multiprocessing as mp
    from tests import _dist_worker
    from tests import cases as K

    mp.start_processes(_dist_worker.worker, args=(world, free_port(), case, str(tmp_path), False, kind),
                       nprocs=world, join=True, start_method="spawn")
    spec, cfg = {
        "sai-scalar2d-periodic": (K.scalar(16, 2, K.P, degree=1), K.cfg("sai", level=1, nu=2)),
        "sai-scalar2d-dirichlet-p2": (K.scalar(16, 2, K.D, degree=2), K.cfg("sai", level=1, nu=1)),
        "jacobi-scalar2d-periodic": (K.scalar(16, 2, K.P, degree=1), K.cfg("jacobi", omega=0.7, nu=2)),
        "sai-stokes2d-stress": (K.stokes(8, 2, K.P, gamma=1.0, degree=1), K.cfg("sai", level=1, zeta=0.13, nu=1)),
    }[case]
    want = ref.RefMultigrid(spec, cfg).eta(kind, 3, 1e-12, 30)
    for rank in range(world):
        z = np.load(tmp_path / f"rank{rank}.npz")
        assert np.array_equal(z["residuals"], want["residuals"]), rank
        assert int(z["iterations"]) == want["iterations"]
        assert float(z["rho"]) == want["rho"] and float(z["eta"]) == want["eta"]


def test_partition_depth_c5_48():
    """C5 at 48^3 (levels 110592, 13824, 1728, 216, 27; children of c are
    8c..8c+7): with 128 rows per rank the partitioned prefix is 3 levels at
    P = 2, 4, 8 (every rank boundary lands on a sibling-group boundary), and a
    boundary inside a sibling group stops the prefix."""
    from paper_2412_12506_b200.parallel import partition_depth
    sizes = [110592, 13824, 1728, 216, 27]
    transfers = [(np.arange(n) // 8, np.arange(n) % 8) for n in sizes[:-1]]
    for P in (2, 4, 8):
        assert partition_depth(sizes, transfers, P, 128) == 3
    assert partition_depth(sizes, transfers, 2, 8) == 3  # 216 / 2 = 108 = 13.5 groups: level 3 stays whole
    assert partition_depth(sizes, transfers, 16, 1) == 2  # 1728 / 16 = 108: level 2 stays whole
    assert partition_depth([36, 9], [(np.arange(36) // 4, np.arange(36) % 4)], 3, 1) == 1  # forced first level


def test_split_b_index_and_boundary_rows():
    """The rank-local B layout (own rows, then the ghost rows' owned-column
    blocks) and its transposed view reproduce B's rows and B^T's rows of the
    rank, the latter in ascending global row order; interior / boundary
    rows partition the rank's rows by ghost references."""
    from paper_2412_12506_b200.parallel import boundary_rows, partition_level, split_b_rows
    import paper_2412_12506_b200 as g
    from tests import cases as K
    P_ = g.Problem(K.scalar(8, 2, K.P, degree=1), min_depth=1)
    ptr, col, _ = P_.level_matrix(0)
    n, bs = P_.level_shape(0)[:2]
    rng = np.random.default_rng(0)
    val = rng.standard_normal(len(col) * bs * bs)
    dense = np.zeros((n * bs, n * bs))
    for i in range(n):
        for k in range(ptr[i], ptr[i + 1]):
            dense[i * bs:(i + 1) * bs, col[k] * bs:(col[k] + 1) * bs] = val[k * bs * bs:(k + 1) * bs * bs].reshape(bs, bs)
    for world in (2, 3):
        for rank in range(world):
            pl = partition_level(ptr, col, n, world, rank)
            (fptr, fcol, own_val, ghost_val), (tptr, tcol, tperm) = split_b_rows((ptr, col, val), n, bs, pl)
            gid = np.concatenate([np.arange(pl.r0, pl.r1), pl.ghost_gid])
            fval = np.concatenate([own_val, ghost_val]).reshape(-1, bs, bs)
            for c in range(pl.n_own):  # B^T row c of the rank = column (r0 + c) of B, rows ascending
                js = tcol[tptr[c]:tptr[c + 1]]
                assert np.all(np.diff(gid[js]) > 0)
                got = np.zeros((bs, n * bs))
                for q, j in zip(range(tptr[c], tptr[c + 1]), js):
                    got[:, gid[j] * bs:(gid[j] + 1) * bs] = fval[tperm[q]].T
                want = dense[:, (pl.r0 + c) * bs:(pl.r0 + c + 1) * bs].T
                assert np.array_equal(got, want)
            interior, boundary = boundary_rows(fptr[:pl.n_own + 1], fcol[:fptr[pl.n_own]], pl.n_own)
            assert sorted(np.concatenate([interior, boundary]).tolist()) == list(range(pl.n_own))
            for r in boundary:
                assert np.any(fcol[fptr[r]:fptr[r + 1]] >= pl.n_own)
            for r in interior:
                assert np.all(fcol[fptr[r]:fptr[r + 1]] < pl.n_own)
