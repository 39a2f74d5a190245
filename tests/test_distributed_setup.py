"""Distributed setup: each rank assembles only its element
range plus a halo (ldgmg_problem_create_partial) and solves only the SAI
columns its rows need (parallel.local_sai).

CPU: every assembled row is bit-identical to the full assembly; the SAI rows
and columns of each rank built from its partial operator (with the
reference's own build_sai, oracle/_ref) equal the global reference build bit
for bit; and the partitioned V-cycle fed with this distributed setup matches
the single-process reference V-cycle over gloo (2 and 4 ranks).
GPU: the column-masked GPU SAI build on the partial operator equals the
global GPU build on every rank's rows and columns."""
import numpy as np
import pytest

import paper_2412_12506_b200 as g
from paper_2412_12506_b200 import parallel
from tests import cases as K
from tests.conftest import HAS_GPU

CASES = {
    "scalar2d-periodic-p1": (K.scalar(16, 2, K.P, degree=1), K.cfg("sai", level=1), 16),
    "scalar2d-dirichlet-p2": (K.scalar(16, 2, K.D, degree=2), K.cfg("sai", level=1), 8),
    "scalar3d-periodic-p1": (K.scalar(16, 3, K.P, degree=1), K.cfg("sai", level=1), 32),
    "stokes2d-stress-p1": (K.stokes(32, 2, K.P, gamma=1.0, degree=1), K.cfg("sai", level=1, zeta=0.13), 8),
    "stokes2d-std-p1": (K.stokes(16, 2, K.P, gamma=0.0, degree=1), K.cfg("sai", level=1, zeta=0.13), 8),
    "scalar2d-sai2": (K.scalar(32, 2, K.P, degree=1), K.cfg("sai", level=2), 16),
}


def _rows(ptr):
    return np.nonzero(np.diff(ptr) > 0)[0]


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("nranks", [2, 4])
def test_partial_assembly_rows_bit_identical(name, nranks):
    spec, cfg, min_rows = CASES[name]
    full = g.Problem(spec)
    hops = parallel.sai_halo_hops(spec, cfg.smoother)
    for rank in range(nranks):
        part = g.Problem.partial(spec, nranks, rank, hops, min_rows)
        assert part.depth == full.depth
        for l in range(full.depth):
            fp, fc, fv = full.level_matrix(l)
            pp, pc, pv = part.level_matrix(l)
            n, bs, _ = full.level_shape(l)
            if not part.level_partial(l):
                assert np.array_equal(fp, pp) and np.array_equal(fc, pc) and fv.tobytes() == pv.tobytes()
                continue
            H = _rows(pp)
            r0, r1 = rank * n // nranks, (rank + 1) * n // nranks
            assert set(range(r0, r1)) <= set(H.tolist())
            if l == 0:
                assert len(H) < n  # genuinely partial
            for e in H:
                assert np.array_equal(fc[fp[e]:fp[e + 1]], pc[pp[e]:pp[e + 1]])
                assert (fv[fp[e] * bs * bs:fp[e + 1] * bs * bs].tobytes()
                        == pv[pp[e] * bs * bs:pp[e + 1] * bs * bs].tobytes())
            assert np.array_equal(part.level_transfer(l)[0], full.level_transfer(l)[0])


def _ref_build(ref, P, cfg):
    kind = g.SYSTEM_STOKES if P.n_comp > 1 else g.SYSTEM_SCALAR

    def build(lptr, lcol, lval, n, mask):
        (bp, bc, bv), _ = ref.sai_build(kind, P.dim, P.n_comp, P.bs_scalar, n, lptr, lcol, lval,
                                        cfg.smoother.level, cfg.smoother.zeta)
        return bp, bc, bv
    return build


def _row_block(ptr, col, val, bs, e):
    return col[ptr[e]:ptr[e + 1]], val[ptr[e] * bs * bs:ptr[e + 1] * bs * bs]


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("nranks", [2, 4])
def test_local_sai_matches_global_reference_build(ref, name, nranks):
    spec, cfg, min_rows = CASES[name]
    full = g.Problem(spec)
    n, bs, _ = full.level_shape(0)
    build = _ref_build(ref, full, cfg)
    Bg = build(*full.level_matrix(0), n, None)
    BgT = parallel.transpose_csr(*Bg, n, n, bs)
    hops = parallel.sai_halo_hops(spec, cfg.smoother)
    for rank in range(nranks):
        part = g.Problem.partial(spec, nranks, rank, hops, min_rows)
        assert part.level_partial(0)
        r0, r1 = rank * n // nranks, (rank + 1) * n // nranks
        Bl = parallel.local_sai(*part.level_matrix(0), n, bs, r0, r1, cfg.smoother.level, build)
        BlT = parallel.transpose_csr(*Bl, n, n, bs)
        for e in range(r0, r1):
            for M, W in ((Bl, Bg), (BlT, BgT)):
                c1, v1 = _row_block(*M, bs, e)
                c2, v2 = _row_block(*W, bs, e)
                assert np.array_equal(c1, c2), (rank, e)
                assert v1.tobytes() == v2.tobytes(), (rank, e)


def test_too_small_halo_is_detected(ref):
    spec, cfg, min_rows = CASES["scalar2d-periodic-p1"]
    full = g.Problem(spec)
    n, bs, _ = full.level_shape(0)
    part = g.Problem.partial(spec, 4, 1, 0, min_rows)  # no halo
    with pytest.raises(ValueError, match="halo too small"):
        parallel.local_sai(*part.level_matrix(0), n, bs, n // 4, n // 2, 1, _ref_build(ref, full, cfg))


def test_partial_rejects_bad_rank():
    spec, _, _ = CASES["scalar2d-periodic-p1"]
    with pytest.raises(g.InvalidArgument, match="rank"):
        g.Problem.partial(spec, 2, 2, 1, 16)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["scalar2d-dirichlet-p2", "scalar3d-periodic-p1", "stokes2d-stress-p1"])
@pytest.mark.parametrize("nranks", [2, 4])
def test_gpu_masked_sai_matches_global_gpu_build(ctx, name, nranks):
    spec, cfg, min_rows = CASES[name]
    full = g.Problem(spec)
    n, bs, _ = full.level_shape(0)
    kind = g.SYSTEM_STOKES if full.n_comp > 1 else g.SYSTEM_SCALAR
    Ag = g.DeviceBsr(ctx, n, n, bs, bs, *full.level_matrix(0))
    Bg_dev, _ = g.sai_build(ctx, Ag, kind, full.n_velocity, cfg.smoother.level, cfg.smoother.zeta)
    Bg = Bg_dev.download()
    BgT = parallel.transpose_csr(*Bg, n, n, bs)

    def gpu_build(lptr, lcol, lval, nl, mask):
        A = g.DeviceBsr(ctx, nl, nl, bs, bs, lptr, lcol, lval)
        B, _ = g.sai_build(ctx, A, kind, full.n_velocity, cfg.smoother.level, cfg.smoother.zeta, col_mask=mask)
        return B.download()

    hops = parallel.sai_halo_hops(spec, cfg.smoother)
    for rank in range(nranks):
        part = g.Problem.partial(spec, nranks, rank, hops, min_rows)
        r0, r1 = rank * n // nranks, (rank + 1) * n // nranks
        Bl = parallel.local_sai(*part.level_matrix(0), n, bs, r0, r1, cfg.smoother.level, gpu_build)
        BlT = parallel.transpose_csr(*Bl, n, n, bs)
        for e in range(r0, r1):
            for M, W in ((Bl, Bg), (BlT, BgT)):
                c1, v1 = _row_block(*M, bs, e)
                c2, v2 = _row_block(*W, bs, e)
                assert np.array_equal(c1, c2)
                assert v1.tobytes() == v2.tobytes()
