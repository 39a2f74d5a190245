"""GPU SAI build (batched least squares) against the reference build_sai
(smoothers.hpp:259-367): identical pattern / index arrays, identical cache
statistics and LS shapes (tests/test_smoothers.cpp:398-543,
tests/test_multigrid.cpp:309-325), B within 1e-12 relative Frobenius norm of
the reference's LAPACK-dgels B, and the stored-block normal equations
(test_smoothers.cpp:324-348)."""
import numpy as np
import pytest

import paper_2412_12506_b200 as g
from tests import cases as K

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

B_RTOL = 1e-12  # measured: <= 8.1e-15 on every case below


def build_pair(ctx, ref, spec, level, zeta=0.1, cache=True):
    R = ref.RefMultigrid(spec, K.cfg("jacobi", min_depth=1))
    n, bs, _ = R.shape(0)
    ptr, col, val = R.matrix(0)
    kind = g.SYSTEM_STOKES if R.n_comp > 1 else g.SYSTEM_SCALAR
    (bp, bc, bv), st = ref.sai_build(kind, R.dim, R.n_comp, R.bs_scalar, n, ptr, col, val, level, zeta, cache)
    A = g.DeviceBsr(ctx, n, n, bs, bs, ptr, col, val)
    S = g.Smoother(ctx, A, g.SmootherConfig.sai(level, zeta, cache), system_kind=kind, n_velocity=R.n_velocity)
    return R, (ptr, col, val), (bp, bc, bv), st, S


def dense(ptr, col, val, n, bs):
    D = np.zeros((n * bs, n * bs))
    B = val.reshape(-1, bs, bs)
    for i in range(n):
        for k in range(ptr[i], ptr[i + 1]):
            D[i * bs:(i + 1) * bs, col[k] * bs:(col[k] + 1) * bs] = B[k]
    return D


SYSTEMS = {
    "scalar2d-dirichlet-p1": (K.scalar(4, 2, K.D, degree=1, mu=1.3), [0, 1, 2], 0.1),
    "scalar2d-periodic-p2": (K.scalar(8, 2, K.P, degree=2), [0, 1, 2], 0.1),
    "scalar2d-mixed-p1": (K.scalar(4, 2, (K.N, K.N, K.D, K.D, K.P, K.P), degree=1, mu=0.7), [1], 0.1),
    "scalar3d-periodic-p2-C2": (K.scalar(4, 3, K.P, degree=2, beta=4.0), [1], 0.1),
    "scalar2d-ball-p4-C3": (K.baseline_configs()["C3-SAI"][0], [1], 0.1),
    "stokes2d-stress-p1": (K.stokes(4, 2, K.P, gamma=1.0, degree=1), [0, 1], 0.1),
    "stokes2d-standard-p3-C4": (K.baseline_configs()["C4"][0], [1], 0.0990),
    # C5 shape (2700x756 least squares, k=108: the wide-panel cuBLAS path)
    "stokes3d-unsteady-p2-C5": (K.baseline_configs()["C5"][0], [1], 0.107),
}


@pytest.mark.parametrize("name", sorted(SYSTEMS))
def test_gpu_sai_matches_reference(ctx, ref, name):
    spec, levels, zeta = SYSTEMS[name]
    for level in levels:
        R, A, Bref, st, S = build_pair(ctx, ref, spec, level, zeta)
        bp, bc, bv = S.sai_matrix()
        assert np.array_equal(bp, Bref[0]) and np.array_equal(bc, Bref[1])
        err = np.linalg.norm(bv - Bref[2]) / np.linalg.norm(Bref[2])
        assert err <= B_RTOL, (name, level, err)
        # every block, not only the aggregate (a few wrong columns must not hide)
        assert np.max(np.abs(bv - Bref[2])) <= 1e-12 * np.max(np.abs(Bref[2])), (name, level)
        gs = S.sai_stats()
        assert (gs.cache_hits, gs.cache_misses) == (st.cache_hits, st.cache_misses)
        assert gs.rank_deficient_columns == st.rank_deficient_columns
        assert gs.ls_dims() == st.ls_dims()


@pytest.mark.parametrize("case", [
    ("scalar2d", K.scalar(8, 2, K.P), 5, [1, 5, 13], [(5, 1), (13, 5), (25, 13)], [0, 1, 2]),
    ("scalar3d", K.scalar(8, 3, K.P), 7, [1, 7, 25], [(7, 1), (25, 7), (63, 25)], [0, 1]),
    ("stokes-standard", K.stokes(8, 2, K.P, gamma=0.0), 5, [1, 5, 13], [(5, 1), (13, 5), (25, 13)], [0, 1, 2]),
    ("stokes-stress", K.stokes(8, 2, K.P, gamma=1.0), 7, [1, 7, 19], [(7, 1), (19, 7), (37, 19)], [0, 1, 2]),
])
def test_stencil_table(ctx, ref, case):
    """tests/test_smoothers.cpp:467-543 (Table 3 of the paper)."""
    _, spec, a_st, b_st, shapes, levels = case
    P = g.Problem(spec, min_depth=1)
    ptr, col, val = P.level_matrix(0)
    n, bs, _ = P.level_shape(0)
    assert set(np.diff(ptr)) == {a_st}
    A = g.DeviceBsr(ctx, n, n, bs, bs, ptr, col, val)
    for lvl in levels:
        S = g.Smoother(ctx, A, g.SmootherConfig.sai(lvl), system_kind=spec.kind, n_velocity=P.n_velocity)
        bp, _, _ = S.sai_matrix()
        assert set(np.diff(bp)) == {b_st[lvl]}
        assert S.sai_stats().ls_dims() == {shapes[lvl]: n}


def test_cache_transparent_and_counts(ctx, ref):
    """test_smoothers.cpp:398-416: 1 miss + 63 hits on the wrapped 8^2 grid,
    bitwise-identical B with and without the cache."""
    spec = K.scalar(8, 2, K.P)
    P = g.Problem(spec, min_depth=1)
    n, bs, _ = P.level_shape(0)
    A = g.DeviceBsr(ctx, n, n, bs, bs, *P.level_matrix(0))
    for lvl in (0, 1):
        S1 = g.Smoother(ctx, A, g.SmootherConfig.sai(lvl, 0.1, True))
        S2 = g.Smoother(ctx, A, g.SmootherConfig.sai(lvl, 0.1, False))
        assert np.array_equal(S1.sai_matrix()[2], S2.sai_matrix()[2])
        s1, s2 = S1.sai_stats(), S2.sai_stats()
        assert (s2.cache_hits, s2.cache_misses) == (0, 0)
        assert (s1.cache_misses, s1.cache_hits) == (1, 63)


def test_hierarchy_shares_one_solve(ctx, ref):
    """test_multigrid.cpp:309-325: cache stats per level of a 16^2 hierarchy."""
    spec = K.scalar(16, 2, K.P, degree=2)
    mg = g.Multigrid(ctx, K.cfg("sai", level=1), g.Problem(spec))
    assert mg.depth == 4
    want = [(1, 255), (0, 64), (1, 15)]
    for l, (miss, hit) in enumerate(want):
        st = mg.smoother(l).sai_stats()
        assert (st.cache_misses, st.cache_hits) == (miss, hit)


def test_rank_deficient_fallback(ctx, ref):
    """test_smoothers.cpp:434-449: periodic 2x2, level 2: 4 rank-deficient
    columns, finite B, normal equations satisfied."""
    spec = K.scalar(2, 2, K.P)
    R, (ptr, col, val), Bref, st, S = build_pair(ctx, ref, spec, 2, cache=False)
    gs = S.sai_stats()
    assert gs.rank_deficient_columns == 4 == st.rank_deficient_columns
    bp, bc, bv = S.sai_matrix()
    assert np.all(np.isfinite(bv))
    n, bs, _ = R.shape(0)
    alpha = ref.balance_vector(g.SYSTEM_SCALAR, 2, 1, bs, n, ptr, col, val, 0.1)
    At = dense(ptr, col, val, n, bs) * np.outer(alpha, alpha)
    Bt = dense(bp, bc, bv, n, bs) / np.outer(alpha, alpha)
    T = At.T @ (At @ Bt - np.eye(n * bs))
    assert np.linalg.norm(T) <= 1e-8 * np.linalg.norm(At)
    assert np.linalg.norm(bv - Bref[2]) <= 1e-8 * np.linalg.norm(Bref[2])


@pytest.mark.parametrize("name", ["scalar2d-dirichlet-p1", "stokes2d-stress-p1"])
def test_normal_equations_on_stored_blocks(ctx, ref, name):
    """test_smoothers.cpp:324-348."""
    spec, levels, zeta = SYSTEMS[name]
    for level in levels:
        R, (ptr, col, val), _, _, S = build_pair(ctx, ref, spec, level, zeta)
        n, bs, _ = R.shape(0)
        kind = g.SYSTEM_STOKES if R.n_comp > 1 else g.SYSTEM_SCALAR
        alpha = ref.balance_vector(kind, R.dim, R.n_comp, R.bs_scalar, n, ptr, col, val, zeta)
        At = dense(ptr, col, val, n, bs) * np.outer(alpha, alpha)
        bp, bc, bv = S.sai_matrix()
        Bt = dense(bp, bc, bv, n, bs) / np.outer(alpha, alpha)
        T = At.T @ (At @ Bt - np.eye(n * bs))
        bound = 1e-8 * np.linalg.norm(At)
        for r in range(n):
            for k in range(bp[r], bp[r + 1]):
                c = bc[k]
                assert np.linalg.norm(T[r * bs:(r + 1) * bs, c * bs:(c + 1) * bs]) <= bound


def test_balance_errors(ctx, ref):
    """test_smoothers.cpp:304-321."""
    P = g.Problem(K.stokes(4, 2, K.P, gamma=0.0), min_depth=1)
    n, bs, _ = P.level_shape(0)
    A = g.DeviceBsr(ctx, n, n, bs, bs, *P.level_matrix(0))
    with pytest.raises(g.InvalidArgument, match="zeta must be positive"):
        g.Smoother(ctx, A, g.SmootherConfig.sai(1, 0.0), system_kind=g.SYSTEM_STOKES, n_velocity=P.n_velocity)
    A1 = g.DeviceBsr(ctx, 1, 1, 3, 3, [0, 1], [0], np.eye(3).ravel())
    with pytest.raises(g.LdgmgRuntimeError, match="zero velocity-pressure coupling"):
        g.Smoother(ctx, A1, g.SmootherConfig.sai(1, 0.1), system_kind=g.SYSTEM_STOKES, n_velocity=2)
