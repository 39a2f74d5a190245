"""The product's built-in host setup (mesh chain + LDG assembly,
csrc/setup.cpp) against the reference assembly (oracle/_ref): level
operators, coarsening maps and injection matrices must be BIT-identical.
CPU only."""
import numpy as np
import pytest

import paper_2412_12506_b200 as g
from tests import cases as K

CASES = {
    "scalar2d-periodic-p1": (K.scalar(8, 2, K.P), 2),
    "scalar2d-dirichlet-p2-mu1.7": (K.scalar(8, 2, K.D, degree=2, mu=1.7), 2),
    "scalar2d-mixed-p3": (K.scalar(8, 2, (K.N, K.N, K.D, K.D, K.P, K.P), degree=3), 2),
    "scalar3d-periodic-p2": (K.scalar(4, 3, K.P, degree=2), 2),
    "scalar2d-box-phases": (K.scalar(16, 2, K.P, phase_shape=g.PHASE_BOXES, center=(0.25, 0.25, 0.25),
                                     radii=(0.75, 0.75, 0.75), mu_in=100.0), 2),
    "stokes2d-standard-p2": (K.stokes(4, 2, K.P, gamma=0.0, degree=2), 2),
    "stokes2d-stress-p1": (K.stokes(4, 2, K.P, gamma=1.0, degree=1), 2),
    "stokes2d-stress-neumann": (K.stokes(4, 2, K.N, gamma=1.0, degree=1), 2),
    "stokes2d-unsteady-dirichlet": (K.stokes(4, 2, K.D, gamma=1.0, degree=2, delta=0.05), 2),
    "stokes3d-stress-p1": (K.stokes(4, 3, K.P, gamma=1.0, degree=1), 2),
}
CASES.update({f"baseline-{k}": (v[0], v[1].min_depth) for k, v in K.baseline_configs().items()})


@pytest.mark.parametrize("name", sorted(CASES))
def test_levels_bit_identical(name, ref):
    spec, min_depth = CASES[name]
    cfg = K.cfg("jacobi", min_depth=min_depth)
    R = ref.RefMultigrid(spec, cfg)
    P = g.Problem(spec, min_depth=min_depth, bottom_max_elements=64)
    assert P.depth == R.depth
    assert (P.dim, P.n_comp, P.bs_scalar) == (R.dim, R.n_comp, R.bs_scalar)
    assert (P.kernel_constants, P.kernel_pressure) == (R.kernel_constants, R.kernel_pressure)
    for l in range(R.depth):
        assert P.level_shape(l) == R.shape(l)
        pp, pc, pv = P.level_matrix(l)
        rp, rc, rv = R.matrix(l)
        assert np.array_equal(pp, rp) and np.array_equal(pc, rc)
        assert np.array_equal(pv.view(np.uint64), rv.view(np.uint64)), f"level {l} values differ"
        if l + 1 < R.depth:
            a, b = P.level_transfer(l)
            c, d = R.transfer(l)
            assert np.array_equal(a, c) and np.array_equal(b, d)
    if R.depth > 1:
        # the oracle reads K back through interpolate_add, which turns exact
        # zeros into -0.0; values must agree exactly
        assert np.array_equal(P.injection(), R.injection())


def test_rejections_mirror_reference():
    with pytest.raises(g.InvalidArgument, match="power of two"):
        g.Problem(K.scalar(6, 2))
    with pytest.raises(g.InvalidArgument, match="degree"):
        g.Problem(K.scalar(8, 3, degree=4))
    with pytest.raises(g.InvalidArgument, match="stress form"):
        g.Problem(K.stokes(4, 2, K.N, gamma=0.0))
    with pytest.raises(g.InvalidArgument, match="depth below"):
        g.Problem(K.scalar(2, 2), min_depth=2)
    with pytest.raises(g.InvalidArgument, match="element budget"):
        g.Problem(K.scalar(16, 2, phase_shape=g.PHASE_BOXES, center=(0.25, 0.25, 0), radii=(0.75, 0.75, 1),
                            mu_in=100.0), bottom_max_elements=8)
