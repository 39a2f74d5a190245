"""Device assembly (assembly_gpu.cu, ldgmg_problem_create_ex with
LDGMG_PROBLEM_DEVICE_ASSEMBLY): the level operators evaluated on the GPU from
the recorded accumulate_AtDB / saddle-scatter program are BIT-identical to the
host assembly (itself bit-identical to the reference, test_setup_parity.py)
for scalar and Stokes systems, every level, and a device-assembled hierarchy
gives the same cycles as the host-assembled one."""
import numpy as np
import pytest

import paper_2412_12506_b200 as g
from tests import cases as K

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SPECS = {
    "scalar2d-periodic-p2": K.scalar(8, 2, K.P, degree=2),
    "scalar2d-dirichlet-p4-ball": K.baseline_configs()["C3-GS"][0],
    "scalar2d-mixed-p1": K.scalar(8, 2, (K.N, K.N, K.D, K.D, K.P, K.P), degree=1, mu=0.7),
    "scalar3d-periodic-p2": K.scalar(4, 3, K.P, degree=2, beta=4.0),
    "stokes2d-standard-p3-C4": K.baseline_configs()["C4"][0],
    "stokes2d-stress-p1": K.stokes(8, 2, K.P, gamma=1.0, degree=1),
    "stokes2d-stress-neumann": K.stokes(4, 2, (K.N, K.N, K.P, K.P, K.P, K.P), gamma=1.0, degree=2),
    "stokes3d-unsteady-p2-C5": K.baseline_configs()["C5"][0],
    # extension A1 (the C5 48^3 mesh shape at test scale): non-power-of-two
    # restricted-Morton mesh, 6^3 -> 3^3
    "stokes3d-unsteady-p2-C5-6cubed-any-n": K.stokes(6, 3, K.P, gamma=0.0, degree=2, beta=4.0, beta_p=1 / 16,
                                                     delta=0.01, phase_shape=g.PHASE_BALL, center=(0.5, 0.5, 0.5),
                                                     radii=(0.25, 0.25, 0.25), mu_in=1e2, mu_out=1.0),
}
ANY_N = {"stokes3d-unsteady-p2-C5-6cubed-any-n"}


@pytest.mark.parametrize("name", sorted(SPECS))
def test_device_assembly_bit_identical(ctx, name):
    spec = SPECS[name]
    an = name in ANY_N
    host = g.Problem(spec, min_depth=1, any_n=an)
    dev = g.Problem(spec, min_depth=1, device_assembly=True, any_n=an)
    assert dev.depth == host.depth
    for l in range(host.depth):
        hp, hc, hv = host.level_matrix(l)
        dp, dc = dev.level_pattern(l)
        assert np.array_equal(hp, dp) and np.array_equal(hc, dc)
        p2, c2, v2 = dev.device_operator(ctx, l).download()
        assert np.array_equal(p2, hp) and np.array_equal(c2, hc)
        assert v2.tobytes() == hv.tobytes(), (name, l)
    with pytest.raises(g.LogicError, match="assembled on the device"):
        dev.level_matrix(0)


def test_device_assembled_hierarchy_same_cycles(ctx):
    spec, cfg = K.baseline_configs()["C2"]
    a = g.Multigrid(ctx, cfg, g.Problem(spec, min_depth=cfg.min_depth))
    b = g.Multigrid(ctx, cfg, g.Problem(spec, min_depth=cfg.min_depth, device_assembly=True))
    rhs = torch.as_tensor(g.random_rhs(a.n, a.bs, 0)).cuda()
    xa, xb = torch.zeros_like(rhs), torch.zeros_like(rhs)
    for _ in range(2):
        a.cycle(xa, rhs)
        b.cycle(xb, rhs)
    torch.cuda.synchronize()
    assert np.array_equal(xa.cpu().numpy(), xb.cpu().numpy())
