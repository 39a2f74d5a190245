"""The persistent cooperative coarse-level program (csrc/coarse_program.cu)
is bit-identical to the launch-per-pass V-cycle, for every smoother, and is
captured in the CUDA graph (LDGMG_COARSE_ROWS=0 disables it)."""
import os
import subprocess
import sys

import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2412_12506_b200 as g
from tests import cases as K
out = []
for spec, cfg in [(K.scalar(32, 2, K.D, degree=2), K.cfg("gs")),
                  (K.scalar(32, 2, K.P, degree=3, beta=9.0), K.cfg("jacobi", omega=0.7, nu=2)),
                  (K.scalar(16, 3, K.P, degree=2, beta=4.0), K.cfg("sai", level=1)),
                  (K.stokes(16, 2, K.P, gamma=1.0, degree=1), K.cfg("sai", level=1, zeta=0.13))]:
    ctx = g.Context(0)
    mg = g.Multigrid(ctx, cfg, g.Problem(spec))
    mg.set_strict_order(True)
    b = torch.as_tensor(np.random.default_rng(1).uniform(-1, 1, mg.n * mg.bs)).cuda()
    x = torch.zeros_like(b)
    mg.cycle(x, b)          # direct launches
    mg.cycles(x, b, 3)      # graph replay
    y = torch.empty_like(b)
    mg.apply(b, y)
    torch.cuda.synchronize()
    out.append(np.concatenate([x.cpu().numpy(), y.cpu().numpy()]))
np.save(sys.argv[1], np.concatenate(out))
"""


def run(env_rows, path, tail="0"):
    env = dict(os.environ, LDGMG_COARSE_ROWS=str(env_rows), LDGMG_TAIL=tail)
    subprocess.run([sys.executable, "-c", SCRIPT % ROOT, path], env=env, check=True, timeout=600)


def test_coarse_program_bitwise(ctx, tmp_path):
    """grid-wide cooperative program, cluster tail and the default
    launch-per-pass V-cycle give the same bits"""
    import numpy as np
    a, b, c = str(tmp_path / "coop.npy"), str(tmp_path / "tail.npy"), str(tmp_path / "off.npy")
    run(4096, a)
    run(0, b, tail="1")
    run(0, c)
    assert np.array_equal(np.load(a), np.load(c))
    assert np.array_equal(np.load(b), np.load(c))
