"""Every runtime knob that survives ("Runtime knobs") against
its default, in a fresh process each (knobs are read once per process):

* LDGMG_SOLVE_GRAPH=0: ldgmg_mg_solve_host through the host-driven loop
  instead of the one-graph device WHILE loop -- same iterate and history,
  bit for bit;
* LDGMG_HOST_FACTORS=1: per-element diagonal factors by the host
  eigensolver instead of the GPU Jacobi eigensolver -- Jacobi cycles within
  1e-12 (different eigenvector bits, same smoother);
* LDGMG_DGEMM_VARIANT=1..5: every tile variant of the batched DMMA GEMM
  gives an SAI build within 1e-12 of the default.
(LDGMG_SPLIT_ROWS, LDGMG_TVIEW, LDGMG_GPU_EIG_MIN and LDGMG_GUARD_BYTES are
covered by test_gpu_streaming_path.py, test_gpu_kernels.py,
test_gpu_vcycle.py and test_gpu_guards.py.)"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2412_12506_b200 as g
from tests import cases as K
what = %r
ctx = g.Context(0)
if what == "solve":
    spec, cfg = K.baseline_configs()["C2"]
    mg = g.Multigrid(ctx, cfg, g.Problem(spec, min_depth=cfg.min_depth))
    b = g.random_rhs(mg.n, mg.bs, 3)
    x, hist, its = mg.solve_host(b, tol=1e-10, maxit=30)
    np.save(sys.argv[1], np.concatenate([x, hist, [its]]))
elif what == "factors":
    spec, cfg = K.baseline_configs()["C1"]
    mg = g.Multigrid(ctx, cfg, g.Problem(spec, min_depth=cfg.min_depth))
    b = torch.as_tensor(g.random_rhs(mg.n, mg.bs, 3)).cuda()
    x = torch.zeros_like(b)
    mg.cycles(x, b, 3)
    np.save(sys.argv[1], x.cpu().numpy())
else:
    spec, cfg = K.baseline_configs()["C4"]
    P = g.Problem(spec, min_depth=cfg.min_depth)
    n, bs, _ = P.level_shape(0)
    A = g.DeviceBsr(ctx, n, n, bs, bs, *P.level_matrix(0))
    B, _ = g.sai_build(ctx, A, g.SYSTEM_STOKES, P.n_velocity, 1, cfg.smoother.zeta)
    np.save(sys.argv[1], B.download()[2])
"""


def run(tmp_path, what, env_extra, tag):
    out = tmp_path / f"{what}_{tag}.npy"
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT % (ROOT, what), str(out)], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


def test_solve_host_loop_equals_device_loop(tmp_path):
    a = run(tmp_path, "solve", {}, "graph")
    b = run(tmp_path, "solve", {"LDGMG_SOLVE_GRAPH": "0"}, "host")
    assert np.array_equal(a.view(np.int64), b.view(np.int64))


def test_host_factors_match_gpu_factors(tmp_path):
    a = run(tmp_path, "factors", {}, "gpu")
    b = run(tmp_path, "factors", {"LDGMG_HOST_FACTORS": "1"}, "host")
    assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(a)


@pytest.mark.parametrize("variant", ["1", "2", "3", "4", "5"])
def test_dgemm_variants_same_sai(tmp_path, variant):
    a = run(tmp_path, "sai", {}, "default")
    b = run(tmp_path, "sai", {"LDGMG_DGEMM_VARIANT": variant}, f"v{variant}")
    assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(a)
