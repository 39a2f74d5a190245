"""Parity of the STREAMING row pass (rowpass_kernel, the TMA ring that runs
every level with more than 8 x SMs rows -- all of the headline V-cycle's
fine-level traffic) against the reference.

The kernel suites use small systems, which run on the split-row kernels; here
(1) the bitwise kernel and V-cycle suites are re-run with LDGMG_SPLIT_ROWS=0,
which sends every pass of every size through the streaming kernel, and
(2) a C2-stencil level large enough to take the streaming path by default
(16^3, p=2: 4096 rows of 27x27 blocks) is checked bitwise against the
reference's spmv / Jacobi / coloured-GS / SAI sweeps (blockla.hpp:136-176,
smoothers.hpp:406-450)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2412_12506_b200 as g
from tests import cases as K
from tests.conftest import ROOT

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a, np.float64)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def bits_equal(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.int64), b.view(np.int64))


def rand(n, seed):
    return np.random.default_rng(seed).uniform(-1, 1, n)


def test_bitwise_suites_on_streaming_path(ctx):
    env = dict(os.environ, LDGMG_SPLIT_ROWS="0")
    out = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_kernels.py", "tests/test_gpu_vcycle.py",
                          "tests/test_gpu_krylov.py", "-x", "-q", "-m", "gpu", "-k", "bitwise", "-p",
                          "no:cacheprovider"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=2400)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert " passed" in out.stdout


@pytest.fixture(scope="module")
def c2_16(ref):
    spec = K.scalar(16, 3, K.P, degree=2, beta=4.0)
    out = {}
    for kind in ("jacobi", "gs", "sai"):
        cfg = K.cfg(kind, omega=0.7, level=1)
        out[kind] = ref.RefMultigrid(spec, cfg)
    return out


def test_large_level_spmv_residual_bitwise(ctx, c2_16):
    R = c2_16["jacobi"]
    n, bs, _ = R.shape(0)
    assert n > 8 * 148  # default streaming path
    A = g.DeviceBsr(ctx, n, n, bs, bs, *R.matrix(0))
    x, b = rand(n * bs, 5), rand(n * bs, 6)
    y = torch.empty(n * bs, dtype=torch.float64, device="cuda")
    g.spmv(ctx, A, dev(x), y)
    want = R.spmv(0, x)
    assert bits_equal(host(y), want)
    r = torch.empty_like(y)
    g.residual(ctx, A, dev(b), dev(x), r)
    assert bits_equal(host(r), b - want)


def test_large_level_smoothers_bitwise(ctx, c2_16):
    b = rand(0, 0)
    for kind, R in c2_16.items():
        n, bs, _ = R.shape(0)
        A = g.DeviceBsr(ctx, n, n, bs, bs, *R.matrix(0))
        if kind == "jacobi":
            S = g.Smoother(ctx, A, g.SmootherConfig.jacobi(0.7), factors=R.diag_factors(0))
        elif kind == "gs":
            S = g.Smoother(ctx, A, g.SmootherConfig.coloured_gs(), factors=R.diag_factors(0))
        else:
            S = g.Smoother(ctx, A, g.SmootherConfig.sai(1), sai=R.sai_matrix(0))
        b = rand(n * bs, 41)
        for sweep in (g.SWEEP_FORWARD, g.SWEEP_REVERSE):
            x = rand(n * bs, 42)
            xd = dev(x)
            for _ in range(2):
                S.apply(dev(b), xd, sweep)
                x = R.smoother_apply(0, b, x, sweep)
                assert bits_equal(host(xd), x), (kind, sweep)
