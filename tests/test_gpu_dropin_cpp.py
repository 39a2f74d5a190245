"""The C++ drop-in (include/ldgmg_b200.hpp): the reference's ldgmg::Multigrid
and ldgmg::gpu::Multigrid built from the same Mesh / LevelAssembler /
MultigridConfig agree (tests/cpp/test_dropin.cpp, built by
`make -C oracle dropin` against the reference headers)."""
import os
import subprocess

import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_dropin_matches_reference(ctx):
    exe = os.path.join(ROOT, "oracle", "_ref", "test_dropin")
    if not os.path.exists(exe):
        pytest.skip("test_dropin not built (make -C oracle dropin)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    lines = [l for l in r.stdout.splitlines() if l.startswith(("PASS", "FAIL"))]
    assert len(lines) >= 5, r.stdout + r.stderr
    assert all(l.startswith("PASS") for l in lines), r.stdout
    assert r.returncode == 0
