"""Memory safety and determinism of the device code without compute-sanitizer
(closed on this GPU pool): every kernel family runs with guard zones around
every library allocation (LDGMG_GUARD_BYTES, csrc/devmem.cpp) and the zones
must come back untouched; the V-cycles of every smoother kind run twice
(direct launches and graph replay, PDL on) and must agree bit for bit; and
the detector itself is shown to fire on a deliberate overrun."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tview", ["0", "1"])
def test_no_out_of_bounds_writes_and_deterministic(tview):
    env = dict(os.environ, LDGMG_GUARD_BYTES="4096", LDGMG_TVIEW=tview)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")], env=env,
                         capture_output=True, text=True, timeout=1800)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "guard zones: 0 violations" in out.stdout, out.stdout[-2000:]


POSITIVE = r"""
import ctypes as C, sys, numpy as np
sys.path.insert(0, %r)
import paper_2412_12506_b200 as g
from paper_2412_12506_b200 import _lib as L
ctx = g.Context(0)
p = C.c_void_p()
L.check(L.lib.ldgmg_device_alloc(ctx.h, 1000, C.byref(p)))
src = np.zeros(126)                                   # 1008 bytes into a 1000-byte buffer
L.check(L.lib.ldgmg_copy_h2d(ctx.h, p, src.ctypes.data, 1008))
print("violations", int(L.lib.ldgmg_debug_guard_check()))
"""


def test_guard_detector_fires():
    env = dict(os.environ, LDGMG_GUARD_BYTES="4096")
    out = subprocess.run([sys.executable, "-c", POSITIVE % ROOT], env=env, capture_output=True, text=True,
                         timeout=600)
    assert "violations 1" in out.stdout, out.stdout + out.stderr[-2000:]
