"""The drop-in boundary: the C-ABI library loads, exports exactly what
include/ldgmg_b200.h declares, and fails loudly without a device (no CPU
fallback).  Runs on CPU."""
import ctypes
import os
import re

import pytest

from tests.conftest import HAS_GPU, ROOT


def _declared():
    text = open(os.path.join(ROOT, "include", "ldgmg_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ldgmg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import paper_2412_12506_b200._lib as L
    lib = ctypes.CDLL(L.LIB_PATH)
    names = _declared()
    assert len(names) >= 50
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python mirror binds every one of them
    assert set(names) == set(L.EXPORTED)


def test_abi_version_and_errors_without_touching_device():
    import paper_2412_12506_b200 as g
    assert g._lib.lib.ldgmg_abi_version() == 1
    assert g.launch_count() >= 0
    rhs = g.random_rhs(3, 2, seed=0)
    assert rhs.shape == (6,) and (abs(rhs) <= 1).all()


@pytest.mark.skipif(HAS_GPU, reason="checks the no-device path")
def test_no_cpu_fallback():
    import paper_2412_12506_b200 as g
    with pytest.raises(g.CudaError, match="no CUDA device"):
        g.Context(0)


def test_random_rhs_matches_reference_generator(ref):
    import numpy as np
    import paper_2412_12506_b200 as g
    for seed in (0, 1, 12345):
        assert np.array_equal(g.random_rhs(37, 9, seed), ref.random_rhs(37, 9, seed))
