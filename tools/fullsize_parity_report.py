"""Measured deviations of the product route from the reference's full-size
histories (tests/golden/histories, tests/test_gpu_fullsize_parity.py): one
JSON line per config -- the numbers DESIGN.md §2.4 records and the test's
per-config bars are set from."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2412_12506_b200 as g  # noqa: E402
from tests import cases as K  # noqa: E402
from tests.test_gpu_fullsize_parity import HIST, measure  # noqa: E402


def main():
    torch.cuda.set_device(0)
    ctx = g.Context(0)
    for name in (sys.argv[1:] or list(K.fullsize_configs())):
        want = np.load(os.path.join(HIST, f"{name}.npz"))
        print(json.dumps({"config": name, **measure(ctx, name, want)}), flush=True)


if __name__ == "__main__":
    main()
