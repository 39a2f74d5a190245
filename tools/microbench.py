"""Kernel microbenchmarks (CUDA events, inputs >> L2): residual / spmv /
Jacobi sweep on the BASELINE stencils.  Prints one JSON line per kernel."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_12506_b200 as g  # noqa: E402
from tests import cases as K  # noqa: E402


def timeit(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3


def main():
    ctx = g.Context(0)
    torch.cuda.set_stream(torch.cuda.Stream())
    ctx.set_stream(torch.cuda.current_stream())
    cases = [("C2-32^3-p2", K.scalar(32, 3, K.P, degree=2, beta=4.0)),
             ("C1-512^2-p3", K.scalar(512, 2, K.P, degree=3, beta=9.0)),
             ("C3-256^2-p4", K.scalar(256, 2, K.D, degree=4, beta=16.0)),
             ("C4-128^2-stokes-p3", K.stokes(128, 2, K.P, degree=3, beta=9.0, beta_p=1 / 16))]
    for name, spec in cases:
        t0 = time.time()
        P = g.Problem(spec)
        tsetup = time.time() - t0
        ptr, col, val = P.level_matrix(0)
        n, bs, nnzb = P.level_shape(0)
        A = g.DeviceBsr(ctx, n, n, bs, bs, ptr, col, val)
        x = torch.rand(n * bs, dtype=torch.float64, device="cuda")
        b = torch.rand(n * bs, dtype=torch.float64, device="cuda")
        r = torch.empty_like(x)
        t = timeit(lambda: g.residual(ctx, A, b, x, r))
        byts = 8.0 * (bs * bs * nnzb + 3 * bs * n)
        print(json.dumps({"kernel": "residual", "case": name, "ms": t * 1e3, "alg_GBps": byts / t / 1e9,
                          "bytes": byts, "setup_s": round(tsetup, 2)}), flush=True)
        t0 = time.time()
        S = g.Smoother(ctx, A, g.SmootherConfig.jacobi(0.7))
        tf = time.time() - t0
        t = timeit(lambda: S.apply(b, x))
        byts = 8.0 * (bs * bs * (nnzb - n) + (bs * bs + 2 * bs) * n + 3 * bs * n) + 16.0 * bs * n
        print(json.dumps({"kernel": "jacobi_sweep", "case": name, "ms": t * 1e3, "alg_GBps": byts / t / 1e9,
                          "factor_setup_s": round(tf, 2)}), flush=True)
        del S, A


if __name__ == "__main__":
    main()
