"""Where the end-to-end solve time goes (C2): ldgmg_mg_solve_host from pageable
host buffers vs the device-resident graph-replayed cycles, plus the bare
pageable H2D / D2H of one vector.  Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2412_12506_b200 as g  # noqa: E402


def main():
    spec, cfg = bench.workload()
    ctx = g.Context(0)
    P = g.Problem(spec, min_depth=cfg.min_depth, bottom_max_elements=cfg.bottom_max_elements)
    mg = g.Multigrid(ctx, cfg, P)
    n, bs = mg.n, mg.bs
    b = bench.rhs(n, bs)
    mg.solve_host(b, tol=1e-10, maxit=100)
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        x, hist, iters = mg.solve_host(b, tol=1e-10, maxit=100)
    t_solve = (time.perf_counter() - t0) / reps
    bd = torch.as_tensor(b).cuda()
    xd = torch.zeros_like(bd)
    mg.cycles(xd, bd, 2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    mg.cycles(xd, bd, iters)
    e1.record()
    torch.cuda.synchronize()
    t_cycles = e0.elapsed_time(e1) * 1e-3
    hb = np.array(b)
    t0 = time.perf_counter()
    for _ in range(reps):
        bd.copy_(torch.from_numpy(hb))
        torch.cuda.synchronize()
    t_h2d = (time.perf_counter() - t0) / reps
    t0 = time.perf_counter()
    for _ in range(reps):
        hb[:] = bd.cpu().numpy()
    t_d2h = (time.perf_counter() - t0) / reps
    print(json.dumps({"iters": iters, "solve_host_ms": t_solve * 1e3, "cycles_ms": t_cycles * 1e3,
                      "overhead_ms": (t_solve - t_cycles) * 1e3, "torch_h2d_ms": t_h2d * 1e3,
                      "torch_d2h_ms": t_d2h * 1e3, "vector_mb": 8 * n * bs / 1e6}))


if __name__ == "__main__":
    main()
