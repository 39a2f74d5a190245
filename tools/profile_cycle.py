"""Profiling target: build a bench workload (C5 at 48^3 by default, `--n` for
another size, `--workload C2`), warm up, then run either `--cycles` V-cycles
or (`--pair`) the level-0 SAI sweep pair between cudaProfilerStart/Stop, so
`ncu --profile-from-start off` sees exactly that region."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2412_12506_b200 as g  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C5")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--cycles", type=int, default=2)
ap.add_argument("--graph", type=int, default=1)
ap.add_argument("--pair", action="store_true", help="profile one level-0 SAI sweep (residual + B r) only")
a = ap.parse_args()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = g.Context(0, stream=stream)
if a.workload in ("C5", "C2"):
    spec, cfg, _ = bench.product_workload(a.workload, a.n)
else:  # any tools/configs_bench.py config (C1, C3-GS, C4, ...)
    from tools import configs_bench as cb
    spec, cfg, _ = cb.configs(a.n or 16)[a.workload]
pow2 = spec.n & (spec.n - 1) == 0
P = g.Problem(spec, min_depth=cfg.min_depth, device_assembly=True, any_n=not pow2)
mg = g.Multigrid(ctx, cfg, P)
offs = bench.kernel_offsets(spec.kind, P.dim, P.bs_scalar, P.kernel_constants, P.kernel_pressure)
b = torch.as_tensor(bench.remove_kernel(g.random_rhs(mg.n, mg.bs, 0), mg.n, mg.bs, offs)).cuda()
x = torch.zeros_like(b)
mg.cycles(x, b, 3)
S0 = mg.smoother(0)
if a.pair:
    S0.apply(b, x, g.SWEEP_FORWARD)
torch.cuda.synchronize()
torch.cuda.profiler.start()
if a.pair:
    S0.apply(b, x, g.SWEEP_FORWARD)
else:
    for _ in range(a.cycles):
        if a.graph:
            mg.cycles(x, b, 1)
        else:
            mg.cycle(x, b)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled", "pair" if a.pair else f"{a.cycles} cycles", flush=True)
