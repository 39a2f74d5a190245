"""Profiling target: build a workload (bench C2 by default, or any
tools/configs_bench.py config), warm up, then run `--cycles` V-cycles between
cudaProfilerStart/Stop (use ncu --profile-from-start off)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2412_12506_b200 as g  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cycles", type=int, default=2)
ap.add_argument("--graph", type=int, default=0)
ap.add_argument("--config", default="")
a = ap.parse_args()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = g.Context(0, stream=stream)
if a.config:
    from tools import configs_bench as cb
    spec, cfg, _ = cb.configs(16)[a.config]
else:
    spec, cfg = bench.workload()
P = g.Problem(spec, min_depth=cfg.min_depth)
mg = g.Multigrid(ctx, cfg, P)
b = torch.as_tensor(bench.rhs(mg.n, mg.bs)).cuda()
x = torch.zeros_like(b)
for _ in range(3):
    mg.cycle(x, b)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(a.cycles):
    if a.graph:
        mg.cycles(x, b, 1)
    else:
        mg.cycle(x, b)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled", a.cycles, "cycles")
