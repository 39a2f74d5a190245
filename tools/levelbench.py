"""Per-level kernel timing of the C2 hierarchy (CUDA events, warm caches):
residual + SAI sweep per level, transfers, bottom -- the V-cycle budget."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2412_12506_b200 as g  # noqa: E402


def timeit(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3  # us


stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = g.Context(0, stream=stream)
spec, cfg = bench.workload()
P = g.Problem(spec)
mg = g.Multigrid(ctx, cfg, P)
b = torch.as_tensor(bench.rhs(mg.n, mg.bs)).cuda()
x = torch.zeros_like(b)
out = {"vcycle_us": timeit(lambda: mg.cycles(x, b, 1))}
for l in range(P.depth - 1):
    n, bs, nnzb = P.level_shape(l)
    A = g.DeviceBsr(ctx, n, n, bs, bs, *P.level_matrix(l))
    xl = torch.rand(n * bs, dtype=torch.float64, device="cuda")
    bl = torch.rand_like(xl)
    rl = torch.empty_like(xl)
    S = mg.smoother(l)
    out[f"L{l}_rows"] = n
    out[f"L{l}_residual_us"] = timeit(lambda: g.residual(ctx, A, bl, xl, rl))
    out[f"L{l}_sai_fwd_us"] = timeit(lambda: S.apply(bl, xl, g.SWEEP_FORWARD))
    out[f"L{l}_sai_rev_us"] = timeit(lambda: S.apply(bl, xl, g.SWEEP_REVERSE))
    out[f"L{l}_residual_GBps"] = 8.0 * (bs * bs * nnzb + 3 * bs * n) / out[f"L{l}_residual_us"] / 1e3
print(json.dumps(out, indent=1))
