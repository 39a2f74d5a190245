"""Row-pass time of one level's residual (C2 hierarchy) under the current
LDGMG_NS / grid settings: python tools/level_ns_probe.py [level]"""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2412_12506_b200 as g  # noqa: E402

lv = int(sys.argv[1]) if len(sys.argv) > 1 else 1
spec, cfg = bench.workload()
ctx = g.Context(0)
P = g.Problem(spec, min_depth=cfg.min_depth)
A = P.device_operator(ctx, lv)
n, bs = A.brows, A.row_bs
b = torch.rand(n * bs, dtype=torch.float64, device="cuda")
x = torch.rand_like(b)
r = torch.empty_like(b)
for _ in range(5):
    g.residual(ctx, A, b, x, r)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    g.residual(ctx, A, b, x, r)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 50 * 1e3
byts = 8 * (bs * bs * A.nnzb + 3 * bs * n)
print(json.dumps({"level": lv, "rows": n, "NS": os.environ.get("LDGMG_NS", "3"), "us": us, "GBps": byts / us / 1e3}))
