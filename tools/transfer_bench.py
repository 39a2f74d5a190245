import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2412_12506_b200 as g
from tests import cases as K
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
ctx = g.Context(0, stream=stream)
spec = K.scalar(32, 3, K.P, degree=2, beta=4.0)
P = g.Problem(spec)
Kinj = P.injection()
for l in range(P.depth - 1):
    nf = P.level_shape(l)[0]; nc = P.level_shape(l + 1)[0]; bs = P.bs
    p, o = P.level_transfer(l)
    T = g.Transfer(ctx, nf, nc, p, o, 3, P.bs_scalar, P.n_comp, Kinj)
    rf = torch.rand(nf * bs, dtype=torch.float64, device='cuda'); rc = torch.empty(nc * bs, dtype=torch.float64, device='cuda')
    for _ in range(5): T.restrict(rf, rc); T.interpolate_add(rc, rf)
    torch.cuda.synchronize()
    for name, fn in (("restrict", lambda: T.restrict(rf, rc)), ("prolong", lambda: T.interpolate_add(rc, rf))):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(100): fn()
        e1.record(stream); torch.cuda.synchronize()
        print(f"level {l} nf={nf} nc={nc} {name}: {e0.elapsed_time(e1)*10:.2f} us/call")
