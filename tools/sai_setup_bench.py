"""Time the GPU SAI build (batched least squares) of one level of a config.

  python tools/sai_setup_bench.py C5 [--level 0] [--reps 2]

Each rep builds a fresh SAI smoother (cache off between reps, so every rep
solves every unique local problem) and reports wall seconds, the unique
least-squares problem count and shapes, and the QR flop rate
(2 m n^2 - 2/3 n^3 per problem, Householder).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2412_12506_b200 as g  # noqa: E402
from tools.configs_bench import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--level", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--c5n", type=int, default=16)
    a = ap.parse_args()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = g.Context(0, stream=stream)
    spec, cfg, _ = configs(a.c5n)[a.name]
    P = g.Problem(spec, min_depth=cfg.min_depth, bottom_max_elements=cfg.bottom_max_elements)
    n, bs, _ = P.level_shape(a.level)
    A = g.DeviceBsr(ctx, n, n, bs, bs, *P.level_matrix(a.level))
    sc = cfg.smoother
    kind = g._lib.SYSTEM_STOKES if P.n_velocity else g._lib.SYSTEM_SCALAR
    for rep in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        S = g.Smoother(ctx, A, g.SmootherConfig.sai(sc.level, sc.zeta, cache=True), system_kind=kind,
                       n_velocity=P.n_velocity)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        st = S.sai_stats()
        shapes = st.ls_dims()
        print(json.dumps({"config": a.name, "level": a.level, "rep": rep, "seconds": round(dt, 4),
                          "unique_problems": st.cache_misses, "columns": st.cache_misses + st.cache_hits,
                          "rank_deficient_columns": st.rank_deficient_columns,
                          "shapes": {f"{k[0]}x{k[1]}": v for k, v in list(shapes.items())[:6]}}), flush=True)
        del S


if __name__ == "__main__":
    main()
