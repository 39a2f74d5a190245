"""All five BASELINE.json configs at their stated sizes on one B200 (the
headline bench.py line is C2; this records the others for DESIGN.md /
profiles).  Per config: setup times (host assembly, GPU hierarchy incl. the
GPU SAI least-squares build), V-cycle time (CUDA graph, CUDA events),
DOF-updates/s and algorithmic GB/s, and the solve to 1e-10: stationary
V-cycles when they converge, otherwise left-preconditioned GMRES (the paper's
protocol).  One JSON line per config.

  python tools/configs_bench.py [C1 C2 C3-GS C3-SAI C4 C5] [--c5n 16]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_12506_b200 as g  # noqa: E402

P_, D_ = g.BC_PERIODIC, g.BC_DIRICHLET


def configs(c5n):
    ball3 = dict(phase_shape=g.PHASE_BALL, center=(0.5, 0.5, 0.5), radii=(0.3, 0.3, 0.3), mu_in=1e4, mu_out=1.0)
    ell = dict(phase_shape=g.PHASE_ELLIPSE, center=(0.5, 0.5, 0.5), radii=(0.35, 0.2, 0.2), mu_in=1e3, mu_out=1.0)
    sph = dict(phase_shape=g.PHASE_BALL, center=(0.5, 0.5, 0.5), radii=(0.25, 0.25, 0.25), mu_in=1e2, mu_out=1.0)
    S = g.SYSTEM_SCALAR
    T = g.SYSTEM_STOKES

    def mg(sm, nu):
        return g.MultigridConfig(smoother=sm, nu1=nu, nu2=nu)

    return {
        "C1": (g.ProblemSpec(kind=S, dim=2, n=64, degree=3, bc=(P_,) * 6, beta=9.0),
               mg(g.SmootherConfig.jacobi(0.7), 2), "uniform"),
        "C1-512": (g.ProblemSpec(kind=S, dim=2, n=512, degree=3, bc=(P_,) * 6, beta=9.0),
                   mg(g.SmootherConfig.jacobi(0.7), 2), "uniform"),
        "C2": (g.ProblemSpec(kind=S, dim=3, n=32, degree=2, bc=(P_,) * 6, beta=4.0),
               mg(g.SmootherConfig.sai(1), 3), "uniform"),
        "C3-GS": (g.ProblemSpec(kind=S, dim=2, n=256, degree=4, bc=(D_,) * 6, beta=16.0, **ball3),
                  mg(g.SmootherConfig.coloured_gs(), 3), "normal"),
        "C3-SAI": (g.ProblemSpec(kind=S, dim=2, n=256, degree=4, bc=(D_,) * 6, beta=16.0, **ball3),
                   mg(g.SmootherConfig.sai(1), 3), "normal"),
        # reference-native conforming interface (catalogue box (1/4,3/4)^2,
        # harness.hpp:57-64): the hierarchy stops before phase mixing (4x4)
        "C3-box-GS": (g.ProblemSpec(kind=S, dim=2, n=256, degree=4, bc=(D_,) * 6, beta=16.0,
                                    phase_shape=g.PHASE_BOXES, center=(0.25, 0.25, 0.25), radii=(0.75, 0.75, 0.75),
                                    mu_in=1e4, mu_out=1.0),
                      mg(g.SmootherConfig.coloured_gs(), 3), "normal"),
        "C3-box-SAI": (g.ProblemSpec(kind=S, dim=2, n=256, degree=4, bc=(D_,) * 6, beta=16.0,
                                     phase_shape=g.PHASE_BOXES, center=(0.25, 0.25, 0.25), radii=(0.75, 0.75, 0.75),
                                     mu_in=1e4, mu_out=1.0),
                       mg(g.SmootherConfig.sai(1), 3), "normal"),
        "C3-box-PGS4": (g.ProblemSpec(kind=S, dim=2, n=256, degree=4, bc=(D_,) * 6, beta=16.0,
                                      phase_shape=g.PHASE_BOXES, center=(0.25, 0.25, 0.25), radii=(0.75, 0.75, 0.75),
                                      mu_in=1e4, mu_out=1.0),
                        mg(g.SmootherConfig.proc_block_gs(4), 3), "normal"),
        "C3-beta4p2-GS": (g.ProblemSpec(kind=S, dim=2, n=256, degree=4, bc=(D_,) * 6, beta=64.0, **ball3),
                          mg(g.SmootherConfig.coloured_gs(), 3), "normal"),
        "C4": (g.ProblemSpec(kind=T, dim=2, n=128, degree=3, bc=(P_,) * 6, beta=9.0, beta_p=1 / 16, gamma=0.0, **ell),
               mg(g.SmootherConfig.sai(1, 0.0990), 3), "uniform"),
        "C5": (g.ProblemSpec(kind=T, dim=3, n=c5n, degree=2, bc=(P_,) * 6, beta=4.0, beta_p=1 / 16, gamma=0.0,
                             delta=0.01, **sph),
               mg(g.SmootherConfig.sai(1, 0.107), 3), "uniform"),
    }


def rhs(P, kind, seed=0):
    n, bs, _ = P.level_shape(0)
    v = g.random_rhs(n, bs, seed)
    if kind == "normal":  # extension A5: Box-Muller on consecutive uniforms of the same stream
        u = (v + 1.0) / 2.0
        u1, u2 = u[0::2], u[1::2]
        z = np.sqrt(-2.0 * np.log(np.maximum(u1, 1e-300)))
        out = np.empty_like(v)
        out[0::2] = z * np.cos(2 * np.pi * u2)
        out[1::2] = z * np.sin(2 * np.pi * u2)
        v = out
    offs = []
    if P.kernel_constants:
        offs += [c * P.bs_scalar for c in range(1 if P.n_comp == 1 else P.dim)]
    if P.kernel_pressure:
        offs.append(P.dim * P.bs_scalar)
    for off in offs:
        idx = np.arange(n) * bs + off
        v[idx] -= v[idx].mean()
    return v


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=["C1", "C1-512", "C2", "C3-GS", "C3-SAI", "C4", "C5"])
    ap.add_argument("--c5n", type=int, default=16)
    ap.add_argument("--csv", default=None, help="also write reference-format CSV rows (+perf columns)")
    ap.add_argument("--host-assembly", action="store_true", help="assemble the operators on the host (default: GPU)")
    ap.add_argument("--cycles", type=int, default=20)
    ap.add_argument("--no-solve", action="store_true", help="V-cycle timing only (no stationary / GMRES solve)")
    ap.add_argument("--props", action="store_true",
                    help="also check size-independent V-cycle properties at this size: apply(2b) == 2 apply(b) "
                         "bit for bit, graph replay == direct launches")
    a = ap.parse_args()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = g.Context(0, stream=stream)
    cfgs = configs(a.c5n)
    rows = []
    for name in a.names:
        spec, cfg, rk = cfgs[name]
        t0 = time.time()
        pow2 = spec.n & (spec.n - 1) == 0
        P = g.Problem(spec, min_depth=cfg.min_depth, bottom_max_elements=cfg.bottom_max_elements,
                      device_assembly=not a.host_assembly, any_n=not pow2)
        t_asm = time.time() - t0
        t0 = time.time()
        mg = g.Multigrid(ctx, cfg, P)
        torch.cuda.synchronize()
        t_mg = time.time() - t0
        dof, byts = mg.cycle_costs()
        bh = rhs(P, rk)
        b = torch.as_tensor(bh).cuda()
        x = torch.zeros_like(b)
        mg.cycles(x, b, 3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        mg.cycles(x, b, a.cycles)
        e1.record(stream)
        torch.cuda.synchronize()
        tc = e0.elapsed_time(e1) * 1e-3 / a.cycles
        rec = {"config": name, "N": P.level_shape(0)[0], "bs": P.bs, "fine_dof": P.level_shape(0)[0] * P.bs,
               "levels": P.depth, "setup_s": {"assembly": round(t_asm, 2), "gpu_hierarchy": round(t_mg, 2)},
               "vcycle_ms": tc * 1e3, "dof_updates_per_s": dof / tc, "alg_GBps": byts / tc / 1e9,
               "alg_bytes_per_cycle": byts, "device_mem_used_GB": round((lambda f, t: (t - f) / 1e9)(
                   *torch.cuda.mem_get_info()), 1)}
        if cfg.smoother.kind == g.SAI:
            st = mg.smoother(0).sai_stats()
            rec["sai_level0"] = {"cache_misses": st.cache_misses, "cache_hits": st.cache_hits,
                                 "ls_shapes": {f"{k[0]}x{k[1]}": v for k, v in st.ls_dims().items()}}
        if a.props:
            y1, y2 = torch.empty_like(b), torch.empty_like(b)
            mg.apply(b, y1)
            mg.apply(2.0 * b, y2)
            xa, xg = torch.zeros_like(b), torch.zeros_like(b)
            mg.cycle(xa, b)
            mg.cycle(xa, b)
            mg.cycles(xg, b, 2)
            torch.cuda.synchronize()
            rec["properties"] = {"apply_homogeneous_bitwise": bool(torch.equal(y2, 2.0 * y1)),
                                 "graph_equals_direct_bitwise": bool(torch.equal(xa, xg))}
            del y1, y2, xa, xg
        if a.no_solve:
            print(json.dumps(rec), flush=True)
            del mg, P
            continue
        t0 = time.perf_counter()
        xs, hist, its = mg.solve_host(bh, tol=1e-10, maxit=40)
        ts = time.perf_counter() - t0
        rec["stationary"] = {"iterations": its, "final_relres": float(hist[-1]), "seconds": round(ts, 4),
                             "converged": bool(hist[-1] <= 1e-10)}
        if hist[-1] > 1e-10:
            xg = torch.zeros_like(b)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep = mg.krylov_solve(b, xg, kind=g._lib.KRYLOV_GMRES, tol=1e-10, maxit=60)
            torch.cuda.synchronize()
            rec["gmres"] = {"iterations": rep["iterations"], "converged": rep["converged"],
                            "eta": rep["eta"], "seconds": round(time.perf_counter() - t0, 4)}
        print(json.dumps(rec), flush=True)
        if a.csv:
            from paper_2412_12506_b200 import report as R
            sm = cfg.smoother
            fam = {g.JACOBI: "J", g.COLOURED_GS: "GS", g.SAI: f"SAI{sm.level}",
                   g.PROC_BLOCK_GS: f"PGS{sm.partitions}"}[sm.kind]
            sweeps = "" if sm.kind == g.JACOBI else "-" + "".join("f" if s_ == g.SWEEP_FORWARD else "r"
                                                                 for s_ in (cfg.pre, cfg.post))
            et = mg.estimate_eta(g._lib.KRYLOV_GMRES, seed=0)
            rows.append(R.CellRow(name, spec.dim, spec.degree, spec.n, f"GMRES-{fam}{sweeps}", rho=et["rho"],
                                  eta=et["eta"], iterations=et["iterations"],
                                  classification=R.CLASSIFICATIONS.index(et["classification"]),
                                  perf={"setup_s": t_asm + t_mg, "vcycle_ms": tc * 1e3,
                                        "dof_updates_per_s": dof / tc, "alg_gbps": byts / tc / 1e9}))
        del mg, P
    if a.csv:
        from paper_2412_12506_b200 import report as R
        with open(a.csv, "w") as f:
            R.write_csv(f, rows)


if __name__ == "__main__":
    main()
