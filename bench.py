"""Benchmark driver (contract in the task statement; workload in DESIGN.md §5).

Headline workload = BASELINE.json configs[4] (C5), the config the metric's
1/2/4/8-GPU figures are quoted on, at its stated size, which fits one B200:
3D unsteady Stokes (rho/dt = 1e2 -> delta = 0.01), LDG p=2 on the periodic
48^3 mesh (110,592 elements, 108x108 FP64 blocks, gamma = 0 -> 7-block
stencil), viscosity 1e2 inside the sphere r = 0.25 at the centre and 1
outside (extension A2), velocity/pressure-balanced SAI1 (zeta = 0.107,
PAPER.md Table 2), nu1 = nu2 = 3, pre forward / post reverse, 5 levels
48 -> 24 -> 12 -> 6 -> 3 (extension A1: restricted Morton order), B^T read
through the transpose view.  The operators come from the built-in setup
(device assembly, GPU SAI build); the forcing is the reference's seeded
uniform[-1,1] draw (random_rhs, krylov.hpp:279-287) with the kernel
(pressure constant) removed.  C2 (configs[1], 3D Poisson 32^3 SAI1) is
measured in the same run and reported under "extra".

A step is one V-cycle (CUDA-graph replay) on device-resident x, b.
metric = V-cycle DOF-updates/s = sum_{l<L} (nu1+nu2) N_l bs per cycle x cycles / s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N > 1 runs under torchrun: the mesh-partitioned V-cycle.
`--impl reference` times the reference's own CPU V-cycle (oracle/_ref, built
from the unmodified reference headers) on the host cores; it never loads the
product library.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "V-cycle DOF-updates/sec"
UNIT = "DOF-updates/s"

# plain-data workload descriptions: turned into the product's ProblemSpec in
# the GPU arm and into the oracle's in the reference arm
PERIODIC = 0
SPHERE = dict(phase_shape=2, center=(0.5, 0.5, 0.5), radii=(0.25, 0.25, 0.25), mu_in=1e2, mu_out=1.0)


def workload_desc(name, n=None):
    if name == "C5":
        n = n or 48
        spec = dict(kind=1, dim=3, n=n, degree=2, bc=(PERIODIC,) * 6, beta=4.0, beta_p=1 / 16, gamma=0.0,
                    delta=0.01, **SPHERE)
        sm = dict(kind=3, level=1, zeta=0.107)
        label = (f"C5: 3D unsteady Stokes (rho/dt=1e2, delta=0.01) LDG p=2 periodic {n}^3, sphere mu=1e2/1, "
                 f"108x108 FP64 blocks, gamma=0 (7-block stencil), balanced SAI1 zeta=0.107, nu=3+3 fwd/rev")
    elif name == "C2":
        n = n or 32
        spec = dict(kind=0, dim=3, n=n, degree=2, bc=(PERIODIC,) * 6, beta=4.0)
        sm = dict(kind=3, level=1, zeta=0.1)
        label = f"C2: 3D Poisson LDG p=2 periodic {n}^3, 27x27 FP64 blocks, SAI1 nu=3+3 fwd/rev"
    else:
        raise ValueError(name)
    return spec, sm, label


def product_workload(name, n=None):
    import paper_2412_12506_b200 as g
    spec_d, sm, label = workload_desc(name, n)
    spec = g.ProblemSpec(**spec_d)
    cfg = g.MultigridConfig(smoother=g.SmootherConfig.sai(sm["level"], sm["zeta"]), pre=g.SWEEP_FORWARD,
                            post=g.SWEEP_REVERSE, nu1=3, nu2=3, bottom_max_elements=64, bottom_tol=1e-10,
                            min_depth=2)
    return spec, cfg, label


def kernel_offsets(kind, dim, bs_scalar, kernel_constants, kernel_pressure):
    offs = []
    if kernel_constants:
        offs += [c * bs_scalar for c in range(1 if kind == 0 else dim)]
    if kernel_pressure:
        offs.append(dim * bs_scalar)
    return offs


def remove_kernel(v, n, bs, offs):
    """random_rhs protocol (krylov.hpp:295-299): the constant-mode component
    of each kernel vector is removed, i.e. the mean of its mode-0 entries."""
    for off in offs:
        idx = np.arange(n) * bs + off
        v[idx] -= v[idx].mean()
    return v


class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md)."""

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except Exception:
            return None
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 5 + i and "Active" in r[5 + i]
                          and "Not" not in r[5 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(rows), "reasons": reasons}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def lscpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_reference(name, n_sample, steps, warmup, max_hierarchies=None):
    """The reference's own CPU V-cycle (oracle/_ref: the unmodified reference
    headers compiled by oracle/Makefile), never the product library.

    Headline: ONE hierarchy on one core (the reference is single-threaded per
    solve: OpenBLAS pinned to 1 thread, blockla.hpp:30-37, no OpenMP).
    Aggregate: k INDEPENDENT hierarchies of the same problem, one per host
    thread, all cycling together (the reference's run_cells parallelism,
    harness.hpp:305-327: each cell owns its hierarchy); they share only the
    least-squares cache (MultigridConfig::cache, multigrid.hpp:35), so the
    extra setups are cache hits.  k = min(nproc, what fits in 60 % of free
    host memory)."""
    from oracle import ref
    spec_d, sm, label = workload_desc(name, n_sample)
    spec = ref.problem_spec(**spec_d)
    cfg = ref.mg_config(smoother_kind=sm["kind"], level=sm["level"], zeta=sm["zeta"])
    cache = ref.SaiCache()
    try:
        import psutil
        proc = psutil.Process()
        rss0 = proc.memory_info().rss
    except Exception:
        psutil = None
    t0 = time.time()
    R0 = ref.RefMultigrid(spec, cfg, cache)
    t_setup = time.time() - t0
    per_h = (proc.memory_info().rss - rss0) if psutil else 2e9
    n, bs, _ = R0.shape(0)
    offs = kernel_offsets(spec_d["kind"], R0.dim, R0.bs_scalar, R0.kernel_constants, R0.kernel_pressure)
    b = remove_kernel(ref.random_rhs(n, bs, 0), n, bs, offs)
    dof = sum(6 * R0.shape(l)[0] * R0.shape(l)[1] for l in range(R0.depth - 1))
    ref.cycles_multi([R0], b, max(1, warmup))
    s1 = ref.cycles_multi([R0], b, steps)
    v1 = dof * steps / s1
    nproc = os.cpu_count() or 1
    k = nproc
    if psutil:
        k = max(1, min(nproc, int(0.6 * psutil.virtual_memory().available / max(per_h, 1)) + 1))
    if max_hierarchies:
        k = min(k, max_hierarchies)
    hs = [R0]
    t1 = time.time()
    if k > 1:
        extra = [None] * (k - 1)

        def mk(i):
            extra[i] = ref.RefMultigrid(spec, cfg, cache)

        th = [threading.Thread(target=mk, args=(i,)) for i in range(k - 1)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        hs += extra
    t_setup_k = time.time() - t1
    sk = ref.cycles_multi(hs, b, steps)
    vk = dof * steps * k / sk
    sample = (f"{name} at {n_sample}^3 (N={n}, bs={bs}, {R0.depth} levels, SAI1, nu=3+3): {steps} V-cycles; "
              f"1 hierarchy on 1 core ({s1:.2f} s) and {k} independent hierarchies on {k} threads ({sk:.2f} s)")
    info = {"sample": sample, "cores": k, "value_1core": v1, "value_aggregate": vk, "aggregate_threads": k,
            "nproc": nproc, "cpu_model": lscpu_model(), "setup_s": round(t_setup, 1),
            "setup_extra_hierarchies_s": round(t_setup_k, 1), "dof_updates_per_cycle": dof,
            "seconds_per_cycle_1core": s1 / steps,
            "note": "reference headers compiled -O3 -DNDEBUG against the oracle's Eigen/LAPACKE shims; "
                    "C5 at 48^3 (and 32^3) cannot be built by the reference (power-of-two meshes, host memory), "
                    "its 16^3 setup alone takes ~10 min on one core, so the timed sample is 8^3; "
                    "the metric is per DOF-update"}
    del hs, R0
    return vk, info


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    try:
        from oracle import ref
        if not ref.available():
            raise FileNotFoundError("oracle/_ref not built")
    except Exception as e:  # pragma: no cover
        print(json.dumps({"impl": "reference", "unavailable": str(e)}))
        return
    name = args.workload
    _, _, label = workload_desc(name, args.n)
    value, info = cpu_reference(name, args.cpu_n, max(1, args.steps), args.warmup)
    print(json.dumps({
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": label, "cpu_sample": info["sample"]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": info["cores"], "kind": "reference",
                         "sample": info["sample"],
                         **{k: v for k, v in info.items() if k not in ("sample", "cores")}},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_partitioned(args, ctx, stream, ws, rank, local):
    """N > 1: the mesh-partitioned V-cycle (paper_2412_12506_b200.parallel) on
    the headline workload (C5 at 48^3 by default), strong scaling over the
    ranks: contiguous (restricted-)Morton ranges, one ghost-layer exchange
    per operator application over NCCL overlapped with the interior rows,
    B^T read through a per-rank transposed view, agglomerated coarse levels,
    P-independent kernel projection, distributed setup (each rank assembles
    its rows + SAI halo and solves its SAI columns).  Time = max over ranks
    of the device time of K cycles."""
    import torch
    import torch.distributed as dist
    import paper_2412_12506_b200 as g
    from paper_2412_12506_b200 import parallel

    spec, cfg, label = product_workload(args.workload, args.n)
    t0 = time.time()
    dm = parallel.from_problem_partial(ctx, spec, cfg, dist, min_rows_per_rank=args.min_rows,
                                       overlap=not args.no_overlap)
    P = dm._problem
    torch.cuda.synchronize()
    t_setup = time.time() - t0
    cc = torch.tensor(dm.cycle_costs(), device="cuda", dtype=torch.float64)
    dist.all_reduce(cc)
    dof_cycle, bytes_cycle = float(cc[0]), float(cc[1])
    n, bs = P.level_shape(0)[:2]
    offs = kernel_offsets(spec.kind, P.dim, P.bs_scalar, P.kernel_constants, P.kernel_pressure)
    b_host = remove_kernel(g.random_rhs(n, bs, 0), n, bs, offs)
    r0, r1 = dm.owned_range()
    b_own = torch.as_tensor(b_host[r0 * bs:r1 * bs].copy()).cuda()
    x_own = torch.zeros_like(b_own)
    dist.barrier()
    # whole-cycle CUDA graph (V-cycle kernels + NCCL exchanges + device-side
    # deterministic projection), validated bitwise against the eager cycle;
    # eager fast-mode cycles if capture is unsupported
    use_graph = dm.enable_graph(torch.zeros_like(b_own), b_own) if not args.no_graph else False
    for _ in range(args.warmup):
        dm.cycle(x_own, b_own, fast=True)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    l0 = g.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            dm.cycle(x_own, b_own, fast=True)
        e1.record(stream)
        torch.cuda.synchronize()
    launches = g.launch_count() - l0
    if use_graph:  # replays launch the captured kernels without host-side launch calls
        launches += args.steps * dm.graph_kernels
    t = e0.elapsed_time(e1) * 1e-3
    tt = torch.tensor([t], device="cuda", dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t = float(tt.item())
    value = dof_cycle * args.steps / t
    # end to end: per step the pinned H2D of the owned b slice, e2e_cycles
    # cycles, the D2H of the owned x slice; wall time, max over ranks
    b_pin = torch.as_tensor(b_host[r0 * bs:r1 * bs].copy()).pin_memory()
    x_pin = torch.empty_like(b_pin).pin_memory()
    dist.barrier()
    ne = 2
    te0 = time.perf_counter()
    for _ in range(ne):
        b_own.copy_(b_pin, non_blocking=True)
        x_own.zero_()
        for _ in range(args.e2e_cycles):
            dm.cycle(x_own, b_own, fast=True)
        x_pin.copy_(x_own, non_blocking=True)
        torch.cuda.synchronize()
    te = time.perf_counter() - te0
    te_t = torch.tensor([te], device="cuda", dtype=torch.float64)
    dist.all_reduce(te_t, op=dist.ReduceOp.MAX)
    e2e_value = dof_cycle * ne * args.e2e_cycles / float(te_t.item())
    # roofline: this rank's level-0 SAI sweep pair (residual + B r row passes on
    # its rows, no exchange) timed alone with CUDA events; max time over ranks
    roof = None
    d0 = dm.L[0]
    if "B" in d0 and "nnzB" in d0:
        n_own = d0["plan"].n_own
        x_ext, rext = d0["x"], d0["rext"]

        def pair():
            dm.ops.residual(d0["A"], b_own, x_ext, rext[:n_own * bs])
            dm.ops.spmv_add(d0["B"], rext, x_ext[:n_own * bs])

        for _ in range(3):
            pair()
        torch.cuda.synchronize()
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        k0.record(stream)
        for _ in range(reps):
            pair()
        k1.record(stream)
        torch.cuda.synchronize()
        tk_t = torch.tensor([k0.elapsed_time(k1) * 1e-3 / reps], device="cuda", dtype=torch.float64)
        dist.all_reduce(tk_t, op=dist.ReduceOp.MAX)
        tk = float(tk_t.item())
        alg = 8.0 * (bs * bs * (d0["nnzA"] + d0["nnzB"]) + 6 * bs * n_own)
        peak = peaks().get("hbm_gbs", 6650.0)
        roof = {"bound": "hbm", "kernel": "level-0 SAI sweep pair on each rank's rows (rowpass_kernel)",
                "achieved": alg / tk / 1e9, "peak": peak, "unit": "GB/s", "frac": alg / tk / 1e9 / peak,
                "traffic": None, "alg_bytes_per_launch_pair": alg, "ms": tk * 1e3,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy), per GPU; time = max over ranks",
                "peak_theoretical": 8000.0, "frac_theoretical": alg / tk / 1e9 / 8000.0}
    ghosts = torch.tensor([float(d0["plan"].n_ghost)], device="cuda", dtype=torch.float64)
    dist.all_reduce(ghosts)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": label + ", mesh-partitioned over the ranks",
                       "fine_elements": n, "fine_dof": n * bs, "dof_updates_per_cycle": dof_cycle,
                       "alg_bytes_per_cycle": bytes_cycle, "parallelism": f"mesh-partitioned x{ws}",
                       "owned_elements_rank0": r1 - r0, "partitioned_levels": dm.ld,
                       "level0_ghost_elements_all_ranks": float(ghosts.item()),
                       "overlap": not args.no_overlap, "cuda_graph": bool(use_graph),
                       "graph_note": getattr(dm, "_graph_error", None) or "validated bitwise vs the eager cycle",
                       "projection": "fast (device, 256 fixed ranges, P-independent)",
                       "l2": "no flush: per-rank working set >> 126 MB L2",
                       "setup_s": round(t_setup, 2)},
            "vcycle_hbm_GBps_total": bytes_cycle * args.steps / t / 1e9,
            "roofline": roof,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(8 * (r1 - r0) * bs),
                    "d2h_bytes_per_step": int(8 * (r1 - r0) * bs),
                    "step": f"pinned H2D of the owned b slice + {args.e2e_cycles} partitioned V-cycles + D2H of the "
                            f"owned x slice (per rank)"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }), flush=True)
    dist.destroy_process_group()


def measure_single(args, ctx, stream, name, n, steps, warmup, e2e_cycles, clocks=True):
    """One workload on one GPU: setup, K graph-replayed V-cycles timed with
    CUDA events, the level-0 SAI sweep pair timed alone (roofline), and the
    end-to-end figure through the C ABI from pinned host buffers."""
    import torch
    import paper_2412_12506_b200 as g

    spec, cfg, label = product_workload(name, n)
    pow2 = spec.n & (spec.n - 1) == 0
    t0 = time.time()
    P = g.Problem(spec, min_depth=cfg.min_depth, bottom_max_elements=cfg.bottom_max_elements,
                  device_assembly=True, any_n=not pow2)
    t_asm = time.time() - t0
    t0 = time.time()
    mg = g.Multigrid(ctx, cfg, P)
    mg.setup()
    torch.cuda.synchronize()
    t_mg = time.time() - t0
    n_el, bs = mg.n, mg.bs
    dof_cycle, bytes_cycle = mg.cycle_costs()
    offs = kernel_offsets(spec.kind, P.dim, P.bs_scalar, P.kernel_constants, P.kernel_pressure)
    b_host = remove_kernel(g.random_rhs(n_el, bs, 0), n_el, bs, offs)
    b = torch.as_tensor(b_host).cuda()
    x = torch.zeros_like(b)

    mg.cycles(x, b, warmup)  # warm-up (also captures the CUDA graph)
    torch.cuda.synchronize()
    l0 = g.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = Clocks(ctx.device) if clocks else None
    torch.cuda.cudart().cudaProfilerStart()  # ncu --profile-from-start off sees the timed region only
    if clk:
        clk.__enter__()
    e0.record(stream)
    mg.cycles(x, b, steps)
    e1.record(stream)
    torch.cuda.synchronize()
    if clk:
        clk.__exit__()
    torch.cuda.cudart().cudaProfilerStop()
    launches = g.launch_count() - l0
    t = e0.elapsed_time(e1) * 1e-3
    value = dof_cycle * steps / t
    finite = bool(torch.isfinite(x).all())

    # ---- dominant kernel pair: the level-0 SAI sweep (residual + B r row passes)
    S0 = mg.smoother(0)
    nnzb_a = P.level_shape(0)[2]
    nnzb_b = S0.sai_nnzb()
    alg = 8.0 * (bs * bs * (nnzb_a + nnzb_b) + 6 * bs * n_el)
    xs = torch.rand_like(b)
    for _ in range(3):
        S0.apply(b, xs, g.SWEEP_FORWARD)
    torch.cuda.synchronize()
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    k0.record(stream)
    for _ in range(reps):
        S0.apply(b, xs, g.SWEEP_FORWARD)
    k1.record(stream)
    torch.cuda.synchronize()
    tk = k0.elapsed_time(k1) * 1e-3 / reps
    del xs

    # ---- end to end through the C ABI (ldgmg_mg_solve_host): per step the
    # pinned H2D of b, `e2e_cycles` V-cycles (graph-resident loop, residual
    # checks on the device, tol = 0 so the count is fixed), the D2H of x
    b_pin_t = torch.from_numpy(np.ascontiguousarray(b_host)).pin_memory()
    x_pin_t = torch.empty_like(b_pin_t).pin_memory()
    b_pin, x_pin = b_pin_t.numpy(), x_pin_t.numpy()
    mg.solve_host(b_pin, tol=0.0, maxit=e2e_cycles, out=x_pin)  # captures the solve graph
    torch.cuda.synchronize()
    n_e2e = 2
    te0 = time.perf_counter()
    for _ in range(n_e2e):
        _, hist, iters = mg.solve_host(b_pin, tol=0.0, maxit=e2e_cycles, out=x_pin)
    te = (time.perf_counter() - te0) / n_e2e
    e2e_value = dof_cycle * iters / te
    pk = peaks()
    peak = pk.get("hbm_gbs", 6650.0)
    res = {
        "label": label, "value": value, "ms_per_step": t / steps * 1e3, "t": t, "launches": launches,
        "finite": finite, "clocks": clk.summary() if clk else None,
        "config": {"workload": label, "fine_elements": n_el, "fine_dof": n_el * bs, "levels": P.depth,
                   "dof_updates_per_cycle": dof_cycle, "alg_bytes_per_cycle": bytes_cycle,
                   "setup_s": {"assembly": round(t_asm, 2), "hierarchy_gpu": round(t_mg, 2)},
                   "device_mem_used_GB": round((lambda f, tot: (tot - f) / 1e9)(*torch.cuda.mem_get_info()), 1)},
        "vcycle_hbm_GBps": bytes_cycle * steps / t / 1e9,
        "roofline": {"bound": "hbm", "kernel": f"level-0 SAI sweep, bs={bs}: residual + B r row passes "
                                              f"(rowpass_kernel)",
                     "achieved": alg / tk / 1e9, "peak": peak, "unit": "GB/s", "frac": alg / tk / 1e9 / peak,
                     "traffic": None, "alg_bytes_per_launch_pair": alg, "ms": tk * 1e3,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy; a read-mostly stream can exceed it)",
                     "peak_theoretical": 8000.0, "frac_theoretical": alg / tk / 1e9 / 8000.0},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(8 * n_el * bs),
                "d2h_bytes_per_step": int(8 * n_el * bs + 8 * (iters + 1)),
                "step": f"one ldgmg_mg_solve_host call from pinned host buffers: H2D of b, {iters} V-cycles "
                        f"(tol=0, device-side residual checks), D2H of x",
                "seconds_per_step": te, "final_relres": float(hist[-1])},
    }
    del mg, P, b, x
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C5", choices=["C5", "C2"])
    ap.add_argument("--n", type=int, default=None, help="mesh size (default: the BASELINE size, 48 / 32)")
    ap.add_argument("--cpu-n", type=int, default=8, help="reference CPU sample mesh size")
    ap.add_argument("--e2e-cycles", type=int, default=10)
    ap.add_argument("--no-extra", action="store_true", help="skip the C2 extra measurement")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--partitioned", action="store_true", help="force the mesh-partitioned path at N=1 (testing)")
    ap.add_argument("--no-graph", action="store_true", help="N>1: eager distributed cycles (no CUDA graph)")
    ap.add_argument("--no-overlap", action="store_true", help="N>1: no interior/boundary split of the passes")
    ap.add_argument("--min-rows", type=int, default=128, help="N>1: partition levels with >= this many rows per rank")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import paper_2412_12506_b200 as g

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = g.Context(local, stream=stream)
    if ws > 1 or args.partitioned:
        if not torch.distributed.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            torch.distributed.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
        run_partitioned(args, ctx, stream, ws, rank, local)
        return

    extra = {}
    if args.workload == "C5" and not args.no_extra:
        # C2 (configs[1], the round-1 headline) first, freed before C5 is built
        c2 = measure_single(args, ctx, stream, "C2", None, max(10, args.steps), args.warmup, 13, clocks=False)
        extra["C2"] = {k: c2[k] for k in ("value", "ms_per_step", "roofline", "e2e", "config", "vcycle_hbm_GBps")}
    r = measure_single(args, ctx, stream, args.workload, args.n, args.steps, args.warmup, args.e2e_cycles)
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        traffic = tr.get(f"sai_sweep_level0_bytes_{args.workload}")
    except Exception:
        pass
    r["roofline"]["traffic"] = traffic

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            from oracle import ref
            if ref.available():
                cv, info = cpu_reference(args.workload, args.cpu_n, 2, 1)
                cpu = {"value": cv, "unit": UNIT, "cores": info["cores"], "kind": "reference",
                       "sample": info["sample"], **{k: v for k, v in info.items() if k not in ("sample", "cores")}}
        except Exception as e:
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        cfgd = dict(r["config"])
        cfgd.update({"parallelism": "single GPU",
                     "l2": "no flush: per-cycle working set (A + B, read every cycle) >> 126 MB L2"})
        line = {
            "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": cfgd,
            "roofline": r["roofline"],
            "vcycle_hbm_GBps": r["vcycle_hbm_GBps"],
            "cpu_baseline": cpu,
            "e2e": r["e2e"],
            "gpu_launches": r["launches"],
            "iterate_finite": r["finite"],
            "clocks": r["clocks"],
            "extra": extra,
        }
        print(json.dumps(line), flush=True)
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
