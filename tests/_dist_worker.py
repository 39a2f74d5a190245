"""Worker for tests/test_parallel_gloo.py (spawned; must be importable).

Runs the product's partitioned V-cycle (paper_2412_12506_b200.parallel:
partition plans from the C ABI, ghost exchange / agglomeration /
P-independent projection over torch.distributed gloo) with a CPU compute
double -- the numpy oracle port -- and writes this rank's owned slice of x
after a few cycles."""
import os
import sys

import numpy as np


class CpuOps:
    """Test double for GpuOps: the same local operations on torch CPU tensors,
    computed by the oracle port (oracle/port.py)."""

    def __init__(self):
        import torch
        from oracle import port
        self.torch, self.port = torch, port

    def tensor(self, n):
        return self.torch.zeros(int(n), dtype=self.torch.float64)

    def itensor(self, a):
        return self.torch.as_tensor(np.ascontiguousarray(a, np.int64))

    def matrix(self, brows, bcols, bs, ptr, col, val):
        return (np.asarray(ptr), np.asarray(col), np.asarray(val), int(brows), int(bcols), int(bs))

    def matrix_pieces(self, brows, bcols, bs, ptr, col, pieces):
        nnz = int(np.asarray(ptr)[-1])
        val = np.zeros(nnz * bs * bs)
        for k0, v in pieces:
            v = np.asarray(v)
            val[k0 * bs * bs:k0 * bs * bs + v.size] = v
        return self.matrix(brows, bcols, bs, ptr, col, val)

    def prefix_view(self, M, nrows):
        ptr, col, val, _, bcols, bs = M
        k = int(ptr[nrows])
        return (ptr[:nrows + 1], col[:k], val[:k * bs * bs], int(nrows), bcols, bs)

    def transposed_view(self, M, brows, bcols, ptr, col, perm):
        bs = M[5]
        blocks = np.asarray(M[2]).reshape(-1, bs, bs)[np.asarray(perm)]
        return (np.asarray(ptr), np.asarray(col), np.ascontiguousarray(blocks.transpose(0, 2, 1)).reshape(-1),
                int(brows), int(bcols), bs)

    def residual_rows(self, A, b, x_ext, r, rows):
        ptr, col, val, _, _, bs = A
        full = b.numpy() - self.port.spmv(ptr, col, val, bs, bs, x_ext.numpy())
        rr = rows.numpy()
        r.view(-1, bs)[self.torch.as_tensor(rr)] = self.torch.as_tensor(full.reshape(-1, bs)[rr])

    def spmv_add_rows(self, B, r_ext, x_own, rows):
        ptr, col, val, _, _, bs = B
        y = self.port.spmv(ptr, col, val, bs, bs, r_ext.numpy()).reshape(-1, bs)
        rr = rows.numpy()
        xo = x_own.view(-1, bs)
        xo[self.torch.as_tensor(rr)] = xo[self.torch.as_tensor(rr)] + self.torch.as_tensor(y[rr])

    def factors(self, n, bs, V, lam, s):
        return (np.asarray(V), np.asarray(lam), np.asarray(s))

    def transfer(self, n_fine, n_coarse, parent, orth, dim, bss, ncomp, K):
        return (np.asarray(parent), np.asarray(orth), np.asarray(K), bss, ncomp, int(n_coarse))

    def residual(self, A, b, x_ext, r):
        ptr, col, val, _, _, bs = A
        r.copy_(self.torch.as_tensor(b.numpy() - self.port.spmv(ptr, col, val, bs, bs, x_ext.numpy())))

    def upload(self, a):
        return self.torch.as_tensor(np.ascontiguousarray(a, np.float64).copy())

    def spmv(self, A, x_ext, y):
        ptr, col, val, _, _, bs = A
        y.copy_(self.torch.as_tensor(self.port.spmv(ptr, col, val, bs, bs, x_ext.numpy())))

    def spmv_add(self, B, r_ext, x_own):
        ptr, col, val, _, _, bs = B
        x_own.copy_(self.torch.as_tensor(x_own.numpy() + self.port.spmv(ptr, col, val, bs, bs, r_ext.numpy())))

    def relax(self, A, F, b, x_src, x_live, x_out, omega):
        ptr, col, val, n, _, bs = A
        out = self.port.relax_rows(np.arange(n), ptr, col, val, bs, b.numpy(), x_src.numpy(), x_live.numpy(), *F,
                                   omega)
        x_out.copy_(self.torch.as_tensor(out.reshape(-1)))

    def relax_rows(self, A, F, b, x_src, x_live, x_out, omega, rows):
        ptr, col, val, n, _, bs = A
        r = rows.numpy()
        out = self.port.relax_rows(r, ptr, col, val, bs, b.numpy(), x_src.numpy(), x_live.numpy(), *F, omega)
        xo = x_out.view(-1, bs)
        xo[self.torch.as_tensor(r)] = self.torch.as_tensor(out)

    def restrict(self, T, rf, rc):
        parent, orth, K, bss, ncomp, nc = T
        rc.copy_(self.torch.as_tensor(self.port.restrict(parent, orth, K, bss, ncomp, nc, rf.numpy())))

    def prolong(self, T, xc, xf):
        parent, orth, K, bss, ncomp, nc = T
        xf.copy_(self.torch.as_tensor(self.port.interpolate_add(parent, orth, K, bss, ncomp, xc.numpy(),
                                                                xf.numpy())))

    def gather(self, x, idx, n, bs, out):
        out[:n * bs] = x.view(-1, bs)[idx[:n]].reshape(-1)

    def to_host(self, t):
        return t.numpy()


def case_spec(case, world):
    """(spec, cfg, min_rows_per_rank) of a test case; processor-block GS uses
    one partition per rank (the reference's smoother with partitions = P)."""
    from tests import cases as K
    return {
        "sai-scalar2d-periodic": lambda: (K.scalar(16, 2, K.P, degree=1), K.cfg("sai", level=1, nu=2), 16),
        "sai-scalar2d-dirichlet-p2": lambda: (K.scalar(16, 2, K.D, degree=2), K.cfg("sai", level=1, nu=1), 8),
        "jacobi-scalar2d-periodic": lambda: (K.scalar(16, 2, K.P, degree=1), K.cfg("jacobi", omega=0.7, nu=2), 16),
        "sai-stokes2d-stress": lambda: (K.stokes(8, 2, K.P, gamma=1.0, degree=1),
                                        K.cfg("sai", level=1, zeta=0.13, nu=1), 8),
        "sai-scalar3d-periodic": lambda: (K.scalar(8, 3, K.P, degree=1), K.cfg("sai", level=1, nu=1), 32),
        "gs-scalar2d-dirichlet-p2": lambda: (K.scalar(16, 2, K.D, degree=2), K.cfg("gs", nu=1), 8),
        "gs-stokes2d-stress": lambda: (K.stokes(8, 2, K.P, gamma=1.0, degree=1), K.cfg("gs", nu=1), 8),
        "pgs-scalar2d-dirichlet-p2": lambda: (K.scalar(16, 2, K.D, degree=2),
                                              K.cfg("pgs", nu=1, omega=0.8, partitions=world), 8),
        "pgs-stokes2d-stress": lambda: (K.stokes(8, 2, K.P, gamma=1.0, degree=1),
                                        K.cfg("pgs", nu=1, omega=0.7, partitions=world), 8),
        # extension A1 (non-power-of-two, restricted Morton order): C5's
        # physics (unsteady Stokes, sphere phase) on a 12^3 mesh, p = 1
        "sai-stokes3d-unsteady-n12": lambda: (
            K.stokes(12, 3, K.P, gamma=0.0, degree=1, beta=1.0, beta_p=1 / 16, delta=0.01, phase_shape=2,
                     center=(0.5, 0.5, 0.5), radii=(0.25, 0.25, 0.25), mu_in=1e2, mu_out=1.0),
            K.cfg("sai", level=1, zeta=0.107, nu=1), 64),
    }[case]()


def any_n_truth(spec, cfg):
    """Single-process truth for a non-power-of-two mesh the reference cannot
    build (build_uniform needs 2^k, mesh.hpp:143-149): the product's host
    setup (bit-identical to the reference's assembly on every mesh both can
    build, tests/test_setup_parity.py, and re-checked on these meshes by
    tests/test_mesh_any_n.py), the reference's own build_sai and sym_eig on
    those operators, and the oracle port's V-cycle."""
    import paper_2412_12506_b200 as g
    from oracle import port, ref
    prob = g.Problem(spec, min_depth=cfg.min_depth, bottom_max_elements=cfg.bottom_max_elements, any_n=True)
    kind = g.SYSTEM_STOKES if prob.n_comp > 1 else g.SYSTEM_SCALAR
    levels = []
    for l in range(prob.depth):
        n, bs, _ = prob.level_shape(l)
        lv = {"n": n, "bs": bs, "A": prob.level_matrix(l)}
        if l + 1 < prob.depth:
            (bp, bc, bv), _ = ref.sai_build(kind, prob.dim, prob.n_comp, prob.bs_scalar, n, *lv["A"],
                                            cfg.smoother.level, cfg.smoother.zeta)
            lv["B"] = (bp, bc, bv)
        levels.append(lv)
    transfers = [prob.level_transfer(l) for l in range(prob.depth - 1)]
    nb, bs, _ = prob.level_shape(prob.depth - 1)
    ptr, col, val = levels[-1]["A"]
    D = np.zeros((nb * bs, nb * bs))
    for i in range(nb):
        for k in range(ptr[i], ptr[i + 1]):
            D[i * bs:(i + 1) * bs, col[k] * bs:(col[k] + 1) * bs] = val[k * bs * bs:(k + 1) * bs * bs].reshape(bs, bs)
    lam, V = ref.sym_eig(D)
    offs = []
    if prob.kernel_constants:
        offs += [c * prob.bs_scalar for c in range(1 if prob.n_comp == 1 else prob.dim)]
    if prob.kernel_pressure:
        offs.append(prob.dim * prob.bs_scalar)
    pm = port.PortMultigrid(levels, transfers, prob.injection(), (V, lam), cfg, prob.bs_scalar, prob.n_comp, offs)
    return pm, prob


def worker(rank, world, port_no, case, outdir, partial=False, krylov=None, overlap_min_rows=1):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist
    from oracle import port, ref
    from paper_2412_12506_b200 import parallel

    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec, cfg, min_rows = case_spec(case, world)
    any_n = spec.n & (spec.n - 1) != 0
    if any_n:
        P, R = any_n_truth(spec, cfg)
    else:
        R = ref.RefMultigrid(spec, cfg)
        P = port.from_reference(R, cfg)
    levels = P.levels
    transfers = P.transfers

    def coarse_factory(ld):
        tail = port.PortMultigrid(levels[ld:], transfers[ld:], P.K, P.bottom, cfg, P.bss, P.ncomp, [])

        class Coarse:
            def vcycle(self, x, b):
                x.copy_(torch.as_tensor(tail.v_cycle(0, np.zeros(x.numel()), b.numpy())))
        return Coarse()

    if partial:
        # distributed setup: this rank's rows + halo only, SAI columns solved
        # by the reference's own build_sai on the rank's partial operator
        import paper_2412_12506_b200 as g
        prob = g.Problem.partial(spec, world, rank, parallel.sai_halo_hops(spec, cfg.smoother), min_rows,
                                 any_n=any_n)
        kind = g.SYSTEM_STOKES if prob.n_comp > 1 else g.SYSTEM_SCALAR

        def ref_build(lptr, lcol, lval, nl, mask):
            (bp, bc, bv), _ = ref.sai_build(kind, prob.dim, prob.n_comp, prob.bs_scalar, nl, lptr, lcol, lval,
                                            cfg.smoother.level, cfg.smoother.zeta)
            return bp, bc, bv
        def ref_factors(l, r0, r1, bs, D):
            V, lam, s_ = R.diag_factors(l)
            return V[r0 * bs * bs:r1 * bs * bs], lam[r0 * bs:r1 * bs], s_[r0 * bs:r1 * bs]

        def bcast(q, mine):
            t = torch.as_tensor(np.ascontiguousarray(mine, np.int64))
            dist.broadcast(t, src=q)
            return t.numpy().astype(np.int32)
        plevels, ptransfers = parallel.partial_levels(prob, cfg, world, rank, min_rows, ref_build, ref_factors,
                                                      bcast)
        # the agglomerated tail keeps the reference's full data (identical by construction)
        dm = parallel.DistMultigrid(CpuOps(), dist, cfg, plevels, ptransfers, prob.injection(), prob.dim,
                                    prob.bs_scalar, prob.n_comp, P.koffs, coarse_factory,
                                    min_rows_per_rank=min_rows, overlap_min_rows=overlap_min_rows)
    else:
        dm = parallel.DistMultigrid(CpuOps(), dist, cfg, levels, transfers, P.K, R.dim, P.bss, P.ncomp, P.koffs,
                                    coarse_factory, min_rows_per_rank=min_rows, overlap_min_rows=overlap_min_rows)
    if krylov is not None:
        rep = parallel.DistKrylov(dm).estimate_eta(kind=krylov, seed=3, tol=1e-12, maxit=30)
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), residuals=rep["residuals"], iterations=rep["iterations"],
                 rho=rep["rho"], eta=rep["eta"], converged=rep["converged"])
        dist.barrier()
        dist.destroy_process_group()
        return
    n, bs = levels[0]["n"], levels[0]["bs"]
    rng = np.random.default_rng(5)
    b = rng.uniform(-1, 1, n * bs)
    r0, r1 = dm.owned_range()
    x_own = torch.zeros((r1 - r0) * bs, dtype=torch.float64)
    b_own = torch.as_tensor(b[r0 * bs:r1 * bs].copy())
    for _ in range(2):
        dm.cycle(x_own, b_own)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), x=x_own.numpy(), r0=r0, r1=r1, ld=dm.ld)
    dist.barrier()
    dist.destroy_process_group()
