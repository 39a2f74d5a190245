"""Mesh-partitioned multi-GPU V-cycle.

One process per GPU.  Rank p owns the contiguous Morton element range
[p*N/P, (p+1)*N/P) of every distributed level (partition_ranges,
smoothers.hpp:87-94); for uniform meshes the children of coarse element c are
8c..8c+7, so the ranges are nested and restriction / prolongation are
rank-local.  Each operator application gathers one ghost layer of its input
(x before the residual / relaxation, r before B r or B^T r) with
torch.distributed point-to-point ops (NCCL over NVLink on B200, gloo in the
CPU tests); the kernel projection reduces in the reference's sequential order
over all elements (all-gather of the per-element products), so results are
independent of the rank count and bit-identical to the single-GPU strict
mode.  Levels with fewer than `min_rows_per_rank * P` elements are
agglomerated: every rank gathers the coarse right-hand side and runs the rest
of the V-cycle redundantly (identical bits everywhere).

All local compute is in the C ABI's sm_100a kernels (GpuOps); the ops object
is injectable only so that the partition / exchange / agglomeration logic can
be tested on CPU against the reference (tests/test_parallel_gloo.py).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from ._lib import check, lib


@dataclass
class Plan:
    """Partition plan of one operator's rows on one rank (ldgmg_partition_level)."""
    r0: int
    r1: int
    n_own: int
    n_ghost: int
    local_col: np.ndarray
    ghost_gid: np.ndarray
    recv_count: np.ndarray
    send_count: np.ndarray
    send_idx: np.ndarray

    @property
    def recv_off(self):
        return np.concatenate([[0], np.cumsum(self.recv_count)])

    @property
    def send_off(self):
        return np.concatenate([[0], np.cumsum(self.send_count)])


def partition_level(ptr, col, N, nranks, rank) -> Plan:
    ptr = np.ascontiguousarray(ptr, np.int32)
    col = np.ascontiguousarray(col, np.int32)
    r0, r1, ng, ns = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    check(lib.ldgmg_partition_level(N, ptr.ctypes.data, col.ctypes.data, nranks, rank, C.byref(r0), C.byref(r1),
                                    C.byref(ng), C.byref(ns), None, None, None, None, None))
    nnz_loc = int(ptr[r1.value] - ptr[r0.value])
    lc = np.empty(max(nnz_loc, 1), np.int32)
    gg = np.empty(max(ng.value, 1), np.int32)
    rc = np.empty(nranks, np.int32)
    sc = np.empty(nranks, np.int32)
    si = np.empty(max(ns.value, 1), np.int32)
    check(lib.ldgmg_partition_level(N, ptr.ctypes.data, col.ctypes.data, nranks, rank, C.byref(r0), C.byref(r1),
                                    C.byref(ng), C.byref(ns), lc.ctypes.data, gg.ctypes.data, rc.ctypes.data,
                                    sc.ctypes.data, si.ctypes.data))
    return Plan(r0.value, r1.value, r1.value - r0.value, ng.value, lc[:nnz_loc], gg[:ng.value], rc, sc,
                si[:ns.value])


def local_rows(ptr, col, val, bs_r, bs_c, plan: Plan):
    """Rows [r0, r1) of a global BSR with the plan's renumbered columns."""
    ptr = np.asarray(ptr)
    lptr = (ptr[plan.r0:plan.r1 + 1] - ptr[plan.r0]).astype(np.int32)
    k0, k1 = int(ptr[plan.r0]), int(ptr[plan.r1])
    lval = np.asarray(val)[k0 * bs_r * bs_c:k1 * bs_r * bs_c]
    return lptr, plan.local_col, lval


def transpose_csr(ptr, col, val, n_rows, n_cols, bs):
    """Host transpose of a square-block BSR (B^T for the reverse sweep):
    block (j, i) of the result = (B_ij)^T, rows i ascending per column j."""
    ptr, col = np.asarray(ptr), np.asarray(col)
    B = np.asarray(val).reshape(-1, bs, bs)
    rows = np.repeat(np.arange(n_rows), np.diff(ptr))
    order = np.lexsort((rows, col))
    tptr = np.zeros(n_cols + 1, np.int32)
    np.add.at(tptr, col + 1, 1)
    tptr = np.cumsum(tptr).astype(np.int32)
    return tptr, rows[order].astype(np.int32), np.ascontiguousarray(B[order].transpose(0, 2, 1)).reshape(-1)


def partition_depth(sizes, transfers, P, min_rows_per_rank):
    """Number of leading levels partitioned over the ranks: a level is
    partitioned while it has >= P * min_rows_per_rank elements and no rank
    boundary splits a sibling group of its restriction (the coarse residual
    of a parent must be summed by ONE rank in child order, multigrid.hpp:
    127-149); the rest of the V-cycle is agglomerated.  At least one level."""
    depth = len(sizes)
    if depth < 2:
        return 0
    ld = 0
    while ld < depth - 1 and sizes[ld] >= P * min_rows_per_rank:
        n, parent = sizes[ld], np.asarray(transfers[ld][0])
        bounds = [q * n // P for q in range(1, P)]
        if any(0 < bq < n and int(parent[bq - 1]) == int(parent[bq]) for bq in bounds):
            break
        ld += 1
    return max(ld, 1)


def split_b_index(ptr, col, n, plan: Plan):
    """The rank's SAI matrix as ONE device matrix serving both sweep
    directions: rows [0, n_own) are the rank's B rows (the
    plan's local column numbering, block order unchanged), rows n_own + g are
    the plan's ghost rows g restricted to the rank's own columns -- exactly
    the entries B[j][c], c owned, that the rank's B^T rows need.  Index-only:
    returns (fptr, fcol, src) with src[q] = the global B block behind local
    block q, and the transposed view pattern (tptr, tcol, tperm): B^T row c
    lists the blocks B[j][c] in ascending GLOBAL row order j (spmv_transpose's
    scatter order, blockla.hpp:163-175), columns = the local ids of j, which
    are the ghost-slot numbering of the forward plan (B's pattern is
    symmetric, so B and B^T reach the same ghosts)."""
    ptr, col = np.asarray(ptr, np.int64), np.asarray(col)
    r0, r1, n_own = plan.r0, plan.r1, plan.n_own
    lptr = ptr[r0:r1 + 1] - ptr[r0]
    own_src = np.arange(ptr[r0], ptr[r1], dtype=np.int64)
    gcnt = np.zeros(len(plan.ghost_gid), np.int64)
    gsrc, gcol = [], []
    for i, g in enumerate(plan.ghost_gid):
        ks = np.arange(ptr[g], ptr[g + 1])
        cs = col[ks]
        m = (cs >= r0) & (cs < r1)
        gsrc.append(ks[m])
        gcol.append(cs[m] - r0)
        gcnt[i] = int(m.sum())
    gsrc = np.concatenate(gsrc).astype(np.int64) if gsrc else np.zeros(0, np.int64)
    gcol = np.concatenate(gcol).astype(np.int32) if gcol else np.zeros(0, np.int32)
    fptr = np.concatenate([lptr, lptr[-1] + np.cumsum(gcnt)]).astype(np.int32)
    fcol = np.concatenate([plan.local_col.astype(np.int32), gcol])
    src = np.concatenate([own_src, gsrc])
    # every stored B[j][c] with c owned must come from an own or ghost row
    ghost_set = np.zeros(n, bool)
    ghost_set[plan.ghost_gid] = True
    ghost_set[r0:r1] = True
    rows_of = np.repeat(np.arange(n), np.diff(ptr))
    hit = (col >= r0) & (col < r1)
    if not np.all(ghost_set[rows_of[hit]]):
        raise ValueError("distributed B^T: the SAI pattern is not symmetric (a row outside the ghost layer "
                         "references an owned column)")
    # transposed view: entries (j, c) of the local matrix with c < n_own
    nrows_f = n_own + len(plan.ghost_gid)
    frow = np.repeat(np.arange(nrows_f), np.diff(fptr))
    gid = np.concatenate([np.arange(r0, r1), plan.ghost_gid]).astype(np.int64)
    sel = np.nonzero(fcol < n_own)[0]
    order = np.lexsort((gid[frow[sel]], fcol[sel]))
    q = sel[order]
    tptr = np.zeros(n_own + 1, np.int64)
    np.add.at(tptr, fcol[q] + 1, 1)
    tptr = np.cumsum(tptr).astype(np.int32)
    return (fptr, fcol, src), (tptr, frow[q].astype(np.int32), q.astype(np.int32))


def split_b_rows(Bg, n, bs, plan: Plan):
    """split_b_index with the values gathered on the host: (fptr, fcol, own
    values (a view of Bg), ghost values), (tptr, tcol, tperm)."""
    ptr, col, val = (np.asarray(a) for a in Bg)
    (fptr, fcol, src), tpat = split_b_index(ptr, col, n, plan)
    k0, k1 = int(ptr[plan.r0]), int(ptr[plan.r1])
    own_val = val[k0 * bs * bs:k1 * bs * bs]
    gk = src[k1 - k0:]
    ghost_val = val.reshape(-1, bs * bs)[gk].reshape(-1) if gk.size else np.zeros(0)
    return (fptr, fcol, own_val, ghost_val), tpat


def boundary_rows(ptr, col, n_own):
    """(interior, boundary) local rows of a rank's operator: boundary rows
    read a ghost column (>= n_own), interior rows only owned ones."""
    ptr, col = np.asarray(ptr), np.asarray(col)
    rows_of = np.repeat(np.arange(len(ptr) - 1), np.diff(ptr))
    bnd = np.zeros(len(ptr) - 1, bool)
    bnd[rows_of[col >= n_own]] = True
    return np.nonzero(~bnd)[0].astype(np.int32), np.nonzero(bnd)[0].astype(np.int32)


def pgs_schedule(n_own, ptr, col, reverse):
    """Wavefronts of the rank's processor-block GS sweep (ldgmg_pgs_schedule):
    a list of local row arrays, one per launch."""
    p = np.ascontiguousarray(ptr, np.int32)
    c = np.ascontiguousarray(col, np.int32)
    nl = C.c_int()
    check(lib.ldgmg_pgs_schedule(int(n_own), p.ctypes.data, c.ctypes.data, int(reverse), None, None, C.byref(nl)))
    rows = np.empty(max(n_own, 1), np.int32)
    lp = np.empty(nl.value + 1, np.int32)
    check(lib.ldgmg_pgs_schedule(int(n_own), p.ctypes.data, c.ctypes.data, int(reverse), rows.ctypes.data,
                                 lp.ctypes.data, C.byref(nl)))
    return [rows[lp[i]:lp[i + 1]] for i in range(nl.value)]


class GpuOps:
    """Local compute through the C ABI (the product path)."""

    def __init__(self, ctx):
        import torch
        self.torch = torch
        self.ctx = ctx

    def tensor(self, n):
        return self.torch.zeros(int(n), dtype=self.torch.float64, device="cuda")

    def itensor(self, a):
        return self.torch.as_tensor(np.ascontiguousarray(a, np.int32)).cuda()

    def upload(self, a):
        return self.torch.as_tensor(np.ascontiguousarray(a, np.float64)).cuda()

    def matrix(self, brows, bcols, bs, ptr, col, val):
        h = C.c_void_p()
        p = np.ascontiguousarray(ptr, np.int32)
        c = np.ascontiguousarray(col, np.int32)
        v = np.ascontiguousarray(val, np.float64)
        check(lib.ldgmg_bsr_upload_ex(self.ctx.h, int(brows), int(bcols), bs, bs, p.ctypes.data, c.ctypes.data,
                                      v.ctypes.data, 1, C.byref(h)))  # LDGMG_BSR_UNSORTED_COLUMNS
        return _Handle(h, lib.ldgmg_bsr_destroy)

    def matrix_pieces(self, brows, bcols, bs, ptr, col, pieces):
        """Upload the pattern, then the values piece by piece (no host
        concatenation): pieces = [(first_block, row-major values), ...]."""
        h = C.c_void_p()
        p = np.ascontiguousarray(ptr, np.int32)
        c = np.ascontiguousarray(col, np.int32)
        check(lib.ldgmg_bsr_upload_ex(self.ctx.h, int(brows), int(bcols), bs, bs, p.ctypes.data, c.ctypes.data,
                                      None, 1, C.byref(h)))
        M = _Handle(h, lib.ldgmg_bsr_destroy)
        for k0, v in pieces:
            v = np.ascontiguousarray(v, np.float64)
            if v.size:
                check(lib.ldgmg_bsr_set_values(self.ctx.h, M.h, int(k0), int(v.size // (bs * bs)), v.ctypes.data))
        return M

    def gather_matrix(self, M, brows, bcols, ptr, col, src_blocks):
        """New device matrix: pattern (ptr, col), block q = M's block src_blocks[q] (device copy)."""
        h = C.c_void_p()
        p = np.ascontiguousarray(ptr, np.int32)
        c = np.ascontiguousarray(col, np.int32)
        q = np.ascontiguousarray(src_blocks, np.int64)
        check(lib.ldgmg_bsr_gather(self.ctx.h, M.h, int(brows), int(bcols), p.ctypes.data, c.ctypes.data,
                                   q.ctypes.data, C.byref(h)))
        return _Handle(h, lib.ldgmg_bsr_destroy)

    def prefix_view(self, M, nrows):
        h = C.c_void_p()
        check(lib.ldgmg_bsr_row_prefix_view(self.ctx.h, M.h, int(nrows), C.byref(h)))
        V = _Handle(h, lib.ldgmg_bsr_destroy)
        V.base = M  # keep the values alive
        return V

    def transposed_view(self, M, brows, bcols, ptr, col, perm):
        h = C.c_void_p()
        p, c, q = (np.ascontiguousarray(a, np.int32) for a in (ptr, col, perm))
        check(lib.ldgmg_bsr_transposed_view(self.ctx.h, M.h, int(brows), int(bcols), p.ctypes.data, c.ctypes.data,
                                            q.ctypes.data, C.byref(h)))
        V = _Handle(h, lib.ldgmg_bsr_destroy)
        V.base = M
        return V

    def residual_rows(self, A, b, x_ext, r, rows):
        check(lib.ldgmg_residual_rows(self.ctx.h, A.h, b.data_ptr(), x_ext.data_ptr(), r.data_ptr(),
                                      rows.data_ptr(), int(rows.numel())))

    def spmv_add_rows(self, B, r_ext, x_own, rows):
        check(lib.ldgmg_spmv_add_rows(self.ctx.h, B.h, r_ext.data_ptr(), x_own.data_ptr(), rows.data_ptr(),
                                      int(rows.numel())))

    def factors(self, n, bs, V, lam, s):
        h = C.c_void_p()
        arrs = [np.ascontiguousarray(a, np.float64) for a in (V, lam, s)]
        check(lib.ldgmg_factors_upload(self.ctx.h, int(n), int(bs), *(a.ctypes.data for a in arrs), C.byref(h)))
        return _Handle(h, lib.ldgmg_factors_destroy)

    def transfer(self, n_fine, n_coarse, parent, orth, dim, bss, ncomp, K):
        from .api import Transfer
        return Transfer(self.ctx, n_fine, n_coarse, parent, orth, dim, bss, ncomp, K)

    def residual(self, A, b, x_ext, r):
        check(lib.ldgmg_residual(self.ctx.h, A.h, b.data_ptr(), x_ext.data_ptr(), r.data_ptr()))

    def spmv_add(self, B, r_ext, x_own):
        check(lib.ldgmg_spmv_add(self.ctx.h, B.h, r_ext.data_ptr(), x_own.data_ptr()))

    def spmv(self, A, x_ext, y):
        check(lib.ldgmg_spmv(self.ctx.h, A.h, x_ext.data_ptr(), y.data_ptr()))

    def relax(self, A, F, b, x_src, x_live, x_out, omega):
        check(lib.ldgmg_relax(self.ctx.h, A.h, F.h, b.data_ptr(), x_src.data_ptr(), x_live.data_ptr(),
                              x_out.data_ptr(), float(omega)))

    def relax_rows(self, A, F, b, x_src, x_live, x_out, omega, rows):
        check(lib.ldgmg_relax_rows(self.ctx.h, A.h, F.h, b.data_ptr(), x_src.data_ptr(), x_live.data_ptr(),
                                   x_out.data_ptr(), float(omega), rows.data_ptr(), int(rows.numel())))

    def restrict(self, T, rf, rc):
        T.restrict(rf, rc)

    def prolong(self, T, xc, xf):
        T.interpolate_add(xc, xf)

    def gather(self, x, idx, n, bs, out):
        check(lib.ldgmg_gather_blocks(self.ctx.h, x.data_ptr(), idx.data_ptr(), int(n), int(bs), out.data_ptr()))

    def project_partials(self, v_own, N, r0, r1, bs, offs, kval, part):
        check(lib.ldgmg_project_partials(self.ctx.h, v_own.data_ptr(), int(N), int(r0), int(r1), int(bs),
                                         offs.data_ptr(), int(offs.numel()), float(kval), part.data_ptr()))

    def project_apply(self, v_own, N, r0, r1, bs, offs, kval, part):
        check(lib.ldgmg_project_apply(self.ctx.h, v_own.data_ptr(), int(N), int(r0), int(r1), int(bs),
                                      offs.data_ptr(), int(offs.numel()), float(kval), part.data_ptr()))

    def to_host(self, t):
        return t.detach().cpu().numpy()


class _Handle:
    def __init__(self, h, dtor):
        self.h, self._dtor = h, dtor

    def __del__(self):
        if getattr(self, "h", None):
            self._dtor(self.h)
            self.h = None


class Exchanger:
    """Ghost exchange of one plan: pack owned blocks the neighbours need,
    point-to-point send / receive straight into the ghost slots."""

    def __init__(self, plan: Plan, bs: int, ops, dist, group, rank):
        self.plan, self.bs, self.ops, self.dist, self.group, self.rank = plan, bs, ops, dist, group, rank
        self.idx = ops.itensor(plan.send_idx if len(plan.send_idx) else np.zeros(1, np.int32))
        self.sendbuf = ops.tensor(max(1, len(plan.send_idx)) * bs)
        self.so, self.ro = plan.send_off, plan.recv_off

    def start(self, x_ext):
        """Pack and post the exchange; returns the pending works (None when
        this plan has no traffic).  With NCCL the transfers run on NCCL's
        stream while the caller's stream goes on (the interior rows)."""
        p, bs = self.plan, self.bs
        if p.n_ghost == 0 and len(p.send_idx) == 0:
            return None
        self.ops.gather(x_ext, self.idx, len(p.send_idx), bs, self.sendbuf)
        # the op list only depends on the (fixed) buffers: build it once per target
        key = x_ext.data_ptr() if hasattr(x_ext, "data_ptr") else id(x_ext)
        reqs = self._reqs.get(key) if hasattr(self, "_reqs") else None
        if reqs is None:
            P2P = self.dist.P2POp
            reqs = []
            for q in range(len(p.send_count)):
                if q == self.rank:
                    continue
                if p.send_count[q]:
                    reqs.append(P2P(self.dist.isend, self.sendbuf[self.so[q] * bs:self.so[q + 1] * bs], q,
                                    self.group))
                if p.recv_count[q]:
                    g0 = (p.n_own + self.ro[q]) * bs
                    reqs.append(P2P(self.dist.irecv, x_ext[g0:g0 + int(p.recv_count[q]) * bs], q, self.group))
            if not hasattr(self, "_reqs"):
                self._reqs = {}
            self._reqs[key] = reqs
        return self.dist.batch_isend_irecv(reqs) if reqs else None

    @staticmethod
    def finish(works):
        """Make the caller's stream (NCCL) / the host (gloo) wait for the ghosts."""
        for w in works or ():
            w.wait()

    def __call__(self, x_ext):
        self.finish(self.start(x_ext))


class DistMultigrid:
    """The V-cycle over P ranks (see module docstring).

    `levels[l]` (global, host numpy): dict with A=(ptr, col, val), n, bs and,
    for smoothed levels, B=(ptr,col,val) for SAI or factors=(V, lam, s) for
    Jacobi; `transfers[l]` = (parent_of, orthant_of); K injection matrices;
    `coarse` = an object with .vcycle(x, b) on full coarse vectors (the
    agglomerated tail, e.g. an api.Multigrid over levels >= ld)."""

    def __init__(self, ops, dist, cfg, levels, transfers, K, dim, bss, ncomp, kernel_offsets, coarse_factory,
                 group=None, min_rows_per_rank=64, overlap=True, overlap_min_rows=2048):
        """overlap: split every pass of a level with >= overlap_min_rows owned
        rows into interior rows (run while the ghost layer is in flight) and
        boundary rows (after it landed); per-row arithmetic is unchanged, so
        the result is bit-identical either way."""
        self.ops, self.dist, self.cfg, self.group = ops, dist, cfg, group
        kind = cfg.smoother.kind
        self.dim = dim
        self.rank = dist.get_rank(group)
        self.P = dist.get_world_size(group)
        self.bs = levels[0]["bs"]
        self.koffs = list(kernel_offsets)
        self.N0 = levels[0]["n"]
        depth = len(levels)
        self.ld = partition_depth([lv["n"] for lv in levels], transfers, self.P, min_rows_per_rank)
        if self.ld == 0:
            raise ValueError("distributed V-cycle needs at least one partitioned level")
        bs = self.bs
        self.L = []
        for l in range(self.ld):
            lv = levels[l]
            n = lv["n"]
            if "A_local" in lv:  # built on the device already (device_partial_levels)
                pa, lrA = lv["plan_A"], lv["A_local_pattern"]
                Aloc = lv["A_local"]
            else:
                pa = partition_level(*lv["A"][:2], n, self.P, self.rank)
                lrA = local_rows(*lv["A"], bs, bs, pa)
                Aloc = ops.matrix(pa.n_own, pa.n_own + pa.n_ghost, bs, *lrA)
            d = {"n": n, "plan": pa, "A": Aloc, "xA": Exchanger(pa, bs, ops, dist, group, self.rank),
                 "nnzA": int(lrA[0][-1])}
            if "B_full" in lv or "B" in lv:
                # one device matrix for both sweep directions: the rank's B
                # rows (forward, a row-prefix view) and, behind them, the
                # ghost rows' owned-column blocks the B^T rows read through
                # a transposed view (no host transpose, no B^T copy)
                if "B_full" in lv:
                    pb, Bfull = lv["plan_B"], lv["B_full"]
                    (fptr, fcol), (tptr, tcol, tperm) = lv["B_index"]
                    nf = pb.n_own + pb.n_ghost
                    nnz_own = int(fptr[pb.n_own])
                else:
                    pb = partition_level(lv["B"][0], lv["B"][1], n, self.P, self.rank)
                    (fptr, fcol, own_val, ghost_val), (tptr, tcol, tperm) = split_b_rows(lv["B"], n, bs, pb)
                    nf = pb.n_own + pb.n_ghost
                    nnz_own = int(fptr[pb.n_own])
                    Bfull = ops.matrix_pieces(nf, nf, bs, fptr, fcol, [(0, own_val), (nnz_own, ghost_val)])
                d["Bfull"] = Bfull
                d["B"] = ops.prefix_view(Bfull, pb.n_own)
                d["BT"] = ops.transposed_view(Bfull, pb.n_own, nf, tptr, tcol, tperm)
                d["nnzB"], d["nnzBT"] = nnz_own, int(tptr[-1])
                d["xB"] = Exchanger(pb, bs, ops, dist, group, self.rank)
                d["ngB"] = d["ngBT"] = pb.n_ghost
                if overlap and pb.n_own >= overlap_min_rows:
                    d["splitB"] = tuple(ops.itensor(a) for a in boundary_rows(fptr[:pb.n_own + 1], fcol[:nnz_own],
                                                                                   pb.n_own))
                    d["splitBT"] = tuple(ops.itensor(a) for a in boundary_rows(tptr, tcol, pb.n_own))
            if overlap and pa.n_own >= overlap_min_rows:
                d["splitA"] = tuple(ops.itensor(a) for a in boundary_rows(lrA[0], lrA[1], pa.n_own))
            if kind == L.PROC_BLOCK_GS:
                if cfg.smoother.partitions != self.P:
                    raise ValueError("distributed processor-block GS needs smoother.partitions == ranks "
                                     "(each rank is one partition, smoothers.hpp:87-94)")
                d["pgs"] = [[ops.itensor(w) for w in pgs_schedule(pa.n_own, lrA[0], lrA[1], rev)]
                            for rev in (0, 1)]
            if "factors_own" in lv and kind != L.SAI:
                d["F"] = ops.factors(pa.n_own, bs, *lv["factors_own"])
            elif "factors" in lv and kind != L.SAI:  # Jacobi, coloured GS, processor-block GS
                V, lam, s = lv["factors"]
                a, b = pa.r0, pa.r1
                d["F"] = ops.factors(pa.n_own, bs, V[a * bs * bs:b * bs * bs], lam[a * bs:b * bs], s[a * bs:b * bs])
            if "colour" in lv:  # coloured GS: own rows per colour, local ids, ascending
                col_own = np.asarray(lv["colour"])[pa.r0:pa.r1]
                nc = int(np.max(lv["colour"])) + 1 if len(lv["colour"]) else 0
                d["crows"] = [ops.itensor(np.nonzero(col_own == c)[0]) for c in range(nc)]
            # transfer to level l+1, rank-local (nested ranges)
            parent, orth = transfers[l]
            nc = levels[l + 1]["n"]
            c0, c1 = self.rank * nc // self.P, (self.rank + 1) * nc // self.P
            lp = np.asarray(parent[pa.r0:pa.r1])
            bounds = [q * n // self.P for q in range(self.P + 1)]
            if any(int(parent[bq - 1]) == int(parent[bq]) for bq in bounds[1:-1] if 0 < bq < n):
                raise ValueError("a rank boundary splits a sibling group; use P dividing N/2^dim")
            if l + 1 < self.ld and (lp.min(initial=c0) < c0 or lp.max(initial=c0) >= c1):
                raise ValueError("partition ranges are not nested across levels")
            # children-induced coarse ranges of every rank (agglomeration gather)
            d["cranges"] = [(int(parent[bounds[q]]) if bounds[q] < n else nc,
                             int(parent[bounds[q + 1] - 1]) + 1 if bounds[q + 1] > bounds[q] else int(parent[bounds[q]]))
                            for q in range(self.P)]
            d["c0"], d["c1"], d["nc"] = c0, c1, nc
            d["T"] = ops.transfer(pa.n_own, c1 - c0 if l + 1 < self.ld else nc, lp - (c0 if l + 1 < self.ld else 0),
                                  orth[pa.r0:pa.r1], dim, bss, ncomp, K)
            d["x"] = ops.tensor((pa.n_own + pa.n_ghost) * bs)
            d["snap"] = ops.tensor((pa.n_own + pa.n_ghost) * bs)
            d["r"] = ops.tensor(pa.n_own * bs)
            d["rext"] = ops.tensor((pa.n_own + max(d.get("ngB", 0), d.get("ngBT", 0))) * bs)
            d["b"] = ops.tensor(pa.n_own * bs)
            self.L.append(d)
        # agglomerated tail: levels >= ld on every rank
        self.coarse = coarse_factory(self.ld)
        nct = levels[self.ld]["n"]
        self.rc_full = ops.tensor(nct * bs)
        self.xc_full = ops.tensor(nct * bs)
        self.rc_part = ops.tensor(nct * bs)  # this rank's restriction contribution

    # ---------------------------------------------------------------- smoothing
    def _pass(self, l, key, xkey, x_ext, full, split):
        """One operator application after its ghost exchange: with a split,
        the interior rows run while the ghosts are in flight."""
        d = self.L[l]
        if split is None:
            d[xkey](x_ext)
            full()
            return
        works = d[xkey].start(x_ext)
        split(d[key][0])
        Exchanger.finish(works)
        split(d[key][1])

    def residual(self, l, b, x_ext, r):
        d = self.L[l]
        sp = d.get("splitA")
        self._pass(l, "splitA", "xA", x_ext, lambda: self.ops.residual(d["A"], b, x_ext, r),
                   sp and (lambda rows: self.ops.residual_rows(d["A"], b, x_ext, r, rows)))

    def smooth(self, l, b, sweep):
        d, bs = self.L[l], self.bs
        n_own = d["plan"].n_own
        x_ext = d["x"]
        kind = self.cfg.smoother.kind
        if kind == L.SAI:
            rext = d["rext"]
            self.residual(l, b, x_ext, rext[:n_own * bs])
            key = "B" if sweep == L.SWEEP_FORWARD else "BT"
            M, x_own = d[key], x_ext[:n_own * bs]
            sp = d.get("split" + key)
            self._pass(l, "split" + key, "xB", rext, lambda: self.ops.spmv_add(M, rext, x_own),
                       sp and (lambda rows: self.ops.spmv_add_rows(M, rext, x_own, rows)))
        elif kind == L.JACOBI:
            d["xA"](x_ext)
            snap = d["snap"]
            snap.copy_(x_ext)
            self.ops.relax(d["A"], d["F"], b, snap, snap[:n_own * bs], x_ext[:n_own * bs], self.cfg.smoother.omega)
        elif kind == L.COLOURED_GS:
            # colours ascending (reverse for a reverse sweep), one ghost
            # exchange per colour phase (smoothers.hpp:417-425), omega = 1
            crows = d["crows"]
            order = range(len(crows)) if sweep == L.SWEEP_FORWARD else range(len(crows) - 1, -1, -1)
            for c in order:
                d["xA"](x_ext)
                if crows[c].numel():
                    self.ops.relax_rows(d["A"], d["F"], b, x_ext, x_ext[:n_own * bs], x_ext[:n_own * bs], 1.0,
                                        crows[c])
        elif kind == L.PROC_BLOCK_GS:
            # each rank is one partition (smoothers.hpp:426-436): its ghosts
            # are exchanged once and stay frozen for the sweep (= the
            # reference's sweep-start snapshot of the other partitions); its
            # own rows are relaxed in sequential order, one wavefront of the
            # dependency DAG per launch, in-partition neighbours read live
            d["xA"](x_ext)
            own = x_ext[:n_own * bs]
            for rows in d["pgs"][0 if sweep == L.SWEEP_FORWARD else 1]:
                self.ops.relax_rows(d["A"], d["F"], b, x_ext, own, own, self.cfg.smoother.omega, rows)
        else:
            raise ValueError("distributed V-cycle supports the Jacobi, coloured GS, processor-block GS and SAI "
                             "smoothers")

    # ---------------------------------------------------------------- V-cycle
    def _vcycle(self, l, b):
        """x lives in self.L[l]['x'][:own]; b is the owned right-hand side."""
        d, bs = self.L[l], self.bs
        n_own = d["plan"].n_own
        x_ext = d["x"]
        for _ in range(self.cfg.nu1):
            self.smooth(l, b, self.cfg.pre)
        self.residual(l, b, x_ext, d["r"])
        if l + 1 < self.ld:
            nxt = self.L[l + 1]
            self.ops.restrict(d["T"], d["r"], nxt["b"])
            nxt["x"].zero_()
            self._vcycle(l + 1, nxt["b"])
            self.ops.prolong(d["T"], nxt["x"][:nxt["plan"].n_own * bs], x_ext[:n_own * bs])
        else:
            # agglomerate: every rank restricts its children into the full
            # coarse vector (disjoint parents), all-reduce assembles it exactly
            self.rc_part.zero_()
            self.ops.restrict(d["T"], d["r"], self.rc_part)
            self._allgather_coarse(l)
            self.xc_full.zero_()
            self.coarse.vcycle(self.xc_full, self.rc_full)
            self.ops.prolong(d["T"], self.xc_full, x_ext[:n_own * bs])
        for _ in range(self.cfg.nu2):
            self.smooth(l, b, self.cfg.post)

    def _allgather(self, mine, sizes):
        """all_gather of unevenly sized slices (padded to the largest)."""
        m = max(sizes)
        buf = self.ops.tensor(m)
        buf[:mine.numel()] = mine
        parts = [self.ops.tensor(m) for _ in sizes]
        self.dist.all_gather(parts, buf, group=self.group)
        return [p[:sz] for p, sz in zip(parts, sizes)]

    def _allgather_coarse(self, l):
        d, bs = self.L[l], self.bs
        cr = d["cranges"]
        a, b = cr[self.rank]
        parts = self._allgather(self.rc_part[a * bs:b * bs], [(y - x) * bs for x, y in cr])
        for (x, y), part in zip(cr, parts):
            self.rc_full[x * bs:y * bs] = part

    def project(self, v_own):
        """multigrid.hpp:243-245 with the dot in the reference's sequential
        order over all elements (P-independent, = single-GPU strict mode)."""
        if not self.koffs:
            return
        bs, n_own = self.bs, self.L[0]["plan"].n_own
        kval = 1.0 / np.sqrt(float(self.N0))
        sizes = [(q + 1) * self.N0 // self.P - q * self.N0 // self.P for q in range(self.P)]
        for off in self.koffs:
            own = v_own[off::bs][:n_own] * kval
            parts = self._allgather(own.contiguous(), sizes)
            prods = np.concatenate([self.ops.to_host(p) for p in parts])
            dsum = float(np.add.accumulate(np.concatenate([[0.0], prods]))[-1])
            v_own[off::bs][:n_own] += (-dsum) * kval

    def apply(self, b_own, x_own):
        """Multigrid::apply on the owned slices (multigrid.hpp:90-101): the
        V-cycle from zero on the projected right-hand side, then project."""
        d, bs = self.L[0], self.bs
        n_own = d["plan"].n_own
        if self.koffs:
            bp = b_own.clone()
            self.project(bp)
        else:
            bp = b_own
        d["x"].zero_()
        self._vcycle(0, bp)
        x_own.copy_(d["x"][:n_own * bs])
        self.project(x_own)

    def project_fast(self, v_own):
        """Kernel projection in the deterministic FAST mode, entirely on the
        device (capturable): the 256 fixed global ranges of the single-GPU
        fast projection, each summed by the rank that owns it, all-gathered
        and combined in the same fixed tree -- bit-identical to the single-GPU
        fast mode and independent of P (P must divide 256)."""
        if not self.koffs:
            return
        torch = self.ops.torch
        N0, bs = self.N0, self.bs
        r0, r1 = self.owned_range()
        if not hasattr(self, "_pf"):
            nc = len(self.koffs)
            owner = np.array([next(q for q in range(self.P)
                                   if q * N0 // self.P <= k * N0 // 256 < (q + 1) * N0 // self.P)
                              for k in range(256)])
            idx = torch.as_tensor(np.concatenate([owner * (256 * nc) + c * 256 + np.arange(256)
                                                  for c in range(nc)])).to(self.ops.tensor(1).device)
            self._pf = {"offs": self.ops.itensor(np.asarray(self.koffs, np.int32)),
                        "part": self.ops.tensor(256 * nc), "all": [self.ops.tensor(256 * nc) for _ in range(self.P)],
                        "idx": idx, "full": self.ops.tensor(256 * nc),
                        "kval": 1.0 / np.sqrt(float(N0))}
        pf = self._pf
        pf["part"].zero_()
        self.ops.project_partials(v_own, N0, r0, r1, bs, pf["offs"], pf["kval"], pf["part"])
        self.dist.all_gather(pf["all"], pf["part"], group=self.group)
        pf["full"].copy_(torch.cat(pf["all"])[pf["idx"]])
        self.ops.project_apply(v_own, N0, r0, r1, bs, pf["offs"], pf["kval"], pf["full"])

    def _cycle_body(self, x_own, b_own, fast):
        d, bs = self.L[0], self.bs
        n_own = d["plan"].n_own
        d["x"][:n_own * bs] = x_own
        self._vcycle(0, b_own)
        x_own.copy_(d["x"][:n_own * bs])
        if fast:
            self.project_fast(x_own)
        else:
            self.project(x_own)

    def cycle(self, x_own, b_own, fast=False):
        """Multigrid::cycle on the owned slices (multigrid.hpp:82-85).  fast:
        device-side deterministic projection (and the captured graph when
        enable_graph succeeded) instead of the reference-order host sum."""
        g = getattr(self, "_graph", None)
        if fast and g is not None:
            self._gx.copy_(x_own)
            self._gb.copy_(b_own)
            g.replay()
            x_own.copy_(self._gx)
            return
        self._cycle_body(x_own, b_own, fast)

    def enable_graph(self, x_probe, b_probe):
        """Capture one fast-mode cycle (V-cycle kernels, NCCL exchanges and
        the device projection) as a CUDA graph, then VALIDATE it: a replay
        from (x_probe, b_probe) must equal an eager fast cycle bit for bit.
        Any capture error or mismatch leaves the eager path in place.
        Returns True when the graph is in use."""
        torch = self.ops.torch
        self._graph = None
        ok, g = False, None
        if torch.cuda.current_stream() == torch.cuda.default_stream():
            self._graph_error = "graph capture needs the hierarchy on a non-default stream"
        try:
            if getattr(self, "_graph_error", None):
                raise RuntimeError(self._graph_error)
            x_e = x_probe.clone()
            self._cycle_body(x_e, b_probe, True)  # eager reference + warm-up
            self._gx = x_probe.clone()
            self._gb = b_probe.clone()
            g = torch.cuda.CUDAGraph()
            torch.cuda.synchronize()
            n0 = L.launch_count()
            with torch.cuda.graph(g, stream=torch.cuda.current_stream()):
                self._cycle_body(self._gx, self._gb, True)
            self.graph_kernels = L.launch_count() - n0  # our kernels per replay
            ok = True
        except Exception as exc:  # capture not supported for some op: stay eager
            self._graph_error = repr(exc)
            ok = False
        # a replay posts NCCL exchanges: replay only if EVERY rank captured
        # (a lone replay would wait forever on its peers)
        capt = torch.tensor([1 if ok else 0], dtype=torch.int32, device=x_probe.device)
        self.dist.all_reduce(capt, op=self.dist.ReduceOp.MIN, group=self.group)
        if int(capt.item()) == 1:
            try:
                self._gx.copy_(x_probe)
                self._gb.copy_(b_probe)
                g.replay()
                torch.cuda.synchronize()
                ok = bool(torch.equal(self._gx, x_e))
            except Exception as exc:
                self._graph_error = repr(exc)
                ok = False
        else:
            ok = False
        # every rank reaches this collective, whatever happened above
        okt = torch.tensor([1 if ok else 0], dtype=torch.int32, device=x_probe.device)
        self.dist.all_reduce(okt, op=self.dist.ReduceOp.MIN, group=self.group)
        if int(okt.item()) == 1:
            self._graph = g
        return self._graph is not None

    def cycle_costs(self):
        """(DOF-updates, algorithmic HBM bytes) of one cycle on THIS rank: its
        rows of the partitioned levels (SURVEY.md §8d formulas on the local
        operators) plus, on rank 0 only, the agglomerated tail (replicated
        work is counted once).  Sum over ranks = the whole job."""
        W, bs = 8.0, self.bs
        dof = byts = 0.0
        nu1, nu2 = self.cfg.nu1, self.cfg.nu2
        for l, d in enumerate(self.L):
            n = d["plan"].n_own
            dof += (nu1 + nu2) * n * bs
            if self.cfg.smoother.kind == L.SAI:
                sweep = lambda key: W * (bs * bs * (d["nnzA"] + d["nnz" + key]) + 6.0 * n * bs)  # noqa: E731
                byts += nu1 * sweep("B" if self.cfg.pre == L.SWEEP_FORWARD else "BT")
                byts += nu2 * sweep("B" if self.cfg.post == L.SWEEP_FORWARD else "BT")
            else:
                byts += (nu1 + nu2) * W * (bs * bs * (d["nnzA"] - n) + (bs * bs + 2.0 * bs) * n + 3.0 * n * bs)
            byts += W * (bs * bs * d["nnzA"] + 3.0 * n * bs)  # residual
            nc = d["c1"] - d["c0"] if l + 1 < self.ld else n // (1 << self.dim)
            byts += W * (bs * n + bs * nc) + W * (bs * nc + 2.0 * bs * n)  # restrict + prolong
        if self.rank == 0:
            td, tb = self.coarse.cycle_costs()
            dof += td
            byts += tb
        return dof, byts

    def symmetric(self):
        """symmetric_plan (multigrid.hpp:41-43)"""
        return self.cfg.smoother.kind == L.JACOBI or self.cfg.pre != self.cfg.post

    def owned_range(self, level=0):
        p = self.L[level]["plan"]
        return p.r0, p.r1


def from_problem(ctx, problem, cfg, dist, group=None, min_rows_per_rank=64):
    """Distributed hierarchy from the built-in setup.  Setup data (SAI B,
    factors) come from a replicated single-GPU hierarchy on each rank."""
    from .api import DeviceBsr, Multigrid, MultigridConfig, Transfer
    full = Multigrid(ctx, cfg, problem)
    depth = problem.depth
    levels, transfers = [], []
    for l in range(depth):
        n, bs, _ = problem.level_shape(l)
        lv = {"n": n, "bs": bs, "A": problem.level_matrix(l)}
        if l + 1 < depth:
            S = full.smoother(l)
            if cfg.smoother.kind == L.SAI:
                lv["B"] = S.sai_matrix()
            else:
                lv["factors"] = S.diag_factors()
                if cfg.smoother.kind == L.COLOURED_GS:
                    lv["colour"] = S.colours()
            transfers.append(problem.level_transfer(l))
        levels.append(lv)
    K = problem.injection()

    def coarse_factory(ld):
        As = [DeviceBsr(ctx, levels[l]["n"], levels[l]["n"], levels[l]["bs"], levels[l]["bs"], *levels[l]["A"])
              for l in range(ld, depth)]
        Ts = [Transfer(ctx, levels[l]["n"], levels[l + 1]["n"], *transfers[l], problem.dim, problem.bs_scalar,
                       problem.n_comp, K) for l in range(ld, depth - 1)]
        ccfg = MultigridConfig(smoother=cfg.smoother, pre=cfg.pre, post=cfg.post, nu1=cfg.nu1, nu2=cfg.nu2,
                               bottom_max_elements=cfg.bottom_max_elements, bottom_tol=cfg.bottom_tol, min_depth=1)
        return Multigrid(ctx, ccfg, levels=As, transfers=Ts,
                         system_kind=L.SYSTEM_STOKES if problem.n_comp > 1 else L.SYSTEM_SCALAR, dim=problem.dim,
                         n_comp=problem.n_comp, bs_scalar=problem.bs_scalar)

    offs = []
    if problem.kernel_constants:
        offs += [c * problem.bs_scalar for c in range(1 if problem.n_comp == 1 else problem.dim)]
    if problem.kernel_pressure:
        offs.append(problem.dim * problem.bs_scalar)
    dm = DistMultigrid(GpuOps(ctx), dist, cfg, levels, transfers, K, problem.dim, problem.bs_scalar,
                       problem.n_comp, offs, coarse_factory, group=group, min_rows_per_rank=min_rows_per_rank)
    dm._full = full
    return dm


# --------------------------------------------------------- distributed setup
def sai_halo_hops(spec, smoother) -> int:
    """Face-graph layers a rank must assemble around its range.  SAI: every
    SAI column its B / B^T rows need must be solved exactly -- B row i needs
    the columns c in pattern^l(i), whose least-squares rows reach
    pattern^(2l+1) of the range, so (2l+1) operator hops.  Other smoothers:
    one operator hop, so that the rank sees its neighbours' rows that
    reference it (the ghost send lists are derived from them).  One operator
    hop is one face layer, two for the stress-form Stokes operator (its
    G_j^T G_i cross terms couple diagonal neighbours) and for any problem with
    a phase interface: the u-hat donor of an interface face is the more
    viscous side (ldg_core.hpp:122-127), so G_k^T D G_k couples elements two
    face layers apart there."""
    two = (spec.kind == L.SYSTEM_STOKES and spec.gamma != 0.0) or \
        (spec.phase_shape != L.PHASE_SINGLE and spec.mu_in != spec.mu_out)
    r_a = 2 if two else 1
    if smoother.kind != L.SAI:
        return r_a
    return (2 * smoother.level + 1) * r_a


def csr_ring(ptr, col, seed_mask, hops):
    """Rows within `hops` steps of the seed rows on the block pattern."""
    ptr, col = np.asarray(ptr), np.asarray(col)
    mask = np.asarray(seed_mask, bool).copy()
    frontier = np.nonzero(mask)[0]
    for _ in range(hops):
        if frontier.size == 0:
            break
        idx = np.concatenate([col[ptr[r]:ptr[r + 1]] for r in frontier]) if frontier.size else np.zeros(0, int)
        new = np.unique(idx[~mask[idx]])
        mask[new] = True
        frontier = new
    return mask


def local_sai(ptr, col, val, n, bs, r0, r1, level, build):
    """B columns for the rank's SAI rows from its assembled rows only.

    (ptr, col, val) is the rank's global-numbered level operator with the
    rows of its range plus halo assembled (the others empty).  The operator
    restricted to the assembled rows H is renumbered locally; `build(lptr,
    lcol, lval, nH, col_mask)` returns the local B (any solver of the
    reference's build_sai); the columns pattern^level(range) -- all B / B^T
    rows of the range need -- are solved.  Returns B in global numbering
    (rows of H, global-shaped CSR).  Every returned entry of the range's
    rows and columns equals the global build's (tests/test_distributed_setup.py)."""
    ptr, col, val = np.asarray(ptr), np.asarray(col), np.asarray(val)
    H = np.nonzero(np.diff(ptr) > 0)[0]
    loc = np.full(n, -1, np.int64)
    loc[H] = np.arange(H.size)
    keep = loc[col] >= 0
    rows_of = np.repeat(np.arange(n), np.diff(ptr))
    kk = np.nonzero(keep)[0]
    lrows = loc[rows_of[kk]]
    lptr = np.zeros(H.size + 1, np.int32)
    np.add.at(lptr, lrows + 1, 1)
    lptr = np.cumsum(lptr).astype(np.int32)
    lcol = loc[col[kk]].astype(np.int32)
    lval = val.reshape(-1, bs * bs)[kk].reshape(-1)
    own = np.zeros(n, bool)
    own[r0:r1] = True
    want = csr_ring(ptr, col, own, level)
    if not np.all(np.diff(ptr)[want] > 0):
        raise ValueError("distributed setup: halo too small for the SAI columns of this range")
    Bp, Bc, Bv = build(lptr, lcol, lval, int(H.size), want[H])
    Bp, Bc = np.asarray(Bp), np.asarray(Bc)
    gptr = np.zeros(n + 1, np.int64)
    gptr[H + 1] = np.diff(Bp)
    gptr = np.cumsum(gptr).astype(np.int32)
    return gptr, H[Bc].astype(np.int32), np.asarray(Bv)


def distributed_colouring(ptr, col, n, nranks, rank, bcast):
    """colour_mesh (smoothers.hpp:63-84: greedy, elements ascending, smallest
    colour unused by the already-coloured neighbours) from the ranks' own rows
    only.  An element's colour depends on its lower-numbered neighbours, which
    live on this or lower ranks, so the ranks colour their ranges in rank
    order; `bcast(q, colours_of_q)` (collective) publishes rank q's range
    before rank q+1 starts.  Identical to the sequential colouring."""
    ptr, col = np.asarray(ptr), np.asarray(col)
    colour = np.full(n, -1, np.int32)
    for q in range(nranks):
        r0, r1 = q * n // nranks, (q + 1) * n // nranks
        mine = np.zeros(r1 - r0, np.int32)
        if q == rank:
            for e in range(r0, r1):
                nb = col[ptr[e]:ptr[e + 1]]
                used = set(int(colour[j]) for j in nb if j != e and colour[j] >= 0)
                c = 0
                while c in used:
                    c += 1
                colour[e] = c
            mine = colour[r0:r1].copy()
        colour[r0:r1] = bcast(q, mine)
    return colour


def partial_levels(prob, cfg, nranks, rank, min_rows_per_rank, sai_fn, factors_fn, bcast=None):
    """Per-level data for DistMultigrid from a Problem.partial: global-shaped
    operators (assembled rows only), transfers, and for the distributed
    levels the rank's SAI matrix (local_sai with `sai_fn`) or diagonal
    factors (`factors_fn(diag_blocks) -> (V, lam, s)` of the rank's rows)."""
    depth = prob.depth
    shapes = [prob.level_shape(l) for l in range(depth)]
    ld = partition_depth([sh[0] for sh in shapes], [prob.level_transfer(l) for l in range(depth - 1)], nranks,
                         min_rows_per_rank)
    levels, transfers = [], []
    for l in range(depth):
        n, bs, _ = shapes[l]
        lv = {"n": n, "bs": bs, "A": prob.level_matrix(l)}
        if l >= ld and prob.level_partial(l):
            raise ValueError(f"distributed setup: level {l} is assembled per rank but agglomerated by the "
                             "V-cycle (a rank boundary splits a sibling group); raise min_rows_per_rank")
        if l + 1 < depth:
            transfers.append(prob.level_transfer(l))
            if l < ld:
                r0, r1 = rank * n // nranks, (rank + 1) * n // nranks
                if cfg.smoother.kind == L.SAI:
                    lv["B"] = local_sai(*lv["A"], n, bs, r0, r1, cfg.smoother.level, sai_fn)
                else:
                    ptr, col, val = lv["A"]
                    dk = np.array([ptr[e] + int(np.nonzero(col[ptr[e]:ptr[e + 1]] == e)[0][0])
                                   for e in range(r0, r1)], np.int64)
                    D = np.asarray(val).reshape(-1, bs * bs)[dk].reshape(-1)
                    V, lam, s = factors_fn(l, r0, r1, bs, D)
                    Vg, lg, sg = np.zeros(n * bs * bs), np.zeros(n * bs), np.zeros(n * bs)
                    Vg[r0 * bs * bs:r1 * bs * bs], lg[r0 * bs:r1 * bs], sg[r0 * bs:r1 * bs] = V, lam, s
                    lv["factors"] = (Vg, lg, sg)
                    if cfg.smoother.kind == L.COLOURED_GS:
                        lv["colour"] = distributed_colouring(ptr, col, n, nranks, rank, bcast)
        levels.append(lv)
    return levels, transfers


def device_partial_levels(ctx, prob, cfg, nranks, rank, min_rows_per_rank, bcast):
    """Per-level data for DistMultigrid with every operator value kept on
    the device: the rank's rows + halo are ASSEMBLED on the device
    (Problem.partial with device assembly, global numbering, other rows
    empty); its SAI columns pattern^l(range) are solved by the column-masked
    GPU build directly on that operator (rows outside the halo enter no
    requested problem); the rank's local A and its B (own rows + the ghost
    rows' owned-column blocks, split_b_index) are cut out of the global-
    shaped device matrices by block gathers.  Only index arrays (ptr / col /
    plans) live on the host; the values never cross PCIe.  Levels past the
    partitioned ones are built in full (device operators) for the
    agglomerated tail."""
    from .api import DeviceBsr, Smoother, SmootherConfig, sai_build
    ops = GpuOps(ctx)
    depth = prob.depth
    shapes = [prob.level_shape(l) for l in range(depth)]
    transfers = [prob.level_transfer(l) for l in range(depth - 1)]
    ld = partition_depth([sh[0] for sh in shapes], transfers, nranks, min_rows_per_rank)
    kind = L.SYSTEM_STOKES if prob.n_comp > 1 else L.SYSTEM_SCALAR
    levels = []
    for l in range(depth):
        n, bs, _ = shapes[l]
        ptr, col = prob.level_pattern(l)
        lv = {"n": n, "bs": bs, "pattern": (ptr, col)}
        if l < ld:
            r0, r1 = rank * n // nranks, (rank + 1) * n // nranks
            Ad = prob.device_operator(ctx, l)
            pa = partition_level(ptr, col, n, nranks, rank)
            lptr = (np.asarray(ptr[r0:r1 + 1], np.int64) - int(ptr[r0])).astype(np.int32)
            lv["plan_A"], lv["A_local_pattern"] = pa, (lptr, pa.local_col)
            whole = pa.n_ghost == 0 and r0 == 0 and r1 == n  # one rank: the local operator IS the global one
            lv["A_local"] = Ad if whole else ops.gather_matrix(
                Ad, pa.n_own, pa.n_own + pa.n_ghost, lptr, pa.local_col,
                np.arange(int(ptr[r0]), int(ptr[r1]), dtype=np.int64))
            if cfg.smoother.kind == L.SAI:
                own = np.zeros(n, bool)
                own[r0:r1] = True
                want = csr_ring(ptr, col, own, cfg.smoother.level)
                Bd, _ = sai_build(ctx, Ad, kind, prob.n_velocity, cfg.smoother.level, cfg.smoother.zeta,
                                  cfg.smoother.cache, col_mask=want)
                del Ad
                Bp, Bc = Bd.pattern()
                pb = partition_level(Bp, Bc, n, nranks, rank)
                (fptr, fcol, src), tpat = split_b_index(Bp, Bc, n, pb)
                nf = pb.n_own + pb.n_ghost
                lv["B_full"] = Bd if (whole and pb.n_ghost == 0) else ops.gather_matrix(Bd, nf, nf, fptr, fcol, src)
                del Bd
                lv["plan_B"], lv["B_index"] = pb, ((fptr, fcol), tpat)
            else:
                dk = np.array([int(ptr[e]) + int(np.nonzero(col[ptr[e]:ptr[e + 1]] == e)[0][0])
                               for e in range(r0, r1)], np.int64)
                n_own = r1 - r0
                Dm = ops.gather_matrix(Ad, n_own, n_own, np.arange(n_own + 1, dtype=np.int32),
                                       np.arange(n_own, dtype=np.int32), dk)
                del Ad
                Dw = DeviceBsr.adopt(ctx, Dm.h)
                Dm.h = None  # ownership moves to Dw
                lv["factors_own"] = Smoother(ctx, Dw, SmootherConfig.jacobi(cfg.smoother.omega)).diag_factors()
                if cfg.smoother.kind == L.COLOURED_GS:
                    lv["colour"] = distributed_colouring(ptr, col, n, nranks, rank, bcast)
        else:
            if prob.level_partial(l):  # the setup assembled only a halo here, but the V-cycle agglomerates it
                raise ValueError(f"distributed setup: level {l} is assembled per rank but agglomerated by the "
                                 "V-cycle (a rank boundary splits a sibling group); raise min_rows_per_rank")
            lv["A_dev"] = prob.device_operator(ctx, l)
        levels.append(lv)
    return levels, transfers


def from_problem_partial(ctx, spec, cfg, dist, group=None, min_rows_per_rank=64, any_n=None, overlap=True,
                         device=True, overlap_min_rows=2048):
    """Distributed hierarchy with DISTRIBUTED setup: each rank builds only
    its rows plus the SAI halo, solves only the SAI columns its rows need
    (column-masked GPU build), and computes the diagonal factors of its own
    rows on the GPU.  device=True (default): operators assembled and cut on
    the device (device_partial_levels, no operator values on the host);
    False: host assembly (Problem.partial + partial_levels, the path the CPU
    tests drive).  The agglomerated tail is set up in full on every rank (it
    is small).  Results are identical either way and to from_problem
    (tests/test_distributed_setup.py)."""
    from .api import DeviceBsr, Multigrid, MultigridConfig, Problem, Smoother, SmootherConfig, Transfer, sai_build
    rank, P = dist.get_rank(group), dist.get_world_size(group)
    if any_n is None:  # extension A1 for non-power-of-two meshes (C5 at 48^3)
        any_n = spec.n & (spec.n - 1) != 0
    prob = Problem.partial(spec, P, rank, sai_halo_hops(spec, cfg.smoother), min_rows_per_rank,
                           min_depth=cfg.min_depth, bottom_max_elements=cfg.bottom_max_elements, any_n=any_n,
                           device_assembly=device)
    depth = prob.depth
    kind = L.SYSTEM_STOKES if prob.n_comp > 1 else L.SYSTEM_SCALAR

    def bcast(q, mine):
        import torch
        t = torch.as_tensor(np.ascontiguousarray(mine, np.int32).astype(np.int64)).cuda()
        dist.broadcast(t, src=dist.get_global_rank(group, q) if group is not None else q, group=group)
        return t.cpu().numpy().astype(np.int32)

    if device:
        levels, transfers = device_partial_levels(ctx, prob, cfg, P, rank, min_rows_per_rank, bcast)
    else:
        def gpu_sai(lptr, lcol, lval, nH, mask):
            A = DeviceBsr(ctx, nH, nH, prob.bs, prob.bs, lptr, lcol, lval)
            B, _ = sai_build(ctx, A, kind, prob.n_velocity, cfg.smoother.level, cfg.smoother.zeta,
                             cfg.smoother.cache, col_mask=mask)
            return B.download()

        def gpu_factors(l, r0, r1, bs, D):
            n_own = r1 - r0
            Ad = DeviceBsr(ctx, n_own, n_own, bs, bs, np.arange(n_own + 1, dtype=np.int32),
                           np.arange(n_own, dtype=np.int32), D)
            return Smoother(ctx, Ad, SmootherConfig.jacobi(cfg.smoother.omega)).diag_factors()

        levels, transfers = partial_levels(prob, cfg, P, rank, min_rows_per_rank, gpu_sai, gpu_factors, bcast)
    K = prob.injection()

    def coarse_factory(ld_):
        As = [levels[l]["A_dev"] if "A_dev" in levels[l] else
              DeviceBsr(ctx, levels[l]["n"], levels[l]["n"], levels[l]["bs"], levels[l]["bs"], *levels[l]["A"])
              for l in range(ld_, depth)]
        Ts = [Transfer(ctx, levels[l]["n"], levels[l + 1]["n"], *transfers[l], prob.dim, prob.bs_scalar,
                       prob.n_comp, K) for l in range(ld_, depth - 1)]
        ccfg = MultigridConfig(smoother=cfg.smoother, pre=cfg.pre, post=cfg.post, nu1=cfg.nu1, nu2=cfg.nu2,
                               bottom_max_elements=cfg.bottom_max_elements, bottom_tol=cfg.bottom_tol, min_depth=1)
        return Multigrid(ctx, ccfg, levels=As, transfers=Ts, system_kind=kind, dim=prob.dim, n_comp=prob.n_comp,
                         bs_scalar=prob.bs_scalar)

    offs = []
    if prob.kernel_constants:
        offs += [c * prob.bs_scalar for c in range(1 if prob.n_comp == 1 else prob.dim)]
    if prob.kernel_pressure:
        offs.append(prob.dim * prob.bs_scalar)
    dm = DistMultigrid(GpuOps(ctx), dist, cfg, levels, transfers, K, prob.dim, prob.bs_scalar, prob.n_comp, offs,
                       coarse_factory, group=group, min_rows_per_rank=min_rows_per_rank, overlap=overlap,
                       overlap_min_rows=overlap_min_rows)
    dm._problem = prob
    return dm


# ------------------------------------------------------ distributed Krylov
_libm = C.CDLL("libm.so.6")
_libm.hypot.restype = C.c_double
_libm.hypot.argtypes = [C.c_double, C.c_double]


def fit_rate(residuals):
    """fit_rate (krylov.hpp:54-95) restated: (rho, eta, classification,
    low_confidence) from a residual history (same libm log/exp)."""
    import math
    r = list(residuals)
    if not r or r[0] <= 0.0:
        return 0.0, 0.0, 0, True
    floor = 1e-13 * r[0]
    K = 0
    while K + 1 < len(r) and r[K + 1] > floor:
        K += 1
    low = True
    if K >= 2:
        sx = sy = sxx = sxy = 0.0
        for k in range(1, K + 1):
            x, y = float(k), math.log(r[k])
            sx += x
            sy += y
            sxx += x * x
            sxy += x * y
        slope = (K * sxy - sx * sy) / (K * sxx - sx * sx)
        low = K < 3
    elif len(r) >= 2:
        slope = math.log(max(r[1], 1e-300)) - math.log(r[0])
    else:
        return 0.0, 0.0, 0, True
    rho = math.exp(slope)
    if rho >= 1.0:
        return rho, float("inf"), 2, low
    eta = math.log(0.1) / math.log(rho)
    return rho, eta, (0 if eta < 2.0 else 1 if eta < 10.0 else 2), low


class DistKrylov:
    """pcg / gmres_left / estimate_eta (krylov.hpp:117-306) over the ranks of
    a DistMultigrid: vectors are the owned slices, the operator is the level-0
    spmv after a ghost exchange, the preconditioner DistMultigrid.apply.
    Dot products gather the per-entry products and sum them in the global
    entry order on every rank (the reference's sequential dot, blockla.hpp:60-63),
    so every scalar -- and the whole residual history -- is independent of the
    rank count and bit-identical to the single-process reference."""

    def __init__(self, dm):
        self.dm = dm
        self.ops, self.bs = dm.ops, dm.bs
        d = dm.L[0]
        self.n_own = d["plan"].n_own * self.bs
        N0, P = dm.N0, dm.P
        self.sizes = [((q + 1) * N0 // P - q * N0 // P) * self.bs for q in range(P)]

    def dot(self, a, b):
        parts = self.dm._allgather((a * b).contiguous(), self.sizes)
        prods = np.concatenate([[0.0]] + [self.ops.to_host(p) for p in parts])
        return float(np.add.accumulate(prods)[-1])

    def norm2(self, a):
        return float(np.sqrt(self.dot(a, a)))

    def spmv(self, x_own, y_own):
        d = self.dm.L[0]
        x_ext = d["x"]
        x_ext[:self.n_own] = x_own
        d["xA"](x_ext)
        self.ops.spmv(d["A"], x_ext, y_own)

    def apply(self, b_own):
        x = self.ops.tensor(self.n_own)
        self.dm.apply(b_own, x)
        return x

    @staticmethod
    def _axpy(alpha, x, y):  # y += alpha * x, two roundings (no FMA)
        y.add_(x * alpha)

    def pcg(self, b_own, tol=1e-12, maxit=60):
        if not self.dm.symmetric():
            raise L.InvalidArgument("pcg: preconditioner plan is not symmetric")
        res, it, conv, brk = [], 0, False, False
        x = self.ops.tensor(self.n_own)
        r = b_own.clone()
        z = self.apply(r)
        rz = self.dot(r, z)
        r0 = float(np.sqrt(max(rz, 0.0)))
        res.append(r0)
        if r0 == 0.0:
            return x, self._report(res, 0, True, False)
        p = z.clone()
        Ap = self.ops.tensor(self.n_own)
        for k in range(1, maxit + 1):
            self.spmv(p, Ap)
            pAp = self.dot(p, Ap)
            if pAp <= 0.0:
                brk = True
                break
            alpha = rz / pAp
            self._axpy(alpha, p, x)
            self._axpy(-alpha, Ap, r)
            z = self.apply(r)
            rz_new = self.dot(r, z)
            rk = float(np.sqrt(max(rz_new, 0.0)))
            res.append(rk)
            it = k
            if rz_new < 0.0:
                brk = True
                break
            if rk <= tol * r0:
                conv = True
                break
            beta = rz_new / rz
            rz = rz_new
            p.mul_(beta).add_(z)
        return x, self._report(res, it, conv, brk)

    def gmres(self, b_own, tol=1e-12, maxit=60):
        res, conv, brk = [], False, False
        x = self.ops.tensor(self.n_own)
        r0 = self.apply(b_own)
        g0 = self.norm2(r0)
        res.append(g0)
        if g0 == 0.0:
            return x, self._report(res, 0, True, False)
        r0.mul_(1.0 / g0)
        basis = [r0]
        H = np.zeros((maxit + 1, maxit))
        gamma = np.zeros(maxit + 1)
        cs, sn = np.zeros(maxit), np.zeros(maxit)
        gamma[0] = g0
        m = 0
        Av = self.ops.tensor(self.n_own)
        for j in range(maxit):
            self.spmv(basis[j], Av)
            w = self.apply(Av)
            pre_norm = self.norm2(w)
            for i in range(j + 1):
                h = self.dot(w, basis[i])
                H[i, j] = h
                self._axpy(-h, basis[i], w)
            hn = self.norm2(w)
            H[j + 1, j] = hn
            happy = hn <= 1e-14 * pre_norm
            if not happy:
                w.mul_(1.0 / hn)
                basis.append(w)
            for i in range(j):
                t = float(cs[i]) * float(H[i, j]) + float(sn[i]) * float(H[i + 1, j])
                H[i + 1, j] = -float(sn[i]) * float(H[i, j]) + float(cs[i]) * float(H[i + 1, j])
                H[i, j] = t
            d = _libm.hypot(float(H[j, j]), float(H[j + 1, j]))
            if d == 0.0:
                cs[j], sn[j] = 1.0, 0.0
            else:
                cs[j], sn[j] = float(H[j, j]) / d, float(H[j + 1, j]) / d
            H[j, j] = d
            H[j + 1, j] = 0.0
            gamma[j + 1] = -float(sn[j]) * float(gamma[j])
            gamma[j] = float(cs[j]) * float(gamma[j])
            m = j + 1
            rk = abs(float(gamma[j + 1]))
            res.append(rk)
            if happy:
                brk = conv = True
                break
            if rk <= tol * g0:
                conv = True
                break
        y = np.zeros(m)
        for i in range(m - 1, -1, -1):
            s_ = float(gamma[i])
            for k in range(i + 1, m):
                s_ -= float(H[i, k]) * float(y[k])
            y[i] = s_ / float(H[i, i]) if H[i, i] != 0.0 else 0.0
        for i in range(m):
            self._axpy(float(y[i]), basis[i], x)
        return x, self._report(res, m, conv, brk)

    @staticmethod
    def _report(res, iters, conv, brk):
        rho, eta, cls, low = fit_rate(res)
        return {"residuals": np.array(res), "iterations": iters, "converged": conv, "breakdown": brk, "rho": rho,
                "eta": eta, "classification": ["fast", "slow", "nonconvergent"][cls], "low_confidence": low}

    def estimate_eta(self, kind=L.KRYLOV_GMRES, seed=0, tol=1e-12, maxit=60):
        """estimate_eta (krylov.hpp:293-306): the seeded random rhs (generated
        in full on every rank), the kernel projected out in the reference's
        order, zero guess, then CG or GMRES on the ranks."""
        from .api import random_rhs
        N0, bs = self.dm.N0, self.bs
        b = random_rhs(N0, bs, seed)
        offs = self.dm.koffs
        if offs:
            kv = 1.0 / np.sqrt(float(N0))
            s_ = float(np.add.accumulate(np.full(N0 + 1, kv * kv) * np.r_[0.0, np.ones(N0)])[-1])
            nrm = float(np.sqrt(s_))
            if nrm > 1e-10:
                kv = kv * (1.0 / nrm)
            for off in offs:
                kvec = np.zeros(N0 * bs)
                kvec[off::bs] = kv
                dd = float(np.add.accumulate(np.r_[0.0, b * kvec])[-1])
                b = b + (-dd) * kvec
        r0_, r1_ = self.dm.owned_range()
        b_own = self.ops.upload(b[r0_ * bs:r1_ * bs]) if hasattr(self.ops, "upload") else \
            self.ops.torch.as_tensor(b[r0_ * bs:r1_ * bs].copy())
        if kind == L.KRYLOV_CG:
            _, rep = self.pcg(b_own, tol, maxit)
        else:
            _, rep = self.gmres(b_own, tol, maxit)
        return rep
