"""TEST INFRASTRUCTURE -- numpy restatement of the reference's hot path
(the CPU oracle the GPU kernels are checked against).  Never imported by the
product.  Pinned against the compiled reference (oracle/_ref, see
tests/test_oracle_pin.py) and against the committed golden fixtures
(tests/golden/, generated from the reference by tests/golden/make_golden.py).

Every function reproduces the reference's floating-point evaluation order
exactly (numpy elementwise ops are IEEE single-rounding, never fused), so the
port is BIT-identical to the reference built against oracle/shim:

  spmv            blockla.hpp:136-154   per block s = 0 + b[r,0]x0 + b[r,1]x1 + ...
                                        y_i = 0 + s_k1 + s_k2 + ... (CSR order)
  spmv_transpose  blockla.hpp:157-176   rows i ascending scatter
  pattern_power   blockla.hpp:197-226
  pinv_apply      blockla.hpp:330-339   t = V^T r (k ascending), cut, V t
  colour_mesh     smoothers.hpp:63-84
  relax           smoothers.hpp:496-518 (Jacobi :411-416, coloured GS :417-425)
  SAI sweep       smoothers.hpp:437-448
  restrict        multigrid.hpp:127-149
  interpolate_add multigrid.hpp:104-123
  v_cycle         multigrid.hpp:247-264, cycle :82-85, apply :90-101
  project_kernel  multigrid.hpp:243-245 (dot/axpy blockla.hpp:60-68)
"""
from __future__ import annotations

import numpy as np


# --------------------------------------------------------------- BSR ops
def _block_dots(val, rbs, cbs, X, transpose=False):
    """s[k, r] = 0 + sum_c B_k[r, c] * X[k, c] sequentially in c
    (transpose: s[k, c] = sum_r B_k[r, c] * X[k, r], r sequential)."""
    B = val.reshape(-1, rbs, cbs)
    if not transpose:
        s = np.zeros((B.shape[0], rbs))
        for c in range(cbs):
            s = s + B[:, :, c] * X[:, c:c + 1]
    else:
        s = np.zeros((B.shape[0], cbs))
        for r in range(rbs):
            s = s + B[:, r, :] * X[:, r:r + 1]
    return s


def _row_slots(ptr):
    ptr = np.asarray(ptr)
    lens = np.diff(ptr)
    return lens, (int(lens.max()) if len(lens) else 0)


def spmv(ptr, col, val, rbs, cbs, x):
    ptr, col = np.asarray(ptr), np.asarray(col)
    brows = len(ptr) - 1
    X = np.asarray(x).reshape(-1, cbs)[col]
    s = _block_dots(np.asarray(val), rbs, cbs, X)
    y = np.zeros((brows, rbs))
    lens, mx = _row_slots(ptr)
    for t in range(mx):
        rows = np.nonzero(lens > t)[0]
        y[rows] = y[rows] + s[ptr[rows] + t]
    return y.reshape(-1)


def spmv_transpose(ptr, col, val, rbs, cbs, bcols, x):
    ptr, col = np.asarray(ptr), np.asarray(col)
    brows = len(ptr) - 1
    rows_of = np.repeat(np.arange(brows), np.diff(ptr))
    X = np.asarray(x).reshape(-1, rbs)[rows_of]
    s = _block_dots(np.asarray(val), rbs, cbs, X, transpose=True)
    y = np.zeros((bcols, cbs))
    # ascending row order per output column j: process block list in CSR order,
    # grouped so that no two blocks in one step hit the same j
    order = np.argsort(col, kind="stable")  # CSR order is already row-ascending
    cj = col[order]
    start = np.searchsorted(cj, np.arange(bcols))
    cnt = np.bincount(col, minlength=bcols)
    for t in range(int(cnt.max()) if len(cnt) else 0):
        js = np.nonzero(cnt > t)[0]
        k = order[start[js] + t]
        y[js] = y[js] + s[k]
    return y.reshape(-1)


def pattern_power(ptr, col, level):
    n = len(ptr) - 1
    out = []
    for i in range(n):
        seen = {i}
        frontier = [i]
        for _ in range(level):
            nxt = []
            for u in frontier:
                for v in col[ptr[u]:ptr[u + 1]]:
                    if v not in seen:
                        seen.add(int(v))
                        nxt.append(int(v))
            frontier = nxt
        out.append(sorted(seen))
    return out


def colour_mesh(ptr, col):
    n = len(ptr) - 1
    colour = [-1] * n
    ncol = 0
    for e in range(n):
        used = [False] * (ncol + 1)
        for j in col[ptr[e]:ptr[e + 1]]:
            if j != e and colour[j] >= 0:
                used[colour[j]] = True
        c = 0
        while used[c]:
            c += 1
        colour[e] = c
        ncol = max(ncol, c + 1)
    return np.array(colour, np.int32)


# ----------------------------------------------------------- smoothers
def pinv_apply(V, lam, r, tol):
    """V column-major n x n (V(k,i) at i*n+k)."""
    n = len(lam)
    Vm = np.asarray(V).reshape(n, n)  # Vm[i, k] = V(k, i)
    lmax = np.max(np.abs(lam)) if n else 0.0
    t = np.zeros(n)
    for k in range(n):
        t = t + Vm[:, k] * r[k]
    cut = np.abs(lam) <= tol * lmax
    t = np.where(cut, 0.0, t / np.where(cut, 1.0, lam))
    x = np.zeros(n)
    for k in range(n):
        x = x + Vm[k, :] * t[k]
    return x


def relax_rows(rows, ptr, col, val, bs, b, x_src, x_live, V, lam, scal, omega, kernel_tol=1e-12):
    """relax (smoothers.hpp:496-518) of the element list `rows`, vectorised
    over elements; returns the new x values for those rows (N_rows x bs)."""
    ptr, col = np.asarray(ptr), np.asarray(col)
    rows = np.asarray(rows)
    Bv = np.asarray(val).reshape(-1, bs, bs)
    Xs = np.asarray(x_src).reshape(-1, bs)
    r = np.asarray(b).reshape(-1, bs)[rows].copy()
    lens = np.diff(ptr)[rows]
    for t in range(int(lens.max()) if len(lens) else 0):
        sel = np.nonzero(lens > t)[0]
        k = ptr[rows[sel]] + t
        offd = col[k] != rows[sel]
        sel, k = sel[offd], k[offd]
        s = np.zeros((len(sel), bs))
        for c in range(bs):
            s = s + Bv[k, :, c] * Xs[col[k], c:c + 1]
        r[sel] = r[sel] - s
    S = np.asarray(scal).reshape(-1, bs)[rows]
    L = np.asarray(lam).reshape(-1, bs)[rows]
    Vm = np.asarray(V).reshape(-1, bs, bs)[rows]  # Vm[e, i, k] = V(k, i)
    u = S * r
    tt = np.zeros_like(u)
    for k in range(bs):
        tt = tt + Vm[:, :, k] * u[:, k:k + 1]
    lmax = np.max(np.abs(L), axis=1, keepdims=True)
    cut = np.abs(L) <= kernel_tol * lmax
    tt = np.where(cut, 0.0, tt / np.where(cut, 1.0, L))
    w = np.zeros_like(u)
    for k in range(bs):
        w = w + Vm[:, k, :] * tt[:, k:k + 1]
    y = S * w
    xe = np.asarray(x_live).reshape(-1, bs)[rows]
    return (1.0 - omega) * xe + omega * y


def jacobi_sweep(ptr, col, val, bs, b, x, V, lam, scal, omega):
    N = len(ptr) - 1
    snap = np.array(x, copy=True)
    out = np.array(x, copy=True).reshape(-1, bs)
    out[:] = relax_rows(np.arange(N), ptr, col, val, bs, b, snap, snap, V, lam, scal, omega)
    return out.reshape(-1)


def gs_sweep(ptr, col, val, bs, b, x, V, lam, scal, colour, reverse=False):
    x = np.array(x, copy=True).reshape(-1, bs)
    nc = int(colour.max()) + 1 if len(colour) else 0
    for ci in range(nc):
        c = nc - 1 - ci if reverse else ci
        rows = np.nonzero(colour == c)[0]
        x[rows] = relax_rows(rows, ptr, col, val, bs, b, x.reshape(-1), x.reshape(-1), V, lam, scal, 1.0)
    return x.reshape(-1)


def pgs_sweep(ptr, col, val, bs, b, x, V, lam, scal, omega, partitions, reverse=False):
    """Processor-block GS (smoothers.hpp:426-436): each partition of
    partition_ranges(N, P) (:87-94) sweeps its elements in order (reverse:
    descending), in-partition neighbours read live, the rest from the
    snapshot.  Element-by-element (pure restatement; small cases only)."""
    N = len(ptr) - 1
    if partitions < 1 or partitions > N:
        raise ValueError("partition_ranges: partition count must lie in [1, N]")
    part = np.empty(N, np.int64)
    for p in range(partitions):
        part[p * N // partitions:(p + 1) * N // partitions] = p
    snap = np.array(x, copy=True)
    live = np.array(x, copy=True).reshape(-1, bs)
    for p in range(partitions):
        s0, s1 = p * N // partitions, (p + 1) * N // partitions
        order = range(s1 - 1, s0 - 1, -1) if reverse else range(s0, s1)
        for e in order:
            # neighbour source per block: live x inside the partition, snapshot outside
            src = np.where(np.repeat(part == part[e], bs), live.reshape(-1), snap)
            live[e] = relax_rows([e], ptr, col, val, bs, b, src, live.reshape(-1), V, lam, scal, omega)[0]
    return live.reshape(-1)


def sai_sweep(A, B, bs, b, x, reverse=False):
    ax = spmv(A[0], A[1], A[2], bs, bs, x)
    r = np.asarray(b) - ax
    if reverse:
        dx = spmv_transpose(B[0], B[1], B[2], bs, bs, len(B[0]) - 1, r)
    else:
        dx = spmv(B[0], B[1], B[2], bs, bs, r)
    return np.asarray(x) + 1.0 * dx


# ------------------------------------------------------------ transfers
def restrict(parent, orth, K, bss, ncomp, n_coarse, rf):
    BS = bss * ncomp
    nk = len(K) // (bss * bss)
    Km = np.asarray(K).reshape(nk, bss, bss)
    src = np.asarray(rf).reshape(-1, ncomp, bss)
    rc = np.zeros((n_coarse, ncomp, bss))
    order = np.argsort(parent, kind="stable")
    cnt = np.bincount(parent, minlength=n_coarse)
    start = np.concatenate([[0], np.cumsum(cnt)[:-1]])
    for t in range(int(cnt.max()) if len(cnt) else 0):
        ps = np.nonzero(cnt > t)[0]
        fs = order[start[ps] + t]
        o = np.asarray(orth)[fs]
        cp = o < 0
        if cp.any():
            rc[ps[cp]] = rc[ps[cp]] + src[fs[cp]]
        m = ~cp
        if m.any():
            s = np.zeros((m.sum(), ncomp, bss))
            Ko = Km[o[m]]  # (n, i, j)
            for i in range(bss):
                s = s + Ko[:, None, i, :] * src[fs[m]][:, :, i:i + 1]
            rc[ps[m]] = rc[ps[m]] + s
    return rc.reshape(-1)


def interpolate_add(parent, orth, K, bss, ncomp, xc, xf):
    nk = len(K) // (bss * bss)
    Km = np.asarray(K).reshape(nk, bss, bss)
    src = np.asarray(xc).reshape(-1, ncomp, bss)[np.asarray(parent)]
    dst = np.array(xf, copy=True).reshape(-1, ncomp, bss)
    o = np.asarray(orth)
    cp = o < 0
    if cp.any():
        dst[cp] = dst[cp] + src[cp]
    m = ~cp
    Ko = Km[o[m]]  # (n, i, j)
    s = np.zeros((m.sum(), ncomp, bss))
    sm = src[m]
    for j in range(bss):
        s = s + Ko[:, None, :, j] * sm[:, :, j:j + 1]
    dst[m] = dst[m] + s
    return dst.reshape(-1)


# ------------------------------------------------------------- V-cycle
class PortMultigrid:
    """The V-cycle on level data extracted from the reference hierarchy."""

    def __init__(self, levels, transfers, K, bottom, cfg, bs_scalar, n_comp, kernel_offsets):
        self.levels, self.transfers, self.K = levels, transfers, K
        self.bottom, self.cfg = bottom, cfg
        self.bss, self.ncomp = bs_scalar, n_comp
        self.koffs = kernel_offsets

    def smooth(self, l, b, x, sweep):
        L = self.levels[l]
        bs = L["bs"]
        kind = self.cfg.smoother.kind
        if kind == 0:
            return jacobi_sweep(*L["A"], bs, b, x, *L["factors"], self.cfg.smoother.omega)
        if kind == 1:
            return gs_sweep(*L["A"], bs, b, x, *L["factors"], L["colour"], reverse=sweep == 1)
        if kind == 2:
            return pgs_sweep(*L["A"], bs, b, x, *L["factors"], self.cfg.smoother.omega,
                             self.cfg.smoother.partitions, reverse=sweep == 1)
        if kind == 3:
            return sai_sweep(L["A"], L["B"], bs, b, x, reverse=sweep == 1)
        raise ValueError("unsupported smoother")

    def v_cycle(self, l, x, b):
        if l + 1 == len(self.levels):
            V, lam = self.bottom
            return pinv_apply(V, lam, b, self.cfg.bottom_tol)
        L = self.levels[l]
        bs = L["bs"]
        for _ in range(self.cfg.nu1):
            x = self.smooth(l, b, x, self.cfg.pre)
        r = np.asarray(b) - spmv(*L["A"], bs, bs, x)
        p, o = self.transfers[l]
        nc = self.levels[l + 1]["n"]
        rc = restrict(p, o, self.K, self.bss, self.ncomp, nc, r)
        xc = self.v_cycle(l + 1, np.zeros(nc * bs), rc)
        x = interpolate_add(p, o, self.K, self.bss, self.ncomp, xc, x)
        for _ in range(self.cfg.nu2):
            x = self.smooth(l, b, x, self.cfg.post)
        return x

    def project(self, v):
        v = np.array(v, copy=True)
        N, bs = self.levels[0]["n"], self.levels[0]["bs"]
        kval = 1.0 / np.sqrt(float(N))
        for off in self.koffs:
            idx = np.arange(N) * bs + off
            d = np.add.accumulate(v[idx] * kval)[-1]
            v[idx] = v[idx] + (-d) * kval
        return v

    def cycle(self, x, b):
        return self.project(self.v_cycle(0, np.asarray(x), np.asarray(b)))

    def apply(self, b):
        N, bs = self.levels[0]["n"], self.levels[0]["bs"]
        if not self.koffs:
            return self.v_cycle(0, np.zeros(N * bs), np.asarray(b))
        bp = self.project(b)
        return self.project(self.v_cycle(0, np.zeros(N * bs), bp))


def from_reference(R, cfg):
    """Build a PortMultigrid from a RefMultigrid's extracted level data."""
    levels = []
    for l in range(R.depth):
        n, bs, _ = R.shape(l)
        L = {"n": n, "bs": bs, "A": R.matrix(l)}
        if l + 1 < R.depth:
            if cfg.smoother.kind == 3:
                L["B"] = R.sai_matrix(l)
            else:
                L["factors"] = R.diag_factors(l)
                if cfg.smoother.kind == 1:
                    L["colour"] = R.colours(l)[0]
        levels.append(L)
    transfers = [R.transfer(l) for l in range(R.depth - 1)]
    K = R.injection() if R.depth > 1 else np.zeros(0)
    offs = []
    if R.kernel_constants:
        offs += [c * R.bs_scalar for c in range(1 if R.n_comp == 1 else R.dim)]
    if R.kernel_pressure:
        offs.append(R.dim * R.bs_scalar)
    return PortMultigrid(levels, transfers, K, R.bottom(), cfg, R.bs_scalar, R.n_comp, offs)
