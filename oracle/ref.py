"""TEST INFRASTRUCTURE -- ctypes binding of the CPU oracle built from the
unmodified reference headers (oracle/_ref/libldgmg_ref.so, see oracle/Makefile
and oracle/ref_capi.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline -- never as part of the product path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libldgmg_ref.so")

# Constants and struct layouts of include/ldgmg_b200.h, the plain-C header
# ref_capi.cpp is compiled against.  Restated here so the oracle never loads
# the product library (bench.py's reference arm and the tests' checker stay
# independent of libldgmg_b200.so).
SWEEP_FORWARD, SWEEP_REVERSE = 0, 1
JACOBI, COLOURED_GS, PROC_BLOCK_GS, SAI = 0, 1, 2, 3
SYSTEM_SCALAR, SYSTEM_STOKES = 0, 1
BC_PERIODIC, BC_DIRICHLET, BC_NEUMANN = 0, 1, 2
PHASE_SINGLE, PHASE_BOXES, PHASE_BALL, PHASE_ELLIPSE = 0, 1, 2, 3


class _SmootherC(C.Structure):
    _fields_ = [("kind", C.c_int), ("omega", C.c_double), ("partitions", C.c_int),
                ("level", C.c_int), ("zeta", C.c_double), ("cache", C.c_int)]


class _MgConfigC(C.Structure):
    _fields_ = [("smoother", _SmootherC), ("pre", C.c_int), ("post", C.c_int),
                ("nu1", C.c_int), ("nu2", C.c_int), ("bottom_max_elements", C.c_int),
                ("bottom_tol", C.c_double), ("min_depth", C.c_int)]


class SaiStats(C.Structure):
    _fields_ = [("rank_deficient_columns", C.c_int), ("cache_hits", C.c_int64),
                ("cache_misses", C.c_int64), ("n_shapes", C.c_int),
                ("shape_rows", C.c_int * 8), ("shape_cols", C.c_int * 8),
                ("shape_count", C.c_int * 8)]

    def ls_dims(self):
        return {(self.shape_rows[i], self.shape_cols[i]): self.shape_count[i]
                for i in range(min(self.n_shapes, 8))}


class _ProblemSpecC(C.Structure):
    _fields_ = [("kind", C.c_int), ("dim", C.c_int), ("n", C.c_int), ("degree", C.c_int),
                ("bc", C.c_int * 6), ("beta", C.c_double), ("beta_p", C.c_double),
                ("gamma", C.c_double), ("delta", C.c_double), ("phase_shape", C.c_int),
                ("center", C.c_double * 3), ("radii", C.c_double * 3),
                ("mu_in", C.c_double), ("mu_out", C.c_double), ("rho_in", C.c_double),
                ("rho_out", C.c_double)]


def _spec_c(spec) -> _ProblemSpecC:
    """Any object with the ProblemSpec attributes (the product's dataclass or
    a types.SimpleNamespace) -> the C struct."""
    s = _ProblemSpecC()
    s.kind, s.dim, s.n, s.degree = spec.kind, spec.dim, spec.n, spec.degree
    for i in range(6):
        s.bc[i] = spec.bc[i]
    s.beta, s.beta_p, s.gamma, s.delta = spec.beta, spec.beta_p, spec.gamma, spec.delta
    s.phase_shape = spec.phase_shape
    for i in range(3):
        s.center[i] = spec.center[i]
        s.radii[i] = spec.radii[i]
    s.mu_in, s.mu_out, s.rho_in, s.rho_out = spec.mu_in, spec.mu_out, spec.rho_in, spec.rho_out
    return s


def _cfg_c(cfg) -> _MgConfigC:
    sm = cfg.smoother
    return _MgConfigC(_SmootherC(sm.kind, sm.omega, sm.partitions, sm.level, sm.zeta, int(sm.cache)), cfg.pre,
                      cfg.post, cfg.nu1, cfg.nu2, cfg.bottom_max_elements, cfg.bottom_tol, cfg.min_depth)


def problem_spec(**kw):
    """A ProblemSpec with the product API's defaults (harness.hpp:30-40)."""
    from types import SimpleNamespace
    d = dict(kind=SYSTEM_SCALAR, dim=2, n=8, degree=1, bc=(BC_PERIODIC,) * 6, beta=-1.0, beta_p=1.0, gamma=0.0,
             delta=0.0, phase_shape=PHASE_SINGLE, center=(0.5, 0.5, 0.5), radii=(0.25, 0.25, 0.25), mu_in=1.0,
             mu_out=1.0, rho_in=1.0, rho_out=1.0)
    d.update(kw)
    return SimpleNamespace(**d)


def mg_config(smoother_kind=SAI, omega=1.0, partitions=1, level=1, zeta=0.1, cache=True, **kw):
    """A MultigridConfig with the reference defaults (multigrid.hpp:26-36)."""
    from types import SimpleNamespace
    sm = SimpleNamespace(kind=smoother_kind, omega=omega, partitions=partitions, level=level, zeta=zeta, cache=cache)
    d = dict(smoother=sm, pre=SWEEP_FORWARD, post=SWEEP_REVERSE, nu1=3, nu2=3, bottom_max_elements=64,
             bottom_tol=1e-10, min_depth=2)
    d.update(kw)
    return SimpleNamespace(**d)


def available() -> bool:
    return os.path.exists(REF_LIB)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{REF_LIB} not built (make -C oracle)")
        _lib = C.CDLL(REF_LIB)
        P, I, D, LL = C.c_void_p, C.c_int, C.c_double, C.c_longlong
        IP, LLP = C.POINTER(C.c_int), C.POINTER(C.c_longlong)
        sigs = {
            "ref_last_error": ([], C.c_char_p),
            "ref_mg_create": ([C.POINTER(_ProblemSpecC), C.POINTER(_MgConfigC)], P),
            "ref_mg_destroy": ([P], None),
            "ref_mg_depth": ([P], I),
            "ref_level_shape": ([P, I, IP, IP, LLP], I),
            "ref_level_matrix": ([P, I, P, P, P], I),
            "ref_level_rhs": ([P, I, P], I),
            "ref_system_info": ([P, IP, IP, IP, IP, IP, IP], I),
            "ref_level_transfer": ([P, I, P, P], I),
            "ref_injection": ([P, P], I),
            "ref_diag_factors": ([P, I, P, P, P], I),
            "ref_colours": ([P, I, P, IP], I),
            "ref_sai_nnzb": ([P, I, LLP], I),
            "ref_sai_matrix": ([P, I, P, P, P], I),
            "ref_sai_stats": ([P, I, C.POINTER(SaiStats)], I),
            "ref_bottom_size": ([P], I),
            "ref_bottom": ([P, P, P], I),
            "ref_kernel": ([P, IP, P], I),
            "ref_spmv": ([P, I, P, P, I], I),
            "ref_smoother_apply": ([P, I, P, P, I], I),
            "ref_restrict": ([P, I, P, P], I),
            "ref_interpolate_add": ([P, I, P, P], I),
            "ref_cycle": ([P, P, P], I),
            "ref_apply": ([P, P, P], I),
            "ref_solve": ([P, P, P, D, I, P, IP], I),
            "ref_cycles_parallel": ([P, P, I, I, C.POINTER(D)], I),
            "ref_cache_new": ([], P),
            "ref_cache_free": ([P], None),
            "ref_cache_entries": ([P], LL),
            "ref_mg_create_shared": ([C.POINTER(_ProblemSpecC), C.POINTER(_MgConfigC), P], P),
            "ref_cycles_multi": ([C.POINTER(P), I, P, I, C.POINTER(D)], I),
            "ref_random_rhs": ([I, I, C.c_ulonglong, P], I),
            "ref_eta": ([P, I, C.c_ulonglong, D, I, P, IP, IP, IP, C.POINTER(D), C.POINTER(D)], I),
            "ref_bsr_spmv": ([I, I, I, I, P, P, P, P, P, I, C.POINTER(C.c_ulonglong)], I),
            "ref_dump_block_coo": ([I, I, I, I, P, P, P, C.c_char_p], I),
            "ref_pattern_power_nnz": ([I, P, P, I, LLP], I),
            "ref_pattern_power": ([I, P, P, I, P, P], I),
            "ref_dense_lstsq": ([I, I, I, P, P, P, IP], I),
            "ref_sym_eig": ([I, P, P, P], I),
            "ref_sai_build": ([I, I, I, I, I, P, P, P, I, D, I], P),
            "ref_sai_raw_nnzb": ([P], LL),
            "ref_sai_raw_matrix": ([P, P, P, P], None),
            "ref_sai_raw_stats": ([P, C.POINTER(SaiStats)], None),
            "ref_sai_raw_free": ([P], None),
            "ref_balance_vector": ([I, I, I, I, I, P, P, P, D, P], I),
            "ref_colour_mesh": ([I, P, P, P], I),
        }
        for name, (args, res) in sigs.items():
            f = getattr(_lib, name)
            f.argtypes = args
            f.restype = res
    return _lib


class RefError(Exception):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def _chk(rc):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def _p(a):
    return a.ctypes.data


class RefMultigrid:
    """The reference Multigrid (multigrid.hpp:45-274) on a catalogue problem."""

    def __init__(self, spec, cfg, cache=None):
        """`cache`: an optional SaiCache shared with other hierarchies
        (MultigridConfig::cache, multigrid.hpp:35)."""
        self.spec, self.cfg, self.cache = spec, cfg, cache
        cs, cc = _spec_c(spec), _cfg_c(cfg)
        if cache is None:
            h = lib().ref_mg_create(C.byref(cs), C.byref(cc))
        else:
            h = lib().ref_mg_create_shared(C.byref(cs), C.byref(cc), cache.h)
        if not h:
            raise RefError(-1, lib().ref_last_error().decode())
        self.h = h
        self._destroy = lib().ref_mg_destroy  # bound now: module globals are gone at interpreter exit
        self.depth = lib().ref_mg_depth(h)
        dim, nc, bss, kc, kp, nv = (C.c_int() for _ in range(6))
        _chk(lib().ref_system_info(h, *(C.byref(v) for v in (dim, nc, bss, kc, kp, nv))))
        self.dim, self.n_comp, self.bs_scalar = dim.value, nc.value, bss.value
        self.kernel_constants, self.kernel_pressure, self.n_velocity = kc.value, kp.value, nv.value

    def __del__(self):
        if getattr(self, "h", None):
            self._destroy(self.h)
            self.h = None

    def shape(self, l):
        n, bs, nnzb = C.c_int(), C.c_int(), C.c_longlong()
        _chk(lib().ref_level_shape(self.h, l, C.byref(n), C.byref(bs), C.byref(nnzb)))
        return n.value, bs.value, nnzb.value

    def matrix(self, l):
        n, bs, nnzb = self.shape(l)
        ptr = np.empty(n + 1, np.int32)
        col = np.empty(max(nnzb, 1), np.int32)
        val = np.empty(max(nnzb * bs * bs, 1))
        _chk(lib().ref_level_matrix(self.h, l, _p(ptr), _p(col), _p(val)))
        return ptr, col[:nnzb], val[: nnzb * bs * bs]

    def transfer(self, l):
        n = self.shape(l)[0]
        p = np.empty(n, np.int32)
        o = np.empty(n, np.int32)
        _chk(lib().ref_level_transfer(self.h, l, _p(p), _p(o)))
        return p, o

    def injection(self):
        K = np.empty((1 << self.dim) * self.bs_scalar ** 2)
        _chk(lib().ref_injection(self.h, _p(K)))
        return K

    def diag_factors(self, l):
        n, bs, _ = self.shape(l)
        V, lam, s = np.empty(n * bs * bs), np.empty(n * bs), np.empty(n * bs)
        _chk(lib().ref_diag_factors(self.h, l, _p(V), _p(lam), _p(s)))
        return V, lam, s

    def colours(self, l):
        n = self.shape(l)[0]
        c = np.empty(n, np.int32)
        nc = C.c_int()
        _chk(lib().ref_colours(self.h, l, _p(c), C.byref(nc)))
        return c, nc.value

    def sai_matrix(self, l):
        n, bs, _ = self.shape(l)
        nnzb = C.c_longlong()
        _chk(lib().ref_sai_nnzb(self.h, l, C.byref(nnzb)))
        ptr = np.empty(n + 1, np.int32)
        col = np.empty(nnzb.value, np.int32)
        val = np.empty(nnzb.value * bs * bs)
        _chk(lib().ref_sai_matrix(self.h, l, _p(ptr), _p(col), _p(val)))
        return ptr, col, val

    def sai_stats(self, l):
        st = SaiStats()
        _chk(lib().ref_sai_stats(self.h, l, C.byref(st)))
        return st

    def bottom(self):
        n = lib().ref_bottom_size(self.h)
        V, lam = np.empty(n * n), np.empty(n)
        _chk(lib().ref_bottom(self.h, _p(V), _p(lam)))
        return V, lam

    def kernel(self):
        nk = C.c_int()
        _chk(lib().ref_kernel(self.h, C.byref(nk), None))
        n, bs, _ = self.shape(0)
        out = np.empty(max(nk.value, 1) * n * bs)
        _chk(lib().ref_kernel(self.h, C.byref(nk), _p(out)))
        return out[: nk.value * n * bs].reshape(nk.value, n * bs)

    def spmv(self, l, x, transpose=False):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty_like(x)
        _chk(lib().ref_spmv(self.h, l, _p(x), _p(y), int(transpose)))
        return y

    def smoother_apply(self, l, b, x, sweep):
        b = np.ascontiguousarray(b, np.float64)
        x = np.array(x, np.float64, copy=True)
        _chk(lib().ref_smoother_apply(self.h, l, _p(b), _p(x), int(sweep)))
        return x

    def restrict(self, l, rf):
        rf = np.ascontiguousarray(rf, np.float64)
        nc, bs, _ = self.shape(l + 1)
        rc = np.empty(nc * bs)
        _chk(lib().ref_restrict(self.h, l, _p(rf), _p(rc)))
        return rc

    def interpolate_add(self, l, xc, xf):
        xc = np.ascontiguousarray(xc, np.float64)
        xf = np.array(xf, np.float64, copy=True)
        _chk(lib().ref_interpolate_add(self.h, l, _p(xc), _p(xf)))
        return xf

    def cycle(self, x, b):
        x = np.array(x, np.float64, copy=True)
        b = np.ascontiguousarray(b, np.float64)
        _chk(lib().ref_cycle(self.h, _p(x), _p(b)))
        return x

    def apply(self, b):
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty_like(b)
        _chk(lib().ref_apply(self.h, _p(b), _p(x)))
        return x

    def solve(self, b, tol=1e-10, maxit=100):
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty_like(b)
        hist = np.empty(maxit + 1)
        it = C.c_int()
        _chk(lib().ref_solve(self.h, _p(b), _p(x), float(tol), int(maxit), _p(hist), C.byref(it)))
        return x, hist[: it.value + 1], it.value

    def cycles_parallel(self, b, ncycles, nthreads):
        b = np.ascontiguousarray(b, np.float64)
        sec = C.c_double()
        _chk(lib().ref_cycles_parallel(self.h, _p(b), int(ncycles), int(nthreads), C.byref(sec)))
        return sec.value

    def eta(self, kind=1, seed=0, tol=1e-12, maxit=60):
        res = np.empty(maxit + 2)
        nres, iters, conv = C.c_int(), C.c_int(), C.c_int()
        rho, eta = C.c_double(), C.c_double()
        _chk(lib().ref_eta(self.h, kind, seed, tol, maxit, _p(res), C.byref(nres), C.byref(iters),
                           C.byref(conv), C.byref(rho), C.byref(eta)))
        return dict(residuals=res[: nres.value], iterations=iters.value, converged=bool(conv.value),
                    rho=rho.value, eta=eta.value)


class SaiCache:
    """The reference's SaiCache (smoothers.hpp:242-250), shareable across hierarchies."""

    def __init__(self):
        self.h = lib().ref_cache_new()
        self._free = lib().ref_cache_free

    def entries(self):
        return int(lib().ref_cache_entries(self.h))

    def __del__(self):
        if getattr(self, "h", None):
            self._free(self.h)
            self.h = None


def cycles_multi(hierarchies, b, ncycles):
    """`ncycles` V-cycles on each hierarchy, one thread per hierarchy, all
    started together; wall seconds (ref_cycles_multi)."""
    b = np.ascontiguousarray(b, np.float64)
    arr = (C.c_void_p * len(hierarchies))(*[m.h for m in hierarchies])
    sec = C.c_double()
    _chk(lib().ref_cycles_multi(arr, len(hierarchies), _p(b), int(ncycles), C.byref(sec)))
    return sec.value


def sym_eig(A):
    """sym_eig (blockla.hpp:318-326) of a dense symmetric matrix: (lambda
    ascending, V column-major flattened)."""
    n = A.shape[0]
    a = np.ascontiguousarray(np.asarray(A, np.float64).reshape(-1, order="F"))  # kept alive over the call
    lam, V = np.empty(n), np.empty(n * n)
    _chk(lib().ref_sym_eig(n, _p(a), _p(lam), _p(V)))
    return lam, V


def random_rhs(nblocks, bs, seed=0):
    out = np.empty(nblocks * bs)
    _chk(lib().ref_random_rhs(nblocks, bs, seed, _p(out)))
    return out


def dump_block_coo(brows, bcols, rbs, cbs, ptr, col, val, path):
    """The reference's dump_block_coo (blockla.hpp:253-268) written to `path`."""
    ptr = np.ascontiguousarray(ptr, np.int32)
    col = np.ascontiguousarray(col, np.int32)
    val = np.ascontiguousarray(val, np.float64)
    _chk(lib().ref_dump_block_coo(brows, bcols, rbs, cbs, _p(ptr), _p(col), _p(val), str(path).encode()))


def bsr_spmv(brows, bcols, rbs, cbs, ptr, col, val, x, transpose=False):
    ptr = np.ascontiguousarray(ptr, np.int32)
    col = np.ascontiguousarray(col, np.int32)
    val = np.ascontiguousarray(val, np.float64)
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty((bcols * cbs) if transpose else (brows * rbs))
    m = C.c_ulonglong()
    _chk(lib().ref_bsr_spmv(brows, bcols, rbs, cbs, _p(ptr), _p(col), _p(val), _p(x), _p(y), int(transpose),
                            C.byref(m)))
    return y, m.value


def sai_build(kind, dim, ncomp, bs_scalar, N, ptr, col, val, level, zeta, cache=True):
    ptr = np.ascontiguousarray(ptr, np.int32)
    col = np.ascontiguousarray(col, np.int32)
    val = np.ascontiguousarray(val, np.float64)
    h = lib().ref_sai_build(kind, dim, ncomp, bs_scalar, N, _p(ptr), _p(col), _p(val), level, zeta, int(cache))
    if not h:
        raise RefError(-1, lib().ref_last_error().decode())
    try:
        nnzb = lib().ref_sai_raw_nnzb(h)
        bs = ncomp * bs_scalar
        bp = np.empty(N + 1, np.int32)
        bc = np.empty(nnzb, np.int32)
        bv = np.empty(nnzb * bs * bs)
        lib().ref_sai_raw_matrix(h, _p(bp), _p(bc), _p(bv))
        st = SaiStats()
        lib().ref_sai_raw_stats(h, C.byref(st))
        return (bp, bc, bv), st
    finally:
        lib().ref_sai_raw_free(h)


def balance_vector(kind, dim, ncomp, bs_scalar, N, ptr, col, val, zeta):
    bs = ncomp * bs_scalar
    a = np.empty(N * bs)
    ptr = np.ascontiguousarray(ptr, np.int32)  # kept alive over the call
    col = np.ascontiguousarray(col, np.int32)
    val = np.ascontiguousarray(val, np.float64)
    _chk(lib().ref_balance_vector(kind, dim, ncomp, bs_scalar, N, _p(ptr), _p(col), _p(val), zeta, _p(a)))
    return a
