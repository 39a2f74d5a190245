"""Python mirror of the reference's operator / smoother / V-cycle interface,
over the C ABI (include/ldgmg_b200.h).  Names follow the reference headers:

    BlockCsr (blockla.hpp:73-92)      -> DeviceBsr
    spmv / spmv_transpose (:136-176)  -> spmv / spmv_transpose
    SmootherConfig / Smoother (smoothers.hpp:23-58, 373-534)
    MultigridConfig / Multigrid (multigrid.hpp:26-36, 45-274)
    random_rhs (krylov.hpp:279-287)

Device vectors are torch CUDA float64 tensors (element-major, BlockVec::data
layout); torch only provides device memory and streams -- every operation is
one of the library's sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from ._lib import check, lib


def _ptr(a) -> int:
    """Data pointer of a torch tensor or a contiguous numpy array."""
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


def _np(a, dtype):
    return np.ascontiguousarray(np.asarray(a, dtype=dtype))


@dataclass
class _Shape:
    brows: int
    bcols: int
    row_bs: int
    col_bs: int


class Context:
    """Device + stream handle (ldgmg_ctx_create)."""

    def __init__(self, device: int = 0, stream=None):
        h = C.c_void_p()
        check(lib.ldgmg_ctx_create(int(device), C.byref(h)))
        self.h = h
        self.device = device
        if stream is None:
            # Device vectors are torch tensors: run on torch's current stream so
            # the caching allocator's stream-ordered reuse stays race-free.
            try:
                import torch
                if torch.cuda.is_available():
                    stream = torch.cuda.current_stream(device)
            except ImportError:
                pass
        if stream is not None:
            self.set_stream(stream)

    def set_stream(self, stream) -> None:
        handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        check(lib.ldgmg_ctx_set_stream(self.h, C.c_void_p(handle)))

    @property
    def stream(self) -> int:
        return int(lib.ldgmg_ctx_stream(self.h) or 0)

    def synchronize(self) -> None:
        check(lib.ldgmg_ctx_synchronize(self.h))

    def close(self) -> None:
        if getattr(self, "h", None):
            lib.ldgmg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceBsr:
    """Device-resident uniform-block CSR (reference BlockCsr, blockla.hpp:73-92)."""

    def __init__(self, ctx: Context, brows, bcols, row_bs, col_bs, ptr, col, val):
        self.ctx = ctx
        ptr = _np(ptr, np.int32)
        col = _np(col, np.int32)
        val = _np(val, np.float64)
        h = C.c_void_p()
        check(lib.ldgmg_bsr_upload(ctx.h, int(brows), int(bcols), int(row_bs), int(col_bs),
                                   ptr.ctypes.data, col.ctypes.data, val.ctypes.data, C.byref(h)))
        self.h = h
        self.brows, self.bcols, self.row_bs, self.col_bs = int(brows), int(bcols), int(row_bs), int(col_bs)
        self.nnzb = int(ptr[-1]) if len(ptr) else 0

    @classmethod
    def from_csr(cls, ctx, A) -> "DeviceBsr":
        return cls(ctx, A.brows, A.bcols, A.row_bs, A.col_bs, A.ptr, A.col, A.val)

    @classmethod
    def adopt(cls, ctx: Context, h) -> "DeviceBsr":
        """Wrap (and own) a matrix handle returned by the C ABI."""
        B = cls.__new__(cls)
        B.ctx, B.h = ctx, h
        br, bc, rb, cb, nz = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int64()
        check(lib.ldgmg_bsr_shape(h, C.byref(br), C.byref(bc), C.byref(rb), C.byref(cb), C.byref(nz)))
        B.brows, B.bcols, B.row_bs, B.col_bs, B.nnzb = br.value, bc.value, rb.value, cb.value, nz.value
        return B

    def pattern(self):
        """(ptr, col) only -- no value download."""
        ptr = np.empty(self.brows + 1, np.int32)
        col = np.empty(max(self.nnzb, 1), np.int32)
        check(lib.ldgmg_bsr_download(self.ctx.h, self.h, ptr.ctypes.data, col.ctypes.data, None))
        return ptr, col[: self.nnzb]

    def download(self):
        ptr = np.empty(self.brows + 1, np.int32)
        col = np.empty(max(self.nnzb, 1), np.int32)
        val = np.empty(max(self.nnzb * self.row_bs * self.col_bs, 1), np.float64)
        check(lib.ldgmg_bsr_download(self.ctx.h, self.h, ptr.ctypes.data, col.ctypes.data, val.ctypes.data))
        return ptr, col[: self.nnzb], val[: self.nnzb * self.row_bs * self.col_bs]

    @property
    def device_bytes(self) -> int:
        return int(lib.ldgmg_bsr_device_bytes(self.h))

    def dump_coo(self, path) -> None:
        """Block-coordinate text dump (the reference's dump_block_coo, blockla.hpp:253-268)."""
        check(lib.ldgmg_bsr_dump_coo(self.ctx.h, self.h, str(path).encode()))

    @classmethod
    def load_coo(cls, ctx: Context, path) -> "DeviceBsr":
        """Upload a block-coordinate dump (duplicates summed, columns ascending)."""
        obj = cls.__new__(cls)
        obj.ctx = ctx
        h = C.c_void_p()
        check(lib.ldgmg_bsr_load_coo(ctx.h, str(path).encode(), C.byref(h)))
        obj.h = h
        br, bc, rb, cb, nz = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int64()
        check(lib.ldgmg_bsr_shape(h, C.byref(br), C.byref(bc), C.byref(rb), C.byref(cb), C.byref(nz)))
        obj.brows, obj.bcols, obj.row_bs, obj.col_bs, obj.nnzb = br.value, bc.value, rb.value, cb.value, nz.value
        return obj

    def __del__(self):
        if getattr(self, "h", None):
            lib.ldgmg_bsr_destroy(self.h)
            self.h = None


def coo_write(path, brows, bcols, row_bs, col_bs, ptr, col, val) -> None:
    """Host-only block-coordinate writer (same text as dump_block_coo)."""
    ptr = _np(ptr, np.int32)
    col = _np(col, np.int32)
    val = _np(val, np.float64)
    check(lib.ldgmg_coo_write_host(str(path).encode(), int(brows), int(bcols), int(row_bs), int(col_bs),
                                   ptr.ctypes.data, col.ctypes.data, val.ctypes.data))


def coo_read(path):
    """Host-only block-coordinate reader -> (brows, bcols, row_bs, col_bs, ptr, col, val)."""
    br, bc, rb, cb, nz = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int64()
    p = str(path).encode()
    check(lib.ldgmg_coo_read_host(p, C.byref(br), C.byref(bc), C.byref(rb), C.byref(cb), C.byref(nz),
                                  None, None, None))
    ptr = np.empty(br.value + 1, np.int32)
    col = np.empty(max(nz.value, 1), np.int32)
    val = np.empty(max(nz.value * rb.value * cb.value, 1), np.float64)
    check(lib.ldgmg_coo_read_host(p, None, None, None, None, None, ptr.ctypes.data, col.ctypes.data,
                                  val.ctypes.data))
    return (br.value, bc.value, rb.value, cb.value, ptr, col[: nz.value], val[: nz.value * rb.value * cb.value])


def spmv(ctx: Context, A: DeviceBsr, x, y) -> None:
    """y = A x (blockla.hpp:136-154); throws on shape mismatch like the reference."""
    if x.numel() != A.bcols * A.col_bs or y.numel() != A.brows * A.row_bs:
        raise L.InvalidArgument("spmv: shape mismatch")
    check(lib.ldgmg_spmv(ctx.h, A.h, _ptr(x), _ptr(y)))


def spmv_transpose(ctx: Context, A: DeviceBsr, x, y) -> None:
    """y = A^T x (blockla.hpp:157-176)."""
    if x.numel() != A.brows * A.row_bs or y.numel() != A.bcols * A.col_bs:
        raise L.InvalidArgument("spmv_transpose: shape mismatch")
    check(lib.ldgmg_spmv_transpose(ctx.h, A.h, _ptr(x), _ptr(y)))


def residual(ctx: Context, A: DeviceBsr, b, x, r) -> None:
    """r = b - A x, fused (multigrid.hpp:256-258)."""
    check(lib.ldgmg_residual(ctx.h, A.h, _ptr(b), _ptr(x), _ptr(r)))


@dataclass
class SmootherConfig:
    """smoothers.hpp:23-58 (same defaults and factory names)."""
    kind: int = L.JACOBI
    omega: float = 0.8
    partitions: int = 1
    level: int = 1
    zeta: float = 0.1
    cache: bool = True

    @staticmethod
    def jacobi(omega: float = 0.8) -> "SmootherConfig":
        return SmootherConfig(kind=L.JACOBI, omega=omega)

    @staticmethod
    def coloured_gs() -> "SmootherConfig":
        return SmootherConfig(kind=L.COLOURED_GS, omega=1.0)

    @staticmethod
    def proc_block_gs(partitions: int, omega: float = 0.8) -> "SmootherConfig":
        return SmootherConfig(kind=L.PROC_BLOCK_GS, omega=omega, partitions=partitions)

    @staticmethod
    def sai(level: int, zeta: float = 0.1, cache: bool = True) -> "SmootherConfig":
        return SmootherConfig(kind=L.SAI, level=level, zeta=zeta, cache=cache)

    def c(self) -> L.SmootherConfig:
        return L.SmootherConfig(self.kind, self.omega, self.partitions, self.level, self.zeta,
                                int(bool(self.cache)))


class Smoother:
    """GPU smoother bound to one operator (smoothers.hpp:373-534)."""

    def __init__(self, ctx: Context, A: DeviceBsr, cfg: SmootherConfig, system_kind=L.SYSTEM_SCALAR,
                 n_velocity=0, factors=None, sai=None, _handle=None, _owner=None):
        self.ctx, self.A, self.cfg = ctx, A, cfg
        self._owner = _owner
        if _handle is not None:
            self.h = _handle
            self._owned = False
            return
        h = C.c_void_p()
        cc = cfg.c()
        if factors is not None:
            V, lam, s = (_np(f, np.float64) for f in factors)
            check(lib.ldgmg_smoother_create_with_factors(ctx.h, A.h, C.byref(cc), V.ctypes.data,
                                                         lam.ctypes.data, s.ctypes.data, C.byref(h)))
        elif sai is not None:
            bp, bc, bv = _np(sai[0], np.int32), _np(sai[1], np.int32), _np(sai[2], np.float64)
            check(lib.ldgmg_smoother_create_with_sai(ctx.h, A.h, C.byref(cc), bp.ctypes.data,
                                                     bc.ctypes.data, bv.ctypes.data, C.byref(h)))
        else:
            check(lib.ldgmg_smoother_create(ctx.h, A.h, int(system_kind), int(n_velocity), C.byref(cc),
                                            C.byref(h)))
        self.h = h
        self._owned = True

    def apply(self, b, x, sweep=L.SWEEP_FORWARD) -> None:
        n = self.A.brows * self.A.row_bs
        if b.numel() != n or x.numel() != n:
            raise L.InvalidArgument("Smoother::apply: shape mismatch")
        check(lib.ldgmg_smoother_apply(self.ctx.h, self.h, _ptr(b), _ptr(x), int(sweep)))

    def colours(self) -> np.ndarray:
        n = C.c_int()
        out = np.empty(self.A.brows, np.int32)
        check(lib.ldgmg_smoother_colours(self.h, out.ctypes.data, C.byref(n)))
        return out

    def n_colours(self) -> int:
        n = C.c_int()
        check(lib.ldgmg_smoother_colours(self.h, None, C.byref(n)))
        return n.value

    def sai_nnzb(self) -> int:
        nnzb = C.c_int64()
        check(lib.ldgmg_smoother_sai_nnzb(self.h, C.byref(nnzb)))
        return nnzb.value

    def sai_matrix(self):
        nnzb = C.c_int64()
        check(lib.ldgmg_smoother_sai_nnzb(self.h, C.byref(nnzb)))
        bs = self.A.row_bs
        ptr = np.empty(self.A.brows + 1, np.int32)
        col = np.empty(max(nnzb.value, 1), np.int32)
        val = np.empty(max(nnzb.value * bs * bs, 1), np.float64)
        check(lib.ldgmg_smoother_sai_matrix(self.ctx.h, self.h, ptr.ctypes.data, col.ctypes.data,
                                            val.ctypes.data))
        return ptr, col[: nnzb.value], val[: nnzb.value * bs * bs]

    def sai_stats(self) -> L.SaiStats:
        st = L.SaiStats()
        check(lib.ldgmg_smoother_sai_stats(self.h, C.byref(st)))
        return st

    def diag_factors(self):
        N, bs = self.A.brows, self.A.row_bs
        V = np.empty(N * bs * bs)
        lam = np.empty(N * bs)
        s = np.empty(N * bs)
        check(lib.ldgmg_smoother_diag_factors(self.ctx.h, self.h, V.ctypes.data, lam.ctypes.data,
                                              s.ctypes.data))
        return V, lam, s

    def __del__(self):
        if getattr(self, "_owned", False) and getattr(self, "h", None):
            lib.ldgmg_smoother_destroy(self.h)
            self.h = None


class Transfer:
    """Restriction / prolongation between two levels (multigrid.hpp:104-149)."""

    def __init__(self, ctx: Context, n_fine, n_coarse, parent_of, orthant_of, dim, bs_scalar, n_comp, K):
        self.ctx = ctx
        p = _np(parent_of, np.int32)
        o = _np(orthant_of, np.int32)
        k = _np(K, np.float64)
        h = C.c_void_p()
        check(lib.ldgmg_transfer_create(ctx.h, int(n_fine), int(n_coarse), p.ctypes.data, o.ctypes.data,
                                        int(dim), int(bs_scalar), int(n_comp), k.ctypes.data, C.byref(h)))
        self.h = h

    def restrict(self, rf, rc) -> None:
        check(lib.ldgmg_restrict(self.ctx.h, self.h, _ptr(rf), _ptr(rc)))

    def interpolate_add(self, xc, xf) -> None:
        check(lib.ldgmg_interpolate_add(self.ctx.h, self.h, _ptr(xc), _ptr(xf)))

    def __del__(self):
        if getattr(self, "h", None):
            lib.ldgmg_transfer_destroy(self.h)
            self.h = None


@dataclass
class MultigridConfig:
    """multigrid.hpp:26-36 (same defaults)."""
    smoother: SmootherConfig = field(default_factory=SmootherConfig.jacobi)
    pre: int = L.SWEEP_FORWARD
    post: int = L.SWEEP_REVERSE
    nu1: int = 3
    nu2: int = 3
    bottom_max_elements: int = 64
    bottom_tol: float = 1e-10
    min_depth: int = 2

    def c(self) -> L.MgConfig:
        return L.MgConfig(self.smoother.c(), self.pre, self.post, self.nu1, self.nu2,
                          self.bottom_max_elements, self.bottom_tol, self.min_depth)


@dataclass
class ProblemSpec:
    """Problem catalogue entry for the built-in host setup (harness.hpp:30-40)."""
    kind: int = L.SYSTEM_SCALAR
    dim: int = 2
    n: int = 8
    degree: int = 1
    bc: tuple = (L.BC_PERIODIC,) * 6
    beta: float = -1.0
    beta_p: float = 1.0
    gamma: float = 0.0
    delta: float = 0.0
    phase_shape: int = L.PHASE_SINGLE
    center: tuple = (0.5, 0.5, 0.5)
    radii: tuple = (0.25, 0.25, 0.25)
    mu_in: float = 1.0
    mu_out: float = 1.0
    rho_in: float = 1.0
    rho_out: float = 1.0

    def c(self) -> L.ProblemSpec:
        s = L.ProblemSpec()
        s.kind, s.dim, s.n, s.degree = self.kind, self.dim, self.n, self.degree
        for i in range(6):
            s.bc[i] = self.bc[i]
        s.beta, s.beta_p, s.gamma, s.delta = self.beta, self.beta_p, self.gamma, self.delta
        s.phase_shape = self.phase_shape
        for i in range(3):
            s.center[i] = self.center[i]
            s.radii[i] = self.radii[i]
        s.mu_in, s.mu_out, s.rho_in, s.rho_out = self.mu_in, self.mu_out, self.rho_in, self.rho_out
        return s


class Problem:
    """Built-in host setup: mesh chain + LDG operators per level."""

    def __init__(self, spec: ProblemSpec, min_depth=2, bottom_max_elements=64, device_assembly=False, any_n=False):
        """device_assembly: the level operators are assembled on the GPU when a
        hierarchy / device operator is created (bit-identical to the host
        assembly; level_matrix then returns no values).
        any_n: extension A1 -- spec.n need not be a
        power of two (Morton order of the bounding grid, restricted)."""
        self.spec = spec
        cs = spec.c()
        h = C.c_void_p()
        flags = (L.PROBLEM_DEVICE_ASSEMBLY if device_assembly else 0) | (L.PROBLEM_ANY_N if any_n else 0)
        if flags:
            check(lib.ldgmg_problem_create_ex(C.byref(cs), int(min_depth), int(bottom_max_elements), 1, 0, 0, 0, flags,
                                              C.byref(h)))
        else:
            check(lib.ldgmg_problem_create(C.byref(cs), int(min_depth), int(bottom_max_elements), C.byref(h)))
        self.h = h
        self.device_assembly = bool(device_assembly)
        self._init_info()

    def _init_info(self):
        h = self.h
        self.depth = int(lib.ldgmg_problem_depth(h))
        dim, nc, bss, kc, kp, nv = (C.c_int() for _ in range(6))
        check(lib.ldgmg_problem_info(h, C.byref(dim), C.byref(nc), C.byref(bss), C.byref(kc), C.byref(kp),
                                     C.byref(nv)))
        self.dim, self.n_comp, self.bs_scalar = dim.value, nc.value, bss.value
        self.kernel_constants, self.kernel_pressure, self.n_velocity = kc.value, kp.value, nv.value
        self.bs = self.n_comp * self.bs_scalar

    @classmethod
    def partial(cls, spec: ProblemSpec, nranks: int, rank: int, halo_hops: int, min_rows_per_rank: int = 64,
                min_depth=2, bottom_max_elements=64, device_assembly=False, any_n=False) -> "Problem":
        """Distributed setup (ldgmg_problem_create_partial): levels with >=
        nranks*min_rows_per_rank elements assemble only this rank's rows plus
        `halo_hops` face layers (other rows empty, global numbering kept)."""
        obj = cls.__new__(cls)
        obj.spec = spec
        cs = spec.c()
        h = C.c_void_p()
        check(lib.ldgmg_problem_create_ex(C.byref(cs), int(min_depth), int(bottom_max_elements), int(nranks),
                                          int(rank), int(halo_hops), int(min_rows_per_rank),
                                          (L.PROBLEM_DEVICE_ASSEMBLY if device_assembly else 0)
                                          | (L.PROBLEM_ANY_N if any_n else 0), C.byref(h)))
        obj.h = h
        obj.device_assembly = bool(device_assembly)
        obj._init_info()
        return obj

    def device_operator(self, ctx: "Context", l: int) -> "DeviceBsr":
        """The level operator on the device (device assembly or upload)."""
        h = C.c_void_p()
        check(lib.ldgmg_problem_device_operator(ctx.h, self.h, int(l), C.byref(h)))
        B = DeviceBsr.__new__(DeviceBsr)
        B.ctx, B.h = ctx, h
        br, bc, rb, cb, nz = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int64()
        check(lib.ldgmg_bsr_shape(h, C.byref(br), C.byref(bc), C.byref(rb), C.byref(cb), C.byref(nz)))
        B.brows, B.bcols, B.row_bs, B.col_bs, B.nnzb = br.value, bc.value, rb.value, cb.value, nz.value
        return B

    def level_partial(self, l) -> bool:
        return bool(lib.ldgmg_problem_level_partial(self.h, int(l)))

    def level_shape(self, l):
        n, bs, nnzb = C.c_int(), C.c_int(), C.c_int64()
        check(lib.ldgmg_problem_level_shape(self.h, l, C.byref(n), C.byref(bs), C.byref(nnzb)))
        return n.value, bs.value, nnzb.value

    def level_matrix(self, l):
        n, bs, nnzb = self.level_shape(l)
        ptr = np.empty(n + 1, np.int32)
        col = np.empty(max(nnzb, 1), np.int32)
        val = np.empty(max(nnzb * bs * bs, 1), np.float64)
        check(lib.ldgmg_problem_level_matrix(self.h, l, ptr.ctypes.data, col.ctypes.data, val.ctypes.data))
        return ptr, col[:nnzb], val[: nnzb * bs * bs]

    def level_pattern(self, l):
        n, bs, nnzb = self.level_shape(l)
        ptr = np.empty(n + 1, np.int32)
        col = np.empty(max(nnzb, 1), np.int32)
        check(lib.ldgmg_problem_level_matrix(self.h, l, ptr.ctypes.data, col.ctypes.data, None))
        return ptr, col[:nnzb]

    def level_transfer(self, l):
        n, _, _ = self.level_shape(l)
        p = np.empty(n, np.int32)
        o = np.empty(n, np.int32)
        check(lib.ldgmg_problem_level_transfer(self.h, l, p.ctypes.data, o.ctypes.data))
        return p, o

    def injection(self):
        K = np.empty((1 << self.dim) * self.bs_scalar ** 2)
        check(lib.ldgmg_problem_injection(self.h, K.ctypes.data))
        return K

    def __del__(self):
        if getattr(self, "h", None):
            lib.ldgmg_problem_destroy(self.h)
            self.h = None


class Multigrid:
    """GPU V-cycle hierarchy (multigrid.hpp:45-274).

    Either built from a Problem (the product's own setup) or from already
    assembled level operators + transfers (the drop-in path: the caller's
    reference objects did the setup)."""

    def __init__(self, ctx: Context, cfg: MultigridConfig, problem: Problem | None = None, *,
                 levels=None, transfers=None, system_kind=L.SYSTEM_SCALAR, dim=2, n_comp=1, bs_scalar=1,
                 kernel_constants=False, kernel_pressure=False, bottom=None):
        self.ctx, self.cfg = ctx, cfg
        h = C.c_void_p()
        cc = cfg.c()
        self._keep = []
        if problem is not None:
            check(lib.ldgmg_mg_create_from_problem(ctx.h, problem.h, C.byref(cc), C.byref(h)))
            self.n, self.bs = problem.level_shape(0)[:2]
            self.level_shapes = [problem.level_shape(l)[:2] for l in range(problem.depth)]
            self._keep = [problem]
        else:
            arrA = (C.c_void_p * len(levels))(*[A.h.value for A in levels])
            arrT = (C.c_void_p * max(1, len(transfers)))(*[T.h.value for T in transfers])
            self._keep = [levels, transfers, arrA, arrT]
            bV = bL = None
            if bottom is not None:
                bV = _np(bottom[0], np.float64)
                bL = _np(bottom[1], np.float64)
                self._keep += [bV, bL]
            check(lib.ldgmg_mg_create(ctx.h, len(levels), arrA, arrT, int(system_kind), int(dim), int(n_comp),
                                      int(bs_scalar), int(bool(kernel_constants)), int(bool(kernel_pressure)),
                                      C.byref(cc), bV.ctypes.data if bV is not None else None,
                                      bL.ctypes.data if bL is not None else None, C.byref(h)))
            self.n, self.bs = levels[0].brows, levels[0].row_bs
            self.level_shapes = [(A.brows, A.row_bs) for A in levels]
        self.h = h
        self.depth = int(lib.ldgmg_mg_depth(h))

    def set_smoother(self, level: int, S: Smoother) -> None:
        check(lib.ldgmg_mg_set_smoother(self.h, level, S.h))
        self._keep.append(S)

    def smoother(self, level: int) -> Smoother:
        h = C.c_void_p()
        check(lib.ldgmg_mg_smoother(self.h, level, C.byref(h)))
        n, bs = self.level_shapes[level]
        return Smoother(self.ctx, _Shape(n, n, bs, bs), None, _handle=h, _owner=self)

    def set_strict_order(self, strict: bool = True) -> None:
        """Reference-order (sequential) kernel-projection dots: bitwise parity mode."""
        check(lib.ldgmg_mg_set_strict_order(self.h, int(bool(strict))))

    def cycle(self, x, b) -> None:
        check(lib.ldgmg_mg_cycle(self.ctx.h, self.h, _ptr(x), _ptr(b)))

    def apply(self, b, x) -> None:
        check(lib.ldgmg_mg_apply(self.ctx.h, self.h, _ptr(b), _ptr(x)))

    def vcycle(self, x, b) -> None:
        """Bare v_cycle(0, x, b) without kernel projection (multigrid.hpp:247-264)."""
        check(lib.ldgmg_mg_vcycle(self.ctx.h, self.h, _ptr(x), _ptr(b)))

    def cycles(self, x, b, n: int) -> None:
        check(lib.ldgmg_mg_cycles(self.ctx.h, self.h, _ptr(x), _ptr(b), int(n)))

    def solve_host(self, b: np.ndarray, tol=1e-10, maxit=100, out: np.ndarray | None = None):
        """Stationary V-cycle solve from host buffers (H2D, cycles, D2H).
        `out` (optional): the host array receiving x; page-locked buffers
        (e.g. a pinned torch tensor's .numpy()) are written by DMA directly."""
        b = _np(b, np.float64)
        if b.ndim != 1 or b.size != self.n * self.bs:
            raise L.InvalidArgument("solve_host: b must hold n * bs entries")
        if int(maxit) < 0:
            raise L.InvalidArgument("mg_solve_host: maxit must be nonnegative")
        if out is not None:
            if out.dtype != np.float64 or out.shape != b.shape or not out.flags["C_CONTIGUOUS"]:
                raise L.InvalidArgument("solve_host: out must be a contiguous float64 array shaped like b")
            x = out
        else:
            x = np.empty_like(b)
        hist = np.empty(maxit + 1)
        it = C.c_int()
        check(lib.ldgmg_mg_solve_host(self.ctx.h, self.h, b.ctypes.data, x.ctypes.data, float(tol), int(maxit),
                                      hist.ctypes.data, C.byref(it)))
        return x, hist[: it.value + 1], it.value

    def _report(self, fn, maxit):
        buf = np.empty(maxit + 2)
        rep = L.SolveReportC()
        rep.residuals = buf.ctypes.data_as(C.POINTER(C.c_double))
        rep.capacity = maxit + 2
        check(fn(C.byref(rep)))
        return {"residuals": buf[: rep.n_residuals].copy(), "iterations": rep.iterations,
                "converged": bool(rep.converged), "breakdown": bool(rep.breakdown), "rho": rep.rho,
                "eta": rep.eta, "classification": ["fast", "slow", "nonconvergent"][rep.classification],
                "low_confidence": bool(rep.low_confidence)}

    def krylov_solve(self, b, x, kind=L.KRYLOV_GMRES, tol=1e-12, maxit=60):
        """pcg / gmres_left with this V-cycle as preconditioner (krylov.hpp:117-251)."""
        return self._report(lambda r: lib.ldgmg_krylov_solve(self.ctx.h, self.h, int(kind), _ptr(b), _ptr(x),
                                                             float(tol), int(maxit), r), maxit)

    def estimate_eta(self, kind=L.KRYLOV_GMRES, seed=0, tol=1e-12, maxit=60):
        """The paper-protocol measurement (krylov.hpp:293-306)."""
        return self._report(lambda r: lib.ldgmg_estimate_eta(self.ctx.h, self.h, int(kind), int(seed), float(tol),
                                                             int(maxit), r), maxit)

    def setup(self) -> None:
        """Build the smoothers not set by set_smoother (else the first cycle does)."""
        check(lib.ldgmg_mg_setup(self.ctx.h, self.h))

    def cycle_costs(self):
        self.setup()
        d, b = C.c_double(), C.c_double()
        check(lib.ldgmg_mg_cycle_costs(self.h, C.byref(d), C.byref(b)))
        return d.value, b.value

    def __del__(self):
        if getattr(self, "h", None):
            lib.ldgmg_mg_destroy(self.h)
            self.h = None


def sai_build(ctx: Context, A: DeviceBsr, system_kind=L.SYSTEM_SCALAR, n_velocity=0, level=1, zeta=0.1,
              cache=True, col_mask=None):
    """build_sai (smoothers.hpp:259-367) on a device operator -> (DeviceBsr B, SaiStats).
    `col_mask` (N bools) restricts the solved columns (the others stay zero)."""
    st = L.SaiStats()
    h = C.c_void_p()
    m = None
    if col_mask is not None:
        m = np.ascontiguousarray(np.asarray(col_mask) != 0, np.int32)
        if m.size != A.brows:
            raise L.InvalidArgument("build_sai: column mask size mismatch")
    check(lib.ldgmg_sai_build(ctx.h, A.h, int(system_kind), int(n_velocity), int(level), float(zeta), int(bool(cache)),
                              m.ctypes.data if m is not None else None, C.byref(h), C.byref(st)))
    B = DeviceBsr.__new__(DeviceBsr)
    B.ctx, B.h = ctx, h
    br, bc, rb, cb, nz = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int64()
    check(lib.ldgmg_bsr_shape(h, C.byref(br), C.byref(bc), C.byref(rb), C.byref(cb), C.byref(nz)))
    B.brows, B.bcols, B.row_bs, B.col_bs, B.nnzb = br.value, bc.value, rb.value, cb.value, nz.value
    return B, st


def random_rhs(nblocks: int, bs: int, seed: int = 0) -> np.ndarray:
    """krylov.hpp:279-287: mt19937_64, u = (rng()>>11)*2^-53, v = 2u-1."""
    out = np.empty(nblocks * bs)
    check(lib.ldgmg_random_rhs(int(nblocks), int(bs), int(seed), out.ctypes.data))
    return out
