"""ctypes binding of the in-tree C ABI library ``libldgmg_b200.so``.

The library is the product: every operator application runs in the sm_100a
kernels behind it.  There is no Python or CPU fallback -- if the shared object
is missing the import fails loudly, and without a CUDA device every compute
entry point returns LDGMG_ERR_CUDA.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libldgmg_b200.so")

OK = 0
ERR_INVALID_ARGUMENT = 1
ERR_RUNTIME = 2
ERR_LOGIC = 3
ERR_CUDA = 4
ERR_NCCL = 5

SWEEP_FORWARD, SWEEP_REVERSE = 0, 1
JACOBI, COLOURED_GS, PROC_BLOCK_GS, SAI = 0, 1, 2, 3
SYSTEM_SCALAR, SYSTEM_STOKES = 0, 1
BC_PERIODIC, BC_DIRICHLET, BC_NEUMANN = 0, 1, 2
PHASE_SINGLE, PHASE_BOXES, PHASE_BALL, PHASE_ELLIPSE = 0, 1, 2, 3


class LdgmgError(Exception):
    """Base class; subclasses mirror the reference's exception types."""


class InvalidArgument(LdgmgError, ValueError):
    """std::invalid_argument in the reference."""


class LdgmgRuntimeError(LdgmgError, RuntimeError):
    """std::runtime_error in the reference."""


class LogicError(LdgmgError):
    """std::logic_error in the reference."""


class CudaError(LdgmgError, RuntimeError):
    """Device failure (no CUDA device, launch error...)."""


_ERRORS = {
    ERR_INVALID_ARGUMENT: InvalidArgument,
    ERR_RUNTIME: LdgmgRuntimeError,
    ERR_LOGIC: LogicError,
    ERR_CUDA: CudaError,
    ERR_NCCL: CudaError,
}


class SmootherConfig(C.Structure):
    _fields_ = [("kind", C.c_int), ("omega", C.c_double), ("partitions", C.c_int),
                ("level", C.c_int), ("zeta", C.c_double), ("cache", C.c_int)]


class MgConfig(C.Structure):
    _fields_ = [("smoother", SmootherConfig), ("pre", C.c_int), ("post", C.c_int),
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


class ProblemSpec(C.Structure):
    _fields_ = [("kind", C.c_int), ("dim", C.c_int), ("n", C.c_int), ("degree", C.c_int),
                ("bc", C.c_int * 6), ("beta", C.c_double), ("beta_p", C.c_double),
                ("gamma", C.c_double), ("delta", C.c_double), ("phase_shape", C.c_int),
                ("center", C.c_double * 3), ("radii", C.c_double * 3),
                ("mu_in", C.c_double), ("mu_out", C.c_double), ("rho_in", C.c_double),
                ("rho_out", C.c_double)]


class SolveReportC(C.Structure):
    _fields_ = [("residuals", C.POINTER(C.c_double)), ("capacity", C.c_int), ("n_residuals", C.c_int),
                ("iterations", C.c_int), ("converged", C.c_int), ("breakdown", C.c_int), ("rho", C.c_double),
                ("eta", C.c_double), ("classification", C.c_int), ("low_confidence", C.c_int)]


KRYLOV_CG, KRYLOV_GMRES = 0, 1
PROBLEM_DEVICE_ASSEMBLY, PROBLEM_ANY_N = 1, 2  # ldgmg_problem_create_ex flags


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_2412_12506_b200/csrc). The B200 path has no CPU fallback.")
    return C.CDLL(LIB_PATH)


lib = _load()

_P = C.c_void_p
_I = C.c_int
_D = C.c_double
_I64 = C.c_int64
_IP = C.POINTER(C.c_int)
_DP = C.POINTER(C.c_double)

_SIGS = {
    "ldgmg_last_error": ([], C.c_char_p),
    "ldgmg_abi_version": ([], _I),
    "ldgmg_launch_count": ([], _I64),
    "ldgmg_debug_guard_check": ([], _I64),
    "ldgmg_debug_guard_live": ([], _I64),
    "ldgmg_ctx_create": ([_I, C.POINTER(_P)], _I),
    "ldgmg_ctx_destroy": ([_P], _I),
    "ldgmg_ctx_set_stream": ([_P, _P], _I),
    "ldgmg_ctx_stream": ([_P], _P),
    "ldgmg_ctx_synchronize": ([_P], _I),
    "ldgmg_device_alloc": ([_P, C.c_size_t, C.POINTER(_P)], _I),
    "ldgmg_device_free": ([_P, _P], _I),
    "ldgmg_copy_h2d": ([_P, _P, _P, C.c_size_t], _I),
    "ldgmg_copy_d2h": ([_P, _P, _P, C.c_size_t], _I),
    "ldgmg_bsr_upload": ([_P, _I, _I, _I, _I, _P, _P, _P, C.POINTER(_P)], _I),
    "ldgmg_bsr_shape": ([_P, _IP, _IP, _IP, _IP, C.POINTER(_I64)], _I),
    "ldgmg_bsr_download": ([_P, _P, _P, _P, _P], _I),
    "ldgmg_bsr_device_bytes": ([_P], _I64),
    "ldgmg_bsr_dump_coo": ([_P, _P, C.c_char_p], _I),
    "ldgmg_bsr_load_coo": ([_P, C.c_char_p, _P], _I),
    "ldgmg_coo_write_host": ([C.c_char_p, _I, _I, _I, _I, _P, _P, _P], _I),
    "ldgmg_coo_read_host": ([C.c_char_p, _P, _P, _P, _P, _P, _P, _P, _P], _I),
    "ldgmg_bsr_destroy": ([_P], _I),
    "ldgmg_bsr_upload_ex": ([_P, _I, _I, _I, _I, _P, _P, _P, _I, C.POINTER(_P)], _I),
    "ldgmg_spmv_add": ([_P, _P, _P, _P], _I),
    "ldgmg_bsr_set_values": ([_P, _P, _I64, _I64, _P], _I),
    "ldgmg_dgemm_nt_batched": ([_P, _I, _I, _I, _D, _P, _I64, _I64, _P, _I64, _I64, _D, _P, _I64, _I64, _I], _I),
    "ldgmg_bsr_row_prefix_view": ([_P, _P, _I, C.POINTER(_P)], _I),
    "ldgmg_bsr_gather": ([_P, _P, _I, _I, _P, _P, _P, C.POINTER(_P)], _I),
    "ldgmg_bsr_transposed_view": ([_P, _P, _I, _I, _P, _P, _P, C.POINTER(_P)], _I),
    "ldgmg_residual_rows": ([_P, _P, _P, _P, _P, _P, _I], _I),
    "ldgmg_spmv_add_rows": ([_P, _P, _P, _P, _P, _I], _I),
    "ldgmg_pgs_schedule": ([_I, _P, _P, _I, _P, _P, _IP], _I),
    "ldgmg_factors_upload": ([_P, _I, _I, _P, _P, _P, C.POINTER(_P)], _I),
    "ldgmg_factors_destroy": ([_P], _I),
    "ldgmg_relax": ([_P, _P, _P, _P, _P, _P, _P, _D], _I),
    "ldgmg_relax_rows": ([_P, _P, _P, _P, _P, _P, _P, _D, _P, _I], _I),
    "ldgmg_project_partials": ([_P, _P, _I, _I, _I, _I, _P, _I, _D, _P], _I),
    "ldgmg_project_apply": ([_P, _P, _I, _I, _I, _I, _P, _I, _D, _P], _I),
    "ldgmg_gather_blocks": ([_P, _P, _P, _I, _I, _P], _I),
    "ldgmg_partition_level": ([_I, _P, _P, _I, _I, _IP, _IP, _IP, _IP, _P, _P, _P, _P, _P], _I),
    "ldgmg_spmv": ([_P, _P, _P, _P], _I),
    "ldgmg_spmv_transpose": ([_P, _P, _P, _P], _I),
    "ldgmg_residual": ([_P, _P, _P, _P, _P], _I),
    "ldgmg_dot": ([_P, _I64, _P, _P, _DP], _I),
    "ldgmg_axpy": ([_P, _I64, _D, _P, _P], _I),
    "ldgmg_smoother_create": ([_P, _P, _I, _I, C.POINTER(SmootherConfig), C.POINTER(_P)], _I),
    "ldgmg_smoother_create_with_factors": ([_P, _P, C.POINTER(SmootherConfig), _P, _P, _P, C.POINTER(_P)], _I),
    "ldgmg_smoother_create_with_sai": ([_P, _P, C.POINTER(SmootherConfig), _P, _P, _P, C.POINTER(_P)], _I),
    "ldgmg_smoother_apply": ([_P, _P, _P, _P, _I], _I),
    "ldgmg_smoother_colours": ([_P, _P, _IP], _I),
    "ldgmg_smoother_sai_nnzb": ([_P, C.POINTER(_I64)], _I),
    "ldgmg_smoother_sai_matrix": ([_P, _P, _P, _P, _P], _I),
    "ldgmg_smoother_sai_stats": ([_P, C.POINTER(SaiStats)], _I),
    "ldgmg_sai_build": ([_P, _P, _I, _I, _I, _D, _I, _P, C.POINTER(_P), C.POINTER(SaiStats)], _I),
    "ldgmg_smoother_diag_factors": ([_P, _P, _P, _P, _P], _I),
    "ldgmg_smoother_destroy": ([_P], _I),
    "ldgmg_transfer_create": ([_P, _I, _I, _P, _P, _I, _I, _I, _P, C.POINTER(_P)], _I),
    "ldgmg_restrict": ([_P, _P, _P, _P], _I),
    "ldgmg_interpolate_add": ([_P, _P, _P, _P], _I),
    "ldgmg_transfer_destroy": ([_P], _I),
    "ldgmg_mg_create": ([_P, _I, _P, _P, _I, _I, _I, _I, _I, _I, C.POINTER(MgConfig), _P, _P, C.POINTER(_P)], _I),
    "ldgmg_mg_set_smoother": ([_P, _I, _P], _I),
    "ldgmg_mg_smoother": ([_P, _I, C.POINTER(_P)], _I),
    "ldgmg_mg_depth": ([_P], _I),
    "ldgmg_mg_cycle": ([_P, _P, _P, _P], _I),
    "ldgmg_mg_apply": ([_P, _P, _P, _P], _I),
    "ldgmg_mg_vcycle": ([_P, _P, _P, _P], _I),
    "ldgmg_mg_cycles": ([_P, _P, _P, _P, _I], _I),
    "ldgmg_mg_solve_host": ([_P, _P, _P, _P, _D, _I, _P, _IP], _I),
    "ldgmg_mg_set_strict_order": ([_P, _I], _I),
    "ldgmg_mg_setup": ([_P, _P], _I),
    "ldgmg_mg_cycle_costs": ([_P, _DP, _DP], _I),
    "ldgmg_mg_destroy": ([_P], _I),
    "ldgmg_krylov_solve": ([_P, _P, _I, _P, _P, _D, _I, C.POINTER(SolveReportC)], _I),
    "ldgmg_estimate_eta": ([_P, _P, _I, C.c_uint64, _D, _I, C.POINTER(SolveReportC)], _I),
    "ldgmg_problem_create": ([C.POINTER(ProblemSpec), _I, _I, C.POINTER(_P)], _I),
    "ldgmg_problem_create_partial": ([C.POINTER(ProblemSpec), _I, _I, _I, _I, _I, _I, C.POINTER(_P)], _I),
    "ldgmg_problem_level_partial": ([_P, _I], _I),
    "ldgmg_problem_create_ex": ([C.POINTER(ProblemSpec), _I, _I, _I, _I, _I, _I, _I, C.POINTER(_P)], _I),
    "ldgmg_problem_device_operator": ([_P, _P, _I, C.POINTER(_P)], _I),
    "ldgmg_problem_depth": ([_P], _I),
    "ldgmg_problem_level_shape": ([_P, _I, _IP, _IP, C.POINTER(_I64)], _I),
    "ldgmg_problem_level_matrix": ([_P, _I, _P, _P, _P], _I),
    "ldgmg_problem_level_transfer": ([_P, _I, _P, _P], _I),
    "ldgmg_problem_info": ([_P, _IP, _IP, _IP, _IP, _IP, _IP], _I),
    "ldgmg_problem_injection": ([_P, _P], _I),
    "ldgmg_mg_create_from_problem": ([_P, _P, C.POINTER(MgConfig), C.POINTER(_P)], _I),
    "ldgmg_problem_destroy": ([_P], _I),
    "ldgmg_random_rhs": ([_I, _I, C.c_uint64, _P], _I),
    "ldgmg_injection_matrices": ([_I, _I, _P], _I),
}

for _name, (_args, _res) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_SIGS)


def check(status: int) -> None:
    """Raise the exception type that mirrors the reference's for a status."""
    if status != OK:
        msg = lib.ldgmg_last_error().decode(errors="replace")
        raise _ERRORS.get(status, LdgmgError)(msg)


def launch_count() -> int:
    return int(lib.ldgmg_launch_count())
