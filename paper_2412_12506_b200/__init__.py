"""B200-native FP64 block-sparse multigrid V-cycle core (arXiv 2412.12506 `ldgmg` hot path).

The compute path is the in-tree C-ABI library ``libldgmg_b200.so`` (sm_100a
CUDA kernels); this package is its Python mirror of the reference interface.
"""
from . import _lib
from ._lib import (BC_DIRICHLET, BC_NEUMANN, BC_PERIODIC, COLOURED_GS, JACOBI, PHASE_BALL, PHASE_BOXES,
                   PHASE_ELLIPSE, PHASE_SINGLE, PROC_BLOCK_GS, SAI, SWEEP_FORWARD, SWEEP_REVERSE,
                   SYSTEM_SCALAR, SYSTEM_STOKES, CudaError, InvalidArgument, LdgmgError, LdgmgRuntimeError,
                   LogicError, launch_count)
from .api import (Context, DeviceBsr, Multigrid, MultigridConfig, Problem, ProblemSpec, Smoother,
                  SmootherConfig, Transfer, coo_read, coo_write, random_rhs, sai_build, residual, spmv, spmv_transpose)

__all__ = [n for n in dir() if not n.startswith("_")]
