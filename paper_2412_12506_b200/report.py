"""Solver combo strings and CSV result rows.

The reference's measurement harness names a solver by a combo string
("GMRES-SAI1-rf", harness.hpp:185-255) and writes one CSV row per
(problem, solver) cell with round-trip doubles (harness.hpp:329-357).  This
module keeps both formats so results from the GPU path line up with the
reference's CSVs, and appends the performance columns the reference does not
have (setup time, V-cycle time, DOF-updates/s, algorithmic GB/s).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

from . import _lib as L
from .api import SmootherConfig

#: harness.hpp:340-342
CSV_HEADER = "problem,dim,degree,n,solver,rho,eta,iterations,classification"
#: columns appended by this framework (empty when not measured)
PERF_COLUMNS = ("setup_s", "vcycle_ms", "dof_updates_per_s", "alg_gbps")
CLASSIFICATIONS = ("fast", "slow", "nonconvergent")  # krylov.hpp:21-35


@dataclass
class SolverSpec:
    """harness.hpp:177-183: Krylov kind, smoother, sweep directions, canonical name."""
    kind: int = L.KRYLOV_GMRES
    smoother: SmootherConfig = field(default_factory=SmootherConfig.coloured_gs)
    pre: int = L.SWEEP_FORWARD
    post: int = L.SWEEP_REVERSE
    name: str = ""


def parse_combo(text: str, zeta: float = 0.131) -> SolverSpec:
    """parse_combo (harness.hpp:185-255): "METHOD-SMOOTHER[-sweeps]".

    METHOD is CG or GMRES; SMOOTHER is J, GS, PGS[n] or SAI<level> (level
    0..2); the optional sweep suffix is two of {f, r} (default "fr"; Jacobi
    takes none).  Raises InvalidArgument with the reference's messages."""
    def fail(why):
        raise L.InvalidArgument(f'solver "{text}": {why}')

    def digits(s):
        if not s:
            fail("expected digits")
        if not all(c.isdigit() and c.isascii() for c in s):
            fail("malformed count")
        if len(s) > 6:
            fail("count out of range")
        return int(s)

    parts = text.split("-")
    if len(parts) < 2 or len(parts) > 3:
        fail("expected METHOD-SMOOTHER[-sweeps]")
    out = SolverSpec()
    if parts[0] == "CG":
        out.kind = L.KRYLOV_CG
    elif parts[0] == "GMRES":
        out.kind = L.KRYLOV_GMRES
    else:
        fail("method must be CG or GMRES")
    fam = parts[1]
    fam_name = fam
    jacobi = False
    if fam == "J":
        out.smoother = SmootherConfig.jacobi()
        jacobi = True
    elif fam == "GS":
        out.smoother = SmootherConfig.coloured_gs()
    elif fam.startswith("PGS"):
        P = 4 if len(fam) == 3 else digits(fam[3:])
        if P < 1:
            fail("partition count must be positive")
        out.smoother = SmootherConfig.proc_block_gs(P)
        fam_name = f"PGS{P}"
    elif fam.startswith("SAI"):
        if len(fam) == 3:
            fail("SAI needs a level, e.g. SAI1")
        level = digits(fam[3:])
        if level > 2:
            fail("SAI level must be 0, 1 or 2")
        out.smoother = SmootherConfig.sai(level, zeta)
    else:
        fail(f'unknown smoother family "{fam}"')
    sweeps = "fr"
    if len(parts) == 3:
        if jacobi:
            fail("Jacobi has no sweep suffix")
        sweeps = parts[2]
    if len(sweeps) != 2 or any(c not in "fr" for c in sweeps):
        fail("sweep suffix must be two of {f, r}")
    out.pre = L.SWEEP_FORWARD if sweeps[0] == "f" else L.SWEEP_REVERSE
    out.post = L.SWEEP_FORWARD if sweeps[1] == "f" else L.SWEEP_REVERSE
    out.name = f"{parts[0]}-{fam_name}"
    if not jacobi:
        out.name += f"-{sweeps}"
    return out


def format_double(v: float) -> str:
    """format_double (harness.hpp:330-338): %.17g, infinities spelled inf/-inf."""
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    return "%.17g" % v


@dataclass
class CellRow:
    """One CSV row: the reference's cell result plus optional perf columns."""
    problem: str
    dim: int
    degree: int
    n: int
    solver: str
    ok: bool = True
    rho: float = 0.0
    eta: float = 0.0
    iterations: int = 0
    classification: int = 0
    perf: dict = field(default_factory=dict)


def csv_header(perf: bool = True) -> str:
    return CSV_HEADER + ("," + ",".join(PERF_COLUMNS) if perf else "")


def csv_row(r: CellRow, perf: bool = True) -> str:
    """write_csv's row (harness.hpp:344-357); failed cells read ",,0,error"."""
    head = f"{r.problem},{r.dim},{r.degree},{r.n},{r.solver},"
    if r.ok:
        body = (f"{format_double(r.rho)},{format_double(r.eta)},{r.iterations},"
                f"{CLASSIFICATIONS[r.classification]}")
    else:
        body = ",,0,error"
    if perf:
        body += "," + ",".join("" if r.perf.get(k) is None else format_double(float(r.perf[k]))
                               for k in PERF_COLUMNS)
    return head + body


def write_csv(stream, rows, perf: bool = True) -> None:
    stream.write(csv_header(perf) + "\n")
    for r in rows:
        stream.write(csv_row(r, perf) + "\n")
