"""Combo strings and CSV rows, restating the reference's harness tests
(tests/test_harness.cpp:9-51, 260-270) against paper_2412_12506_b200.report."""
import io

import pytest

import paper_2412_12506_b200 as g
from paper_2412_12506_b200 import report as R


def test_combo_strings_parse_to_canonical_specs():
    s = R.parse_combo("GMRES-GS")
    assert s.kind == g._lib.KRYLOV_GMRES and s.smoother.kind == g.COLOURED_GS
    assert (s.pre, s.post, s.name) == (g.SWEEP_FORWARD, g.SWEEP_REVERSE, "GMRES-GS-fr")
    s = R.parse_combo("CG-J")
    assert s.kind == g._lib.KRYLOV_CG and s.smoother.kind == g.JACOBI and s.smoother.omega == 0.8
    assert s.name == "CG-J"
    s = R.parse_combo("GMRES-PGS")
    assert s.smoother.kind == g.PROC_BLOCK_GS and s.smoother.partitions == 4 and s.name == "GMRES-PGS4-fr"
    s = R.parse_combo("CG-PGS16-rf")
    assert s.smoother.partitions == 16 and (s.pre, s.post) == (g.SWEEP_REVERSE, g.SWEEP_FORWARD)
    assert s.name == "CG-PGS16-rf"
    s = R.parse_combo("GMRES-SAI2-rr", 0.27)
    assert s.smoother.kind == g.SAI and s.smoother.level == 2 and s.smoother.zeta == 0.27
    assert (s.pre, s.post, s.name) == (g.SWEEP_REVERSE, g.SWEEP_REVERSE, "GMRES-SAI2-rr")
    assert R.parse_combo("GMRES-GS-ff", 0.5).name == "GMRES-GS-ff"


@pytest.mark.parametrize("bad", ["GMRES", "NEWTON-GS", "GMRES-XX", "GMRES-SAI", "GMRES-SAI3", "CG-J-ff",
                                 "GMRES-GS-fx", "GMRES-GS-frr", "GMRES-GS-ff-x", "CG-PGS0", "GMRES-SAIx"])
def test_malformed_combo_strings_are_rejected(bad):
    with pytest.raises(g.InvalidArgument, match=f'solver "{bad}"'):
        R.parse_combo(bad)


def test_csv_doubles_round_trip_and_infinities_spell_inf():
    assert R.format_double(0.1) == "0.10000000000000001"
    assert R.format_double(float("inf")) == "inf"
    assert R.format_double(float("-inf")) == "-inf"
    assert R.format_double(2.0) == "2"


def test_empty_matrix_is_header_only():
    s = io.StringIO()
    R.write_csv(s, [], perf=False)
    assert s.getvalue() == "problem,dim,degree,n,solver,rho,eta,iterations,classification\n"


def test_rows_and_perf_columns():
    rows = [R.CellRow("poisson-2d", 2, 3, 64, "GMRES-J", rho=0.25, eta=1.6609640474436813, iterations=19,
                      classification=0, perf={"vcycle_ms": 0.29, "dof_updates_per_s": 1.21e9}),
            R.CellRow("stokes-3d", 3, 2, 16, "GMRES-SAI1-fr", ok=False)]
    s = io.StringIO()
    R.write_csv(s, rows)
    lines = s.getvalue().splitlines()
    assert lines[0] == R.CSV_HEADER + ",setup_s,vcycle_ms,dof_updates_per_s,alg_gbps"
    assert lines[1] == "poisson-2d,2,3,64,GMRES-J,0.25,1.6609640474436813,19,fast,,0.28999999999999998,1210000000,"
    assert lines[2] == "stokes-3d,3,2,16,GMRES-SAI1-fr,,,0,error,,,,"
