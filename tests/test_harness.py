"""SURVEY.md §8(f)2 harness parity: include/rd_gpu_harness.hpp (the reference's ExperimentConfig,
validate, config JSON, EocTable/CSV conventions, run_precond_bench, MatrixMarket I/O) and the
rdbench bench-precond CLI (paper_2102_03515_b200/cli/rdbench.cpp) with the reference's exit codes
(tools/rdbench.cpp:121-125, :186-190: 0 converged, 1 a row did not converge, 2 an exception)."""
import csv
import io
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2102_03515_b200")
RDBENCH = os.path.join(PKG, "_build", "rdbench")
HARNESS = os.path.join(ROOT, "tests", "cpp", "test_harness")


def _built(path):
    if not os.path.exists(path):
        subprocess.run(["make", "-s", "-C", PKG], check=True)
    return path


def test_harness_host_checks(tmp_path):
    out = subprocess.run([_built(HARNESS), str(tmp_path)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr


@pytest.mark.parametrize("args", [["bench-precond", "--rho", "-1"], ["bench-precond", "--n", "0"],
                                  ["bench-precond", "--tol", "0"], ["bench-precond", "--precond", "jacobi"],
                                  ["bench-precond", "--precond", "ilu"], ["bench-precond", "--example", "ball"],
                                  ["bench-precond", "--bogus"], ["table-h"], ["adapt", "--example", "smooth"],
                                  ["adapt", "--budget", "0"], ["adapt", "--precond", "jacobi"], ["nope"], []])
def test_rdbench_rejects_with_exit_2(args):
    """Rejected configs raise std::invalid_argument before any device work: exit code 2 and an
    'error:' line (rdbench.cpp:186-190); the other subcommands are outside the device path."""
    out = subprocess.run([_built(RDBENCH)] + args, capture_output=True, text=True, timeout=60)
    assert out.returncode == 2, (args, out.stdout, out.stderr)
    assert out.stdout == ""


@pytest.mark.gpu
def test_rdbench_bench_precond_rows(O, tmp_path):
    """bench-precond rows (bench.cpp:392-423) from the device: the reference's columns and
    number formats, rho outer / n inner, iteration counts equal to the oracle's."""
    path = tmp_path / "rows.csv"
    out = subprocess.run([_built(RDBENCH), "bench-precond", "--rho", "1", "1e-4", "--n", "8", "12",
                          "--out", str(path)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    text = path.read_text()
    rows = list(csv.DictReader(io.StringIO(text)))
    assert text.splitlines()[0] == "rho,n,dofs,iterations,converged,setup_seconds,solve_seconds"
    assert [(r["rho"], r["n"]) for r in rows] == [("1.000000e+00", "8"), ("1.000000e+00", "12"),
                                                  ("1.000000e-04", "8"), ("1.000000e-04", "12")]
    for r in rows:
        n, rho = int(r["n"]), float(r["rho"])
        ref = O.solve_system_amg(O.build_system(O.build_structured_cube(n), rho, "smooth"), 1e-8)
        assert int(r["dofs"]) == (n - 1) ** 3 and int(r["converged"]) == 1
        assert int(r["iterations"]) == ref.iterations
        assert float(r["setup_seconds"]) > 0 and float(r["solve_seconds"]) > 0


@pytest.mark.gpu
@pytest.mark.parametrize("n", [16, 24])
def test_rdbench_unattainable_tolerance(tmp_path, n):
    """An unattainable tolerance drives PCG past the rounding floor.  Where it ends depends on
    the last bits of every dot product: either the residual becomes exactly zero (rel = 0 <=
    tol: a converged row, exit 0) or p'Ap / r'z loses its sign, pcg throws (linalg.cpp:81-89)
    and rdbench reports the exception with exit code 2 and nothing on stdout, as the reference
    does (rdbench.cpp:186-190).  The exit-1 rule for non-converged rows is covered host-side."""
    out = subprocess.run([_built(RDBENCH), "bench-precond", "--rho", "1", "--n", str(n), "--tol", "1e-300",
                          "--gnuplot"], capture_output=True, text=True, timeout=300)
    assert out.returncode in (0, 2), out.stdout + out.stderr
    if out.returncode == 2:
        assert "not positive definite" in out.stderr and out.stdout == ""
    else:
        rows = [l.split() for l in out.stdout.splitlines() if l and not l.startswith("#")]
        assert len(rows) == 1 and rows[0][4] == "1", out.stdout


@pytest.mark.gpu
def test_rdbench_adapt(O, tmp_path):
    """rdbench adapt (rdbench.cpp:99-104, 140-151; bench.cpp:425-474): the level history per rho,
    a blank line, then the eoc summary; the history matches the oracle's adaptive_solve from
    build_structured_cube(8) level for level (dofs and iterations equal; the columns agree to the
    CSV's %.6e, i.e. within 1e-6 relative)."""
    path = tmp_path / "adapt.csv"
    out = subprocess.run([_built(RDBENCH), "adapt", "--rho", "1e-2", "--budget", "3000", "--tol", "1e-10",
                          "--out", str(path)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    hist_text, summ_text = path.read_text().split("\n\n")
    rows = list(csv.DictReader(io.StringIO(hist_text)))
    summ = list(csv.DictReader(io.StringIO(summ_text)))
    assert list(rows[0].keys()) == ["rho", "level", "dofs", "eta", "l2_sq", "hm1_sq", "iterations", "seconds"]
    assert list(summ[0].keys()) == ["rho", "dofs", "l2_sq", "l2_eoc", "hm1_sq", "hm1_eoc"]
    orows, _, _ = O.adaptive_solve(O.build_structured_cube(8), "box", 1e-2, 3000, tol=1e-10)
    assert len(rows) == len(orows) >= 2
    for r, o in zip(rows, orows):
        assert int(r["level"]) == o["level"] and int(r["dofs"]) == o["dofs"]
        assert int(r["iterations"]) == o["iterations"]
        for k, ok in (("eta", "eta"), ("l2_sq", "err_l2_sq"), ("hm1_sq", "err_hm1_sq")):
            assert float(r[k]) == pytest.approx(o[ok], rel=1e-6), k
    assert int(summ[0]["dofs"]) == orows[-1]["dofs"]
