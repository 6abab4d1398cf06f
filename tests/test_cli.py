"""CLI.  CPU: argument and input
errors exit 2 with a message naming the problem, reps=0 prints an empty
table; GPU: the SPEC examples of run_track / run_monodromy / run_pieri /
run_evalbench through the product."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def cli(*args, cwd=None):
    r = subprocess.run([sys.executable, "-m", "paper_1501_06625_b200.cli", *args], capture_output=True, text=True,
                       cwd=cwd or ROOT)
    return r.returncode, r.stdout, r.stderr


def test_unknown_flag_is_a_usage_error():
    rc, _, err = cli("--mode", "evalbench", "--bogus")
    assert rc == 2 and "unrecognized" in err


def test_pieri_shape_error():
    rc, _, err = cli("--mode", "pieri", "--pieri", "5,2,2")
    assert rc == 2 and "M + P = N" in err


def test_missing_system_file(tmp_path):
    rc, _, err = cli("--mode", "track", "--system", str(tmp_path / "nope.sys"))
    assert rc == 2 and "nope.sys" in err


def test_parse_error_reports_line_and_column(tmp_path):
    p = tmp_path / "bad.sys"
    p.write_text("vars: x0 x1\nx0 + * x1;\n")
    rc, _, err = cli("--mode", "track", "--system", str(p))
    assert rc == 2 and "line 2, column" in err


def test_missing_witness_names_the_file():
    rc, _, err = cli("--mode", "monodromy", "--cyclic", "32")
    assert rc == 2 and "--witness FILE" in err


def test_evalbench_zero_reps_is_an_empty_table():
    rc, out, _ = cli("--mode", "evalbench", "--cyclic", "16", "--reps", "0")
    assert rc == 0 and out.split() == ["prec", "n", "N", "reps", "ms/eval"]


def test_step_control_validation():
    rc, _, err = cli("--mode", "track", "--cyclic", "16", "--max-step", "2")
    assert rc == 2 and "step control" in err


@pytest.mark.gpu
def test_track_trivial_fixture(gpu, tmp_path):
    """trivial 1-variable homotopy fixture -> exit 0, s = 1;
    the end solution is written in the solutions format."""
    f = tmp_path / "f.sys"
    f.write_text("vars: x\nx - 2;\n")
    g = tmp_path / "g.sys"
    g.write_text("vars: x\nx - 1;\n")
    out = tmp_path / "end.sol"
    rc, stdout, err = cli("--mode", "track", "--system", str(f), "--start-system", str(g), "--out", str(out),
                          "--trace", str(tmp_path / "t.txt"))
    assert rc == 0, err
    row = stdout.splitlines()[1].split()
    assert row[2] == "1"
    from paper_1501_06625_b200 import PrecisionMode as PM, read_solutions
    sol = read_solutions(out.read_text(), PM.DD)
    assert abs(complex(sol[0].point[0, 0, 0], sol[0].point[1, 0, 0]) - 2) < 1e-15
    assert len((tmp_path / "t.txt").read_text().splitlines()) > 2


@pytest.mark.gpu
def test_track_max_steps_one_fails(gpu):
    """maxSteps = 1 on the cyclic-4 leg -> exit nonzero, s = 0."""
    rc, out, _ = cli("--mode", "track", "--cyclic", "4", "--max-steps", "1")
    assert rc == 1 and out.splitlines()[1].split()[2] == "0"


@pytest.mark.gpu
def test_track_deterministic_rows(gpu):
    """same config + seed -> identical report rows except wall time."""
    a = cli("--mode", "track", "--cyclic", "16", "--seed", "3")[1].splitlines()[1].split()[:-1]
    b = cli("--mode", "track", "--cyclic", "16", "--seed", "3")[1].splitlines()[1].split()[:-1]
    assert a == b


@pytest.mark.gpu
def test_monodromy_cyclic4_degree_2(gpu):
    """--cyclic 4 --precision dd -> degree 2."""
    rc, out, err = cli("--mode", "monodromy", "--cyclic", "4", "--precision", "dd", "--seed", "11")
    assert rc == 0, err
    assert "degree estimate 2" in out


@pytest.mark.gpu
def test_pieri_4_2_2(gpu):
    """n=4, m=2, p=2 in D -> success, residual <= 1e-10."""
    rc, out, err = cli("--mode", "pieri", "--pieri", "4,2,2", "--precision", "d")
    assert rc == 0, err
    res = float(out.strip().splitlines()[-1].split("final residual ")[1].split(",")[0])
    assert res <= 1e-10


@pytest.mark.gpu
def test_evalbench_cyclic16(gpu):
    """cyclic-16 -> a D / DD / QD table, times nondecreasing with precision."""
    rc, out, err = cli("--mode", "evalbench", "--cyclic", "16", "--reps", "100")
    assert rc == 0, err
    rows = [l.split() for l in out.splitlines()[1:]]
    assert [r[0] for r in rows] == ["d", "dd", "qd"]
    t = [float(r[-1]) for r in rows]
    assert t[0] <= t[1] <= t[2]
