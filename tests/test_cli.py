"""CLI contract (reference tools/main.cpp exit codes and output formats,
mirrored from the reference's cli_test.cpp expectations)."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXAMPLE = "3*x^8-x^7+2*x^6+x^5-4*x^4+9*x^3-3*x^2-2*x+1"


def run(*args):
    r = subprocess.run([sys.executable, "-m", "paper_1307_5655_b200", *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout, r.stderr


def test_compile_stats_horner():
    code, out, err = run("compile", "--poly", EXAMPLE, "--scheme", "horner", "--stats")
    assert code == 0 and err == ""
    assert "nodes: 9" in out and "max_lazy_height: 0" in out and "exponents[x]: 1" in out


def test_compile_dot_single_node(tmp_path):
    dot = tmp_path / "t.dot"
    code, _, _ = run("compile", "--poly", "x", "--scheme", "estrin", "--dot", str(dot))
    assert code == 0 and "c=1 d=1 lh=0" in dot.read_text()


def test_syntax_error_is_exit_one():
    code, out, err = run("compile", "--poly", "3*x^^2")
    assert code == 1 and out == "" and "position" in err


def test_unknown_scheme_is_exit_two():
    code, out, err = run("compile", "--poly", "x+1", "--scheme", "nope")
    assert code == 2 and out == "" and err


def test_threshold_scheme_name():
    code, out, _ = run("compile", "--poly", EXAMPLE, "--scheme", "balanced:horner@2", "--stats")
    assert code == 0 and "nodes: 9" in out


def test_unwritable_dot_is_exit_four():
    code, out, _ = run("compile", "--poly", "x", "--dot", "/nonexistent/dir/t.dot")
    assert code == 4 and out == ""


def test_parser_matches_reference_grammar():
    from paper_1307_5655_b200.parser import ParseError, parse_polynomial
    p = parse_polynomial("x^2*y^2 + 2*x*y + 1")
    assert p.variables == ("x", "y")
    assert sorted(map(tuple, p.exponents.tolist())) == [(0, 0), (1, 1), (2, 2)]
    q = parse_polynomial("x*x*x - 2", ["x"])  # repeated factors add exponents
    assert q.exponents.tolist() == [[3], [0]] and q.coefficients.tolist() == [1, -2]
    for bad in ("", "2*3", "x+", "x y", "x^-1", "+-x"):
        with pytest.raises(ParseError):
            parse_polynomial(bad)
    with pytest.raises(ParseError):
        parse_polynomial("z", ["x"])  # unknown variable in a fixed order


@pytest.mark.gpu
def test_eval_integer_domain_all_schemes():
    for s in ("direct", "horner", "estrin", "balanced"):
        code, out, _ = run("eval", "--poly", EXAMPLE, "--scheme", s, "--domain", "int", "--at", "x=2")
        assert code == 0 and out == "793\n"


@pytest.mark.gpu
def test_eval_float_and_interval():
    code, out, _ = run("eval", "--poly", "x^2+1", "--domain", "float", "--at", "x=1.5")
    assert code == 0 and out == "3.25\n"
    code, out, _ = run("eval", "--poly", "x^2+1", "--domain", "interval", "--at", "x=[0.9,1.1]")
    lo, hi = (float(v) for v in out.strip()[1:-1].split(","))
    assert code == 0 and lo <= 2.0 <= hi


@pytest.mark.gpu
def test_eval_binding_errors_are_exit_three():
    code, out, err = run("eval", "--poly", "x*y", "--domain", "int", "--at", "x=2")
    assert code == 3 and out == "" and "unbound" in err
    code, _, _ = run("eval", "--poly", "x", "--domain", "int", "--at", "x=abc")
    assert code == 3


@pytest.mark.gpu
def test_eval_multivariate_and_batch_file(tmp_path):
    code, out, _ = run("eval", "--poly", "x^2*y^2 + 2*x*y + 1", "--scheme", "horner",
                       "--domain", "int", "--at", "x=2,y=3")
    assert code == 0 and out == "49\n"
    pts = np.array([[2, 3], [0, 0], [1, -1], [-2, 5]], dtype=np.int64)
    np.save(tmp_path / "p.npy", pts)
    code, _, err = run("eval", "--poly", "x^2*y^2 + 2*x*y + 1", "--domain", "int",
                       "--points", str(tmp_path / "p.npy"), "--out", str(tmp_path / "o.npy"))
    assert code == 0, err
    x, y = pts[:, 0], pts[:, 1]
    assert np.load(tmp_path / "o.npy").tolist() == (x * x * y * y + 2 * x * y + 1).tolist()


@pytest.mark.gpu
def test_bench_writes_reference_csv_header(tmp_path):
    csvp = tmp_path / "b.csv"
    code, out, err = run("bench", "--schemes", "horner,balanced", "--degrees", "16,32",
                         "--points", "20000", "--reps", "3", "--csv", str(csvp))
    assert code == 0, err
    text = csvp.read_text()
    assert text.startswith("scheme,degree,terms,coeff_bits,point_bits,workers,reps,median_ns,"
                           "ratio_vs_balanced\n")
    assert text.count("\n") == 5 and ",1.0000\n" in text and "degree 16" in out
