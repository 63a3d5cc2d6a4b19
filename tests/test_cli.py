"""The command-line front end (paper_2409_05572_b200/blockeig):
the reference CLI's subcommands, CSV/JSON schemas and exit codes
(tools/blockeig_cli.cpp:214-221,245-400), driven over the product library and,
as the comparison, the same source linked against the oracle
(oracle/_build/blockeig_oracle, test infrastructure)."""
import csv
import io
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PRODUCT_CLI = os.path.join(ROOT, "paper_2409_05572_b200", "blockeig")
ORACLE_CLI = os.path.join(ROOT, "oracle", "_build", "blockeig_oracle")
HIST_COLS = ["iteration", "r_overall", "n_now", "event", "spmv_cols_cum", "solve_cols_cum", "ortho_flops_cum",
             "rr_dim"]
CMP_COLS = ["strategy", "status", "iterations", "r_final", "spmv_cols", "solve_cols", "ortho_flops", "rr_flops",
            "combined_work", "save_pct"]


def cli(exe, *args, env=None):
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.dirname(exe) if exe == ORACLE_CLI else
                        os.path.join(ROOT, "paper_2409_05572_b200", "csrc")], check=True)
    e = dict(os.environ, **(env or {}))
    return subprocess.run([exe, *args], capture_output=True, text=True, timeout=600, env=e)


def rows(text):
    return list(csv.DictReader(io.StringIO(text)))


SOLVE = ["--gen", "laplacian1d:100", "--solver", "lobpcg", "--nev", "4", "--seed", "11"]


# ---------------------------------------------------------------- CPU (oracle build + argument handling)
def test_solve_csv_schema_and_exit_codes():
    r = cli(ORACLE_CLI, "solve", *SOLVE, "--strategy", "fix")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0] == ",".join(HIST_COLS)
    h = rows(r.stdout)
    assert [int(x["iteration"]) for x in h] == list(range(1, len(h) + 1))
    assert {x["event"].split("(")[0] for x in h} <= {"none", "shrink", "expand", "lock"}
    assert "status=converged" in r.stderr and "values:" in r.stderr
    # not converged -> 2; bad input -> 1
    assert cli(ORACLE_CLI, "solve", *SOLVE, "--max-iters", "3").returncode == 2
    assert cli(ORACLE_CLI, "solve", "--solver", "lobpcg").returncode == 1
    assert cli(ORACLE_CLI, "solve", *SOLVE, "--strategy", "bogus").returncode == 1
    assert cli(ORACLE_CLI, "solve", *SOLVE, "--nev", "x").returncode == 1
    assert cli(ORACLE_CLI, "nonsense").returncode == 1


def test_solve_json_and_out_file(tmp_path):
    out = tmp_path / "h.json"
    r = cli(ORACLE_CLI, "solve", *SOLVE, "--strategy", "slope", "--format", "json", "--out", str(out))
    assert r.returncode == 0, r.stderr
    assert "status=converged" in r.stdout  # summary to stdout when --out is given
    d = json.loads(out.read_text())
    assert d["command"] == "solve" and d["status"] == "converged" and len(d["values"]) == 4
    assert set(d["work"]) == {"spmv_cols", "solve_cols", "ortho_flops", "rr_flops", "combined"}
    assert len(d["history"]) == d["iterations"]


def test_compare_concurrent_equals_sequential():
    """compare runs the four strategies concurrently on one matrix handle
    (blockeig_cli.cpp:346-353); each row must equal a sequential solve"""
    r = cli(ORACLE_CLI, "compare", *SOLVE)
    assert r.returncode == 0, r.stderr
    got = rows(r.stdout)
    assert [x["strategy"] for x in got] == ["none", "fix", "slope", "slopek"]
    assert list(got[0].keys()) == CMP_COLS
    for x in got:
        s = cli(ORACLE_CLI, "solve", *SOLVE, "--strategy", x["strategy"], "--format", "json")
        d = json.loads(s.stdout)
        assert int(x["iterations"]) == d["iterations"]
        assert int(x["ortho_flops"]) == d["work"]["ortho_flops"] and int(x["rr_flops"]) == d["work"]["rr_flops"]
        assert float(x["r_final"]) == d["r_final"]
    assert float(got[0]["save_pct"]) == 0.0


def test_gen_writes_matrix_market(tmp_path):
    """gen on the product (host-only path, no device): a symmetric coordinate file
    that the library reads back to the same matrix"""
    out = tmp_path / "a.mtx"
    r = cli(PRODUCT_CLI, "gen", "--gen", "laplacian1d:50", "--out", str(out))
    assert r.returncode == 0, r.stderr
    assert "wrote 50x50 matrix (99 stored entries)" in r.stdout
    text = out.read_text().splitlines()
    assert text[0].startswith("%%MatrixMarket matrix coordinate real symmetric")
    from paper_2409_05572_b200 import blockeig as B
    L = B.Library(os.path.join(ROOT, "paper_2409_05572_b200", "libblockeig_b200.so"))
    a = L.read(str(out))
    assert a.rows == 50 and a.nnz_lower == 99


def test_product_cli_argument_errors_need_no_gpu():
    assert cli(PRODUCT_CLI, "--help").returncode == 0
    assert cli(PRODUCT_CLI, "solve", "--gen", "laplacian1d:10", "--format", "xml").returncode == 1
    assert cli(PRODUCT_CLI, "theory", "example3x3").returncode == 1  # out of scope: library refuses


# ---------------------------------------------------------------- GPU: product vs oracle
@pytest.mark.gpu
@pytest.mark.parametrize("solver", ["si", "sd", "lobpcg", "tracemin"])
def test_product_history_csv_matches_oracle(solver):
    args = ["solve", "--gen", "laplacian1d:100", "--solver", solver, "--nev", "4", "--seed", "11",
            "--strategy", "fix"]
    g = cli(PRODUCT_CLI, *args)
    o = cli(ORACLE_CLI, *args)
    assert g.returncode == o.returncode == 0, (g.stderr, o.stderr)
    hg, ho = rows(g.stdout), rows(o.stdout)
    # r_overall: 1e-6 relative plus an absolute floor of 1e-12 (the residual ratio
    # is relative to ||A||: its rounding noise does not shrink with it, and a ratio
    # near tol 1e-8 differs by ~4e-14).  SD keeps a residual column whose remaining
    # norm sits at the 1e-8 drop threshold for hundreds of iterations (DESIGN.md
    # "Parity"): its drift grows ~10x per 50 iterations past ~300 (2e-6 at 292,
    # 2e-2 at 465 on the B200) until a K4 drop decision flips (kept counts, hence
    # spmv_cols, differ by ~iteration 565 with the same widths): SD's records are
    # compared over the first 250 iterations
    rtol = 1e-6
    for a, b in zip(hg, ho):
        if (a["n_now"], a["event"]) != (b["n_now"], b["event"]):
            break  # a rounding flip (tests/test_gpu_flips.py); the prefix is compared
        if solver == "sd" and int(a["iteration"]) > 250:
            break
        for c in HIST_COLS:
            if c == "r_overall":
                assert abs(float(a[c]) - float(b[c])) <= rtol * float(b[c]) + 1e-12, (a, b)
            else:
                assert a[c] == b[c], (c, a, b)


@pytest.mark.gpu
def test_product_compare_concurrent_equals_sequential():
    """four concurrent product solves on one beig_matrix (per-solve streams and
    workspaces, one shared device CSR) equal the sequential runs bit for bit"""
    r = cli(PRODUCT_CLI, "compare", *SOLVE, "--format", "json", env={"BLOCKEIG_THREADS": "4"})
    assert r.returncode == 0, r.stderr
    conc = {x["strategy"]: x for x in json.loads(r.stdout)["rows"]}
    for strat, x in conc.items():
        s = cli(PRODUCT_CLI, "solve", *SOLVE, "--strategy", strat, "--format", "json")
        d = json.loads(s.stdout)
        assert x["iterations"] == d["iterations"] and x["values"] == d["values"]
        assert x["r_final"] == d["r_final"] and x["work"] == d["work"]
