"""The batch driver's commands on the GPU against the reference driver's
own outputs for the same job files (tests/golden/cli, make_cli_golden.py;
bg/cli.py:191-261)."""

import contextlib
import csv
import io
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, relerr

pytestmark = pytest.mark.gpu

CLI = os.path.join(GOLDEN, "cli")


def _run(args):
    from paper_1305_4886_b200 import cli
    buf = io.StringIO()
    cwd = os.getcwd()
    os.chdir(ROOT)  # the job files name the data relative to the repo
    try:
        with contextlib.redirect_stdout(buf):
            rc = cli.main(args)
    finally:
        os.chdir(cwd)
    return rc, buf.getvalue()


def test_loglik_matches_reference_driver():
    rc, out = _run(["loglik", os.path.join(CLI, "job.cfg"), "tile=128"])
    assert rc == 0
    want = float(open(os.path.join(CLI, "loglik.txt")).read().split()[1])
    got = float(out.split()[1])
    assert abs(got - want) <= 1e-10 * abs(want)


def test_predict_csv_matches_reference_driver(tmp_path):
    out = tmp_path / "pred.csv"
    rc, _ = _run(["predict", os.path.join(CLI, "job.cfg"), "se_fit=true", f"out={out}", "tile=128"])
    assert rc == 0
    got = list(csv.reader(open(out)))
    want = list(csv.reader(open(os.path.join(CLI, "predict.csv"))))
    assert got[0] == want[0] == ["mean", "se"]
    g, w = np.array(got[1:], dtype=float), np.array(want[1:], dtype=float)
    assert relerr(g[:, 0], w[:, 0]) <= 1e-9 and relerr(g[:, 1], w[:, 1]) <= 1e-9


def test_bench_chol_csv_schema_and_residuals(tmp_path):
    out = tmp_path / "bench.csv"
    rc, log = _run(["bench-chol", os.path.join(CLI, "bench.cfg"), f"out={out}", "tile=128",
                    "bench_n=64,600"])
    assert rc == 0 and "bench-chol n=600 P=1 h=2" in log
    got = list(csv.reader(open(out)))
    want = list(csv.reader(open(os.path.join(CLI, "bench.csv"))))
    assert got[0] == want[0] == ["n", "P", "h", "seconds", "residual"]
    assert [r[:3] for r in got[1:]] == [["64", "1", "1"], ["64", "1", "2"], ["600", "1", "1"],
                                        ["600", "1", "2"]]
    for r in got[1:]:
        assert float(r[3]) > 0 and float(r[4]) <= 1e-14


def test_fit_and_simulate_write_outputs(tmp_path):
    fit = tmp_path / "fit.json"
    rc, _ = _run(["fit", os.path.join(CLI, "job.cfg"), f"out={fit}", "max_evals=30", "tile=128"])
    assert rc == 0
    doc = json.load(open(fit))
    assert set(doc) == {"theta", "log_density", "converged", "n_evals", "trace"}
    assert len(doc["theta"]) == 3 and doc["n_evals"] == len(doc["trace"])
    want = float(open(os.path.join(CLI, "loglik.txt")).read().split()[1])
    assert doc["log_density"] >= want - 1e-9  # the optimizer starts at theta0
    sims = tmp_path / "sims.csv"
    rc, _ = _run(["simulate", os.path.join(CLI, "job.cfg"), f"out={sims}", "r=4", "post=false",
                  "tile=128"])
    assert rc == 0
    rows = list(csv.reader(open(sims)))
    assert rows[0] == ["sim1", "sim2", "sim3", "sim4"] and len(rows) == 301


def test_numerical_error_exits_3(tmp_path, capsys):
    # a nugget-free exponential kernel on duplicated points is singular
    data = tmp_path / "dup.csv"
    data.write_text("x,y\n0.5,1.0\n0.5,2.0\n")
    rc, _ = _run(["loglik", os.path.join(CLI, "job.cfg"), f"data={data}", "kernel=matern",
                  "theta0=1,0.2", "tile=128"])
    assert rc == 3
    assert "numerical error at theta 1,0.2" in capsys.readouterr().err
