"""Golden outputs of the REFERENCE command-line driver (bg/cli.py).

Run in the build container only (needs /root/reference, read-only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cli_golden.py

Writes tests/golden/cli/: a small data set (data.csv, grid.csv), the job
configs, and what the reference's `blockgp` printed / wrote for them
(loglik.txt, predict.csv, bench.csv).  tests/test_gpu_cli.py runs this
package's driver on the same files and compares.
"""

import contextlib
import io
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from blockgp import cli  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cli")


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(11)
    n, m = 300, 25
    X = rng.uniform(0, 1, (n, 2))
    d = np.sqrt(((X[:, None] - X[None]) ** 2).sum(-1))
    C = 1.5 * np.exp(-d / 0.2) + 0.05 * np.eye(n)
    y = np.linalg.cholesky(C) @ rng.standard_normal(n)
    g = np.linspace(0.05, 0.95, 5)
    G = np.stack(np.meshgrid(g, g, indexing="xy"), -1).reshape(-1, 2)
    cli.write_csv(os.path.join(OUT, "data.csv"), ["x1", "x2", "y"], np.column_stack([X, y]))
    cli.write_csv(os.path.join(OUT, "grid.csv"), ["x1", "x2"], G)
    base = ("kernel = matern-nugget\ntheta0 = 1.5,0.2,0.05\nnu = 0.5\n"
            "data = tests/golden/cli/data.csv\npred_grid = tests/golden/cli/grid.csv\n")
    with open(os.path.join(OUT, "job.cfg"), "w") as f:
        f.write("# reference job (workers = 1, in-process)\nworkers = 1\n" + base)
    with open(os.path.join(OUT, "bench.cfg"), "w") as f:
        f.write("bench_n = 64,200\nbench_p = 1\nbench_h = 1,2\nseed = 0\n")
    root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.chdir(root)
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        assert cli.main(["loglik", os.path.join(OUT, "job.cfg")]) == 0
    with open(os.path.join(OUT, "loglik.txt"), "w") as f:
        f.write(buf.getvalue())
    assert cli.main(["predict", os.path.join(OUT, "job.cfg"), "se_fit=true",
                     f"out={os.path.join(OUT, 'predict.csv')}"]) == 0
    assert cli.main(["bench-chol", os.path.join(OUT, "bench.cfg"),
                     f"out={os.path.join(OUT, 'bench.csv')}"]) == 0
    print(buf.getvalue())


if __name__ == "__main__":
    main()
