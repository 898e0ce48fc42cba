"""The batch driver (paper_1305_4886_b200/cli.py) on the host: config
parsing, CSV round trips and the configuration exit code, against the
reference driver's formats (bg/cli.py:31-148; tests/golden/cli from
make_cli_golden.py).  The GPU commands are in test_gpu_cli.py."""

import os

import numpy as np
import pytest

from conftest import GOLDEN

from paper_1305_4886_b200 import cli
from paper_1305_4886_b200.errors import ConfigError

CLI = os.path.join(GOLDEN, "cli")


def test_reads_reference_config_and_overrides(tmp_path):
    cfg = cli.read_config(os.path.join(CLI, "job.cfg"), ["theta0=2,0.3,0.1", "tile = 128"])
    assert cfg.get("kernel") == "matern-nugget"
    assert cfg.get("theta0") == [2.0, 0.3, 0.1]
    assert cfg.get("nu") == 0.5 and cfg.get("tile") == 128 and cfg.get("workers") == 1
    assert cfg.get("se_fit") is False and cfg.get("bench_h") == [1, 2, 3]
    with pytest.raises(ConfigError, match="out"):
        cfg.get("out")
    p = tmp_path / "bad.cfg"
    p.write_text("kernel matern\n")
    with pytest.raises(ConfigError, match="expected key = value"):
        cli.read_config(str(p))
    with pytest.raises(ConfigError, match="bad value for 'workers'"):
        cli.read_config(os.path.join(CLI, "job.cfg"), ["workers=two"]).get("workers")


def test_tables_round_trip_reference_csv(tmp_path):
    X, y = cli.load_table(os.path.join(CLI, "data.csv"), with_y=True)
    assert X.shape == (300, 2) and y.shape == (300,)
    G, none = cli.load_table(os.path.join(CLI, "grid.csv"), with_y=False)
    assert G.shape == (25, 2) and none is None
    out = tmp_path / "t.csv"
    cli.save_table(str(out), ["x1", "x2", "y"], np.column_stack([X, y]))
    # byte-identical to the reference driver's writer (repr precision)
    assert out.read_text() == open(os.path.join(CLI, "data.csv")).read()
    with pytest.raises(ConfigError, match="last column must be 'y'"):
        cli.load_table(os.path.join(CLI, "grid.csv"), with_y=True)
    with pytest.raises(ConfigError, match="must not have a 'y'"):
        cli.load_table(os.path.join(CLI, "data.csv"), with_y=False)
    rag = tmp_path / "rag.csv"
    rag.write_text("a,y\n1,2\n3\n")
    with pytest.raises(ConfigError, match="ragged"):
        cli.load_table(str(rag), with_y=True)


def test_configuration_errors_exit_2(tmp_path, capsys):
    assert cli.main(["loglik", str(tmp_path / "missing.cfg")]) == 2
    assert cli.main(["loglik", os.path.join(CLI, "job.cfg"), "backend=in-process"]) == 2
    assert "config error" in capsys.readouterr().err
