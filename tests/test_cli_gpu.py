"""CLI on the GPU path (paper_2605_29284_b200/cli.py) against files written by the reference
CLI (tests/golden/cli, oracle/make_golden.py:gen_cli): same headers, fields within 1e-10,
byte-identical reruns (test_acceptance.py:246-266), RAPIDKRIG_SEED, exit statuses."""
import os

import numpy as np
import pytest

from rk_testutil import has_gpu, rel_err

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

CLI = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")
OBS = os.path.join(CLI, "obs.csv")
MODEL = ["--sigma2", "1.0", "--alpha", "5.0", "--nu", "1.0", "--tau2", "0.05"]
RUNS = {
    "predict_rapid": ["predict", "--grid", "32x24", "--L", "3", "--covariates", "1+x+y"],
    "predict_exact": ["predict", "--grid", "32x24", "--method", "exact", "--domain", "0,1,0,1"],
    "simulate": ["simulate", "--grid", "32x32", "--draws", "10", "--seed", "7", "--save-draws"],
}


@pytest.fixture(scope="module")
def cli():
    from paper_2605_29284_b200.cli import cli_main
    from paper_2605_29284_b200.io import read_grid_output
    return cli_main, read_grid_output


@pytest.mark.parametrize("name", sorted(RUNS))
def test_cli_outputs_match_reference(cli, tmp_path, name):
    cli_main, read = cli
    out = str(tmp_path / "o.rkg")
    assert cli_main([*RUNS[name], "--obs", OBS, "--out", out, *MODEL]) == 0
    ours, ref = read(out), read(os.path.join(CLI, name + ".rkg"))
    assert ours.header == ref.header
    for k, v in ref.fields.items():
        assert rel_err(ours.fields[k], v) < 1e-10, k
    out2 = str(tmp_path / "o2.rkg")
    assert cli_main([*RUNS[name], "--obs", OBS, "--out", out2, *MODEL]) == 0
    assert open(out, "rb").read() == open(out2, "rb").read()


def test_seed_env_exit_codes(cli, tmp_path, monkeypatch, capsys):
    cli_main, read = cli
    base = ["simulate", "--obs", OBS, "--grid", "12x12", "--draws", "4", *MODEL]
    a, b = str(tmp_path / "a.rkg"), str(tmp_path / "b.rkg")
    assert cli_main([*base, "--seed", "3", "--out", a]) == 0
    monkeypatch.setenv("RAPIDKRIG_SEED", "3")
    assert cli_main([*base, "--seed", "99", "--out", b]) == 0
    assert open(a, "rb").read() == open(b, "rb").read()
    monkeypatch.delenv("RAPIDKRIG_SEED")
    assert cli_main(["predict", "--obs", OBS, "--frobnicate"]) == 1
    assert "usage" in capsys.readouterr().err.lower()
    assert cli_main(["predict", "--obs", str(tmp_path / "nope.csv"), "--out", a, "--grid", "8x8", *MODEL]) == 1
    # a correlation range comparable to the domain breaks the circulant embedding (numeric)
    rc = cli_main(["simulate", "--obs", OBS, "--out", a, "--grid", "24x24", "--domain", "0,1,0,1", "--draws", "3",
                   "--seed", "1", "--sigma2", "1.0", "--alpha", "1.0", "--nu", "1.5", "--tau2", "0.05"])
    assert rc == 2
    assert "numeric error" in capsys.readouterr().err
