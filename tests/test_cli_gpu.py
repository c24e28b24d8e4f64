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


def test_timing_study_and_its_data(tmp_path):
    """studies.run_timing rows (studies.py:289-390) and its data: the (seed, n) Philox stream's
    uniforms then normals, identical to numpy Philox + scipy ndtri."""
    import scipy.special as sp
    from paper_2605_29284_b200 import studies
    from paper_2605_29284_b200.cli import cli_main
    from paper_2605_29284_b200.simulate import std_normals
    n, seed = 70, 3
    rng = np.random.Generator(np.random.Philox(key=seed + (n << 64)))
    rng.uniform(0, 1, n), rng.uniform(0, 1, n)
    ref = sp.ndtri((rng.integers(0, 1 << 53, size=n).astype(float) + 0.5) / float(1 << 53))
    assert rel_err(std_normals(seed, n, n, start=2 * n), ref) < 1e-14
    rows = studies.run_timing(ns=(60,), grid_ladder=((20, 16),), methods=("exact", "rapid-L2", "cs-fast"), reps=1)
    assert [r.method for r in rows] == ["exact", "rapid-L2", "cs-fast"]
    assert all(r.grid == (20, 16) and r.predict_seconds > 0 and not r.censored for r in rows)
    out = str(tmp_path / "t.csv")
    assert cli_main(["bench-time", "--out", out, "--ns", "40", "--grids", "16x16", "--methods", "rapid-L4",
                     "--reps", "1"]) == 0
    assert open(out).read().splitlines()[0] == "method,n,grid,setup_seconds,predict_seconds,reps,censored"
    assert cli_main(["bench-error", "--out", out]) == 1
