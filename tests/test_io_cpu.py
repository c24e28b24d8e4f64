"""RKGRID1 / observation-file host code (paper_2605_29284_b200/io.py) against the reference's
format (io.py:1-178): reads the reference-written files in tests/golden/cli, rewrites them
byte for byte, and covers the loader's and writer's error paths."""
import os
import warnings

import numpy as np
import pytest

from paper_2605_29284_b200 import io as rio
from paper_2605_29284_b200.errors import DomainError

CLI = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")


@pytest.mark.parametrize("name", ["predict_rapid", "predict_exact", "simulate"])
def test_reads_and_rewrites_reference_files_bytewise(tmp_path, name):
    src = os.path.join(CLI, name + ".rkg")
    g = rio.read_grid_output(src)
    nx, ny = g.dims
    assert all(f.shape == (ny, nx) and np.all(np.isfinite(f)) for f in g.fields.values())
    base = {"version", "nx", "ny", "x0", "y0", "dx", "dy", "fields"}
    extra = {k: v for k, v in g.header.items() if k not in base}
    out = tmp_path / "re.rkg"
    rio.write_grid_output(out, nx=nx, ny=ny, x0=float(g.header["x0"]), y0=float(g.header["y0"]),
                          dx=float(g.header["dx"]), dy=float(g.header["dy"]), fields=g.fields, extra=extra)
    assert open(out, "rb").read() == open(src, "rb").read()


def test_roundtrip_bitwise_and_validation(tmp_path):
    rng = np.random.default_rng(0)
    f = {"a": rng.normal(size=(3, 5)), "b": np.array([[np.pi] * 5] * 3) * 1e300}
    p = tmp_path / "g.rkg"
    rio.write_grid_output(p, nx=5, ny=3, x0=0.1, y0=-2.0, dx=0.25, dy=0.5, fields=f, extra={"k": 7})
    g = rio.read_grid_output(p)
    assert g.header["k"] == "7" and g.header["fields"] == "a,b" and g.dims == (5, 3)
    assert all(np.array_equal(g.fields[k].view(np.uint64), f[k].view(np.uint64)) for k in f)
    with pytest.raises(DomainError):
        rio.write_grid_output(p, nx=5, ny=3, x0=0, y0=0, dx=1, dy=1, fields={"a": np.zeros((5, 3))})
    with pytest.raises(DomainError):
        rio.write_grid_output(p, nx=5, ny=3, x0=0, y0=0, dx=1, dy=1, fields={})
    bad = tmp_path / "bad.rkg"
    bad.write_bytes(b"RKGRID2\nnx=1\n\n")
    with pytest.raises(DomainError):
        rio.read_grid_output(bad)
    bad.write_bytes(open(p, "rb").read()[:-8])
    with pytest.raises(DomainError):
        rio.read_grid_output(bad)


def test_observation_loader(tmp_path):
    p = tmp_path / "o.txt"
    p.write_text("x y z elev\n0 0 1 10\n1 0.5 2 20\n\n0.25 1 3 30\n")
    t = rio.load_observations(p)
    assert len(t) == 3 and t.bbox == (0.0, 1.0, 0.0, 1.0)
    assert np.array_equal(t.covariates["elev"], [10.0, 20.0, 30.0])
    t2 = rio.load_observations(os.path.join(CLI, "obs.csv"))
    assert len(t2) == 60 and not t2.covariates
    for text in ("x,y\n0,0\n", "x,y,z\n0,0\n", "x,y,z\n0,a,1\n", ""):
        p.write_text(text)
        with pytest.raises(DomainError):
            rio.load_observations(p)
    with pytest.raises(DomainError):
        rio.load_observations(tmp_path / "missing.csv")
    p.write_text("x,y,z\n0,0,1\n0,0,2\n1,1,3\n")
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        assert len(rio.load_observations(p)) == 3
    assert any("duplicate" in str(x.message) for x in w)


def test_formula_and_covariates():
    assert rio.parse_formula(" 1 + x+y+ x*y ") == ["1", "x", "y", "x*y"]
    for bad in ("", "+", "1+z", "x^2"):
        with pytest.raises(DomainError):
            rio.parse_formula(bad)
    X = rio.build_covariates(["1", "x*y", "y"], [1.0, 2.0], [3.0, 4.0])
    assert np.array_equal(X, [[1.0, 3.0, 3.0], [1.0, 8.0, 4.0]])
