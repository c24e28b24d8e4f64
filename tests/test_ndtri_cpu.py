"""The generated inverse-normal approximation (csrc/rk_ndtri.cuh, tools/gen_ndtri.py) against
scipy.special.ndtri -- the function the reference samples with (simulate.py:71-74) -- in float64
on the host: the device evaluates the same formulas with FMAs."""
import os
import re

import numpy as np
import pytest

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2605_29284_b200", "csrc",
                   "rk_ndtri.cuh")


def _consts():
    src = open(HDR).read()
    scal = {m.group(1): float.fromhex(m.group(2))
            for m in re.finditer(r"constexpr double (\w+) = (\S+);", src)}
    arrs = {}
    for m in re.finditer(r"__constant__ (?:const )?double (\w+)\[\d+\] = \{(.*?)\};", src, re.S):
        arrs[m.group(1)] = [float.fromhex(t.split("/*")[0].strip()) for t in m.group(2).split(",")]
    return scal, arrs


def _horner(c, x):
    acc = np.full_like(x, c[-1])
    for a in c[-2::-1]:
        acc = acc * x + a
    return acc


def _ndtri_host(u):
    s, a = _consts()
    u = np.asarray(u, dtype=np.float64)
    z = np.empty_like(u)
    tail = np.abs(u - 0.5) > s["kNdtriQmax"]
    q = u[~tail] - 0.5
    v = s["kNdtriR2"] - q * q
    z[~tail] = q * (_horner(a["kNdtriP"], v) / _horner(a["kNdtriQ"], v))
    ut = u[tail]
    m = np.where(ut > 0.5, 1.0 - ut, ut)
    with np.errstate(divide="ignore"):
        t = np.sqrt(-np.log(m)) - s["kNdtriS0"]
    with np.errstate(invalid="ignore", divide="ignore"):
        zt = np.where(m > 0, _horner(a["kNdtriT"], t) / _horner(a["kNdtriS"], t), np.inf)
    z[tail] = np.where(ut > 0.5, zt, -zt)
    return z


def _sample_us():
    rng = np.random.default_rng(1)
    k = np.concatenate([np.arange(0, 4096, dtype=np.uint64),                       # smallest u
                        rng.integers(0, 2 ** 53, size=200000, dtype=np.uint64),
                        np.uint64(2 ** 53) - 1 - np.arange(0, 4096, dtype=np.uint64)])   # largest u
    u = (k.astype(np.float64) + 0.5) * 2.0 ** -53
    edges = np.array([0.04, 0.96, 0.5 - 0.46, 0.5 + 0.46, 0.5, 0.25, 0.75])
    edges = np.concatenate([edges, np.nextafter(edges, 0), np.nextafter(edges, 1)])
    return np.concatenate([u, edges])


def test_ndtri_approximation_matches_scipy():
    sp = pytest.importorskip("scipy.special")
    u = _sample_us()
    ref = sp.ndtri(u)
    z = _ndtri_host(u)
    fin = np.isfinite(ref) & (ref != 0)
    rel = np.abs(z[fin] - ref[fin]) / np.abs(ref[fin])
    assert rel.max() < 2e-15, rel.max()
    assert np.array_equal(z[~fin], ref[~fin])      # u = 1/2 -> 0; u rounding to 1 -> +inf
    assert np.all(np.sign(z[fin]) == np.sign(ref[fin]))
