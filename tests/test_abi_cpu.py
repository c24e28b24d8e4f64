"""CPU-only checks: the C-ABI library loads and exports every declared symbol;
host-side logic (model constants, seeds, chunking, FFT planning) matches the
reference/oracle.  No device computation here."""

import math
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import rk_oracle as ro
from rk_testutil import ROOT, load_golden

HEADER = os.path.join(ROOT, "include", "rapidkrig_b200.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(rk_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2605_29284_b200 import _native as N
    if not os.path.exists(N.LIB_PATH):
        from paper_2605_29284_b200 import build
        build.build()
    return N.load(require_gpu=False)


def test_library_exports_every_declared_symbol(lib):
    declared = _declared()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    from paper_2605_29284_b200 import _native as N
    assert sorted(N.exported_symbols()) == declared
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2605_29284_b200",
                                                                     "librapidkrig_b200.so")],
                         capture_output=True, text=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_library_is_sm100a_native(lib):
    from paper_2605_29284_b200 import _native as N
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_seed_helper(lib):
    assert lib.rk_version() == 1
    g = load_golden("rng")
    for si, s in enumerate(g["seeds"]):
        for ji, j in enumerate(g["js"]):
            assert lib.rk_draw_seed(int(s), int(j)) == int(g["sub"][si, ji])


def test_model_constants_match_reference_arithmetic():
    from paper_2605_29284_b200 import _native as N
    for nu in (0.5, 1.5, 2.5, 12.5, 1.0, 0.75, 3.7):
        m = N.make_model(1.0, 2.0, nu, 0.1)
        n = ro.half_integer_n(nu)
        if n is None:
            assert m.half_n == -1
            gp, gm, g1, g2 = ro.temme_constants(nu - int(nu + 0.5))
            assert (m.temme_gampl, m.temme_gammi, m.temme_gam1, m.temme_gam2) == (gp, gm, g1, g2)
        else:
            coef, pref = ro.half_integer_coeffs(n)
            assert m.half_n == n and list(m.half_coef)[: n + 1] == coef and m.half_pref == pref
        assert m.gamma_nu == math.gamma(nu)


@pytest.mark.parametrize("n_draws", [2, 3, 7, 256, 1001, 1024])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 5, 8, 16])
def test_next_fft_len_and_shards(n_draws, world):
    from paper_2605_29284_b200.rapid import next_fft_len
    from paper_2605_29284_b200.simulate import shard_ranges
    g = load_golden("fft_len")
    assert [next_fft_len(int(k)) for k in g["n"]] == list(g["p"])
    sh = shard_ranges(n_draws, world)
    assert len(sh) == world
    flat = [j for a, b in sh for j in range(a, b)]
    assert flat == list(range(n_draws))
    sizes = [b - a for a, b in sh]
    assert max(sizes) - min(sizes) <= 1


def test_draw_seed_host():
    from paper_2605_29284_b200.simulate import draw_seed
    assert draw_seed(7, 0) != 7
    assert 0 <= draw_seed(2 ** 63, 123) < 2 ** 64
    assert draw_seed(5, 9) == ro.sub_seed(5, 9)


def test_neighborhood_host_matches_oracle():
    from paper_2605_29284_b200.gridding import PaddedGrid, neighborhood
    g = load_golden("grids")
    for i in range(int(g["n"])):
        dims, L, obs = tuple(int(v) for v in g[f"dims_{i}"]), int(g[f"L_{i}"]), g[f"obs_{i}"]
        og = ro.make_grid((0.0, 1.0, 0.0, 1.0), dims, L, obs)
        grid = PaddedGrid(og.origin, og.spacing, og.interior_dims, og.pad)
        for k in range(obs.shape[0]):
            nb = neighborhood(grid, obs[k], L)
            assert np.array_equal(nb.indices, g[f"indices_{i}"][k])


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2605_29284_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            src = open(os.path.join(pkg, f)).read()
            assert "import oracle" not in src and "from oracle" not in src, f
