"""The XOR swizzles between the first two Stockham stages (csrc/rk_fft.cuh, fft_stage SWZ 1-4):
each is a bijection of the line's element indices, the first stage's stores (8 lanes of a quarter
warp = one 128-byte shared-memory wavefront of 16-byte elements) hit eight distinct 16-byte bank
groups, and so do the next stage's loads.  Host-side restatement of the index maps, checked
exhaustively for the line lengths the plans produce."""
import pytest


def swz_pow2(i):      # SWZ 1 / 2: radix-8 pair of a 2^a line
    return i ^ ((i >> 3) & 7)


def swz_r6(i):        # SWZ 3 / 4: radix 6 followed by radix 9 / 8
    return i ^ ((i >> 3) & 1)


def groups_distinct(addrs):
    return len({a % 8 for a in addrs}) == len(addrs)


@pytest.mark.parametrize("n", [64, 512, 2048, 4096, 32768])
def test_pow2_swizzle(n):
    assert sorted(swz_pow2(i) for i in range(n)) == list(range(n))
    nb = n // 8
    for j0 in range(0, nb, 8):          # stage 1 stores: butterfly j writes 8 j + k
        for k in range(8):
            assert groups_distinct([swz_pow2(8 * j + k) for j in range(j0, j0 + 8)])
            # the kernel's closed form of the same address
            assert all(swz_pow2(8 * j + k) == 8 * j + (k ^ (j & 7)) for j in range(j0, j0 + 8))
    for j0 in range(0, nb, 8):          # stage 2 loads: butterfly j reads j + k nb
        for k in range(8):
            assert groups_distinct([swz_pow2(j + k * nb) for j in range(j0, j0 + 8)])
            assert all(swz_pow2(j + k * nb) == (j + k * nb) ^ (((j >> 3) + k * (nb >> 3)) & 7)
                       for j in range(j0, j0 + 8))


@pytest.mark.parametrize("n,r2", [(54, 9), (486, 9), (4374, 9), (432, 9), (3888, 9), (1944, 9), (384, 8), (3072, 8)])
def test_radix6_swizzle(n, r2):
    assert sorted(swz_r6(i) for i in range(n)) == list(range(n))
    nb6 = n // 6
    for j0 in range(0, nb6 - 7, 8):     # stage 1 stores: butterfly j writes 6 j + k
        for k in range(6):
            assert groups_distinct([swz_r6(6 * j + k) for j in range(j0, j0 + 8)])
    nb = n // r2
    assert nb % 2 == 0
    for j0 in range(0, nb - 7, 8):      # stage 2 loads: butterfly j reads j + k nb
        for k in range(r2):
            assert groups_distinct([swz_r6(j + k * nb) for j in range(j0, j0 + 8)])
