"""Pins for the oracle's partition (DESIGN reading R2).

The paper only says the states are "shuffled and then selected and processed
in blocks of m" before every operator application and that the
theory holds for any order (L162, L605).  We fix a counter-based permutation;
these tests pin the oracle's implementation to values that do not come from it.
"""
import collections

import numpy as np
import pytest

import oracle
from conftest import golden


def test_mix64_splitmix_kats():
    kat = golden("partition_kat.json")
    for x, y in kat["mix64"]:
        assert oracle.mix64(int(x, 16)) == int(y, 16)


def test_prefix_kat_from_survey():
    kat = golden("partition_kat.json")["prefix"]
    perm = oracle.partition(kat["n"], kat["seed"], kat["k"])
    assert list(perm[: len(kat["pi_prefix"])]) == kat["pi_prefix"]


@pytest.mark.parametrize("n", [1, 2, 3, 5, 50, 64, 65, 1000, 10_000, 50_000, 1_000_000])
def test_bijection(n):
    perm = oracle.partition(n, 7, 3)
    assert np.array_equal(np.sort(perm), np.arange(n, dtype=np.uint32))


@pytest.mark.parametrize("n", [1, 2, 7, 50, 4097, 100_000])
def test_inverse_composes_to_identity(n):
    perm = oracle.partition(n, 123, 9)
    inv = oracle.partition_inverse(n, 123, 9)
    assert np.array_equal(inv[perm], np.arange(n, dtype=np.uint32))
    assert np.array_equal(perm[inv], np.arange(n, dtype=np.uint32))


def test_identity_flag_is_paper_ascending_order():
    # "we assume that the states are processed in ascending order"
    assert np.array_equal(oracle.partition(17, 5, 1, identity=True), np.arange(17))


def test_sweeps_and_seeds_draw_different_orders():
    a = oracle.partition(1000, 1, 1)
    assert not np.array_equal(a, oracle.partition(1000, 1, 2))
    assert not np.array_equal(a, oracle.partition(1000, 2, 1))
    assert np.array_equal(a, oracle.partition(1000, 1, 1))  # deterministic


def test_positions_are_roughly_uniform():
    # a dropped round or key mixing would leave strong structure: over 4000
    # sweeps every (position, state) cell of n=5 must be hit ~1/5 of the time
    n, K = 5, 4000
    counts = np.zeros((n, n))
    for k in range(1, K + 1):
        p = oracle.partition(n, 99, k)
        counts[np.arange(n), p] += 1
    freq = counts / K
    assert np.all(np.abs(freq - 0.2) < 0.035), freq


def test_independent_python_reading_of_the_spec():
    """A second, from-the-text implementation (pure Python) of SURVEY 8(c)-1."""
    M = (1 << 64) - 1

    def mix(z):
        z = (z + 0x9E3779B97F4A7C15) & M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)

    def perm(n, seed, k):
        w = max(2, (n - 1).bit_length())
        w += w & 1
        h = w // 2
        key = mix(mix(seed) ^ k)
        rk = [mix(key ^ r) for r in range(6)]

        def enc(x):
            L, R = x >> h, x & ((1 << h) - 1)
            for r in range(6):
                L, R = R, L ^ (mix(rk[r] ^ R) >> (64 - h))
            return (L << h) | R

        out = []
        for p in range(n):
            x = enc(p)
            while x >= n:
                x = enc(x)
            out.append(x)
        return out

    for n, seed, k in [(1, 0, 1), (2, 3, 4), (50, 42, 7), (333, 2**63 + 5, 12), (1024, 0, 1)]:
        assert list(oracle.partition(n, seed, k)) == perm(n, seed, k)


def test_batches_follow_eq_M():
    # Eq. M(i) under the identity order: the states updated before
    # position p are exactly positions < b*floor(p/b); last batch short (R4).
    n, b = 5, 2
    groups = collections.defaultdict(list)
    for p, s in enumerate(oracle.partition(n, 0, 1, identity=True)):
        groups[p // b].append(int(s))
    assert list(groups.values()) == [[0, 1], [2, 3], [4]]
