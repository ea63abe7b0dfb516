"""Pins the product library's host generators (std::mt19937_64 + libstdc++ distributions, the
reference's RNG stack) against golden vectors produced by the real libstdc++
(tests/golden/make_rng_golden.cpp -> tests/golden/rng_golden.json)."""
import json
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "rng_golden.json")))


@pytest.fixture(scope="module")
def cp(built_lib):
    import paper_2603_25691_b200 as cp
    return cp


def test_mt19937_64_stream(cp):
    g = cp.Mt19937_64(0)
    assert [str(v) for v in g.next_u64(8)] == GOLD["mt19937_64_seed0"]
    g2 = cp.Mt19937_64(5489)
    g2.next_u64(9999)
    assert str(g2()) == GOLD["mt19937_64_default_10000th"][0]  # the standard's check value


def test_uniform_real(cp):
    g = cp.Mt19937_64(7)
    got = g.uniform_real(-1.0, 1.0, 64)
    assert np.array_equal(got, np.array(GOLD["uniform_real_m1_1_seed7"]))


def test_uniform_int(cp):
    g = cp.Mt19937_64(11)
    ranges = [(0, 0), (0, 1), (3, 10), (1, 60), (0, 1999999), (5, 1 << 40), (-7, 7), (0, (1 << 62) + 12345),
              (100, 100)]
    got = []
    for _ in range(4):
        for lo, hi in ranges:
            got.append(int(g.uniform_int(lo, hi, 1)[0]))
    assert got == GOLD["uniform_int_mixed_seed11"]


def test_normal(cp):
    g = cp.Mt19937_64(3)
    got = g.normal(0.0, 1.0, 65)
    assert np.array_equal(got, np.array(GOLD["normal_0_1_seed3"]))
    g.normal_reset()  # the golden continues with a fresh distribution object
    got2 = g.normal(2.0, 0.1, 9)
    assert np.array_equal(got2, np.array(GOLD["normal_2_01_seed3_continued"]))


def test_sample_uniform(cp):
    from tests.refinst import sample
    idx, _ = sample([64], np.arange(64, dtype=np.float64), 20, 2)
    assert idx[0].tolist() == GOLD["sample_uniform_N64_q20_seed2"]
    flat = np.zeros(2000000)
    idx, _ = sample([2000000], flat, 50, 1)
    assert idx[0].tolist() == GOLD["sample_uniform_N2000000_q50_seed1"]
    idx, _ = sample([2000000], flat, 200000, 1)
    h = 1469598103934665603
    for x in idx[0].astype(np.int64).tolist():
        h ^= x
        h = (h * 1099511628211) % (1 << 64)
    assert str(h) == GOLD["sample_uniform_N2000000_q200000_seed1_fnv1a"][0]
