"""Sampling module of the oracle and the generator pins.

The SPEC leaves the generator open ("counter-based / splittable", SPEC.md:125,
162); this build pins Philox4x32-10 and checks it against the published
Random123 known-answer vectors (Salmon et al., SC'11; kat_vectors in Random123
v1.14), which also match CUDA's curand_philox4x32_x.h round function.
"""
import json
import os

import numpy as np
import pytest
from scipy import stats

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")

PHILOX_KATS = [
    ((0x00000000, 0x00000000, 0x00000000, 0x00000000), (0x00000000, 0x00000000),
     (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF), (0xFFFFFFFF, 0xFFFFFFFF),
     (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,expect", PHILOX_KATS)
def test_philox_known_answers(orc, ctr, key, expect):
    assert orc.philox4x32_10(ctr, key) == expect


def test_bits53_layout(orc):
    # draw k of (seed, stream, layer): ctr = {k>>1, layer, stream_lo, stream_hi}, key = {seed_lo, seed_hi}
    seed, stream, layer = 0x0123456789ABCDEF, 0xFEDCBA9876543210, 7
    x = orc.philox4x32_10((5, layer, stream & 0xFFFFFFFF, stream >> 32), (seed & 0xFFFFFFFF, seed >> 32))
    assert orc.bits53(seed, stream, layer, 10) == (((x[1] << 32) | x[0]) >> 11)
    assert orc.bits53(seed, stream, layer, 11) == (((x[3] << 32) | x[2]) >> 11)


def test_make_distribution_examples(orc):
    d = orc.make_distribution([1, 1, 1, 1])
    assert np.array_equal(d.probs, [0.25] * 4)
    d = orc.make_distribution([9, 16])                                          # :143
    np.testing.assert_allclose(d.probs, [0.36, 0.64], rtol=0, atol=1e-16)
    with pytest.raises(orc.OracleDegenerateError):                              # :144
        orc.make_distribution([0, 0])
    with pytest.raises(orc.OracleDomainError):                                  # :140
        orc.make_distribution([1, -1])


def test_distribution_invariants(orc):
    rng = np.random.default_rng(5)
    w = rng.uniform(0, 1, 300) ** 4
    w[[3, 77, 299]] = 0.0
    d = orc.make_distribution(w)
    assert abs(d.probs.sum() - 1.0) <= 1e-12
    assert np.all(np.diff(d.cdf) >= 0) and d.cdf[-1] == 1.0
    draws = orc.draw_indices(d, 200_000, seed=9, stream=1)
    assert not np.isin(draws, [3, 77, 299]).any()                               # :132


def test_tiny_probabilities_are_clamped(orc):
    d = orc.make_distribution([1.0, 1e-17, 1.0])
    assert d.probs[1] == 0.0 and d.probs[0] == 0.5 and d.probs[2] == 0.5
    assert not np.any(orc.draw_indices(d, 10_000, seed=1, stream=0) == 1)


def test_draw_point_mass(orc):
    d = orc.make_distribution([0, 1])
    assert np.all(orc.draw_indices(d, 1000, seed=3, stream=4) == 1)


def test_draw_fair_coin(orc):
    d = orc.make_distribution([0.5, 0.5])
    f = np.mean(orc.draw_indices(d, 100_000, seed=11, stream=0) == 0)
    assert 0.494 <= f <= 0.506


def test_draw_determinism_and_stream_independence(orc):
    d = orc.make_distribution(np.arange(1, 9))
    a = orc.draw_indices(d, 500, seed=7, stream=3)
    _ = orc.draw_indices(d, 500, seed=7, stream=4)                              # interleave another stream
    b = orc.draw_indices(d, 500, seed=7, stream=3)
    assert np.array_equal(a, b)
    c = orc.draw_indices(d, 500, seed=7, stream=4)
    assert not np.array_equal(a, c)
    with pytest.raises(orc.OracleDomainError):
        orc.draw_indices(d, 0, seed=7, stream=3)


def test_draw_prefix_property(orc):
    # draw k depends only on (seed, stream, layer, k): a longer draw extends a shorter one
    d = orc.make_distribution(np.arange(1, 30))
    assert np.array_equal(orc.draw_indices(d, 37, 5, 6, 2), orc.draw_indices(d, 100, 5, 6, 2)[:37])


def test_chi_square_goodness_of_fit(orc):
    probs = np.array([0.05, 0.1, 0.2, 0.15, 0.05, 0.25, 0.12, 0.08])
    d = orc.make_distribution(probs)
    draws = orc.draw_indices(d, 1_000_000, seed=2024, stream=0)
    counts = np.bincount(draws, minlength=8)
    p = stats.chisquare(counts, d.probs * len(draws)).pvalue
    assert p > 0.001


def test_golden_draws(orc):
    """Regression pin: index streams of the oracle for fixed inputs
    (tests/golden/make_golden.py). The GPU parity tests check the device draws
    against the same file."""
    with open(os.path.join(GOLDEN, "draws.json")) as f:
        g = json.load(f)
    for case in g["cases"]:
        w = np.array(case["w"])
        dist = orc.weight_probs(w)
        got = orc.draw_indices(dist, case["r"], case["seed"], case["stream"], case["layer"])
        assert got.tolist() == case["indices"]
