"""Pins for oracle.philox and oracle.noise (no GPU)."""
import numpy as np
import pytest

from oracle.noise import noise_code, noise_codes_np
from oracle.philox import philox4x32_10, philox4x32_10_np
from tq_testutil import golden_rows


def test_philox_known_answer_vectors():
    rows = golden_rows("philox_kat.txt")
    assert len(rows) == 3
    for r in rows:
        vals = [int(v, 16) for v in r]
        ctr, key, want = vals[0:4], vals[4:6], tuple(vals[6:10])
        assert philox4x32_10(ctr, key) == want
        got = philox4x32_10_np(*[np.array([v]) for v in ctr], np.array([key[0]]), np.array([key[1]]))
        assert tuple(int(g[0]) for g in got) == want


def test_philox_vectorised_matches_scalar():
    rng = np.random.default_rng(1)
    c = rng.integers(0, 2 ** 32, size=(4, 64), dtype=np.uint64)
    k = rng.integers(0, 2 ** 32, size=(2, 64), dtype=np.uint64)
    out = philox4x32_10_np(c[0], c[1], c[2], c[3], k[0], k[1])
    for i in range(64):
        want = philox4x32_10([int(c[t, i]) for t in range(4)], [int(k[0, i]), int(k[1, i])])
        assert tuple(int(o[i]) for o in out) == want


def test_noise_code_vectorised_matches_scalar():
    g = np.arange(300) % 37
    j = np.arange(300) * 7919 + (1 << 33) * (np.arange(300) % 3)
    two = (np.arange(300) % 2) == 1
    p = np.where(two, 0.3, 0.2)
    v = noise_codes_np(g, j, 12345, p, two)
    for i in range(300):
        assert v[i] == noise_code(int(g[i]), int(j[i]), 12345, float(p[i]), bool(two[i]))


def test_noise_rates_and_uniform_paulis():
    # Statistical pin of reading R1/R8: P(error) = p, codes uniform over 3 / 15.
    n = 200_000
    j = np.arange(n, dtype=np.uint64)
    for two, ncodes in ((False, 3), (True, 15)):
        p = 0.25
        v = noise_codes_np(5, j, 7, p, two)
        rate = np.mean(v > 0)
        assert abs(rate - p) < 5 * np.sqrt(p * (1 - p) / n)
        counts = np.bincount(v[v > 0], minlength=ncodes + 1)[1:]
        assert counts.size == ncodes and np.all(counts > 0)
        exp = counts.sum() / ncodes
        chi2 = np.sum((counts - exp) ** 2 / exp)
        assert chi2 < ncodes + 6 * np.sqrt(2 * ncodes)   # loose chi^2 bound
        assert v.max() <= ncodes


def test_noise_extremes():
    assert noise_code(3, 4, 0, 0.0, False) == 0
    assert all(noise_code(g, 1, 0, 1.0, False) in (1, 2, 3) for g in range(50))
    assert all(1 <= noise_code(g, 1, 0, 1.0, True) <= 15 for g in range(50))


def test_error_threshold_rule_is_exact():
    # error iff w0 * 2^-32 < p (R8): a draw with w0 == floor(p 2^32) is an error iff
    # w0 * 2^-32 < p exactly; check the rule on a manufactured boundary.
    w0 = 4294967      # floor(1e-3 * 2^32)
    assert float(w0) * 2.0 ** -32 < 1e-3
    assert not (float(w0 + 1) * 2.0 ** -32 < 1e-3)
