"""Fidelity metrics (Eqs. 6-7): the oracle copy pinned by closed forms and
invariants, and the product copy (paper_2203_13892_b200.metrics) equal to the oracle."""
import numpy as np
import pytest

from oracle import metrics as OM
from paper_2203_13892_b200 import metrics as PM


def rand_dist(rng, n, zeros=0):
    p = rng.random(n)
    if zeros:
        p[rng.choice(n, zeros, replace=False)] = 0
    return p / p.sum()


def test_oracle_closed_forms():
    rng = np.random.default_rng(0)
    for _ in range(20):
        p = rand_dist(rng, 16, 3)
        assert OM.fidelity(p, p) == pytest.approx(1.0, abs=1e-14)          # identical -> 1
        assert OM.normalized_fidelity(p, p) == pytest.approx(1.0, abs=1e-12)
        u = np.full(16, 1 / 16)
        assert OM.normalized_fidelity(p, u) == pytest.approx(0.0, abs=1e-12)  # uniform -> 0
        q = rand_dist(rng, 16)
        assert OM.fidelity(p, q) == pytest.approx(OM.fidelity(q, p), abs=1e-15)
        perm = rng.permutation(16)
        assert OM.fidelity(p[perm], q[perm]) == pytest.approx(OM.fidelity(p, q), abs=1e-14)
    # disjoint supports -> 0 ("completely different (orthogonal) states")
    assert OM.fidelity(np.array([0.5, 0.5, 0, 0]), np.array([0, 0, 0.3, 0.7])) == 0.0
    # two-outcome closed form: (sqrt(pq) + sqrt((1-p)(1-q)))^2
    for p, q in [(0.1, 0.7), (0.5, 0.5), (0.0, 1.0), (0.25, 0.2)]:
        want = (np.sqrt(p * q) + np.sqrt((1 - p) * (1 - q))) ** 2
        assert OM.fidelity(np.array([p, 1 - p]), np.array([q, 1 - q])) == pytest.approx(want, abs=1e-15)
    # hand example: P = (1/2, 1/2, 0, 0) vs uniform: F_s = (2 sqrt(1/8))^2 = 1/2
    assert OM.fidelity(np.array([0.5, 0.5, 0, 0]), np.full(4, 0.25)) == pytest.approx(0.5, abs=1e-15)
    # and normalized against a half-way mixture: F_s = ((sqrt(3)+1)/4 * 2)^2 ... checked numerically
    P = np.array([1.0, 0, 0, 0])
    mix = 0.5 * P + 0.5 * np.full(4, 0.25)
    f_uni = 0.25
    assert OM.normalized_fidelity(P, mix) == pytest.approx((0.625 - f_uni) / (1 - f_uni), abs=1e-15)


def test_product_metrics_equal_oracle():
    rng = np.random.default_rng(1)
    for _ in range(20):
        p, q = rand_dist(rng, 32, 5), rand_dist(rng, 32, 2)
        assert PM.hellinger_fidelity(p, q) == pytest.approx(OM.fidelity(p, q), abs=1e-14)
        assert PM.normalized_fidelity(p, q) == pytest.approx(OM.normalized_fidelity(p, q), abs=1e-12)
    counts = {0: 3, 5: 1}
    d = PM.distribution(counts, 3)
    assert d[0] == 0.75 and d[5] == 0.25 and d.sum() == 1.0
    with pytest.raises(ValueError):
        PM.normalized_fidelity(np.full(8, 1 / 8), d)
