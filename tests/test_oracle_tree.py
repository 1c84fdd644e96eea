"""Tree-reuse invariants and sampling pins for the oracle (no GPU).

BASELINE north_star check 4: "a tree with arity 1 at every level equals the
flat per-shot baseline"; reuse is exact: DFS == per-leaf flat recompute with
inherited keys; sampling == brute-force linear scan (smallest x with C(x) > t).
"""
import numpy as np
import pytest

from oracle import gates as G
from oracle.planner import Plan, fixed_plan, flat_plan, split_equal
from oracle.tree import (NoiseModel, leaf_ancestors, measure_uniform, sample_leaf,
                         simulate_leaf_flat, simulate_tree)
from workloads import load_config, random_circuit


def _c1():
    w = load_config("c1_qft5")
    return w, G.lower(w.circuit.gates), NoiseModel(w.p1, w.p2, w.readout_p01, w.readout_p10)


def test_arity_one_tree_equals_flat():
    w, low, nm = _c1()
    N = 60
    flat = simulate_tree(5, low, flat_plan(len(low), N), nm, 3)
    for b in ([0, 20, 63], [0, 5, 40, 50, 63], [0, 62, 63]):
        L = len(b) - 1
        plan = Plan([N] + [1] * (L - 1), b)
        tree = simulate_tree(5, low, plan, nm, 3)
        for l in range(N):
            assert tree.leaves[l].outcome == flat.leaves[l].outcome
            assert tree.leaves[l].x == flat.leaves[l].x


def test_dfs_equals_per_leaf_recompute():
    w, low, nm = _c1()
    nm = NoiseModel(0.05, 0.1, 0.02, 0.02)       # many errors
    plan = fixed_plan(len(low), [3, 2, 4])
    dumps = [(d, j) for d in range(3) for j in range(plan.instances()[d])]
    tree = simulate_tree(5, low, plan, nm, 9, dump=dumps)
    for leaf in range(plan.n_outcomes):
        r, psi, states = simulate_leaf_flat(5, low, plan, nm, 9, leaf, want_states=True)
        assert r.outcome == tree.leaves[leaf].outcome
        for key, st in states.items():
            assert np.array_equal(st, tree.dumps[key])


def test_leaf_ancestors():
    plan = fixed_plan(30, [3, 2, 4])
    for leaf in range(24):
        anc = leaf_ancestors(plan, leaf)
        assert anc[-1] == leaf
        assert anc[1] == leaf // 4 and anc[0] == leaf // 8


def test_shards_partition_the_tree():
    w, low, nm = _c1()
    plan = fixed_plan(len(low), [4, 5])
    full = simulate_tree(5, low, plan, nm, 1)
    parts = {}
    for lo, hi in ((0, 1), (1, 3), (3, 4)):
        parts.update(simulate_tree(5, low, plan, nm, 1, top_range=(lo, hi)).leaves)
    assert sorted(parts) == list(range(20))
    assert all(parts[l].outcome == full.leaves[l].outcome for l in range(20))


def test_sampling_matches_linear_scan():
    rng = np.random.default_rng(5)
    n = 6
    nm = NoiseModel(0, 0)
    for leaf in range(200):
        psi = rng.normal(size=64) + 1j * rng.normal(size=64)
        if leaf % 3 == 0:
            psi[rng.integers(0, 64, 20)] = 0              # zero-probability entries
        r = sample_leaf(psi, n, leaf, 4, nm)
        p = np.abs(psi) ** 2
        t = measure_uniform(leaf, 4) * np.sum(np.cumsum(p)[-1])
        acc, x = 0.0, None
        for i in range(64):
            acc += p[i]
            if acc > t:
                x = i
                break
        assert r.x == x and p[r.x] > 0


def test_uniform_magnitude_sampling_closed_form():
    n = 10
    psi = np.exp(1j * np.arange(2 ** n)) / 2 ** (n / 2)
    for leaf in range(300):
        r = sample_leaf(psi, n, leaf, 2, NoiseModel(0, 0))
        u = measure_uniform(leaf, 2)
        if not r.flagged:
            assert r.x == int(np.floor(u * 2 ** n))


def test_u53_range_and_determinism():
    us = [measure_uniform(l, 0) for l in range(2000)]
    assert all(0.0 <= u < 1.0 for u in us)
    assert abs(np.mean(us) - 0.5) < 0.03
    w, low, nm = _c1()
    a = simulate_tree(5, low, fixed_plan(len(low), [2, 3]), nm, 77)
    b = simulate_tree(5, low, fixed_plan(len(low), [2, 3]), nm, 77)
    assert [a.leaves[i].outcome for i in range(6)] == [b.leaves[i].outcome for i in range(6)]


def test_u53_is_uniform_on_the_2pow53_lattice():
    """R9's u = ((w0 >> 5) 2^26 + (w1 >> 6)) 2^-53: every value is a multiple of 2^-53 in
    [0, 1); its top 27 bits are w0's top 27 bits (u >= 1/2 iff w0's top bit is set, floor(u
    2^27) == w0 >> 5), the next 26 are w1's top 26; the values pass a Kolmogorov-Smirnov test
    for U[0, 1) (scipy.stats.kstest, 20,000 leaves)."""
    from scipy import stats
    from oracle.philox import philox4x32_10, seed_key
    us = np.array([measure_uniform(l, 11) for l in range(20000)])
    assert np.all((us >= 0) & (us < 1))
    assert np.all(np.floor(us * 2.0 ** 53) == us * 2.0 ** 53)
    for l in range(0, 20000, 997):
        w0, w1, _, _ = philox4x32_10((0, l, 1, 0), seed_key(11))
        assert int(np.floor(us[l] * 2.0 ** 27)) == w0 >> 5
        assert int(us[l] * 2.0 ** 53) & ((1 << 26) - 1) == w1 >> 6
    assert stats.kstest(us, "uniform").pvalue > 1e-4


def test_readout_word_selection_and_rates():
    """R11: bit b of leaf l flips iff word (b & 3) of Philox(ctr = (b >> 2, l, 2, 0)) * 2^-32 is
    below p10 (bit set) / p01 (bit clear).  With p01 = p10 = p the flip of bit b equals that
    word's threshold test (checked against the words directly for 5-qubit outcomes, both
    values of every bit), and the per-bit flip rates over 20,000 leaves are p within 5 sigma."""
    from oracle.philox import philox4x32_10, seed_key
    from oracle.tree import readout_mask
    p = 0.2
    n = 6
    flips = np.zeros(n)
    L = 20000
    for l in range(L):
        m0 = readout_mask(0, n, l, 4, p, p)
        m1 = readout_mask((1 << n) - 1, n, l, 4, p, p)
        assert m0 == m1                     # symmetric p: the flips do not depend on x
        if l < 200:
            for b in range(n):
                w = philox4x32_10((b >> 2, l, 2, 0), seed_key(4))[b & 3]
                assert ((m0 >> b) & 1) == (w * 2.0 ** -32 < p)
        flips += [(m0 >> b) & 1 for b in range(n)]
    rate = flips / L
    assert np.all(np.abs(rate - p) < 5 * np.sqrt(p * (1 - p) / L))
    # asymmetric: a set bit uses p10, a clear bit p01
    assert readout_mask(0, n, 3, 4, 1.0, 0.0) == (1 << n) - 1
    assert readout_mask((1 << n) - 1, n, 3, 4, 1.0, 0.0) == 0
