"""Pins of oracle/kraus.py (non-Pauli channels as trajectories, R31-R37; P:467-475
§4.3.2, Table 2) against what the mathematics fixes: Kraus completeness, the density-matrix
channel by exact branch enumeration, closed forms for T1/T2 relaxation and single-qubit
damping, the choice rule on states whose branch probabilities are known, the trajectory
ensemble vs the channel (Monte Carlo), tree reuse, and the reduction to the Pauli oracle."""
import math

import numpy as np
import pytest

from oracle import gates as OG
from oracle import kraus as K
from oracle.planner import fixed_plan
from oracle.statevector import apply_1q, zero_state
from oracle.tree import NoiseModel, simulate_tree as pauli_tree
from workloads import random_circuit, qft_gates

NM0 = NoiseModel(0.0, 0.0)


def test_kraus_sets_are_complete():
    for ops in (K.ad_ops(0.01), K.ad_ops(0.37), K.pd_ops(0.01), K.pd_ops(0.8)):
        s = sum(k.conj().T @ k for k in ops)
        assert np.max(np.abs(s - np.eye(2))) < 1e-15
    km = K.KrausModel(t1=50e-6, t2=70e-6, gate_time_1q=50e-9, gate_time_2q=300e-9)
    g, l = K.tr_params(km, True)
    assert abs(g - (1 - math.exp(-300e-9 / 50e-6))) < 1e-18 and 0 < l < g


KM_CASES = [K.KrausModel(amp_damping=0.2, phase_damping=0.3),
            K.KrausModel(t1=10e-6, t2=15e-6, gate_time_1q=1e-6, gate_time_2q=2e-6),
            K.KrausModel(amp_damping=0.1, phase_damping=0.05, t1=10e-6, t2=15e-6, gate_time_1q=1e-6,
                         gate_time_2q=2e-6)]


@pytest.mark.parametrize("case", [0, 1, 2])
def test_dm_channel_equals_branch_enumeration(case):
    """rho -> sum_k K_k rho K_k^dag on the full-space operators (evolve_dm) equals the sum
    over every sequence of Kraus choices applied to the statevector (enumerate_branches)."""
    rng = np.random.default_rng(case)
    n = 2
    gates = [("u", 0, -1, *rng.uniform(0, 6.28, 3)), ("cx", 0, 1, 0, 0, 0),
             ("ry", 1, -1, float(rng.uniform(0, 6.28)), 0, 0)]
    if case < 2:
        gates.append(("h", 1, -1, 0, 0, 0))
    low = OG.lower(gates)
    km = KM_CASES[case]
    a = K.evolve_dm(n, low, 0.0, 0.0, km)
    b = K.enumerate_branches(n, low, km)
    assert np.max(np.abs(a - b)) < 1e-13
    assert abs(np.trace(a).real - 1.0) < 1e-13


def test_thermal_relaxation_closed_forms():
    """TR (R32): after k identity-like gates of duration t, P(1) of |1> = exp(-k t / T1)
    (populations) and |rho_01| of |+> = exp(-k t / T2) / 2 (coherences)."""
    t1, t2, t = 20e-6, 30e-6, 1e-6
    km = K.KrausModel(t1=t1, t2=t2, gate_time_1q=t, gate_time_2q=t)
    k = 7
    ident = [("u", 0, -1, 0.0, 0.0, 0.0)] * k
    rho = K.evolve_dm(1, OG.lower([("x", 0, -1, 0, 0, 0)] + ident), 0.0, 0.0, km)
    # the X itself is a location too: k + 1 relaxations of |1>
    assert abs(rho[1, 1].real - math.exp(-(k + 1) * t / t1)) < 1e-14
    rho = K.evolve_dm(1, OG.lower([("h", 0, -1, 0, 0, 0)] + ident), 0.0, 0.0, km)
    assert abs(abs(rho[0, 1]) - 0.5 * math.exp(-(k + 1) * t / t2)) < 1e-14


def test_single_qubit_damping_closed_forms():
    g, l = 0.01, 0.01
    rho = K.evolve_dm(1, OG.lower([("x", 0, -1, 0, 0, 0)]), 0.0, 0.0, K.KrausModel(amp_damping=g))
    assert abs(rho[1, 1].real - (1 - g)) < 1e-15 and abs(rho[0, 0].real - g) < 1e-15
    rho = K.evolve_dm(1, OG.lower([("h", 0, -1, 0, 0, 0)]), 0.0, 0.0, K.KrausModel(phase_damping=l))
    assert abs(rho[0, 1].real - 0.5 * math.sqrt(1 - l)) < 1e-15 and abs(rho[1, 1].real - 0.5) < 1e-15


def test_choice_rule_on_known_branch_probabilities():
    """|1> under AD(g): p_0 = 1-g, p_1 = g, so K1 (decay to |0>) iff r >= 1-g (R35);
    |0> never decays; |1> under PD(l): K1 iff r >= 1-l, the state stays |1>."""
    g = 0.3
    one = apply_1q(zero_state(1), 1, 0, OG.PAULI[1])
    hits = 0
    for j in range(400):
        r = K.kraus_uniform(5, j, 4, 11)
        psi, k, f = K.choose(one, 1, 0, K.ad_ops(g), r)
        assert k == (1 if r >= 1 - g else 0)
        assert np.allclose(psi, [1, 0] if k else [0, 1], atol=1e-15)
        hits += k
        psi, k, _ = K.choose(zero_state(1), 1, 0, K.ad_ops(g), r)
        assert k == 0
        psi, k, _ = K.choose(one, 1, 0, K.pd_ops(g), r)
        assert k == (1 if r >= 1 - g else 0) and np.allclose(psi, [0, 1], atol=1e-15)
    assert 0.2 * 400 < hits < 0.4 * 400


def test_kraus_uniform_is_the_keyed_philox_word():
    from oracle.philox import philox4x32_10, seed_key
    for s in range(8):
        w = philox4x32_10((17, 9, 3 + (s >> 2), 0), seed_key(5))[s & 3]
        assert K.kraus_uniform(17, 9, s, 5) == w * 2.0 ** -32


def test_trajectory_ensemble_matches_channel():
    """Monte Carlo: the average of |psi><psi| over independent keyed trajectories converges
    to the density-matrix channel (the unravelling is unbiased)."""
    n = 2
    low = OG.lower([("h", 0, -1, 0, 0, 0), ("cx", 0, 1, 0, 0, 0), ("ry", 1, -1, 0.7, 0, 0),
                    ("x", 0, -1, 0, 0, 0)])
    km = K.KrausModel(amp_damping=0.25, phase_damping=0.2, t1=5e-6, t2=7e-6, gate_time_1q=1e-6,
                      gate_time_2q=2e-6)
    nm = NoiseModel(0.1, 0.2)
    want = K.evolve_dm(n, low, nm.p1, nm.p2, km)
    M = 3000
    acc = np.zeros((4, 4), dtype=np.complex128)
    for j in range(M):
        psi, _ = K.run_slice(zero_state(n), n, low, 0, len(low), j, 3, nm, km)
        acc += np.outer(psi, psi.conj())
    acc /= M
    assert np.max(np.abs(acc - want)) < 3.0 / math.sqrt(M)      # ~6 sigma of an entry


def test_tree_dfs_equals_per_leaf_flat_and_norms():
    rng = np.random.default_rng(4)
    n = 4
    low = OG.lower(random_circuit(n, 24, rng))
    km = K.KrausModel(amp_damping=0.05, phase_damping=0.05, t1=10e-6, t2=12e-6, gate_time_1q=0.2e-6,
                      gate_time_2q=0.5e-6)
    nm = NoiseModel(0.02, 0.05, 0.01, 0.02)
    plan = fixed_plan(len(low), [3, 2, 2])
    tree = K.simulate_tree(n, low, plan, nm, km, 8, dump=[(2, 5)])
    for leaf in range(12):
        r, psi = K.simulate_leaf_flat(n, low, plan, nm, km, 8, leaf)
        assert r == tree.leaves[leaf]
        assert abs(np.vdot(psi, psi).real - 1.0) < 1e-12
        if leaf == 5:
            assert np.array_equal(psi, tree.dumps[(2, 5)])


def test_no_kraus_reduces_to_pauli_oracle():
    n = 5
    low = OG.lower(qft_gates(n))
    nm = NoiseModel(0.05, 0.1, 0.02, 0.02)
    plan = fixed_plan(len(low), [4, 5])
    a = K.simulate_tree(n, low, plan, nm, K.KrausModel(), 3)
    b = pauli_tree(n, low, plan, nm, 3)
    assert a.leaves == b.leaves
