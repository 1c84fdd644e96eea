"""Noise-semantics pins (no GPU): trajectories vs density matrix by exact
enumeration of every error pattern, analytic channel values, and a Monte-Carlo
check of the keyed draws through the tree simulator.

BASELINE north_star check 2: "a trajectory average versus exact density-matrix
evolution with the depolarizing channel on 2-4 qubits".
"""
import itertools

import numpy as np
import pytest

from oracle import density
from oracle import gates as G
from oracle.planner import flat_plan
from oracle.statevector import apply_1q, apply_2q, zero_state
from oracle.tree import NoiseModel, simulate_tree
from workloads import random_circuit


def enumerate_trajectories(n, lowered, p1, p2):
    """rho = sum over all error patterns of weight * |psi><psi|, with psi
    built by the oracle's own statevector + Pauli application."""
    opts = []
    for g in lowered:
        two = g[0] in G.TWO_QUBIT_PRIMS
        p = p2 if two else p1
        codes = range(16) if two else range(4)
        opts.append([(c, (1 - p) if c == 0 else p / (15 if two else 3)) for c in codes])
    dim = 2 ** n
    rho = np.zeros((dim, dim), complex)
    for pattern in itertools.product(*opts):
        w = 1.0
        psi = zero_state(n)
        for (kind, a, b, th, ph, la), (code, pw) in zip(lowered, pattern):
            w *= pw
            if kind in G.TWO_QUBIT_PRIMS:
                psi = apply_2q(psi, n, a, b, G.matrix_2q(kind))
                if code:
                    psi = apply_1q(psi, n, a, G.PAULI[code >> 2])
                    psi = apply_1q(psi, n, b, G.PAULI[code & 3])
            else:
                psi = apply_1q(psi, n, a, G.matrix_1q(kind, th, ph, la))
                if code:
                    psi = apply_1q(psi, n, a, G.PAULI[code])
        if w == 0:
            continue
        rho += w * np.outer(psi, psi.conj())
    return rho


@pytest.mark.parametrize("seed,n,ng", [(0, 2, 4), (1, 3, 4), (2, 3, 5), (3, 4, 3)])
def test_trajectory_enumeration_equals_density_matrix(seed, n, ng):
    rng = np.random.default_rng(seed)
    low = G.lower(random_circuit(n, ng, rng, kinds=("h", "u", "rx", "cx", "cz", "t", "ry")))
    low = low[:5]
    p1, p2 = 0.13, 0.21
    rho_t = enumerate_trajectories(n, low, p1, p2)
    rho_d = density.evolve(n, low, p1, p2)
    assert np.max(np.abs(rho_t - rho_d)) < 1e-13
    assert abs(np.trace(rho_d) - 1) < 1e-13


def test_analytic_single_qubit_depolarizing():
    # X on |0> then depolarizing p: P(0) = 2p/3 (X and Y flip back; Z does not)
    p = 0.3
    rho = density.evolve(1, [("x", 0, -1, 0, 0, 0)], p, 0.0)
    assert abs(rho[0, 0].real - 2 * p / 3) < 1e-15
    # CX on |00> then 15-Pauli p2: P(00) = 1 - p2 + 3 p2/15 = 1 - 0.8 p2
    rho = density.evolve(2, [("cx", 0, 1, 0, 0, 0)], 0.0, p)
    assert abs(rho[0, 0].real - (1 - 0.8 * p)) < 1e-15


def test_monte_carlo_keyed_draws_match_density_matrix():
    # flat plan, many shots: empirical histogram (through Philox draws, tree
    # sampling and readout) vs the exact DM + readout distribution.
    n = 2
    low = [("h", 0, -1, 0, 0, 0), ("cx", 0, 1, 0, 0, 0), ("ry", 1, -1, 0.7, 0, 0)]
    nm = NoiseModel(0.05, 0.1, 0.02, 0.04)
    shots = 12000
    res = simulate_tree(n, low, flat_plan(len(low), shots), nm, seed=11)
    hist = np.bincount([r.outcome for r in res.leaves.values()], minlength=4) / shots
    rho = density.evolve(n, low, nm.p1, nm.p2)
    want = density.readout_distribution(np.real(np.diag(rho)), n, nm.readout_p01, nm.readout_p10)
    tvd = 0.5 * np.sum(np.abs(hist - want))
    assert tvd < 0.02


def test_readout_extremes():
    n = 3
    low = [("x", 0, -1, 0, 0, 0), ("x", 2, -1, 0, 0, 0)]       # |101> = 5
    res = simulate_tree(n, low, flat_plan(2, 50), NoiseModel(0, 0, 1.0, 1.0), 0)
    assert all(r.x == 5 and r.outcome == 0b010 for r in res.leaves.values())
    res = simulate_tree(n, low, flat_plan(2, 50), NoiseModel(0, 0, 0.0, 0.0), 0)
    assert all(r.outcome == 5 for r in res.leaves.values())
    res = simulate_tree(n, low, flat_plan(2, 50), NoiseModel(0, 0, 1.0, 0.0), 0)   # only 0->1
    assert all(r.outcome == 0b111 for r in res.leaves.values())
