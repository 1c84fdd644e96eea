"""Closed-form pins for the oracle's noise-free path (no GPU).

QFT|x> = sum_y exp(+2 pi i x y / 2^n) |y> / sqrt(2^n) (textbook; SURVEY §4 "QFT
closed form"); GHZ = (|0..0> + |1..1>)/sqrt2; "noise-free runs equal the
ideal state" (BASELINE north_star check 3).
"""
import numpy as np
import pytest

from oracle import gates as G
from oracle.planner import fixed_plan
from oracle.tree import NoiseModel, ideal_state, simulate_tree
from workloads import basis_prep_gates, ghz_gates, load_config, qft_gates


def qft_closed_form(x, n):
    y = np.arange(2 ** n)
    return np.exp(2j * np.pi * x * y / 2 ** n) / np.sqrt(2 ** n)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6])
def test_qft_basis_states(n):
    for x in range(2 ** n):
        low = G.lower(basis_prep_gates(x, n) + qft_gates(n))
        psi = ideal_state(n, low)
        assert np.max(np.abs(psi - qft_closed_form(x, n))) < 1e-13


def test_qft_config_instances():
    w = load_config("c1_qft5")
    psi = ideal_state(5, G.lower(w.circuit.gates))
    assert np.max(np.abs(psi - qft_closed_form(5, 5))) < 1e-14
    w = load_config("c2_qft15")
    assert w.meta["basis_x"] == 27873
    psi = ideal_state(15, G.lower(w.circuit.gates))
    assert np.max(np.abs(psi - qft_closed_form(27873, 15))) < 1e-12
    # uniform magnitudes (north_star closed-form check)
    assert np.allclose(np.abs(psi) ** 2, 2.0 ** -15, atol=1e-14)


@pytest.mark.parametrize("n", [2, 5, 9])
def test_ghz_two_equal_peaks(n):
    psi = ideal_state(n, G.lower(ghz_gates(n)))
    want = np.zeros(2 ** n, complex)
    want[0] = want[-1] = 2 ** -0.5
    assert np.max(np.abs(psi - want)) < 1e-15


def test_noise_free_tree_equals_ideal():
    w = load_config("c1_qft5")
    low = G.lower(w.circuit.gates)
    ideal = ideal_state(5, low)
    plan = fixed_plan(len(low), [3, 4])
    dumps = [(1, j) for j in range(12)] + [(0, j) for j in range(3)]
    res = simulate_tree(5, low, plan, NoiseModel(0.0, 0.0), 0, dump=dumps)
    for j in range(12):
        assert np.array_equal(res.dumps[(1, j)], res.dumps[(1, 0)])
        assert np.max(np.abs(res.dumps[(1, j)] - ideal)) < 1e-15
