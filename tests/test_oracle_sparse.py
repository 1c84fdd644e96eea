"""Pins of the sparse-state oracle against the dense oracle (no GPU)."""
import numpy as np
import pytest

from oracle import gates as OG
from oracle import sparse as SP
from oracle.planner import fixed_plan
from oracle.tree import NoiseModel, simulate_tree
from workloads import ghz_gates, hea_gates, monomial_brickwork_gates, make_variant


@pytest.mark.parametrize("n,seed", [(4, 0), (6, 1), (7, 2)])
def test_sparse_equals_dense_monomial(n, seed):
    gates = monomial_brickwork_gates(n, 6, np.random.default_rng(seed))
    low = OG.lower(gates)
    plan = fixed_plan(len(low), [3, 2, 3])
    nm = NoiseModel(0.05, 0.1, 0.02, 0.03)
    d = simulate_tree(n, low, plan, nm, seed)
    s = SP.simulate_tree(n, low, plan, nm, seed, max_terms=1)
    for l in range(plan.n_outcomes):
        assert s.leaves[l].outcome == d.leaves[l].outcome
        assert s.leaves[l].x == d.leaves[l].x


def test_sparse_equals_dense_ghz_ladder():
    n = 8
    low = OG.lower(hea_gates(n, 2, np.zeros((2, n))))
    plan = fixed_plan(len(low), [4, 3])
    nm = NoiseModel(0.02, 0.05, 0.01, 0.01)
    d = simulate_tree(n, low, plan, nm, 3, dump=[(1, j) for j in range(12)])
    s = SP.simulate_tree(n, low, plan, nm, 3, max_terms=2)
    for l in range(12):
        assert s.leaves[l].outcome == d.leaves[l].outcome


def test_sparse_states_match_dense_states():
    n = 6
    low = OG.lower(ghz_gates(n) + monomial_brickwork_gates(n, 3, np.random.default_rng(4)))
    nm = NoiseModel(0.1, 0.1)
    for j in range(5):
        st = SP.run_slice({0: 1 + 0j}, low, 0, len(low), j, 1, nm)
        from oracle.tree import run_slice
        from oracle.statevector import zero_state
        dense = run_slice(zero_state(n), n, low, 0, len(low), j, 1, nm)
        assert np.max(np.abs(SP.to_dense(st, n) - dense)) < 1e-14


def test_structured_variants_shapes():
    for name, n, G in (("c3_brick20_monomial", 20, 590), ("c4_qaoa24_beta0", 24, 288),
                       ("c5_hea28_ry0", 28, 248)):
        w = make_variant(name)
        assert w.circuit.n_qubits == n and len(OG.lower(w.circuit.gates)) == G
