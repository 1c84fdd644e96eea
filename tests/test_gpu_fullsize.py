"""Full-size parity at BASELINE.json's widths (20/24/28 qubits) with the plans
bench.py uses (DCP, default launch configuration).

* C3 (20q): structured monomial-gate variant -> every trajectory is 1-sparse,
  so the sparse oracle predicts ALL 10,240 leaves; plus the general-angle C3
  config with per-leaf dense recompute of sampled leaves and their states.
* C4 (24q): beta = 0 variant -> |a_x|^2 = 2^-24 for every trajectory, so each
  leaf's outcome is floor(u * 2^24) (closed form) except draws within the 1e-9
  boundary band; all 8,192 leaves checked.
* C5 (28q, 4 GiB states): RY = 0 variant -> GHZ-like 2-term trajectories; the
  shard rank 0 of 16 (8 top-level subtrees, 2,048 leaves) against the sparse
  oracle on the same shard.
"""
import numpy as np
import pytest

import paper_2203_13892_b200.tqsim as T
from oracle import gates as OG
from oracle import sparse as SP
from oracle.planner import Plan
from oracle.tree import NoiseModel, measure_uniform, simulate_leaf_flat
from workloads import load_config, make_variant

pytestmark = pytest.mark.gpu


def nm_of(w):
    return NoiseModel(w.p1, w.p2, w.readout_p01, w.readout_p10)


def test_c3_monomial_all_leaves_sparse_oracle():
    w = make_variant("c3_brick20_monomial")
    res = T.tqsim_run(*T.workload_args(w), seed=w.seed)
    plan = Plan(res.plan.arity_list, res.plan.boundary_list)
    assert plan.arities == [20] + [2] * 9
    ref = SP.simulate_tree(20, OG.lower(w.circuit.gates), plan, nm_of(w), w.seed, max_terms=1)
    bad = [l for l, r in ref.leaves.items()
           if not r.flagged and int(res.leaf_outcomes[l]) != r.outcome]
    assert not bad, bad[:10]
    assert len(ref.leaves) == 10240


def test_c4_beta0_all_leaves_closed_form():
    w = make_variant("c4_qaoa24_beta0")
    n, gates, noise, shots, ar = T.workload_args(w)
    res = T.tqsim_run_ex(n, gates, noise, shots, ar, w.seed, None, [(9, 0), (9, 8191)])
    assert res.plan.n_outcomes == 8192
    for st in res.dumps:                       # uniform magnitudes (the structural property)
        assert np.max(np.abs(np.abs(st) ** 2 - 2.0 ** -24)) < 1e-20
    skipped = 0
    for l in range(8192):
        v = measure_uniform(l, w.seed) * 2 ** 24
        frac = v - np.floor(v)
        if frac < 0.02 or frac > 0.98:        # within the 1e-9 CDF boundary band (R9)
            skipped += 1
            continue
        assert int(res.leaf_outcomes[l]) == int(np.floor(v)), l
    assert skipped < 0.06 * 8192


def test_c5_ry0_shard_sparse_oracle():
    torch = pytest.importorskip("torch")
    T.tqsim_release_run_cache()        # earlier tests' tqsim_run arena (tens of GB)
    torch.cuda.empty_cache()
    w = make_variant("c5_hea28_ry0")
    n, gates, noise, shots, ar = T.workload_args(w)
    h = T.tqsim_create(n, gates, noise, shots, ar)
    p = h.plan
    assert p.arity_list == [128] + [2] * 8
    world = 16
    t0, t1, l0, l1 = T.tqsim_shard_range(p, 0, world)
    ws = torch.empty(h.workspace_bytes(0, world), dtype=torch.uint8, device="cuda")
    out = torch.zeros(int(p.n_outcomes), dtype=torch.int32, device="cuda")
    h.execute(w.seed, 0, world, torch.cuda.current_stream().cuda_stream, ws.data_ptr(), ws.numel(),
              out.data_ptr())
    got = out.cpu().numpy()
    plan = Plan(p.arity_list, p.boundary_list)
    ref = SP.simulate_tree(n, OG.lower(gates), plan, nm_of(w), w.seed, top_range=(t0, t1),
                           max_terms=2)
    assert sorted(ref.leaves) == list(range(l0, l1))
    bad = [l for l, r in ref.leaves.items() if not r.flagged and int(got[l]) != r.outcome]
    assert not bad, bad[:10]
    assert not got[l1:].any()                  # other shards' leaves untouched
    h.close()


def test_c3_general_sampled_leaves_dense_oracle():
    w = load_config("c3_brick20")
    n, gates, noise, shots, ar = T.workload_args(w)
    L = T.tqsim_plan_circuit(n, gates, noise, shots, ar).n_levels
    leaves = [0, 10239]
    res = T.tqsim_run_ex(n, gates, noise, shots, ar, w.seed, None, [(L - 1, l) for l in leaves])
    plan = Plan(res.plan.arity_list, res.plan.boundary_list)
    low = OG.lower(gates)
    for i, l in enumerate(leaves):
        r, psi, _ = simulate_leaf_flat(n, low, plan, nm_of(w), w.seed, l, want_states=True)
        assert np.max(np.abs(res.dumps[i] - psi)) <= 1e-10
        if not r.flagged:
            assert int(res.leaf_outcomes[l]) == r.outcome


def test_c4_general_sampled_leaves_dense_oracle():
    """C4 (24 qubits, general angles) at its full plan: two leaves in different
    top-level subtrees recomputed flat by the dense oracle (amplitudes + outcomes)."""
    w = load_config("c4_qaoa24")
    n, gates, noise, shots, ar = T.workload_args(w)
    L = T.tqsim_plan_circuit(n, gates, noise, shots, ar).n_levels
    leaves = [3, 8190]
    res = T.tqsim_run_ex(n, gates, noise, shots, ar, w.seed, None, [(L - 1, l) for l in leaves])
    plan = Plan(res.plan.arity_list, res.plan.boundary_list)
    low = OG.lower(gates)
    for i, l in enumerate(leaves):
        r, psi, _ = simulate_leaf_flat(n, low, plan, nm_of(w), w.seed, l, want_states=True)
        assert np.max(np.abs(res.dumps[i] - psi)) <= 1e-10
        if not r.flagged:
            assert int(res.leaf_outcomes[l]) == r.outcome
