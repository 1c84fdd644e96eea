"""GPU parity of the Kraus engine (non-Pauli channels, kraus.cu; P:467-475
§4.3.2, Table 2) against oracle/kraus.py, element by element on the same keyed draws.

Bars: amplitudes of dumped node states within 1e-10; leaf outcomes bit-exact except leaves the
oracle flags (a sampling draw or a Kraus decision within 1e-9 of a boundary, R9 / R36);
histograms identical when nothing is flagged.  The noise models are Table 2's: DC, TR, AD,
PD, each with and without readout error (R), and ALL.
"""
import numpy as np
import pytest

import paper_2203_13892_b200.tqsim as T
from oracle import gates as OG
from oracle import kraus as K
from oracle.planner import Plan
from oracle.tree import NoiseModel
from workloads import basis_prep_gates, qft_gates, random_circuit

pytestmark = pytest.mark.gpu

AMP_TOL = 1e-10
TR = dict(t1=50e-6, t2=70e-6, gate_time_1q=50e-9, gate_time_2q=300e-9)   # reading R32's parameters


def table2_models(scale=1.0):
    """Table 2 noise models: (name, depolarizing p1/p2, readout, Kraus model)."""
    dc = (1e-3 * scale, 1e-2 * scale)
    ro = 1e-2 * scale
    ad, pd = 0.01 * scale, 0.01 * scale
    tr = K.KrausModel(t1=TR["t1"] / scale, t2=TR["t2"] / scale, gate_time_1q=TR["gate_time_1q"],
                      gate_time_2q=TR["gate_time_2q"])
    return {
        "TR": ((0, 0), 0.0, tr), "TRR": ((0, 0), ro, tr),
        "AD": ((0, 0), 0.0, K.KrausModel(amp_damping=ad)), "ADR": ((0, 0), ro, K.KrausModel(amp_damping=ad)),
        "PD": ((0, 0), 0.0, K.KrausModel(phase_damping=pd)), "PDR": ((0, 0), ro, K.KrausModel(phase_damping=pd)),
        "ALL": (dc, ro, K.KrausModel(amp_damping=ad, phase_damping=pd, **{k: v for k, v in
                                                                          vars(tr).items() if k.startswith(("t", "gate"))})),
    }


def noise_of(dep, ro, km):
    return T.noise_arg(dep[0], dep[1], ro, ro, km.amp_damping, km.phase_damping, km.t1, km.t2, km.gate_time_1q,
                       km.gate_time_2q)


def run_compare(n, gates, dep, ro, km, shots, arities, seed, dumps=()):
    noise = noise_of(dep, ro, km)
    res = T.tqsim_run_ex(n, gates, noise, shots, arities, seed, None, dumps)
    dbg = T.tqsim_run_ex(n, gates, noise, shots, arities, seed, None, (), leaf_debug=True)
    assert np.array_equal(res.leaf_outcomes, dbg.leaf_outcomes)
    plan = Plan(res.plan.arity_list, res.plan.boundary_list)
    nm = NoiseModel(dep[0], dep[1], ro, ro)
    ref = K.simulate_tree(n, OG.lower(gates), plan, nm, km, seed, dump=dumps)
    flagged = 0
    for l, r in ref.leaves.items():
        assert dbg.leaf_u[l] == r.u
        if r.flagged:
            flagged += 1
            continue
        assert not dbg.leaf_flagged[l], l
        assert int(res.leaf_outcomes[l]) == r.outcome, (l, int(res.leaf_outcomes[l]), r.outcome)
    if flagged == 0:
        want = {}
        for r in ref.leaves.values():
            want[r.outcome] = want.get(r.outcome, 0) + 1
        assert res.counts == want
    for i, key in enumerate(dumps):
        err = np.max(np.abs(res.dumps[i] - ref.dumps[key]))
        assert err <= AMP_TOL, (key, err)
    return res, ref


@pytest.mark.parametrize("model", ["TR", "TRR", "AD", "ADR", "PD", "PDR", "ALL"])
def test_table2_models_random_circuits(model):
    """Every Table 2 model with its rates scaled up 20x (many decisions take K1) on random
    circuits of every gate kind, tree (3, 2, 4): amplitudes, outcomes, histogram."""
    dep, ro, km = table2_models(20.0)[model]
    rng = np.random.default_rng(sum(map(ord, model)))
    for it in range(2):
        n = int(rng.integers(3, 9))
        gates = random_circuit(n, int(rng.integers(15, 40)), rng)
        run_compare(n, gates, dep, ro, km, 24, [3, 2, 4], 50 + it, dumps=[(0, 0), (1, 3), (2, 23)])


def test_qft12_all_channels_paper_rates():
    """The paper's QFT_12 study circuit (H prelude) under ALL at the paper's rates
    (AD = PD = 0.01), 200 shots on a (10, 20) tree: the full oracle tree."""
    n = 12
    gates = [("h", q, -1, 0.0, 0.0, 0.0) for q in range(n)] + qft_gates(n)
    dep, ro, km = table2_models(1.0)["ALL"]
    run_compare(n, gates, dep, ro, km, 200, [10, 20], 7, dumps=[(0, 3), (1, 150)])


def test_max_width_13_and_width_check():
    n = 13
    gates = basis_prep_gates(4321, n) + qft_gates(n)[:80]
    dep, ro, km = table2_models(5.0)["AD"]
    run_compare(n, gates, dep, ro, km, 12, [3, 4], 3, dumps=[(1, 11)])
    with pytest.raises(T.TqsimError) as e:
        T.tqsim_run(17, qft_gates(17), noise_of(dep, ro, km), 8, [8], 0)
    assert e.value.status == 2


@pytest.mark.parametrize("n", [14, 15, 16])
def test_cluster_engine_widths_14_to_16(n):
    """Widths 14..16 run in the cluster kernel (the state over 2^(n-13) CTAs' shared memory,
    gates on the top qubits through DSMEM): random circuits that touch the top qubits, every
    Table 2 channel at 20x rates, a (3, 4) tree -- dumped amplitudes, outcomes, histogram vs
    the oracle."""
    rng = np.random.default_rng(100 + n)
    gates = random_circuit(n, 40, rng)
    gates += [("cx", n - 1, 0, 0.0, 0.0, 0.0), ("h", n - 2, -1, 0.0, 0.0, 0.0), ("cz", n - 2, n - 1, 0.0, 0.0, 0.0),
              ("rx", n - 1, -1, 0.7, 0.0, 0.0), ("cx", 3, n - 1, 0.0, 0.0, 0.0)]
    dep, ro, km = table2_models(20.0)["ALL"]
    run_compare(n, gates, dep, ro, km, 12, [3, 4], 11, dumps=[(0, 1), (1, 7)])


def test_qft15_all_channels_paper_rates_cluster():
    """C2's circuit (QFT-15, BASELINE configs[1]) under ALL at the paper's rates through the
    cluster engine (4 CTAs per trajectory): 20 shots on a (4, 5) tree, the full oracle tree."""
    n = 15
    gates = [("h", q, -1, 0.0, 0.0, 0.0) for q in range(n)] + qft_gates(n)
    dep, ro, km = table2_models(1.0)["ALL"]
    run_compare(n, gates, dep, ro, km, 20, [4, 5], 5, dumps=[(0, 2), (1, 17)])


def test_vanishing_damping_equals_pauli_engine():
    """gamma = 1e-18: every Kraus decision takes K0 = diag(1, 1) (to fp64), so the Kraus engine
    must reproduce the Pauli engine's outcomes (GPU vs GPU, two independent kernels)."""
    rng = np.random.default_rng(9)
    n = 10
    gates = random_circuit(n, 60, rng)
    a = T.tqsim_run(n, gates, T.noise_arg(0.05, 0.1, 0.02, 0.02, amp_damping=1e-18), 60, [4, 15], 5)
    b = T.tqsim_run(n, gates, T.noise_arg(0.05, 0.1, 0.02, 0.02), 60, [4, 15], 5)
    assert np.array_equal(a.leaf_outcomes, b.leaf_outcomes)


def test_kraus_tree_equals_flat_and_shards():
    """Arity-1 invariant and serial shards (split below level 0) with Kraus channels."""
    torch = pytest.importorskip("torch")
    n = 8
    gates = random_circuit(n, 40, np.random.default_rng(3))
    noise = noise_of(*table2_models(10.0)["ALL"])
    flat = T.tqsim_run_ex(n, gates, noise, 30, [30], 2)
    tree = T.tqsim_run_ex(n, gates, noise, 30, [30, 1, 1], 2)
    assert np.array_equal(flat.leaf_outcomes, tree.leaf_outcomes)
    h = T.tqsim_create(n, gates, noise, 30, [5, 6])
    acc = np.zeros(30, dtype=np.int64)
    for r in range(4):
        ws = torch.empty(h.workspace_bytes(r, 4), dtype=torch.uint8, device="cuda")
        o = torch.zeros(30, dtype=torch.int32, device="cuda")
        h.execute(2, r, 4, torch.cuda.current_stream().cuda_stream, ws.data_ptr(), ws.numel(), o.data_ptr())
        acc += o.cpu().numpy()
    single = T.tqsim_run(n, gates, noise, 30, [5, 6], 2)
    assert np.array_equal(acc.astype(np.uint32), single.leaf_outcomes)
    h.close()
