"""GPU parity of the small-state tree kernel (csrc/small.cu; SURVEY §8(a)
kernel notes "n <= 10 takes the small_state_tree path") against the oracle.

The kernel recomputes each leaf's root-to-leaf path with the inherited keys, so its outcomes
must equal the oracle's tree DFS (oracle.tree.simulate_tree; the oracle's own pin
"per-leaf flat recompute == DFS" is tests/test_oracle_tree.py) for every leaf the oracle does
not flag (R9's 1e-9 band), its u53 must equal the oracle's bit for bit, and it must agree with
the general tree engine (options.small_tree = 2) on the same inputs.
"""
import numpy as np
import pytest

import paper_2203_13892_b200.tqsim as T
from oracle import gates as OG
from oracle.planner import Plan
from oracle.tree import NoiseModel, simulate_tree
from workloads import ghz_gates, load_config, qft_gates, random_circuit

pytestmark = pytest.mark.gpu

SMALL_ON = 1
SMALL_OFF = 2


def run(n, gates, nm, shots, arities, seed, small, **kw):
    noise = T.noise_arg(nm.p1, nm.p2, nm.readout_p01, nm.readout_p10)
    opts = T.default_options(small_tree=small, **kw)
    return T.tqsim_run_ex(n, gates, noise, shots, arities, seed, opts, leaf_debug=True)


def check_vs_oracle(n, gates, nm, shots, arities, seed, **kw):
    res = run(n, gates, nm, shots, arities, seed, SMALL_ON, **kw)
    assert res.plan.small_tree == 1
    plan = Plan(res.plan.arity_list, res.plan.boundary_list)
    ref = simulate_tree(n, OG.lower(gates), plan, nm, seed)
    assert res.leaf_outcomes.shape[0] == plan.n_outcomes
    flagged = 0
    for l, r in ref.leaves.items():
        assert res.leaf_u[l] == r.u, l                      # same keyed u53 (R7, R9)
        if r.flagged:
            flagged += 1
            continue
        assert int(res.leaf_outcomes[l]) == r.outcome, (l, int(res.leaf_outcomes[l]), r.outcome)
        assert not res.leaf_flagged[l], l
    if flagged == 0:
        want = {}
        for r in ref.leaves.values():
            want[r.outcome] = want.get(r.outcome, 0) + 1
        assert res.counts == want
    # the general engine on the same inputs: identical outcomes outside the flagged band
    gen = run(n, gates, nm, shots, arities, seed, SMALL_OFF, **kw)
    assert gen.plan.small_tree == 0
    for l, r in ref.leaves.items():
        if not r.flagged:
            assert int(gen.leaf_outcomes[l]) == int(res.leaf_outcomes[l]), l
    return res, ref


def test_c1_qft5_small_tree_full():
    w = load_config("c1_qft5")
    nm = NoiseModel(w.p1, w.p2, w.readout_p01, w.readout_p10)
    res, _ = check_vs_oracle(5, w.circuit.gates, nm, w.shots, w.arities, w.seed)
    assert res.plan.n_outcomes == 1000
    assert res.stats.kernel_launches == 2          # the seed kernel + the whole tree
    assert res.stats.pass_launches == 1


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 7, 8, 9, 10])
def test_random_circuits_every_width(n):
    """Every width up to the limit (n < 5 runs padded to 5 qubits, R28), heavy noise (every Pauli
    code, readout flips on every bit), three-level ragged trees."""
    rng = np.random.default_rng(700 + n)
    gates = random_circuit(n, int(rng.integers(30, 90)), rng)
    if not gates:
        pytest.skip("no gates")
    check_vs_oracle(n, gates, NoiseModel(0.08, 0.15, 0.03, 0.05), 60, [3, 4, 5], 11 + n)


@pytest.mark.parametrize("p", [0.0, 1.0])
def test_noise_extremes(p):
    """p = 0 (noise-free: one outcome distribution for every leaf) and p = 1 (every gate errs)."""
    rng = np.random.default_rng(71)
    n = 8
    gates = random_circuit(n, 70, rng)
    check_vs_oracle(n, gates, NoiseModel(p, p, 0.0, 0.0), 40, [4, 10], 5)


def test_structured_circuits():
    """GHZ (two-peak distribution: the CDF has flat runs) and QFT on a basis state."""
    check_vs_oracle(9, ghz_gates(9), NoiseModel(0.01, 0.02, 0.01, 0.01), 200, [10, 20], 3)
    check_vs_oracle(7, qft_gates(7), NoiseModel(0.02, 0.05, 0.0, 0.0), 150, [5, 5, 6], 4)


def test_flat_and_long_slices():
    """Arity-1 / flat plans and slices longer than 32 gates (codes drawn 32 at a time)."""
    rng = np.random.default_rng(72)
    n = 6
    gates = random_circuit(n, 140, rng)
    check_vs_oracle(n, gates, NoiseModel(0.03, 0.06, 0.02, 0.02), 50, [50], 6)
    check_vs_oracle(n, gates, NoiseModel(0.03, 0.06, 0.02, 0.02), 48, [1, 6, 1, 8], 7)


def test_auto_choice_and_limits(monkeypatch):
    """Auto (options.small_tree = 0) picks the kernel for C1; never above 10 qubits, never for the
    Kraus engine; state dumps run the general tree on a small handle (and agree with it)."""
    monkeypatch.delenv("TQSIM_SMALL", raising=False)
    w = load_config("c1_qft5")
    n, gates, noise, shots, ar = T.workload_args(w)
    a = T.tqsim_run_ex(n, gates, noise, shots, ar, w.seed, T.default_options())
    assert a.plan.small_tree == 1
    rng = np.random.default_rng(73)
    g11 = random_circuit(11, 40, rng)
    big = T.tqsim_run_ex(11, g11, noise, 20, [4, 5], 1, T.default_options(small_tree=SMALL_ON))
    assert big.plan.small_tree == 0
    kn = T.noise_arg(0.01, 0.02, 0.0, 0.0)
    kn.amp_damping = 0.01
    kr = T.tqsim_run_ex(6, random_circuit(6, 30, rng), kn, 20, [4, 5], 1, T.default_options(small_tree=SMALL_ON))
    assert kr.plan.small_tree == 0
    d = T.tqsim_run_ex(n, gates, noise, shots, ar, w.seed, T.default_options(small_tree=SMALL_ON),
                       dumps=[(1, 3)])
    assert d.stats.pass_launches > 1                # the general engine ran (stored-state path)
    ref = simulate_tree(n, OG.lower(gates), Plan(d.plan.arity_list, d.plan.boundary_list),
                        NoiseModel(w.p1, w.p2, w.readout_p01, w.readout_p10), w.seed)
    for l, r in ref.leaves.items():
        if not r.flagged:
            assert int(d.leaf_outcomes[l]) == r.outcome == int(a.leaf_outcomes[l])


@pytest.mark.parametrize("world", [2, 3, 7])
def test_serial_shards_equal_single_run(world):
    """tqsim_execute shards (split-level ranges) of a small-tree handle add up to
    the single run."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(74)
    n = 7
    gates = random_circuit(n, 50, rng)
    noise = T.noise_arg(0.05, 0.1, 0.02, 0.02)
    ar = [5, 4, 3]
    shots = int(np.prod(ar))
    opts = T.default_options(small_tree=SMALL_ON)
    h = T.tqsim_create(n, gates, noise, shots, ar, opts)
    assert h.plan.small_tree == 1
    single = T.tqsim_run_ex(n, gates, noise, shots, ar, 9, opts).leaf_outcomes
    acc = np.zeros(shots, dtype=np.int64)
    for r in range(world):
        ws = torch.empty(max(1, h.workspace_bytes(r, world)), dtype=torch.uint8, device="cuda")
        o = torch.zeros(shots, dtype=torch.int32, device="cuda")
        h.execute(9, r, world, torch.cuda.current_stream().cuda_stream, ws.data_ptr(), ws.numel(), o.data_ptr())
        acc += o.cpu().numpy()
    assert np.array_equal(acc.astype(np.uint32), single)
    h.close()
