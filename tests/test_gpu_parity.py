"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by element.

Bars (BASELINE north_star): per-trajectory amplitudes max-abs <= 1e-10 (fp64);
sampled outcomes bit-exact except draws the oracle flags as lying within 1e-9
of a cumulative-probability boundary; histograms identical otherwise.
"""
import numpy as np
import pytest

import paper_2203_13892_b200.tqsim as T
from oracle import gates as OG
from oracle.noise import noise_codes_np
from oracle.philox import philox4x32_10
from oracle.planner import Plan, fixed_plan, dcp_plan
from oracle.tree import (NoiseModel, error_rates, ideal_state, leaf_ancestors,
                         simulate_leaf_flat, simulate_tree)
from tq_testutil import golden_rows
from workloads import basis_prep_gates, ghz_gates, load_config, qft_gates, random_circuit

pytestmark = pytest.mark.gpu

AMP_TOL = 1e-10


def oracle_plan_of(res_plan) -> Plan:
    return Plan(res_plan.arity_list, res_plan.boundary_list)


def assert_leaves_match(gpu_leaf, oracle_leaves, allow_flag=True):
    flagged = 0
    for l, r in oracle_leaves.items():
        if r.flagged and allow_flag:
            flagged += 1
            continue
        assert int(gpu_leaf[l]) == r.outcome, (l, int(gpu_leaf[l]), r.outcome, r.x)
    return flagged


def run_and_compare(n, gates, nm: NoiseModel, shots, arities, seed, opts=None, dumps=()):
    noise = T.noise_arg(nm.p1, nm.p2, nm.readout_p01, nm.readout_p10)
    res = T.tqsim_run_ex(n, gates, noise, shots, arities, seed, opts, dumps)
    plan = oracle_plan_of(res.plan)
    low = OG.lower(gates)
    ref = simulate_tree(n, low, plan, nm, seed, dump=dumps)
    assert res.leaf_outcomes.shape[0] == plan.n_outcomes
    flagged = assert_leaves_match(res.leaf_outcomes, ref.leaves)
    if flagged == 0:
        want = {}
        for r in ref.leaves.values():
            want[r.outcome] = want.get(r.outcome, 0) + 1
        assert res.counts == want
    for i, key in enumerate(dumps):
        err = np.max(np.abs(res.dumps[i] - ref.dumps[key]))
        assert err <= AMP_TOL, (key, err)
    return res, ref


def test_device_philox_known_answers_and_oracle():
    rows = golden_rows("philox_kat.txt")
    words = np.array([[int(v, 16) for v in r[:6]] for r in rows], dtype=np.uint32)
    out = T.tqsim_debug_philox(words)
    for r, o in zip(rows, out):
        assert tuple(int(v) for v in o) == tuple(int(v, 16) for v in r[6:10])
    rng = np.random.default_rng(0)
    words = rng.integers(0, 2 ** 32, size=(500, 6), dtype=np.uint64).astype(np.uint32)
    out = T.tqsim_debug_philox(words)
    for w, o in zip(words, out):
        assert tuple(int(v) for v in o) == philox4x32_10(w[:4], w[4:6])


def test_noise_tables_match_oracle():
    w = load_config("c2_qft15")
    n, gates, noise, shots, ar = T.workload_args(w)
    h = T.tqsim_create(n, gates, noise, shots, ar)
    p = h.plan
    low = OG.lower(gates)
    for level in (0, p.n_levels - 1):
        b0, b1 = p.boundaries[level], p.boundaries[level + 1]
        count = 300
        got = h.noise_table(5, level, 17, count)
        g = np.arange(b0, b1)[None, :]
        j = np.arange(17, 17 + count)[:, None]
        two = np.array([OG.is_two_qubit(low[i]) for i in range(b0, b1)])[None, :]
        want = noise_codes_np(g, j, 5, np.where(two, w.p2, w.p1), two)
        assert np.array_equal(got, want)
    h.close()


def test_c1_qft5_full_tree():
    w = load_config("c1_qft5")
    nm = NoiseModel(w.p1, w.p2, w.readout_p01, w.readout_p10)
    dumps = [(0, j) for j in range(10)] + [(1, j) for j in (0, 1, 99, 500, 999)]
    res, ref = run_and_compare(5, w.circuit.gates, nm, w.shots, w.arities, w.seed, dumps=dumps)
    assert res.plan.n_outcomes == 1000


@pytest.mark.parametrize("tile", [0, 4, 7, 9, 10, 12, 13])
def test_random_circuits_all_tiles(tile):
    rng = np.random.default_rng(100 + tile)
    for it in range(3):
        n = int(rng.integers(4, 15))
        gates = random_circuit(n, int(rng.integers(20, 80)), rng)
        nm = NoiseModel(0.05, 0.1, 0.02, 0.03)          # many errors: every Pauli path
        arities = [3, 2, 4] if it % 2 == 0 else None
        shots = 24 if arities else 40
        opts = T.default_options(tile_qubits=tile, batch_log2_amps=n + 2)  # ragged batches
        dumps = [(0, 0), (0, 2)]
        run_and_compare(n, gates, nm, shots, arities, 1234 + it, opts, dumps)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_tiny_widths(n):
    rng = np.random.default_rng(n)
    gates = random_circuit(n, 30, rng)
    if not gates:
        pytest.skip("no gates")
    run_and_compare(n, gates, NoiseModel(0.1, 0.2, 0.05, 0.05), 30, [5, 6], 3,
                    dumps=[(1, 0), (1, 29)])


def test_qft_noise_free_equals_closed_form():
    n = 13
    x = 4321
    gates = basis_prep_gates(x, n) + qft_gates(n)
    res = T.tqsim_run_ex(n, gates, T.noise_arg(0, 0), 8, [2, 4], 0, None, [(1, 0), (1, 7)])
    y = np.arange(2 ** n)
    want = np.exp(2j * np.pi * x * y / 2 ** n) / np.sqrt(2 ** n)
    for i in range(2):
        assert np.max(np.abs(res.dumps[i] - want)) < 1e-12


def test_ghz_two_peaks_and_outcomes():
    n = 16
    res = T.tqsim_run_ex(n, ghz_gates(n), T.noise_arg(0, 0), 2000, [2000], 0, None, [(0, 5)])
    st = res.dumps[0]
    assert abs(st[0] - 2 ** -0.5) < 1e-15 and abs(st[-1] - 2 ** -0.5) < 1e-15
    assert set(res.counts) == {0, 2 ** n - 1}
    assert abs(res.counts[0] - 1000) < 5 * np.sqrt(500)


def test_arity_one_tree_equals_flat_on_gpu():
    w = load_config("c1_qft5")
    noise = T.noise_arg(0.02, 0.05, 0.01, 0.01)
    flat = T.tqsim_run_ex(5, w.circuit.gates, noise, 300, [300], 9)
    tree = T.tqsim_run_ex(5, w.circuit.gates, noise, 300, [300, 1, 1, 1], 9)
    assert np.array_equal(flat.leaf_outcomes, tree.leaf_outcomes)


def test_c2_qft15_full_config_leaf_subset():
    w = load_config("c2_qft15")
    n, gates, noise, shots, ar = T.workload_args(w)
    nm = NoiseModel(w.p1, w.p2, w.readout_p01, w.readout_p10)
    plan0 = T.tqsim_plan_circuit(n, gates, noise, shots, ar)
    L = plan0.n_levels
    leaves = [0, 1, 777, 5119, 5120, 10239] + list(np.random.default_rng(0).integers(0, 10240, 6))
    dumps = [(L - 1, int(l)) for l in leaves[:4]]
    res = T.tqsim_run_ex(n, gates, noise, shots, ar, w.seed, None, dumps)
    plan = oracle_plan_of(res.plan)
    assert plan.arities == [20] + [2] * 9
    low = OG.lower(gates)
    for i, l in enumerate(leaves):
        r, psi, _ = simulate_leaf_flat(n, low, plan, nm, w.seed, int(l), want_states=True)
        if not r.flagged:
            assert int(res.leaf_outcomes[l]) == r.outcome
        if i < len(dumps):
            assert np.max(np.abs(res.dumps[i] - psi)) <= AMP_TOL
    assert sum(res.counts.values()) == 10240


def test_serial_shards_equal_single_run():
    torch = pytest.importorskip("torch")
    w = load_config("c1_qft5")
    n, gates, noise, shots, ar = T.workload_args(w)
    h = T.tqsim_create(n, gates, noise, shots, ar)
    N = h.plan.n_outcomes
    outs = []
    for world in (1, 2, 3, 4):
        acc = torch.zeros(N, dtype=torch.int64, device="cuda")
        for r in range(world):
            ws = torch.empty(h.workspace_bytes(r, world), dtype=torch.uint8, device="cuda")
            o = torch.zeros(N, dtype=torch.int32, device="cuda")
            h.execute(7, r, world, torch.cuda.current_stream().cuda_stream, ws.data_ptr(),
                      ws.numel(), o.data_ptr())
            acc += o.to(torch.int64)
        outs.append(acc.cpu().numpy())
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    h.close()


def test_device_philox_matches_curand():
    import ctypes as C
    import os
    from tq_testutil import ROOT
    so = os.path.join(ROOT, "tests", "_curand_ref.so")
    ref = C.CDLL(so)
    rng = np.random.default_rng(42)
    words = rng.integers(0, 2 ** 32, size=(4096, 6), dtype=np.uint64).astype(np.uint32)
    want = np.zeros((4096, 4), dtype=np.uint32)
    assert ref.curand_philox_ref(words.ctypes.data_as(C.c_void_p), C.c_uint64(4096),
                                 want.ctypes.data_as(C.c_void_p)) == 0
    assert np.array_equal(T.tqsim_debug_philox(words), want)


def _structured_circuit(n, rng):
    """QFT (lowered CP runs) + RZZ (CX.RZ.CX runs) + SWAPs + a general layer: every
    fused-run kind of the fast path, so errors land inside diagonal runs (generic
    propagated diagonals), inside SWAP relabelings and on single gates."""
    from workloads.generators import g1, g2, random_3_regular_edges
    gates = basis_prep_gates(int(rng.integers(0, 2 ** n)), n) + qft_gates(n)
    edges = random_3_regular_edges(n, rng) if n % 2 == 0 else [(q, (q + 3) % n) for q in range(n)]
    for (u, v) in edges:
        gates += [g2("cx", u, v), g1("rz", v, float(rng.uniform(0, 6.28))), g2("cx", u, v)]
    for q in range(n):
        gates.append(g1("u", q, *[float(a) for a in rng.uniform(0, 6.28, 3)]))
    for q in range(0, n - 1, 2):
        gates.append(g2("swap", q, n - 1 - q))
    gates.append(g2("cp", 0, n - 1, 0.7))
    return gates


@pytest.mark.parametrize("tile,p", [(0, 0.05), (7, 0.3), (9, 0.1), (12, 0.3), (10, 1.0)])
def test_error_frame_structured(tile, p):
    """The careful path (fused ops under a run-time Pauli frame) vs the oracle with many
    errors per pass, including p = 1 (every gate draws a Pauli)."""
    rng = np.random.default_rng(int(p * 1000) + tile)
    n = 12
    gates = _structured_circuit(n, rng)
    nm = NoiseModel(p, min(1.0, 2 * p), 0.02, 0.03)
    opts = T.default_options(tile_qubits=tile, batch_log2_amps=n + 2)
    run_and_compare(n, gates, nm, 24, [3, 2, 4], 77 + tile, opts,
                    dumps=[(0, 0), (0, 2), (1, 5), (2, 23)])


def test_run_plan_cache_reuse():
    """tqsim_run reuses its prepared plan for byte-identical inputs: results are the
    same as a fresh preparation (run_ex with explicit default options = another key)."""
    w = load_config("c1_qft5")
    n, gates, noise, shots, ar = T.workload_args(w)
    ca = T.CircuitArg(n, gates)
    a = T.tqsim_run(n, ca, noise, shots, ar, 5)
    b = T.tqsim_run(n, ca, noise, shots, ar, 5)
    c = T.tqsim_run(n, ca, noise, shots, ar, 6)
    fresh = T.tqsim_run_ex(n, gates, noise, shots, ar, 6, T.default_options())
    assert np.array_equal(a.leaf_outcomes, b.leaf_outcomes)
    assert np.array_equal(c.leaf_outcomes, fresh.leaf_outcomes)
    assert not np.array_equal(a.leaf_outcomes, c.leaf_outcomes)
    other = T.tqsim_run(n, ca, T.noise_arg(0, 0), shots, ar, 5)   # noise model is part of the key
    ref = T.tqsim_run_ex(n, gates, T.noise_arg(0, 0), shots, ar, 5, T.default_options())
    assert np.array_equal(other.leaf_outcomes, ref.leaf_outcomes)


def test_qasm_program_runs_like_generator():
    """A QASM program through tqsim_parse_qasm runs to the same leaf
    outcomes as the same circuit from the generator, and matches the oracle."""
    from test_qasm import to_qasm
    w = load_config("c1_qft5")
    n, gates, noise, shots, ar = T.workload_args(w)
    n2, g2, measured = T.tqsim_parse_qasm(to_qasm(n, [tuple(g) for g in w.circuit.gates]))
    assert n2 == n and measured
    a = T.tqsim_run_ex(n, gates, noise, shots, ar, 3)
    b = T.tqsim_run_ex(n2, g2, noise, shots, ar, 3)
    assert np.array_equal(a.leaf_outcomes, b.leaf_outcomes)
    run_and_compare(n2, g2, NoiseModel(w.p1, w.p2, w.readout_p01, w.readout_p10), shots, ar, 3)


def test_copy_cost_profiler_feeds_dcp():
    """the measured B200 copy cost (gate units) is finite and positive,
    and as tqsim_options.copy_cost_gates it sets DCP's first-slice length."""
    c, cm, gm = T.tqsim_profile_copy_cost(15, 64, 0)
    assert np.isfinite(c) and c > 0 and cm > 0 and gm > 0
    assert abs(c - cm / gm) <= 1e-9 * c
    w = load_config("c2_qft15")
    n, gates, noise, shots, ar = T.workload_args(w)
    p = T.tqsim_plan_circuit(n, gates, noise, shots, None, T.default_options(copy_cost_gates=c))
    m = max(1, int(np.floor(c + 0.5)))
    if p.n_levels > 1:
        assert p.boundary_list[1] == m


def test_accuracy_tree_vs_flat_normalized_fidelity():
    """the tree output's normalized fidelity (Eq.7)
    matches the flat per-shot baseline's.  Tree and flat use independent seeds; the bound is
    the paper's maximum difference 0.016 plus 3 sigma of the difference of the two means
    (sigma from the per-seed spreads of both runs)."""
    import importlib.util
    import os
    from tq_testutil import ROOT
    spec = importlib.util.spec_from_file_location("tq_accuracy", os.path.join(ROOT, "scripts", "accuracy.py"))
    acc = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(acc)
    n, gates = acc.circuit("qft10h")
    r = acc.compare(n, gates, T.noise_arg(1e-3, 1e-2, 1e-2, 1e-2), 16000, 6)
    assert 0.0 < r["F_tree_mean"] <= 1.0 and 0.0 < r["F_flat_mean"] <= 1.0
    assert len(r["tree_arities"]) > 1                      # a real tree (DCP), not the flat plan
    assert r["diff_of_means"] <= 0.016 + 3.0 * r["sigma_diff"], r


@pytest.mark.parametrize("cfg,p", [("c1_qft5", 0.05), ("c2_qft15", None)])
def test_leaf_without_state_store_equals_stored_path(cfg, p):
    """The leaf measurement without a stored leaf state (run sums -> select -> recompute
    the run's tile -> finish) gives the same outcomes as the stored-state path (state
    dumps force it), including careful (error-frame) leaves; and matches the oracle."""
    w = load_config(cfg)
    n, gates, noise, shots, ar = T.workload_args(w)
    if p is not None:
        noise = T.noise_arg(p, 2 * p, 0.02, 0.03)
    L = T.tqsim_plan_circuit(n, gates, noise, shots, ar).n_levels
    a = T.tqsim_run_ex(n, gates, noise, shots, ar, 11)                       # no store
    b = T.tqsim_run_ex(n, gates, noise, shots, ar, 11, None, [(L - 1, 0)])   # stored
    assert np.array_equal(a.leaf_outcomes, b.leaf_outcomes)
    if cfg == "c1_qft5":
        nm = NoiseModel(noise.p1, noise.p2, noise.readout_p01, noise.readout_p10)
        ref = simulate_tree(n, OG.lower(gates), oracle_plan_of(a.plan), nm, 11)
        assert_leaves_match(a.leaf_outcomes, ref.leaves)


@pytest.mark.parametrize("tile,p", [(7, 0.1), (8, 0.4), (9, 1.0)])
def test_offtile_diagonal_units(tile, p):
    """QAOA (CX.RZ.CX) + QFT (lowered CP) on 14 qubits with tiles of 2^7..2^9: the first
    pass of a level applies diagonal units whose qubits lie off the tile, reading them
    from the tile index; errors inside those units flip off-tile qubits, which the
    out-of-place store applies as an address XOR."""
    from workloads.generators import qaoa_gates, random_3_regular_edges
    rng = np.random.default_rng(tile * 7 + int(p * 10))
    n = 14
    gates = qaoa_gates(n, random_3_regular_edges(n, rng), [0.4, 0.9], [0.3, 0.7]) + qft_gates(n)
    nm = NoiseModel(p, min(1.0, 2 * p), 0.02, 0.03)
    opts = T.default_options(tile_qubits=tile, batch_log2_amps=n + 2)
    noise = T.noise_arg(nm.p1, nm.p2, nm.readout_p01, nm.readout_p10)
    low = OG.lower(gates)
    recs = T.tqsim_describe_passes(n, gates, noise, 24, [3, 2, 4], opts)
    qm = lambda g: (1 << low[g][1]) | ((1 << low[g][2]) if low[g][2] >= 0 else 0)
    offtile = [r for r in recs if qm(r.gate) & ~r.tile_qubit_mask]
    assert offtile, "no off-tile diagonal unit in the plan"
    run_and_compare(n, gates, nm, 24, [3, 2, 4], 5 + tile, opts,
                    dumps=[(0, 0), (0, 2), (1, 4), (2, 23)])


@pytest.mark.parametrize("tile,p,ar", [(7, 0.2, [3, 2, 4]), (8, 1.0, [4, 6]), (10, 0.05, [4, 6])])
def test_store_map_cx_ladders(tile, p, ar):
    """HEA (RY layers + CX ladders) on 14 qubits with small tiles: the first pass of a
    level absorbs the CX gates that do not fit into a GF(2)-linear map of the store
    address; their errors conjugate through the map in the careful path; the leaf
    sampler inverts the map to find a run's tile (no-store leaf path)."""
    from workloads.generators import hea_gates
    rng = np.random.default_rng(tile + int(p * 100))
    n = 14
    gates = hea_gates(n, 3, rng.uniform(0, 6.28, (3, n)))
    gates += [("swap", 3, 11, 0.0, 0.0, 0.0), ("cx", 12, 5, 0.0, 0.0, 0.0), ("swap", 0, 9, 0.0, 0.0, 0.0)]
    nm = NoiseModel(p, min(1.0, 2 * p), 0.02, 0.03)
    opts = T.default_options(tile_qubits=tile, batch_log2_amps=n + 2)
    noise = T.noise_arg(nm.p1, nm.p2, nm.readout_p01, nm.readout_p10)
    recs = T.tqsim_describe_passes(n, gates, noise, 24, ar, opts)
    assert any(r.role == 3 for r in recs), "no absorbed CX in the plan"
    if len(ar) == 2:   # store maps in the leaf level's pass too
        assert any(r.role == 3 and r.level == 1 for r in recs)
    dumps = [(0, 0), (0, 2), (1, 4), (2, 23)] if len(ar) == 3 else [(0, 0), (0, 3), (1, 5), (1, 23)]
    run_and_compare(n, gates, nm, 24, ar, 11 + tile, opts, dumps=dumps)
    # the leaf sampler without stored leaf states (select -> recompute -> finish)
    res = T.tqsim_run_ex(n, gates, noise, 24, ar, 11 + tile, opts)
    low = OG.lower(gates)
    ref = simulate_tree(n, low, oracle_plan_of(res.plan), nm, 11 + tile)
    assert_leaves_match(res.leaf_outcomes, ref.leaves)


@pytest.mark.parametrize("n,ar,blog,tile", [(19, [2, 3, 4], 0, 0), (12, [3, 5, 3], 15, 6),
                                            (16, [2, 7], 19, 0), (14, [4, 4], 0, 7)])
def test_leaf_dedup_equals_stored_path(n, ar, blog, tile):
    """Error-free sibling leaves share one computed state (only the first error-free
    sibling of a batch runs the leaf passes; the sampler reads its run sums): outcomes
    equal the stored-state path bit for bit, through the chunk-sum sampler (n = 19) and
    with sibling groups cut by batch boundaries (batch of 2^blog amplitudes, arity 3 / 7),
    and with several leaf passes (small tiles: the recompute reads the representative's
    in-place slot)."""
    rng = np.random.default_rng(n + len(ar))
    gates = random_circuit(n, 60, rng)
    noise = T.noise_arg(0.003, 0.01, 0.02, 0.03)   # most leaves error-free: many duplicates
    shots = int(np.prod(ar))
    opts = T.default_options(batch_log2_amps=blog, tile_qubits=tile)
    recs = T.tqsim_describe_passes(n, gates, noise, shots, ar, opts)
    if tile:
        assert max(r.pass_ for r in recs if r.level == len(ar) - 1) >= 1   # multi-pass leaf level
    a = T.tqsim_run_ex(n, gates, noise, shots, ar, 5, opts)                          # dedup
    b = T.tqsim_run_ex(n, gates, noise, shots, ar, 5, opts, [(len(ar) - 1, 0)])      # stored
    assert np.array_equal(a.leaf_outcomes, b.leaf_outcomes)
    nm = NoiseModel(0.003, 0.01, 0.02, 0.03)
    if n <= 16:
        ref = simulate_tree(n, OG.lower(gates), oracle_plan_of(a.plan), nm, 5)
        assert_leaves_match(a.leaf_outcomes, ref.leaves)


def test_release_run_cache_then_run_again():
    """tqsim_release_run_cache frees the plan cache, arena and pinned buffer; the next
    tqsim_run plans and allocates again and gives the same outcomes."""
    w = load_config("c1_qft5")
    n, gates, noise, shots, ar = T.workload_args(w)
    a = T.tqsim_run(n, gates, noise, shots, ar, 3)
    T.tqsim_release_run_cache()
    b = T.tqsim_run(n, gates, noise, shots, ar, 3)
    assert np.array_equal(a.leaf_outcomes, b.leaf_outcomes)
    assert a.counts == b.counts


@pytest.mark.parametrize("tile,p", [(0, 0.002), (6, 0.01), (9, 0.05), (11, 0.002)])
def test_random_circuits_dedup_vs_oracle(tile, p):
    """Random circuits (every gate kind, SWAP / CP / CX ladders) through the default path --
    no state dumps, so shared states are computed once (dedup maps) and the leaves are
    sampled without stored states -- against the oracle's outcomes."""
    rng = np.random.default_rng(500 + tile)
    for it in range(3):
        n = int(rng.integers(5, 15))
        gates = random_circuit(n, int(rng.integers(30, 90)), rng)
        nm = NoiseModel(p, 2 * p, 0.02, 0.03)
        arities = [[3, 2, 4], [4, 4, 2], [2, 3, 2, 2]][it]
        shots = int(np.prod(arities))
        opts = T.default_options(tile_qubits=tile, batch_log2_amps=n + 3)
        run_and_compare(n, gates, nm, shots, arities, 900 + it, opts)


@pytest.mark.parametrize("n,tile,p,ar", [(14, 7, 0.05, [3, 2, 4]), (14, 8, 1.0, [3, 2, 4]), (12, 6, 0.002, [2, 2, 2, 3]),
                                         (13, 0, 0.2, [4, 6]), (20, 4, 0.01, [2, 3, 4])])
def test_conditional_leaf_sampling_vs_oracle(n, tile, p, ar):
    """Leaf slices ending in a single-qubit layer (QAOA mixers) are sampled top bits first
    (marginals of the top bits from the gates touching them, then the
    conditional state of the chosen bits): the outcomes equal the oracle's full-state
    inverse CDF and the stored-state path's, with errors in every kernel (p up to 1), dedup
    maps (p = 0.002), and the stage-2 chunk sampler (n = 20, one top bit)."""
    from workloads.generators import qaoa_gates, random_3_regular_edges
    rng = np.random.default_rng(n * 10 + tile)
    edges = random_3_regular_edges(n, rng) if n % 2 == 0 else [(q, (q + 1) % n) for q in range(n)]
    gates = qaoa_gates(n, edges, list(rng.uniform(0, 3, 2)), list(rng.uniform(0, 3, 2)))
    nm = NoiseModel(p, min(1.0, 2 * p), 0.02, 0.03)
    noise = T.noise_arg(nm.p1, nm.p2, nm.readout_p01, nm.readout_p10)
    opts = T.default_options(tile_qubits=tile, batch_log2_amps=n + 2)
    shots = int(np.prod(ar))
    plan = T.tqsim_plan_circuit(n, gates, noise, shots, ar, opts)
    assert plan.trail_top_bits > 0, "the plan does not use conditional leaf sampling"
    a = T.tqsim_run_ex(n, gates, noise, shots, ar, 21, opts, (), leaf_debug=True)           # conditional
    b = T.tqsim_run_ex(n, gates, noise, shots, ar, 21, opts, [(len(ar) - 1, 0)])             # stored path
    ref = simulate_tree(n, OG.lower(gates), oracle_plan_of(a.plan), nm, 21)
    flagged = {l for l, r in ref.leaves.items() if r.flagged}
    for l, r in ref.leaves.items():
        assert a.leaf_u[l] == r.u
        if l in flagged:
            continue
        assert int(a.leaf_outcomes[l]) == r.outcome, (l, int(a.leaf_outcomes[l]), r.outcome)
        assert int(b.leaf_outcomes[l]) == r.outcome
        assert not a.leaf_flagged[l]
    nd = T.tqsim_run_ex(n, gates, noise, shots, ar, 21, T.default_options(tile_qubits=tile, batch_log2_amps=n + 2,
                                                                       no_dedup=1))
    assert np.array_equal(nd.leaf_outcomes, a.leaf_outcomes)


def _fast_trail_circuit(n, m, rng):
    """RZZ units within the top m qubits and within the rest, CZ / T / RZ / P / U and RX layers:
    the leaf slice is diagonal units followed by top-qubit 1q gates (the streaming projection)."""
    from workloads.generators import g1, g2
    top, low = list(range(n - m, n)), list(range(n - m))
    gs = [g1("h", q) for q in range(n)]
    for _ in range(2):
        for (a, b) in [(top[0], top[1]), (top[2], top[-1]), (low[0], low[3]), (low[2], low[5]), (top[1], top[3])]:
            gs += [g2("cx", a, b), g1("rz", b, float(rng.uniform(0, 6))), g2("cx", a, b)]
        gs += [g2("cz", top[0], top[2]), g1("t", low[1]), g1("rz", top[1], 0.3)]
        gs += [g1("rx", q, float(rng.uniform(0, 3))) for q in range(n)]
        gs += [g1("p", top[0], 0.4), g1("u", top[2], 0.1, 0.2, 0.3)]
    return gs


@pytest.mark.parametrize("n,tile,p,ar,tl", [(14, 8, 0.05, [3, 2, 4], 3), (12, 7, 0.5, [2, 3, 4], 3),
                                            (18, 10, 0.002, [2, 2, 2, 3], 3), (14, 8, 1.0, [2, 3, 4], 3),
                                            (14, 8, 0.05, [3, 2, 4], 4), (18, 10, 0.01, [2, 2, 2, 3], 4),
                                            (16, 11, 0.5, [2, 3, 4], 5), (14, 8, 0.05, [3, 4, 2], 3),
                                            (18, 10, 0.3, [2, 3, 2], 4), (13, 9, 0.02, [3, 5, 2], 3)])
def test_streaming_projection_vs_oracle(n, tile, p, ar, tl):
    """The hand-written projection (diagonal units folded into per-leaf coefficients, top-qubit
    gates with their keyed Paulis) and its hand-over of leaves with a Pauli inside a unit to
    the generated kernel (p = 0.5, 1): outcomes equal the oracle's and the stored path's.
    tl = options.trail_low: the marginal pass's tile holds qubits 0..tl-1 and the top tile - tl."""
    rng = np.random.default_rng(n + tile)
    gates = _fast_trail_circuit(n, tile - tl, rng)
    nm = NoiseModel(p, min(1.0, 2 * p), 0.02, 0.03)
    noise = T.noise_arg(nm.p1, nm.p2, nm.readout_p01, nm.readout_p10)
    opts = T.default_options(tile_qubits=tile, batch_log2_amps=n + 2, trail_low=tl)
    shots = int(np.prod(ar))
    plan = T.tqsim_plan_circuit(n, gates, noise, shots, ar, opts)
    assert plan.trail_top_bits == tile - tl and plan.trail_fast == 1
    a = T.tqsim_run_ex(n, gates, noise, shots, ar, 33, opts, (), leaf_debug=True)
    b = T.tqsim_run_ex(n, gates, noise, shots, ar, 33, opts, [(len(ar) - 1, 1)])
    ref = simulate_tree(n, OG.lower(gates), oracle_plan_of(a.plan), nm, 33)
    for l, r in ref.leaves.items():
        if r.flagged:
            continue
        assert int(a.leaf_outcomes[l]) == r.outcome, (l, int(a.leaf_outcomes[l]), r.outcome)
        assert int(b.leaf_outcomes[l]) == r.outcome
        assert not a.leaf_flagged[l]


@pytest.mark.parametrize("world", [3, 5])
def test_conditional_sampling_split_level_shards(world):
    """Conditional leaf sampling under split-level sharding (W does not divide A_0,
    the leaf batches are clipped to the shard): serial shards add up to the single run."""
    torch = pytest.importorskip("torch")
    from workloads.generators import qaoa_gates, random_3_regular_edges
    rng = np.random.default_rng(40 + world)
    n = 14
    gates = qaoa_gates(n, random_3_regular_edges(n, rng), [0.7, 1.1], [0.4, 0.9])
    noise = T.noise_arg(0.01, 0.03, 0.01, 0.01)
    opts = T.default_options(tile_qubits=7, batch_log2_amps=n + 2)
    ar = [4, 3, 2]
    shots = int(np.prod(ar))
    h = T.tqsim_create(n, gates, noise, shots, ar, opts)
    assert h.plan.trail_top_bits > 0
    single = T.tqsim_run_ex(n, gates, noise, shots, ar, 8, opts).leaf_outcomes
    acc = np.zeros(shots, dtype=np.int64)
    split, lo, hi = T.tqsim_shard_levels(h.plan, 0, world)
    assert split > 0
    for r in range(world):
        ws = torch.empty(h.workspace_bytes(r, world), dtype=torch.uint8, device="cuda")
        o = torch.zeros(shots, dtype=torch.int32, device="cuda")
        h.execute(8, r, world, torch.cuda.current_stream().cuda_stream, ws.data_ptr(), ws.numel(), o.data_ptr())
        acc += o.cpu().numpy()
    assert np.array_equal(acc.astype(np.uint32), single)
    h.close()


@pytest.mark.parametrize("ar,world,blog", [([2, 3, 4], 3, 2), ([3, 5, 2], 2, 2), ([2, 7, 2], 5, 1)])
def test_streaming_projection_split_level_shards(ar, world, blog):
    """The streaming projection (clipped leaf batches, parent slots of a split shard; leaf
    arity 2: the sibling-pair kernel, batches of 2 or 4 leaves that may cut a pair) under
    serial shards equals the single run."""
    torch = pytest.importorskip("torch")
    n, tile = 14, 8
    gates = _fast_trail_circuit(n, tile - 3, np.random.default_rng(5))
    noise = T.noise_arg(0.02, 0.05, 0.01, 0.01)
    opts = T.default_options(tile_qubits=tile, batch_log2_amps=n + blog, trail_low=3)
    shots = int(np.prod(ar))
    h = T.tqsim_create(n, gates, noise, shots, ar, opts)
    assert h.plan.trail_fast == 1
    single = T.tqsim_run_ex(n, gates, noise, shots, ar, 12, opts).leaf_outcomes
    acc = np.zeros(shots, dtype=np.int64)
    assert T.tqsim_shard_levels(h.plan, 0, world)[0] > 0
    for r in range(world):
        ws = torch.empty(h.workspace_bytes(r, world), dtype=torch.uint8, device="cuda")
        o = torch.zeros(shots, dtype=torch.int32, device="cuda")
        h.execute(12, r, world, torch.cuda.current_stream().cuda_stream, ws.data_ptr(), ws.numel(), o.data_ptr())
        acc += o.cpu().numpy()
    assert np.array_equal(acc.astype(np.uint32), single)
    h.close()


@pytest.mark.parametrize("p", [0.05, 1.0])
def test_relabel_with_store_map_case_vs_oracle(p):
    """The stress-run case of a low-low SWAP relabeling next to an absorbed SWAP(7, 2) in a first
    pass (tests/golden/stress_relabel_map_case.json): outcomes and state dumps equal the oracle's."""
    import json
    import os
    from tq_testutil import ROOT
    d = json.load(open(os.path.join(ROOT, "tests", "golden", "stress_relabel_map_case.json")))
    gates = [tuple(g) for g in d["gates"]]
    opts = T.default_options(tile_qubits=d["tile_qubits"])
    run_and_compare(d["n_qubits"], gates, NoiseModel(p, p, 0.02, 0.03), int(np.prod(d["arities"])), d["arities"],
                    d["seed"] % (1 << 40), opts, dumps=[(0, 1), (1, 5), (2, 17)])
    run_and_compare(d["n_qubits"], gates, NoiseModel(p, p, 0.02, 0.03), int(np.prod(d["arities"])), d["arities"],
                    d["seed"] % (1 << 40), opts)


@pytest.mark.parametrize("n,tile,ar", [(14, 8, [2, 4, 6]), (16, 10, [3, 2, 8]), (12, 7, [2, 2, 2, 5])])
def test_conditional_sampling_b_only_errors_share_marginals(n, tile, ar):
    """Leaves whose errors all fall in the stage-2 gates B share their representative's marginals
    (the dedup map of the conditional-sampling leaf level counts pass A's gates only, DESIGN.md
    §6.2): noise on 1q gates only (p2 = 0), so many leaves draw errors only on the low-qubit RX
    layer.  Outcomes equal the oracle's, and the run with every instance computed."""
    from workloads.generators import qaoa_gates, random_3_regular_edges
    rng = np.random.default_rng(3 * n + tile)
    gates = qaoa_gates(n, random_3_regular_edges(n, rng), list(rng.uniform(0, 3, 2)), list(rng.uniform(0, 3, 2)))
    nm = NoiseModel(0.03, 0.0, 0.02, 0.0)
    noise = T.noise_arg(nm.p1, nm.p2, nm.readout_p01, nm.readout_p10)
    opts = T.default_options(tile_qubits=tile, batch_log2_amps=n + 4)
    shots = int(np.prod(ar))
    a = T.tqsim_run_ex(n, gates, noise, shots, ar, 5, opts, (), leaf_debug=True)
    assert a.plan.trail_top_bits > 0
    ref = simulate_tree(n, OG.lower(gates), oracle_plan_of(a.plan), nm, 5)
    for l, r in ref.leaves.items():
        assert a.leaf_u[l] == r.u
        if not r.flagged:
            assert int(a.leaf_outcomes[l]) == r.outcome, (l, int(a.leaf_outcomes[l]), r.outcome)
    nd = T.tqsim_run_ex(n, gates, noise, shots, ar, 5, T.default_options(tile_qubits=tile, batch_log2_amps=n + 4,
                                                                      no_dedup=1), leaf_debug=True)
    assert np.array_equal(nd.leaf_outcomes, a.leaf_outcomes)
    assert a.stats.computed_node_executions < nd.stats.computed_node_executions


@pytest.mark.parametrize("n,tile,p,ar,tl", [(14, 8, 0.2, [8, 8], 3), (16, 10, 0.1, [8, 8], 4),
                                            (12, 7, 0.6, [4, 16], 3)])
def test_streaming_projection_top_unit_paulis_vs_oracle(n, tile, p, ar, tl):
    """Paulis inside diagonal units on the TOP bits stay in the streaming projection (the unit
    with its Paulis is monomial: per-leaf effective diagonal + top-bit flips, kernels.cu
    proj_unit_eff); the leaf slice's units are all on the top bits, so no leaf is handed over.
    Outcomes equal the oracle's and the stored-state path's."""
    from workloads.generators import g1, g2
    rng = np.random.default_rng(n + tile)
    m = tile - tl
    top = list(range(n - m, n))
    suffix = []   # the leaf slice: top units (CX.RZ.CX, CZ), low gates, the RX layer
    for (a, b) in [(top[0], top[1]), (top[2], top[-1]), (top[1], top[3]), (top[-1], top[0])]:
        suffix += [g2("cx", a, b), g1("rz", b, float(rng.uniform(0, 6))), g2("cx", a, b)]
    suffix += [g2("cz", top[0], top[2]), g1("t", 1), g2("cx", 0, 2)]
    suffix += [g1("rx", q, float(rng.uniform(0, 3))) for q in range(n)]
    prefix = [g1("h", q) for q in range(n)]   # as many lowered gates: the first slice of a 2-level plan
    while len(OG.lower(prefix)) < len(OG.lower(suffix)):
        q = int(rng.integers(0, n - 1))
        prefix += [g1("ry", q, float(rng.uniform(0, 3))), g2("cx", q, q + 1)]
    while len(OG.lower(prefix)) > len(OG.lower(suffix)):
        prefix = prefix[:-1]
    gs = prefix + suffix
    nm = NoiseModel(p, p, 0.02, 0.03)
    noise = T.noise_arg(nm.p1, nm.p2, nm.readout_p01, nm.readout_p10)
    opts = T.default_options(tile_qubits=tile, batch_log2_amps=n + 3, trail_low=tl)
    shots = int(np.prod(ar))
    a = T.tqsim_run_ex(n, gs, noise, shots, ar, 17, opts, (), leaf_debug=True)
    assert a.plan.trail_top_bits > 0 and a.plan.trail_fast == 1
    b = T.tqsim_run_ex(n, gs, noise, shots, ar, 17, opts, [(len(ar) - 1, 0)])            # stored path
    ref = simulate_tree(n, OG.lower(gs), oracle_plan_of(a.plan), nm, 17)
    for l, r in ref.leaves.items():
        if r.flagged:
            continue
        assert int(a.leaf_outcomes[l]) == r.outcome, (l, int(a.leaf_outcomes[l]), r.outcome)
        assert int(b.leaf_outcomes[l]) == r.outcome


@pytest.mark.gpu
@pytest.mark.parametrize("p", [1.0, 0.2])
def test_nonmonomial_suffix_run_case_vs_oracle(p):
    """The stress-run case of a run H Tdg T H (product 1, suffix products not monomial;
    tests/golden/stress_nonmonomial_run_case.json): outcomes equal the oracle's, with and without
    dedup, and so do those of the minimal circuit."""
    import json
    import os
    from tq_testutil import ROOT
    d = json.load(open(os.path.join(ROOT, "tests", "golden", "stress_nonmonomial_run_case.json")))
    gates = [tuple(g) for g in d["gates"]]
    ar = d["arities"]
    for nd in (0, 1):
        opts = T.default_options(trail_low=4, batch_log2_amps=9, no_dedup=nd)
        run_and_compare(d["n_qubits"], gates, NoiseModel(p, min(1.0, 2 * p), 0.02, 0.03), int(np.prod(ar)), ar,
                        d["seed"] % (1 << 40), opts)
    mini = [("h", 1, -1, 0.0, 0.0, 0.0), ("tdg", 1, -1, 0.0, 0.0, 0.0), ("t", 1, -1, 0.0, 0.0, 0.0),
            ("h", 1, -1, 0.0, 0.0, 0.0), ("cx", 0, 1, 0.0, 0.0, 0.0), ("ry", 2, -1, 0.7, 0.0, 0.0)]
    run_and_compare(4, mini, NoiseModel(p, p, 0.0, 0.0), 24, [2, 3, 4], 5, T.default_options(small_tree=0))
