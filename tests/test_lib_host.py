"""Host-side tests of the C-ABI library (no GPU): it loads, exports every
symbol of include/tqsim.h, and its host logic (lowering, DCP planner, pass
planner, shard ranges) agrees with the oracle / invariants.  GPU entry points
must fail loudly without a device (no CPU fallback)."""
import os
import re

import numpy as np
import pytest

import paper_2203_13892_b200.tqsim as T
from oracle import gates as OG
from oracle.planner import dcp_plan, fixed_plan
from oracle.tree import NoiseModel, error_rates
from tq_testutil import ROOT
from workloads import config_names, load_config, qft_gates, random_circuit

HAVE_GPU = False
try:
    import torch
    HAVE_GPU = torch.cuda.is_available()
except Exception:  # pragma: no cover
    pass


def header_functions():
    src = open(os.path.join(ROOT, "include", "tqsim.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tqsim_[a-z_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = T.lib()
    names = header_functions()
    assert len(names) >= 18
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(T.EXPORTS)
    assert "sm_100a" in T.tqsim_version()


def test_lowering_matches_oracle():
    for name in config_names():
        w = load_config(name)
        mine = T.tqsim_lower_circuit(w.circuit.n_qubits, w.circuit.gates)
        ref = OG.lower(w.circuit.gates)
        assert [(k, a, (b if b >= 0 else 0)) for (k, a, b, *_r) in ref] == \
               [(k, a, (b if k in ("cx", "cz") else 0)) for (k, a, b) in mine]


def _oracle_plan(w, arities=None, **kw):
    low = OG.lower(w.circuit.gates)
    if arities is not None:
        return fixed_plan(len(low), arities)
    rates = error_rates(low, NoiseModel(w.p1, w.p2))
    return dcp_plan(rates, w.shots, w.circuit.n_qubits, w.copy_cost_gates, **kw)


def test_plan_matches_oracle_on_configs():
    for name in config_names():
        w = load_config(name)
        n, gates, noise, shots, ar = T.workload_args(w)
        p = T.tqsim_plan_circuit(n, gates, noise, shots, ar)
        o = _oracle_plan(w, ar)
        assert p.arity_list == o.arities, name
        assert p.boundary_list == o.boundaries, name
        assert p.n_outcomes == o.n_outcomes
        assert p.node_executions == sum(o.instances())
        assert abs(p.predicted_speedup_nodes - o.node_ratio_speedup()) < 1e-12
        assert abs(p.first_error_rate - o.first_error_rate) < 1e-15


def test_plan_matches_oracle_random_sweep():
    rng = np.random.default_rng(3)
    for it in range(60):
        n = int(rng.integers(1, 12))
        G = int(rng.integers(1, 400))
        gates = random_circuit(n, G, rng)
        if not gates:
            continue
        p1 = float(rng.choice([0.0, 1e-4, 1e-3, 1e-2, 0.2]))
        p2 = float(rng.choice([0.0, 1e-3, 1e-2, 0.3]))
        shots = int(rng.integers(1, 40000))
        cc = float(rng.choice([1, 3, 10, 20.4]))
        topup = int(rng.integers(0, 2))
        opts = T.default_options(copy_cost_gates=cc, topup=topup)
        p = T.tqsim_plan_circuit(n, gates, T.noise_arg(p1, p2), shots, None, opts)
        low = OG.lower(gates)
        o = dcp_plan(error_rates(low, NoiseModel(p1, p2)), shots, n, cc, topup=topup)
        assert p.arity_list == o.arities and p.boundary_list == o.boundaries


def test_invalid_inputs_rejected():
    noise = T.noise_arg(1e-3, 1e-2)
    with pytest.raises(T.TqsimError) as e:
        T.tqsim_plan_circuit(3, [("cx", 0, 0, 0, 0, 0)], noise, 10)
    assert e.value.status == 2
    with pytest.raises(T.TqsimError):
        T.tqsim_plan_circuit(3, [("h", 3, -1, 0, 0, 0)], noise, 10)
    with pytest.raises(T.TqsimError):
        T.tqsim_plan_circuit(3, [("h", 0, -1, 0, 0, 0)], T.noise_arg(1.5, 0), 10)
    with pytest.raises(T.TqsimError):
        T.tqsim_plan_circuit(3, [("h", 0, -1, 0, 0, 0)] * 4, noise, 100, arities=[5, 5])
    with pytest.raises(T.TqsimError):
        T.tqsim_plan_circuit(3, [("h", 0, -1, 0, 0, 0)] * 2, noise, 8, arities=[2, 2, 2])
    with pytest.raises(T.TqsimError):
        T.tqsim_plan_circuit(31, [("h", 0, -1, 0, 0, 0)], noise, 8)
    with pytest.raises(T.TqsimError):
        T.tqsim_plan_circuit(3, [("h", 0, -1, 0, 0, 0)], noise, 0)
    # memory budget too small for the DCP limit -> flat plan; for execution -> ECAPACITY
    p = T.tqsim_plan_circuit(20, [("h", 0, -1, 0, 0, 0)] * 100, noise, 1000,
                             options=T.default_options(mem_budget_bytes=16 << 20))
    assert p.n_levels == 1


def _check_pass_invariants(n, gates, noise, shots, arities=None, options=None):
    recs = T.tqsim_describe_passes(n, gates, noise, shots, arities, options)
    plan = T.tqsim_plan_circuit(n, gates, noise, shots, arities, options)
    low = OG.lower(gates)
    assert sorted(r.gate for r in recs) == list(range(len(low)))     # every gate exactly once
    def in_swap_triple(g):   # CX(a,b) CX(b,a) CX(a,b): one lowered SWAP
        for s0 in (g - 2, g - 1, g):
            if s0 < 0 or s0 + 2 >= len(low):
                continue
            x, y, z = low[s0], low[s0 + 1], low[s0 + 2]
            if x[0] == y[0] == z[0] == "cx" and x[1:3] == z[1:3] and y[1:3] == (x[2], x[1]):
                return True
        return False

    def is_diag(g):
        k, a, c, th, ph, la = low[g]
        if k in ("cx", "cz"):
            return k == "cz"
        m = OG.matrix_1q(k, th, ph, la)
        return m[0, 1] == 0 and m[1, 0] == 0

    def in_diag_unit(g):   # a diagonal gate, or CX(a,b) D(b) CX(a,b) (lowered RZZ / CP middle)
        if is_diag(g):
            return True
        for s0 in (g - 2, g):
            if s0 < 0 or s0 + 2 >= len(low):
                continue
            x, y, z = low[s0], low[s0 + 1], low[s0 + 2]
            if x[0] == z[0] == "cx" and x[1:3] == z[1:3] and is_diag(s0 + 1) and y[1] == x[2]:
                return True
        return False

    pos = {}
    for i, r in enumerate(recs):
        b = plan.boundary_list
        assert b[r.level] <= r.gate < b[r.level + 1]                 # in its own slice
        k, a, c = low[r.gate][0], low[r.gate][1], low[r.gate][2]
        qm = (1 << a) | ((1 << c) if c >= 0 else 0)
        # roles (tqsim_op_record.role): 0 register op; in the first (out-of-place) pass
        # of a level: 1 diagonal unit reading off-tile qubits from the tile index, 2
        # absorbed SWAP (store relabeling, qubits >= 3), 3 absorbed CX (store map)
        if r.role == 0:
            assert qm & ~r.reg_qubit_mask == 0, r.gate                # gate qubits in registers
        else:
            assert r.pass_ == 0, (r.gate, r.pass_, r.role)
        if r.role == 1:
            assert in_diag_unit(r.gate), r.gate
        elif r.role == 2:
            assert in_swap_triple(r.gate) and min(a, c) >= 3, r.gate
        elif r.role == 3:   # control a, target c; a low control only above the leaf level
            assert k == "cx" and (c < 3 or a >= 3 or (a == 2 and r.level + 1 < plan.n_levels)), r.gate
        assert r.reg_qubit_mask & ~r.tile_qubit_mask == 0            # registers within the tile
        assert bin(r.reg_qubit_mask).count("1") == min(4, max(n, 4))
        # store maps / relabelings act at the end of the pass
        if r.role in (2, 3):
            pos[r.gate] = (r.level, r.pass_, 1 << 30, i)
            continue
        pos[r.gate] = (r.level, r.pass_, r.phase, i)
    # order preserved between any two gates sharing a qubit
    last = {}
    for g, (k, a, c, *_r) in enumerate(low):
        for q in (a, c):
            if q < 0:
                continue
            if q in last:
                assert pos[last[q]] < pos[g], (last[q], g)
            last[q] = g
    return recs, plan


def test_pass_plan_invariants_configs():
    for name in config_names():
        w = load_config(name)
        recs, plan = _check_pass_invariants(*T.workload_args(w))
        assert plan.hbm_passes > 0


def test_pass_plan_invariants_random():
    rng = np.random.default_rng(9)
    for it in range(40):
        n = int(rng.integers(1, 22))
        gates = random_circuit(n, int(rng.integers(1, 200)), rng)
        if not gates:
            continue
        tq = int(rng.choice([0, 4, 7, 9, 12, 13]))
        _check_pass_invariants(n, gates, T.noise_arg(1e-3, 1e-2), int(rng.integers(1, 3000)),
                               None, T.default_options(tile_qubits=tq))


def test_shard_ranges_partition():
    w = load_config("c5_hea28")
    plan = T.tqsim_plan_circuit(*T.workload_args(w))
    for world in (1, 2, 3, 4, 8, 200):
        leaves, tops = [], []
        for r in range(world):
            t0, t1, l0, l1 = T.tqsim_shard_range(plan, r, world)
            tops.append((t0, t1))
            leaves.append((l0, l1))
        assert tops[0][0] == 0 and tops[-1][1] == plan.arities[0]
        assert leaves[0][0] == 0 and leaves[-1][1] == plan.n_outcomes
        assert all(a[1] == b[0] for a, b in zip(leaves, leaves[1:]))
    with pytest.raises(T.TqsimError):
        T.tqsim_shard_range(plan, 2, 2)


@pytest.mark.skipif(HAVE_GPU, reason="checks the no-GPU failure mode")
def test_gpu_entry_points_fail_loudly_without_device():
    w = load_config("c1_qft5")
    with pytest.raises(T.TqsimError) as e:
        T.tqsim_create(*T.workload_args(w))
    assert e.value.status == 4
    with pytest.raises(T.TqsimError) as e:
        T.tqsim_run(*T.workload_args(w))
    assert e.value.status == 4


def test_jit_compiles_every_variant_on_host():
    """NVRTC compiles every generated pass kernel (incl. the leaf no-store / recompute
    variants) without a GPU: a host-side check of the code generator."""
    for name in ("c1_qft5", "c2_qft15"):
        w = load_config(name)
        k, nbytes, sec = T.tqsim_compile_passes(*T.workload_args(w))
        assert k > 0 and nbytes > 0
    rng = np.random.default_rng(7)
    for tq in (0, 7, 12):
        n = int(rng.integers(5, 14))
        gates = random_circuit(n, 50, rng)
        k, _, _ = T.tqsim_compile_passes(n, gates, T.noise_arg(0.1, 0.2), 40, [4, 10],
                                         T.default_options(tile_qubits=tq))
        assert k > 0


def test_kernel_generator_accepts_every_random_plan():
    """The code generator (host side, no compile) accepts every pass of random circuits
    -- CP / RZZ / SWAP-heavy and general -- at every tile width, in particular first
    passes whose diagonal units sit off the tile (passplan.cpp diag_unit_at)."""
    from workloads.generators import g1, g2
    rng = np.random.default_rng(21)
    noise = T.noise_arg(0.05, 0.1)
    for it in range(24):
        n = int(rng.integers(4, 15))
        if it % 2:
            gates = random_circuit(n, int(rng.integers(20, 90)), rng)
        else:   # diagonal-unit heavy
            gates = []
            for _ in range(int(rng.integers(10, 40))):
                a, b = (int(v) for v in rng.choice(n, size=2, replace=False))
                r = int(rng.integers(0, 4))
                if r == 0:
                    gates += [g2("cx", a, b), g1("rz", b, float(rng.uniform(0, 6))), g2("cx", a, b)]
                elif r == 1:
                    gates.append(g2("cp", a, b, float(rng.uniform(0, 6))))
                elif r == 2:
                    gates.append(g2("swap", a, b))
                else:
                    gates.append(g1("rx", a, float(rng.uniform(0, 6))))
        arities = [3, 2, 4] if it % 3 else None
        for tile in (4, 6, 8, 10, 12):
            opts = T.default_options(tile_qubits=tile)
            recs = T.tqsim_describe_passes(n, gates, noise, 24, arities, opts)
            npass = {}
            for r in recs:
                npass[r.level] = max(npass.get(r.level, 0), r.pass_ + 1)
            for lv, k in npass.items():
                for ps in range(k):
                    assert T.tqsim_pass_source(n, gates, noise, 24, arities, opts, lv, ps)


def test_fused_copy_cost_first_slice():
    """copy_cost_gates = -1: the first slice is half the gates one
    HBM pass holds when the whole circuit is planned as one slice (the fused fan-out adds no pass;
    a level boundary costs the pass it splits), then DCP as usual."""
    import paper_2203_13892_b200.tqsim as T
    from workloads import load_config
    w = load_config("c4_qaoa24")
    n, gates, noise, shots, ar = T.workload_args(w)
    recs = T.tqsim_describe_passes(n, gates, noise, 1, [1])
    passes = len({r.pass_ for r in recs})
    G = len(T.tqsim_lower_circuit(n, gates))
    m = max(1, int(np.floor(max(1.0, 0.5 * G / passes) + 0.5)))
    p = T.tqsim_plan_circuit(n, gates, noise, shots, None, T.default_options(copy_cost_gates=-1.0))
    assert p.boundary_list[1] == m
    assert p.boundary_list[1] != 10
    with pytest.raises(T.TqsimError):
        T.tqsim_plan_circuit(n, gates, noise, shots, None, T.default_options(copy_cost_gates=-2.0))


def test_small_tree_choice_host(monkeypatch):
    """Host-side choice of the small-state tree kernel (options.small_tree):
    auto for C1 (n_outcomes x gates x 2^5 = 2.0e6 <= 2^24), never for C2 (15 qubits), above 10
    qubits, with a non-Pauli channel, or with small_tree = 2; TQSIM_SMALL=0 only stops auto."""
    monkeypatch.delenv("TQSIM_SMALL", raising=False)
    w = load_config("c1_qft5")
    n, gates, noise, shots, ar = T.workload_args(w)
    assert T.tqsim_plan_circuit(n, gates, noise, shots, ar).small_tree == 1
    assert T.tqsim_plan_circuit(n, gates, noise, shots, ar, T.default_options(small_tree=2)).small_tree == 0
    w2 = load_config("c2_qft15")
    n2, g2, noise2, s2, ar2 = T.workload_args(w2)
    assert T.tqsim_plan_circuit(n2, g2, noise2, s2, ar2, T.default_options(small_tree=1)).small_tree == 0
    rng = np.random.default_rng(3)
    g10 = random_circuit(10, 60, rng)
    # 88 lowered gates x 2^10: 2^24 / 90,112 = 186 outcomes -- 100 shots auto, 1,000 not
    assert T.tqsim_plan_circuit(10, g10, noise, 100, [10, 10]).small_tree == 1
    assert T.tqsim_plan_circuit(10, g10, noise, 1000, [10, 100]).small_tree == 0
    assert T.tqsim_plan_circuit(10, g10, noise, 1000, [10, 100], T.default_options(small_tree=1)).small_tree == 1
    kn = T.noise_arg(0.01, 0.02, 0.0, 0.0, amp_damping=0.01)
    assert T.tqsim_plan_circuit(6, random_circuit(6, 20, rng), kn, 100, [10, 10],
                                T.default_options(small_tree=1)).small_tree == 0
    monkeypatch.setenv("TQSIM_SMALL", "0")
    assert T.tqsim_plan_circuit(n, gates, noise, shots, ar).small_tree == 0
    assert T.tqsim_plan_circuit(n, gates, noise, shots, ar, T.default_options(small_tree=1)).small_tree == 1
    with pytest.raises(T.TqsimError):
        T.tqsim_plan_circuit(n, gates, noise, shots, ar, T.default_options(small_tree=3))


def test_relabel_with_store_map_regression():
    """A first pass holding both a low-low SWAP (a relabeling of physical qubits 0 and 2) and an
    absorbed SWAP(7, 2) (store-map CX gates on logical qubit 2): every pass kernel of the plan
    generates (before the fix the relabeling carried the mapped qubit onto physical 0 and the
    generator raised TQSIM_EINTERNAL).  Case from scripts/stress_parity.py (fixture: inputs only)."""
    import json
    d = json.load(open(os.path.join(ROOT, "tests", "golden", "stress_relabel_map_case.json")))
    gates = [tuple(g) for g in d["gates"]]
    n, ar = d["n_qubits"], d["arities"]
    noise = T.noise_arg(0.05, 0.1)
    opts = T.default_options(tile_qubits=d["tile_qubits"])
    plan = T.tqsim_plan_circuit(n, gates, noise, int(np.prod(ar)), ar, opts)
    for lv in range(plan.n_levels):
        p = 0
        while True:
            try:
                src = T.tqsim_pass_source(n, gates, noise, int(np.prod(ar)), ar, opts, lv, p)
            except T.TqsimError as e:
                assert "out of range" in str(e), (lv, p, str(e))
                break
            assert "__global__" in src
            p += 1
        assert p >= 1


def test_kraus_width_limit_host():
    """The Kraus engine's width limit (include/tqsim.h TQSIM_KRAUS_MAX_QUBITS = 16: one CTA up
    to 13 qubits, a thread-block cluster of 2^(n-13) CTAs for 14..16): 16 plans, 17 is
    TQSIM_EINVAL; the same widths without non-Pauli channels are not limited."""
    kn = T.noise_arg(1e-3, 1e-2, 0.0, 0.0, amp_damping=0.01)
    for n in (13, 14, 16):
        assert T.tqsim_plan_circuit(n, qft_gates(n), kn, 32, [4, 8]).n_outcomes == 32
    with pytest.raises(T.TqsimError) as e:
        T.tqsim_plan_circuit(17, qft_gates(17), kn, 32, [4, 8])
    assert e.value.status == 2
    assert T.tqsim_plan_circuit(17, qft_gates(17), T.noise_arg(1e-3, 1e-2), 32, [4, 8]).n_outcomes == 32


def test_nonmonomial_suffix_run_regression():
    """A run of single-qubit gates whose product is diagonal (H Tdg T H = 1) but whose suffix
    products are not monomial (an error after Tdg pushed through T H is (Z - Y)/sqrt 2) must not be
    fused into one DIAG / NOP op: every pass kernel of the plan generates and compiles (before the
    fix the generator raised TQSIM_EINTERNAL 'not an X-type permutation').  Case from
    scripts/stress_parity.py (fixture: inputs only)."""
    import json
    d = json.load(open(os.path.join(ROOT, "tests", "golden", "stress_nonmonomial_run_case.json")))
    gates = [tuple(g) for g in d["gates"]]
    n, ar = d["n_qubits"], d["arities"]
    for p in (1.0, 0.2):
        k, _, _ = T.tqsim_compile_passes(n, gates, T.noise_arg(p, p), int(np.prod(ar)), ar,
                                         T.default_options(trail_low=4, batch_log2_amps=9))
        assert k > 0
    mini = [("h", 1, -1, 0.0, 0.0, 0.0), ("tdg", 1, -1, 0.0, 0.0, 0.0), ("t", 1, -1, 0.0, 0.0, 0.0),
            ("h", 1, -1, 0.0, 0.0, 0.0), ("cx", 0, 1, 0.0, 0.0, 0.0), ("ry", 2, -1, 0.7, 0.0, 0.0)]
    k, _, _ = T.tqsim_compile_passes(4, mini, T.noise_arg(0.3, 0.3), 6, [2, 3])
    assert k > 0
