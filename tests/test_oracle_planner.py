"""Pins for oracle.planner against numbers the paper prints (no GPU)."""
import math

import pytest

from oracle.planner import (Plan, dcp_plan, eq4_first_arity, fixed_plan, flat_plan,
                            int_root_floor, split_equal)
from oracle import gates as G
from oracle.tree import NoiseModel, error_rates
from tq_testutil import golden_rows
from workloads import load_config


def test_table3_node_ratio_speedups():
    rows = golden_rows("table3_qpe_structures.txt")
    assert len(rows) == 5
    for r in rows:
        ar = [int(v) for v in r[:3]]
        p = fixed_plan(120, ar)                       # QPE_9 has 120 gates
        assert p.n_outcomes == 1000
        assert round(p.node_ratio_speedup(), 2) == float(r[3])


def test_tree_node_counts_from_captions():
    for r in golden_rows("tree_node_counts.txt"):
        ar = [int(v) for v in r[0].split(",")]
        p = fixed_plan(9, ar)
        assert p.total_nodes() == int(r[1])
        assert p.n_outcomes == int(r[2])


def test_qft14_plan_p527():
    d = {r[0]: r[1] for r in golden_rows("qft14_plan.txt")}
    G_, e, N = int(d["n_gates"]), float(d["error_rate"]), int(d["shots"])
    for m in range(int(d["copy_cost_min"]), int(d["copy_cost_max"]) + 1):
        p = dcp_plan([e] * G_, N, 14, copy_cost_gates=m)
        assert p.n_levels == int(d["n_subcircuits"])
        assert p.arities[0] == int(d["first_arity"])
        assert p.arities == [500, 2, 2, 2, 2, 2, 2]
        assert round(p.node_ratio_speedup(), 2) == float(d["max_speedup"])
        assert p.boundaries[1] == m and p.boundaries[-1] == G_


def test_eq4_closed_form_values():
    # p_hat = 0.5 maximises p(1-p): n0 = 1.96^2/(4*0.05^2) = 384.16 -> 384.16/(1+384.16/32000)
    assert eq4_first_arity(0.5, 32000) == math.ceil(384.16 / (1 + 384.16 / 32000)) == 380
    assert eq4_first_arity(0.9, 32000) == 380           # clamped to 0.5 (R12)
    assert eq4_first_arity(0.0, 32000) == 1             # noise-free -> 1
    assert eq4_first_arity(0.5, 10) == 10               # clamp to N
    p = 1 - (1 - 1e-3) ** 10
    n0 = 1.96 ** 2 * p * (1 - p) / 0.05 ** 2
    assert eq4_first_arity(p, 32000) == math.ceil(n0 / (1 + n0 / 32000)) == 16


def test_eq5_integer_root():
    assert int_root_floor(1000, 3) == 10                # float pow gives 9.999999999999998
    assert math.floor(1000 ** (1 / 3)) == 9             # the pitfall (R15)
    assert int_root_floor(125, 3) == 5
    assert int_root_floor(64, 6) == 2 and int_root_floor(63, 6) == 1
    for q in range(1, 3000, 37):
        for k in range(1, 6):
            a = int_root_floor(q, k)
            assert a ** k <= q < (a + 1) ** k


def test_degenerate_plans():
    assert dcp_plan([1e-3] * 100, 1, 10).arities == [1]                  # N = 1 -> flat
    assert dcp_plan([1e-3] * 15, 1000, 10).arities == [1000]             # G < 2m -> flat
    p = dcp_plan([0.0] * 200, 1000, 10)                                  # noise-free: A0 = 1 ...
    assert p.arities[1:] == [2] * 9 and p.arities[0] == 2                # ... then top-up to 2
    assert split_equal(10, 11, 3) == [10, 14, 18, 21]
    assert fixed_plan(63, [10, 100]).boundaries == [0, 32, 63]


def test_memory_limit_caps_levels():
    # k + 2 <= floor(budget / S): S = 16 * 2^28 = 4 GiB, budget 6 states -> k <= 4
    p = dcp_plan([1e-3] * 1000, 32000, 28, mem_budget_bytes=6 * 16 * 2 ** 28)
    assert p.n_levels - 1 <= 4


def test_every_plan_meets_shots():
    for N in (2, 3, 7, 64, 100, 999, 1000, 4097, 32000):
        for e in (0.0, 1e-4, 1e-3, 1e-2, 0.1):
            for G_ in (5, 20, 100, 600):
                for topup in (0, 1):
                    p = dcp_plan([e] * G_, N, 12, topup=topup)
                    assert p.n_outcomes >= N
                    assert p.boundaries[0] == 0 and p.boundaries[-1] == G_
                    assert all(b1 > b0 for b0, b1 in zip(p.boundaries, p.boundaries[1:]))
                    assert all(a >= 1 for a in p.arities)


def _plan_of(name):
    w = load_config(name)
    low = G.lower(w.circuit.gates)
    rates = error_rates(low, NoiseModel(w.p1, w.p2))
    return dcp_plan(rates, w.shots, w.circuit.n_qubits, w.copy_cost_gates), len(low)


def test_config_plans_appendix_a():
    # SURVEY Appendix A, derived by hand from rule §8(c) step 2 (regression pin)
    exp = {"c2_qft15": ([20] + [2] * 9, 20460), "c3_brick20": ([20] + [2] * 9, 20460),
           "c4_qaoa24": ([16] + [2] * 9, 16368), "c5_hea28": ([128] + [2] * 8, 65408)}
    for name, (ar, nodes) in exp.items():
        p, G_ = _plan_of(name)
        assert p.arities == ar, name
        assert p.total_nodes() - 1 == nodes
    p, _ = _plan_of("c5_hea28")
    assert abs(p.first_error_rate - 0.044588) < 1e-6
    assert p.boundaries == [0, 10] + [10 + 30 * i for i in range(1, 7)] + [219, 248]
