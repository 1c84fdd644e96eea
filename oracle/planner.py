"""Tree planning -- oracle copy (test infrastructure only).

Tree notation (A_0, ..., A_{k-1}) and instances of subcircuit i = prod_{j<=i} A_j
(§3.1, Eq.2, counting the level-i nodes; the paper's 0-based product
bound is read as "including the node's own arity", which is what makes
(64,1,1) have 192 subcircuit nodes, fig:graphical-representation P:233).

Dynamic Circuit Partition (§3.2, §3.3) in the reading of
SURVEY §8(c) step 2 (R12-R18):

  1. m = max(1, round(copy_cost_gates))           first-slice length
     if G < 2m or N == 1: flat plan (N)
  2. p_hat = 1 - prod_{g<m} (1 - e_g)              Eq.3, readout excluded
  3. p_hat = min(p_hat, 0.5); n0 = z^2 p_hat (1-p_hat) / eps^2
     A_0 = clamp(ceil(n0 / (1 + n0/N)), 1, N)     Eq.4, z=1.96, eps=0.05
  4. k = max k <= min(floor((G-m)/m), floor(budget/S) - 2) with 2^k A_0 <= N
     ("maximum value of k such that A_r >= 2"; limits P:310-316); none -> flat
  5. A_r = largest integer a with a^k A_0 <= N    Eq.5 IN INTEGERS
  6. top-up: A_0 = max(A_0, ceil(N / A_r^k))      P:294 "adding one ... starting from
     the first subcircuit" (reading R18; topup=1 selects SPEC's round-robin)
  7. slices: [m] + k near-equal slices of the remaining G-m gates, extra gates
     to the earliest slices (R17).
Fixed arities: equal split of G into len(arities) slices (R20).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional, Sequence


@dataclass
class Plan:
    arities: List[int]
    boundaries: List[int]            # len = L+1, slice d = gates [b[d], b[d+1])
    first_error_rate: float = 0.0    # p_hat (Eq.3), 0 for fixed/flat plans

    @property
    def n_levels(self) -> int:
        return len(self.arities)

    def instances(self) -> List[int]:
        """Eq.2: number of level-d nodes = prod_{i<=d} A_i."""
        out, acc = [], 1
        for a in self.arities:
            acc *= a
            out.append(acc)
        return out

    @property
    def n_outcomes(self) -> int:
        return self.instances()[-1]

    def total_nodes(self) -> int:
        """Subcircuit nodes + the root (initial-state) node."""
        return sum(self.instances()) + 1

    def node_ratio_speedup(self) -> float:
        """Max speedup as node ratio vs the baseline tree (N,1,...,1) (Table 3)."""
        inst = self.instances()
        return len(inst) * inst[-1] / float(sum(inst))

    def gate_ratio_speedup(self) -> float:
        inst = self.instances()
        tree = sum(i * (self.boundaries[d + 1] - self.boundaries[d]) for d, i in enumerate(inst))
        flat = inst[-1] * self.boundaries[-1]
        return flat / float(tree)

    def tree_gate_apps(self) -> int:
        inst = self.instances()
        return sum(i * (self.boundaries[d + 1] - self.boundaries[d]) for d, i in enumerate(inst))


def split_equal(g_start: int, g_count: int, parts: int) -> List[int]:
    """Boundaries splitting [g_start, g_start+g_count) into `parts` slices whose
    lengths differ by at most one, extra gates going to the earliest slices."""
    base, extra = divmod(g_count, parts)
    b = [g_start]
    for i in range(parts):
        b.append(b[-1] + base + (1 if i < extra else 0))
    return b


def fixed_plan(n_gates: int, arities: Sequence[int]) -> Plan:
    return Plan(list(int(a) for a in arities), split_equal(0, n_gates, len(arities)))


def flat_plan(n_gates: int, n_shots: int) -> Plan:
    return Plan([int(n_shots)], [0, int(n_gates)])


def eq4_first_arity(p_hat: float, n_shots: int, z: float = 1.96, eps: float = 0.05) -> int:
    """Eq.4 evaluated in exactly this fp64 order, ceil, clamp [1, N]."""
    p = min(p_hat, 0.5)
    n0 = (z * z * p * (1.0 - p)) / (eps * eps)
    a0 = math.ceil(n0 / (1.0 + n0 / float(n_shots)))
    return int(min(max(a0, 1), n_shots))


def int_root_floor(q: int, k: int) -> int:
    """Largest integer a with a^k <= q (Eq.5 floor of the k-th root, in integers)."""
    if q < 1:
        return 0
    a = 1
    while (a + 1) ** k <= q:
        a += 1
    return a


def dcp_plan(error_rates: Sequence[float], n_shots: int, n_qubits: int,
             copy_cost_gates: float = 10.0, z: float = 1.96, eps: float = 0.05,
             mem_budget_bytes: int = 180_000_000_000, topup: int = 0) -> Plan:
    """error_rates[g] = e_g of lowered gate g (p1 for 1q, p2 for 2q)."""
    G = len(error_rates)
    N = int(n_shots)
    m = max(1, int(math.floor(copy_cost_gates + 0.5)))
    if G < 2 * m or N == 1:
        return flat_plan(G, N)
    prod = 1.0
    for g in range(m):
        prod *= (1.0 - error_rates[g])
    p_hat = 1.0 - prod
    a0 = eq4_first_arity(p_hat, N, z, eps)
    state_bytes = 16 * (2 ** n_qubits)
    k_max = min((G - m) // m, mem_budget_bytes // state_bytes - 2)
    k = 0
    for kk in range(1, max(k_max, 0) + 1):
        if (2 ** kk) * a0 <= N:
            k = kk
    if k < 1:
        p = flat_plan(G, N)
        p.first_error_rate = p_hat
        return p
    ar = int_root_floor(N // a0, k)         # a^k * a0 <= N  <=>  a^k <= floor(N/a0)
    ar_k = ar ** k
    if topup == 0:
        a0 = max(a0, -(-N // ar_k))
        arities = [a0] + [ar] * k
    else:
        arities = [a0] + [ar] * k
        i = 0
        while math.prod(arities) < N:
            arities[i % len(arities)] += 1
            i += 1
    boundaries = [0] + split_equal(m, G - m, k)
    return Plan(arities, boundaries, p_hat)
