"""Sparse-state oracle for structured full-size variants -- TEST INFRASTRUCTURE ONLY.

Same algorithm as oracle.tree (P:224 tree, P:173/P:277 noise after each gate,
P:139 sampling, P:475 readout; readings R1-R11), but the state is a dict
{basis index: amplitude} holding only non-zero entries, so circuits whose noisy
trajectories stay k-sparse (monomial gates, GHZ-like states) are simulated at
any width (SURVEY §8(c) "structured variants").  A 1q matrix maps |x> to
m[0][b]|x with bit q = 0> + m[1][b]|x with bit q = 1> (b = bit q of x); entries
that are exactly zero are not stored.  Pinned against oracle.tree on small n by
tests/test_oracle_sparse.py.
"""
from __future__ import annotations

from typing import Dict, Optional, Tuple

import numpy as np

from . import gates as G
from .noise import noise_code
from .planner import Plan
from .tree import FLAG_EPS, LeafResult, NoiseModel, TreeResult, measure_uniform, readout_mask

SState = Dict[int, complex]


def apply_1q(st: SState, q: int, m: np.ndarray) -> SState:
    out: SState = {}
    bit = 1 << q
    for x, a in st.items():
        b = (x >> q) & 1
        x0 = x & ~bit
        for r in (0, 1):
            c = m[r, b]
            if c != 0:
                y = x0 | (r << q)
                out[y] = out.get(y, 0j) + c * a
    return {k: v for k, v in out.items() if v != 0}


def apply_2q(st: SState, a_q: int, b_q: int, m4: np.ndarray) -> SState:
    out: SState = {}
    mask = (1 << a_q) | (1 << b_q)
    for x, amp in st.items():
        col = (((x >> a_q) & 1) << 1) | ((x >> b_q) & 1)
        base = x & ~mask
        for row in range(4):
            c = m4[row, col]
            if c != 0:
                y = base | ((row >> 1) << a_q) | ((row & 1) << b_q)
                out[y] = out.get(y, 0j) + c * amp
    return {k: v for k, v in out.items() if v != 0}


def run_slice(st: SState, lowered, g0: int, g1: int, j: int, seed: int, noise: NoiseModel) -> SState:
    for g in range(g0, g1):
        kind, a, b, th, ph, la = lowered[g]
        if kind in G.TWO_QUBIT_PRIMS:
            st = apply_2q(st, a, b, G.matrix_2q(kind))
            code = noise_code(g, j, seed, noise.p2, True)
            if code:
                st = apply_1q(st, a, G.PAULI[code >> 2])
                st = apply_1q(st, b, G.PAULI[code & 3])
        else:
            st = apply_1q(st, a, G.matrix_1q(kind, th, ph, la))
            code = noise_code(g, j, seed, noise.p1, False)
            if code:
                st = apply_1q(st, a, G.PAULI[code])
    return st


def sample_leaf(st: SState, n: int, leaf: int, seed: int, noise: NoiseModel) -> LeafResult:
    keys = sorted(st)
    probs = [st[k].real ** 2 + st[k].imag ** 2 for k in keys]
    c = np.cumsum(probs)
    total = c[-1]
    u = measure_uniform(leaf, seed)
    target = u * total
    i = int(np.searchsorted(c, target, side="right"))
    i = min(i, len(keys) - 1)
    lo = c[i - 1] if i > 0 else 0.0
    flagged = bool(abs(target - lo) < FLAG_EPS or abs(c[i] - target) < FLAG_EPS)
    x = keys[i]
    mask = readout_mask(x, n, leaf, seed, noise.readout_p01, noise.readout_p10)
    return LeafResult(x, x ^ mask, flagged, u)


def simulate_tree(n: int, lowered, plan: Plan, noise: NoiseModel, seed: int,
                  top_range: Optional[Tuple[int, int]] = None, max_terms: int = 64) -> TreeResult:
    res = TreeResult()
    A, B, L = plan.arities, plan.boundaries, len(plan.arities)

    def node(d: int, j: int, parent: SState) -> None:
        st = run_slice(dict(parent), lowered, B[d], B[d + 1], j, seed, noise)
        if len(st) > max_terms:
            raise ValueError("state not sparse (%d terms)" % len(st))
        if d == L - 1:
            res.leaves[j] = sample_leaf(st, n, j, seed, noise)
            return
        for br in range(A[d + 1]):
            node(d + 1, j * A[d + 1] + br, st)

    lo, hi = top_range if top_range is not None else (0, A[0])
    for j0 in range(lo, hi):
        node(0, j0, {0: 1.0 + 0j})
    return res


def to_dense(st: SState, n: int) -> np.ndarray:
    v = np.zeros(2 ** n, dtype=np.complex128)
    for k, a in st.items():
        v[k] = a
    return v
