"""Tree simulation with reuse, leaf sampling and readout -- oracle copy
(test infrastructure only).

Follows the algorithm step by step in the paper's order (SURVEY §8(c)
"Oracle algorithm", R1-R11):

* Tree (§3): the root is the initial state |0...0>; a depth-(d+1) node is
  an instance of subcircuit d; a node's output state is reused by its A_{d+1}
  children.  Node (d, j_d), j_d in [0, prod_{i<=d} A_i), has parent
  j_{d-1} = j_d // A_d (i.e. j_d = j_{d-1} * A_d + branch).
* Node execution (§2.5): start from a copy of the parent state; for
  each gate g of slice d: psi <- G_g psi, then the keyed draw (oracle.noise) and,
  on error, the Pauli(s) after the gate.
* Leaf l (§2.3 "the final outcome is sampled"; one sample per leaf, R10):
  p_x = |a_x|^2, C = sequential cumsum, total = C[-1];
  (w0, w1) = Philox(ctr = (0, l, 1, 0)), u = ((w0>>5) 2^26 + (w1>>6)) 2^-53;
  x = smallest x with C(x) > u*total (np.searchsorted side='right', clamped);
  flagged if u*total is within 1e-9 of C(x-1) or C(x) (R9);
  readout: bit b flips iff word (b&3) of Philox(ctr=(b>>2, l, 2, 0)),
  times 2^-32, is < p10 (bit = 1) or p01 (bit = 0).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, Iterable, List, Optional, Sequence, Tuple

import numpy as np

from . import gates as G
from .noise import TAG_MEASURE, TAG_READOUT, noise_code
from .philox import philox4x32_10, seed_key
from .planner import Plan
from .statevector import apply_1q, apply_2q, zero_state

FLAG_EPS = 1e-9


@dataclass
class NoiseModel:
    p1: float
    p2: float
    readout_p01: float = 0.0
    readout_p10: float = 0.0


@dataclass
class LeafResult:
    x: int                 # sampled basis index before readout
    outcome: int           # after readout flips
    flagged: bool          # draw within FLAG_EPS of a CDF boundary
    u: float


def apply_gate_with_noise(psi: np.ndarray, n: int, gate, g: int, j: int, seed: int,
                          noise: NoiseModel) -> np.ndarray:
    kind, a, b, th, ph, la = gate
    if kind in G.TWO_QUBIT_PRIMS:
        psi = apply_2q(psi, n, a, b, G.matrix_2q(kind))
        code = noise_code(g, j, seed, noise.p2, True)
        if code:
            psi = apply_1q(psi, n, a, G.PAULI[code >> 2])
            psi = apply_1q(psi, n, b, G.PAULI[code & 3])
    else:
        psi = apply_1q(psi, n, a, G.matrix_1q(kind, th, ph, la))
        code = noise_code(g, j, seed, noise.p1, False)
        if code:
            psi = apply_1q(psi, n, a, G.PAULI[code])
    return psi


def run_slice(psi: np.ndarray, n: int, lowered, g_begin: int, g_end: int, j: int,
              seed: int, noise: NoiseModel) -> np.ndarray:
    for g in range(g_begin, g_end):
        psi = apply_gate_with_noise(psi, n, lowered[g], g, j, seed, noise)
    return psi


def measure_uniform(leaf: int, seed: int) -> float:
    k = seed_key(seed)
    w0, w1, _, _ = philox4x32_10((0, leaf & 0xFFFFFFFF, TAG_MEASURE, leaf >> 32), k)
    return ((w0 >> 5) * 67108864.0 + (w1 >> 6)) * (1.0 / 9007199254740992.0)


def readout_mask(x: int, n: int, leaf: int, seed: int, p01: float, p10: float) -> int:
    if p01 == 0.0 and p10 == 0.0:
        return 0
    k = seed_key(seed)
    mask = 0
    words = None
    for bit in range(n):
        if bit % 4 == 0:
            words = philox4x32_10((bit >> 2, leaf & 0xFFFFFFFF, TAG_READOUT, leaf >> 32), k)
        w = words[bit & 3]
        p = p10 if (x >> bit) & 1 else p01
        if float(w) * 2.0 ** -32 < p:
            mask |= 1 << bit
    return mask


def sample_leaf(psi: np.ndarray, n: int, leaf: int, seed: int, noise: NoiseModel) -> LeafResult:
    prob = psi.real ** 2 + psi.imag ** 2
    c = np.cumsum(prob)
    total = c[-1]
    u = measure_uniform(leaf, seed)
    target = u * total
    x = int(np.searchsorted(c, target, side="right"))
    x = min(x, 2 ** n - 1)
    lo = c[x - 1] if x > 0 else 0.0
    flagged = bool(abs(target - lo) < FLAG_EPS or abs(c[x] - target) < FLAG_EPS)
    mask = readout_mask(x, n, leaf, seed, noise.readout_p01, noise.readout_p10)
    return LeafResult(x, x ^ mask, flagged, u)


@dataclass
class TreeResult:
    leaves: Dict[int, LeafResult] = field(default_factory=dict)
    dumps: Dict[Tuple[int, int], np.ndarray] = field(default_factory=dict)

    def outcome_array(self, n_outcomes: int) -> np.ndarray:
        out = np.zeros(n_outcomes, dtype=np.uint32)
        for l, r in self.leaves.items():
            out[l] = r.outcome
        return out


def simulate_tree(n: int, lowered, plan: Plan, noise: NoiseModel, seed: int,
                  top_range: Optional[Tuple[int, int]] = None,
                  dump: Iterable[Tuple[int, int]] = ()) -> TreeResult:
    """DFS over the tree with state reuse.  top_range restricts the level-0
    instances (a shard / bounded sample).  dump = {(level, instance)} whose
    post-slice states are recorded."""
    dump = set(dump)
    res = TreeResult()
    A = plan.arities
    B = plan.boundaries
    L = len(A)

    def node(d: int, j: int, parent: np.ndarray) -> None:
        psi = run_slice(parent.copy(), n, lowered, B[d], B[d + 1], j, seed, noise)
        if (d, j) in dump:
            res.dumps[(d, j)] = psi.copy()
        if d == L - 1:
            res.leaves[j] = sample_leaf(psi, n, j, seed, noise)
            return
        for br in range(A[d + 1]):
            node(d + 1, j * A[d + 1] + br, psi)

    root = zero_state(n)
    lo, hi = top_range if top_range is not None else (0, A[0])
    for j0 in range(lo, hi):
        node(0, j0, root)
    return res


def leaf_ancestors(plan: Plan, leaf: int) -> List[int]:
    """j_d for d = 0..L-1 of the path to `leaf` (j_{L-1} = leaf)."""
    A = plan.arities
    L = len(A)
    out = [0] * L
    j = leaf
    for d in range(L - 1, -1, -1):
        out[d] = j
        j //= A[d]
    return out


def simulate_leaf_flat(n: int, lowered, plan: Plan, noise: NoiseModel, seed: int,
                       leaf: int, want_states: bool = False):
    """Per-leaf flat recompute with inherited keys: run every slice d on one
    state with key j_d.  Must equal the tree DFS exactly (reuse is exact)."""
    anc = leaf_ancestors(plan, leaf)
    psi = zero_state(n)
    states = {}
    for d, j in enumerate(anc):
        psi = run_slice(psi, n, lowered, plan.boundaries[d], plan.boundaries[d + 1], j, seed, noise)
        if want_states:
            states[(d, j)] = psi.copy()
    r = sample_leaf(psi, n, leaf, seed, noise)
    return (r, psi, states) if want_states else r


def histogram(outcomes: Sequence[int]) -> Dict[int, int]:
    h: Dict[int, int] = {}
    for o in outcomes:
        h[int(o)] = h.get(int(o), 0) + 1
    return h


def ideal_state(n: int, lowered) -> np.ndarray:
    psi = zero_state(n)
    for (kind, a, b, th, ph, la) in lowered:
        if kind in G.TWO_QUBIT_PRIMS:
            psi = apply_2q(psi, n, a, b, G.matrix_2q(kind))
        else:
            psi = apply_1q(psi, n, a, G.matrix_1q(kind, th, ph, la))
    return psi


def error_rates(lowered, noise: NoiseModel) -> List[float]:
    return [noise.p2 if g[0] in G.TWO_QUBIT_PRIMS else noise.p1 for g in lowered]
