"""Non-Pauli error channels as quantum trajectories -- oracle copy (test infrastructure only).

The paper's sensitivity study (§4.3.2, Table 2, results P:627-661)
adds to the depolarizing channel (DC) the thermal relaxation (TR), amplitude damping (AD,
"damping ratio of 0.01") and phase damping (PD, "damping ratio of 0.01") channels, each
"through a set of Kraus operators", plus readout error; ALL combines them.  The paper
gives no Kraus matrices, no TR parameters, no order and no sampling rule; the readings
below (R31-R37) fix them, and this module follows them step by step.

R31 Kraus sets (standard forms):
      AD(g):  K0 = [[1, 0], [0, sqrt(1-g)]],  K1 = [[0, sqrt(g)], [0, 0]]
      PD(l):  K0 = [[1, 0], [0, sqrt(1-l)]],  K1 = [[0, 0], [0, sqrt(l)]]
R32 TR(T1, T2, t) = AD(g_T) followed by PD(l_T) with g_T = 1 - exp(-t/T1) and
      l_T = 1 - exp(-2t/T2 + t/T1) (T2 <= 2 T1): populations relax as exp(-t/T1) and
      coherences decay as sqrt(1-g_T) sqrt(1-l_T) = exp(-t/T2).  t = the gate's duration
      (1q or 2q class).
R33 Locations: after every lowered gate, after its depolarizing Pauli ("after each
      of the gates"), on every qubit the gate acts on.  Sub-location order
      s = 2c + i: channel c in (0 TR-amplitude, 1 TR-phase, 2 AD, 3 PD), qubit i in
      (0: q0, 1: q1 of a 2q gate); disabled channels / absent qubits are skipped.
R34 Draw: r = w * 2^-32, w = word (s & 3) of Philox4x32-10(ctr = (g, j mod 2^32,
      3 + (s >> 2), j >> 32), key = seed) -- keyed like the Pauli draw (tags 0..2 are
      noise / measure / readout), so CPU and GPU draw the same r.
R35 Choice (quantum-trajectory unravelling): with psi normalised, p_k = ||K_k psi||^2;
      the smallest k with r < p_0 + ... + p_k is taken (K0 first), psi <- K_k psi / sqrt(p_k).
      The ensemble over r reproduces rho -> sum_k K_k rho K_k^dag (pinned against the
      density-matrix channel by exact branch enumeration, tests/test_oracle_kraus.py).
R36 Flag: a decision whose r lies within 1e-9 of a cumulative boundary p_0 + .. + p_k is
      flagged, and every leaf below a flagged decision is flagged (a rounding difference
      could flip it), as R9 does for the sampling draw.
R37 Planning: the tree structure comes from the depolarizing rates ("we use
      the parameters from depolarizing channel to generate the TQSim structure and use it
      across all noise models").
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Dict, Iterable, List, Optional, Tuple

import numpy as np

from . import gates as G
from .noise import noise_code
from .philox import philox4x32_10, seed_key
from .planner import Plan
from .statevector import apply_1q, apply_2q, full_unitary_1q, full_unitary_2q, zero_state
from .tree import FLAG_EPS, LeafResult, NoiseModel, TreeResult, sample_leaf

TAG_KRAUS = 3          # tags 3 (sub-locations 0..3) and 4 (4..7)
CH_TR_AMP, CH_TR_PHASE, CH_AD, CH_PD = 0, 1, 2, 3


@dataclass
class KrausModel:
    amp_damping: float = 0.0       # AD gamma (0.01)
    phase_damping: float = 0.0     # PD lambda (0.01)
    t1: float = 0.0                # TR T1 (0 = TR off); seconds
    t2: float = 0.0                # TR T2 (<= 2 T1)
    gate_time_1q: float = 0.0
    gate_time_2q: float = 0.0

    @property
    def enabled(self) -> bool:
        return self.amp_damping > 0 or self.phase_damping > 0 or self.t1 > 0


def ad_ops(g: float) -> List[np.ndarray]:
    return [np.array([[1.0, 0.0], [0.0, math.sqrt(1.0 - g)]], dtype=np.complex128),
            np.array([[0.0, math.sqrt(g)], [0.0, 0.0]], dtype=np.complex128)]


def pd_ops(l: float) -> List[np.ndarray]:
    return [np.array([[1.0, 0.0], [0.0, math.sqrt(1.0 - l)]], dtype=np.complex128),
            np.array([[0.0, 0.0], [0.0, math.sqrt(l)]], dtype=np.complex128)]


def tr_params(km: KrausModel, two: bool) -> Tuple[float, float]:
    """(g_T, l_T) of R32 for a gate of the given class."""
    t = km.gate_time_2q if two else km.gate_time_1q
    g = 1.0 - math.exp(-t / km.t1)
    l = 1.0 - math.exp(-2.0 * t / km.t2 + t / km.t1)
    return g, l


def channels(km: KrausModel, two: bool) -> List[Tuple[int, List[np.ndarray]]]:
    """The enabled channels in R33 order, as (c, Kraus list)."""
    out = []
    if km.t1 > 0:
        g, l = tr_params(km, two)
        out.append((CH_TR_AMP, ad_ops(g)))
        out.append((CH_TR_PHASE, pd_ops(l)))
    if km.amp_damping > 0:
        out.append((CH_AD, ad_ops(km.amp_damping)))
    if km.phase_damping > 0:
        out.append((CH_PD, pd_ops(km.phase_damping)))
    return out


def kraus_uniform(g: int, j: int, s: int, seed: int) -> float:
    """R34: r in [0, 1) for sub-location s of gate g at node instance j."""
    w = philox4x32_10((g, j & 0xFFFFFFFF, TAG_KRAUS + (s >> 2), j >> 32), seed_key(seed))
    return float(w[s & 3]) * 2.0 ** -32


def choose(psi: np.ndarray, n: int, q: int, ops: List[np.ndarray], r: float):
    """R35/R36: (new psi, chosen k, flagged)."""
    outs, cum, k_sel, flagged = [], 0.0, None, False
    for k, K in enumerate(ops):
        phi = apply_1q(psi, n, q, K)
        p = float(np.vdot(phi, phi).real)
        cum += p
        outs.append((phi, p))
        if abs(r - cum) < FLAG_EPS:
            flagged = True
        if k_sel is None and r < cum:
            k_sel = k
    if k_sel is None:                       # r beyond the total (rounding): the last non-zero
        k_sel = max(k for k, (_, p) in enumerate(outs) if p > 0.0)
        flagged = True
    phi, p = outs[k_sel]
    return phi / math.sqrt(p), k_sel, flagged


def apply_location(psi: np.ndarray, n: int, gate, g: int, j: int, seed: int, noise: NoiseModel,
                   km: KrausModel):
    """Gate g, its depolarizing Pauli (oracle.noise, R1/R8), then the Kraus
    channels of R33 on its qubits.  Returns (psi, flagged)."""
    kind, a, b, th, ph, la = gate
    two = kind in G.TWO_QUBIT_PRIMS
    if two:
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
    flagged = False
    qs = (a, b) if two else (a,)
    for c, ops in channels(km, two):
        for i, q in enumerate(qs):
            s = 2 * c + i
            psi, _, f = choose(psi, n, q, ops, kraus_uniform(g, j, s, seed))
            flagged |= f
    return psi, flagged


def run_slice(psi, n, lowered, g0, g1, j, seed, noise, km):
    flagged = False
    for g in range(g0, g1):
        psi, f = apply_location(psi, n, lowered[g], g, j, seed, noise, km)
        flagged |= f
    return psi, flagged


def simulate_tree(n: int, lowered, plan: Plan, noise: NoiseModel, km: KrausModel, seed: int,
                  top_range: Optional[Tuple[int, int]] = None,
                  dump: Iterable[Tuple[int, int]] = ()) -> TreeResult:
    """DFS with state reuse (§3) of the trajectories with Kraus channels; a leaf is
    flagged if its sampling draw (R9) or any Kraus decision on its path (R36) is."""
    dump = set(dump)
    res = TreeResult()
    A, B, L = plan.arities, plan.boundaries, len(plan.arities)

    def node(d, j, parent, pflag):
        psi, f = run_slice(parent.copy(), n, lowered, B[d], B[d + 1], j, seed, noise, km)
        f |= pflag
        if (d, j) in dump:
            res.dumps[(d, j)] = psi.copy()
        if d == L - 1:
            r = sample_leaf(psi, n, j, seed, noise)
            res.leaves[j] = LeafResult(r.x, r.outcome, r.flagged or f, r.u)
            return
        for br in range(A[d + 1]):
            node(d + 1, j * A[d + 1] + br, psi, f)

    lo, hi = top_range if top_range is not None else (0, A[0])
    for j0 in range(lo, hi):
        node(0, j0, zero_state(n), False)
    return res


def simulate_leaf_flat(n, lowered, plan: Plan, noise: NoiseModel, km: KrausModel, seed: int, leaf: int):
    """Per-leaf flat recompute with inherited keys (must equal the DFS exactly)."""
    A = plan.arities
    anc = [0] * len(A)
    j = leaf
    for d in range(len(A) - 1, -1, -1):
        anc[d] = j
        j //= A[d]
    psi, fl = zero_state(n), False
    for d, jd in enumerate(anc):
        psi, f = run_slice(psi, n, lowered, plan.boundaries[d], plan.boundaries[d + 1], jd, seed, noise, km)
        fl |= f
    r = sample_leaf(psi, n, leaf, seed, noise)
    return LeafResult(r.x, r.outcome, r.flagged or fl, r.u), psi


# ---------------------------------------------------------------- density-matrix pins
def evolve_dm(n: int, lowered, p1: float, p2: float, km: KrausModel) -> np.ndarray:
    """rho after the circuit with the depolarizing channel (as oracle.density) and the Kraus
    channels of R31-R33 applied as maps rho -> sum_k K_k rho K_k^dag (Eq.1)."""
    import itertools
    dim = 2 ** n
    rho = np.zeros((dim, dim), dtype=np.complex128)
    rho[0, 0] = 1.0
    for (kind, a, b, th, ph, la) in lowered:
        two = kind in G.TWO_QUBIT_PRIMS
        if two:
            u = full_unitary_2q(n, a, b, G.matrix_2q(kind))
            rho = u @ rho @ u.conj().T
            acc = np.zeros_like(rho)
            for pa, pb in itertools.product(range(4), range(4)):
                if pa or pb:
                    op = full_unitary_1q(n, a, G.PAULI[pa]) @ full_unitary_1q(n, b, G.PAULI[pb])
                    acc += op @ rho @ op.conj().T
            rho = (1.0 - p2) * rho + (p2 / 15.0) * acc
        else:
            u = full_unitary_1q(n, a, G.matrix_1q(kind, th, ph, la))
            rho = u @ rho @ u.conj().T
            acc = np.zeros_like(rho)
            for pa in (1, 2, 3):
                op = full_unitary_1q(n, a, G.PAULI[pa])
                acc += op @ rho @ op.conj().T
            rho = (1.0 - p1) * rho + (p1 / 3.0) * acc
        for c, ops in channels(km, two):
            for q in ((a, b) if two else (a,)):
                new = np.zeros_like(rho)
                for K in ops:
                    op = full_unitary_1q(n, q, K)
                    new += op @ rho @ op.conj().T
                rho = new
    return rho


def enumerate_branches(n: int, lowered, km: KrausModel) -> np.ndarray:
    """Brute force without the sampling rule: sum over every sequence of Kraus choices of
    the unnormalised K..K psi psi^dag K^dag..K^dag (no depolarizing), which must equal
    evolve_dm(p1 = p2 = 0) -- the trajectory ensemble's definition."""
    branches = [zero_state(n)]
    for (kind, a, b, th, ph, la) in lowered:
        two = kind in G.TWO_QUBIT_PRIMS
        if two:
            branches = [apply_2q(v, n, a, b, G.matrix_2q(kind)) for v in branches]
        else:
            branches = [apply_1q(v, n, a, G.matrix_1q(kind, th, ph, la)) for v in branches]
        for c, ops in channels(km, two):
            for q in ((a, b) if two else (a,)):
                branches = [apply_1q(v, n, q, K) for v in branches for K in ops]
    rho = np.zeros((2 ** n, 2 ** n), dtype=np.complex128)
    for v in branches:
        rho += np.outer(v, v.conj())
    return rho
