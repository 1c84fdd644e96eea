"""Circuit / workload generators (inputs only; see package docstring).

A circuit is a list of gate tuples ``(kind, q0, q1, theta, phi, lam)`` where
``kind`` is one of GATE_KINDS (OpenQASM-2 style names), ``q1`` is -1 for
single-qubit gates, and unused angles are 0.0.  For ``cp`` the control is q0
and the target q1; for ``cx``/``cz`` q0 is the control.

Config recipes follow BASELINE.json ``configs`` (C1..C5) and SURVEY.md §8(c)
row 23/24 (seed 0 everywhere; numpy ``default_rng(0)`` draws).  The generated
configs are frozen as JSON under ``configs/`` by ``workloads/freeze.py`` so that
neither side depends on numpy's stream stability.
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

# Order matters: it is the tqsim_gate_kind enum order of include/tqsim.h.
GATE_KINDS = ("x", "y", "z", "h", "s", "sdg", "t", "tdg", "rx", "ry", "rz",
              "p", "u", "cx", "cz", "swap", "cp")
TWO_QUBIT = frozenset(("cx", "cz", "swap", "cp"))

Gate = Tuple[str, int, int, float, float, float]

_CONFIG_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "configs")


def g1(kind: str, q: int, theta: float = 0.0, phi: float = 0.0, lam: float = 0.0) -> Gate:
    return (kind, int(q), -1, float(theta), float(phi), float(lam))


def g2(kind: str, a: int, b: int, theta: float = 0.0) -> Gate:
    return (kind, int(a), int(b), float(theta), 0.0, 0.0)


@dataclass
class Circuit:
    n_qubits: int
    gates: List[Gate]


@dataclass
class Workload:
    name: str
    circuit: Circuit
    p1: float
    p2: float
    readout_p01: float
    readout_p10: float
    shots: int
    arities: Optional[List[int]]          # None = auto (DCP)
    seed: int = 0
    copy_cost_gates: float = 10.0
    meta: dict = field(default_factory=dict)

    def to_json(self) -> dict:
        return {
            "name": self.name, "n_qubits": self.circuit.n_qubits,
            "gates": [list(g) for g in self.circuit.gates],
            "noise": {"p1": self.p1, "p2": self.p2,
                      "readout_p01": self.readout_p01, "readout_p10": self.readout_p10},
            "shots": self.shots, "arities": self.arities, "seed": self.seed,
            "copy_cost_gates": self.copy_cost_gates, "meta": self.meta,
        }

    @staticmethod
    def from_json(d: dict) -> "Workload":
        gates = [(str(g[0]), int(g[1]), int(g[2]), float(g[3]), float(g[4]), float(g[5]))
                 for g in d["gates"]]
        nz = d["noise"]
        return Workload(d["name"], Circuit(int(d["n_qubits"]), gates), float(nz["p1"]),
                        float(nz["p2"]), float(nz["readout_p01"]), float(nz["readout_p10"]),
                        int(d["shots"]), None if d["arities"] is None else [int(a) for a in d["arities"]],
                        int(d["seed"]), float(d["copy_cost_gates"]), d.get("meta", {}))


# ---------------------------------------------------------------- circuits
def qft_gates(n: int) -> List[Gate]:
    """Textbook QFT (SURVEY §8(c) 'QFT construction'): for j = n-1..0: H(j);
    for m = j-1..0: CP(pi/2^(j-m)) control m target j; then SWAP(i, n-1-i)."""
    out: List[Gate] = []
    for j in range(n - 1, -1, -1):
        out.append(g1("h", j))
        for m in range(j - 1, -1, -1):
            out.append(g2("cp", m, j, math.pi / (2 ** (j - m))))
    for i in range(n // 2):
        out.append(g2("swap", i, n - 1 - i))
    return out


def basis_prep_gates(x: int, n: int) -> List[Gate]:
    """X on every set bit of x (little endian: qubit q = bit q), ascending."""
    return [g1("x", q) for q in range(n) if (x >> q) & 1]


def ghz_gates(n: int) -> List[Gate]:
    return [g1("h", 0)] + [g2("cx", i, i + 1) for i in range(n - 1)]


def brickwork_gates(n: int, layers: int, rng: np.random.Generator) -> List[Gate]:
    """C3: per layer a U3 on every qubit (angles U[0,2pi)^3, layer-major,
    qubit-minor) then CX on even pairs (even layer) / odd pairs (odd layer),
    control = lower index."""
    out: List[Gate] = []
    for layer in range(layers):
        for q in range(n):
            th, ph, la = rng.uniform(0.0, 2 * math.pi, 3)
            out.append(g1("u", q, th, ph, la))
        start = 0 if layer % 2 == 0 else 1
        for a in range(start, n - 1, 2):
            out.append(g2("cx", a, a + 1))
    return out


def random_3_regular_edges(n: int, rng: np.random.Generator) -> List[Tuple[int, int]]:
    """Uniform-ish random simple 3-regular graph by the configuration model
    with rejection (no self loops / multi-edges)."""
    assert (3 * n) % 2 == 0
    while True:
        stubs = np.repeat(np.arange(n), 3)
        perm = rng.permutation(stubs)
        edges = set()
        ok = True
        for i in range(0, len(perm), 2):
            a, b = int(perm[i]), int(perm[i + 1])
            if a == b:
                ok = False
                break
            e = (min(a, b), max(a, b))
            if e in edges:
                ok = False
                break
            edges.add(e)
        if ok:
            return sorted(edges)


def qaoa_gates(n: int, edges: Sequence[Tuple[int, int]], gammas: Sequence[float],
               betas: Sequence[float]) -> List[Gate]:
    """MaxCut QAOA: H layer, then per layer for each edge CX(u,v) RZ(2g)(v) CX(u,v)
    (RZZ lowered to CX-RZ-CX, BASELINE config 4), then RX(2b) on every qubit."""
    out: List[Gate] = [g1("h", q) for q in range(n)]
    for gm, bt in zip(gammas, betas):
        for (u, v) in edges:
            out.append(g2("cx", u, v))
            out.append(g1("rz", v, 2 * gm))
            out.append(g2("cx", u, v))
        for q in range(n):
            out.append(g1("rx", q, 2 * bt))
    return out


def hea_gates(n: int, layers: int, angles: np.ndarray) -> List[Gate]:
    """C5: GHZ prep (H + CX ladder) then `layers` x [RY per qubit + CX ladder]."""
    out = ghz_gates(n)
    for layer in range(layers):
        for q in range(n):
            out.append(g1("ry", q, float(angles[layer, q])))
        for i in range(n - 1):
            out.append(g2("cx", i, i + 1))
    return out


def inverse_qft_gates(qubits: Sequence[int]) -> List[Gate]:
    """The textbook QFT on `qubits` (qft_gates' order: H(j), CP(pi/2^(j-m)) control m target
    j, then the SWAPs), reversed with negated angles."""
    m = len(qubits)
    fwd: List[Gate] = []
    for j in range(m - 1, -1, -1):
        fwd.append(g1("h", qubits[j]))
        for k in range(j - 1, -1, -1):
            fwd.append(g2("cp", qubits[k], qubits[j], math.pi / (2 ** (j - k))))
    for i in range(m // 2):
        fwd.append(g2("swap", qubits[i], qubits[m - 1 - i]))
    return [(k, a, b, -th, ph, la) for (k, a, b, th, ph, la) in reversed(fwd)]


def qpe_gates(n_count: int, phase: float) -> List[Gate]:
    """Quantum phase estimation of U = P(2 pi phase) on its eigenstate |1> (the paper's QPE_9:
    8 counting qubits + 1 target, phase 1/3, "cannot be exactly represented by a 9-bit
    fixed-point number"): counting qubits 0..n_count-1, target n_count;
    X(target), H(counting), CP(2 pi phase 2^k) control k -> target, inverse QFT(counting).
    The counting register then reads ~ phase * 2^n_count."""
    t = n_count
    out: List[Gate] = [g1("x", t)] + [g1("h", q) for q in range(n_count)]
    for k in range(n_count):
        out.append(g2("cp", k, t, 2 * math.pi * phase * (2 ** k)))
    return out + inverse_qft_gates(list(range(n_count)))


def bv_gates(n: int, hidden: int) -> List[Gate]:
    """Bernstein-Vazirani on n qubits (n-1 data + ancilla n-1; the paper's BV_10 with the
    hidden string all ones): X + H on the ancilla, H on the data, CX(data_i -> ancilla)
    for every set bit of `hidden`, H on all -- the ideal output is the single bitstring
    hidden + 2^(n-1) (the ancilla returns to |1>)."""
    a = n - 1
    out: List[Gate] = [g1("x", a), g1("h", a)] + [g1("h", q) for q in range(a)]
    out += [g2("cx", q, a) for q in range(a) if (hidden >> q) & 1]
    return out + [g1("h", q) for q in range(n)]


def random_circuit(n: int, n_gates: int, rng: np.random.Generator,
                   kinds: Sequence[str] = GATE_KINDS) -> List[Gate]:
    """Random gate list over every kind (for parity/unit tests)."""
    out: List[Gate] = []
    for _ in range(n_gates):
        k = kinds[int(rng.integers(0, len(kinds)))]
        if k in TWO_QUBIT:
            if n < 2:
                continue
            a, b = rng.choice(n, size=2, replace=False)
            out.append(g2(k, int(a), int(b), float(rng.uniform(0, 2 * math.pi))))
        else:
            th, ph, la = rng.uniform(0, 2 * math.pi, 3)
            out.append(g1(k, int(rng.integers(0, n)), th, ph, la))
    return out


# ---------------------------------------------------------------- configs
def make_config(name: str) -> Workload:
    """Build one BASELINE.json config from its recipe (seed 0)."""
    if name == "c1_qft5":
        n = 5
        gates = basis_prep_gates(0b00101, n) + qft_gates(n)   # |10100>: X on q0, q2
        return Workload(name, Circuit(n, gates), 1e-3, 1e-2, 1e-2, 1e-2, 1000, [10, 100], 0,
                        meta={"basis_x": 5})
    if name == "c2_qft15":
        n = 15
        rng = np.random.default_rng(0)
        x = int(rng.integers(0, 2 ** n))
        gates = basis_prep_gates(x, n) + qft_gates(n)
        return Workload(name, Circuit(n, gates), 1e-3, 1e-2, 1e-2, 1e-2, 10000, None, 0,
                        meta={"basis_x": x})
    if name == "c3_brick20":
        n = 20
        rng = np.random.default_rng(0)
        gates = brickwork_gates(n, 20, rng)
        return Workload(name, Circuit(n, gates), 1e-3, 1e-2, 1e-2, 1e-2, 10000, None, 0)
    if name == "c4_qaoa24":
        n = 24
        rng = np.random.default_rng(0)
        edges = random_3_regular_edges(n, rng)
        g0, b0, g1_, b1 = (float(v) for v in rng.uniform(0.0, math.pi, 4))
        gates = qaoa_gates(n, edges, [g0, g1_], [b0, b1])
        return Workload(name, Circuit(n, gates), 1e-3, 1e-2, 0.0, 0.0, 8192, None, 0,
                        meta={"edges": edges, "gammas": [g0, g1_], "betas": [b0, b1]})
    if name == "c5_hea28":
        n = 28
        rng = np.random.default_rng(0)
        angles = rng.uniform(0.0, 2 * math.pi, (4, n))
        gates = hea_gates(n, 4, angles)
        return Workload(name, Circuit(n, gates), 5e-4, 5e-3, 1e-2, 1e-2, 32768, None, 0)
    raise KeyError(name)


MONOMIAL_1Q = ("x", "y", "z", "s", "sdg", "t", "tdg", "p", "rz")


def monomial_brickwork_gates(n: int, layers: int, rng: np.random.Generator) -> List[Gate]:
    """C3-shaped brickwork whose 1q gates are monomial matrices (one non-zero per
    row/column), so every noisy trajectory of |0..0> stays 1-sparse."""
    out: List[Gate] = []
    for layer in range(layers):
        for q in range(n):
            k = MONOMIAL_1Q[int(rng.integers(0, len(MONOMIAL_1Q)))]
            out.append(g1(k, q, float(rng.uniform(0.0, 2 * math.pi))))
        start = 0 if layer % 2 == 0 else 1
        for a in range(start, n - 1, 2):
            out.append(g2("cx", a, a + 1))
    return out


def make_variant(name: str) -> Workload:
    """Structured full-size variants of C3/C4/C5 (SURVEY §8(c) "What pins each
    part"): same widths, gate counts, noise and shots as the configs, with the
    structure changed so the oracle can predict every leaf at full size."""
    if name == "c3_brick20_monomial":
        base = make_config("c3_brick20")
        gates = monomial_brickwork_gates(20, 20, np.random.default_rng(1))
        return Workload(name, Circuit(20, gates), base.p1, base.p2, base.readout_p01,
                        base.readout_p10, base.shots, None, 0)
    if name == "c4_qaoa24_beta0":
        base = make_config("c4_qaoa24")
        m = base.meta
        gates = qaoa_gates(24, m["edges"], m["gammas"], [0.0, 0.0])
        return Workload(name, Circuit(24, gates), base.p1, base.p2, 0.0, 0.0, base.shots, None, 0,
                        meta={"edges": m["edges"], "gammas": m["gammas"], "betas": [0.0, 0.0]})
    if name == "c5_hea28_ry0":
        base = make_config("c5_hea28")
        gates = hea_gates(28, 4, np.zeros((4, 28)))
        return Workload(name, Circuit(28, gates), base.p1, base.p2, base.readout_p01,
                        base.readout_p10, base.shots, None, 0)
    raise KeyError(name)


def config_names() -> List[str]:
    return ["c1_qft5", "c2_qft15", "c3_brick20", "c4_qaoa24", "c5_hea28"]


def load_config(name: str) -> Workload:
    """Load a frozen config JSON (configs/<name>.json); falls back to the recipe."""
    path = os.path.join(_CONFIG_DIR, name + ".json")
    if os.path.exists(path):
        with open(path) as f:
            return Workload.from_json(json.load(f))
    return make_config(name)
