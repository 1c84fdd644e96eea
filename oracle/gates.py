"""Gate matrices and lowering -- oracle copy (test infrastructure only).

The paper fixes the gate set only loosely ("X, Y, Z, Hadamard (H), and CNOT",
P:117 §2.2; gates are "matrix representations" multiplied into the
Statevector, §2.3).  Global phases matter for amplitude parity, so the
standard OpenQASM-2 forms of SURVEY §8(c) "Gate matrices" are used (reading
rows 4-5 of the ambiguity register, R4/R5):

  H = [[1,1],[1,-1]]/sqrt2   X, Y = [[0,-i],[i,0]], Z   S = diag(1,i)  T = diag(1,e^{i pi/4})
  RX(t) = [[c,-is],[-is,c]]  RY(t) = [[c,-s],[s,c]]  RZ(t) = diag(e^{-it/2}, e^{it/2})
  P(l) = diag(1, e^{il})     U(t,p,l) = [[c, -e^{il} s], [e^{ip} s, e^{i(p+l)} c]]
  with c = cos(t/2), s = sin(t/2).

Two-qubit matrices are written in the textbook basis |a b> with a = q0 the
more significant local bit: CX(a,b) flips b when a = 1; CZ = diag(1,1,1,-1).

Lowering (one noise location per LOWERED gate, row 1):
  CP(t; a, b)  -> P(t/2) a, CX(a,b), P(-t/2) b, CX(a,b), P(t/2) b
  SWAP(a, b)   -> CX(a,b), CX(b,a), CX(a,b)
"""
from __future__ import annotations

import math
from typing import List, Sequence, Tuple

import numpy as np

SQ2 = 1.0 / math.sqrt(2.0)

ONE_QUBIT = ("x", "y", "z", "h", "s", "sdg", "t", "tdg", "rx", "ry", "rz", "p", "u")
TWO_QUBIT_PRIMS = ("cx", "cz")

PAULI = {
    0: np.array([[1, 0], [0, 1]], dtype=np.complex128),     # I
    1: np.array([[0, 1], [1, 0]], dtype=np.complex128),     # X
    2: np.array([[0, -1j], [1j, 0]], dtype=np.complex128),  # Y
    3: np.array([[1, 0], [0, -1]], dtype=np.complex128),    # Z
}


def matrix_1q(kind: str, theta: float = 0.0, phi: float = 0.0, lam: float = 0.0) -> np.ndarray:
    c = math.cos(theta / 2.0)
    s = math.sin(theta / 2.0)
    if kind == "x":
        m = [[0, 1], [1, 0]]
    elif kind == "y":
        m = [[0, -1j], [1j, 0]]
    elif kind == "z":
        m = [[1, 0], [0, -1]]
    elif kind == "h":
        m = [[SQ2, SQ2], [SQ2, -SQ2]]
    elif kind == "s":
        m = [[1, 0], [0, 1j]]
    elif kind == "sdg":
        m = [[1, 0], [0, -1j]]
    elif kind == "t":
        m = [[1, 0], [0, complex(math.cos(math.pi / 4), math.sin(math.pi / 4))]]
    elif kind == "tdg":
        m = [[1, 0], [0, complex(math.cos(math.pi / 4), -math.sin(math.pi / 4))]]
    elif kind == "rx":
        m = [[c, -1j * s], [-1j * s, c]]
    elif kind == "ry":
        m = [[c, -s], [s, c]]
    elif kind == "rz":
        m = [[complex(math.cos(theta / 2), -math.sin(theta / 2)), 0],
             [0, complex(math.cos(theta / 2), math.sin(theta / 2))]]
    elif kind == "p":
        # P(lambda): the angle is carried in `theta` for p/rz/rx/ry (single-angle gates)
        m = [[1, 0], [0, complex(math.cos(theta), math.sin(theta))]]
    elif kind == "u":
        eil = complex(math.cos(lam), math.sin(lam))
        eip = complex(math.cos(phi), math.sin(phi))
        eipl = complex(math.cos(phi + lam), math.sin(phi + lam))
        m = [[c, -eil * s], [eip * s, eipl * c]]
    else:
        raise ValueError("not a 1q gate: " + kind)
    return np.array(m, dtype=np.complex128)


def matrix_2q(kind: str) -> np.ndarray:
    if kind == "cx":
        return np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], dtype=np.complex128)
    if kind == "cz":
        return np.diag([1, 1, 1, -1]).astype(np.complex128)
    raise ValueError("not a 2q primitive: " + kind)


LoweredGate = Tuple[str, int, int, float, float, float]


def lower(gates: Sequence[Tuple]) -> List[LoweredGate]:
    """Lower a workload gate list to primitives {1q kinds, cx, cz}."""
    out: List[LoweredGate] = []
    for (k, a, b, th, ph, la) in gates:
        if k == "cp":
            out.append(("p", a, -1, th / 2.0, 0.0, 0.0))
            out.append(("cx", a, b, 0.0, 0.0, 0.0))
            out.append(("p", b, -1, -th / 2.0, 0.0, 0.0))
            out.append(("cx", a, b, 0.0, 0.0, 0.0))
            out.append(("p", b, -1, th / 2.0, 0.0, 0.0))
        elif k == "swap":
            out.append(("cx", a, b, 0.0, 0.0, 0.0))
            out.append(("cx", b, a, 0.0, 0.0, 0.0))
            out.append(("cx", a, b, 0.0, 0.0, 0.0))
        elif k in ("cx", "cz"):
            out.append((k, a, b, 0.0, 0.0, 0.0))
        else:
            out.append((k, a, -1, th, ph, la))
    return out


def is_two_qubit(g: LoweredGate) -> bool:
    return g[0] in TWO_QUBIT_PRIMS
