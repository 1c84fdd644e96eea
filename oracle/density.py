"""Density-matrix evolution -- oracle copy, brute-force pin only (test
infrastructure; tiny n).

rho = sum_i p_i |psi_i><psi_i| (Eq.1).  Gates act as rho <- U rho U^dag
with U the dense Kronecker-product operator; the depolarizing channel after a
gate (readings R1/R2) is
  1q:  rho <- (1-p) rho + p/3  sum_{P in X,Y,Z} P rho P
  2q:  rho <- (1-p) rho + p/15 sum_{(P,Q) != (I,I)} (P⊗Q) rho (P⊗Q)^dag
and readout error acts on the diagonal as independent bit flips.
"""
from __future__ import annotations

import itertools

import numpy as np

from . import gates as G
from .statevector import full_unitary_1q, full_unitary_2q


def evolve(n: int, lowered, p1: float, p2: float) -> np.ndarray:
    dim = 2 ** n
    rho = np.zeros((dim, dim), dtype=np.complex128)
    rho[0, 0] = 1.0
    for (kind, a, b, th, ph, la) in lowered:
        if kind in G.TWO_QUBIT_PRIMS:
            u = full_unitary_2q(n, a, b, G.matrix_2q(kind))
            rho = u @ rho @ u.conj().T
            acc = np.zeros_like(rho)
            for pa, pb in itertools.product(range(4), range(4)):
                if pa == 0 and pb == 0:
                    continue
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
    return rho


def readout_distribution(prob: np.ndarray, n: int, p01: float, p10: float) -> np.ndarray:
    """Apply independent classical bit flips (P(0->1)=p01, P(1->0)=p10) to a distribution."""
    out = np.zeros_like(prob)
    for x in range(2 ** n):
        for y in range(2 ** n):
            w = 1.0
            for b in range(n):
                xb, yb = (x >> b) & 1, (y >> b) & 1
                if xb == 0:
                    w *= p01 if yb == 1 else 1.0 - p01
                else:
                    w *= p10 if yb == 0 else 1.0 - p10
            out[y] += w * prob[x]
    return out
