"""Accuracy metrics of the tree method (the paper's §4.1 figure of merit).

Eq.6:  F_s(P, Q) = (sum_x sqrt(P(x) Q(x)))^2
Eq.7:  F(P_ideal, P_out) = (F_s(P_ideal, P_out) - F_s(P_ideal, P_uni)) / (1 - F_s(P_ideal, P_uni))

The paper compares the normalized fidelity of TQSim's output with that of the flat
per-shot baseline ("closely matched normalized fidelity values show the baseline
result and TQSim result are interchangeable"; max difference 0.016).
Host-side arithmetic on histograms; the distributions come from the GPU path.
"""
from __future__ import annotations

from typing import Dict

import numpy as np


def distribution(counts: Dict[int, int], n_qubits: int) -> np.ndarray:
    """Histogram {bitstring: count} -> probability vector of length 2^n."""
    p = np.zeros(1 << n_qubits)
    total = 0
    for x, c in counts.items():
        p[int(x)] += c
        total += c
    if total <= 0:
        raise ValueError("empty histogram")
    return p / total


def hellinger_fidelity(p: np.ndarray, q: np.ndarray) -> float:
    """Eq.6: the squared Bhattacharyya coefficient of two distributions."""
    return float(np.dot(np.sqrt(np.asarray(p, float)), np.sqrt(np.asarray(q, float))) ** 2)


def normalized_fidelity(p_ideal: np.ndarray, p_out: np.ndarray) -> float:
    """Eq.7: 0 for a uniform output, 1 for the ideal one (undefined if P_ideal is uniform)."""
    p_ideal = np.asarray(p_ideal, float)
    f_uni = float(np.sum(np.sqrt(p_ideal / p_ideal.size)) ** 2)
    if not (1.0 - f_uni > 1e-12):
        raise ValueError("normalized fidelity is undefined for a uniform ideal distribution")
    return (hellinger_fidelity(p_ideal, p_out) - f_uni) / (1.0 - f_uni)
