"""Fidelity metrics -- oracle copy (test infrastructure only; pinned by closed forms and
invariants in tests/test_metrics.py).

Eq.6:  F_s(P, Q) = (sum_x sqrt(P(x) Q(x)))^2
Eq.7:  F(P_ideal, P_out) = (F_s(P_ideal, P_out) - F_s(P_ideal, P_uni))
                                        / (1 - F_s(P_ideal, P_uni))
"""
from __future__ import annotations

import numpy as np


def fidelity(p_ideal: np.ndarray, p_out: np.ndarray) -> float:
    return float(np.sum(np.sqrt(p_ideal * p_out)) ** 2)


def normalized_fidelity(p_ideal: np.ndarray, p_out: np.ndarray) -> float:
    uni = np.full_like(p_ideal, 1.0 / p_ideal.size)
    fu = fidelity(p_ideal, uni)
    return (fidelity(p_ideal, p_out) - fu) / (1.0 - fu)
