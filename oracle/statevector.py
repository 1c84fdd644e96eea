"""Plain statevector operations -- oracle copy (test infrastructure only).

"An ideal quantum circuit simulator multiplies the matrix representations of
the quantum gates in the given circuit to the initial Statevector" (P:139
§2.3).  The state is a length-2^n complex128 vector; basis index
x = sum_q bit_q * 2^q (little endian).

The vector is viewed as an n-axis tensor T[i_{n-1}, ..., i_0] (C order), so
qubit q lives on axis n-1-q; a k-qubit matrix is contracted on those axes with
np.tensordot.  No blocking, fusion or reordering.
"""
from __future__ import annotations

import numpy as np


def zero_state(n: int) -> np.ndarray:
    psi = np.zeros(2 ** n, dtype=np.complex128)
    psi[0] = 1.0
    return psi


def apply_1q(psi: np.ndarray, n: int, q: int, m: np.ndarray) -> np.ndarray:
    """psi <- (I ⊗ .. ⊗ m_q ⊗ .. ⊗ I) psi."""
    t = psi.reshape((2,) * n)
    ax = n - 1 - q
    out = np.tensordot(m, t, axes=([1], [ax]))      # new axis 0 = qubit q
    out = np.moveaxis(out, 0, ax)
    return np.ascontiguousarray(out).reshape(-1)


def apply_2q(psi: np.ndarray, n: int, a: int, b: int, m4: np.ndarray) -> np.ndarray:
    """Apply a 4x4 matrix written in the local basis |bit_a bit_b> (a more significant)."""
    t = psi.reshape((2,) * n)
    ax_a, ax_b = n - 1 - a, n - 1 - b
    u = m4.reshape(2, 2, 2, 2)                      # u[a', b', a, b]
    out = np.tensordot(u, t, axes=([2, 3], [ax_a, ax_b]))
    out = np.moveaxis(out, [0, 1], [ax_a, ax_b])
    return np.ascontiguousarray(out).reshape(-1)


def full_unitary_1q(n: int, q: int, m: np.ndarray) -> np.ndarray:
    """Dense 2^n x 2^n operator by Kronecker products (used only by pins / DM)."""
    op = np.array([[1.0 + 0j]])
    for k in range(n - 1, -1, -1):                  # most significant qubit first
        op = np.kron(op, m if k == q else np.eye(2))
    return op


def full_unitary_2q(n: int, a: int, b: int, m4: np.ndarray) -> np.ndarray:
    """Dense operator for a 2q matrix by explicit basis enumeration (independent of tensordot)."""
    dim = 2 ** n
    op = np.zeros((dim, dim), dtype=np.complex128)
    for x in range(dim):
        ba, bb = (x >> a) & 1, (x >> b) & 1
        col = (ba << 1) | bb
        for row in range(4):
            amp = m4[row, col]
            if amp == 0:
                continue
            na, nb = row >> 1, row & 1
            y = (x & ~((1 << a) | (1 << b))) | (na << a) | (nb << b)
            op[y, x] += amp
    return op
