"""Pins for oracle.gates and oracle.statevector (no GPU).

Each pin is independent of the code it checks: algebraic identities of the
textbook matrices, basis-state truth tables computed with integer bit
operations, and Kronecker-product / explicit-enumeration dense operators.
"""
import cmath
import math

import numpy as np
import pytest

from oracle import gates as G
from oracle.statevector import apply_1q, apply_2q, full_unitary_1q, full_unitary_2q, zero_state

ANG = (0.3, 1.1, -2.2)


def mats():
    for k in G.ONE_QUBIT:
        yield k, G.matrix_1q(k, *ANG)


def test_unitarity():
    for k, m in mats():
        assert np.allclose(m.conj().T @ m, np.eye(2), atol=1e-15), k
    for k in G.TWO_QUBIT_PRIMS:
        m = G.matrix_2q(k)
        assert np.allclose(m.conj().T @ m, np.eye(4), atol=0)


def test_algebraic_identities():
    X, Y, Z = G.PAULI[1], G.PAULI[2], G.PAULI[3]
    M = G.matrix_1q
    assert np.allclose(X @ Y, 1j * Z)                      # Pauli algebra fixes Y's sign
    assert np.allclose(M("h") @ M("h"), np.eye(2))
    assert np.allclose(M("h") @ X @ M("h"), Z)
    assert np.allclose(M("s") @ M("s"), Z)
    assert np.allclose(M("t") @ M("t"), M("s"))
    assert np.allclose(M("s") @ M("sdg"), np.eye(2))
    assert np.allclose(M("t") @ M("tdg"), np.eye(2))
    for th in (0.0, 0.7, math.pi, 5.0):
        c, s = math.cos(th / 2), math.sin(th / 2)
        assert np.allclose(M("rx", th), c * np.eye(2) - 1j * s * X)     # exp(-i th X/2)
        assert np.allclose(M("ry", th), c * np.eye(2) - 1j * s * Y)
        assert np.allclose(M("rz", th), c * np.eye(2) - 1j * s * Z)
        assert np.allclose(M("p", th), cmath.exp(1j * th / 2) * M("rz", th))
        assert np.allclose(M("u", th, 0.0, 0.0), M("ry", th))
    assert np.allclose(M("u", math.pi, 0.0, math.pi), X)
    # U(t,p,l) = e^{i(p+l)/2} RZ(p) RY(t) RZ(l)  (OpenQASM 2 definition)
    t, p, l = ANG
    assert np.allclose(M("u", t, p, l),
                       cmath.exp(1j * (p + l) / 2) * M("rz", p) @ M("ry", t) @ M("rz", l))


def test_cx_cz_truth_tables_by_bits():
    n = 3
    for a, b in ((0, 1), (2, 0), (1, 2)):
        for x in range(2 ** n):
            psi = np.zeros(2 ** n, complex)
            psi[x] = 1
            out = apply_2q(psi, n, a, b, G.matrix_2q("cx"))
            y = x ^ (((x >> a) & 1) << b)
            assert out[y] == 1 and np.count_nonzero(out) == 1
            outz = apply_2q(psi, n, a, b, G.matrix_2q("cz"))
            sign = -1 if ((x >> a) & 1) and ((x >> b) & 1) else 1
            assert outz[x] == sign


def test_apply_1q_matches_kron_and_bit_rule():
    rng = np.random.default_rng(0)
    n = 4
    psi = rng.normal(size=16) + 1j * rng.normal(size=16)
    for q in range(n):
        for k, m in mats():
            ref = full_unitary_1q(n, q, m) @ psi
            assert np.allclose(apply_1q(psi, n, q, m), ref, atol=1e-14)
        # bit rule: X on qubit q maps index x to x ^ (1<<q)
        xs = apply_1q(psi, n, q, G.PAULI[1])
        assert np.array_equal(xs, psi[np.arange(16) ^ (1 << q)])


def test_apply_2q_matches_enumeration():
    rng = np.random.default_rng(1)
    n = 4
    psi = rng.normal(size=16) + 1j * rng.normal(size=16)
    m4 = rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4))
    for a in range(n):
        for b in range(n):
            if a != b:
                ref = full_unitary_2q(n, a, b, m4) @ psi
                assert np.allclose(apply_2q(psi, n, a, b, m4), ref, atol=1e-13)


def test_lowering_cp_and_swap():
    n = 3
    for (a, b) in ((0, 2), (2, 1)):
        th = 0.9
        op = np.eye(8, dtype=complex)
        for (k, qa, qb, t, p, l) in G.lower([("cp", a, b, th, 0, 0)]):
            if k == "cx":
                op = full_unitary_2q(n, qa, qb, G.matrix_2q("cx")) @ op
            else:
                op = full_unitary_1q(n, qa, G.matrix_1q(k, t, p, l)) @ op
        want = np.diag([cmath.exp(1j * th) if ((x >> a) & 1 and (x >> b) & 1) else 1 for x in range(8)])
        assert np.allclose(op, want, atol=1e-15)
        op = np.eye(8, dtype=complex)
        for (k, qa, qb, t, p, l) in G.lower([("swap", a, b, 0, 0, 0)]):
            op = full_unitary_2q(n, qa, qb, G.matrix_2q("cx")) @ op
        perm = np.zeros((8, 8))
        for x in range(8):
            ba, bb = (x >> a) & 1, (x >> b) & 1
            y = (x & ~((1 << a) | (1 << b))) | (bb << a) | (ba << b)
            perm[y, x] = 1
        assert np.array_equal(op, perm)


def test_lowered_gate_counts():
    from workloads import load_config
    # QFT_n lowered: n H + 5 n(n-1)/2 (CP) + 3 floor(n/2) (SWAP) + prep X's
    for name, n, nx in (("c1_qft5", 5, 2), ("c2_qft15", 15, 8)):
        w = load_config(name)
        low = G.lower(w.circuit.gates)
        assert len(low) == n + 5 * n * (n - 1) // 2 + 3 * (n // 2) + nx
    assert len(G.lower(load_config("c3_brick20").circuit.gates)) == 590
    assert len(G.lower(load_config("c4_qaoa24").circuit.gates)) == 288
    assert len(G.lower(load_config("c5_hea28").circuit.gates)) == 248
