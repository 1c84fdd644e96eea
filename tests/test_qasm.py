"""OpenQASM 2.0 subset ingestion (SPEC circuit-ir S:52-60) through
the C ABI (tqsim_parse_qasm) -- host only, no GPU."""
import math

import pytest

import paper_2203_13892_b200.tqsim as T
from workloads import qft_gates


def parse(text):
    return T.tqsim_parse_qasm(text)


def to_qasm(n, gates):
    """Test-side writer (repr keeps every angle exact)."""
    lines = ["OPENQASM 2.0;", 'include "qelib1.inc";', "qreg q[%d];" % n, "creg c[%d];" % n]
    for kind, a, b, th, ph, la in gates:
        if kind in ("cx", "cz", "swap"):
            lines.append("%s q[%d],q[%d];" % (kind, a, b))
        elif kind == "cp":
            lines.append("cp(%r) q[%d],q[%d];" % (th, a, b))
        elif kind in ("rx", "ry", "rz", "p"):
            lines.append("%s(%r) q[%d];" % (kind, th, a))
        elif kind == "u":
            lines.append("u(%r,%r,%r) q[%d];" % (th, ph, la, a))
        else:
            lines.append("%s q[%d];" % (kind, a))
    lines.append("measure q -> c;")
    return "\n".join(lines) + "\n"


def test_spec_examples():
    # S:59-61 examples
    assert parse("qreg q[1]; x q[0]; measure q -> c;") == (1, [("x", 0, -1, 0.0, 0.0, 0.0)], True)
    n, g, m = parse("qreg q[2]; h q[0]; cx q[0],q[1];")
    assert (n, m) == (2, False)
    assert [(k, a, b) for k, a, b, *_ in g] == [("h", 0, -1), ("cx", 0, 1)]
    with pytest.raises(T.TqsimError) as e:
        parse("qreg q[1]; frobnicate q[0];")
    assert e.value.status == 2 and "frobnicate" in str(e.value) and "line 1" in str(e.value)


def test_pi_expressions_and_param_gates():
    n, g, _ = parse("""OPENQASM 2.0;
include "qelib1.inc";   // ignored
qreg q[2];
rz(-pi/4) q[0];
rx(2*(pi-1)/3) q[1];
u3(pi/2, 0, pi) q[0];
u2(0.5, -pi) q[1];
u1(1.5e-1) q[0];
cu1(3*pi/4) q[1], q[0];
id q[1];
barrier q;
""")
    assert n == 2
    assert g[0][:4] == ("rz", 0, -1, -math.pi / 4)
    assert g[1][3] == pytest.approx(2 * (math.pi - 1) / 3, abs=0)
    assert g[2] == ("u", 0, -1, math.pi / 2, 0.0, math.pi)
    assert g[3] == ("u", 1, -1, math.pi / 2, 0.5, -math.pi)        # u2 = U(pi/2, phi, lambda)
    assert g[4][:4] == ("p", 0, -1, 0.15)                         # u1 = P
    assert g[5][:4] == ("cp", 1, 0, 3 * math.pi / 4)
    assert g[6] == ("u", 1, -1, 0.0, 0.0, 0.0)                    # id: still a gate (noise location)
    assert len(g) == 7                                            # barrier dropped


def test_broadcast_and_registers():
    n, g, _ = parse("qreg a[2]; qreg b[2]; creg c[4]; h a; cx a, b; swap a[1], b[0]; measure a[0] -> c[0];")
    assert n == 4
    assert [(k, x, y) for k, x, y, *_ in g] == [("h", 0, -1), ("h", 1, -1), ("cx", 0, 2), ("cx", 1, 3),
                                                ("swap", 1, 2)]


@pytest.mark.parametrize("text,msg", [
    ("qreg q[2]; x q[2];", "out of range"),
    ("qreg q[2]; rx q[0];", "takes 1 parameter"),
    ("qreg q[2]; cx q[0];", "takes 2 qubit"),
    ("qreg q[2]; cx q[1],q[1];", "same qubit"),
    ("qreg q[2]; h r[0];", "unknown quantum register"),
    ("qreg q[31];", "more than 30"),
    ("qreg q[2];\nh q[0]\nx q[1];", "line 3"),
    ("qreg q[1]; rz(1/0) q[0];", "division by zero"),
    ("qreg q[2]; gate g a { x a; }", "not supported"),
    ("h q[0];", "unknown quantum register"),
])
def test_errors(text, msg):
    with pytest.raises(T.TqsimError) as e:
        parse(text)
    assert e.value.status == 2 and msg in str(e.value), str(e.value)


def test_round_trip_qft_and_lowering():
    gates = [(k, a, b, th, ph, la) for (k, a, b, th, ph, la) in qft_gates(7)]
    n, g, m = parse(to_qasm(7, gates))
    assert (n, m) == (7, True)
    assert g == gates
    assert T.tqsim_lower_circuit(n, g) == T.tqsim_lower_circuit(7, gates)
