// Circuit IR: validation, lowering and gate matrices.
//
// Paper: a circuit is "a list of quantum gates that need to be applied, in
// order" (§2.2); noise operators are inserted "after each of the gates"
// (P:277).  Readings: R4 lowering CP -> P,CX,P,CX,P and SWAP -> 3 CX;
// R5 OpenQASM-2 matrices with fixed global phases (see include/tqsim.h).
#include <cmath>
#include <sstream>

#include "tq_internal.h"

namespace tq {

namespace {

void mat_set(LGate& g, double r00, double i00, double r01, double i01, double r10, double i10,
             double r11, double i11) {
  g.m[0] = r00; g.m[1] = i00; g.m[2] = r01; g.m[3] = i01;
  g.m[4] = r10; g.m[5] = i10; g.m[6] = r11; g.m[7] = i11;
}

LGate make_1q(uint32_t kind, uint32_t q, double th, double ph, double la) {
  LGate g{};
  g.kind = kind; g.q0 = q; g.q1 = q; g.two = false;
  const double c = std::cos(th / 2.0), s = std::sin(th / 2.0);
  const double r2 = 1.0 / std::sqrt(2.0);
  switch (kind) {
    case TQ_X: mat_set(g, 0, 0, 1, 0, 1, 0, 0, 0); break;
    case TQ_Y: mat_set(g, 0, 0, 0, -1, 0, 1, 0, 0); break;
    case TQ_Z: mat_set(g, 1, 0, 0, 0, 0, 0, -1, 0); break;
    case TQ_H: mat_set(g, r2, 0, r2, 0, r2, 0, -r2, 0); break;
    case TQ_S: mat_set(g, 1, 0, 0, 0, 0, 0, 0, 1); break;
    case TQ_SDG: mat_set(g, 1, 0, 0, 0, 0, 0, 0, -1); break;
    case TQ_T: mat_set(g, 1, 0, 0, 0, 0, 0, std::cos(M_PI / 4), std::sin(M_PI / 4)); break;
    case TQ_TDG: mat_set(g, 1, 0, 0, 0, 0, 0, std::cos(M_PI / 4), -std::sin(M_PI / 4)); break;
    case TQ_RX: mat_set(g, c, 0, 0, -s, 0, -s, c, 0); break;
    case TQ_RY: mat_set(g, c, 0, -s, 0, s, 0, c, 0); break;
    case TQ_RZ:
      mat_set(g, std::cos(th / 2), -std::sin(th / 2), 0, 0, 0, 0, std::cos(th / 2), std::sin(th / 2));
      break;
    case TQ_P: mat_set(g, 1, 0, 0, 0, 0, 0, std::cos(th), std::sin(th)); break;
    case TQ_U: {
      // [[c, -e^{il} s], [e^{ip} s, e^{i(p+l)} c]]
      const double cl = std::cos(la), sl = std::sin(la), cp = std::cos(ph), sp = std::sin(ph);
      const double cpl = std::cos(ph + la), spl = std::sin(ph + la);
      mat_set(g, c, 0, -cl * s, -sl * s, cp * s, sp * s, cpl * c, spl * c);
      break;
    }
    default: break;
  }
  const bool diag = g.m[2] == 0 && g.m[3] == 0 && g.m[4] == 0 && g.m[5] == 0;
  g.op = diag ? OP_DIAG : OP_GEN;
  return g;
}

LGate make_2q(uint32_t kind, uint32_t a, uint32_t b) {
  LGate g{};
  g.kind = kind; g.q0 = a; g.q1 = b; g.two = true;
  g.op = kind == TQ_CX ? OP_CX : OP_CZ;
  return g;
}

Error einval(const std::string& m) { return Error{TQSIM_EINVAL, m}; }

}  // namespace

std::vector<LGate> lower(const tqsim_circuit* c) {
  if (!c) throw einval("circuit is NULL");
  if (c->n_qubits < 1 || c->n_qubits > TQSIM_MAX_QUBITS)
    throw einval("n_qubits must be in [1, 30]");
  if (c->n_gates < 1 || !c->gates) throw einval("circuit has no gates");
  std::vector<LGate> out;
  out.reserve(c->n_gates * 2);
  for (uint64_t i = 0; i < c->n_gates; ++i) {
    const tqsim_gate& g = c->gates[i];
    std::ostringstream where;
    where << "gate " << i << ": ";
    if (g.kind > TQ_CP) throw einval(where.str() + "unknown kind");
    if (g.q0 >= c->n_qubits) throw einval(where.str() + "qubit out of range");
    const bool two = g.kind == TQ_CX || g.kind == TQ_CZ || g.kind == TQ_SWAP || g.kind == TQ_CP;
    if (two) {
      if (g.q1 >= c->n_qubits) throw einval(where.str() + "qubit out of range");
      if (g.q1 == g.q0) throw einval(where.str() + "2q gate on identical qubits");
    }
    if (!std::isfinite(g.theta) || !std::isfinite(g.phi) || !std::isfinite(g.lambda))
      throw einval(where.str() + "non-finite angle");
    switch (g.kind) {
      case TQ_CX: case TQ_CZ: out.push_back(make_2q(g.kind, g.q0, g.q1)); break;
      case TQ_SWAP:
        out.push_back(make_2q(TQ_CX, g.q0, g.q1));
        out.push_back(make_2q(TQ_CX, g.q1, g.q0));
        out.push_back(make_2q(TQ_CX, g.q0, g.q1));
        break;
      case TQ_CP:
        out.push_back(make_1q(TQ_P, g.q0, g.theta / 2.0, 0, 0));
        out.push_back(make_2q(TQ_CX, g.q0, g.q1));
        out.push_back(make_1q(TQ_P, g.q1, -g.theta / 2.0, 0, 0));
        out.push_back(make_2q(TQ_CX, g.q0, g.q1));
        out.push_back(make_1q(TQ_P, g.q1, g.theta / 2.0, 0, 0));
        break;
      default: out.push_back(make_1q(g.kind, g.q0, g.theta, g.phi, g.lambda)); break;
    }
  }
  if (out.size() >= (1ull << 32)) throw einval("too many gates");
  return out;
}

}  // namespace tq
