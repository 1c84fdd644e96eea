// OpenQASM 2.0 subset ingestion (SPEC circuit-ir S:52-60).
//
// The paper's benchmark circuits come from QASMBench / Qiskit / Cirq / Qulacs
// (§4.2); none ship with this build, so user programs come in as text.
// Grammar (extended where OpenQASM 2 programs commonly need it):
//   OPENQASM 2.0;  include "...";  qreg name[n];  creg name[n];
//   gate statements  name[(expr, ...)] arg, arg ...;   arg = reg | reg[i]
//     x y z h s sdg t tdg id | rx ry rz p u1 (1 angle) | u2 (2) | u u3 (3)
//     cx CX cz swap cp cu1 (1 angle)
//   barrier ...;  measure a -> b;  (terminal full measurement; only the flag is kept)
//   expr: decimal / scientific literals, pi, + - * /, unary minus, parentheses
// Several qregs are concatenated in declaration order (qubit 0 = first qreg[0],
// little endian, R6).  A register argument broadcasts the gate over the register.
// `id` becomes U(0,0,0): it is a gate of the program, hence a noise location
// (P:277).  Errors: TQSIM_EINVAL "line L col C: message".
#include <cctype>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "tq_internal.h"

namespace tq {

namespace {

struct Parser {
  const char* s;
  size_t i = 0, line = 1, col = 1;
  std::map<std::string, std::pair<uint32_t, uint32_t>> qregs;   // name -> (offset, size)
  std::map<std::string, uint32_t> cregs;
  uint32_t width = 0;
  bool measured = false;
  std::vector<tqsim_gate> gates;

  [[noreturn]] void fail(const std::string& m) const {
    throw Error{TQSIM_EINVAL, "line " + std::to_string(line) + " col " + std::to_string(col) + ": " + m};
  }
  char peek() const { return s[i]; }
  void adv() {
    if (s[i] == '\n') {
      ++line;
      col = 1;
    } else {
      ++col;
    }
    ++i;
  }
  void ws() {
    for (;;) {
      while (s[i] && std::isspace((unsigned char)s[i])) adv();
      if (s[i] == '/' && s[i + 1] == '/') {
        while (s[i] && s[i] != '\n') adv();
        continue;
      }
      break;
    }
  }
  bool eat(char c) {
    ws();
    if (peek() == c) {
      adv();
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) fail(std::string("expected '") + c + "'");
  }
  std::string ident() {
    ws();
    if (!(std::isalpha((unsigned char)peek()) || peek() == '_')) fail("expected an identifier");
    std::string r;
    while (std::isalnum((unsigned char)peek()) || peek() == '_') {
      r.push_back(peek());
      adv();
    }
    return r;
  }
  uint64_t integer() {
    ws();
    if (!std::isdigit((unsigned char)peek())) fail("expected an integer");
    uint64_t v = 0;
    while (std::isdigit((unsigned char)peek())) {
      v = v * 10 + (uint64_t)(peek() - '0');
      if (v > (1ull << 31)) fail("integer too large");
      adv();
    }
    return v;
  }
  // expr := term (('+'|'-') term)* ; term := unary (('*'|'/') unary)* ;
  // unary := '-' unary | '+' unary | primary ; primary := number | pi | '(' expr ')'
  double expr() {
    double v = term();
    for (;;) {
      if (eat('+')) v += term();
      else if (eat('-')) v -= term();
      else return v;
    }
  }
  double term() {
    double v = unary();
    for (;;) {
      if (eat('*')) v *= unary();
      else if (eat('/')) {
        const double d = unary();
        if (d == 0.0) fail("division by zero");
        v /= d;
      } else {
        return v;
      }
    }
  }
  double unary() {
    if (eat('-')) return -unary();
    if (eat('+')) return unary();
    return primary();
  }
  double primary() {
    ws();
    if (eat('(')) {
      const double v = expr();
      expect(')');
      return v;
    }
    if (std::isalpha((unsigned char)peek())) {
      const std::string id = ident();
      if (id == "pi") return M_PI;
      fail("unknown symbol '" + id + "' in expression");
    }
    const char* b = s + i;
    char* e = nullptr;
    const double v = std::strtod(b, &e);
    if (e == b) fail("expected a number");
    while (s + i < e) adv();
    return v;
  }
  // reg | reg[i] -> list of global qubits
  std::vector<uint32_t> qarg() {
    const std::string name = ident();
    auto it = qregs.find(name);
    if (it == qregs.end()) fail("unknown quantum register '" + name + "'");
    const uint32_t off = it->second.first, size = it->second.second;
    if (eat('[')) {
      const uint64_t k = integer();
      expect(']');
      if (k >= size) fail("qubit index " + std::to_string(k) + " out of range for '" + name + "'");
      return {off + (uint32_t)k};
    }
    std::vector<uint32_t> r;
    for (uint32_t k = 0; k < size; ++k) r.push_back(off + k);
    return r;
  }
  void skip_statement() {
    while (peek() && peek() != ';') adv();
    expect(';');
  }
  void add(uint32_t kind, uint32_t a, uint32_t b, double th, double ph, double la) {
    tqsim_gate g{};
    g.kind = kind;
    g.q0 = a;
    g.q1 = b;
    g.theta = th;
    g.phi = ph;
    g.lambda = la;
    gates.push_back(g);
  }

  void parse() {
    for (;;) {
      ws();
      if (!peek()) break;
      const std::string kw = ident();
      if (kw == "OPENQASM") {
        skip_statement();
      } else if (kw == "include") {
        skip_statement();
      } else if (kw == "qreg" || kw == "creg") {
        const std::string name = ident();
        expect('[');
        const uint64_t n = integer();
        expect(']');
        expect(';');
        if (qregs.count(name) || cregs.count(name)) fail("register '" + name + "' redeclared");
        if (kw == "qreg") {
          if (n == 0) fail("empty quantum register");
          if (width + n > TQSIM_MAX_QUBITS) fail("more than " + std::to_string(TQSIM_MAX_QUBITS) + " qubits");
          qregs[name] = {width, (uint32_t)n};
          width += (uint32_t)n;
        } else {
          cregs[name] = (uint32_t)n;
        }
      } else if (kw == "barrier") {
        skip_statement();
      } else if (kw == "measure") {
        qarg();
        ws();
        if (!(peek() == '-' && s[i + 1] == '>')) fail("expected '->'");
        adv();
        adv();
        ident();   // classical target (only the terminal-measurement flag is kept)
        if (eat('[')) {
          integer();
          expect(']');
        }
        expect(';');
        measured = true;
      } else if (kw == "gate" || kw == "opaque" || kw == "if" || kw == "reset") {
        fail("'" + kw + "' is not supported (SPEC non-goals: custom gates, classical control)");
      } else {
        gate_statement(kw);
      }
    }
    if (qregs.empty()) fail("no qreg declared");
  }

  void gate_statement(const std::string& name) {
    static const std::map<std::string, std::pair<int, int>> table = {
        // name -> (kind or -1 special, number of angles)
        {"x", {TQ_X, 0}}, {"y", {TQ_Y, 0}}, {"z", {TQ_Z, 0}}, {"h", {TQ_H, 0}},
        {"s", {TQ_S, 0}}, {"sdg", {TQ_SDG, 0}}, {"t", {TQ_T, 0}}, {"tdg", {TQ_TDG, 0}},
        {"id", {-1, 0}}, {"rx", {TQ_RX, 1}}, {"ry", {TQ_RY, 1}}, {"rz", {TQ_RZ, 1}},
        {"p", {TQ_P, 1}}, {"u1", {TQ_P, 1}}, {"u2", {-2, 2}}, {"u", {TQ_U, 3}}, {"u3", {TQ_U, 3}},
        {"U", {TQ_U, 3}}, {"cx", {TQ_CX, 0}}, {"CX", {TQ_CX, 0}}, {"cz", {TQ_CZ, 0}},
        {"swap", {TQ_SWAP, 0}}, {"cp", {TQ_CP, 1}}, {"cu1", {TQ_CP, 1}}};
    auto it = table.find(name);
    if (it == table.end()) fail("unsupported gate '" + name + "'");
    const int kind = it->second.first, nang = it->second.second;
    std::vector<double> ang;
    if (eat('(')) {
      if (!eat(')')) {
        ang.push_back(expr());
        while (eat(',')) ang.push_back(expr());
        expect(')');
      }
    }
    if ((int)ang.size() != nang)
      fail("gate '" + name + "' takes " + std::to_string(nang) + " parameter(s), got " + std::to_string(ang.size()));
    std::vector<std::vector<uint32_t>> args;
    args.push_back(qarg());
    while (eat(',')) args.push_back(qarg());
    expect(';');
    const bool two = kind == TQ_CX || kind == TQ_CZ || kind == TQ_SWAP || kind == TQ_CP;
    if ((int)args.size() != (two ? 2 : 1))
      fail("gate '" + name + "' takes " + std::to_string(two ? 2 : 1) + " qubit argument(s)");
    size_t reps = 1;
    for (auto& a : args)
      if (a.size() > 1) {
        if (reps > 1 && a.size() != reps) fail("register arguments of different sizes");
        reps = a.size();
      }
    for (size_t r = 0; r < reps; ++r) {
      const uint32_t a = args[0][args[0].size() > 1 ? r : 0];
      if (two) {
        const uint32_t b = args[1][args[1].size() > 1 ? r : 0];
        if (a == b) fail("gate '" + name + "' on the same qubit twice");
        add((uint32_t)kind, a, b, ang.empty() ? 0.0 : ang[0], 0.0, 0.0);
      } else if (kind == -1) {   // id -> U(0,0,0): a gate, hence a noise location
        add(TQ_U, a, 0, 0.0, 0.0, 0.0);
      } else if (kind == -2) {   // u2(phi, lambda) = U(pi/2, phi, lambda)
        add(TQ_U, a, 0, M_PI / 2, ang[0], ang[1]);
      } else {
        add((uint32_t)kind, a, 0, nang > 0 ? ang[0] : 0.0, nang > 1 ? ang[1] : 0.0, nang > 2 ? ang[2] : 0.0);
      }
    }
  }
};

}  // namespace

}  // namespace tq

extern "C" tqsim_status tqsim_parse_qasm(const char* text, tqsim_gate* out, uint64_t cap,
                                         uint64_t* n_gates, uint32_t* n_qubits, uint32_t* measured) {
  try {
    if (!text || !n_gates || !n_qubits) throw tq::Error{TQSIM_EINVAL, "NULL argument"};
    tq::Parser p;
    p.s = text;
    p.parse();
    *n_gates = p.gates.size();
    *n_qubits = p.width;
    if (measured) *measured = p.measured ? 1u : 0u;
    if (out)
      for (uint64_t k = 0; k < p.gates.size() && k < cap; ++k) out[k] = p.gates[k];
    return TQSIM_OK;
  } catch (const tq::Error& e) {
    tq::set_error(e.msg);
    return e.status;
  } catch (...) {
    tq::set_error("internal error in the QASM parser");
    return TQSIM_EINTERNAL;
  }
}
