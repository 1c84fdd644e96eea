// Run-time specialization of the gate-pass kernels.
//
// Each HBM pass of the pass plan becomes one kernel whose gate sequence,
// tile/register qubit positions and gate matrices are compile-time constants:
//   * register tile of 16 complex128 amplitudes per thread in named registers;
//   * CX, SWAP-parts and X gates are register RENAMINGS (no instructions);
//   * diagonal gates touch only the amplitudes they change; zero matrix
//     components are skipped (real matrices cost half the FMAs);
//   * the keyed Pauli error of every gate (codes computed per CTA by the shared
//     tq_noise_code) is applied right AFTER its gate on a rarely-taken branch
//     ("noise operators ... after each of the gates");
//   * the first pass of a node reads its PARENT's state (fused fan-out) or
//     synthesizes |0..0> (root); passes with one phase need no shared memory.
// Sources are compiled with NVRTC for sm_100a (one program per pass, in
// parallel host threads) and cached in-process by source text.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <set>
#include <mutex>
#include <sstream>
#include <thread>
#include <unordered_map>

#include "tq_internal.h"

namespace tq {

namespace {

const char* kPrelude =
#include "jit_prelude.inc"
    ;

const char* kJitTypes = R"TQ(
struct __align__(16) tq_d2 { double x, y; };
struct TqJitArgs {
  const tq_d2* src; tq_d2* dst; tq_u64 seed; double p1, p2;
  tq_u64 child_first, parent_first; tq_u32 arity, batch;
  double* runsum;   // leaf level: |a|^2 sums of 8-amplitude runs, 2^(n-3) per state
  const unsigned char* rows; tq_u32 row_bytes;   // noise rows of the batch (launch_noise_rows)
  // leaf measurement without the state store (variants 1/2, see gen_pass)
  const tq_u32* tiles; const tq_u32* runsel; tq_d2* scratch; tq_u32* xlout;
  // dedup maps (launch_dedup_map) of the batch and of the parent batch, or null
  const tq_u32* rep; const tq_u32* prep;
  // projection (variant 3) work list: leaves and their count, or null (every leaf)
  const tq_u32* wlist; const tq_u32* wcount;
};
// 16-byte global load the compiler may not sink below the error-branch: the tile loads
// are issued before the (dependent) noise-row mask load is waited on
__device__ __forceinline__ tq_d2 tq_ld(const tq_d2* p) {
  tq_d2 r;
  asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
// one 32-byte access = two consecutive amplitudes (LDG/STG.256 on sm_100)
__device__ __forceinline__ void tq_ld2(const tq_d2* p, tq_d2& a, tq_d2& b) {
  asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y) : "l"(p));
}
__device__ __forceinline__ void tq_st2(tq_d2* p, const tq_d2& a, const tq_d2& b) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" :: "l"(p), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y) : "memory");
}
// TMA staging (TQSIM_TMA): tensor map by value, mbarrier + cp.async.bulk.tensor (5-D tile)
struct __align__(64) TqTmap { unsigned long long v[16]; };
__device__ __forceinline__ unsigned tq_smem(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tq_mbar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(tq_smem(bar)) : "memory");
}
__device__ __forceinline__ void tq_fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void tq_fence_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tq_tma_load(void* dst, const TqTmap* tm, unsigned long long* bar, int c0, int c1, int c2,
                                            int c3, int c4, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(tq_smem(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
               :: "r"(tq_smem(dst)), "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(tq_smem(bar)) : "memory");
}
__device__ __forceinline__ void tq_mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok = 0u;
  while (!ok)
    asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                 : "=r"(ok) : "r"(tq_smem(bar)), "r"(parity) : "memory");
}
// r *= i^q
__device__ __forceinline__ void tq_rot(tq_d2& r, tq_u32 q) {
  const double a = (q & 1u) ? r.y : r.x, b = (q & 1u) ? r.x : r.y;
  r.x = (((q + 1u) >> 1) & 1u) ? -a : a;
  r.y = ((q >> 1) & 1u) ? -b : b;
}
)TQ";

struct HostJitArgs {   // mirrors TqJitArgs
  const void* src;
  void* dst;
  uint64_t seed;
  double p1, p2;
  uint64_t child_first, parent_first;
  uint32_t arity, batch;
  double* runsum;
  const void* rows;
  uint32_t row_bytes;
  const uint32_t* tiles;
  const uint32_t* runsel;
  void* scratch;
  uint32_t* xlout;
  const uint32_t* rep;
  const uint32_t* prep;
  const uint32_t* wlist;
  const uint32_t* wcount;
};

std::string hexd(double v) {
  char b[64];
  std::snprintf(b, sizeof(b), "%a", v);
  return b;
}

uint32_t host_swz(uint32_t i) { return i ^ (((i >> 3) ^ (i >> 6) ^ (i >> 9) ^ (i >> 12)) & 7u); }

// Gate-matrix coefficients: FP64 literals in the generated code (default), or --
// TQSIM_JIT_COEF=0 -- a by-value kernel parameter table, which makes the source
// (and the compiled-kernel cache key) depend only on the circuit's structure
// (gate kinds, qubits, which components are 0 or +-1), not on its angles.
struct ConstPool {
  std::vector<double> vals;
  std::map<uint64_t, int> index;
  std::map<uint64_t, std::string> local;   // per gate: value bits -> register name
  std::ostringstream decl;
  int nlocal = 0;
  void begin_op() {
    local.clear();
    decl.str("");
    nlocal = 0;
  }
  // 2 (default): FP64 literals -- fastest (the measured best on B200);
  // 0: by-value kernel parameter -- source (and cache key) independent of angles
  int mode = 2;
  std::string ref(double v) {
    if (v == 1.0) return "1.0";
    if (v == -1.0) return "-1.0";
    if (mode == 2) return hexd(v);
    uint64_t bits;
    std::memcpy(&bits, &v, 8);
    auto lt = local.find(bits);
    if (lt != local.end()) return lt->second;
    auto it = index.find(bits);
    int k;
    if (it == index.end()) {
      k = (int)vals.size();
      vals.push_back(v);
      index[bits] = k;
    } else {
      k = it->second;
    }
    const std::string name = "q" + std::to_string(nlocal++);
    decl << "      const double " << name << " = cf.v[" << k << "];\n";
    local[bits] = name;
    return name;
  }
};
thread_local ConstPool* g_pool = nullptr;   // set while one kernel is generated

// re/im of  a*x + b*y  with a = (ar, ai), b = (br, bi); zero components skipped.
std::string lin(double ar, double ai, const std::string& x, double br, double bi,
                const std::string& y, bool imag) {
  std::vector<std::pair<double, std::string>> t;
  if (!imag) {
    if (ar != 0) t.push_back({ar, x + ".x"});
    if (ai != 0) t.push_back({-ai, x + ".y"});
    if (br != 0) t.push_back({br, y + ".x"});
    if (bi != 0) t.push_back({-bi, y + ".y"});
  } else {
    if (ar != 0) t.push_back({ar, x + ".y"});
    if (ai != 0) t.push_back({ai, x + ".x"});
    if (br != 0) t.push_back({br, y + ".y"});
    if (bi != 0) t.push_back({bi, y + ".x"});
  }
  if (t.empty()) return "0.0";
  std::string e = "(" + g_pool->ref(t.back().first) + " * " + t.back().second + ")";
  for (int i = (int)t.size() - 2; i >= 0; --i)
    e = "fma(" + g_pool->ref(t[i].first) + ", " + t[i].second + ", " + e + ")";
  return e;
}

struct Gen {
  std::ostringstream o;
  int rm[16];   // logical register index -> slot
  void reset_map() {
    for (int k = 0; k < 16; ++k) rm[k] = k;
  }
  std::string r(int logical) { return "r" + std::to_string(rm[logical]); }
};


// ---------------------------------------------------------------- error-free fast path
// In the fast path (no Pauli drawn for any gate of the pass) runs of consecutive gates
// on at most two qubits whose product is DIAGONAL (e.g. the 5-gate lowered CP, or
// CX.RZ.CX) are fused into one diagonal op.  A diagonal op needs no register slot:
// its phase is a function of index bits the thread knows -- register bits at code
// generation time, thread/tile bits at run time -- so the fast path is planned into
// phases around the non-diagonal gates only (fewer shared-memory tile exchanges).
typedef std::complex<double> cplx;

// re/im of sum_j c_j * v_j (complex coefficients, compile-time; zero terms skipped)
std::string linN(const cplx* c, const std::string* v, int nterms, bool imag) {
  std::vector<std::pair<double, std::string>> t;
  for (int j = 0; j < nterms; ++j) {
    if (!imag) {
      if (c[j].real() != 0) t.push_back({c[j].real(), v[j] + ".x"});
      if (c[j].imag() != 0) t.push_back({-c[j].imag(), v[j] + ".y"});
    } else {
      if (c[j].real() != 0) t.push_back({c[j].real(), v[j] + ".y"});
      if (c[j].imag() != 0) t.push_back({c[j].imag(), v[j] + ".x"});
    }
  }
  if (t.empty()) return "0.0";
  std::string e = "(" + g_pool->ref(t.back().first) + " * " + t.back().second + ")";
  for (int i = (int)t.size() - 2; i >= 0; --i)
    e = "fma(" + g_pool->ref(t[i].first) + ", " + t[i].second + ", " + e + ")";
  return e;
}


// Effect of the keyed Pauli of one gate (code c) propagated to the END of the fused
// run containing the gate: E' = R E R^dagger with R the run's later gates (monomial,
// so E' = (diagonal) x (bit flips)).  Either Pauli-type E' = i^k X^x Z^z, or generic
// E' = D X^x with D a diagonal on the run's two qubits.  Masks over PHYSICAL qubits
// (after the run's SWAP relabeling, if any).
struct ErrEff {
  uint32_t x = 0, z = 0, k = 0;
  bool generic = false;
  cplx D[4];                // generic: entry for local index bit_s0 | bit_s1 << 1
};
struct ErrSite {
  uint32_t gate = 0;        // lowered gate index g
  uint32_t local = 0;       // index of the gate in the pass's op list
  std::vector<ErrEff> eff;  // per code c = 1..(3 or 15)
};

struct FOp {
  // AMAP: an absorbed CX (ROLE_STOREMAP), applied by the store-address map; no code in
  // the fast path, a frame conjugation (+ its errors) in the careful path
  enum Kind { GEN, XPERM, CX, DIAG, NOP, GEN2, AMAP } kind = GEN;
  cplx m4[16];            // GEN2: row-major 4x4, local index bit_qa | bit_qb << 1
  std::vector<FOp> comps; // GEN2: its gates (careful path), each with its own site
  int qa = -1, qb = -1;   // global (physical) qubits (qb = -1: one-qubit op)
  cplx m[4];              // GEN: row-major 2x2
  cplx d[4];              // DIAG: entry for index bit_qa | bit_qb << 1
  // careful path: the run's gates in order, and its two PHYSICAL qubits after the run
  // (the local frame of generic error diagonals; -1 = dummy slot)
  std::vector<ErrSite> sites;
  int ea = -1, eb = -1;
};

struct PhaseSpec {
  PhaseDesc P;
  std::vector<int> items;   // careful path: indices into pp.ops; fast path: into fops
};

// 4x4 over (s0, s1), local index = bit_s0 | bit_s1 << 1
struct M4 {
  cplx a[4][4];
  static M4 id() {
    M4 r;
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) r.a[i][j] = i == j ? cplx(1, 0) : cplx(0, 0);
    return r;
  }
  M4 mul(const M4& b) const {   // this * b
    M4 r;
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) {
        cplx acc(0, 0);
        for (int k = 0; k < 4; ++k)
          if (a[i][k] != cplx(0, 0) && b.a[k][j] != cplx(0, 0)) acc += a[i][k] * b.a[k][j];
        r.a[i][j] = acc;
      }
    return r;
  }
  bool diagonal() const {
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j)
        if (i != j && a[i][j] != cplx(0, 0)) return false;
    return true;
  }
  // a permutation times a diagonal (decompose()'s 1e-12 threshold): one entry per column
  // and per row
  bool monomial() const {
    int rows = 0;
    for (int j = 0; j < 4; ++j) {
      int cnt = 0, r0 = -1;
      for (int i = 0; i < 4; ++i)
        if (std::abs(a[i][j]) > 1e-12) ++cnt, r0 = i;
      if (cnt != 1) return false;
      rows |= 1 << r0;
    }
    return rows == 15;
  }
};

M4 op_matrix(const LGate& g, int s0, int s1) {
  M4 r;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) r.a[i][j] = cplx(0, 0);
  auto bit = [&](int idx, int q) { return q == s0 ? (idx & 1) : ((idx >> 1) & 1); };
  if (!g.two) {
    const cplx m[4] = {cplx(g.m[0], g.m[1]), cplx(g.m[2], g.m[3]), cplx(g.m[4], g.m[5]),
                       cplx(g.m[6], g.m[7])};
    const int q = (int)g.q0, o = q == s0 ? 1 : 0;   // bit position of the other slot
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) {
        const int oi = o ? ((i >> 1) & 1) : (i & 1), oj = o ? ((j >> 1) & 1) : (j & 1);
        if (oi != oj) continue;
        r.a[i][j] = m[bit(i, q) * 2 + bit(j, q)];
      }
    return r;
  }
  const int c = (int)g.q0, t = (int)g.q1;
  for (int j = 0; j < 4; ++j) {
    if (g.op == OP_CX) {
      int i = j;
      if (bit(j, c)) i ^= (t == s0 ? 1 : 2);
      r.a[i][j] = cplx(1, 0);
    } else {   // CZ
      r.a[j][j] = (bit(j, c) && bit(j, t)) ? cplx(-1, 0) : cplx(1, 0);
    }
  }
  return r;
}

bool is_x_gate(const LGate& lg) {
  const double* m = lg.m;
  return !lg.two && m[0] == 0 && m[1] == 0 && m[2] == 1 && m[3] == 0 && m[4] == 1 && m[5] == 0 &&
         m[6] == 0 && m[7] == 0;
}

bool is_swap(const M4& P) {   // exchanges |01> and |10>, fixes |00>, |11>
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      const int si = (i == 1) ? 2 : (i == 2) ? 1 : i;
      if (P.a[i][j] != (j == si ? cplx(1, 0) : cplx(0, 0))) return false;
    }
  return true;
}

// Fast-path op list.  SWAPs (a fused run whose product is the swap permutation) are
// not executed: both qubits are tile qubits, so the swap is a relabeling of tile
// positions -- later ops are rewritten to PHYSICAL qubit labels and the final store
// writes position p to logical qubit log_of_phys[tile_q[p]].
// Pauli p (0 I, 1 X, 2 Y, 3 Z) as a 2x2
void pauli2(int p, cplx m[2][2]) {
  const cplx I(0, 1);
  m[0][0] = m[1][1] = m[0][1] = m[1][0] = 0;
  if (p == 0) m[0][0] = m[1][1] = 1;
  else if (p == 1) m[0][1] = m[1][0] = 1;
  else if (p == 2) { m[0][1] = -I; m[1][0] = I; }
  else { m[0][0] = 1; m[1][1] = -1; }
}

// 4x4 of Pauli pa on slot a and pb on slot b (local index bit_s0 | bit_s1 << 1)
M4 pauli4(int pa, int slot_a, int pb, int slot_b) {
  cplx A[2][2], B[2][2];
  pauli2(pa, A);
  pauli2(pb, B);
  M4 r;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      const int ia = (i >> slot_a) & 1, ja = (j >> slot_a) & 1;
      const int ib = (i >> slot_b) & 1, jb = (j >> slot_b) & 1;
      r.a[i][j] = A[ia][ja] * B[ib][jb];
    }
  return r;
}

M4 dagger(const M4& m) {
  M4 r;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) r.a[i][j] = std::conj(m.a[j][i]);
  return r;
}

bool near(const cplx& a, const cplx& b) { return std::abs(a - b) < 1e-13; }

// The four frame variants of a one-qubit matrix are c [[1, s u], [s w, 1]] with one sign s
// per variant (RX, RY; c real, |u|, |w| <= 1)
bool sign_variants(const cplx V[4][4]) {
  const cplx c = V[0][0];
  if (c.imag() != 0.0 || c.real() <= 0.0) return false;
  if (std::abs(V[0][1]) > c.real() || std::abs(V[0][2]) > c.real()) return false;
  for (int v = 0; v < 4; ++v) {
    if (V[v][0] != c || V[v][3] != c) return false;
    const bool same = std::abs(V[v][1] - V[0][1]) < 1e-15 && std::abs(V[v][2] - V[0][2]) < 1e-15;
    const bool flip = std::abs(V[v][1] + V[0][1]) < 1e-15 && std::abs(V[v][2] + V[0][2]) < 1e-15;
    if (!same && !flip) return false;
  }
  return true;
}

// exact 0 / +-1 for components within rounding of them (phases composed at generation time)
cplx snap(cplx v) {
  auto s1 = [](double x) {
    for (double t : {0.0, 1.0, -1.0})
      if (std::abs(x - t) < 1e-14) return t;
    return x;
  };
  return cplx(s1(v.real()), s1(v.imag()));
}

// ZYZ form of a 2x2 unitary: m = e^{ia} diag(1, e^{if}) [[c, -s], [s, c]] diag(1, e^{il}),
// c, s >= 0.  ea = e^{ia}, eaf = e^{i(a+f)}, el = e^{il}.  False when m is not of this
// form to 1e-12 (not unitary up to a phase) or is diagonal / anti-diagonal-free.
struct Zyz {
  double c = 0, s = 0;
  cplx ea, eaf, el;
};
bool zyz_of(const cplx* m, Zyz& z) {
  z.c = std::abs(m[0]);
  z.s = std::abs(m[2]);
  if (z.s < 1e-12 || std::abs(z.c * z.c + z.s * z.s - 1.0) > 1e-12) return false;
  z.eaf = m[2] / z.s;
  if (z.c > 1e-12) {
    z.ea = m[0] / z.c;
  } else {
    z.ea = cplx(1.0, 0.0);
    z.c = 0.0;
  }
  z.el = (-m[1] / z.s) / z.ea;
  const cplx m11 = z.eaf * z.el * z.c;
  if (std::abs(m11 - m[3]) > 1e-12 || std::abs(std::abs(z.el) - 1.0) > 1e-12) return false;
  return true;
}

// real 2x2 whose entries are +-c (H, and H up to signs)
bool hadamard_like(const cplx* m) {
  const double c = std::abs(m[0].real());
  if (c == 0.0) return false;
  for (int e = 0; e < 4; ++e)
    if (m[e].imag() != 0.0 || std::abs(m[e].real()) != c) return false;
  return true;
}

// E' = R E R^dagger (monomial) -> Pauli-type i^k X^x Z^z or generic D X^x, local masks
ErrEff decompose(const M4& M) {
  ErrEff e;
  int xe = -1;
  for (int r = 0; r < 4; ++r)
    if (std::abs(M.a[r][0]) > 1e-12) xe = r;
  if (xe < 0) throw Error{TQSIM_EINTERNAL, "error propagation: not monomial"};
  cplx v[4];
  for (int j = 0; j < 4; ++j) {
    for (int r = 0; r < 4; ++r)
      if (r != (j ^ xe) && std::abs(M.a[r][j]) > 1e-12)
        throw Error{TQSIM_EINTERNAL, "error propagation: not an X-type permutation"};
    v[j] = M.a[j ^ xe][j];
  }
  e.x = (uint32_t)xe;
  const cplx I(0, 1), ph[4] = {cplx(1, 0), I, cplx(-1, 0), -I};
  int k = -1;
  for (int t = 0; t < 4; ++t)
    if (near(v[0], ph[t])) k = t;
  bool pauli = k >= 0;
  uint32_t z = 0;
  if (pauli) {
    for (int b = 0; b < 2; ++b) {
      const cplx rr = v[1 << b] / v[0];
      if (near(rr, cplx(-1, 0))) z |= 1u << b;
      else if (!near(rr, cplx(1, 0))) pauli = false;
    }
    if (pauli)
      for (int j = 0; j < 4; ++j)
        if (!near(v[j], v[0] * ((__builtin_popcount(z & (uint32_t)j) & 1) ? -1.0 : 1.0))) pauli = false;
  }
  if (pauli) {
    e.k = (uint32_t)k;
    e.z = z;
  } else {
    // M = D X^x: D(i) = M[i][i ^ x]
    e.generic = true;
    for (int i = 0; i < 4; ++i) e.D[i] = M.a[i][i ^ xe];
  }
  return e;
}

// Fast-path op list.  SWAPs (a fused run whose product is the swap permutation) are
// not executed: both qubits are tile qubits, so the swap is a relabeling of tile
// positions -- later ops are rewritten to PHYSICAL qubit labels and the final store
// writes position p to logical qubit log_of_phys[tile_q[p]].  Runs that cancel to
// the identity become NOPs (they still carry their gates' error sites).
// FP64 cost (per amplitude) of one gate applied alone in the fast path: a general
// complex 2x2 8, a real one 4, diagonals / permutations ~free.
int gate_cost(const LGate& g) {
  if (g.two || g.op == OP_DIAG) return g.two ? 0 : 1;
  if (is_x_gate(g)) return 0;
  bool real = true;
  for (int k = 1; k < 8; k += 2)
    if (g.m[k] != 0.0) real = false;
  return real ? 4 : 8;
}

// Commutation-aware 2-qubit blocks: gates on disjoint qubits commute, so a gate joins
// the open block(s) holding its qubits while their union has <= 2 qubits; otherwise
// those blocks close (are emitted, in order) and the gate opens a new block.  Emitting
// a block when it closes is a valid topological order (blocks open at the same time
// are on disjoint qubits).  Returns the pass's local op indices, block by block.
std::vector<int> block_order(int n, const std::function<const LGate&(int)>& lg_of) {
  struct Blk {
    std::vector<int> ops;
    uint64_t qm = 0;
    bool open = true;
  };
  std::vector<Blk> blks;
  std::map<int, int> owner;   // qubit -> open block
  std::vector<int> ord;
  auto close = [&](int bi) {
    if (!blks[bi].open) return;
    blks[bi].open = false;
    for (int q = 0; q < 64; ++q)
      if (blks[bi].qm >> q & 1) owner.erase(q);
    ord.insert(ord.end(), blks[bi].ops.begin(), blks[bi].ops.end());
  };
  for (int i = 0; i < n; ++i) {
    const LGate& g = lg_of(i);
    const uint64_t Q = (1ull << g.q0) | (g.two ? 1ull << g.q1 : 0ull);
    std::vector<int> own;
    for (int q = 0; q < 64; ++q)
      if (Q >> q & 1) {
        auto it = owner.find(q);
        if (it != owner.end() && std::find(own.begin(), own.end(), it->second) == own.end()) own.push_back(it->second);
      }
    std::sort(own.begin(), own.end());
    uint64_t U = Q;
    for (int bi : own) U |= blks[bi].qm;
    if (__builtin_popcountll(U) <= 2) {
      Blk nb;
      for (int bi : own) {
        nb.ops.insert(nb.ops.end(), blks[bi].ops.begin(), blks[bi].ops.end());
        blks[bi].open = false;
        blks[bi].ops.clear();
      }
      nb.ops.push_back(i);
      nb.qm = U;
      blks.push_back(nb);
      for (int q = 0; q < 64; ++q)
        if (U >> q & 1) owner[q] = (int)blks.size() - 1;
      continue;
    }
    for (int bi : own) close(bi);
    Blk nb;
    nb.ops.push_back(i);
    nb.qm = Q;
    blks.push_back(nb);
    for (int q = 0; q < 64; ++q)
      if (Q >> q & 1) owner[q] = (int)blks.size() - 1;
  }
  for (size_t bi = 0; bi < blks.size(); ++bi) close((int)bi);
  return ord;
}

// Fast-path op list.  SWAPs (a fused run whose product is the swap permutation) are
// not executed: both qubits are tile qubits, so the swap is a relabeling of tile
// positions -- later ops are rewritten to PHYSICAL qubit labels and the final store
// writes position p to logical qubit log_of_phys[tile_q[p]].  Runs that cancel to
// the identity become NOPs (they still carry their gates' error sites).  A run on two
// qubits whose gates cost more than a dense 4x4 (16 FP64 / amplitude) becomes one GEN2
// op; its gates are kept as components for the careful path.
std::vector<FOp> fuse_fast_ops(const PassDesc& pd, const PassPlan& pp,
                               const std::vector<LGate>& gates, bool allow_swap,
                               std::vector<int>& log_of_phys, bool block_reorder) {
  std::vector<FOp> out;
  std::vector<int> phys_of(64);
  for (int q = 0; q < 64; ++q) phys_of[q] = q;
  const int n = (int)(pd.op_end - pd.op_begin);
  auto lg_raw = [&](int li) -> const LGate& { return gates[pp.ops[pd.op_begin + li].gate]; };
  static const bool fuse2 = [] {
    const char* e = std::getenv("TQSIM_FUSE2");
    return !(e && e[0] == '0');
  }();
  std::vector<int> ord(n);
  for (int i = 0; i < n; ++i) ord[i] = i;
  if (block_reorder && fuse2) ord = block_order(n, lg_raw);
  auto lg_of = [&](int i) -> const LGate& { return lg_raw(ord[i]); };
  auto is_map = [&](int i) { return pp.ops[pd.op_begin + ord[i]].role == ROLE_STOREMAP; };
  // With a store map in the pass, SWAP relabelings stay within {0..2} or within the
  // qubits >= 3, so address bits 0..2 stay on physical qubits 0..2.
  bool has_map = false;
  for (int t = 0; t < n; ++t) has_map |= pp.ops[pd.op_begin + t].role == ROLE_STOREMAP;
  bool lowhigh_relabel = false;
  // error effects of the gates [i, e_end] of a run on slots (s0, S1), pushed to the run end
  auto make_sites = [&](FOp& f, int i, int e_end, int s0, int S1) {
    const int slot1 = S1 >= 0 ? S1 : (s0 == 0 ? 1 : 0);
    std::vector<M4> mats;
    for (int t = i; t <= e_end; ++t) mats.push_back(op_matrix(lg_of(t), s0, slot1));
    f.ea = phys_of[s0];
    f.eb = S1 >= 0 ? phys_of[S1] : -1;
    M4 R = M4::id();   // product of the gates after t
    std::vector<ErrSite> sites(e_end - i + 1);
    for (int t = e_end; t >= i; --t) {
      const LGate& lg = lg_of(t);
      ErrSite& es = sites[t - i];
      es.gate = pp.ops[pd.op_begin + ord[t]].gate;
      es.local = (uint32_t)ord[t];
      const M4 Rd = dagger(R);
      auto slot = [&](int q) { return q == s0 ? 0 : 1; };
      const int ncode = lg.two ? 15 : 3;
      for (int c = 1; c <= ncode; ++c) {
        M4 E = lg.two ? pauli4(c >> 2, slot((int)lg.q0), c & 3, slot((int)lg.q1))
                      : pauli4(c, slot((int)lg.q0), 0, 1 - slot((int)lg.q0));
        ErrEff ef = decompose(R.mul(E).mul(Rd));
        auto to_pos = [&](uint32_t m) {   // local slot masks -> physical qubits after the run
          uint32_t r = 0;
          if (m & 1u) r |= 1u << f.ea;
          if (m & 2u) {
            if (f.eb < 0) throw Error{TQSIM_EINTERNAL, "error propagation touched the placeholder slot"};
            r |= 1u << f.eb;
          }
          return r;
        };
        ef.x = to_pos(ef.x);
        ef.z = to_pos(ef.z);
        es.eff.push_back(ef);
      }
      R = R.mul(mats[t - i]);
    }
    f.sites = std::move(sites);
  };
  // one gate as its own op (GEN2 components)
  auto single = [&](int t) {
    const LGate& g = lg_of(t);
    FOp f;
    f.qa = phys_of[g.q0];
    if (g.two && g.op == OP_CX) {
      f.kind = FOp::CX;
      f.qb = phys_of[g.q1];
    } else if (g.two) {   // CZ
      f.kind = FOp::DIAG;
      f.qb = phys_of[g.q1];
      f.d[0] = f.d[1] = f.d[2] = 1.0;
      f.d[3] = -1.0;
    } else if (is_x_gate(g)) {
      f.kind = FOp::XPERM;
    } else if (g.op == OP_DIAG) {
      f.kind = FOp::DIAG;
      f.d[0] = cplx(g.m[0], g.m[1]);
      f.d[1] = cplx(g.m[6], g.m[7]);
      f.d[2] = f.d[0];
      f.d[3] = f.d[1];
    } else {
      f.kind = FOp::GEN;
      for (int k = 0; k < 4; ++k) f.m[k] = cplx(g.m[2 * k], g.m[2 * k + 1]);
    }
    make_sites(f, t, t, (int)g.q0, g.two ? (int)g.q1 : -1);
    return f;
  };
  // gates touching a qubit off the tile (diagonal units / absorbed SWAPs of the first
  // pass, passplan.cpp) may only fuse into a DIAG op or a relabeling, never with tile gates
  auto off_tile = [&](const LGate& g) {
    return !((pd.tile_mask >> phys_of[g.q0]) & 1) || (g.two && !((pd.tile_mask >> phys_of[g.q1]) & 1));
  };
  int i = 0;
  while (i < n) {
    const LGate& g0 = lg_of(i);
    if (is_map(i)) {
      FOp f;
      f.kind = FOp::AMAP;
      f.qa = phys_of[g0.q0];
      f.qb = phys_of[g0.q1];
      if (f.qa < LOW_Q && f.qb >= LOW_Q && pd.leaf_sums)
        throw Error{TQSIM_EINTERNAL, "absorbed CX from a low control in the leaf-sum pass"};
      make_sites(f, i, i, (int)g0.q0, (int)g0.q1);
      out.push_back(f);
      ++i;
      continue;
    }
    const bool restricted = off_tile(g0);
    int s0 = (int)g0.q0, s1 = g0.two ? (int)g0.q1 : -1;
    M4 P = op_matrix(g0, s0, s1 < 0 ? (s0 == 0 ? 1 : 0) : s1);
    int best = P.diagonal() ? i : -1, best_swap = -1;
    M4 bestP = P;
    int bs1 = s1, sw1 = -1;
    int jmax = i, cost = gate_cost(g0), gens = cost >= 4 ? 1 : 0;
    M4 Pmax = P;
    // A run [i, j] is fused into one DIAG / NOP op only if every error of its gates can be
    // pushed to the run's end as a monomial (make_sites): the product R_t of the gates after
    // each t must itself be monomial.  (H Tdg T H is the identity, but X after Tdg pushed
    // through T H is (Z - Y)/sqrt 2: such a run is left to the single-gate ops.)
    auto sites_monomial = [&](int j, int S1) {
      const int slot1 = S1 >= 0 ? S1 : (s0 == 0 ? 1 : 0);
      M4 R = M4::id();
      for (int t = j; t > i; --t) {
        R = R.mul(op_matrix(lg_of(t), s0, slot1));
        if (!R.monomial()) return false;
      }
      return true;
    };
    for (int j = i + 1; j < n && j < i + 12; ++j) {
      const LGate& gj = lg_of(j);
      if (is_map(j) || (!restricted && off_tile(gj))) break;
      int ns1 = s1;
      const int qs[2] = {(int)gj.q0, gj.two ? (int)gj.q1 : -1};
      bool ok = true;
      for (int q : qs) {
        if (q < 0 || q == s0 || q == ns1) continue;
        if (ns1 < 0) ns1 = q;
        else ok = false;
      }
      if (!ok) break;
      // (a product over s0 alone used a placeholder second slot on which it acts
      // as the identity, so the 4x4 is unchanged when s1 becomes a real qubit)
      s1 = ns1;
      P = op_matrix(gj, s0, s1 < 0 ? (s0 == 0 ? 1 : 0) : s1).mul(P);
      jmax = j;
      Pmax = P;
      cost += gate_cost(gj);
      gens += gate_cost(gj) >= 4 ? 1 : 0;
      if (P.diagonal()) {
        if (restricted || sites_monomial(j, s1)) {
          best = j;
          bestP = P;
          bs1 = s1;
        }
      } else if (allow_swap && s1 >= 0 && is_swap(P) && sites_monomial(j, s1) &&
                 // with store maps only high-high relabelings: a low-low one could carry a
                 // mapped logical qubit (2 above the leaf level) onto physical 0 / 1, whose
                 // address bits a map must not move (map_ok below)
                 (!has_map || (phys_of[s0] >= LOW_Q && phys_of[s1] >= LOW_Q))) {
        best_swap = j;
        sw1 = s1;
      }
    }
    FOp f;
    int e_end, S1;
    if (restricted && best < 0 && best_swap < 0)
      throw Error{TQSIM_EINTERNAL, "pass planner placed a non-diagonal gate off the tile"};
    if (!restricted && fuse2 && best < 0 && best_swap < 0 && s1 >= 0 && gens >= 2 && cost > 16) {
      // dense 4x4 on (s0, s1): 16 FP64 per amplitude instead of `cost`
      f.kind = FOp::GEN2;
      f.qa = phys_of[s0];
      f.qb = phys_of[s1];
      for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) f.m4[r * 4 + c] = Pmax.a[r][c];
      for (int t = i; t <= jmax; ++t) f.comps.push_back(single(t));
      out.push_back(f);
      i = jmax + 1;
      continue;
    }
    if (best_swap > best) {   // relabel instead of moving amplitudes
      e_end = best_swap;
      S1 = sw1;
      lowhigh_relabel |= (phys_of[s0] < LOW_Q) != (phys_of[sw1] < LOW_Q);
      std::swap(phys_of[s0], phys_of[sw1]);
      f.kind = FOp::NOP;
      f.qa = phys_of[s0];   // the pair of physical qubits the relabeling exchanges
      f.qb = phys_of[sw1];
    } else if (best >= 0) {
      e_end = best;
      S1 = bs1;
      f.kind = FOp::DIAG;
      f.qa = phys_of[s0];
      f.qb = bs1 >= 0 ? phys_of[bs1] : -1;
      for (int k = 0; k < 4; ++k) f.d[k] = bestP.a[k][k];
      bool trivial = true;
      for (int k = 0; k < 4; ++k)
        if (f.d[k] != cplx(1, 0)) trivial = false;
      if (trivial) f.kind = FOp::NOP;
    } else {
      out.push_back(single(i));
      ++i;
      continue;
    }
    make_sites(f, i, e_end, s0, S1);
    out.push_back(f);
    i = e_end + 1;
  }
  // Trailing CX ops -- no later op of the pass (other than store maps and relabelings)
  // touches their qubits -- also become store maps: they then need no registers (fewer
  // phases).  In the leaf-sum pass only those whose target is < 3 or whose control is
  // >= 3, so the stored high address bits stay functions of the physical high bits
  // (leaf runs in one tile); elsewhere a low control only splits 128-byte lines into
  // 32-byte-complete halves.  Not with a low/high relabeling in the pass (address bits
  // 0..2 must stay on physical qubits 0..2 under a map).
  // The composed map must keep the columns of physical qubits 0, 1 (and 2 in the
  // leaf-sum pass) within address bits 0..2: lanes on qubits 0..1 then still store
  // 64-byte-contiguous groups (measured: fully scattered 16-byte stores run at ~60% of
  // the HBM rate, scripts/microbench/io_layout_bench.cu).
  auto map_ok = [&]() {
    uint32_t col[3] = {1u, 2u, 4u};
    for (const FOp& f : out)
      if (f.kind == FOp::AMAP)
        for (int q = 0; q < 3; ++q) col[q] ^= ((col[q] >> f.qa) & 1u) << f.qb;
    return col[0] < 8u && col[1] < 8u && (!pd.leaf_sums || col[2] < 8u);
  };
  if (!lowhigh_relabel) {
    uint64_t touched = 0;
    for (int t = (int)out.size() - 1; t >= 0; --t) {
      FOp& f = out[t];
      if (f.kind == FOp::AMAP || f.kind == FOp::NOP) continue;
      uint64_t qm = 1ull << f.qa;
      if (f.qb >= 0) qm |= 1ull << f.qb;
      if (f.kind == FOp::CX && !(qm & touched)) {
        f.kind = FOp::AMAP;
        if (map_ok()) continue;
        f.kind = FOp::CX;
      }
      touched |= qm;
    }
  }
  if (!map_ok()) throw Error{TQSIM_EINTERNAL, "absorbed CX maps split the 64-byte store groups"};
  log_of_phys.assign(64, 0);
  for (int q = 0; q < 64; ++q) log_of_phys[phys_of[q]] = q;
  return out;
}

// Register layout of one phase: the 4 tile positions R held in registers, the
// other K-4 on thread-index bits.  `coalesced` (the phases that touch HBM: the
// first loads, the last stores) puts lanes on the remaining positions in
// ascending order, so with R free of positions 0..2 lanes 0..2 walk qubits 0..2
// and every warp access covers whole 128-byte lines (measured: scattered lanes
// cost ~30% of HBM throughput, scripts/microbench/stream_bench.cu).  Exchange
// phases put lanes 0..2 on positions of distinct residue mod 3, which makes the
// 16-byte shared-memory accesses conflict-free under tq_swz.
PhaseDesc make_phase_layout(uint64_t R, int K, int low, bool coalesced) {
  for (int p = K - 1; p >= 0 && __builtin_popcountll(R) < RBITS; --p)
    if (!(R >> p & 1) && p >= low) R |= 1ull << p;
  for (int p = 0; p < K && __builtin_popcountll(R) < RBITS; ++p)
    if (!(R >> p & 1)) R |= 1ull << p;
  PhaseDesc P{};
  int rb = 0;
  for (int p = 0; p < K; ++p)
    if (R >> p & 1) P.rpos[rb++] = (uint8_t)p;
  std::vector<int> nonr;
  for (int p = 0; p < K; ++p)
    if (!(R >> p & 1)) nonr.push_back(p);
  std::vector<int> tmap;
  if (!coalesced && nonr.size() >= 3) {
    std::vector<int> rest = nonr;
    for (int r = 0; r < 3; ++r)
      for (size_t i = 0; i < rest.size(); ++i)
        if (rest[i] % 3 == r) {
          tmap.push_back(rest[i]);
          rest.erase(rest.begin() + i);
          break;
        }
    tmap.insert(tmap.end(), rest.begin(), rest.end());
  } else {
    tmap = nonr;
  }
  for (size_t m = 0; m < tmap.size(); ++m) P.tpos[m] = (uint8_t)tmap[m];
  return P;
}

// Layout of a phase that touches HBM, coalesced in the address order `key` (key[p] =
// address bit of tile position p: the physical qubit for loads, the LOGICAL qubit for
// stores after SWAP relabelings): registers padded with the lowest keys >= 5, lanes on
// the rest in ascending key order, so lanes 0..2 walk address bits 0..2 when R holds
// none of them.
// An I/O phase may also hold low address bits in registers when they move as 32-byte
// pairs: address bit 0 in registers (registers k, k | b0 are one LDG/STG.256) plus at
// most one of bits 1, 2; the lanes then start at the lowest other bit.  Measured at the
// full HBM rate of the lane-coalesced layout; bits 0..2 all in registers are not
// (scripts/microbench/io_layout_bench.cu).
bool io_pairs_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TQSIM_IO_PAIRS");
    return !(e && e[0] == '0');
  }();
  return on;
}
bool io_regs_ok(uint64_t R, const int* key, int K) {
  bool has0 = false;
  int low = 0;
  for (int p = 0; p < K; ++p)
    if (R >> p & 1) {
      if (key[p] == 0) has0 = true;
      else if (key[p] < LOW_Q) ++low;
    }
  return has0 && io_pairs_enabled() ? low <= 1 : low == 0 && !has0;
}
// R plus the position of address bit 0 when R holds a low address bit
uint64_t io_with_pair(uint64_t R, const int* key, int K) {
  bool any_low = false;
  int p0 = -1;
  for (int p = 0; p < K; ++p) {
    if ((R >> p & 1) && key[p] < LOW_Q) any_low = true;
    if (key[p] == 0) p0 = p;
  }
  return any_low && p0 >= 0 ? R | 1ull << p0 : R;
}

PhaseDesc make_io_layout(uint64_t R, int K, const int* key) {
  std::vector<int> order(K);
  for (int p = 0; p < K; ++p) order[p] = p;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return key[a] < key[b]; });
  if (__builtin_popcountll(R) < RBITS) R = io_with_pair(R, key, K);
  // pad the registers with address bits 5, 6, ... (lanes keep bits 0..4: every warp
  // access is 512 contiguous bytes, and the leaf run sums a warp holds are consecutive)
  for (int i = 0; i < K && __builtin_popcountll(R) < RBITS; ++i)
    if (!(R >> order[i] & 1) && key[order[i]] >= LOW_Q + 2) R |= 1ull << order[i];
  for (int i = 0; i < K && __builtin_popcountll(R) < RBITS; ++i)
    if (!(R >> order[i] & 1) && key[order[i]] >= LOW_Q) R |= 1ull << order[i];
  for (int i = 0; i < K && __builtin_popcountll(R) < RBITS; ++i)
    if (!(R >> order[i] & 1)) R |= 1ull << order[i];
  PhaseDesc P{};
  int rb = 0;
  for (int p = 0; p < K; ++p)
    if (R >> p & 1) P.rpos[rb++] = (uint8_t)p;
  std::vector<int> lanes;
  for (int i = 0; i < K; ++i)
    if (!(R >> order[i] & 1)) lanes.push_back(order[i]);
  // With low address bits in registers (32-byte pairs) only the leading lanes on the
  // remaining low bits matter for HBM; fill lanes 1..2 with positions of residues mod 3
  // not yet used, which keeps the 16-byte shared-memory accesses of this phase
  // conflict-free under tq_swz (bank group bit b = XOR of position bits = b mod 3).
  bool low_in_regs = false;
  for (int p = 0; p < K; ++p)
    if ((R >> p & 1) && key[p] < LOW_Q) low_in_regs = true;
  int nf = 0;   // leading lanes on low address bits
  while (nf < (int)lanes.size() && key[lanes[nf]] < LOW_Q) ++nf;
  if (low_in_regs) {
    int used = 0;
    for (int j = 0; j < nf; ++j) used |= 1 << (lanes[j] % 3);
    for (int slot = nf; slot < 3 && slot < (int)lanes.size(); ++slot)
      for (int j = slot; j < (int)lanes.size(); ++j)
        if (!(used >> (lanes[j] % 3) & 1)) {
          const int v = lanes[j];
          lanes.erase(lanes.begin() + j);
          lanes.insert(lanes.begin() + slot, v);
          used |= 1 << (v % 3);
          break;
        }
  }
  for (size_t m = 0; m < lanes.size(); ++m) P.tpos[m] = (uint8_t)lanes[m];
  return P;
}

// One schedulable item of a phase plan: tile positions it needs in registers and
// the global qubits it touches (for the order constraints).
struct PItem {
  uint64_t need, qm;
  int idx;
};

// Greedy in-order grouping of items into register phases with commuting
// look-ahead (an item moves ahead of deferred items only if it shares no qubit
// with them).  Phase 0 is fixed to the register set R0 the kernel loads; the last
// phase is the store layout: when `coal` it must hold no position < low in
// registers, so a trailing re-layout phase is added if the last group needs one.
std::vector<PhaseSpec> plan_phases(const std::vector<PItem>& items, int K, uint64_t R0, bool coal,
                                   const int* store_key, bool runsums_only = false) {
  const int low = std::min(LOW_Q, K);
  const uint64_t lowm = (1ull << low) - 1;
  uint64_t store_low = 0;   // positions of the store's address bits 0..low-1
  bool same_low = true;     // the load's and the store's low lanes coincide
  for (int p = 0; p < K; ++p)
    if (store_key[p] < low) {
      store_low |= 1ull << p;
      if (store_key[p] != p) same_low = false;
    }
  std::vector<std::pair<std::vector<int>, uint64_t>> groups;
  std::vector<int> remaining(items.size());
  for (size_t i = 0; i < items.size(); ++i) remaining[i] = (int)i;
  bool first = true;
  while (first || !remaining.empty()) {
    uint64_t used = first ? R0 : 0, blocked = 0;
    std::vector<int> in, deferred;
    for (int ii : remaining) {
      const PItem& it = items[ii];
      if (it.qm & blocked) {
        deferred.push_back(ii);
        blocked |= it.qm;
        continue;
      }
      const bool ok = first ? (it.need & ~R0) == 0 : __builtin_popcountll(used | it.need) <= RBITS;
      if (ok) {
        used |= it.need;
        in.push_back(ii);
      } else {
        deferred.push_back(ii);
        blocked |= it.qm;
      }
    }
    if (!first && in.empty()) throw Error{TQSIM_EINTERNAL, "phase planner made no progress"};
    groups.emplace_back(std::move(in), used);
    remaining.swap(deferred);
    first = false;
  }
  if (coal) {
    const uint64_t last_regs = io_with_pair(groups.size() == 1 ? R0 : groups.back().second, store_key, K);
    const bool st_ok = __builtin_popcountll(last_regs) <= RBITS && io_regs_ok(last_regs, store_key, K);
    // a pass that stores no state (leaf run sums / the run recompute) needs no coalesced store
    // layout: when its last phase already holds the run's low qubits in registers, the run
    // sums are register sums and the extra (empty) exchange phase is dropped
    const uint64_t last_R = groups.size() == 1 ? R0 : groups.back().second;
    const bool runs_in_regs = (last_R & store_low) == store_low && groups.size() > 1;
    if (!(runsums_only && runs_in_regs) && (!st_ok || (groups.size() == 1 && !same_low)))
      groups.emplace_back(std::vector<int>(), 0);
  }
  (void)lowm;
  std::vector<PhaseSpec> out;
  int load_key[64];
  for (int p = 0; p < K; ++p) load_key[p] = p;
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    PhaseSpec ps;
    const bool ld = gi == 0, st = gi + 1 == groups.size();
    const uint64_t R = gi == 0 ? R0 : groups[gi].second;
    if (st && coal) ps.P = make_io_layout(R, K, store_key);
    else if (ld) ps.P = make_io_layout(R, K, load_key);
    else ps.P = make_phase_layout(R, K, low, st);
    for (int ii : groups[gi].first) ps.items.push_back(items[ii].idx);
    out.push_back(ps);
  }
  return out;
}

// Register set of the load phase: as many leading items as fit in 4 positions
// >= low (positions 0..low-1 stay on lanes: coalesced), padded with high positions.
uint64_t choose_load_regs(const std::vector<PItem>& items, int K, bool coal, bool allow_low) {
  const int low = std::min(LOW_Q, K);
  const uint64_t lowm = (1ull << low) - 1;
  int load_key[64];
  for (int p = 0; p < K; ++p) load_key[p] = p;
  uint64_t used = 0, blocked = 0;
  for (const PItem& it : items) {
    if (it.qm & blocked) continue;
    const uint64_t nu = coal ? io_with_pair(used | it.need, load_key, K) : used | it.need;
    const bool ok = __builtin_popcountll(nu) <= RBITS &&
                    (!coal || (allow_low ? io_regs_ok(nu, load_key, K) : !(nu & lowm)));
    if (ok) used = nu;
    else blocked |= it.qm;
  }
  PhaseDesc P = make_io_layout(used, K, load_key);
  uint64_t R = 0;
  for (int b = 0; b < RBITS; ++b) R |= 1ull << P.rpos[b];
  return R;
}

// variant (leaf-sum passes only): 0 = store the state (and run sums); 1 = run sums only,
// no state store, the instance's store-address frame XOR to xlout; 2 = recompute one
// tile per leaf (tiles[s]) and store only the 8 amplitudes of run runsel[s] to scratch.
// resident threads per SM the register budget targets (TQSIM_JIT_THREADS_PER_SM, default 512:
// 16 warps at <= 128 registers / thread), as many independent CTAs as fit; the clean
// (error-free work item) kernels carry no Pauli-frame state and take their own target
// (TQSIM_JIT_CLEAN_THREADS_PER_SM, default the same).  The __launch_bounds__ minimum of a
// K-qubit-tile kernel of T threads, and the resident CTAs persistent grids are sized by.
int jit_ctas_per_sm(int K, int T, bool clean) {
  static const int tps = [] {
    const char* e = std::getenv("TQSIM_JIT_THREADS_PER_SM");
    return e ? std::max(128, std::atoi(e)) : 512;
  }();
  static const int tps_clean = [] {
    const char* e = std::getenv("TQSIM_JIT_CLEAN_THREADS_PER_SM");
    return e ? std::max(128, std::atoi(e)) : tps;
  }();
  return K >= 13 ? 1
                 : std::max(1, std::min((clean ? tps_clean : tps) / std::max(T, 32),
                                        (int)((227 * 1024) / ((16 << K) + 1024))));
}

std::string gen_pass(const PassDesc& pd, const PassPlan& pp, const std::vector<LGate>& gates,
                     int n, int mode, const std::string& name, int& threads, size_t& smem,
                     std::vector<double>& coefs, int variant = 0,
                     std::vector<uint32_t>* out_row = nullptr, double* fp64_out = nullptr, int proj_m = 0,
                     const TmaGeom* tma = nullptr, bool clean = false) {
  const int K = pd.K, T = 1 << (K - RBITS);
  const int low = std::min(LOW_Q, K);
  const bool coal = K - RBITS >= low;   // enough lane bits to keep qubits 0..2 on lanes 0..2
  const uint32_t CROW = noise_row_bytes(pd.slice_len);
  const int nops = (int)(pd.op_end - pd.op_begin);
  int qpos[64];
  for (int q = 0; q < 64; ++q) qpos[q] = -1;
  for (int p = 0; p < K; ++p) qpos[pd.tile_q[p]] = p;
  auto posm = [&](int qa, int qb) { return (1ull << qpos[qa]) | (qb >= 0 ? 1ull << qpos[qb] : 0ull); };
  auto qmk = [&](int qa, int qb) { return (1ull << qa) | (qb >= 0 ? 1ull << qb : 0ull); };

  // Two candidate op lists -- gates in pass order, or regrouped into 2-qubit blocks (more
  // dense 4x4 fusion) -- each planned into phases; the cheaper one by a per-amplitude
  // cost model (FP64 ops of the fused ops + a shared-memory exchange per extra phase)
  // is generated.
  std::vector<int> log_of_phys;
  std::vector<FOp> fops;
  std::vector<PhaseSpec> fast;
  uint64_t R0 = 0;
  int store_key[64];   // the store writes tile position p to logical qubit log_of_phys[tile_q[p]]
  double best_cost = 0.0;
  // (x2: the load phase may or may not take low address bits into registers as 32-byte
  // pairs -- the greedy load choice is not monotone in phases)
  for (int cand = 0; cand < 4; ++cand) {
    std::vector<int> lop;
    std::vector<FOp> ops = fuse_fast_ops(pd, pp, gates, true, lop, (cand & 1) == 1);
    // diagonal ops need no register slot (index bits are known, jit below)
    std::vector<PItem> items;
    double fcost = 0.0;
    for (size_t i = 0; i < ops.size(); ++i) {
      const FOp& f = ops[i];
      const bool noreg = f.kind == FOp::DIAG || f.kind == FOp::NOP || f.kind == FOp::AMAP;
      if (!noreg && (qpos[f.qa] < 0 || (f.qb >= 0 && qpos[f.qb] < 0)))
        throw Error{TQSIM_EINTERNAL, "a register op on a qubit off the tile"};
      items.push_back({noreg ? 0ull : posm(f.qa, f.qb), qmk(f.qa, f.qb), (int)i});
      fcost += f.kind == FOp::GEN2 ? 16.0 : f.kind == FOp::GEN ? 8.0 : f.kind == FOp::DIAG ? 1.0 : 0.0;
    }
    // One phase plan for both paths: the error-free fast path and the careful path,
    // which runs the same fused ops under a run-time Pauli frame (below).
    const uint64_t r0 = choose_load_regs(items, K, coal, cand >= 2);
    int skey[64];
    for (int p = 0; p < K; ++p) skey[p] = lop[pd.tile_q[p]];
    std::vector<PhaseSpec> ph = plan_phases(items, K, r0, coal, skey,
                                            pd.leaf_sums && (variant == 1 || variant == 2) &&
                                                std::getenv("TQSIM_RUNSUM_PHASE") == nullptr);
    const double cost = fcost + 12.0 * (double)ph.size();
    if (cand == 0 || cost < best_cost) {
      best_cost = cost;
      if (fp64_out) *fp64_out = fcost;
      fops = std::move(ops);
      fast = std::move(ph);
      R0 = r0;
      (void)R0;
      log_of_phys = lop;
      for (int p = 0; p < K; ++p) store_key[p] = skey[p];
    }
  }
  // Store map: the store writes the amplitude at physical index i to address P(i) =
  // L(M(i)), M the absorbed CX gates (GF(2)-linear, composed in op order over physical
  // qubits) and L the SWAP relabeling (physical -> logical bit).  pcol[q] = P(e_q).
  bool has_map = false;
  uint32_t pcol[32];
  {
    uint32_t col[32];
    for (int q = 0; q < 32; ++q) col[q] = q < n ? 1u << q : 0u;
    for (const FOp& f : fops)
      if (f.kind == FOp::AMAP) {
        has_map = true;
        for (int q = 0; q < n; ++q) col[q] ^= ((col[q] >> f.qa) & 1u) << f.qb;
      }
    for (int q = 0; q < 32; ++q) {
      pcol[q] = 0;
      for (int j = 0; j < n; ++j)
        if (col[q] >> j & 1) pcol[q] |= 1u << log_of_phys[j];
    }
    for (int q = 0; has_map && pd.leaf_sums && q < std::min(n, LOW_Q); ++q)
      if (pcol[q] >= (1u << LOW_Q) || !pcol[q])
        throw Error{TQSIM_EINTERNAL, "store map moves address bits 0..2"};
  }
  bool store_moves = false;   // some amplitude is stored at an address other than its own
  for (int q = 0; q < n; ++q) store_moves |= pcol[q] != (1u << q);
  if (out_row) {   // per out-of-tile qubit: the stored-address bits whose parity is its bit
    // invert P over GF(2): rows of P^-1 (Gauss-Jordan on [P | I], row r = address bit r)
    std::vector<uint64_t> A(n);   // bits 0..n-1: P, bits 32..32+n-1: identity
    for (int r = 0; r < n; ++r) {
      uint64_t v = 1ull << (32 + r);
      for (int c = 0; c < n; ++c)
        if (pcol[c] >> r & 1) v |= 1ull << c;
      A[r] = v;
    }
    for (int c = 0; c < n; ++c) {
      int piv = -1;
      for (int r = c; r < n; ++r)
        if (A[r] >> c & 1) { piv = r; break; }
      if (piv < 0) throw Error{TQSIM_EINTERNAL, "store map is singular"};
      std::swap(A[c], A[piv]);
      for (int r = 0; r < n; ++r)
        if (r != c && (A[r] >> c & 1)) A[r] ^= A[c];
    }
    // now row c of [I | P^-1]: physical bit c = parity(P^-1 row c & address)
    out_row->clear();
    for (int i = 0; i < pd.n_out; ++i) out_row->push_back((uint32_t)(A[pd.out_q[i]] >> 32));
  }
  if (const char* e = std::getenv("TQSIM_JIT_DEBUG")) {
    if (e[0] == '1') {
      std::fprintf(stderr, "[tqsim jit] %s: %d ops -> %zu fused ops; %zu phases\n", name.c_str(), nops,
                   fops.size(), fast.size());
      for (size_t ph = 0; ph < fast.size(); ++ph) {
        std::fprintf(stderr, "   phase %zu R=", ph);
        for (int b = 0; b < RBITS; ++b) std::fprintf(stderr, "%d,", pd.tile_q[fast[ph].P.rpos[b]]);
        std::fprintf(stderr, " ops:");
        static const char* kn[] = {"G", "X", "CX", "D", "NOP", "G2", "M"};
        for (int it : fast[ph].items)
          std::fprintf(stderr, " %s(%d,%d)", kn[(int)fops[it].kind], fops[it].qa, fops[it].qb);
        std::fprintf(stderr, "\n");
      }
    }
  }
  // TQSIM_NEXT_PF=1: persistent run-sum / projection loops prefetch the next item's tile into L2
  static const bool next_pf_env = [] {
    const char* e = std::getenv("TQSIM_NEXT_PF");
    return e && e[0] == '1';
  }();
  const bool next_pf = next_pf_env && !tma;
  const bool use_smem = fast.size() > 1;
  threads = T;
  smem = use_smem ? (size_t)16 << K : 0;
  if (tma) smem = 128 + ((size_t)32 << K);   // 2 mbarriers + two tile buffers (prefetch / current)
  Gen g;
  std::ostringstream& o = g.o;
  ConstPool pool;
  {
    const char* e = std::getenv("TQSIM_JIT_COEF");   // "0" = parameter mode
    pool.mode = (e && e[0] == '0') ? 0 : 2;
  }
  g_pool = &pool;
  // Careful-path tables.  GOFF: slice-relative gate index of pass op li (its noise
  // code is codes[4 + GOFF[li]]).  ERRX/ERRZ[li * 16 + c]: the propagated error of
  // code c of op li -- ERRX: bits 0..29 X mask (physical qubits), 30..31 phase power
  // k; ERRZ: Z mask (Pauli-type) or 0x80000000 | index into GD (generic: 4 complex
  // diagonal entries).
  std::vector<uint32_t> errx((size_t)std::max(nops, 1) * 16, 0u), errz(errx.size(), 0u);
  std::vector<double> gd;
  std::map<std::vector<double>, uint32_t> gd_index;
  // every op with error sites (GEN2 components included), in emission order
  std::vector<const FOp*> site_ops;
  std::function<void(const FOp&)> collect = [&](const FOp& f) {
    if (f.kind == FOp::GEN2) {
      for (const FOp& cf : f.comps) collect(cf);
      return;
    }
    if (!f.sites.empty()) site_ops.push_back(&f);
  };
  for (const FOp& f : fops) collect(f);
  std::map<const FOp*, uint32_t> site_off;   // op -> offset of its sites in SITES
  std::vector<uint32_t> site_list;
  for (const FOp* f : site_ops) {
    site_off[f] = (uint32_t)site_list.size();
    for (const ErrSite& es : f->sites) site_list.push_back(es.local);
  }
  for (const FOp* fp : site_ops)
    for (const ErrSite& es : fp->sites)
      for (size_t c = 0; c < es.eff.size(); ++c) {
        const ErrEff& ef = es.eff[c];
        if (ef.x >> 30 || ef.z >> 30) throw Error{TQSIM_EINTERNAL, "error frame needs qubits < 30"};
        uint32_t wx = ef.x | ((ef.k & 3u) << 30), wz = ef.z;
        if (ef.generic) {
          std::vector<double> key;
          for (int i = 0; i < 4; ++i) {
            key.push_back(ef.D[i].real());
            key.push_back(ef.D[i].imag());
          }
          auto it = gd_index.find(key);
          uint32_t di;
          if (it == gd_index.end()) {
            di = (uint32_t)(gd.size() / 8);
            gd_index[key] = di;
            gd.insert(gd.end(), key.begin(), key.end());
          } else {
            di = it->second;
          }
          wz = 0x80000000u | di;
        }
        errx[(size_t)es.local * 16 + c + 1] = wx;
        errz[(size_t)es.local * 16 + c + 1] = wz;
      }
  o << "static __constant__ unsigned short SITES[" << std::max<size_t>(site_list.size(), 1) << "] = {";
  for (size_t i = 0; i < site_list.size(); ++i) o << (i ? "," : "") << site_list[i];
  if (site_list.empty()) o << "0";
  o << "};\n";
  // gate offsets inside the slice (a slice may exceed 65,535 lowered gates: flat plans)
  o << "static __constant__ " << (pd.slice_len > 65535u ? "tq_u32" : "unsigned short") << " GOFF["
    << std::max(nops, 1) << "] = {";
  for (int i = 0; i < nops; ++i) o << (i ? "," : "") << (pp.ops[pd.op_begin + i].gate - pd.slice_begin);
  if (!nops) o << "0";
  o << "};\nstatic __device__ const tq_u32 ERRX[" << errx.size() << "] = {";
  for (size_t i = 0; i < errx.size(); ++i) o << (i ? "," : "") << errx[i] << "u";
  o << "};\nstatic __device__ const tq_u32 ERRZ[" << errz.size() << "] = {";
  for (size_t i = 0; i < errz.size(); ++i) o << (i ? "," : "") << errz[i] << "u";
  o << "};\nstatic __device__ const double GD[" << std::max<size_t>(gd.size(), 8) << "] = {";
  for (size_t i = 0; i < gd.size(); ++i) o << (i ? "," : "") << hexd(gd[i]);
  if (gd.empty()) o << "0.0";
  o << "};\n";
  const int NW = std::max(1, (nops + 31) / 32);
  const int minb = jit_ctas_per_sm(K, T, clean);
  if (tma) {
    // per-kernel work scan and TMA issue: the next computed (representative) work item, and
    // the tensor-map coordinates of its tile (TmaGeom: runs of tile / out-of-tile qubits)
    // warp 0 scans 32 candidates (w, w + G, ...) per step: one dedup-map round trip per 32
    o << "__device__ __forceinline__ tq_u64 tq_next_item(const TqJitArgs& a, tq_u64 w, tq_u64 total) {\n"
      << "  const tq_u32 lane = threadIdx.x & 31u;\n"
      << "  for (; w < total; w += 32ull * gridDim.x) {\n"
      << "    const tq_u64 c = w + (tq_u64)lane * gridDim.x;\n"
      << "    bool ok = false;\n"
      << "    if (c < total) { const tq_u32 s = (tq_u32)(c % a.batch); ok = !a.rep || a.rep[s] == s; }\n"
      << "    const unsigned bal = __ballot_sync(0xffffffffu, ok);\n"
      << "    const int f = bal ? __ffs(bal) - 1 : 32;\n"
      << (variant == 1 ? "    if (c < total && (int)lane < f && !ok && c / a.batch == 0) a.xlout[c % a.batch] = 0u;\n" : "")
      << "    if (bal) return w + (tq_u64)f * gridDim.x;\n"
      << "  }\n  return total;\n}\n";
    o << "__device__ __forceinline__ void tq_issue(const TqJitArgs& a, const TqTmap* tm, tq_u64 w, tq_d2* dst,\n"
      << "                                         unsigned long long* bar) {\n"
      << "  const tq_u32 s = (tq_u32)(w % a.batch);\n  const tq_u64 t = w / a.batch;\n";
    if (mode == 1)
      o << "  tq_u64 pj = ((tq_u64)a.child_first + s) / a.arity - a.parent_first;\n  if (a.prep) pj = a.prep[pj];\n";
    else
      o << "  const tq_u64 pj = s;\n";
    std::string c[5];
    for (int dmi = 0; dmi < 5; ++dmi) c[dmi] = "0";
    for (int dmi = 0; dmi < tma->ndims; ++dmi) {
      if (tma->kind[dmi] == 2) c[dmi] = "(int)pj";
      else if (tma->kind[dmi] == 0)
        c[dmi] = "(int)((t >> " + std::to_string(tma->tbit[dmi]) + ") & " + std::to_string((1ull << tma->len[dmi]) - 1) + "ull)";
    }
    o << "  tq_tma_load(dst, tm, bar, " << c[0] << ", " << c[1] << ", " << c[2] << ", " << c[3] << ", " << c[4] << ", "
      << (16u << K) << "u);\n}\n";
  }
  o << "extern \"C\" __global__ void __launch_bounds__(" << T << ", " << std::min(minb, 32) << ") "
    << name << "(const TqJitArgs a, const TqCoef cf" << (tma ? ", const __grid_constant__ TqTmap tmap" : "") << ") {\n";
  if (tma)
    o << "  extern __shared__ __align__(128) unsigned char tq_sm[];\n"
      << "  unsigned long long* const tq_bar = reinterpret_cast<unsigned long long*>(tq_sm);\n"
      << "  tq_d2* const tq_buf0 = reinterpret_cast<tq_d2*>(tq_sm + 128);\n"
      << "  __shared__ tq_u64 tq_next[2];\n";
  else if (use_smem) o << "  extern __shared__ tq_d2 tile[];\n";
  o << "  __shared__ tq_u32 tq_errb[" << std::max(1, T / 32) << "][" << NW << "];   // per warp: the eb words\n";
  o << "  const tq_u32 tid = threadIdx.x;\n  const tq_u64 bid = blockIdx.x;\n";
  if (tma) {
    // persistent CTAs: the next item's tile streams into the other buffer (TMA) while this
    // one is computed; the current buffer doubles as the exchange tile of the phases
    o << "  const tq_u64 tq_total = (tq_u64)a.batch << " << pd.n_out << ";\n"
      << "  if (tid == 0u) { tq_mbar_init(tq_bar); tq_mbar_init(tq_bar + 1); tq_fence_mbar_init(); }\n"
      << "  __syncthreads();\n"
      << "  if (tid < 32u) {\n    const tq_u64 w0 = tq_next_item(a, bid, tq_total);\n"
      << "    if (tid == 0u) { tq_next[0] = w0; if (w0 < tq_total) tq_issue(a, &tmap, w0, tq_buf0, tq_bar); }\n  }\n"
      << "  __syncthreads();\n"
      << "  tq_u64 tq_w = tq_next[0];\n  tq_u32 tq_b = 0u, tq_par0 = 0u, tq_par1 = 0u;\n"
      << "  while (tq_w < tq_total) {\n"
      << "  if (tid < 32u) {\n    const tq_u64 nx = tq_next_item(a, tq_w + gridDim.x, tq_total);\n"
      << "    if (tid == 0u) {\n      tq_next[tq_b ^ 1u] = nx;\n"
      << "      if (nx < tq_total) tq_issue(a, &tmap, nx, tq_buf0 + ((tq_u64)(tq_b ^ 1u) << " << K << "), tq_bar + (tq_b ^ 1u));\n    }\n  }\n"
      << "  tq_mbar_wait(tq_bar + tq_b, tq_b ? tq_par1 : tq_par0);\n"
      << "  if (tq_b) tq_par1 ^= 1u; else tq_par0 ^= 1u;\n"
      << "  const tq_u32 s = (tq_u32)(tq_w % a.batch);\n  const tq_u64 t = tq_w / a.batch;\n"
      << "  tq_d2* const tile = tq_buf0 + ((tq_u64)tq_b << " << K << ");\n";
  } else if (variant == 2)   // one CTA per leaf, on the tile holding its selected run
    o << "  const tq_u32 s = (tq_u32)bid;\n  const tq_u64 t = a.tiles[s];\n  const tq_u32 rsel = a.runsel[s];\n";
  else if (variant == 0)
    o << "  const tq_u32 s = (tq_u32)(bid % a.batch);\n  const tq_u64 t = bid / a.batch;\n";
  else   // leaf run sums / projection: every (instance, tile), or the instances of a work list
         // (dedup representatives / projection hand-overs) with persistent CTAs
  {
    // the next item's index (and, fan-out, its parent slot) is loaded one item ahead, so the
    // dependent index loads (work list -> parent map -> tile) do not stall each item's start
    // item order: tile-major (w = i + nw t: concurrent CTAs take the same tile of many
    // instances) or instance-major (w = t + 2^n_out i: concurrent CTAs sweep consecutive
    // tiles of few instances).  Instance-major for states of <= 256 tiles (C2's leaf pass
    // 0.90 -> 0.86 ms per tree; neutral on C3/C4: profiles/r02_ab_item_order.txt);
    // TQSIM_ITEM_ORDER=0/1 forces one.
    static const int order_env = [] {
      const char* e = std::getenv("TQSIM_ITEM_ORDER");
      return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    const bool inst_major = order_env >= 0 ? order_env == 1 : pd.n_out <= 8;
    o << "  const tq_u32 nw = a.wlist ? *a.wcount : a.batch;\n"
      << "  const tq_u64 tq_tot = (tq_u64)nw << " << pd.n_out << ";\n";
    if (inst_major)
      o << "  const tq_u32 tq_gm = (tq_u32)(gridDim.x >> " << pd.n_out << ");\n"
        << "  const tq_u64 tq_gd = gridDim.x & " << ((1ull << pd.n_out) - 1) << "ull;\n"
        << "  tq_u32 tq_i = (tq_u32)(bid >> " << pd.n_out << ");\n  tq_u64 tq_t = bid & " << ((1ull << pd.n_out) - 1)
        << "ull;\n";
    else
      o << "  const tq_u32 tq_gm = nw ? (tq_u32)(gridDim.x % nw) : 0u;\n"
        << "  const tq_u64 tq_gd = nw ? gridDim.x / nw : 0ull;\n"
        << "  tq_u32 tq_i = nw ? (tq_u32)(bid % nw) : 0u;\n  tq_u64 tq_t = nw ? bid / nw : 0ull;\n";
    o << "  tq_u32 tq_snx = 0u;\n"
      << "  if (bid < tq_tot) tq_snx = a.wlist ? a.wlist[tq_i] : tq_i;\n";
    if (mode == 1)
      o << "  tq_u64 tq_pnx = ((tq_u64)a.child_first + tq_snx) / a.arity - a.parent_first;\n"
        << "  if (a.prep && bid < tq_tot) tq_pnx = a.prep[tq_pnx];\n";
    o << "  for (tq_u64 w = bid; w < tq_tot; w += gridDim.x) {\n"
      << "  const tq_u32 s = tq_snx;\n  const tq_u64 t = tq_t;\n";
    if (mode == 1) o << "  const tq_u64 tq_pcur = tq_pnx;\n";
    if (inst_major)
      o << "  tq_i += tq_gm;\n  tq_t += tq_gd;\n  if (tq_t >= " << (1ull << pd.n_out) << "ull) { tq_t -= "
        << (1ull << pd.n_out) << "ull; ++tq_i; }\n";   // w + gridDim.x
    else
      o << "  tq_i += tq_gm;\n  tq_t += tq_gd;\n  if (tq_i >= nw) { tq_i -= nw; ++tq_t; }\n";   // w + gridDim.x
    o << "  const tq_u64 tq_wn = w + gridDim.x;\n"
      << "  if (tq_wn < tq_tot) tq_snx = a.wlist ? a.wlist[tq_i] : tq_i;\n";
  }
  if (variant == 3)   // the leaf's chosen top bits (the select kernel's chunk)
    o << "  const tq_u32 hsel = a.runsel[s];\n";
  if (variant != 2 && !tma) {
    // An instance that shares its representative's state (dedup map, launch_dedup_map:
    // no error in its slice, same effective parent) is not computed; readers go through
    // the map.  A skipped leaf's store-address XOR is 0.
    // (a variant-1 work list holds representatives only: compact_reps_kernel)
    o << (variant == 1 ? "  if (!a.wlist && a.rep && a.rep[s] != s) {\n" : "  if (a.rep && a.rep[s] != s) {\n")
      << (variant == 1 ? "    if (t == 0 && tid == 0u) a.xlout[s] = 0u;\n" : "")
      << ((variant == 1 || variant == 3) && mode == 1   // keep the look-ahead parent slot current
              ? "    if (tq_wn < tq_tot) {\n      tq_pnx = ((tq_u64)a.child_first + tq_snx) / a.arity - a.parent_first;\n"
                "      if (a.prep) tq_pnx = a.prep[tq_pnx];\n    }\n"
              : "")
      << (tma || variant == 0 ? "    return;\n" : "    continue;\n")
      << "  }\n";
  }
  o << "  tq_u32 gtile = 0u, gtile_st = 0u;\n";   // the tile's out-of-tile index bits: physical / stored
  for (int i = 0; i < pd.n_out; ++i)
    o << "  gtile |= (tq_u32)((t >> " << i << ") & 1ull) << " << (int)pd.out_q[i] << "; gtile_st ^= (0u - (tq_u32)((t >> "
      << i << ") & 1ull)) & " << pcol[pd.out_q[i]] << "u;\n";
  o << "  tq_d2* __restrict__ dst = a.dst + ((tq_u64)s << " << n << ");\n";
  const bool ahead = (variant == 1 || variant == 3) && !tma;   // the loop above loads indices ahead
  if (mode == 1 && ahead)
    o << "  const tq_u64 pj = tq_pcur;\n"
      << "  const tq_d2* __restrict__ src = a.src + (pj << " << n << ");\n";
  else if (mode == 1)   // fan-out src: the parent, or (skipped duplicate parent) its representative
    o << "  tq_u64 pj = ((tq_u64)a.child_first + s) / a.arity - a.parent_first;\n"
      << "  if (a.prep) pj = a.prep[pj];\n"
      << "  const tq_d2* __restrict__ src = a.src + (pj << " << n << ");\n";
  else if (mode == 2 && variant == 2) {
    // recompute of a leaf whose state was not computed (an error-free duplicate): its
    // representative's slot holds the same state
    o << "  const tq_u32 sr = a.rep ? a.rep[s] : s;\n"
      << "  const tq_d2* src = a.dst + ((tq_u64)sr << " << n << ");\n";
  } else if (mode == 2)
    o << "  const tq_d2* src = dst;\n";
  o << "  tq_d2 r0, r1, r2, r3, r4, r5, r6, r7, r8, r9, r10, r11, r12, r13, r14, r15;\n";

  // phase-0 registers, shared by both paths: the parent state in the first pass of a
  // node (fused fan-out), |0..0> at the root, else the node's own state
  uint32_t lo_last[16];   // tile-local position offsets of the registers (last offsets() call)
  auto offsets = [&](const PhaseDesc& P, const std::vector<int>* lq, uint32_t* goff, uint32_t* soff,
                     std::string& lb, std::string& gb) {
    // column of tile position p: the physical bit, or (lq: the store) its image P(e_q)
    auto col = [&](int p) { return lq ? pcol[pd.tile_q[p]] : 1u << pd.tile_q[p]; };
    std::ostringstream l, gg;
    l << "0u";
    gg << (lq ? "gtile_st" : "gtile");
    for (int m = 0; m < K - RBITS; ++m) {
      l << " | (((tid >> " << m << ") & 1u) << " << (int)P.tpos[m] << ")";
      const uint32_t c = col(P.tpos[m]);
      if (__builtin_popcount(c) == 1)
        gg << " ^ (((tid >> " << m << ") & 1u) << " << __builtin_ctz(c) << ")";
      else
        gg << " ^ ((0u - ((tid >> " << m << ") & 1u)) & " << c << "u)";
    }
    for (int k = 0; k < 16; ++k) {
      uint32_t go = 0, lo = 0;
      for (int b = 0; b < RBITS; ++b)
        if (k >> b & 1) {
          go ^= col(P.rpos[b]);
          lo |= 1u << P.rpos[b];
        }
      goff[k] = go;
      soff[k] = host_swz(lo);
      lo_last[k] = lo;
    }
    lb = l.str();
    gb = gg.str();
  };
  // register bit whose offset is address bit 0 (-1: none): such register pairs move as
  // one 32-byte access (tq_ld2 / tq_st2)
  // (store: only when address bit 0 is the image of one physical bit alone)
  int bit0_cols = 0;
  for (int q = 0; q < n; ++q) bit0_cols += pcol[q] & 1u;
  auto pair_bit = [&](const uint32_t* go, bool store) {
    if (store && bit0_cols != 1) return -1;
    for (int b = 0; b < RBITS; ++b)
      if (go[1 << b] == 1u) return b;
    return -1;
  };
  auto emit_load = [&]() {
    uint32_t goff[16], soff[16];
    std::string lb, gb;
    offsets(fast[0].P, nullptr, goff, soff, lb, gb);
    o << "  {\n    const tq_u32 gb = " << gb << ";\n";
    const int b0 = pair_bit(goff, false);
    if (tma) {   // the tile is in shared memory (TMA box order = tile-local index)
      for (int k = 0; k < 16; ++k) o << "    r" << k << " = tile[(" << lb << ") | " << lo_last[k] << "u];\n";
      if (fast.size() > 1) o << "    __syncthreads();\n";   // the buffer becomes the exchange tile
      o << "  }\n";
      return;
    }
    for (int k = 0; k < 16; ++k) {
      if (mode == 0)
        o << "    r" << k << ".x = (gb + " << goff[k] << "u == 0u) ? 1.0 : 0.0; r" << k << ".y = 0.0;\n";
      else if (b0 < 0)
        o << "    r" << k << " = tq_ld(src + (gb + " << goff[k] << "u));\n";
      else if (!(k >> b0 & 1))   // address bit 0 in registers: 32-byte pair
        o << "    tq_ld2(src + (gb + " << goff[k] << "u), r" << k << ", r" << (k | 1 << b0) << ");\n";
    }
    o << "  }\n";
    if (next_pf && (variant == 1 || variant == 3) && mode != 0) {
      // persistent loop: the CTA's NEXT work item's tile is prefetched into L2 while this one is
      // computed (no registers held; its loads then wait on L2, not HBM)
      o << "  {\n    const tq_u64 wn = w + gridDim.x;\n"
        << "    if (wn < ((tq_u64)nw << " << pd.n_out << ")) {\n"
        << "      const tq_u32 sn = a.wlist ? a.wlist[wn % nw] : (tq_u32)(wn % nw);\n"
        << "      const tq_u64 tn = wn / nw;\n      tq_u32 gtn = 0u;\n";
      for (int i = 0; i < pd.n_out; ++i)
        o << "      gtn |= (tq_u32)((tn >> " << i << ") & 1ull) << " << (int)pd.out_q[i] << ";\n";
      if (mode == 1)
        o << "      tq_u64 pjn = ((tq_u64)a.child_first + sn) / a.arity - a.parent_first;\n"
          << "      if (a.prep) pjn = a.prep[pjn];\n"
          << "      const tq_d2* srcn = a.src + (pjn << " << n << ");\n";
      else
        o << "      const tq_d2* srcn = a.dst + ((tq_u64)sn << " << n << ");\n";
      o << "      const tq_u32 gbn = gtn" << gb.substr(5) << ";\n";
      for (int k = 0; k < 16; ++k) {
        if (b0 >= 0 && (k >> b0 & 1)) continue;
        o << "      asm volatile(\"prefetch.global.L2 [%0];\" :: \"l\"(srcn + (gbn + " << goff[k] << "u)));\n";
      }
      o << "    }\n  }\n";
    }
  };
  emit_load();
  if (mode == 1 && ahead)   // the next item's parent slot (its index arrived during the tile loads)
    o << "  if (tq_wn < tq_tot) {\n"
      << "    tq_pnx = ((tq_u64)a.child_first + tq_snx) / a.arity - a.parent_first;\n"
      << "    if (a.prep) tq_pnx = a.prep[tq_pnx];\n  }\n";
  // noise row of the instance (launch_noise_rows): error-free instances (the common
  // case) run the fused fast path, the others apply each keyed Pauli after its gate
  o << "  const unsigned char* __restrict__ codes = a.rows + (tq_u64)s * " << CROW << "u;\n";
  o << "  const tq_u32 emask = __ldg(reinterpret_cast<const unsigned int*>(codes));\n";
  if (pd.mask_any)   // trail passes: any error in the slice (their bits are not in the row mask)
    o << "  const bool errs = emask != 0u;\n";
  else
    o << "  const bool errs = (emask >> " << std::min<uint32_t>(pd.pass_index, 31) << ") & 1u;\n";

  bool sc_used = false;   // a fast phase scaled the run sums by the run-time tq_sc
  // TQSIM_FRAME_FLUSH=1: careful phases flush the Pauli frame into the exchange tile (see the
  // phase store).  Off by default: measured slower (C2 1.94 -> 2.01 ms, C4 trail pass 154 ->
  // 159 ms per tree; profiles/r02_ab_frame_flush.txt) -- the flush costs more than the fast
  // phases it enables; parity-tested on (the full GPU suite passed with it on)
  static const bool flush_frame = [] {
    const char* e = std::getenv("TQSIM_FRAME_FLUSH");
    return e && e[0] == '1';
  }();
  auto emit_phases = [&](const std::vector<PhaseSpec>& specs, bool with_errors, int ph_only) {
  // amap_upto[ph]: an absorbed CX (store-map op) among the ops of phases 0..ph
  std::vector<char> amap_upto(specs.size(), 0);
  {
    std::function<bool(const FOp&)> has_amap = [&](const FOp& f) {
      if (f.kind == FOp::AMAP) return true;
      for (const FOp& c : f.comps)
        if (has_amap(c)) return true;
      return false;
    };
    bool seen = false;
    for (size_t q = 0; q < specs.size(); ++q) {
      for (int it : specs[q].items) seen = seen || has_amap(fops[it]);
      amap_upto[q] = seen;
    }
  }
  const int nph = (int)specs.size();
  for (int ph = 0; ph < nph; ++ph) {
    if (ph != ph_only) continue;
    const PhaseDesc& P = specs[ph].P;
    const bool last = ph == nph - 1;
    g.reset_map();
    uint32_t goff[16], soff[16];
    std::string lbs, gbs;
    offsets(P, nullptr, goff, soff, lbs, gbs);
    o << "  { // phase " << ph << "\n";
    if (ph > 0) {
      o << "    __syncthreads();\n    const tq_u32 sb = tq_swz(" << lbs << ");\n";
      for (int k = 0; k < 16; ++k) o << "    r" << k << " = tile[sb ^ " << soff[k] << "u];\n";
      o << "    __syncthreads();\n";
    }
    // Error-free path: monomial gates (CX, CZ, X, diagonal) are composed at code
    // generation time into a register renaming + a pending phase per logical
    // amplitude, folded into the next general gate's coefficients or applied once
    // at the end of the phase.  Exact up to fp rounding (R30).
    cplx dph[16];
    for (int k = 0; k < 16; ++k) dph[k] = cplx(1.0, 0.0);
    double sum_scale = 1.0;   // run sums x this (variant 1, last phase; see the flush)
    auto permute = [&](auto perm) {   // new logical k <- old logical perm(k)
      int nrm[16];
      cplx nd[16];
      for (int k = 0; k < 16; ++k) {
        nrm[k] = g.rm[perm(k)];
        nd[k] = dph[perm(k)];
      }
      for (int k = 0; k < 16; ++k) {
        g.rm[k] = nrm[k];
        dph[k] = nd[k];
      }
    };
    // register bit of a global qubit in this phase (-1: not in registers)
    auto rbit = [&](int q) {
      for (int b = 0; b < RBITS; ++b)
        if (pd.tile_q[P.rpos[b]] == q) return b;
      return -1;
    };
    bool gph_on = false, gph_decl = false;
    // a thread-bit diagonal joins the common factor gph (declared once per phase; reset to 1
    // after a flush folded it into the registers)
    auto gph_begin = [&]() {
      if (!gph_decl) o << "    double gphx = 1.0, gphy = 0.0;\n";
      else if (!gph_on) o << "    gphx = 1.0; gphy = 0.0;\n";
      gph_decl = gph_on = true;
    };
    int fb_gen = 0;
    struct FBv {
      bool on = false;
      bool one[2] = {true, true};   // F_b[v] still exactly 1 (never assigned)
      std::string var[2];
    };
    FBv fb[RBITS];
    for (int b = 0; b < RBITS; ++b)
      for (int v = 0; v < 2; ++v) fb[b].var[v] = "fb" + std::to_string(b) + "_" + std::to_string(v);
    std::set<std::string> declared;
    // apply pending F_b to the registers (before an op mixing bit b), then reset it
    auto fb_flush = [&](int b, int& gen) {
      if (b < 0 || !fb[b].on) return;
      // A flush that multiplies all 16 registers also takes the pending common factor gph
      // (a per-thread scalar: it commutes with every register op), two per-thread products
      // instead of 16 register multiplies at the phase end.
      const bool fold = gph_on && !fb[b].one[0] && !fb[b].one[1];
      std::string X[2];
      for (int v = 0; v < 2; ++v) {
        if (fb[b].one[v]) continue;
        X[v] = fb[b].var[v];
        if (fold) {
          const std::string nm = X[v] + "p";
          o << "    const double " << nm << "r = fma(" << X[v] << "r, gphx, -" << X[v] << "i * gphy), " << nm
            << "i = fma(" << X[v] << "r, gphy, " << X[v] << "i * gphx);\n";
          X[v] = nm;
        }
      }
      if (fold) gph_on = false;
      for (int k = 0; k < 16; ++k) {
        const int v = (k >> b) & 1;
        if (X[v].empty()) continue;
        const std::string r = g.r(k);
        o << "    { const tq_d2 x = " << r << "; " << r << ".x = fma(" << X[v] << "r, x.x, -" << X[v] << "i * x.y); " << r
          << ".y = fma(" << X[v] << "r, x.y, " << X[v] << "i * x.x); }\n";
      }
      ++gen;
      fb[b] = FBv();
      for (int v = 0; v < 2; ++v)
        fb[b].var[v] = "fb" + std::to_string(b) + "_" + std::to_string(v) + "g" + std::to_string(gen);
    };
    if (!with_errors) {
      // run-time index bits of the qubits diagonal ops need outside the registers
      uint64_t rtq = 0;
      for (int it : specs[ph].items) {
        const FOp& f = fops[it];
        if (f.kind != FOp::DIAG) continue;
        if (rbit(f.qa) < 0) rtq |= 1ull << f.qa;
        if (f.qb >= 0 && rbit(f.qb) < 0) rtq |= 1ull << f.qb;
      }
      if (rtq) {
        o << "    const tq_u32 gbp = " << gbs << ";\n";
        for (int q = 0; q < 64; ++q)
          if (rtq >> q & 1) o << "    const bool rt" << q << " = (gbp >> " << q << ") & 1u;\n";
      }
      // Diagonals on (thread bit, register bit b) accumulate into per-thread factors
      // F_b[0], F_b[1] (one per value of logical register bit b), applied once -- at
      // the phase end through a product tree, or before an op that mixes bit b.
      Zyz zyz;
      for (int it : specs[ph].items) {
        const FOp& f = fops[it];
        if (f.kind == FOp::CX) {
          const int ba = rbit(f.qa), bb = rbit(f.qb);
          fb_flush(bb, fb_gen);
          permute([&](int k) { return k ^ (((k >> ba) & 1) << bb); });
        } else if (f.kind == FOp::XPERM) {
          const int ba = rbit(f.qa);
          std::swap(fb[ba].var[0], fb[ba].var[1]);
          std::swap(fb[ba].one[0], fb[ba].one[1]);
          permute([&](int k) { return k ^ (1 << ba); });
        } else if (f.kind == FOp::GEN && hadamard_like(f.m)) {
          // c * (+-1 entries), e.g. H: a butterfly of adds.  The pair's pending phases
          // stay pending when equal (the gate commutes with a common factor), else the
          // second input is multiplied by the ratio; c and the signs join the pending
          // phases (applied once at the phase end, or folded into a later gate).
          const int ba = rbit(f.qa);
          fb_flush(ba, fb_gen);
          std::ostringstream oo;
          pool.begin_op();
          const double c = std::abs(f.m[0].real());
          double sg[4];
          for (int e = 0; e < 4; ++e) sg[e] = f.m[e].real() > 0 ? 1.0 : -1.0;
          for (int k = 0; k < 16; ++k) {
            if (k >> ba & 1) continue;
            const int k1 = k | 1 << ba;
            const std::string va = g.r(k), vb = g.r(k1);
            const cplx p = dph[k];
            const cplx q = snap(dph[k1] / p);
            if (q != cplx(1.0, 0.0))   // (zero parts skipped: a factor +-i is a swap with a sign)
              oo << "      { const tq_d2 y = " << vb << "; " << vb << ".x = " << lin(q.real(), q.imag(), "y", 0, 0, "y", false)
                 << "; " << vb << ".y = " << lin(q.real(), q.imag(), "y", 0, 0, "y", true) << "; }\n";
            // out_r = s_r0 * (x + (s_r1 / s_r0) y)
            const char* op0 = sg[1] * sg[0] > 0 ? " + " : " - ";
            const char* op1 = sg[3] * sg[2] > 0 ? " + " : " - ";
            oo << "      { const tq_d2 x = " << va << ", y = " << vb << "; " << va << ".x = x.x" << op0 << "y.x; " << va
               << ".y = x.y" << op0 << "y.y; " << vb << ".x = x.x" << op1 << "y.x; " << vb << ".y = x.y" << op1
               << "y.y; }\n";
            dph[k] = p * (sg[0] * c);
            dph[k1] = p * (sg[2] * c);
          }
          o << "    {\n" << pool.decl.str() << oo.str() << "    }\n";
        } else if (f.kind == FOp::GEN && zyz_of(f.m, zyz)) {
          // U = e^{ia} diag(1, e^{if}) [[c, -s], [s, c]] diag(1, e^{il}): the right phase joins
          // the second input's pending phase (a ratio multiply when the pair's phases then
          // differ), the left phases and the larger of c, s join the outputs' pending phases,
          // and the core is [[1, -t], [t, 1]] or [[u, -1], [1, u]] (|t|, |u| <= 1): one FMA per
          // output component instead of two to four (RX, RY, U3 cores).
          const int ba = rbit(f.qa);
          fb_flush(ba, fb_gen);
          std::ostringstream oo;
          pool.begin_op();
          const bool by_c = std::abs(zyz.c) >= std::abs(zyz.s);
          const double r = by_c ? zyz.s / zyz.c : zyz.c / zyz.s, sc = by_c ? zyz.c : zyz.s;
          for (int k = 0; k < 16; ++k) {
            if (k >> ba & 1) continue;
            const int k1 = k | 1 << ba;
            const std::string va = g.r(k), vb = g.r(k1);
            const cplx p = dph[k];
            const cplx q = snap(zyz.el * dph[k1] / p);
            if (q != cplx(1.0, 0.0))
              oo << "      { const tq_d2 y = " << vb << "; " << vb << ".x = " << lin(q.real(), q.imag(), "y", 0, 0, "y", false)
                 << "; " << vb << ".y = " << lin(q.real(), q.imag(), "y", 0, 0, "y", true) << "; }\n";
            const std::string R = g_pool->ref(r), NR = g_pool->ref(-r);
            oo << "      { const tq_d2 x = " << va << ", y = " << vb << ";\n";
            if (by_c)   // (x - t y, t x + y)
              oo << "        " << va << ".x = fma(" << NR << ", y.x, x.x); " << va << ".y = fma(" << NR << ", y.y, x.y); "
                 << vb << ".x = fma(" << R << ", x.x, y.x); " << vb << ".y = fma(" << R << ", x.y, y.y); }\n";
            else        // (u x - y, x + u y)
              oo << "        " << va << ".x = fma(" << R << ", x.x, -y.x); " << va << ".y = fma(" << R << ", x.y, -y.y); "
                 << vb << ".x = fma(" << R << ", y.x, x.x); " << vb << ".y = fma(" << R << ", y.y, x.y); }\n";
            dph[k] = snap(p * zyz.ea * sc);
            dph[k1] = snap(p * zyz.eaf * sc);
          }
          o << "    {\n" << pool.decl.str() << oo.str() << "    }\n";
        } else if (f.kind == FOp::GEN) {
          const int ba = rbit(f.qa);
          fb_flush(ba, fb_gen);
          std::ostringstream oo;
          pool.begin_op();
          for (int k = 0; k < 16; ++k) {
            if (k >> ba & 1) continue;
            const int k1 = k | 1 << ba;
            const cplx a00 = f.m[0] * dph[k], a01 = f.m[1] * dph[k1], a10 = f.m[2] * dph[k], a11 = f.m[3] * dph[k1];
            dph[k] = dph[k1] = cplx(1.0, 0.0);
            const std::string va = g.r(k), vb = g.r(k1);
            oo << "      { const tq_d2 x = " << va << ", y = " << vb << ";\n";
            oo << "        " << va << ".x = " << lin(a00.real(), a00.imag(), "x", a01.real(), a01.imag(), "y", false) << ";\n";
            oo << "        " << va << ".y = " << lin(a00.real(), a00.imag(), "x", a01.real(), a01.imag(), "y", true) << ";\n";
            oo << "        " << vb << ".x = " << lin(a10.real(), a10.imag(), "x", a11.real(), a11.imag(), "y", false) << ";\n";
            oo << "        " << vb << ".y = " << lin(a10.real(), a10.imag(), "x", a11.real(), a11.imag(), "y", true) << "; }\n";
          }
          o << "    {\n" << pool.decl.str() << oo.str() << "    }\n";
        } else if (f.kind == FOp::GEN2) {   // dense 4x4 on two register bits
          const int ba = rbit(f.qa), bb = rbit(f.qb);
          fb_flush(ba, fb_gen);
          fb_flush(bb, fb_gen);
          std::ostringstream oo;
          pool.begin_op();
          for (int k = 0; k < 16; ++k) {
            if ((k >> ba & 1) || (k >> bb & 1)) continue;
            int idx[4];
            std::string v[4], x[4];
            for (int j = 0; j < 4; ++j) {
              idx[j] = k | ((j & 1) << ba) | ((j >> 1) << bb);
              v[j] = g.r(idx[j]);
              x[j] = "x" + std::to_string(j);
            }
            oo << "      { const tq_d2 x0 = " << v[0] << ", x1 = " << v[1] << ", x2 = " << v[2] << ", x3 = " << v[3]
               << ";\n";
            for (int r = 0; r < 4; ++r) {
              cplx c[4];
              for (int j = 0; j < 4; ++j) c[j] = f.m4[r * 4 + j] * dph[idx[j]];   // pending input phases
              oo << "        " << v[r] << ".x = " << linN(c, x, 4, false) << ";\n";
              oo << "        " << v[r] << ".y = " << linN(c, x, 4, true) << ";\n";
            }
            oo << "      }\n";
            for (int j = 0; j < 4; ++j) dph[idx[j]] = cplx(1.0, 0.0);
          }
          o << "    {\n" << pool.decl.str() << oo.str() << "    }\n";
        } else if (f.kind == FOp::DIAG) {
          const int ra = rbit(f.qa), rb = f.qb >= 0 ? rbit(f.qb) : -2;
          const bool rta = ra < 0, rtb = rb == -1;
          auto entry = [&](int bita, int bitb) { return f.d[bita | (bitb << 1)]; };
          if (!rta && !rtb) {
            for (int k = 0; k < 16; ++k) dph[k] *= entry(k >> ra & 1, rb >= 0 ? (k >> rb & 1) : 0);
          } else if (rta && (rtb || rb == -2)) {   // factor common to the 16 amplitudes
            std::ostringstream oo;
            pool.begin_op();
            std::string sel_r, sel_i;
            auto val = [&](const cplx& v, bool im) { return g_pool->ref(im ? v.imag() : v.real()); };
            if (rb == -2) {
              sel_r = "(rt" + std::to_string(f.qa) + " ? " + val(entry(1, 0), false) + " : " + val(entry(0, 0), false) + ")";
              sel_i = "(rt" + std::to_string(f.qa) + " ? " + val(entry(1, 0), true) + " : " + val(entry(0, 0), true) + ")";
            } else {
              const std::string A = "rt" + std::to_string(f.qa), B = "rt" + std::to_string(f.qb);
              auto sel = [&](bool im) {
                return "(" + B + " ? (" + A + " ? " + val(entry(1, 1), im) + " : " + val(entry(0, 1), im) + ") : (" +
                       A + " ? " + val(entry(1, 0), im) + " : " + val(entry(0, 0), im) + "))";
              };
              sel_r = sel(false);
              sel_i = sel(true);
            }
            gph_begin();
            oo << "      { const double fr = " << sel_r << ", fi = " << sel_i << ";\n"
               << "        const double tx = fma(gphx, fr, -gphy * fi); gphy = fma(gphx, fi, gphy * fr); gphx = tx; }\n";
            o << "    {\n" << pool.decl.str() << oo.str() << "    }\n";
          } else {   // one register bit, one run-time bit
            const bool a_reg = !rta;
            const int rbit_reg = a_reg ? ra : rb;
            const std::string RT = "rt" + std::to_string(a_reg ? f.qb : f.qa);
            std::ostringstream oo;
            pool.begin_op();
            for (int bk = 0; bk < 2; ++bk) {
              // e0 / e1: the entry for thread bit 0 / 1 at register-bit value bk
              const cplx e0 = a_reg ? entry(bk, 0) : entry(0, bk), e1 = a_reg ? entry(bk, 1) : entry(1, bk);
              if (e0 == e1) {   // independent of the thread bit: a compile-time phase
                for (int k = 0; k < 16; ++k)
                  if ((k >> rbit_reg & 1) == bk) dph[k] *= e0;
                continue;
              }
              FBv& F = fb[rbit_reg];
              const std::string fr = RT + " ? " + g_pool->ref(e1.real()) + " : " + g_pool->ref(e0.real());
              const std::string fi = RT + " ? " + g_pool->ref(e1.imag()) + " : " + g_pool->ref(e0.imag());
              const std::string& X = F.var[bk];
              if (F.one[bk]) {
                if (!declared.count(X)) {
                  o << "    double " << X << "r, " << X << "i;\n";
                  declared.insert(X);
                }
                oo << "      " << X << "r = " << fr << "; " << X << "i = " << fi << ";\n";
                F.one[bk] = false;
              } else {
                oo << "      { const double er = " << fr << ", ei = " << fi << ";\n"
                   << "        const double t = fma(" << X << "r, er, -" << X << "i * ei); " << X << "i = fma(" << X
                   << "r, ei, " << X << "i * er); " << X << "r = t; }\n";
              }
              F.on = true;
            }
            o << "    {\n" << pool.decl.str() << oo.str() << "    }\n";
          }
        }
      }
    }
    if (with_errors) {
      // Careful path: the same fused ops on the stored state psi_s, with the true state
      // = F psi_s for the run-time Pauli frame F = i^fk X^fx Z^fz (tile positions,
      // uniform per CTA).  Cliffords (CX, X) run unchanged and conjugate the frame;
      // GEN / DIAG ops run conjugated by the frame (F^+ U F); each drawn error, pushed
      // to the end of its fused run at code generation time (ERRX/ERRZ), multiplies into the
      // frame (and, for errors inside diagonal runs, applies a diagonal).  The frame is
      // applied at the store (address XOR + phase).  Exact up to fp rounding (R30).
      o << "    const tq_u32 lth = " << lbs << ";\n";
      auto pos_bit = [&](int q, const std::string& frame_bit_var, int k, std::string& expr) {
        // index bit of physical qubit q for register k (compile-time, thread bit, or --
        // outside the tile -- the CTA's tile-index bit) ^ frame bit
        const int pos = qpos[q];
        int rb = -1;
        for (int b = 0; b < RBITS; ++b)
          if (pos >= 0 && P.rpos[b] == pos) rb = b;
        const std::string fb = frame_bit_var;
        if (rb >= 0) expr = "(" + fb + " ^ " + std::to_string((k >> rb) & 1) + "u)";
        else if (pos >= 0) expr = "(" + fb + " ^ ((lth >> " + std::to_string(pos) + ") & 1u))";
        else expr = "(" + fb + " ^ ((gtile >> " + std::to_string(q) + ") & 1u))";
        return rb;
      };
      // apply a diagonal with entries E(i) (i = bit_qa | bit_qb << 1, physical qubits)
      // under the frame: register k gets E((bits of k's index) ^ (frame X bits))
      auto emit_frame_diag = [&](int qa, int qb, const std::string* ent /*8 exprs re,im x4*/,
                                 bool rt_entries) {
        const int pb = qb;
        o << "      { const tq_u32 xa = (fx >> " << qa << ") & 1u";
        if (qb >= 0) o << ", xb = (fx >> " << qb << ") & 1u";
        o << ";\n";
        // classes of registers by (bit at qa, bit at qb)
        std::map<std::string, std::vector<int>> cls;
        for (int k = 0; k < 16; ++k) {
          std::string ea, eb = "0u";
          pos_bit(qa, "xa", k, ea);
          if (qb >= 0) pos_bit(qb, "xb", k, eb);
          cls["(" + ea + " | (" + eb + " << 1))"].push_back(k);
        }
        int ci = 0;
        for (auto& kv : cls) {
          bool all_one = !rt_entries;
          if (!rt_entries)
            for (int i = 0; i < (pb >= 0 ? 4 : 2); ++i)
              if (ent[2 * i] != "1.0" || ent[2 * i + 1] != "0.0") all_one = false;
          if (all_one) continue;
          o << "        { const tq_u32 ic = " << kv.first << ";\n";
          // compile-time entries with few non-unit values (CP, CZ: one): a uniform branch per
          // non-unit entry, so only the registers whose (frame-shifted) index selects it pay
          // a complex multiply
          int nonunit = 0;
          for (int i = 0; i < (pb >= 0 ? 4 : 2); ++i)
            if (ent[2 * i] != "1.0" || ent[2 * i + 1] != "0.0") ++nonunit;
          if (!rt_entries && nonunit <= 2) {
            for (int i = 0; i < (pb >= 0 ? 4 : 2); ++i) {
              if (ent[2 * i] == "1.0" && ent[2 * i + 1] == "0.0") continue;
              o << "          if (ic == " << i << "u) {\n";
              for (int k : kv.second) {
                const std::string v = g.r(k);
                o << "            { const tq_d2 x = " << v << "; " << v << ".x = fma(" << ent[2 * i] << ", x.x, -("
                  << ent[2 * i + 1] << ") * x.y); " << v << ".y = fma(" << ent[2 * i] << ", x.y, (" << ent[2 * i + 1]
                  << ") * x.x); }\n";
              }
              o << "          }\n";
            }
            o << "        }\n";
            ++ci;
            continue;
          }
          auto sel = [&](int part) {
            if (pb < 0) return "(ic & 1u) ? " + ent[2 + part] + " : " + ent[part];
            return "(ic & 2u) ? ((ic & 1u) ? " + ent[6 + part] + " : " + ent[4 + part] + ") : ((ic & 1u) ? " +
                   ent[2 + part] + " : " + ent[part] + ")";
          };
          o << "          const double fr = " << sel(0) << ", fi = " << sel(1) << ";\n";
          for (int k : kv.second) {
            const std::string v = g.r(k);
            o << "          { const tq_d2 x = " << v << "; " << v << ".x = fma(fr, x.x, -fi * x.y); " << v
              << ".y = fma(fr, x.y, fi * x.x); }\n";
          }
          o << "        }\n";
          ++ci;
        }
        o << "      }\n";
      };
      std::function<void(const FOp&)> emit_careful = [&](const FOp& f) {
        if (f.kind == FOp::GEN2) {   // its gates one by one, each with its own errors
          for (const FOp& cf : f.comps) emit_careful(cf);
          return;
        }

        if (f.kind == FOp::CX) {
          const int ba = rbit(f.qa), bb = rbit(f.qb);
          fb_flush(bb, fb_gen);
          permute([&](int k) { return k ^ (((k >> ba) & 1) << bb); });
          o << "    fx ^= ((fx >> " << f.qa << ") & 1u) << " << f.qb << "; fz ^= ((fz >> " << f.qb << ") & 1u) << "
            << f.qa << ";\n";
        } else if (f.kind == FOp::AMAP) {   // applied by the store map: conjugate the frame only
          o << "    fx ^= ((fx >> " << f.qa << ") & 1u) << " << f.qb << "; fz ^= ((fz >> " << f.qb << ") & 1u) << "
            << f.qa << ";\n";
        } else if (f.kind == FOp::XPERM) {
          const int ba = rbit(f.qa);
          std::swap(fb[ba].var[0], fb[ba].var[1]);
          std::swap(fb[ba].one[0], fb[ba].one[1]);
          permute([&](int k) { return k ^ (1 << ba); });
          o << "    fk += ((fz >> " << f.qa << ") & 1u) << 1;\n";
        } else if (f.kind == FOp::GEN) {
          // F^+ U F on this qubit: variant v = x | z << 1 of Z^z X^x U X^x Z^z
          const int ba = rbit(f.qa);
          fb_flush(ba, fb_gen);
          cplx V[4][4];   // [v][entry]
          for (int v = 0; v < 4; ++v) {
            cplx u[4] = {f.m[0], f.m[1], f.m[2], f.m[3]};
            if (v & 1) { cplx t[4] = {u[3], u[2], u[1], u[0]}; for (int i = 0; i < 4; ++i) u[i] = t[i]; }
            if (v & 2) { u[1] = -u[1]; u[2] = -u[2]; }
            for (int i = 0; i < 4; ++i) V[v][i] = u[i];
          }
          bool hl = true;
          for (int v = 0; v < 4; ++v) hl = hl && hadamard_like(V[v]) && std::abs(V[v][0].real()) == std::abs(V[0][0].real());
          if (hl) {
            // Hadamard-like: V_v = diag(s00, s10) h [[1, a], [1, b]] (a = s01 s00, b = s11 s10):
            // registers get the add/sub butterfly, h joins the (uniform) pending phases, and
            // diag(s00, s10) = s00 Z^[s10 != s00] joins the frame (fk += 2, fz ^= e_q)
            const double h = std::abs(V[0][0].real());
            double sa[4], sb[4];
            int gneg[4], zfl[4];
            for (int v = 0; v < 4; ++v) {
              const double s00 = V[v][0].real() > 0 ? 1 : -1, s01 = V[v][1].real() > 0 ? 1 : -1;
              const double s10 = V[v][2].real() > 0 ? 1 : -1, s11 = V[v][3].real() > 0 ? 1 : -1;
              sa[v] = s01 * s00;
              sb[v] = s11 * s10;
              gneg[v] = s00 < 0 ? 1 : 0;
              zfl[v] = s10 != s00 ? 1 : 0;
            }
            std::ostringstream oo;
            oo << "      const tq_u32 v = ((fx >> " << f.qa << ") & 1u) | (((fz >> " << f.qa << ") & 1u) << 1);\n";
            auto sel4 = [&](const double* t) {
              std::ostringstream e;
              e << "((v & 2u) ? ((v & 1u) ? " << t[3] << ".0 : " << t[2] << ".0) : ((v & 1u) ? " << t[1] << ".0 : " << t[0] << ".0))";
              return e.str();
            };
            auto bits4 = [&](const int* t) { return (unsigned)(t[0] | t[1] << 1 | t[2] << 2 | t[3] << 3); };
            oo << "      const double sa = " << sel4(sa) << ", sb = " << sel4(sb) << ";\n";
            oo << "      fk += ((" << bits4(gneg) << "u >> v) & 1u) << 1;\n";
            oo << "      fz ^= ((" << bits4(zfl) << "u >> v) & 1u) << " << f.qa << ";\n";
            for (int k = 0; k < 16; ++k) {
              if (k >> ba & 1) continue;
              const std::string va = g.r(k), vb = g.r(k | 1 << ba);
              oo << "      { const tq_d2 x = " << va << ", y = " << vb << "; " << va << ".x = fma(sa, y.x, x.x); " << va
                 << ".y = fma(sa, y.y, x.y); " << vb << ".x = fma(sb, y.x, x.x); " << vb << ".y = fma(sb, y.y, x.y); }\n";
            }
            for (int k = 0; k < 16; ++k) dph[k] *= h;   // uniform: commutes with every later op
            o << "    {\n" << oo.str() << "    }\n";
          } else if (sign_variants(V)) {
            // V_v = c [[1, sg_v u], [sg_v w, 1]] (RX, RY: the frame only flips the sign of the
            // off-diagonal): one FMA per output component per nonzero part of u / w, c joins
            // the (uniform) pending phases
            const double c = V[0][0].real();
            const cplx u = V[0][1] / c, w = V[0][2] / c;
            unsigned neg = 0;
            for (int v = 0; v < 4; ++v)
              if (std::abs(V[v][1] + V[0][1]) < 1e-15 && std::abs(V[0][1]) > 0) neg |= 1u << v;
            pool.begin_op();
            std::ostringstream oo;
            oo << "      const tq_u32 v = ((fx >> " << f.qa << ") & 1u) | (((fz >> " << f.qa << ") & 1u) << 1);\n";
            oo << "      const double sg = ((" << neg << "u >> v) & 1u) ? -1.0 : 1.0;\n";
            auto term = [&](double cv, const std::string& src, std::string& e) {   // e += sg*cv*src
              if (cv == 0.0) return;
              e = "fma(sg * " + g_pool->ref(cv) + ", " + src + ", " + e + ")";
            };
            for (int k = 0; k < 16; ++k) {
              if (k >> ba & 1) continue;
              const std::string va = g.r(k), vb = g.r(k | 1 << ba);
              std::string a0 = "x.x", a1 = "x.y", b0 = "y.x", b1 = "y.y";
              // out0 = x + sg u y: re += u.re y.x - u.im y.y, im += u.re y.y + u.im y.x
              term(u.real(), "y.x", a0); term(-u.imag(), "y.y", a0);
              term(u.real(), "y.y", a1); term(u.imag(), "y.x", a1);
              // out1 = y + sg w x
              term(w.real(), "x.x", b0); term(-w.imag(), "x.y", b0);
              term(w.real(), "x.y", b1); term(w.imag(), "x.x", b1);
              oo << "      { const tq_d2 x = " << va << ", y = " << vb << "; " << va << ".x = " << a0 << "; " << va
                 << ".y = " << a1 << "; " << vb << ".x = " << b0 << "; " << vb << ".y = " << b1 << "; }\n";
            }
            for (int k = 0; k < 16; ++k) dph[k] *= c;
            o << "    {\n" << pool.decl.str() << oo.str() << "    }\n";
          } else {
          pool.begin_op();
          std::ostringstream oo;
          oo << "      const tq_u32 v = ((fx >> " << f.qa << ") & 1u) | (((fz >> " << f.qa << ") & 1u) << 1);\n";
          std::string cr[4], ci[4];   // coefficient expressions
          bool zr[4], zi[4];
          for (int e = 0; e < 4; ++e) {
            for (int part = 0; part < 2; ++part) {
              double val[4];
              bool same = true, zero = true;
              for (int v = 0; v < 4; ++v) {
                val[v] = part ? V[v][e].imag() : V[v][e].real();
                if (val[v] != val[0]) same = false;
                if (val[v] != 0.0) zero = false;
              }
              std::string ex;
              if (same) ex = g_pool->ref(val[0]);
              else {
                const std::string nm = "c" + std::to_string(e) + (part ? "i" : "r");
                oo << "      const double " << nm << " = (v & 2u) ? ((v & 1u) ? " << g_pool->ref(val[3]) << " : "
                   << g_pool->ref(val[2]) << ") : ((v & 1u) ? " << g_pool->ref(val[1]) << " : " << g_pool->ref(val[0])
                   << ");\n";
                ex = nm;
              }
              (part ? ci[e] : cr[e]) = ex;
              (part ? zi[e] : zr[e]) = zero;
            }
          }
          // re/im of a*x + b*y with coefficient expressions (zero terms skipped)
          auto linx = [&](int ea_, const std::string& x, int eb_, const std::string& y, bool imag) {
            std::vector<std::string> t;
            if (!imag) {
              if (!zr[ea_]) t.push_back(cr[ea_] + " * " + x + ".x");
              if (!zi[ea_]) t.push_back("-" + ci[ea_] + " * " + x + ".y");
              if (!zr[eb_]) t.push_back(cr[eb_] + " * " + y + ".x");
              if (!zi[eb_]) t.push_back("-" + ci[eb_] + " * " + y + ".y");
            } else {
              if (!zr[ea_]) t.push_back(cr[ea_] + " * " + x + ".y");
              if (!zi[ea_]) t.push_back(ci[ea_] + " * " + x + ".x");
              if (!zr[eb_]) t.push_back(cr[eb_] + " * " + y + ".y");
              if (!zi[eb_]) t.push_back(ci[eb_] + " * " + y + ".x");
            }
            if (t.empty()) return std::string("0.0");
            std::string e = t[0];
            for (size_t i = 1; i < t.size(); ++i) e += " + " + t[i];
            return "(" + e + ")";
          };
          for (int k = 0; k < 16; ++k) {
            if (k >> ba & 1) continue;
            const std::string va = g.r(k), vb = g.r(k | 1 << ba);
            oo << "      { const tq_d2 x = " << va << ", y = " << vb << ";\n";
            oo << "        " << va << ".x = " << linx(0, "x", 1, "y", false) << ";\n";
            oo << "        " << va << ".y = " << linx(0, "x", 1, "y", true) << ";\n";
            oo << "        " << vb << ".x = " << linx(2, "x", 3, "y", false) << ";\n";
            oo << "        " << vb << ".y = " << linx(2, "x", 3, "y", true) << "; }\n";
          }
          o << "    {\n" << pool.decl.str() << oo.str() << "    }\n";
          }
        } else if (f.kind == FOp::DIAG) {
          pool.begin_op();
          const int ra = rbit(f.qa), rb = f.qb >= 0 ? rbit(f.qb) : -2;
          const bool rta = ra < 0, rtb = rb == -1;
          auto entry = [&](int bita, int bitb) { return f.d[bita | (bitb << 1)]; };
          auto val = [&](const cplx& v, bool im) { return g_pool->ref(im ? v.imag() : v.real()); };
          // thread bit of qubit q XOR its frame bit (frame-conjugated diagonal: D(i ^ x))
          auto tbit = [&](int q) {   // off the tile: the CTA's tile-index bit
            const std::string ib = qpos[q] >= 0 ? "(lth >> " + std::to_string(qpos[q]) + ")" : "(gtile >> " + std::to_string(q) + ")";
            return "((" + ib + " ^ (fx >> " + std::to_string(q) + ")) & 1u)";
          };
          if (!rta && !rtb) {   // both register bits: applied now (frame-dependent, no folding)
            std::string ent[8];
            for (int i = 0; i < 4; ++i) {
              const cplx d = f.d[i];
              ent[2 * i] = d.real() == 1.0 ? "1.0" : d.real() == 0.0 ? "0.0" : g_pool->ref(d.real());
              ent[2 * i + 1] = d.imag() == 0.0 ? "0.0" : g_pool->ref(d.imag());
            }
            o << "    {\n" << pool.decl.str();
            emit_frame_diag(f.qa, f.qb, ent, false);
            o << "    }\n";
          } else if (rta && (rtb || rb == -2)) {   // thread bits only: into the common factor
            std::ostringstream oo;
            const std::string A = tbit(f.qa), B = rb == -2 ? std::string("0u") : tbit(f.qb);
            auto sel = [&](bool im) {
              return "(" + B + " ? (" + A + " ? " + val(entry(1, 1), im) + " : " + val(entry(0, 1), im) + ") : (" +
                     A + " ? " + val(entry(1, 0), im) + " : " + val(entry(0, 0), im) + "))";
            };
            gph_begin();
            oo << "      { const double fr = " << sel(false) << ", fi = " << sel(true) << ";\n"
               << "        const double tx = fma(gphx, fr, -gphy * fi); gphy = fma(gphx, fi, gphy * fr); gphx = tx; }\n";
            o << "    {\n" << pool.decl.str() << oo.str() << "    }\n";
          } else {   // one register bit, one thread bit: per-bit factors F_b[v]
            const bool a_reg = !rta;
            const int rbit_reg = a_reg ? ra : rb, q_reg = a_reg ? f.qa : f.qb, q_rt = a_reg ? f.qb : f.qa;
            const std::string TB = tbit(q_rt), XR = "((fx >> " + std::to_string(q_reg) + ") & 1u)";
            std::ostringstream oo;
            for (int bk = 0; bk < 2; ++bk) {
              // entry at (thread bit t, register value w) in the op's (a, b) orientation
              auto E = [&](int t, int w) { return a_reg ? entry(w, t) : entry(t, w); };
              bool all_one = true;
              for (int t = 0; t < 2; ++t)
                for (int w = 0; w < 2; ++w)
                  if (E(t, w) != cplx(1, 0)) all_one = false;
              if (all_one) continue;
              FBv& F = fb[rbit_reg];
              // register value seen by the diagonal: bk ^ frame bit
              auto sel = [&](bool im) {
                return "(" + XR + " ? (" + TB + " ? " + val(E(1, bk ^ 1), im) + " : " + val(E(0, bk ^ 1), im) +
                       ") : (" + TB + " ? " + val(E(1, bk), im) + " : " + val(E(0, bk), im) + "))";
              };
              const std::string& X = F.var[bk];
              if (F.one[bk]) {
                if (!declared.count(X)) {
                  o << "    double " << X << "r, " << X << "i;\n";
                  declared.insert(X);
                }
                oo << "      " << X << "r = " << sel(false) << "; " << X << "i = " << sel(true) << ";\n";
                F.one[bk] = false;
              } else {
                oo << "      { const double er = " << sel(false) << ", ei = " << sel(true) << ";\n"
                   << "        const double t = fma(" << X << "r, er, -" << X << "i * ei); " << X << "i = fma(" << X
                   << "r, ei, " << X << "i * er); " << X << "r = t; }\n";
              }
              F.on = true;
            }
            o << "    {\n" << pool.decl.str() << oo.str() << "    }\n";
          }
        }
        // the run's drawn errors, in gate order (uniform branch; rare)
        if (!f.sites.empty()) {
          bool any_gen = false;
          for (const ErrSite& es : f.sites)
            for (const ErrEff& ef : es.eff) any_gen |= ef.generic;
          std::map<uint32_t, uint32_t> wm;   // bitmap word -> mask of this op's sites
          for (const ErrSite& es : f.sites) wm[es.local >> 5] |= 1u << (es.local & 31);
          std::ostringstream cond;
          cond << "0u";
          for (auto& kv : wm) cond << " | (eb" << kv.first << " & " << kv.second << "u)";
          const uint32_t so = site_off.at(&f);
          o << "    if (" << cond.str() << ") {\n";
          o << "      for (tq_u32 si = " << so << "u; si < " << so + f.sites.size() << "u; ++si) {\n";
          o << "        const tq_u32 li = SITES[si];\n";
          o << "        if (!((tq_errb[tid >> 5][li >> 5] >> (li & 31u)) & 1u)) continue;\n";
          o << "        const tq_u32 c = codes[4u + GOFF[li]];\n";
          o << "        const tq_u32 wx = __ldg(ERRX + li * 16u + c), wz = __ldg(ERRZ + li * 16u + c);\n";
          o << "        if (!(wz & 0x80000000u)) {\n"
            << "          fk += (wx >> 30) + ((__popc(wz & fx) & 1u) << 1);\n"
            << "          fx ^= wx & 0x3fffffffu; fz ^= wz;\n";
          if (any_gen) {
            o << "        } else {\n          fx ^= wx & 0x3fffffffu;\n"
              << "          const double* __restrict__ D = GD + 8u * (wz & 0x7fffffffu);\n";
            std::string ent[8];
            for (int i = 0; i < 8; ++i) {
              ent[i] = "e" + std::to_string(i);
              o << "          const double e" << i << " = __ldg(D + " << i << ");\n";
            }
            emit_frame_diag(f.ea, f.eb, ent, true);
          }
          o << "        }\n      }\n    }\n";
        }
      };
      for (int it : specs[ph].items) emit_careful(fops[it]);
    }
    {   // flush the pending phases (run-time factors, then compile-time)
      // product tree T[idx] = gph * prod_{b in L} F_b[bit of idx], idx over the pending bits L
      // The leaf variants 1/2 feed only |a|^2: in their last phase the pending run-time
      // factors (diagonal entries: unit modulus) are dropped and the compile-time ones
      // reduce to their modulus.
      const bool mag_only = last && variant != 0 && variant != 3;
      std::vector<int> L;
      for (int b = 0; b < RBITS && !mag_only; ++b)
        if (fb[b].on) L.push_back(b);
      std::vector<std::string> Tn(1, gph_on && !mag_only ? std::string("gph") : std::string());
      int tcount = 0;
      for (size_t li = 0; li < L.size(); ++li) {
        std::vector<std::string> nt(Tn.size() * 2);
        for (size_t i = 0; i < Tn.size(); ++i)
          for (int v = 0; v < 2; ++v) {
            const FBv& F = fb[L[li]];
            if (F.one[v]) { nt[i | (v << li)] = Tn[i]; continue; }
            if (Tn[i].empty()) { nt[i | (v << li)] = F.var[v]; continue; }
            const std::string nm = "tf" + std::to_string(tcount++), A = Tn[i], B = F.var[v];
            auto re = [&](const std::string& x) { return x == "gph" ? std::string("gphx") : x + "r"; };
            auto im = [&](const std::string& x) { return x == "gph" ? std::string("gphy") : x + "i"; };
            o << "    const double " << nm << "r = fma(" << re(A) << ", " << re(B) << ", -" << im(A) << " * " << im(B)
              << "), " << nm << "i = fma(" << re(A) << ", " << im(B) << ", " << im(A) << " * " << re(B) << ");\n";
            nt[i | (v << li)] = nm;
          }
        Tn.swap(nt);
      }
      for (int k = 0; k < 16; ++k) {
        size_t idx = 0;
        for (size_t li = 0; li < L.size(); ++li) idx |= (size_t)((k >> L[li]) & 1) << li;
        const std::string& X = Tn[idx];
        if (X.empty()) continue;
        const std::string xr = X == "gph" ? "gphx" : X + "r", xi = X == "gph" ? "gphy" : X + "i";
        const std::string v = g.r(k);
        o << "    { const tq_d2 x = " << v << "; " << v << ".x = fma(" << xr << ", x.x, -" << xi << " * x.y); " << v
          << ".y = fma(" << xr << ", x.y, " << xi << " * x.x); }\n";
      }
      std::ostringstream oo;
      pool.begin_op();
      // run sums only (variant 1), an earlier phase of the fast path: when no later op of
      // the pass mixes this phase's register qubits (only diagonal ops touch them), the
      // pending per-register phases are unobservable in |a|^2 -- only their modulus is kept,
      // as a run-time factor of the sums when common to the 16 registers
      if (!last && !with_errors && variant == 1 && pd.leaf_sums) {
        uint64_t mixed = 0;
        std::function<void(const FOp&)> mq = [&](const FOp& f) {
          if (f.kind != FOp::DIAG && f.kind != FOp::NOP) {
            if (f.qa >= 0) mixed |= 1ull << f.qa;
            if (f.qb >= 0) mixed |= 1ull << f.qb;
          }
          for (const FOp& c : f.comps) mq(c);
        };
        for (int p2 = ph + 1; p2 < nph; ++p2)
          for (int it : specs[p2].items) mq(fops[it]);
        bool hidden = true;
        for (int b = 0; b < RBITS; ++b) hidden &= !((mixed >> pd.tile_q[P.rpos[b]]) & 1ull);
        if (hidden) {
          const double s0 = std::abs(dph[0]);
          bool uni = true;
          for (int k = 1; k < 16; ++k) uni &= std::abs(dph[k]) == s0;
          if (uni) {
            if (s0 != 1.0) {
              o << "    tq_sc *= " << hexd(s0 * s0) << ";\n";
              sc_used = true;
            }
            for (int k = 0; k < 16; ++k) dph[k] = cplx(1.0, 0.0);
          } else {
            for (int k = 0; k < 16; ++k) dph[k] = snap(cplx(std::abs(dph[k]), 0.0));
          }
        }
      }
      // run sums only (variant 1): a modulus common to the 16 registers scales the sums
      // (one multiply per stored sum) instead of every amplitude
      if (mag_only && variant == 1 && pd.leaf_sums) {
        const double s0 = std::abs(dph[0]);
        bool uni = true;
        for (int k = 1; k < 16; ++k) uni &= std::abs(dph[k]) == s0;
        if (uni && s0 != 1.0) {
          sum_scale = s0 * s0;
          for (int k = 0; k < 16; ++k) dph[k] = cplx(1.0, 0.0);
        }
      }
      for (int k = 0; k < 16; ++k) {
        const cplx d = mag_only ? snap(cplx(std::abs(dph[k]), 0.0)) : dph[k];
        if (d == cplx(1.0, 0.0)) continue;
        const std::string v = g.r(k);
        oo << "      { const tq_d2 x = " << v << "; " << v << ".x = "
           << lin(d.real(), d.imag(), "x", 0, 0, "x", false) << "; " << v << ".y = "
           << lin(d.real(), d.imag(), "x", 0, 0, "x", true) << "; }\n";
      }
      o << "    {\n" << pool.decl.str() << oo.str() << "    }\n";
    }
    if (last) {
      // In place with a single phase, a thread's loads and stores meet no barrier: when
      // the store addresses differ from the loaded ones (a relabeling or store map, or
      // the careful path's frame XOR) another warp may not have loaded them yet.
      if (mode == 2 && nph == 1 && (with_errors || store_moves)) o << "    __syncthreads();\n";
      // fast path: physical tile qubit tile_q[p] holds logical qubit log_of_phys[tile_q[p]]
      uint32_t gofs[16], sofs[16];
      std::string lbx, gbl;
      offsets(P, &log_of_phys, gofs, sofs, lbx, gbl);
      o << "    const tq_u32 gbs = " << gbl << ";\n";
      std::string xl = "";
      if (with_errors) {
        // true state = i^fk X^fx Z^fz psi_s: the amplitude at physical index i goes to
        // i ^ fx, times i^fk (-1)^popc(fz & i); fx mapped to stored (logical) address bits
        uint32_t gph[16], sph[16];
        std::string lbp, gbp;
        offsets(P, nullptr, gph, sph, lbp, gbp);
        o << "    tq_u32 xl = 0u;\n";
        for (int q = 0; q < n; ++q)
          o << "    xl |= ((fx >> " << q << ") & 1u) << " << log_of_phys[q] << ";\n";
        if ((variant == 0 || variant == 3) && !has_map) {   // variants 1/2 feed only |a|^2: the phase does not matter
          o << "    const tq_u32 zt = __popc(fz & (" << gbp << "));\n";
          for (int k = 0; k < 16; ++k)
            o << "    tq_rot(" << g.r(k) << ", fk + ((zt + __popc(fz & " << gph[k] << "u)) << 1));\n";
        } else if (variant == 0 || variant == 3) {
          // the frame acts after the store map: its Z sign is read on the mapped index,
          // i.e. on the stored address with fz relabeled like fx
          o << "    tq_u32 zl = 0u;\n";
          for (int q = 0; q < n; ++q)
            o << "    zl |= ((fz >> " << q << ") & 1u) << " << log_of_phys[q] << ";\n";
          o << "    const tq_u32 zt = __popc(zl & gbs);\n";
          for (int k = 0; k < 16; ++k)
            o << "    tq_rot(" << g.r(k) << ", fk + ((zt + __popc(zl & " << gofs[k] << "u)) << 1));\n";
        }
        xl = " ^ xl";
      }
      if (variant == 0) {
        const int b0 = pair_bit(gofs, true);
        for (int k = 0; k < 16; ++k) {
          if (b0 < 0) {
            o << "    dst[(gbs ^ " << gofs[k] << "u)" << xl << "] = " << g.r(k) << ";\n";
          } else if (!(k >> b0 & 1)) {   // 32-byte pair; a frame X on address bit 0 swaps it
            const std::string ra = g.r(k), rb = g.r(k | 1 << b0);
            if (with_errors)
              o << "    { const tq_u32 ad = (gbs ^ " << gofs[k] << "u)" << xl << "; const bool sw = ad & 1u; tq_st2(dst + (ad & ~1u), sw ? "
                << rb << " : " << ra << ", sw ? " << ra << " : " << rb << "); }\n";
            else
              o << "    tq_st2(dst + (gbs ^ " << gofs[k] << "u), " << ra << ", " << rb << ");\n";
          }
        }
      } else if (variant == 3) {   // projection: the amplitudes whose top bits equal the leaf's choice
        const int n2 = n - proj_m;
        for (int k = 0; k < 16; ++k)
          o << "    { const tq_u32 ad = (gbs ^ " << gofs[k] << "u)" << xl << "; if ((ad >> " << n2
            << ") == hsel) a.scratch[((tq_u64)s << " << n2 << ") | (ad & " << ((1u << n2) - 1u) << "u)] = "
            << g.r(k) << "; }\n";
      } else if (variant == 1) {   // the instance's store-address XOR (uniform per instance)
        o << "    if (t == 0 && tid == 0u) a.xlout[s] = " << (with_errors ? "xl" : "0u") << ";\n";
      } else {                     // the selected run's 8 amplitudes only
        for (int k = 0; k < 16; ++k)
          o << "    { const tq_u32 ad = (gbs ^ " << gofs[k] << "u)" << xl << "; if ((ad >> " << RUN_Q
            << ") == rsel) a.scratch[((tq_u64)s << " << RUN_Q << ") | (ad & " << ((1 << RUN_Q) - 1) << "u)] = "
            << g.r(k) << "; }\n";
      }
      if (pd.leaf_sums && variant != 2 && variant != 3) {
        // |a|^2 sums of the 8-amplitude runs (qubits 0..2): reduce over the register bits
        // holding positions 0..2, then butterfly-shuffle over the lane bits holding the
        // rest (the store layout puts the lowest non-register positions on lanes 0..4).
        int rbits_low = 0;      // register bits holding stored (logical) qubits < RUN_Q
        for (int b = 0; b < RBITS; ++b)
          if (store_key[P.rpos[b]] < RUN_Q) rbits_low |= 1 << b;
        std::vector<int> lane_bits;
        for (int m = 0; m < K - RBITS; ++m)
          if (store_key[P.tpos[m]] < RUN_Q) lane_bits.push_back(m);
        if ((int)lane_bits.size() + __builtin_popcount(rbits_low) != RUN_Q || (!lane_bits.empty() && lane_bits.back() >= 5))
          throw Error{TQSIM_EINTERNAL, "run-sum layout: low qubits not on registers/lanes"};
        std::vector<int> reps;   // one k per run held by this thread
        for (int k = 0; k < 16; ++k)
          if (!(k & rbits_low)) reps.push_back(k);
        for (size_t i = 0; i < reps.size(); ++i) {
          o << "    double rs" << i << " = 0.0;\n";
          for (int k = 0; k < 16; ++k)
            if ((k & ~rbits_low) == reps[i])
              o << "    rs" << i << " = fma(" << g.r(k) << ".x, " << g.r(k) << ".x, fma(" << g.r(k) << ".y, "
                << g.r(k) << ".y, rs" << i << "));\n";
        }
        // Reduce-scatter over the lane bits holding the run's qubits: at each lane bit the
        // lane keeps half of its partial sums (the half selected by its bit) and adds the
        // partner's copy of that half -- R/2 + R/4 + ... shuffles instead of R per bit, and
        // every lane ends with R >> |lane_bits| finished run sums to store.
        const unsigned fm = T >= 32 ? 0xffffffffu : (1u << T) - 1u;
        std::vector<std::string> v;
        for (size_t i = 0; i < reps.size(); ++i) v.push_back("rs" + std::to_string(i));
        std::vector<std::string> base_terms;   // runtime index of the first kept sum
        int stage = 0;
        for (int m : lane_bits) {
          const size_t L = v.size(), half = L / 2;
          if (half == 0) throw Error{TQSIM_EINTERNAL, "run-sum reduce-scatter ran out of sums"};
          o << "    const bool hb" << stage << " = (tid >> " << m << ") & 1u;\n";
          std::vector<std::string> nv;
          for (size_t j = 0; j < half; ++j) {
            const std::string nm = "ru" + std::to_string(stage) + "_" + std::to_string(j);
            o << "    const double " << nm << " = (hb" << stage << " ? " << v[j + half] << " : " << v[j]
              << ") + __shfl_xor_sync(" << fm << "u, hb" << stage << " ? " << v[j] << " : " << v[j + half] << ", "
              << (1 << m) << ");\n";
            nv.push_back(nm);
          }
          base_terms.push_back("(hb" + std::to_string(stage) + " ? " + std::to_string(half) + "u : 0u)");
          v.swap(nv);
          ++stage;
        }
        o << "    const tq_u32 rbase = 0u";
        for (auto& t : base_terms) o << " + " << t;
        o << ";\n";
        o << "    static __constant__ tq_u32 ROFF[" << reps.size() << "] = {";
        for (size_t i = 0; i < reps.size(); ++i) o << (i ? "," : "") << gofs[reps[i]] << "u";
        o << "};\n";
        for (size_t j = 0; j < v.size(); ++j)
          o << "    a.runsum[((tq_u64)s << " << (n - RUN_Q) << ") + (((gbs ^ ROFF[rbase + " << j << "u])" << xl
            << ") >> " << RUN_Q << ")] = " << v[j] << (sum_scale != 1.0 ? " * " + hexd(sum_scale) : std::string())
            << (sc_used ? " * tq_sc" : "")
            << ";\n";
      }
    } else {
      o << "    const tq_u32 sbs = tq_swz(" << lbs << ");\n";
      std::string sx;
      if (with_errors && flush_frame && !amap_upto[ph]) {
        // Frame flush at the exchange: the true state i^fk X^fx Z^fz psi_s is written to the
        // tile explicitly (amplitude at physical index i -> i ^ fx, times i^fk (-1)^popc(fz & i);
        // X only on tile qubits -- an off-tile X keeps the frame), so the next phases start
        // from a trivial frame and run the fast code unless they draw an error themselves.
        // Exact: the frame is a signed permutation.  Not after an absorbed CX (the frame then
        // acts after the deferred store map).
        uint32_t tmask = 0;
        for (int p = 0; p < K; ++p) tmask |= 1u << pd.tile_q[p];
        o << "    tq_u32 tq_sxw = 0u;\n"
          << "    if ((fx & " << ~tmask << "u) == 0u && (fx | fz | fk) != 0u) {\n"
          << "      const tq_u32 tq_zt = __popc(fz & (" << gbs << "));\n";
        for (int k = 0; k < 16; ++k)
          o << "      tq_rot(" << g.r(k) << ", fk + ((tq_zt + __popc(fz & " << goff[k] << "u)) << 1));\n";
        o << "      tq_u32 tq_xt = 0u;\n";
        for (int p = 0; p < K; ++p) o << "      tq_xt |= ((fx >> " << (int)pd.tile_q[p] << ") & 1u) << " << p << ";\n";
        o << "      tq_sxw = tq_swz(tq_xt);\n      fx = 0u; fz = 0u; fk = 0u;\n    }\n";
        sx = " ^ tq_sxw";
      }
      for (int k = 0; k < 16; ++k) o << "    tile[sbs ^ " << soff[k] << "u" << sx << "] = " << g.r(k) << ";\n";
    }
    o << "  }\n";
  }
  };
  // Per phase, CTA-uniform: the error-free fast code while the Pauli frame is trivial
  // and no op of the phase drew an error, else the careful code (the frame carries
  // across phases; both leave the tile in the same canonical shared-memory layout).
  // bitmap of the pass ops whose gate drew an error
  for (int w = 0; w < NW; ++w) o << "  tq_u32 eb" << w << " = 0u;\n";
  // clean: the kernel of the work-list items whose pass drew no error (compact_reps_kernel
  // classifies them): the fast code only -- a third of the instructions, no frame state
  if (!clean) {
  // every warp builds the bitmap itself (one ballot per 32 ops; no block barrier)
  // (CTAs of fewer than 32 threads: the T lanes cover a word's 32 ops in turn)
  {
    const int L = std::min(T, 32);
    char mk[16];
    std::snprintf(mk, sizeof mk, "0x%xu", L >= 32 ? 0xffffffffu : (1u << L) - 1u);
    o << "  if (errs) {\n";
    for (int w = 0; w < NW; ++w)
      o << "    { tq_u32 m = 0u;\n"
        << "      for (tq_u32 l = tid & 31u; l < 32u; l += " << L << "u) {\n"
        << "        const tq_u32 li = " << 32 * w << "u + l;\n"
        << "        if (li < " << nops << "u && codes[4u + GOFF[li]] != 0) m |= 1u << l;\n      }\n"
        << "      eb" << w << " = __reduce_or_sync(" << mk << ", m); }\n";
    o << "    if ((tid & 31u) == 0u) {\n";
    for (int w = 0; w < NW; ++w) o << "      tq_errb[tid >> 5][" << w << "] = eb" << w << ";\n";
    o << "    }\n    __syncwarp(" << mk << ");\n";
    o << "  }\n";
  }
  }
  o << "  tq_u32 fx = 0u, fz = 0u, fk = 0u;\n";
  if (variant == 1 && pd.leaf_sums) o << "  double tq_sc = 1.0;\n";   // run-sum factor (see the flush)
  for (int ph = 0; ph < (int)fast.size(); ++ph) {
    std::vector<uint32_t> pm(NW, 0u);   // error sites of the phase's ops
    std::function<void(const FOp&)> mark = [&](const FOp& f) {
      for (const FOp& cf : f.comps) mark(cf);
      for (const ErrSite& es : f.sites) pm[es.local >> 5] |= 1u << (es.local & 31);
    };
    for (int it : fast[ph].items) mark(fops[it]);
    if (clean) {
      emit_phases(fast, false, ph);
      continue;
    }
    o << "  if ((fx | fz | fk) == 0u";
    for (int w = 0; w < NW; ++w)
      if (pm[w]) o << " && !(eb" << w << " & " << pm[w] << "u)";
    o << ") {\n";
    emit_phases(fast, false, ph);
    o << "  } else {\n";
    emit_phases(fast, true, ph);
    o << "  }\n";
  }
  if (!tma && (variant == 1 || variant == 3)) o << "  __syncthreads();\n  }\n";   // the work loop
  if (tma)   // generic-proxy writes (exchanges) before the buffer's next TMA fill
    o << "  tq_fence_async();\n  __syncthreads();\n  tq_w = tq_next[tq_b ^ 1u];\n  tq_b ^= 1u;\n  }\n";
  o << "}\n";
  g_pool = nullptr;
  coefs = pool.vals;
  // gate coefficients are a by-value kernel parameter (constant bank 0): run-time
  // data, so the source depends only on the circuit's structure
  std::string src = "struct TqCoef { double v[" + std::to_string(std::max<size_t>(coefs.size(), 1)) +
                    "]; };\n" + o.str();
  return src;
}

struct CompiledKernel {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t fn = nullptr;
};

std::mutex g_cache_mu;
std::unordered_map<std::string, CompiledKernel> g_cache;   // full source -> kernel
std::atomic<uint64_t> g_compiles{0};

std::string compile_to_cubin(const std::string& src, const std::string& name) {
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), (name + ".cu").c_str(), 0, nullptr, nullptr) !=
      NVRTC_SUCCESS)
    throw Error{TQSIM_EINTERNAL, "nvrtcCreateProgram failed"};
  // TQSIM_JIT_LINEINFO=1 adds line info for ncu source views (slower compiles, bigger cubins)
  static const bool lineinfo = [] {
    const char* e = std::getenv("TQSIM_JIT_LINEINFO");
    return e && e[0] == '1';
  }();
  const char* opts[] = {"-arch=sm_100a", "-default-device", "-std=c++17", "-lineinfo"};
  const nvrtcResult r = nvrtcCompileProgram(prog, lineinfo ? 4 : 3, opts);
  if (r != NVRTC_SUCCESS) {
    size_t ls = 0;
    nvrtcGetProgramLogSize(prog, &ls);
    std::string log(ls, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    nvrtcDestroyProgram(&prog);
    throw Error{TQSIM_EINTERNAL, "NVRTC failed for " + name + ": " + log.substr(0, 2000)};
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  std::string cubin(n, '\0');
  nvrtcGetCUBIN(prog, &cubin[0]);
  nvrtcDestroyProgram(&prog);
  if (const char* dir = std::getenv("TQSIM_JIT_DUMP"))   // the cubin too (cuobjdump -sass)
    if (FILE* f = std::fopen((std::string(dir) + "/" + name + ".cubin").c_str(), "wb")) {
      std::fwrite(cubin.data(), 1, cubin.size(), f);
      std::fclose(f);
    }
  return cubin;
}

// TMA staging for a kernel (TQSIM_TMA: 0 off (default), 1 the leaf run-sum / trail passes
// (variant 1), 2 every eligible pass): a load from a source batch (fan-out or in place),
// variants 0 / 1, K <= 11 (two 32 KiB tile buffers), and a tile that is one 5-D tensor-map box.
// Off by default: measured on C4 the persistent double-buffered CTAs (3 x 4 warps per SM, 64 KiB
// each) hide the load latency (long_scoreboard 2.1 -> 0.5 stall cycles per issue) but stall at
// the phase barriers with too few warps: the trail marginal pass 203 -> 416 ms per tree
// (profiles/r02_tma_*).
bool tma_wanted(const PassDesc& pd, int n, int mode, int variant, TmaGeom* g) {
  static const int level = [] {
    const char* e = std::getenv("TQSIM_TMA");
    return e ? std::atoi(e) : 0;
  }();
  if (level <= 0 || mode == 0 || pd.K > 11) return false;
  if (variant != 0 && variant != 1) return false;
  if (level == 1 && variant != 1 && !pd.mask_any) return false;
  if (level == 1 && pd.mask_any && variant != 1) return false;
  return tma_geom(pd, n, g);
}

}  // namespace

std::string jit_source(const PassPlan& pp, const std::vector<LGate>& gates, size_t level,
                       size_t pass, const std::string& name) {
  int th;
  size_t sm;
  std::vector<double> cf;
  const int mode = pass > 0 ? 2 : (level == 0 ? 0 : 1);
  int variant = 0;   // TQSIM_JIT_VARIANT=1/2 (leaf-sum passes): the no-store / recompute kernels
  if (const char* e = std::getenv("TQSIM_JIT_VARIANT"))
    if (pp.levels[level][pass].leaf_sums) variant = std::atoi(e);
  return std::string(kPrelude) + kJitTypes +
         gen_pass(pp.levels[level][pass], pp, gates, pp.n_sim, mode, name, th, sm, cf, variant);
}

uint64_t jit_compile_count() { return g_compiles.load(); }

void jit_compile_only(const PassPlan& pp, const std::vector<LGate>& gates, uint64_t* n_kernels,
                      uint64_t* cubin_bytes) {
  std::vector<std::string> srcs, names;
  for (size_t d = 0; d < pp.levels.size(); ++d)
    for (size_t p = 0; p < pp.levels[d].size(); ++p) {
      const int nvar = pp.levels[d][p].leaf_sums ? 4 : 1;
      for (int vv = 0; vv < nvar; ++vv) {   // (3: the clean variant-1 kernel)
        const int v = vv == 3 ? 1 : vv;
        names.push_back("tq_pass_l" + std::to_string(d) + "_p" + std::to_string(p) + (v ? "_v" + std::to_string(v) : "") +
                        (vv == 3 ? "c" : ""));
        const int mode = p > 0 ? 2 : (d == 0 ? 0 : 1);
        int th;
        size_t sm;
        std::vector<double> cf;
        TmaGeom tg;
        const bool tw = vv != 3 && tma_wanted(pp.levels[d][p], pp.n_sim, mode, v, &tg);
        srcs.push_back(std::string(kPrelude) + kJitTypes +
                       gen_pass(pp.levels[d][p], pp, gates, pp.n_sim, mode, names.back(), th, sm, cf, v, nullptr,
                                nullptr, 0, tw ? &tg : nullptr, vv == 3));
      }
    }
  if (pp.trail.on) {   // the conditional leaf sampling kernels (jit_build's trail jobs)
    const TrailPlan& tp = pp.trail;
    for (int vv : {1, 3, 4}) {   // (4: the clean variant-1 kernel)
      const int v = vv == 4 ? 1 : vv;
      names.push_back("tq_trail_a_v" + std::to_string(v) + (vv == 4 ? "c" : ""));
      int th;
      size_t sm;
      std::vector<double> cf;
      TmaGeom tg;
      const bool tw = vv != 4 && tma_wanted(tp.a, pp.n_sim, 1, v, &tg);
      srcs.push_back(std::string(kPrelude) + kJitTypes +
                     gen_pass(tp.a, pp, gates, pp.n_sim, 1, names.back(), th, sm, cf, v, nullptr, nullptr, tp.m,
                              tw ? &tg : nullptr, vv == 4));
    }
    for (size_t p = 0; p < tp.b.size(); ++p)
      for (int v : p + 1 == tp.b.size() ? std::vector<int>{1, 2} : std::vector<int>{0}) {
        names.push_back("tq_trail_b" + std::to_string(p) + "_v" + std::to_string(v));
        int th;
        size_t sm;
        std::vector<double> cf;
        TmaGeom tg;
        const bool tw = tma_wanted(tp.b[p], tp.n2, 2, v, &tg);
        srcs.push_back(std::string(kPrelude) + kJitTypes +
                       gen_pass(tp.b[p], pp, gates, tp.n2, 2, names.back(), th, sm, cf, v, nullptr, nullptr, 0,
                                tw ? &tg : nullptr));
      }
  }
  if (const char* dir = std::getenv("TQSIM_JIT_DUMP"))   // debugging: every generated source
    for (size_t i = 0; i < srcs.size(); ++i)
      if (FILE* f = std::fopen((std::string(dir) + "/" + names[i] + ".cu").c_str(), "w")) {
        std::fwrite(srcs[i].data(), 1, srcs[i].size(), f);
        std::fclose(f);
      }
  std::vector<std::string> errs(srcs.size());
  std::vector<size_t> sizes(srcs.size(), 0);
  std::atomic<size_t> next{0};
  std::vector<std::thread> pool;
  const size_t nt = std::min<size_t>(srcs.size(), std::max(1u, std::thread::hardware_concurrency()));
  for (size_t t = 0; t < nt; ++t)
    pool.emplace_back([&] {
      for (;;) {
        const size_t i = next.fetch_add(1);
        if (i >= srcs.size()) return;
        try {
          sizes[i] = compile_to_cubin(srcs[i], names[i]).size();
        } catch (const Error& e) {
          errs[i] = e.msg;
        }
      }
    });
  for (auto& th : pool) th.join();
  uint64_t tot = 0;
  for (size_t i = 0; i < srcs.size(); ++i) {
    if (!errs[i].empty()) throw Error{TQSIM_EINTERNAL, errs[i]};
    tot += sizes[i];
  }
  if (n_kernels) *n_kernels = srcs.size();
  if (cubin_bytes) *cubin_bytes = tot;
}

std::vector<std::vector<JitPass>> jit_build(const PassPlan& pp, const std::vector<LGate>& gates,
                                            double* compile_seconds, JitTrail* trail) {
  struct Job {
    size_t d, p;
    int which = 0;   // 0 level pass, 1 trail pass A, 2 trail stage-2 pass p
    int variant;
    bool clean = false;   // variant 1 for the items without an error (JitPass::kernel_clean)
    std::string name, src;
    int threads;
    size_t smem;
    std::string cubin;
    std::string err;
    std::vector<double> coefs;
    std::vector<uint32_t> out_row;
    double fp64 = 0.0;
    bool tma = false;
    TmaGeom geom;
    int nsim = -1;
  };
  std::vector<Job> jobs;
  std::vector<std::vector<JitPass>> out(pp.levels.size());
  for (size_t d = 0; d < pp.levels.size(); ++d) {
    out[d].resize(pp.levels[d].size());
    for (size_t p = 0; p < pp.levels[d].size(); ++p) {
      const int nvar = pp.levels[d][p].leaf_sums ? 4 : 1;
      for (int vv = 0; vv < nvar; ++vv) {
        Job j;
        j.d = d;
        j.p = p;
        const int v = vv == 3 ? 1 : vv;
        j.variant = v;
        j.clean = vv == 3;
        j.name = "tq_pass_l" + std::to_string(d) + "_p" + std::to_string(p) + (v ? "_v" + std::to_string(v) : "") +
                 (j.clean ? "c" : "");
        const int mode = p > 0 ? 2 : (d == 0 ? 0 : 1);
        j.tma = !j.clean && tma_wanted(pp.levels[d][p], pp.n_sim, mode, v, &j.geom);
        std::string body = gen_pass(pp.levels[d][p], pp, gates, pp.n_sim, mode, j.name, j.threads,
                                    j.smem, j.coefs, v, &j.out_row, &j.fp64, 0, j.tma ? &j.geom : nullptr,
                                    j.clean);
        j.src = std::string(kPrelude) + kJitTypes + body;
        jobs.push_back(std::move(j));
      }
    }
  }
  if (trail && pp.trail.on) {   // conditional leaf sampling (passplan.cpp plan_trail)
    const TrailPlan& tp = pp.trail;
    for (int vv : {1, 3, 4}) {   // pass A: run sums (marginals; 4: clean) / projection onto the chosen top bits
      Job j;
      j.which = 1;
      j.d = pp.levels.size() - 1;
      j.p = 0;
      const int v = vv == 4 ? 1 : vv;
      j.variant = v;
      j.clean = vv == 4;
      j.name = "tq_trail_a_v" + std::to_string(v) + (j.clean ? "c" : "");
      j.tma = !j.clean && tma_wanted(tp.a, pp.n_sim, 1, v, &j.geom);
      std::string body = gen_pass(tp.a, pp, gates, pp.n_sim, 1, j.name, j.threads, j.smem, j.coefs, v, &j.out_row,
                                  &j.fp64, tp.m, j.tma ? &j.geom : nullptr, j.clean);
      j.src = std::string(kPrelude) + kJitTypes + body;
      jobs.push_back(std::move(j));
    }
    for (size_t p = 0; p < tp.b.size(); ++p) {
      const bool last = p + 1 == tp.b.size();
      for (int v : last ? std::vector<int>{1, 2} : std::vector<int>{0}) {
        Job j;
        j.which = 2;
        j.d = pp.levels.size() - 1;
        j.p = p;
        j.variant = v;
        j.name = "tq_trail_b" + std::to_string(p) + "_v" + std::to_string(v);
        j.tma = tma_wanted(tp.b[p], tp.n2, 2, v, &j.geom);
        std::string body = gen_pass(tp.b[p], pp, gates, tp.n2, 2, j.name, j.threads, j.smem, j.coefs, v, &j.out_row,
                                    &j.fp64, 0, j.tma ? &j.geom : nullptr);
        j.nsim = tp.n2;
        j.src = std::string(kPrelude) + kJitTypes + body;
        jobs.push_back(std::move(j));
      }
    }
    trail->b.assign(tp.b.size(), JitPass{});
  }
  if (const char* dir = std::getenv("TQSIM_JIT_DUMP"))   // debugging: every generated source
    for (const Job& j : jobs)
      if (FILE* f = std::fopen((std::string(dir) + "/" + j.name + ".cu").c_str(), "w")) {
        std::fwrite(j.src.data(), 1, j.src.size(), f);
        std::fclose(f);
      }
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<size_t> todo;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    for (size_t i = 0; i < jobs.size(); ++i)
      if (!g_cache.count(jobs[i].src)) todo.push_back(i);
  }
  if (!todo.empty()) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t nthreads = std::min<size_t>(todo.size(), hw);
    std::atomic<size_t> next{0};
    std::vector<std::thread> pool;
    for (size_t t = 0; t < nthreads; ++t)
      pool.emplace_back([&] {
        for (;;) {
          const size_t i = next.fetch_add(1);
          if (i >= todo.size()) return;
          Job& j = jobs[todo[i]];
          try {
            j.cubin = compile_to_cubin(j.src, j.name);
          } catch (const Error& e) {
            j.err = e.msg;
          }
        }
      });
    for (auto& th : pool) th.join();
    for (size_t i : todo)
      if (!jobs[i].err.empty()) throw Error{TQSIM_EINTERNAL, jobs[i].err};
    std::lock_guard<std::mutex> lk(g_cache_mu);
    for (size_t i : todo) {
      Job& j = jobs[i];
      if (g_cache.count(j.src)) continue;
      CompiledKernel ck;
      cudaError_t e = cudaLibraryLoadData(&ck.lib, j.cubin.data(), nullptr, nullptr, 0, nullptr,
                                          nullptr, 0);
      if (e != cudaSuccess) throw Error{TQSIM_ECUDA, std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e)};
      e = cudaLibraryGetKernel(&ck.fn, ck.lib, j.name.c_str());
      if (e != cudaSuccess) throw Error{TQSIM_ECUDA, std::string("cudaLibraryGetKernel: ") + cudaGetErrorString(e)};
      if (j.smem > 48 * 1024) {
        e = cudaFuncSetAttribute(reinterpret_cast<const void*>(ck.fn),
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)j.smem);
        if (e != cudaSuccess) throw Error{TQSIM_ECUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e)};
      }
      g_cache[j.src] = ck;
      g_compiles++;
    }
  }
  if (compile_seconds)
    *compile_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::lock_guard<std::mutex> lk(g_cache_mu);
  for (Job& j : jobs) {
    const CompiledKernel& ck = g_cache.at(j.src);
    JitPass& jp = j.which == 0 ? out[j.d][j.p] : j.which == 1 ? trail->a : trail->b[j.p];
    if (j.clean) {   // same launch geometry as the variant-1 kernel (same tile, threads, smem)
      jp.kernel_clean = reinterpret_cast<void*>(ck.fn);
      continue;
    }
    if (j.variant == 3) {   // trail projection: its own launch parameters
      jp.kernel_project = reinterpret_cast<void*>(ck.fn);
      jp.threads_project = j.threads;
      jp.smem_project = j.smem;
      jp.coefs_project = j.coefs;
      continue;
    }
    if (j.which != 0 && j.variant == 1) {   // trail kernels without a variant 0: launch parameters
      jp.threads = j.threads;
      jp.smem = j.tma ? (size_t)16 << (j.which == 1 ? pp.trail.a.K : pp.trail.b[j.p].K) : j.smem;
      jp.coefs = j.coefs;
      jp.out_row = j.out_row;
      jp.fp64_per_amp = j.fp64;
    }
    if (j.variant == 0 || j.variant == 1) {   // the TMA decision per variant (tma_wanted)
      jp.tma_v[j.variant] = j.tma;
      if (j.tma) {
        jp.geom = j.geom;
        jp.smem_tma = j.smem;
      }
      jp.n_sim = j.nsim >= 0 ? j.nsim : pp.n_sim;
    }
    if (j.variant == 0) {
      jp.kernel = reinterpret_cast<void*>(ck.fn);
      jp.threads = j.threads;
      jp.smem = j.smem;
      jp.coefs = j.coefs;
      jp.out_row = j.out_row;
      jp.fp64_per_amp = j.fp64;
    } else {
      (j.variant == 1 ? jp.kernel_nostore : jp.kernel_recompute) = reinterpret_cast<void*>(ck.fn);
    }
  }
  return out;
}



bool tma_geom(const PassDesc& pd, int n, TmaGeom* g) {
  TmaGeom r;
  if (pd.K < 4 || n < 4 || pd.tile_q[0] != 0 || pd.tile_q[1] != 1 || pd.tile_q[2] != 2) return false;
  r.kind[0] = 1;
  r.qstart[0] = 0;
  r.len[0] = 3;
  r.ndims = 1;
  int pos_out[64];
  for (int i = 0; i < 64; ++i) pos_out[i] = -1;
  for (int i = 0; i < pd.n_out; ++i) pos_out[pd.out_q[i]] = i;
  for (int q = 3; q < n;) {
    const bool in = (pd.tile_mask >> q) & 1ull;
    int e = q;
    while (e < n && (((pd.tile_mask >> e) & 1ull) != 0) == in && (!in || e - q < 8)) ++e;
    if (r.ndims >= 4) return false;   // the state index needs the last dim
    r.kind[r.ndims] = in ? 1 : 0;
    r.qstart[r.ndims] = q;
    r.len[r.ndims] = e - q;
    r.tbit[r.ndims] = in ? 0 : pos_out[q];
    ++r.ndims;
    q = e;
  }
  r.kind[r.ndims] = 2;
  ++r.ndims;
  *g = r;
  return true;
}

namespace {
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

// The 5-D tensor map over `nstates` states of 2^n amplitudes at `base` with the pass's tile box.
int encode_tile_map(const TmaGeom& g, int n, const void* base, uint64_t nstates, CUtensorMap* out) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return (int)cudaErrorNotSupported;
  cuuint64_t dim[5], stride[4];
  cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
  uint64_t last_stride = 16ull << n;
  for (int d = 0; d < 5; ++d) {
    if (d >= g.ndims) {   // padding
      dim[d] = 1;
      box[d] = 1;
      last_stride *= 2;
      if (d > 0) stride[d - 1] = last_stride;
      continue;
    }
    if (d == 0) {
      dim[0] = 16;
      box[0] = 16;
      continue;
    }
    if (g.kind[d] == 2) {
      dim[d] = nstates;
      box[d] = 1;
      stride[d - 1] = 16ull << n;
      last_stride = (16ull << n) * nstates;
      continue;
    }
    dim[d] = 1ull << g.len[d];
    box[d] = g.kind[d] == 1 ? (1u << g.len[d]) : 1u;
    stride[d - 1] = 16ull << g.qstart[d];
  }
  const CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<void*>(base), dim, stride, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}
}  // namespace

int launch_jit_pass(const JitPass& jp, const PassDesc& pd, const PassLaunch& L, void* stream) {
  HostJitArgs a{L.src, L.dst, L.seed, L.p1, L.p2, L.child_first, L.parent_first,
                L.arity ? L.arity : 1u, L.batch, static_cast<double*>(L.runsum), L.rows, L.row_bytes,
                L.tiles, L.runsel, L.scratch, L.xlout, L.rep, L.prep, L.wlist, L.wcount};
  const void* kern = L.variant == 0 ? jp.kernel
                   : L.variant == 1 ? (L.clean ? jp.kernel_clean : jp.kernel_nostore)
                   : L.variant == 2 ? jp.kernel_recompute : jp.kernel_project;
  if (!kern) return (int)cudaErrorInvalidDeviceFunction;
  uint64_t grid = L.variant == 2 ? (uint64_t)L.batch : (uint64_t)L.batch << pd.n_out;
  if (L.variant == 3 && L.wlist) grid = std::min<uint64_t>(grid, 4 * 148);   // persistent over the work list
  if (L.variant == 1 && L.wlist) {   // persistent over the batch's representatives
    const uint64_t per_sm = (uint64_t)jit_ctas_per_sm(pd.K, (int)jp.threads, L.clean != 0);
    // TQSIM_PERSIST_WAVES: CTAs per resident slot (1 / 2 / 4: C4's marginal pass 148.6 /
    // 145.5 / 142.8 ms per tree, C2 neutral: profiles/r02_ab_item_order.txt)
    static const uint64_t waves = [] {
      const char* e = std::getenv("TQSIM_PERSIST_WAVES");
      return (uint64_t)(e ? std::max(1, std::atoi(e)) : 4);
    }();
    grid = std::min<uint64_t>(grid, per_sm * 148 * waves);
  }
  if (grid == 0) return 0;
  if (grid > 0x7FFFFFFFull) return (int)cudaErrorInvalidConfiguration;
  static const double zero = 0.0;
  const std::vector<double>& cf = L.variant == 3 ? jp.coefs_project : jp.coefs;
  void* args[] = {&a, const_cast<double*>(cf.empty() ? &zero : cf.data())};
  const int threads = L.variant == 3 ? jp.threads_project : jp.threads;
  const size_t smem = L.variant == 3 ? jp.smem_project : jp.smem;
  if ((L.variant == 0 || L.variant == 1) && jp.tma_v[L.variant] && !L.clean) {
    // TMA-staged persistent kernel: the tensor map of the source batch (parents / own states)
    CUtensorMap tm;
    const bool fan = L.src_mode == 1;
    const uint64_t nst = fan ? ((L.child_first + L.batch - 1) / (L.arity ? L.arity : 1) - L.parent_first + 1) : L.batch;
    const int e = encode_tile_map(jp.geom, jp.n_sim, fan ? L.src : L.dst, nst, &tm);
    if (e) return e;
    const uint64_t per_sm = jp.smem_tma > 100 * 1024 ? 1 : jp.smem_tma > 70 * 1024 ? 2 : 3;
    const uint64_t pgrid = std::min<uint64_t>(grid, per_sm * 148);
    void* targs[] = {&a, const_cast<double*>(cf.empty() ? &zero : cf.data()), &tm};
    return (int)cudaLaunchKernel(kern, dim3((unsigned)pgrid), dim3(threads), targs, jp.smem_tma,
                                 static_cast<cudaStream_t>(stream));
  }
  return (int)cudaLaunchKernel(kern, dim3((unsigned)grid), dim3(threads), args, smem,
                               static_cast<cudaStream_t>(stream));
}

}  // namespace tq
