// Pass planner: slice -> HBM passes -> register phases.
//
// Not in the paper (its underlying simulator is Qulacs); this is the
// B200 design of DESIGN.md §6.1.  Every HBM pass stages tiles of 2^K
// amplitudes spanning the K tile qubits {0,1,2} ∪ H (qubits 0..2 give 128-byte
// contiguous runs) in shared memory; inside a tile each thread holds 16
// amplitudes spanning RBITS = 4 tile positions in registers ("phase"), applies
// every consecutive gate on those positions, then the tile is re-shuffled
// through shared memory for the next phase.
//
// Gate order is preserved except that a gate may move ahead of earlier gates
// with which it shares no qubit (they commute); the Pauli error of a gate is
// applied together with the gate, so "noise after its gate" holds.
#include <algorithm>
#include <array>
#include <cstdlib>

#include "tq_internal.h"

namespace tq {

namespace {

inline uint64_t qmask(const LGate& g) { return (1ull << g.q0) | (1ull << g.q1); }
inline int popc(uint64_t v) { return __builtin_popcountll(v); }

// Greedy in-order grouping with commuting look-ahead.  `cost_mask(g)` is the
// set of resources gate g needs beyond the always-present ones; `cap` bounds
// the resources of one group.  Returns groups of gate indices.
// A lowered SWAP: CX(a,b) CX(b,a) CX(a,b) at order positions i, i+1, i+2.
bool swap_triple_at(const std::vector<uint32_t>& v, size_t i, const std::vector<LGate>& gates) {
  if (i + 2 >= v.size()) return false;
  const LGate &x = gates[v[i]], &y = gates[v[i + 1]], &z = gates[v[i + 2]];
  return x.op == OP_CX && y.op == OP_CX && z.op == OP_CX && x.q0 == z.q0 && x.q1 == z.q1 &&
         y.q0 == x.q1 && y.q1 == x.q0;
}

// A diagonal unit starting at order position i: a one-qubit diagonal gate, a CZ, or
// CX(a,b) D(b) CX(a,b) (the lowered RZZ / the middle of a lowered CP).  Returns its
// length (0: none).  Its product is diagonal, so its phase is a function of index bits
// the kernel knows even off the tile (jit.cpp).
size_t diag_unit_at(const std::vector<uint32_t>& v, size_t i, const std::vector<LGate>& gates) {
  const LGate& x = gates[v[i]];
  if ((!x.two && x.op == OP_DIAG) || x.op == OP_CZ) return 1;
  if (x.op != OP_CX || i + 2 >= v.size()) return 0;
  const LGate &y = gates[v[i + 1]], &z = gates[v[i + 2]];
  if (!y.two && y.op == OP_DIAG && y.q0 == x.q1 && z.op == OP_CX && z.q0 == x.q0 && z.q1 == x.q1) return 3;
  return 0;
}

// absorb_swaps also absorbs CX gates that do not fit the tile (or touch
// a qubit of an earlier absorbed CX) into a GF(2)-linear map of the store address: the
// out-of-place store writes amplitude i to M(i) (jit.cpp).  Later gates on their qubits
// that are not themselves absorbed are deferred (they would run before the map).
// Measured: C5 HEA-28 (CX ladders) 261,248 -> 127,616 HBM passes.
//
// absorb_swaps (first pass of a level: out of place, so its store may permute the
// address bits freely): a SWAP on qubits >= low that does not fit the tile joins the
// group as a pure relabeling needing no tile slot; later gates on its qubits are
// deferred to the next pass.  Likewise every diagonal unit joins the first group
// without taking tile slots (its off-tile qubits are read from the tile index): the
// Pauli errors of its gates may flip off-tile qubits, which the out-of-place store
// applies as an address XOR.  (Measured: C4 QAOA-24 37,008 -> 33,808 HBM passes
// against joining only the units that do not fit.)
template <class MaskFn>
std::vector<std::pair<std::vector<uint32_t>, uint64_t>> group_gates(
    const std::vector<uint32_t>& order, const std::vector<LGate>& gates, MaskFn need_mask,
    int cap, size_t max_items = ~size_t(0), bool absorb_swaps = false, int low = 0,
    std::vector<uint8_t>* role = nullptr, bool leaf_level = false) {
  std::vector<std::pair<std::vector<uint32_t>, uint64_t>> groups;
  std::vector<uint32_t> remaining = order;
  bool first_group = true;
  while (!remaining.empty()) {
    uint64_t used = 0, blocked = 0, mapped = 0;   // mapped: qubits of absorbed CX gates
    std::vector<uint32_t> in, deferred;
    for (size_t ri = 0; ri < remaining.size(); ++ri) {
      const uint32_t g = remaining[ri];
      if (absorb_swaps && first_group && swap_triple_at(remaining, ri, gates) && in.size() + 3 <= max_items) {
        const LGate& x = gates[g];
        const uint64_t qm = qmask(x);
        const uint64_t need = need_mask(g);
        if (!(qm & (blocked | mapped)) && popc(used | need) > cap && (int)x.q0 >= low && (int)x.q1 >= low) {
          for (int t = 0; t < 3; ++t) {
            in.push_back(remaining[ri + t]);
            if (role) (*role)[remaining[ri + t]] = ROLE_SWAP;
          }
          blocked |= qm;   // nothing later in this pass touches the relabeled pair
          ri += 2;
          continue;
        }
      }
      if (absorb_swaps && first_group) {
        const size_t du = diag_unit_at(remaining, ri, gates);
        if (du && in.size() + du <= max_items) {
          const uint64_t qm = qmask(gates[g]);
          if (!(qm & (blocked | mapped))) {
            for (size_t t = 0; t < du; ++t) {
              in.push_back(remaining[ri + t]);
              if (role) (*role)[remaining[ri + t]] = ROLE_DIAG;
            }
            ri += du - 1;
            continue;
          }
        }
        const LGate& x = gates[g];
        // (target < low: a permutation inside 128-byte lines; control low - 1 = 2 <= target:
        // splits lines into 64-byte halves, and a leaf run over two tiles, so not at the
        // leaf level; controls 0, 1 would scatter the stores)
        const bool mappable = (int)x.q1 < low || (int)x.q0 >= low || ((int)x.q0 == low - 1 && !leaf_level);
        if (x.op == OP_CX && mappable && in.size() < max_items) {
          const uint64_t qm = qmask(x);
          if (!(qm & blocked) && ((qm & mapped) || popc(used | need_mask(g)) > cap)) {
            in.push_back(g);
            mapped |= qm;
            if (role) (*role)[g] = ROLE_STOREMAP;
            continue;
          }
        }
      }
      const uint64_t qm = qmask(gates[g]);
      if ((qm & (blocked | mapped)) || in.size() >= max_items) {
        deferred.push_back(g);
        blocked |= qm;
        continue;
      }
      const uint64_t need = need_mask(g);
      if (popc(used | need) <= cap) {
        used |= need;
        in.push_back(g);
      } else {
        deferred.push_back(g);
        blocked |= qm;
      }
    }
    if (in.empty()) throw Error{TQSIM_EINTERNAL, "pass planner made no progress"};
    groups.emplace_back(std::move(in), used);
    remaining.swap(deferred);
    first_group = false;
  }
  return groups;
}

}  // namespace

uint64_t PassPlan::passes_total(const std::vector<uint64_t>& inst) const {
  uint64_t t = 0;
  for (size_t d = 0; d < levels.size(); ++d) t += inst[d] * levels[d].size();
  return t;
}

namespace {
PassPlan make_pass_plan_k(const std::vector<LGate>& gates, uint32_t n_qubits, const Plan& plan, int K,
                          uint32_t trail_low);
}

PassPlan make_pass_plan(const std::vector<LGate>& gates, uint32_t n_qubits, const Plan& plan,
                        const Options& o) {
  if (o.tile_qubits) return make_pass_plan_k(gates, n_qubits, plan, (int)o.tile_qubits, o.trail_low);
  // Auto tile width (measured on B200): 2^11-amplitude tiles (4 CTAs x
  // 4 warps per SM) hide HBM latency ~10% better than 2^12 tiles (2 CTAs x 8 warps) but
  // may need more HBM passes; pick the smaller  sum_d instances_d * passes_d / eta_K.
  const std::vector<uint64_t> inst = instances(plan);
  PassPlan best;
  double best_cost = 0.0;
  for (int K : {12, 11}) {
    PassPlan pp = make_pass_plan_k(gates, n_qubits, plan, K, o.trail_low);
    const double eta = K == 11 ? 1.10 : 1.0;
    const double cost = (double)pp.passes_total(inst) / eta;
    if (best.levels.empty() || cost < best_cost) {
      best = std::move(pp);
      best_cost = cost;
    }
  }
  return best;
}

namespace {
// One HBM pass: the tile {0..low-1} ∪ H (padded with the lowest unused high qubits), its
// register phases over the pass's gates (RBITS register positions each), appended to pp.
PassDesc build_pass(PassPlan& pp, const std::vector<LGate>& gates, int K, int n, int low, uint64_t H,
                    const std::vector<uint32_t>& group, const std::vector<uint8_t>& role, uint32_t slice_begin,
                    uint32_t slice_len, uint32_t pass_index, bool leaf_sums) {
  const uint64_t low_mask = (1ull << low) - 1;
  const int hcap = K - low;
  for (int q = low; q < n && popc(H) < hcap; ++q)   // pad with the lowest unused high qubits
    if (!(H >> q & 1)) H |= 1ull << q;
  PassDesc pd;
  pd.K = K;
  pd.slice_begin = slice_begin;
  pd.pass_index = pass_index;
  pd.slice_len = slice_len;
  int pos = 0;
  int qpos[64];
  for (int q = 0; q < 64; ++q) qpos[q] = -1;
  for (int q = 0; q < low; ++q) { pd.tile_q[pos] = (uint8_t)q; qpos[q] = pos++; }
  for (int q = low; q < n; ++q)
    if (H >> q & 1) { pd.tile_q[pos] = (uint8_t)q; qpos[q] = pos++; }
  pd.tile_mask = low_mask | H;
  pd.n_out = 0;
  for (int q = 0; q < n; ++q)
    if (!(pd.tile_mask >> q & 1)) pd.out_q[pd.n_out++] = (uint8_t)q;
  // phases over tile positions
  // absorbed SWAP relabelings (non-tile qubits) and diagonal units need no register
  // slot; a unit's gates thereby stay consecutive in the op list, which is how the
  // kernel generator fuses them back into one diagonal
  auto pos_mask = [&](uint32_t g) {
    const int a = qpos[gates[g].q0], b = qpos[gates[g].q1];
    if (a < 0 || b < 0 || role[g] == ROLE_DIAG || role[g] == ROLE_STOREMAP) return 0ull;
    return (1ull << a) | (1ull << b);
  };
  auto phases = group_gates(group, gates, pos_mask, RBITS);
  pd.phase_begin = (uint32_t)pp.phases.size();
  pd.op_begin = (uint32_t)pp.ops.size();
  for (size_t ph = 0; ph < phases.size(); ++ph) {
    uint64_t R = phases[ph].second;
    for (int p = K - 1; p >= 0 && popc(R) < RBITS; --p)   // pad with high positions
      if (!(R >> p & 1) && p >= low) R |= 1ull << p;
    for (int p = 0; p < K && popc(R) < RBITS; ++p)
      if (!(R >> p & 1)) R |= 1ull << p;
    PhaseDesc pdsc{};
    int rb = 0, rbit_of_pos[MAX_K];
    for (int p = 0; p < K; ++p)
      if (R >> p & 1) { pdsc.rpos[rb] = (uint8_t)p; rbit_of_pos[p] = rb++; }
    // thread-bit -> position map
    std::vector<int> nonr;
    for (int p = 0; p < K; ++p)
      if (!(R >> p & 1)) nonr.push_back(p);
    const bool global_phase = ph == 0 || ph + 1 == phases.size();
    std::vector<int> tmap;
    if (!global_phase && nonr.size() >= 3) {
      // lanes 0..2 on positions of distinct residue mod 3 -> conflict-free 16-byte
      // shared-memory accesses under the XOR swizzle of kernels.cu
      std::vector<int> rest = nonr;
      for (int r = 0; r < 3; ++r)
        for (size_t i = 0; i < rest.size(); ++i)
          if (rest[i] % 3 == r) { tmap.push_back(rest[i]); rest.erase(rest.begin() + i); break; }
      tmap.insert(tmap.end(), rest.begin(), rest.end());
    } else {
      tmap = nonr;
    }
    for (size_t m = 0; m < tmap.size(); ++m) pdsc.tpos[m] = (uint8_t)tmap[m];
    pdsc.op_begin = (uint32_t)pp.ops.size();
    for (uint32_t g : phases[ph].first) {
      const LGate& lg = gates[g];
      OpDesc od{};
      od.type = lg.op;
      od.two = lg.two ? 1 : 0;
      od.gate = g;
      od.role = role[g];
      const bool intile = pos_mask(g) != 0;   // in registers
      od.ra = intile ? (uint8_t)rbit_of_pos[qpos[lg.q0]] : 0;
      od.rb = intile && lg.two ? (uint8_t)rbit_of_pos[qpos[lg.q1]] : od.ra;
      pp.ops.push_back(od);
    }
    pdsc.op_end = (uint32_t)pp.ops.size();
    pp.phases.push_back(pdsc);
  }
  // The leaf level's last pass also writes |a|^2 sums of 2^RUN_Q-amplitude runs
  // (qubits 0..RUN_Q-1) for the sampler (jit.cpp).
  pd.leaf_sums = leaf_sums;
  pd.phase_end = (uint32_t)pp.phases.size();
  pd.op_end = (uint32_t)pp.ops.size();
  return pd;
}

// Conditional sampling through the leaf slice's trailing layer: split the
// leaf slice into A = every gate touching G1 = the top m = K - low qubits, plus every
// diagonal unit, and B = the rest (gates on qubits < n - m only).  If every B gate can move
// after the A gates it precedes (no shared qubit) and A fits one pass over the tile
// {0..low-1} ∪ G1, the leaf is sampled as: marginals over the top bits from A alone (B is
// unitary on the other qubits), then the conditional (n-m)-qubit state of the chosen top
// bits, B applied to it, and the rest of the index by the same inverse CDF.
void plan_trail(PassPlan& pp, const std::vector<LGate>& gates, const Plan& plan, int n, int K, int low) {
  const size_t L = plan.arities.size();
  const int m = K - low, n2 = n - m;
  if (L < 2 || m < 1 || n2 < low + 2 || pp.levels[L - 1].size() < 2) return;
  const uint32_t b0 = (uint32_t)plan.bounds[L - 1], b1 = (uint32_t)plan.bounds[L];
  std::vector<uint32_t> order;
  for (uint32_t g = b0; g < b1; ++g) order.push_back(g);
  const uint64_t G1 = ((1ull << m) - 1) << n2, tile = G1 | ((1ull << low) - 1);
  std::vector<uint8_t> role(gates.size(), ROLE_REG);
  std::vector<char> inA(order.size(), 0);
  for (size_t i = 0; i < order.size();) {
    const size_t du = diag_unit_at(order, i, gates);
    if (du) {
      for (size_t t = 0; t < du; ++t) {
        inA[i + t] = 1;
        role[order[i + t]] = ROLE_DIAG;
      }
      i += du;
      continue;
    }
    const uint64_t qm = qmask(gates[order[i]]);
    if (qm & G1) {
      if (qm & ~tile) return;   // a non-diagonal gate coupling G1 to a qubit off the tile
      inA[i] = 1;
    }
    ++i;
  }
  std::vector<uint32_t> A, B;
  uint64_t bq = 0;   // qubits of the B gates seen so far
  for (size_t i = 0; i < order.size(); ++i) {
    const uint64_t qm = qmask(gates[order[i]]);
    if (inA[i]) {
      if (qm & bq) return;   // an A gate after a B gate on a shared qubit: B cannot move past it
      A.push_back(order[i]);
    } else {
      B.push_back(order[i]);
      bq |= qm;
    }
  }
  if (B.empty() || A.size() > (size_t)MAX_PASS_OPS) return;
  TrailPlan t;
  // the fast projection's spec (ProjSpec): diagonal units before the top-bit 1q gates
  {
    ProjSpec& ps = t.proj;
    ps.m = (uint32_t)m;
    ps.n2 = (uint32_t)n2;
    bool ok = true;
    uint64_t touched = 0;   // top qubits that already got a 1q gate
    std::vector<std::array<double, 8>> ug, ux;
    std::vector<std::pair<uint32_t, uint32_t>> uqg, uqx;
    struct UnitGates {   // the unit's gates (ProjSpec::ugn / ugk / ugoff / ugd)
      uint8_t n = 0, k[3] = {0, 0, 0};
      uint32_t off[3] = {0, 0, 0};
      double d[3][4] = {};
    };
    std::vector<UnitGates> ugg, ugx;
    auto cmul = [](const double* a, const double* b, double* o) {   // o = a * b (complex)
      o[0] = a[0] * b[0] - a[1] * b[1];
      o[1] = a[0] * b[1] + a[1] * b[0];
    };
    for (size_t i = 0; i < A.size() && ok;) {
      const LGate& x = gates[A[i]];
      size_t du = diag_unit_at(A, i, gates);
      const bool top1q = !x.two && (int)x.q0 >= n2;
      if (du && !top1q) {
        // the unit's 4 diagonal entries over (bit a, bit b) by applying its gates to basis states
        const uint32_t qa = x.q0, qb = x.two ? x.q1 : x.q0;
        std::array<double, 8> T{};
        for (int idx = 0; idx < 4 && ok; ++idx) {
          if (qa == qb && (idx == 1 || idx == 2)) continue;
          int ba = idx & 1, bb = idx >> 1;
          double amp[2] = {1.0, 0.0};
          for (size_t t2 = 0; t2 < du; ++t2) {
            const LGate& g = gates[A[i + t2]];
            if (g.op == OP_CX) {
              const int c = g.q0 == qa ? ba : bb;
              if (c) (g.q1 == qa ? ba : bb) ^= 1;
            } else if (g.op == OP_CZ) {
              if (ba && bb) amp[0] = -amp[0], amp[1] = -amp[1];
            } else {   // 1q diagonal on qa or qb
              const int bit = g.q0 == qa ? ba : bb;
              const double d[2] = {g.m[bit ? 6 : 0], g.m[bit ? 7 : 1]};
              double o[2];
              cmul(d, amp, o);
              amp[0] = o[0];
              amp[1] = o[1];
            }
          }
          if (ba != (idx & 1) || bb != (idx >> 1)) ok = false;   // not diagonal
          T[2 * idx] = amp[0];
          T[2 * idx + 1] = amp[1];
        }
        UnitGates ugs;
        ugs.n = (uint8_t)du;
        for (size_t t2 = 0; t2 < du && t2 < 3; ++t2) {
          const LGate& g = gates[A[i + t2]];
          ugs.off[t2] = A[i + t2] - b0;
          if (g.op == OP_CX) ugs.k[t2] = 2;
          else if (g.op == OP_CZ) ugs.k[t2] = 3;
          else {
            ugs.k[t2] = g.q0 == qa ? 0 : 1;
            ugs.d[t2][0] = g.m[0];
            ugs.d[t2][1] = g.m[1];
            ugs.d[t2][2] = g.m[6];
            ugs.d[t2][3] = g.m[7];
          }
        }
        if (du > 3) ok = false;
        const bool ga = (int)qa >= n2, gb = (int)qb >= n2;
        if (ga != gb) ok = false;                                      // couples top and low bits
        if (ga && ((touched >> qa & 1) || (touched >> qb & 1))) ok = false;   // after a top 1q gate
        if (ga) {
          uqg.push_back({qa - n2, qb - n2});
          ug.push_back(T);
          ugg.push_back(ugs);
        } else {
          uqx.push_back({qa, qb});
          ux.push_back(T);
          ugx.push_back(ugs);
        }
        for (size_t t2 = 0; t2 < du; ++t2) {
          if (ps.ndg >= (uint32_t)PROJ_MAX_DG) { ok = false; break; }
          ps.dgoff[ps.ndg++] = A[i + t2] - b0;
        }
        i += du;
        continue;
      }
      if (top1q) {   // a 1q gate on a top qubit (diagonal or not): part of U_j, in order
        if (ps.ng >= (uint32_t)PROJ_MAX_G) { ok = false; break; }
        ps.gbit[ps.ng] = x.q0 - n2;
        ps.goff[ps.ng] = A[i] - b0;
        for (int k = 0; k < 8; ++k) ps.gmat[ps.ng][k] = x.m[k];
        ++ps.ng;
        touched |= 1ull << x.q0;
        ++i;
        continue;
      }
      ok = false;   // a non-diagonal gate among the top qubits (e.g. CX(16, 17))
    }
    if (ok && m <= 10 && ug.size() + ux.size() <= (size_t)PROJ_MAX_U) {
      ps.nug = (uint32_t)ug.size();
      ps.nux = (uint32_t)ux.size();
      size_t k = 0;
      auto put_gates = [&](size_t kk, const UnitGates& s) {
        ps.ugn[kk] = s.n;
        for (int t2 = 0; t2 < 3; ++t2) {
          ps.ugk[kk][t2] = s.k[t2];
          ps.ugoff[kk][t2] = s.off[t2];
          for (int e = 0; e < 4; ++e) ps.ugd[kk][t2][e] = s.d[t2][e];
        }
      };
      for (size_t u = 0; u < ug.size(); ++u, ++k) {
        ps.ua[k] = uqg[u].first;
        ps.ub[k] = uqg[u].second;
        for (int e = 0; e < 8; ++e) ps.uT[k][e] = ug[u][e];
        put_gates(k, ugg[u]);
      }
      for (size_t u = 0; u < ux.size(); ++u, ++k) {
        ps.ua[k] = uqx[u].first;
        ps.ub[k] = uqx[u].second;
        for (int e = 0; e < 8; ++e) ps.uT[k][e] = ux[u][e];
        put_gates(k, ugx[u]);
      }
      t.fast = std::getenv("TQSIM_TRAIL_FAST") == nullptr || std::getenv("TQSIM_TRAIL_FAST")[0] != '0';
    }
  }
  t.on = true;
  t.m = m;
  t.n2 = n2;
  t.a = build_pass(pp, gates, K, n, low, G1, A, role, b0, b1 - b0, 0, true);
  t.a.mask_any = true;
  const int K2 = std::min(K, n2);
  const uint64_t low_mask = (1ull << low) - 1;
  std::vector<uint8_t> role2(gates.size(), ROLE_REG);
  auto groups = group_gates(B, gates, [&](uint32_t g) { return qmask(gates[g]) & ~low_mask; }, K2 - low,
                            MAX_PASS_OPS);
  for (size_t pi = 0; pi < groups.size(); ++pi) {
    PassDesc pd = build_pass(pp, gates, K2, n2, low, groups[pi].second, groups[pi].first, role2, b0, b1 - b0,
                             (uint32_t)(1 + pi), pi + 1 == groups.size());
    pd.mask_any = true;
    t.b.push_back(pd);
  }
  pp.trail = std::move(t);
}

PassPlan make_pass_plan_k(const std::vector<LGate>& gates, uint32_t n_qubits, const Plan& plan, int K,
                          uint32_t trail_low) {
  PassPlan pp;
  const int n = std::max<int>((int)n_qubits, RBITS);
  pp.n_sim = n;
  K = std::max(K, std::min(n, LOW_Q + 2));   // >= 2 free high slots so any 2q gate fits
  K = std::min(K, n);
  const int low = std::min(LOW_Q, K);
  const uint64_t low_mask = (1ull << low) - 1;
  const int hcap = K - low;

  for (size_t d = 0; d + 1 < plan.bounds.size(); ++d) {
    std::vector<uint32_t> order;
    for (uint64_t g = plan.bounds[d]; g < plan.bounds[d + 1]; ++g) order.push_back((uint32_t)g);
    std::vector<uint8_t> role(gates.size(), ROLE_REG);   // roles in the first pass (OpRole)
    auto passes = group_gates(order, gates,
                              [&](uint32_t g) { return qmask(gates[g]) & ~low_mask; }, hcap,
                              MAX_PASS_OPS, /*absorb_swaps=*/true, low, &role,
                              /*leaf_level=*/d + 2 == plan.bounds.size());
    std::vector<PassDesc> lvl;
    for (size_t pi = 0; pi < passes.size(); ++pi)
      lvl.push_back(build_pass(pp, gates, K, n, low, passes[pi].second, passes[pi].first, role,
                               (uint32_t)plan.bounds[d], (uint32_t)(plan.bounds[d + 1] - plan.bounds[d]),
                               (uint32_t)pi, d + 2 == plan.bounds.size() && pi + 1 == passes.size()));
    pp.levels.push_back(std::move(lvl));
  }
  if (const char* e = std::getenv("TQSIM_TRAIL"); !(e && e[0] == '0')) {
    // pass A's tile: the low qubits 0..tlow-1 (contiguous runs of 2^tlow amplitudes) and the
    // top m = K - tlow qubits.  Auto: 4 low qubits for K >= 10 -- one top qubit fewer to
    // rotate per amplitude in the marginal pass and 256-byte runs (C4: 185 -> 165 ms per tree
    // for that pass, the stage-2 passes unchanged; 5 low qubits add a stage-2 pass)
    const int tlow = trail_low ? std::min<int>(K - 1, (int)trail_low) : (K >= 10 ? LOW_Q + 1 : LOW_Q);
    plan_trail(pp, gates, plan, n, K, std::max(low, tlow));
  }
  return pp;
}
}  // namespace

}  // namespace tq
