// Tree planner: Dynamic Circuit Partition and the fixed-arity override
// (SURVEY §8(a) row a2).
//
// DCP (§3.2, §3.3) in the readings R12-R18 of DESIGN.md:
//   m = max(1, round(copy_cost_gates))                first slice length
//   G < 2m or N == 1 -> flat plan (N)
//   p_hat = 1 - prod_{g<m} (1 - e_g)                  Eq.3
//   A_0 = clamp(ceil(n0 / (1 + n0/N)), 1, N),  n0 = z^2 p (1-p) / eps^2, p = min(p_hat, .5)   Eq.4
//   k = max k <= min((G-m)/m, budget/S - 2) with 2^k A_0 <= N
//   A_r = max integer a with a^k A_0 <= N             Eq.5, in integers (R15)
//   top-up A_0 <- max(A_0, ceil(N / A_r^k))           P:294 (R18); topup=1: round robin
//   slices: [m] + k near-equal slices, extras to the earliest (R17)
// Fixed arities: near-equal split into len(arities) slices (R20).
#include <cmath>

#include "tq_internal.h"

namespace tq {

Options options_from(const tqsim_options* o) {
  Options r;
  if (!o) return r;
  r.copy_cost_gates = o->copy_cost_gates;
  r.z = o->z;
  r.eps = o->eps;
  r.mem_budget = o->mem_budget_bytes;
  r.topup = o->topup;
  r.tile_qubits = o->tile_qubits;
  r.batch_log2_amps = o->batch_log2_amps;
  r.profile = o->profile;
  r.no_dedup = o->no_dedup;
  r.trail_low = o->trail_low;
  r.small_tree = o->small_tree;
  if (!(r.copy_cost_gates >= 0 || r.copy_cost_gates == -1.0) || !(r.z > 0) || !(r.eps > 0) || r.topup > 1 ||
      r.no_dedup > 1 || r.small_tree > 2 || (r.trail_low != 0 && (r.trail_low < 3 || r.trail_low > MAX_K - 1)) ||
      (r.tile_qubits != 0 && (r.tile_qubits < RBITS || r.tile_qubits > MAX_K)) ||
      r.batch_log2_amps > 40)
    throw Error{TQSIM_EINVAL, "invalid tqsim_options"};
  return r;
}

namespace {

std::vector<uint64_t> split_equal(uint64_t start, uint64_t count, uint64_t parts) {
  std::vector<uint64_t> b{start};
  const uint64_t base = count / parts, extra = count % parts;
  for (uint64_t i = 0; i < parts; ++i) b.push_back(b.back() + base + (i < extra ? 1 : 0));
  return b;
}

// a^k with saturation above `cap` (returns cap + 1 when exceeded)
uint64_t ipow_sat(uint64_t a, uint32_t k, uint64_t cap) {
  uint64_t r = 1;
  for (uint32_t i = 0; i < k; ++i) {
    if (a != 0 && r > cap / a) return cap + 1;
    r *= a;
  }
  return r;
}

uint64_t int_root_floor(uint64_t q, uint32_t k) {   // largest a with a^k <= q
  if (q < 1) return 0;
  uint64_t a = 1;
  while (ipow_sat(a + 1, k, q) <= q) ++a;
  return a;
}

Plan flat(uint64_t G, uint64_t N) {
  Plan p;
  p.arities = {static_cast<uint32_t>(N)};
  p.bounds = {0, G};
  return p;
}

}  // namespace

std::vector<uint64_t> instances(const Plan& p) {
  std::vector<uint64_t> out;
  uint64_t acc = 1;
  for (uint32_t a : p.arities) {
    acc *= a;
    out.push_back(acc);
  }
  return out;
}

Plan make_plan(const std::vector<LGate>& gates, uint32_t n_qubits, const tqsim_noise_model* nm,
               uint64_t n_shots, const uint32_t* arities, uint32_t n_levels, const Options& o) {
  const uint64_t G = gates.size();
  if (n_shots < 1) throw Error{TQSIM_EINVAL, "n_shots must be >= 1"};
  if (n_shots > 0xFFFFFFFFull) throw Error{TQSIM_EINVAL, "n_shots must be < 2^32"};
  if (arities) {
    if (n_levels < 1 || n_levels > TQSIM_MAX_LEVELS)
      throw Error{TQSIM_EINVAL, "n_levels must be in [1, 64]"};
    if (n_levels > G) throw Error{TQSIM_EINVAL, "n_levels exceeds the lowered gate count"};
    Plan p;
    unsigned __int128 prod = 1;
    for (uint32_t d = 0; d < n_levels; ++d) {
      if (arities[d] < 1) throw Error{TQSIM_EINVAL, "arities must be >= 1"};
      p.arities.push_back(arities[d]);
      prod *= arities[d];
      if (prod > (unsigned __int128)1 << 40) throw Error{TQSIM_EINVAL, "too many outcomes"};
    }
    if ((uint64_t)prod < n_shots) throw Error{TQSIM_EINVAL, "product of arities < n_shots"};
    p.bounds = split_equal(0, G, n_levels);
    return p;
  }
  const uint64_t N = n_shots;
  const uint64_t m = std::max<uint64_t>(1, (uint64_t)std::floor(o.copy_cost_gates + 0.5));
  if (G < 2 * m || N == 1) return flat(G, N);
  double prod = 1.0;
  for (uint64_t g = 0; g < m; ++g) prod *= (1.0 - (gates[g].two ? nm->p2 : nm->p1));
  const double p_hat = 1.0 - prod;
  const double p = std::min(p_hat, 0.5);
  const double n0 = (o.z * o.z * p * (1.0 - p)) / (o.eps * o.eps);
  double a0d = std::ceil(n0 / (1.0 + n0 / (double)N));
  uint64_t a0 = a0d < 1.0 ? 1 : (a0d > (double)N ? N : (uint64_t)a0d);
  const uint64_t S = 16ull << n_qubits;
  const int64_t mem_levels = (int64_t)(o.mem_budget / S) - 2;
  const int64_t k_max = std::min<int64_t>((int64_t)((G - m) / m), mem_levels);
  uint32_t k = 0;
  for (int64_t kk = 1; kk <= k_max && kk < 63; ++kk)
    if ((a0 << kk) <= N && (a0 << kk) >> kk == a0) k = (uint32_t)kk;
  if (k < 1) {
    Plan f = flat(G, N);
    f.p_hat = p_hat;
    return f;
  }
  if (k + 1 > TQSIM_MAX_LEVELS) k = TQSIM_MAX_LEVELS - 1;
  const uint64_t ar = int_root_floor(N / a0, k);
  const uint64_t ar_k = ipow_sat(ar, k, N);
  Plan out;
  out.p_hat = p_hat;
  if (o.topup == 0) {
    a0 = std::max<uint64_t>(a0, (N + ar_k - 1) / ar_k);
    out.arities.push_back((uint32_t)a0);
    for (uint32_t i = 0; i < k; ++i) out.arities.push_back((uint32_t)ar);
  } else {
    out.arities.push_back((uint32_t)a0);
    for (uint32_t i = 0; i < k; ++i) out.arities.push_back((uint32_t)ar);
    for (uint64_t i = 0;; ++i) {
      unsigned __int128 pr = 1;
      for (uint32_t a : out.arities) pr *= a;
      if ((uint64_t)pr >= N) break;
      out.arities[i % out.arities.size()] += 1;
    }
  }
  std::vector<uint64_t> rest = split_equal(m, G - m, k);
  out.bounds.push_back(0);
  out.bounds.insert(out.bounds.end(), rest.begin(), rest.end());
  return out;
}

void fill_plan(const Plan& p, uint32_t n_qubits, uint64_t n_gates, uint64_t hbm_passes,
               tqsim_plan* out) {
  *out = tqsim_plan{};
  out->n_levels = (uint32_t)p.arities.size();
  out->n_qubits = n_qubits;
  for (size_t d = 0; d < p.arities.size(); ++d) out->arities[d] = p.arities[d];
  for (size_t d = 0; d < p.bounds.size(); ++d) out->boundaries[d] = p.bounds[d];
  out->first_error_rate = p.p_hat;
  out->n_lowered_gates = n_gates;
  const std::vector<uint64_t> inst = instances(p);
  uint64_t nodes = 0, tree_apps = 0;
  for (size_t d = 0; d < inst.size(); ++d) {
    nodes += inst[d];
    tree_apps += inst[d] * (p.bounds[d + 1] - p.bounds[d]);
  }
  out->n_outcomes = inst.back();
  out->node_executions = nodes;
  out->predicted_speedup_nodes = (double)inst.size() * (double)inst.back() / (double)nodes;
  out->predicted_speedup_gates = (double)(inst.back() * n_gates) / (double)tree_apps;
  out->gate_amp_updates = tree_apps << n_qubits;
  out->flat_gate_amp_updates = (inst.back() * n_gates) << n_qubits;
  out->hbm_passes = hbm_passes;
}

}  // namespace tq
