// Tree scheduler, workspace layout and the C ABI (SURVEY §8(a) rows a4, a7,
// a8; §8(b)).
//
// The tree (§3, §3.1) is walked level by level in batches:
// run_level(d, [i0, i1)) runs subcircuit d on a batch of <= cap[d] level-d
// instances (fan-out fused into the first pass: every child reads its parent's
// state from the level d-1 batch, "state copy"), then recurses into the
// children of that batch.  Live states are sum_d cap[d], bounded by
// options.mem_budget_bytes (180 GB by default, R25; the paper's "memory
// capacity limit").  Leaves are measured right after their last pass.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <tuple>
#include <new>

#include "tq_internal.h"

struct tqsim_handle {
  uint32_t n_user = 0;
  int n_sim = 0;
  tq::Options opts;
  tqsim_noise_model noise{};
  std::vector<tq::LGate> gates;
  tq::Plan plan;
  tq::PassPlan pp;
  tqsim_plan cplan{};
  std::vector<uint64_t> inst;
  std::vector<std::vector<tq::JitPass>> jit;   // specialized pass kernels [level][pass]
  tq::JitTrail jit_trail;                      // conditional leaf sampling kernels (pp.trail)
  double compile_s = 0.0;
  uint8_t* d_two = nullptr;
  uint8_t* d_pass_of = nullptr;   // per lowered gate: index of its pass in its level (<= 31)
  uint64_t* d_seed = nullptr;     // the run's seed (set by a 1-thread kernel before the tree)
  // CUDA graph of the whole tree (every launch of run_level), replayed by later executes
  // with the same workspace / outcome buffers / shard; seed-independent (read from d_seed)
  cudaGraphExec_t graph_exec = nullptr;
  cudaStream_t capture_stream = nullptr;
  // the leaf branch of the captured tree (see run_level: pipelined penultimate level)
  cudaStream_t leaf_stream = nullptr;
  cudaEvent_t pipe_ev[5] = {};   // level done [2], leaf done [2], join
  std::vector<cudaEvent_t> map_ev; // per level: its dedup map is built (side-stream chain)
  std::vector<uint64_t> graph_key;
  tqsim_stats graph_stats{};
  std::vector<uint8_t> h_tables;  // host copy: [two flags | pass index] per lowered gate
  uint8_t* h_tables_pinned = nullptr;   // the same bytes in page-locked memory (async H2D)
  tqsim_stats stats{};
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<std::pair<int, size_t>> ev_marks;   // (kind 0 pass / 1 measure / 2 noise, event index)
  const tqsim_debug* debug = nullptr;
  cudaStream_t debug_stream = nullptr;
  // per-leaf sampler debug outputs (device, global leaf id; set by tqsim_run_ex for one call)
  double* d_dbg_u = nullptr;
  double* d_dbg_total = nullptr;
  uint8_t* d_dbg_flag = nullptr;
  // tqsim_profile_tree: one tag per event interval (kind, level, pass, batch start, count)
  struct Tag {
    int kind;
    uint32_t level, pass;
    uint64_t b, cnt;
  };
  std::vector<Tag> ev_tags;
  bool tag_launches = false;
  // Kraus engine (non-Pauli channels, kraus.cu): the lowered gate table in HBM
  bool kraus = false;
  tq::KGate* d_kgates = nullptr;   // also read by the small-state tree kernel (small.cu)
  // small-state tree (small.cu): the whole tree as one kernel, one warp per leaf
  bool small = false;
  // conditional leaf sampling: a byte per leaf-slice gate, 1 = in pass A (the gates whose errors
  // change the marginals; NoiseLevel::err_sel of the leaf level's dedup map)
  uint8_t* d_trail_asel = nullptr;
};

namespace tq {

namespace {
thread_local std::string g_last_error;

struct CudaFail {
  int code;
  const char* what;
};

inline void ck(int code, const char* what) {
  if (code != 0) throw CudaFail{code, what};
}
inline void ckc(cudaError_t e, const char* what) { ck((int)e, what); }

template <class F>
tqsim_status guarded(F&& f) {
  try {
    f();
    return TQSIM_OK;
  } catch (const Error& e) {
    g_last_error = e.msg;
    return e.status;
  } catch (const CudaFail& e) {
    g_last_error = std::string(e.what) + ": " + cuda_error_string(e.code);
    return TQSIM_ECUDA;
  } catch (const std::bad_alloc&) {
    g_last_error = "host out of memory";
    return TQSIM_ECAPACITY;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return TQSIM_EINTERNAL;
  } catch (...) {
    g_last_error = "unknown internal error";
    return TQSIM_EINTERNAL;
  }
}

void validate_noise(const tqsim_noise_model* nm) {
  if (!nm) throw Error{TQSIM_EINVAL, "noise model is NULL"};
  const double v[4] = {nm->p1, nm->p2, nm->readout_p01, nm->readout_p10};
  for (double p : v)
    if (!(p >= 0.0 && p <= 1.0)) throw Error{TQSIM_EINVAL, "probabilities must be in [0, 1]"};
  if (!(nm->amp_damping >= 0.0 && nm->amp_damping < 1.0) || !(nm->phase_damping >= 0.0 && nm->phase_damping < 1.0))
    throw Error{TQSIM_EINVAL, "amp_damping / phase_damping must be in [0, 1)"};
  if (!(nm->t1 >= 0.0)) throw Error{TQSIM_EINVAL, "t1 must be >= 0"};
  if (nm->t1 > 0.0 && !(nm->t2 > 0.0 && nm->t2 <= 2.0 * nm->t1 && nm->gate_time_1q >= 0.0 && nm->gate_time_2q >= 0.0))
    throw Error{TQSIM_EINVAL, "thermal relaxation needs 0 < t2 <= 2 t1 and gate times >= 0"};
}

void require_device() {
  int dev = 0, count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    throw Error{TQSIM_ECUDA, "no CUDA device (this library has no CPU fallback)"};
  ckc(cudaGetDevice(&dev), "cudaGetDevice");
  int major = 0;
  ckc(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev), "cc");
  if (major != 10) throw Error{TQSIM_ECUDA, "needs an sm_100 (B200) device"};
}

struct Layout {
  std::vector<uint64_t> cap;       // states per level batch
  std::vector<uint64_t> off;       // byte offset of level buffer
  uint64_t off2 = 0;               // second buffer of the penultimate level (pipelined leaf)
  uint64_t runs_off = 0, sums_off = 0, rows_off = 0, total = 0;
  std::vector<uint64_t> lvl_count;      // the shard's instances per level
  std::vector<uint64_t> rows_lvl_off;   // byte offset of each level's noise rows (in the rows region)
  uint64_t map_off = 0;                 // dedup maps: rep then pos, u32 per instance of the shard
  std::vector<uint64_t> map_lvl;        // entry offset of each level's map
  uint64_t map_entries = 0;
  std::vector<uint64_t> kflag_off;      // Kraus engine: per level, one path-flag byte per batch slot
  std::vector<uint64_t> wl_off;         // per level: the batch's work list (cap u32) + its count
  // conditional leaf sampling (pp.trail): projected states, their run sums, stage-1 outputs
  uint64_t psi_off = 0, runs2_off = 0, hsel_off = 0, htgt_off = 0, glist_off = 0;
  uint64_t sel_off = 0;                 // leaf select / recompute buffers (per leaf of a batch):
                                        // runsel u32, tile u32, xl u32, t3 f64, 8 amplitudes
  int chunk_log2 = 0;
};

constexpr uint64_t ALIGN = 256;
inline uint64_t align_up(uint64_t v) { return (v + ALIGN - 1) / ALIGN * ALIGN; }

// Shard of rank r of W: the tree is split at the split level d*, the first
// level whose instance count I is a multiple of W (else the first with I >= 16 W, else the
// leaf level); rank r owns the level-d* instances [I r / W, I (r+1) / W) and everything
// below them, and recomputes the few ancestors above them (instances are keyed, so a
// recomputed ancestor is bit-identical on every rank).  lo[d], hi[d]: the rank's
// contiguous instance range at level d.
struct ShardRange {
  uint32_t split = 0;
  std::vector<uint64_t> lo, hi;
  uint64_t count(size_t d) const { return hi[d] - lo[d]; }
  bool empty() const { return hi.empty() || hi[0] <= lo[0]; }
};

ShardRange shard_levels(const tqsim_plan& p, uint32_t rank, uint32_t world) {
  if (world < 1 || rank >= world) throw Error{TQSIM_EINVAL, "rank must be < world, world >= 1"};
  const uint32_t L = p.n_levels;
  std::vector<uint64_t> inst(L);
  uint64_t v = 1;
  for (uint32_t d = 0; d < L; ++d) inst[d] = v *= p.arities[d];
  uint32_t ds = L - 1;
  bool found = false;
  for (uint32_t d = 0; d < L && !found; ++d)
    if (inst[d] % world == 0) ds = d, found = true;
  for (uint32_t d = 0; d < L && !found; ++d)
    if (inst[d] >= 16ull * world) ds = d, found = true;
  ShardRange r;
  r.split = ds;
  r.lo.assign(L, 0);
  r.hi.assign(L, 0);
  r.lo[ds] = inst[ds] * rank / world;
  r.hi[ds] = inst[ds] * (rank + 1) / world;
  if (r.hi[ds] > r.lo[ds]) {
    for (uint32_t d = ds; d-- > 0;) {   // ancestors (recomputed)
      r.lo[d] = r.lo[d + 1] / p.arities[d + 1];
      r.hi[d] = (r.hi[d + 1] + p.arities[d + 1] - 1) / p.arities[d + 1];
    }
    for (uint32_t d = ds + 1; d < L; ++d) {
      r.lo[d] = r.lo[d - 1] * p.arities[d];
      r.hi[d] = r.hi[d - 1] * p.arities[d];
    }
  }
  return r;
}

// level-0 range [t0, t1) of the shard (used for the public range query)
void shard(const tqsim_plan& p, uint32_t rank, uint32_t world, uint64_t& t0, uint64_t& t1) {
  const ShardRange r = shard_levels(p, rank, world);
  t0 = r.lo[0];
  t1 = r.hi[0];
}

Layout layout_tl(const tqsim_handle* h, const ShardRange& sr, int tl);

// Batch size: opts.batch_log2_amps, or by default 2^26 amplitudes per level batch -- and for
// 18+ qubits the largest batch up to 2^30 amplitudes whose buffers take <= 55% of the
// memory budget (room for a second, smaller workspace next to tqsim_run's arena): larger
// batches hold more siblings and cousins, so more shared states are computed once (measured:
// C3 251 -> 238 ms, C4 1.21 -> 0.94-0.99 s at 2^28-2^29 (round 1); round 2 C4 with conditional
// leaf sampling 2^27 / 2^28 / 2^29: 738 / 685 / 648 ms; C5 shard 5.1 -> 3.9 s at 2^30, which
// takes ~160 GB and so needs batch_log2_amps = 30 explicitly).
Layout layout(const tqsim_handle* h, const ShardRange& sr) {
  if (h->opts.batch_log2_amps) return layout_tl(h, sr, (int)h->opts.batch_log2_amps);
  if (h->n_sim >= 18)
    for (int tl = 30; tl > 26; --tl) {
      Layout L = layout_tl(h, sr, tl);
      if ((double)L.total <= 0.55 * (double)h->opts.mem_budget) return L;
    }
  return layout_tl(h, sr, 26);
}

Layout layout_tl(const tqsim_handle* h, const ShardRange& sr, int tl) {
  Layout L;
  const int n = h->n_sim;
  const uint64_t S = 16ull << n;
  // >= 2 states per batch by default: sibling pairs share a batch, so error-free
  // duplicates are computed once (measured C5 shard: 8.7 -> 5.5 s); the budget loop
  // below halves the caps again when the buffers would not fit
  const uint64_t target = std::max<uint64_t>(tl >= n ? (1ull << (tl - n)) : 1ull,
                                             h->opts.batch_log2_amps ? 1ull : 2ull);
  const size_t levels = h->plan.arities.size();
  for (size_t d = 0; d < levels; ++d) {
    const uint64_t per = sr.count(d);
    L.cap.push_back(std::max<uint64_t>(1, std::min(per, target)));
    L.lvl_count.push_back(per);
  }
  L.chunk_log2 = std::min(n, 12);
  auto total_of = [&](Layout& l) {
    uint64_t off = 0;
    l.off.clear();
    for (size_t d = 0; d < levels; ++d) {
      l.off.push_back(off);
      off = align_up(off + l.cap[d] * S);
    }
    if (levels >= 2) {   // double buffer of the penultimate level
      l.off2 = off;
      off = align_up(off + l.cap[levels - 2] * S);
    }
    l.runs_off = off;
    off = align_up(off + l.cap.back() * (8ull << (n - RUN_Q)));
    l.sums_off = off;
    {   // chunk sums: the sampler's chunks, or (conditional leaf sampling) 2^m top-bit chunks and
        // the stage-2 sampler's chunks of the n2-qubit states
      uint64_t per = 8ull << (n - l.chunk_log2);
      if (h->pp.trail.on) {
        const int n2 = h->pp.trail.n2;
        per = std::max<uint64_t>(per, 8ull << (n - n2));
        per = std::max<uint64_t>(per, 8ull << (n2 - std::min(n2, 12)));
      }
      off = align_up(off + l.cap.back() * per);
    }
    l.rows_off = off;   // noise rows of every instance of the shard (drawn in one launch)
    uint64_t rows = 0;
    l.rows_lvl_off.clear();
    for (size_t d = 0; d < levels; ++d) {
      l.rows_lvl_off.push_back(rows);
      rows = align_up(rows + l.lvl_count[d] * noise_row_bytes((uint32_t)(h->plan.bounds[d + 1] -
                                                                         h->plan.bounds[d])));
    }
    off = align_up(off + rows);
    l.map_off = off;
    l.map_lvl.clear();
    l.map_entries = 0;
    for (size_t d = 0; d < levels; ++d) {
      l.map_lvl.push_back(l.map_entries);
      l.map_entries += l.lvl_count[d];
    }
    off = align_up(off + 8 * l.map_entries);
    l.kflag_off.clear();
    for (size_t d = 0; d < levels; ++d) {
      l.kflag_off.push_back(off);
      off = align_up(off + (h->kraus ? l.cap[d] : 0));
    }
    l.wl_off.clear();
    for (size_t d = 0; d < levels; ++d) {
      l.wl_off.push_back(off);
      off = align_up(off + 4 * (2 * l.cap[d] + 2));   // two lists (clean, with errors) + counts
    }
    if (h->pp.trail.on) {
      const uint64_t capl = l.cap.back(), n2 = (uint64_t)h->pp.trail.n2;
      l.psi_off = off;
      off = align_up(off + (capl << n2) * 16);
      l.runs2_off = off;
      off = align_up(off + capl * (8ull << (n2 - RUN_Q)));
      l.hsel_off = off;
      off = align_up(off + capl * 4);
      l.htgt_off = off;
      off = align_up(off + capl * 8);
      l.glist_off = off;   // the generated projection's work list + its count
      off = align_up(off + capl * 4 + 4);
    }
    l.sel_off = off;
    off = align_up(off + l.cap.back() * (4 + 4 + 4 + 8 + (16ull << RUN_Q)) + 4 * ALIGN);
    l.total = off;
    return off;
  };
  while (total_of(L) > h->opts.mem_budget) {
    auto it = std::max_element(L.cap.begin(), L.cap.end());
    if (*it <= 1) throw Error{TQSIM_ECAPACITY, "memory budget too small for one state per level"};
    *it = (*it + 1) / 2;
  }
  return L;
}

// ---------------------------------------------------------------- global arena for tqsim_run
std::mutex g_arena_mu;
void* g_arena = nullptr;
size_t g_arena_size = 0;
cudaStream_t g_stream = nullptr;   // tqsim_run's stream (created once)
void* g_pinned = nullptr;          // tqsim_run's page-locked outcome buffer
size_t g_pinned_size = 0;

// Prepared-handle cache of tqsim_run (the plan cache of FFT-style libraries): lowering,
// DCP, pass plan and the run-time specialized kernels of a (circuit, noise, shots,
// arities, options) input are reused by later calls with byte-identical inputs; the
// per-gate device tables are still uploaded every call.  Guarded by g_arena_mu.
struct CachedHandle {
  std::string key;
  tqsim_handle* h;
  uint64_t last_use;
};
std::vector<CachedHandle> g_hcache;
uint64_t g_hcache_clock = 0;
constexpr size_t HCACHE_MAX = 8;

void* arena_get(size_t bytes) {
  if (g_arena_size >= bytes) return g_arena;
  if (g_arena) cudaFree(g_arena);
  g_arena = nullptr;
  g_arena_size = 0;
  ckc(cudaMalloc(&g_arena, bytes), "cudaMalloc workspace");
  g_arena_size = bytes;
  return g_arena;
}

// ---------------------------------------------------------------- scheduler
struct Exec {
  tqsim_handle* h;
  uint64_t seed;
  cudaStream_t st;
  char* ws;
  Layout L;
  uint32_t* d_out;
  std::vector<uint64_t> lvl_first;   // global id of the shard's first instance per level
  std::vector<uint64_t> lvl_end;     // one past the shard's last instance per level
  // Pipelined penultimate level (captured tree only): its batches alternate between two
  // buffers; each batch's leaf work runs on a second stream, so the FP64-bound leaf passes
  // of batch k overlap the HBM-bound passes of batch k+1.
  bool pipe = false;
  cudaStream_t st2 = nullptr;
  const cudaEvent_t* ev = nullptr;   // level done [0..1], leaf done [2..3], join [4]
  uint64_t kD = 0;
  bool slot_used[2] = {false, false};
  bool leaf_issued = false;
  uint64_t pcnt[64] = {};   // instances of the current batch per level
  bool dedup = false;       // dedup maps built for this tree (no state dumps asked for)
  const uint32_t* wl = nullptr;      // the current batch's work list (compact_reps) and count:
  const uint32_t* wlc = nullptr;     //   the computed instances whose variant-1 pass drew no error,
  const uint32_t* wl2 = nullptr;     //   and (wl2, wlc2) those with an error (null: wl holds all)
  const uint32_t* wlc2 = nullptr;
  const cudaEvent_t* map_ev = nullptr;   // side-stream map chain: level d's map is ready
  bool map_waited[64] = {};
};

Exec make_exec(tqsim_handle* h, uint64_t seed, cudaStream_t st, void* ws, const ShardRange& sr, uint32_t* d_out) {
  Exec x{h, seed, st, static_cast<char*>(ws), layout(h, sr), d_out, sr.lo, sr.hi};
  return x;
}

cudaEvent_t next_event(tqsim_handle* h) {
  if (h->ev_used == h->ev_pool.size()) {
    cudaEvent_t e;
    ckc(cudaEventCreate(&e), "cudaEventCreate");
    h->ev_pool.push_back(e);
  }
  return h->ev_pool[h->ev_used++];
}

void mark(Exec& x, int kind, uint32_t level = 0, uint32_t pass = 0, uint64_t b = 0, uint64_t cnt = 0) {
  if (!x.h->opts.profile) return;
  if (x.h->tag_launches && (x.h->ev_marks.size() & 1) == 0)   // an interval opens
    x.h->ev_tags.push_back(tqsim_handle::Tag{kind, level, pass, b, cnt});
  static const bool sync = [] {
    const char* e = std::getenv("TQSIM_PROFILE_SYNC");
    return e && e[0] == '1';
  }();
  if (sync) ckc(cudaStreamSynchronize(x.st), "profile sync");
  cudaEvent_t e = next_event(x.h);
  ckc(cudaEventRecord(e, x.st), "cudaEventRecord");
  x.h->ev_marks.push_back({kind, x.h->ev_used - 1});
}

void dump_if_requested(Exec& x, uint32_t d, uint64_t b, uint64_t cnt, const char* level_buf) {
  const tqsim_debug* dbg = x.h->debug;
  if (!dbg || !dbg->n_dumps) return;
  const uint64_t amps_user = 1ull << x.h->n_user;
  for (uint32_t i = 0; i < dbg->n_dumps; ++i) {
    if (dbg->dump_levels[i] != d) continue;
    const uint64_t j = dbg->dump_instances[i];
    if (j < b || j >= b + cnt) continue;
    ckc(cudaMemcpyAsync(dbg->dump_host + 2 * amps_user * i,
                        level_buf + ((j - b) << (x.h->n_sim + 4)), 16 * amps_user,
                        cudaMemcpyDeviceToHost, x.st),
        "dump copy");
    ckc(cudaStreamSynchronize(x.st), "dump sync");
  }
}

// Conditional leaf sampling of one leaf batch [b, b+cnt) (passplan.cpp
// plan_trail).  The inverse CDF over the index (R9) is taken top bits first: the marginals of
// the top m bits need only the A gates (the B gates act on the other qubits and are unitary
// there), so
//   1. pass A (fan-out + A gates) writes run sums, summed into 2^m chunk sums = marginals;
//   2. stage-1 select: the chunk (top bits) holding u*total and the residual target;
//   3. pass A again, storing only the amplitudes of the chosen top bits (projection, every
//      leaf -- a shared state has per-leaf top bits) -> an n2-qubit state per leaf;
//   4. the B passes on those states (the last writes run sums);
//   5. stage-2 select with the residual target -> recompute the run's tile -> finish
//      (outcome = top bits << n2 | rest, readout flips on every bit).
// Same outcome as sampling the full leaf state (the same inverse CDF, same u) up to rounding
// (draws within 1e-9 of a boundary are flagged, R9); the leaf state is never materialised.
void run_leaf_trail(Exec& x, uint32_t d, uint64_t b, uint64_t cnt, uint64_t parent_first, const char* pbuf,
                    char* buf, const uint8_t* rows, uint32_t row_bytes) {
  tqsim_handle* h = x.h;
  const TrailPlan& tp = h->pp.trail;
  const JitTrail& jt = h->jit_trail;
  const int n = h->n_sim, n2 = tp.n2;
  const uint64_t capl = x.L.cap.back();
  char* sel = x.ws + x.L.sel_off;
  uint32_t* runsel = reinterpret_cast<uint32_t*>(sel);
  uint32_t* tiles = reinterpret_cast<uint32_t*>(sel + align_up(4 * capl));
  uint32_t* xlv = reinterpret_cast<uint32_t*>(sel + 2 * align_up(4 * capl));
  double* t3 = reinterpret_cast<double*>(sel + 3 * align_up(4 * capl));
  void* scratch = sel + 3 * align_up(4 * capl) + align_up(8 * capl);
  double* runs = reinterpret_cast<double*>(x.ws + x.L.runs_off);
  double* sums = reinterpret_cast<double*>(x.ws + x.L.sums_off);
  char* psi = x.ws + x.L.psi_off;
  double* runs2 = reinterpret_cast<double*>(x.ws + x.L.runs2_off);
  uint32_t* hsel = reinterpret_cast<uint32_t*>(x.ws + x.L.hsel_off);
  double* htgt = reinterpret_cast<double*>(x.ws + x.L.htgt_off);
  const uint32_t* maps = reinterpret_cast<const uint32_t*>(x.ws + x.L.map_off);
  const uint32_t* rep = x.dedup && cnt > 1 ? maps + x.L.map_lvl[d] + (b - x.lvl_first[d]) : nullptr;
  const uint32_t* prep = x.dedup && d > 0 && x.pcnt[d - 1] > 1
                             ? maps + x.L.map_lvl[d - 1] + (parent_first - x.lvl_first[d - 1]) : nullptr;
  const uint64_t A = h->plan.arities[d];
  const uint64_t parents = (b + cnt - 1) / A - b / A + 1;
  PassLaunch pl{};
  pl.src_mode = 1u;
  pl.src = pbuf;
  pl.dst = buf;
  pl.child_first = b;
  pl.parent_first = parent_first;
  pl.arity = (uint32_t)A;
  pl.batch = (uint32_t)cnt;
  pl.seed = x.seed;
  pl.p1 = h->noise.p1;
  pl.p2 = h->noise.p2;
  pl.rows = rows;
  pl.row_bytes = row_bytes;
  pl.prep = prep;
  // 1. pass A: run sums of the computed (representative) leaves
  pl.variant = 1u;
  pl.runsum = runs;
  pl.xlout = xlv;
  pl.rep = rep;
  pl.wlist = x.wl;
  pl.wcount = x.wlc;
  mark(x, 0, d, 0, b, cnt);
  if (x.wl2 && jt.a.kernel_clean) {   // the marginals of the clean leaves, then of those with errors
    pl.clean = 1u;
    ck(launch_jit_pass(jt.a, tp.a, pl, x.st), "trail pass A launch (clean)");
    pl.clean = 0u;
    pl.wlist = x.wl2;
    pl.wcount = x.wlc2;
    h->stats.kernel_launches++;
    h->stats.pass_launches++;
  }
  ck(launch_jit_pass(jt.a, tp.a, pl, x.st), "trail pass A launch");
  mark(x, 0, d, 0, b, cnt);
  h->stats.pass_bytes += (cnt << n) * 1 + (parents << n) * 16;
  // 2. chunk sums over the top bits (marginals) and the stage-1 select
  LeafSelect s1{};
  s1.rep = rep;
  s1.hsel = hsel;
  s1.htarget = htgt;
  s1.dbg_u = h->d_dbg_u;
  s1.dbg_total = h->d_dbg_total;
  mark(x, 1, d, 0, b, cnt);
  ck(launch_chunk_sums(runs, (uint32_t)cnt, n, n2, sums, x.st, &s1, b), "trail chunk sums launch");
  ck(launch_sample(buf, runs, sums, (uint32_t)cnt, n, (int)h->n_user, n2, b, h->d_seed, h->noise.readout_p01,
                   h->noise.readout_p10, x.d_out, x.st, &s1),
     "trail select launch");
  mark(x, 1, d, 0, b, cnt);
  // 3. projection onto the chosen top bits (every leaf: a shared state has per-leaf choices):
  //    the hand-written streaming kernel (ProjSpec), and the generated kernel for the leaves
  //    it hands over (a Pauli inside a diagonal unit) -- or the generated one for all
  PassLaunch pb = pl;
  pb.variant = 3u;
  pb.rep = nullptr;
  pb.wlist = nullptr;
  pb.wcount = nullptr;
  pb.runsel = hsel;
  pb.scratch = psi;
  mark(x, 0, d, 100, b, cnt);
  if (tp.fast) {
    uint32_t* glist = reinterpret_cast<uint32_t*>(x.ws + x.L.glist_off);
    uint32_t* gcount = glist + capl;
    ckc(cudaMemsetAsync(gcount, 0, 4, x.st), "trail list reset");
    TrailProjLaunch tl{};
    tl.src = pbuf;
    tl.prep = prep;
    tl.child_first = b;
    tl.parent_first = parent_first;
    tl.arity = (uint32_t)A;
    tl.batch = (uint32_t)cnt;
    tl.n = (uint32_t)n;
    tl.rows = rows;
    tl.row_bytes = row_bytes;
    tl.hsel = hsel;
    tl.psi = psi;
    tl.glist = glist;
    tl.gcount = gcount;
    ck(launch_trail_project(tp.proj, tl, x.st), "trail fast projection launch");
    pb.wlist = glist;
    pb.wcount = gcount;
    h->stats.kernel_launches += 1;
  }
  ck(launch_jit_pass(jt.a, tp.a, pb, x.st), "trail projection launch");
  mark(x, 0, d, 100, b, cnt);
  h->stats.pass_bytes += (parents << n) * 16 + (cnt << n2) * 16;
  // 4. the B passes on the projected n2-qubit states, in place
  PassLaunch last{};
  for (size_t p = 0; p < tp.b.size(); ++p) {
    PassLaunch q = pl;
    q.wlist = nullptr;
    q.wcount = nullptr;
    q.src_mode = 2u;
    q.src = psi;
    q.dst = psi;
    q.prep = nullptr;
    q.rep = nullptr;
    q.child_first = b;
    const bool lastp = p + 1 == tp.b.size();
    q.variant = lastp ? 1u : 0u;
    q.runsum = runs2;
    q.xlout = xlv;
    mark(x, 0, d, 101 + (uint32_t)p, b, cnt);
    ck(launch_jit_pass(jt.b[p], tp.b[p], q, x.st), "trail stage-2 pass launch");
    mark(x, 0, d, 101 + (uint32_t)p, b, cnt);
    h->stats.pass_bytes += (cnt << n2) * (lastp ? 17 : 32);
    if (lastp) last = q;
  }
  h->stats.kernel_launches += 4 + tp.b.size();
  h->stats.pass_launches += 2 + tp.b.size();
  // 5. stage 2: the rest of the index from the residual target; recompute; finish
  const JitPass& jl = jt.b.back();
  LeafSelect s2{};
  s2.runsel = runsel;
  s2.t3 = t3;
  s2.tile = tiles;
  s2.xl = xlv;
  s2.n_out = (uint32_t)jl.out_row.size();
  for (size_t i = 0; i < jl.out_row.size() && i < 32; ++i) s2.out_row[i] = jl.out_row[i];
  s2.tgt = htgt;
  s2.hi = hsel;
  s2.hi_shift = (uint32_t)n2;
  mark(x, 1, d, 1, b, cnt);
  if (n2 - RUN_Q <= SMALL_SAMPLE_RUNS_LOG2) {
    ck(launch_sample_small(psi, runs2, (uint32_t)cnt, n2, (int)h->n_user, b, h->d_seed, h->noise.readout_p01,
                           h->noise.readout_p10, x.d_out, x.st, &s2),
       "trail stage-2 select launch");
    h->stats.kernel_launches += 1;
  } else {
    const int c2 = std::min(n2, 12);
    ck(launch_chunk_sums(runs2, (uint32_t)cnt, n2, c2, sums, x.st, &s2, b), "trail stage-2 chunk sums");
    ck(launch_sample(psi, runs2, sums, (uint32_t)cnt, n2, (int)h->n_user, c2, b, h->d_seed, h->noise.readout_p01,
                     h->noise.readout_p10, x.d_out, x.st, &s2),
       "trail stage-2 select launch");
    h->stats.kernel_launches += 2;
  }
  PassLaunch rc = last;
  rc.variant = 2;
  rc.tiles = tiles;
  rc.runsel = runsel;
  rc.scratch = scratch;
  ck(launch_jit_pass(jl, tp.b.back(), rc, x.st), "trail leaf recompute launch");
  ck(launch_sample_finish(scratch, runsel, t3, (uint32_t)cnt, (int)h->n_user, b, h->d_seed, h->noise.readout_p01,
                          h->noise.readout_p10, x.d_out, x.st, h->d_dbg_flag, hsel, (uint32_t)n2),
     "trail sample finish launch");
  mark(x, 1, d, 1, b, cnt);
  h->stats.kernel_launches += 2;
  h->stats.measure_launches += 5;
  h->stats.measure_bytes += (cnt << (n - RUN_Q)) * 8 + cnt * ((16ull << tp.b.back().K) + (16ull << RUN_Q) * 2);
  h->stats.leaves += cnt;
}

void run_level(Exec& x, uint32_t d, uint64_t i0, uint64_t i1, uint64_t parent_first,
               const char* parent_buf = nullptr) {
  tqsim_handle* h = x.h;
  const int n = h->n_sim;
  const uint32_t levels = (uint32_t)h->plan.arities.size();
  const uint64_t cap = x.L.cap[d];
  char* buf = x.ws + x.L.off[d];
  const char* pbuf = parent_buf ? parent_buf : d > 0 ? x.ws + x.L.off[d - 1] : nullptr;
  const bool piped = x.pipe && d + 2 == levels;
  if (x.map_ev && !x.map_waited[d]) {   // this level's dedup map (side-stream chain)
    ckc(cudaStreamWaitEvent(x.st, x.map_ev[d], 0), "map wait");
    x.map_waited[d] = true;
  }
  const auto& passes = h->pp.levels[d];
  const uint32_t slice_begin = (uint32_t)h->plan.bounds[d];
  const uint32_t slice_len = (uint32_t)(h->plan.bounds[d + 1] - slice_begin);
  const uint32_t row_bytes = noise_row_bytes(slice_len);
  (void)slice_begin;
  for (uint64_t b = i0; b < i1; b += cap) {
    const uint64_t cnt = std::min(cap, i1 - b);
    x.pcnt[d] = cnt;
    int slot = 0;
    if (piped) {   // this batch's buffer: free once the leaf work of batch k-2 is done
      slot = (int)(x.kD++ & 1);
      buf = x.ws + (slot ? x.L.off2 : x.L.off[d]);
      if (x.slot_used[slot]) ckc(cudaStreamWaitEvent(x.st, x.ev[2 + slot], 0), "pipe wait");
    }
    // the batch's noise rows (row a3), drawn for the whole shard at the start of the tree
    uint8_t* rows = reinterpret_cast<uint8_t*>(x.ws + x.L.rows_off + x.L.rows_lvl_off[d]) +
                    (b - x.lvl_first[d]) * row_bytes;
    // leaf: the last pass writes run sums only (no state store) unless state dumps are asked for
    const bool leaf = d + 1 == levels;
    const bool nostore = leaf && !(h->debug && h->debug->n_dumps);
    char* sel = x.ws + x.L.sel_off;
    const uint64_t capl = x.L.cap.back();
    uint32_t* runsel = reinterpret_cast<uint32_t*>(sel);
    uint32_t* tiles = reinterpret_cast<uint32_t*>(sel + align_up(4 * capl));
    uint32_t* xlv = reinterpret_cast<uint32_t*>(sel + 2 * align_up(4 * capl));
    double* t3 = reinterpret_cast<double*>(sel + 3 * align_up(4 * capl));
    void* scratch = sel + 3 * align_up(4 * capl) + align_up(8 * capl);
    // the batch's computed instances as a work list: the pass kernels loop over them with
    // persistent CTAs instead of launching an (empty) CTA per shared instance and tile
    x.wl = x.wlc = x.wl2 = x.wlc2 = nullptr;
    static const bool use_wl = [] {
      const char* e = std::getenv("TQSIM_WORKLIST");
      return !(e && e[0] == '0');
    }();
    static const bool split_clean = [] {   // 0: one variant-1 kernel (with the careful code) for all
      const char* e = std::getenv("TQSIM_CLEAN_SPLIT");
      return !(e && e[0] == '0');
    }();
    if (use_wl && x.dedup && cnt > 1 && leaf && nostore) {   // the leaf run-sum passes (variant 1)
      const uint32_t* maps = reinterpret_cast<const uint32_t*>(x.ws + x.L.map_off);
      uint32_t* wl = reinterpret_cast<uint32_t*>(x.ws + x.L.wl_off[d]);
      const uint64_t c = x.L.cap[d];
      uint32_t* xl0 = leaf && nostore ? reinterpret_cast<uint32_t*>(x.ws + x.L.sel_off + 2 * align_up(4 * x.L.cap.back()))
                                      : nullptr;
      // the variant-1 pass's error bits of the noise row: the trail's marginal pass takes the
      // careful code on any error of the slice (mask_any), a level pass on its own bit
      const uint32_t em = h->pp.trail.on ? ~0u : 1u << std::min<size_t>(passes.size() - 1, 31);
      const bool asel = h->pp.trail.on && h->d_trail_asel;   // (nostore: the trail is active)
      ck(launch_compact_reps(asel ? h->d_trail_asel : nullptr,
                             (uint32_t)(h->plan.bounds[d + 1] - h->plan.bounds[d]),
                             maps + x.L.map_lvl[d] + (b - x.lvl_first[d]), (uint32_t)cnt, wl, wl + c, xl0,
                             split_clean ? rows : nullptr, row_bytes, em, wl + c + 1, split_clean ? wl + 2 * c + 1 : nullptr,
                             x.st),
         "work list launch");
      h->stats.kernel_launches++;
      x.wl = wl;
      x.wlc = wl + c;
      if (split_clean) {
        x.wl2 = wl + c + 1;
        x.wlc2 = wl + 2 * c + 1;
      }
    }
    if (leaf && nostore && h->pp.trail.on) {   // conditional leaf sampling (default path)
      run_leaf_trail(x, d, b, cnt, parent_first, pbuf, buf, rows, row_bytes);
      h->stats.node_executions += cnt;
      h->stats.gate_amp_updates += (cnt * (h->plan.bounds[d + 1] - h->plan.bounds[d])) << h->n_user;
      continue;
    }
    PassLaunch last{};
    for (size_t p = 0; p < passes.size(); ++p) {
      PassLaunch pl{};
      pl.src_mode = p > 0 ? 2u : (d == 0 ? 0u : 1u);
      pl.src = pbuf;
      pl.dst = buf;
      pl.child_first = b;
      pl.parent_first = parent_first;
      pl.arity = h->plan.arities[d];
      pl.batch = (uint32_t)cnt;
      pl.seed = x.seed;
      pl.p1 = h->noise.p1;
      pl.p2 = h->noise.p2;
      pl.runsum = x.ws + x.L.runs_off;
      pl.rows = rows;
      pl.row_bytes = row_bytes;
      const bool runsums_only = nostore && passes[p].leaf_sums;
      pl.variant = runsums_only ? 1u : 0u;
      pl.xlout = xlv;
      // shared states computed once (dedup maps; nobody reads a skipped slot except through
      // the maps: the next level's fan-out, the sampler, the recompute)
      pl.wlist = runsums_only ? x.wl : nullptr;   // only the variant-1 kernels loop over a work list
      pl.wcount = runsums_only ? x.wlc : nullptr;
      if (x.dedup) {
        const uint32_t* maps = reinterpret_cast<const uint32_t*>(x.ws + x.L.map_off);
        if (cnt > 1) pl.rep = maps + x.L.map_lvl[d] + (b - x.lvl_first[d]);
        if (d > 0 && x.pcnt[d - 1] > 1) pl.prep = maps + x.L.map_lvl[d - 1] + (parent_first - x.lvl_first[d - 1]);
      }
      mark(x, 0, d, (uint32_t)p, b, cnt);
      if (runsums_only && x.wl2 && h->jit[d][p].kernel_clean) {   // clean items, then those with errors
        pl.clean = 1u;
        ck(launch_jit_pass(h->jit[d][p], passes[p], pl, x.st), "gate pass launch (clean)");
        pl.clean = 0u;
        pl.wlist = x.wl2;
        pl.wcount = x.wlc2;
        h->stats.kernel_launches++;
        h->stats.pass_launches++;
      }
      ck(launch_jit_pass(h->jit[d][p], passes[p], pl, x.st), "gate pass launch");
      mark(x, 0, d, (uint32_t)p, b, cnt);
      h->stats.kernel_launches++;
      h->stats.pass_launches++;
      if (passes[p].leaf_sums) last = pl;
      const uint64_t amps = cnt << n;
      // write (or, without the leaf state store, the run sums: 8 B per 8 amplitudes)
      uint64_t bytes = runsums_only ? amps : amps * 16;
      if (pl.src_mode == 2) bytes += amps * 16;
      else if (pl.src_mode == 1) {
        const uint64_t A = pl.arity;
        const uint64_t parents = (b + cnt - 1) / A - b / A + 1;
        bytes += (parents << n) * 16;
      }
      h->stats.pass_bytes += bytes;
    }
    h->stats.node_executions += cnt;
    h->stats.gate_amp_updates += (cnt * (h->plan.bounds[d + 1] - h->plan.bounds[d])) << h->n_user;
    dump_if_requested(x, d, b, cnt, buf);
    if (leaf && nostore) {
      // select each leaf's run from the run sums -> recompute the one tile holding it
      // (variant 2 of the last pass, same operands) -> walk its 8 amplitudes
      double* sums = reinterpret_cast<double*>(x.ws + x.L.sums_off);
      const double* runs = reinterpret_cast<const double*>(x.ws + x.L.runs_off);
      const size_t lp = passes.size() - 1;
      const JitPass& jp = h->jit[d][lp];
      LeafSelect ls{};
      ls.runsel = runsel;
      ls.t3 = t3;
      ls.tile = tiles;
      ls.xl = xlv;
      ls.n_out = (uint32_t)jp.out_row.size();
      ls.rep = x.dedup && cnt > 1 ? reinterpret_cast<const uint32_t*>(x.ws + x.L.map_off) + x.L.map_lvl[d] +
                                         (b - x.lvl_first[d])
                                   : nullptr;
      for (size_t i = 0; i < jp.out_row.size() && i < 32; ++i) ls.out_row[i] = jp.out_row[i];
      ls.dbg_u = h->d_dbg_u;
      ls.dbg_total = h->d_dbg_total;
      ls.dbg_flag = nullptr;   // the finish kernel flags the draw
      mark(x, 1, d, 0, b, cnt);
      if (n - RUN_Q <= SMALL_SAMPLE_RUNS_LOG2) {
        ck(launch_sample_small(buf, runs, (uint32_t)cnt, n, (int)h->n_user, b, h->d_seed, h->noise.readout_p01,
                               h->noise.readout_p10, x.d_out, x.st, &ls),
           "sample select launch");
        h->stats.kernel_launches += 1;
        h->stats.measure_launches += 1;
        h->stats.measure_bytes += (cnt << (n - RUN_Q)) * 8;
      } else {
        ck(launch_chunk_sums(runs, (uint32_t)cnt, n, x.L.chunk_log2, sums, x.st, &ls, b), "chunk sums launch");
        ck(launch_sample(buf, runs, sums, (uint32_t)cnt, n, (int)h->n_user, x.L.chunk_log2, b, h->d_seed,
                         h->noise.readout_p01, h->noise.readout_p10, x.d_out, x.st, &ls),
           "sample select launch");
        h->stats.kernel_launches += 2;
        h->stats.measure_launches += 2;
        h->stats.measure_bytes += (cnt << (n - RUN_Q)) * 8 +
                                  cnt * ((8ull << (n - x.L.chunk_log2)) + (8ull << (x.L.chunk_log2 - RUN_Q)));
      }
      PassLaunch rc = last;
      rc.variant = 2;
      rc.tiles = tiles;
      rc.runsel = runsel;
      rc.scratch = scratch;
      ck(launch_jit_pass(jp, passes[lp], rc, x.st), "leaf recompute launch");
      ck(launch_sample_finish(scratch, runsel, t3, (uint32_t)cnt, (int)h->n_user, b, h->d_seed,
                              h->noise.readout_p01, h->noise.readout_p10, x.d_out, x.st, h->d_dbg_flag),
         "sample finish launch");
      mark(x, 1, d, 0, b, cnt);
      h->stats.kernel_launches += 2;
      h->stats.measure_launches += 2;
      // the recomputed tile per leaf (read its share of the source + 8 amplitudes written)
      h->stats.measure_bytes += cnt * ((16ull << passes[lp].K) + (16ull << RUN_Q) * 2);
      h->stats.leaves += cnt;
    } else if (leaf) {
      double* sums = reinterpret_cast<double*>(x.ws + x.L.sums_off);
      const double* runs = reinterpret_cast<const double*>(x.ws + x.L.runs_off);
      LeafSelect dbg{};   // stored-state path: only the debug outputs
      dbg.dbg_u = h->d_dbg_u;
      dbg.dbg_total = h->d_dbg_total;
      dbg.dbg_flag = h->d_dbg_flag;
      mark(x, 1, d, 0, b, cnt);
      if (n - RUN_Q <= SMALL_SAMPLE_RUNS_LOG2) {   // one kernel: all run sums of each leaf
        ck(launch_sample_small(buf, runs, (uint32_t)cnt, n, (int)h->n_user, b, h->d_seed,
                               h->noise.readout_p01, h->noise.readout_p10, x.d_out, x.st, &dbg),
           "sample launch");
        h->stats.kernel_launches += 1;
        h->stats.measure_launches += 1;
        h->stats.measure_bytes += (cnt << (n - RUN_Q)) * 8 + cnt * (16ull << RUN_Q);
      } else {
        ck(launch_chunk_sums(runs, (uint32_t)cnt, n, x.L.chunk_log2, sums, x.st), "chunk sums launch");
        ck(launch_sample(buf, runs, sums, (uint32_t)cnt, n, (int)h->n_user, x.L.chunk_log2, b, h->d_seed,
                         h->noise.readout_p01, h->noise.readout_p10, x.d_out, x.st, &dbg),
           "sample launch");
        h->stats.kernel_launches += 2;
        h->stats.measure_launches += 2;
        // run sums read once; per leaf the chunk sums, one chunk of run sums, 8 amplitudes
        h->stats.measure_bytes += (cnt << (n - RUN_Q)) * 8 +
                                  cnt * ((8ull << (n - x.L.chunk_log2)) +
                                         (8ull << (x.L.chunk_log2 - RUN_Q)) + (16ull << RUN_Q));
      }
      mark(x, 1, d, 0, b, cnt);
      h->stats.leaves += cnt;
    } else if (piped) {
      const uint64_t A = h->plan.arities[d + 1];
      ckc(cudaEventRecord(x.ev[slot], x.st), "pipe record");
      ckc(cudaStreamWaitEvent(x.st2, x.ev[slot], 0), "pipe fork");
      std::swap(x.st, x.st2);
      run_level(x, d + 1, std::max(b * A, x.lvl_first[d + 1]), std::min((b + cnt) * A, x.lvl_end[d + 1]), b, buf);
      std::swap(x.st, x.st2);
      ckc(cudaEventRecord(x.ev[2 + slot], x.st2), "pipe record");
      x.slot_used[slot] = true;
      x.leaf_issued = true;
    } else {
      const uint64_t A = h->plan.arities[d + 1];
      run_level(x, d + 1, std::max(b * A, x.lvl_first[d + 1]), std::min((b + cnt) * A, x.lvl_end[d + 1]), b);
    }
  }
}

// Kraus engine (kraus.cu): level batches as run_level forms them; one CTA per instance runs
// the whole slice with the state in shared memory; leaves are sampled in the same kernel.
void run_level_kraus(Exec& x, uint32_t d, uint64_t i0, uint64_t i1, uint64_t parent_first) {
  tqsim_handle* h = x.h;
  const uint32_t levels = (uint32_t)h->plan.arities.size();
  const tqsim_noise_model& nm = h->noise;
  for (uint64_t b = i0; b < i1; b += x.L.cap[d]) {
    const uint64_t cnt = std::min(x.L.cap[d], i1 - b);
    KrausArgs a{};
    a.gates = h->d_kgates;
    a.src = d > 0 ? x.ws + x.L.off[d - 1] : nullptr;
    a.dst = x.ws + x.L.off[d];
    a.src_flag = d > 0 ? reinterpret_cast<const uint8_t*>(x.ws + x.L.kflag_off[d - 1]) : nullptr;
    a.dst_flag = reinterpret_cast<uint8_t*>(x.ws + x.L.kflag_off[d]);
    a.child_first = b;
    a.parent_first = parent_first;
    a.arity = h->plan.arities[d];
    a.g0 = (uint32_t)h->plan.bounds[d];
    a.g1 = (uint32_t)h->plan.bounds[d + 1];
    a.n = (uint32_t)h->n_sim;   // the layout's state size (n < 4 padded, R28: the pad qubits stay |0>)
    a.n_user = h->n_user;
    a.mode = d > 0 ? 1u : 0u;
    a.leaf = d + 1 == levels ? 1u : 0u;
    a.store_leaf = h->debug && h->debug->n_dumps ? 1u : 0u;
    a.seedp = h->d_seed;
    a.p1 = nm.p1;
    a.p2 = nm.p2;
    a.p01 = nm.readout_p01;
    a.p10 = nm.readout_p10;
    if (nm.t1 > 0.0) {   // R32: TR = AD(1 - e^{-t/T1}) then PD(1 - e^{-2t/T2 + t/T1}), t per gate class
      a.ch_mask |= 1u;
      const double t[2] = {nm.gate_time_1q, nm.gate_time_2q};
      for (int c = 0; c < 2; ++c) {
        a.trg[c] = 1.0 - std::exp(-t[c] / nm.t1);
        a.trl[c] = 1.0 - std::exp(-2.0 * t[c] / nm.t2 + t[c] / nm.t1);
      }
    }
    if (nm.amp_damping > 0.0) a.ch_mask |= 2u, a.ad = nm.amp_damping;
    if (nm.phase_damping > 0.0) a.ch_mask |= 4u, a.pd = nm.phase_damping;
    a.out = x.d_out;
    a.dbg_u = h->d_dbg_u;
    a.dbg_total = h->d_dbg_total;
    a.dbg_flag = h->d_dbg_flag;
    mark(x, 3, d, 0, b, cnt);
    ck(launch_kraus_slice(a, (uint32_t)cnt, x.st), "kraus slice launch");
    mark(x, 3, d, 0, b, cnt);
    h->stats.kernel_launches++;
    h->stats.pass_launches++;
    h->stats.node_executions += cnt;
    h->stats.gate_amp_updates += (cnt * (a.g1 - a.g0)) << h->n_user;
    // one parent read per instance, the state written (not at a leaf): shared memory otherwise
    h->stats.pass_bytes += (cnt << h->n_user) * ((d > 0 ? 16 : 0) + (a.leaf ? 0 : 16));
    dump_if_requested(x, d, b, cnt, x.ws + x.L.off[d]);
    if (a.leaf) {
      h->stats.leaves += cnt;
    } else {
      const uint64_t A = h->plan.arities[d + 1];
      run_level_kraus(x, d + 1, std::max(b * A, x.lvl_first[d + 1]), std::min((b + cnt) * A, x.lvl_end[d + 1]), b);
    }
  }
}

// Small-state tree (small.cu): every leaf of the shard in one launch, one warp per leaf
// recomputing its root-to-leaf path with the inherited keys (the tree's own noise draws).
void run_small_tree(Exec& x) {
  tqsim_handle* h = x.h;
  const uint32_t L = (uint32_t)h->plan.arities.size();
  SmallTreeArgs a{};
  a.gates = h->d_kgates;
  a.leaf_first = x.lvl_first[L - 1];
  a.leaf_count = x.lvl_end[L - 1] - x.lvl_first[L - 1];
  a.levels = L;
  a.n = (uint32_t)std::max(h->n_sim, 5);   // >= one amplitude per lane; pad qubits stay |0> (R28)
  a.n_user = h->n_user;
  for (uint32_t d = 0; d < L; ++d) a.arity[d] = h->plan.arities[d];
  for (uint32_t d = 0; d <= L; ++d) a.bounds[d] = (uint32_t)h->plan.bounds[d];
  a.seedp = h->d_seed;
  a.p1 = h->noise.p1;
  a.p2 = h->noise.p2;
  a.p01 = h->noise.readout_p01;
  a.p10 = h->noise.readout_p10;
  a.out = x.d_out;
  a.dbg_u = h->d_dbg_u;
  a.dbg_total = h->d_dbg_total;
  a.dbg_flag = h->d_dbg_flag;
  mark(x, 0, L - 1, 0, a.leaf_first, a.leaf_count);
  ck(launch_small_tree(a, x.st), "small tree launch");
  mark(x, 0, L - 1, 0, a.leaf_first, a.leaf_count);
  h->stats.kernel_launches++;
  h->stats.pass_launches++;
  uint64_t nodes = 0, gamps = 0;
  for (uint32_t d = 0; d < L; ++d) {   // the tree's nominal work over the shard (as run_level counts it)
    const uint64_t cnt = x.lvl_end[d] - x.lvl_first[d];
    nodes += cnt;
    gamps += (cnt * (h->plan.bounds[d + 1] - h->plan.bounds[d])) << h->n_user;
  }
  h->stats.node_executions += nodes;
  h->stats.gate_amp_updates += gamps;
  h->stats.leaves += a.leaf_count;
}

// Every noise row of the shard (all levels) in one launch, then the tree.
void run_tree(Exec& x) {
  if (x.h->small && !(x.h->debug && x.h->debug->n_dumps)) {
    run_small_tree(x);
    return;
  }
  if (x.h->kraus) {
    run_level_kraus(x, 0, x.lvl_first[0], x.lvl_end[0], 0);
    return;
  }
  tqsim_handle* h = x.h;
  NoiseLevels NL{};
  const size_t levels = h->plan.arities.size();
  if (levels > (size_t)NOISE_MAX_LEVELS) throw Error{TQSIM_EINTERNAL, "too many levels for the noise rows"};
  uint64_t total = 0;
  for (size_t d = 0; d < levels; ++d) {
    NoiseLevel& lv = NL.lv[d];
    lv.inst_first = x.lvl_first[d];
    lv.count = x.L.lvl_count[d];
    lv.rows_off = x.L.rows_lvl_off[d];
    lv.slice_begin = (uint32_t)h->plan.bounds[d];
    lv.slice_len = (uint32_t)(h->plan.bounds[d + 1] - h->plan.bounds[d]);
    lv.row_bytes = noise_row_bytes(lv.slice_len);
    lv.map_off = x.L.map_lvl[d];
    lv.cap = x.L.cap[d];
    lv.arity = h->plan.arities[d];
    lv.err_sel = d + 1 == levels && h->pp.trail.on ? h->d_trail_asel : nullptr;   // (dumps: no maps)
    total += lv.count;
  }
  NL.n_levels = (uint32_t)levels;
  mark(x, 2);
  ck(launch_noise_rows_all(h->d_two, h->d_pass_of, NL, total, h->d_seed, h->noise.p1, h->noise.p2,
                           reinterpret_cast<uint8_t*>(x.ws + x.L.rows_off), x.st),
     "noise rows launch");
  mark(x, 2);
  h->stats.kernel_launches++;
  h->stats.noise_launches++;
  x.dedup = !(h->debug && h->debug->n_dumps) && !h->opts.no_dedup;
  if (x.dedup) {
    uint32_t* maps = reinterpret_cast<uint32_t*>(x.ws + x.L.map_off);
    const uint8_t* rws = reinterpret_cast<const uint8_t*>(x.ws + x.L.rows_off);
    if (x.pipe) {   // per-level kernels on the side stream, ahead of the levels that wait on them
      while (h->map_ev.size() < levels) {
        cudaEvent_t e;
        ckc(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "map event");
        h->map_ev.push_back(e);
      }
      ckc(cudaEventRecord(x.ev[4], x.st), "map fork");
      ckc(cudaStreamWaitEvent(x.st2, x.ev[4], 0), "map fork wait");
      for (size_t d = 0; d < levels; ++d) {
        ck(launch_dedup_map_level(rws, NL, (uint32_t)d, maps, maps + x.L.map_entries, x.st2), "dedup map launch");
        ckc(cudaEventRecord(h->map_ev[d], x.st2), "map record");
        h->stats.kernel_launches++;
      }
      x.map_ev = h->map_ev.data();
      x.leaf_issued = true;   // the side stream joins at the end
    } else {
      ck(launch_dedup_map(rws, NL, maps, maps + x.L.map_entries, x.st), "dedup map launch");
      h->stats.kernel_launches++;
    }
  }
  run_level(x, 0, x.lvl_first[0], x.lvl_end[0], 0);
  if (x.pipe && x.leaf_issued) {   // join the leaf branch
    ckc(cudaEventRecord(x.ev[4], x.st2), "pipe join record");
    ckc(cudaStreamWaitEvent(x.st, x.ev[4], 0), "pipe join");
  }
}

// per-gate device tables: 2q flag (noise class) and pass index (error bitmask bit)
void upload_gate_tables(tqsim_handle* h, cudaStream_t st) {
  const size_t G = h->h_tables.size() / 2;
  const uint8_t* src = h->h_tables.data();
  if (st) {   // page-locked staging (tqsim_run: every call uploads its tables)
    if (!h->h_tables_pinned) {
      ckc(cudaMallocHost(reinterpret_cast<void**>(&h->h_tables_pinned), std::max<size_t>(2 * G, 1)), "cudaMallocHost");
      std::memcpy(h->h_tables_pinned, src, 2 * G);
    }
    src = h->h_tables_pinned;
  }
  ckc(cudaMemcpyAsync(h->d_two, src, G, cudaMemcpyHostToDevice, st), "upload two");
  ckc(cudaMemcpyAsync(h->d_pass_of, src + G, G, cudaMemcpyHostToDevice, st), "upload pass_of");
}

tqsim_handle* create_handle(const tqsim_circuit* c, const tqsim_noise_model* nm, uint64_t n_shots,
                            const uint32_t* arities, uint32_t n_levels, const tqsim_options* o,
                            bool need_gpu) {
  validate_noise(nm);
  Options opts = options_from(o);
  auto* h = new tqsim_handle();
  try {
    h->n_user = c ? c->n_qubits : 0;
    h->gates = lower(c);
    h->opts = opts;
    h->noise = *nm;
    h->kraus = kraus_enabled(*nm);
    if (h->kraus && c->n_qubits > TQSIM_KRAUS_MAX_QUBITS)
      throw Error{TQSIM_EINVAL, "non-Pauli channels (amplitude / phase damping, thermal relaxation) run in the "
                                "shared-memory Kraus engine: n_qubits must be <= 16"};
    if (opts.copy_cost_gates == -1.0 && !arities) {
      // copy cost of this engine's fused fan-out: the child's
      // first pass reads the parent instead of its own state, so the copy adds no HBM pass; what
      // a level boundary costs is the pass it may split, on average half a pass = half the
      // gates one pass holds.  Gates per pass from the pass planner on the whole circuit.
      Plan whole;
      whole.arities = {1};
      whole.bounds = {0, h->gates.size()};
      const PassPlan pw = make_pass_plan(h->gates, c->n_qubits, whole, opts);
      const double gpp = (double)h->gates.size() / (double)std::max<size_t>(1, pw.levels[0].size());
      opts.copy_cost_gates = std::max(1.0, 0.5 * gpp);
      h->opts.copy_cost_gates = opts.copy_cost_gates;
    }
    h->plan = make_plan(h->gates, c->n_qubits, nm, n_shots, arities, n_levels, opts);
    h->pp = make_pass_plan(h->gates, c->n_qubits, h->plan, opts);
    h->n_sim = h->pp.n_sim;
    h->inst = instances(h->plan);
    fill_plan(h->plan, c->n_qubits, h->gates.size(), h->pp.passes_total(h->inst), &h->cplan);
    h->cplan.tile_qubits = h->pp.levels.empty() || h->pp.levels[0].empty() ? 0u : (uint32_t)h->pp.levels[0][0].K;
    h->cplan.trail_top_bits = h->pp.trail.on && !h->kraus ? (uint32_t)h->pp.trail.m : 0u;
    h->cplan.trail_fast = h->pp.trail.on && !h->kraus && h->pp.trail.fast ? 1u : 0u;
    {   // small-state tree: eligible for narrow Pauli-noise circuits; auto when
        // the per-leaf recompute (n_outcomes x lowered gates x 2^n) stays small
      const double flat = (double)h->cplan.n_outcomes * (double)h->gates.size() *
                          (double)(1ull << std::max(h->n_sim, 5));
      const char* env = std::getenv("TQSIM_SMALL");   // "0": auto never picks it (explicit 1 still does)
      // auto: only where the whole tree is a few microseconds of work (measured crossover
      // 2^23..2^25 amplitude-gate updates, profiles/r02_small_tree_sweep.jsonl)
      const bool auto_ok = !(env && env[0] == '0') && flat <= 16777216.0;
      h->small = !h->kraus && h->n_user <= (uint32_t)TQSIM_SMALL_MAX_QUBITS && opts.small_tree != 2 &&
                 (opts.small_tree == 1 || auto_ok);
      h->cplan.small_tree = h->small ? 1u : 0u;
    }
    if (need_gpu) {
      require_device();
      const size_t G = std::max<size_t>(h->gates.size(), 1);
      ckc(cudaMalloc(reinterpret_cast<void**>(&h->d_two), G), "cudaMalloc two");
      ckc(cudaMalloc(reinterpret_cast<void**>(&h->d_pass_of), G), "cudaMalloc pass_of");
      ckc(cudaMalloc(reinterpret_cast<void**>(&h->d_seed), 8), "cudaMalloc seed");
      h->h_tables.assign(2 * G, 0);
      for (size_t g = 0; g < h->gates.size(); ++g) h->h_tables[g] = h->gates[g].two ? 1 : 0;
      for (const auto& lvl : h->pp.levels)
        for (const PassDesc& pd : lvl)
          for (uint32_t oi = pd.op_begin; oi < pd.op_end; ++oi)
            h->h_tables[G + h->pp.ops[oi].gate] = (uint8_t)std::min<uint32_t>(pd.pass_index, 31);
      upload_gate_tables(h, nullptr);
      ckc(cudaStreamSynchronize(nullptr), "upload gate tables");
      if (h->kraus || h->small) {   // the Kraus engine / small tree read the lowered gates from HBM
        std::vector<KGate> kg(h->gates.size());
        for (size_t g = 0; g < h->gates.size(); ++g) {
          const LGate& l = h->gates[g];
          kg[g].two = l.two ? 1u : 0u;
          kg[g].op = l.op;
          kg[g].q0 = l.q0;
          kg[g].q1 = l.q1;
          for (int k = 0; k < 8; ++k) kg[g].m[k] = l.m[k];
        }
        ckc(cudaMalloc(reinterpret_cast<void**>(&h->d_kgates), sizeof(KGate) * std::max<size_t>(kg.size(), 1)),
            "cudaMalloc kraus gates");
        ckc(cudaMemcpy(h->d_kgates, kg.data(), sizeof(KGate) * kg.size(), cudaMemcpyHostToDevice), "kraus gates");
      }
      if (h->pp.trail.on && !h->kraus) {   // pass A's gates within the leaf slice
        const size_t L = h->plan.arities.size();
        const uint64_t b0 = h->plan.bounds[L - 1], len = h->plan.bounds[L] - b0;
        std::vector<uint8_t> asel(std::max<uint64_t>(len, 1), 0);
        const PassDesc& pa = h->pp.trail.a;
        for (uint32_t oi = pa.op_begin; oi < pa.op_end; ++oi) asel.at(h->pp.ops[oi].gate - b0) = 1;
        ckc(cudaMalloc(reinterpret_cast<void**>(&h->d_trail_asel), asel.size()), "cudaMalloc trail asel");
        ckc(cudaMemcpy(h->d_trail_asel, asel.data(), asel.size(), cudaMemcpyHostToDevice), "trail asel");
      }
      if (!h->kraus) {
        // gate tables (gate sequence, qubit positions, matrices) become code + constant banks
        // (small-state handles too: state dumps run the general tree)
        h->jit = jit_build(h->pp, h->gates, &h->compile_s, &h->jit_trail);
      }

    }
  } catch (...) {
    tqsim_destroy(h);
    throw;
  }
  return h;
}

void execute(tqsim_handle* h, uint64_t seed, uint32_t rank, uint32_t world, cudaStream_t st,
             void* ws, uint64_t ws_bytes, uint32_t* d_out) {
  if (!h) throw Error{TQSIM_EINVAL, "handle is NULL"};
  if (!d_out) throw Error{TQSIM_EINVAL, "d_leaf_outcomes is NULL"};
  const ShardRange sr = shard_levels(h->cplan, rank, world);
  Exec x = make_exec(h, seed, st, ws, sr, d_out);
  if (!ws || ws_bytes < x.L.total) throw Error{TQSIM_ECAPACITY, "workspace too small"};
  if (reinterpret_cast<uintptr_t>(ws) % ALIGN) throw Error{TQSIM_EINVAL, "workspace not 256-byte aligned"};
  h->stats = tqsim_stats{};
  h->ev_used = 0;
  h->ev_marks.clear();
  h->ev_tags.clear();
  ck(launch_set_seed(h->d_seed, seed, st), "seed launch");
  static const bool graphs = [] {
    const char* e = std::getenv("TQSIM_GRAPH");
    return !(e && e[0] == '0');
  }();
  const bool dumps = h->debug && h->debug->n_dumps;
  if (!sr.empty() && graphs && !h->opts.profile && !dumps && !h->kraus) {
    // replay the captured tree: one graph launch instead of one host launch per kernel
    const std::vector<uint64_t> key = {reinterpret_cast<uint64_t>(ws), ws_bytes, reinterpret_cast<uint64_t>(d_out),
                                       rank, world, reinterpret_cast<uint64_t>(h->d_dbg_u),
                                       reinterpret_cast<uint64_t>(h->d_dbg_total),
                                       reinterpret_cast<uint64_t>(h->d_dbg_flag)};
    if (!h->graph_exec || h->graph_key != key) {
      if (h->graph_exec) cudaGraphExecDestroy(h->graph_exec);
      h->graph_exec = nullptr;
      if (!h->capture_stream)
        ckc(cudaStreamCreateWithFlags(&h->capture_stream, cudaStreamNonBlocking), "capture stream");
      Exec xc = x;
      xc.st = h->capture_stream;
      static const bool pipe_on = [] {
        const char* e = std::getenv("TQSIM_PIPE");
        return !(e && e[0] == '0');
      }();
      if (pipe_on && h->plan.arities.size() >= 2) {
        if (!h->leaf_stream) {
          // highest priority: as CTAs of the running HBM-bound pass retire, the block
          // scheduler fills the freed slots with the FP64-bound leaf CTAs (node priorities
          // kept by the graph: cudaGraphInstantiateFlagUseNodePriority)
          int lo = 0, hi = 0;
          ckc(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
          ckc(cudaStreamCreateWithPriority(&h->leaf_stream, cudaStreamNonBlocking, hi), "leaf stream");
          for (cudaEvent_t& e : h->pipe_ev) ckc(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "pipe event");
        }
        xc.pipe = true;
        xc.st2 = h->leaf_stream;
        xc.ev = h->pipe_ev;
      }
      ckc(cudaStreamBeginCapture(h->capture_stream, cudaStreamCaptureModeThreadLocal), "begin capture");
      cudaGraph_t g = nullptr;
      try {
        run_tree(xc);
      } catch (...) {
        cudaStreamEndCapture(h->capture_stream, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      ckc(cudaStreamEndCapture(h->capture_stream, &g), "end capture");
      const cudaError_t e = cudaGraphInstantiate(&h->graph_exec, g, cudaGraphInstantiateFlagUseNodePriority);
      cudaGraphDestroy(g);
      ckc(e, "graph instantiate");
      h->graph_key = key;
      h->graph_stats = h->stats;
    }
    h->stats = h->graph_stats;
    h->stats.kernel_launches += 1;   // the seed kernel
    ckc(cudaGraphLaunch(h->graph_exec, st), "graph launch");
    return;
  }
  if (!sr.empty()) run_tree(x);
  h->stats.kernel_launches += 1;     // the seed kernel
  if (h->opts.profile) {
    ckc(cudaStreamSynchronize(st), "profile sync");
    for (size_t i = 0; i + 1 < h->ev_marks.size(); i += 2) {
      float ms = 0.f;
      ckc(cudaEventElapsedTime(&ms, h->ev_pool[h->ev_marks[i].second],
                               h->ev_pool[h->ev_marks[i + 1].second]),
          "cudaEventElapsedTime");
      if (h->ev_marks[i].first == 0) h->stats.pass_ms += ms;
      else if (h->ev_marks[i].first == 1) h->stats.measure_ms += ms;
      else h->stats.noise_ms += ms;
    }
    if (const char* path = std::getenv("TQSIM_PROFILE_DUMP")) {   // every interval: kind, ms
      if (FILE* f = std::fopen(path, "a")) {
        for (size_t i = 0; i + 1 < h->ev_marks.size(); ++i) {
          float ms = 0.f;
          cudaEventElapsedTime(&ms, h->ev_pool[h->ev_marks[i].second], h->ev_pool[h->ev_marks[i + 1].second]);
          std::fprintf(f, "%d %d %.6f\n", h->ev_marks[i].first, (int)(i & 1), ms);
        }
        std::fclose(f);
      }
    }
  }
}

// Work the tree actually executed (DESIGN.md §7 "shared states computed once"): per batch
// of every level, formed exactly as run_level forms them, the instances that were computed
// (dedup representatives; every instance when dedup is off) and the distinct parent states
// their fan-out pass read.  Reads the dedup maps back from the workspace (synchronous).
struct BatchWork {
  uint64_t comp = 0, parents = 0;
  uint64_t parents_all = 0;   // distinct parent states (representatives) read by ALL instances
};
using WorkMap = std::map<std::pair<uint32_t, uint64_t>, BatchWork>;

WorkMap computed_work(const tqsim_handle* h, const ShardRange& sr, const Layout& L, const char* ws, bool dedup) {
  std::vector<uint32_t> maps;
  if (dedup && L.map_entries) {
    maps.resize(2 * L.map_entries);
    ckc(cudaMemcpy(maps.data(), ws + L.map_off, 8 * L.map_entries, cudaMemcpyDeviceToHost), "maps D2H");
  }
  const size_t levels = h->plan.arities.size();
  WorkMap out;
  auto rep = [&](uint32_t d, uint64_t j) -> uint64_t {   // global id of j's representative
    if (!dedup) return j;
    const uint64_t idx = L.map_lvl[d] + (j - sr.lo[d]);
    return j - maps[L.map_entries + idx] + maps[idx];
  };
  std::function<void(uint32_t, uint64_t, uint64_t)> walk = [&](uint32_t d, uint64_t i0, uint64_t i1) {
    for (uint64_t b = i0; b < i1; b += L.cap[d]) {
      const uint64_t cnt = std::min(L.cap[d], i1 - b);
      BatchWork w;
      std::vector<uint64_t> par, pall;
      for (uint64_t j = b; j < b + cnt; ++j) {
        const uint64_t pr = d > 0 ? rep(d - 1, j / h->plan.arities[d]) : 0;
        if (d > 0) pall.push_back(pr);
        if (cnt > 1 && rep(d, j) != j) continue;
        ++w.comp;
        if (d > 0) par.push_back(pr);
      }
      std::sort(par.begin(), par.end());
      w.parents = (uint64_t)(std::unique(par.begin(), par.end()) - par.begin());
      std::sort(pall.begin(), pall.end());
      w.parents_all = (uint64_t)(std::unique(pall.begin(), pall.end()) - pall.begin());
      out[{d, b}] = w;
      if (d + 1 < levels) {
        const uint64_t A = h->plan.arities[d + 1];
        walk(d + 1, std::max(b * A, sr.lo[d + 1]), std::min((b + cnt) * A, sr.hi[d + 1]));
      }
    }
  };
  if (!sr.empty()) walk(0, sr.lo[0], sr.hi[0]);
  return out;
}

// algorithmic bytes of pass p of level d over `comp` computed states reading `parents`
// distinct parent states: in place 32 B / amplitude; fan-out 16 B written
// + 16 B per amplitude of each parent read; root 16 B written; the leaf's run-sums-only
// pass writes 1 B / amplitude instead of 16.
double pass_alg_bytes(const tqsim_handle* h, uint32_t d, size_t p, uint64_t comp, uint64_t parents, bool nostore) {
  if (h->kraus) {   // Kraus engine: one kernel per level; parent read + state write (none at a leaf)
    if (p > 0) return 0.0;
    const double amps = (double)comp * (double)(1ull << h->n_user);
    return amps * ((d > 0 ? 16.0 : 0.0) + (d + 1 == h->plan.arities.size() ? 0.0 : 16.0));
  }
  const double amps = (double)comp * (double)(1ull << h->n_sim);
  const bool runsums_only = nostore && h->pp.levels[d][p].leaf_sums;
  double bytes = runsums_only ? amps : amps * 16.0;
  if (p > 0) bytes += amps * 16.0;
  else if (d > 0) bytes += (double)parents * (double)(1ull << h->n_sim) * 16.0;
  return bytes;
}

// Conditional leaf sampling (run_leaf_trail): algorithmic bytes of its kernels over a leaf
// batch of `cnt` leaves, `comp` of them computed, reading `parents` (computed) / `parents_all`
// distinct parent states.  pass 0 = A (run sums), 100 = projection, 101 + p = stage-2 pass p.
double trail_alg_bytes(const tqsim_handle* h, uint32_t pass, uint64_t cnt, uint64_t comp, uint64_t parents,
                       uint64_t parents_all) {
  const double S = (double)(1ull << h->n_sim), S2 = (double)(1ull << h->pp.trail.n2);
  if (pass == 0) return (double)comp * S + (double)parents * S * 16.0;
  if (pass == 100) return (double)parents_all * S * 16.0 + (double)cnt * S2 * 16.0;
  const bool lastp = pass - 101 + 1 == h->pp.trail.b.size();
  return (double)cnt * S2 * (lastp ? 17.0 : 32.0);
}

bool trail_active(const tqsim_handle* h) { return h->pp.trail.on && !(h->debug && h->debug->n_dumps); }

void fill_computed(tqsim_handle* h, const ShardRange& sr, const Layout& L, const char* ws) {
  const bool dumps = h->debug && h->debug->n_dumps;
  if (h->small && !dumps) {   // small-state tree: every leaf recomputes its whole path, no HBM states
    const size_t Lv = h->plan.arities.size();
    const uint64_t leaves = sr.empty() ? 0 : sr.hi[Lv - 1] - sr.lo[Lv - 1];
    h->stats.computed_node_executions = leaves * Lv;
    h->stats.computed_gate_amp_updates = (leaves * h->plan.bounds[Lv]) << h->n_user;
    h->stats.computed_pass_bytes = 0;
    return;
  }
  const bool dedup = !dumps && !h->opts.no_dedup && !h->kraus;
  const WorkMap wm = computed_work(h, sr, L, ws, dedup);
  tqsim_stats& st = h->stats;
  st.computed_node_executions = st.computed_gate_amp_updates = st.computed_pass_bytes = 0;
  double bytes = 0.0;
  for (const auto& kv : wm) {
    const uint32_t d = kv.first.first;
    const BatchWork& w = kv.second;
    st.computed_node_executions += w.comp;
    st.computed_gate_amp_updates += (w.comp * (h->plan.bounds[d + 1] - h->plan.bounds[d])) << h->n_user;
    if (d + 1 == h->plan.arities.size() && trail_active(h)) {
      const uint64_t b = kv.first.second;
      const uint64_t cnt = std::min(L.cap[d], sr.hi[d] - b);
      const uint64_t pall = w.parents_all;
      bytes += trail_alg_bytes(h, 0, cnt, w.comp, w.parents, pall) + trail_alg_bytes(h, 100, cnt, w.comp, w.parents, pall);
      for (size_t p = 0; p < h->pp.trail.b.size(); ++p)
        bytes += trail_alg_bytes(h, 101 + (uint32_t)p, cnt, w.comp, w.parents, pall);
      continue;
    }
    const size_t np = h->kraus ? 1 : h->pp.levels[d].size();
    for (size_t p = 0; p < np; ++p) bytes += pass_alg_bytes(h, d, p, w.comp, w.parents, !dumps);
  }
  st.computed_pass_bytes = (uint64_t)bytes;
}

void build_result(tqsim_handle* h, const std::vector<uint32_t>& outs, double wall, tqsim_result** out) {
  auto* r = static_cast<tqsim_result*>(std::calloc(1, sizeof(tqsim_result)));
  if (!r) throw std::bad_alloc();
  r->plan = h->cplan;
  r->stats = h->stats;
  r->wall_s = wall;
  std::vector<uint64_t> bits, counts;
  if (h->n_user <= 24 && (1ull << h->n_user) <= 8 * std::max<size_t>(outs.size(), 1)) {
    // counting histogram over the 2^n outcomes (ascending bitstrings, as the sort gives)
    std::vector<uint32_t> hist(1ull << h->n_user, 0u);
    for (uint32_t v : outs) ++hist[v];
    for (size_t v = 0; v < hist.size(); ++v)
      if (hist[v]) {
        bits.push_back(v);
        counts.push_back(hist[v]);
      }
  } else {
    std::vector<uint32_t> sorted = outs;
    std::sort(sorted.begin(), sorted.end());
    for (size_t i = 0; i < sorted.size();) {
      size_t j = i;
      while (j < sorted.size() && sorted[j] == sorted[i]) ++j;
      bits.push_back(sorted[i]);
      counts.push_back(j - i);
      i = j;
    }
  }
  r->n_distinct = bits.size();
  r->bitstrings = static_cast<uint64_t*>(std::malloc(std::max<size_t>(1, bits.size()) * 8));
  r->counts = static_cast<uint64_t*>(std::malloc(std::max<size_t>(1, counts.size()) * 8));
  r->leaf_outcomes = static_cast<uint32_t*>(std::malloc(std::max<size_t>(1, outs.size()) * 4));
  if (!r->bitstrings || !r->counts || !r->leaf_outcomes) {
    tqsim_result_free(r);
    throw std::bad_alloc();
  }
  std::memcpy(r->bitstrings, bits.data(), bits.size() * 8);
  std::memcpy(r->counts, counts.data(), counts.size() * 8);
  std::memcpy(r->leaf_outcomes, outs.data(), outs.size() * 4);
  *out = r;
}

}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }

}  // namespace tq

using namespace tq;

extern "C" {

void tqsim_default_options(tqsim_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->copy_cost_gates = 10.0;
  o->z = 1.96;
  o->eps = 0.05;
  o->mem_budget_bytes = 180000000000ull;
}

const char* tqsim_last_error(void) { return g_last_error.c_str(); }
const char* tqsim_version(void) { return "tqsim-b200 0.1 (sm_100a)"; }

tqsim_status tqsim_lower_circuit(const tqsim_circuit* c, tqsim_gate* out, uint64_t cap,
                                 uint64_t* n_out) {
  return guarded([&] {
    std::vector<LGate> g = lower(c);
    if (!n_out) throw Error{TQSIM_EINVAL, "n_out is NULL"};
    *n_out = g.size();
    for (uint64_t i = 0; i < g.size() && i < cap && out; ++i) {
      out[i] = tqsim_gate{};
      out[i].kind = g[i].kind;
      out[i].q0 = g[i].q0;
      out[i].q1 = g[i].two ? g[i].q1 : 0;
    }
  });
}

tqsim_status tqsim_plan_circuit(const tqsim_circuit* c, const tqsim_noise_model* nm,
                                uint64_t n_shots, const uint32_t* arities, uint32_t n_levels,
                                const tqsim_options* o, tqsim_plan* out) {
  return guarded([&] {
    if (!out) throw Error{TQSIM_EINVAL, "out is NULL"};
    tqsim_handle* h = create_handle(c, nm, n_shots, arities, n_levels, o, false);
    *out = h->cplan;
    tqsim_destroy(h);
  });
}

tqsim_status tqsim_describe_passes(const tqsim_circuit* c, const tqsim_noise_model* nm,
                                   uint64_t n_shots, const uint32_t* arities, uint32_t n_levels,
                                   const tqsim_options* o, tqsim_op_record* out, uint64_t cap,
                                   uint64_t* n_out) {
  return guarded([&] {
    if (!n_out) throw Error{TQSIM_EINVAL, "n_out is NULL"};
    tqsim_handle* h = create_handle(c, nm, n_shots, arities, n_levels, o, false);
    uint64_t k = 0;
    for (size_t d = 0; d < h->pp.levels.size(); ++d)
      for (size_t p = 0; p < h->pp.levels[d].size(); ++p) {
        const PassDesc& pd = h->pp.levels[d][p];
        for (uint32_t ph = pd.phase_begin; ph < pd.phase_end; ++ph) {
          const PhaseDesc& P = h->pp.phases[ph];
          uint64_t rmask = 0;
          for (int b = 0; b < RBITS; ++b) rmask |= 1ull << pd.tile_q[P.rpos[b]];
          for (uint32_t i = P.op_begin; i < P.op_end; ++i, ++k)
            if (out && k < cap)
              out[k] = tqsim_op_record{(uint32_t)d, (uint32_t)p, ph - pd.phase_begin,
                                       h->pp.ops[i].gate, pd.tile_mask, rmask, h->pp.ops[i].role, 0u};
        }
      }
    *n_out = k;
    tqsim_destroy(h);
  });
}

tqsim_status tqsim_compile_passes(const tqsim_circuit* c, const tqsim_noise_model* nm,
                                  uint64_t n_shots, const uint32_t* arities, uint32_t n_levels,
                                  const tqsim_options* o, uint64_t* n_kernels,
                                  uint64_t* cubin_bytes, double* seconds) {
  return guarded([&] {
    tqsim_handle* h = create_handle(c, nm, n_shots, arities, n_levels, o, false);
    const auto t0 = std::chrono::steady_clock::now();
    try {
      jit_compile_only(h->pp, h->gates, n_kernels, cubin_bytes);
    } catch (...) {
      tqsim_destroy(h);
      throw;
    }
    if (seconds)
      *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    tqsim_destroy(h);
  });
}

tqsim_status tqsim_pass_source(const tqsim_circuit* c, const tqsim_noise_model* nm,
                               uint64_t n_shots, const uint32_t* arities, uint32_t n_levels,
                               const tqsim_options* o, uint32_t level, uint32_t pass, char* out,
                               uint64_t cap, uint64_t* n_out) {
  return guarded([&] {
    tqsim_handle* h = create_handle(c, nm, n_shots, arities, n_levels, o, false);
    std::string s;
    try {
      if (level >= h->pp.levels.size() || pass >= h->pp.levels[level].size())
        throw Error{TQSIM_EINVAL, "level/pass out of range"};
      s = jit_source(h->pp, h->gates, level, pass, "tq_pass");
    } catch (...) {
      tqsim_destroy(h);
      throw;
    }
    tqsim_destroy(h);
    if (n_out) *n_out = s.size();
    if (out && cap) {
      const size_t k = std::min<size_t>(cap - 1, s.size());
      std::memcpy(out, s.data(), k);
      out[k] = '\0';
    }
  });
}

tqsim_status tqsim_shard_range(const tqsim_plan* p, uint32_t rank, uint32_t world,
                               uint64_t* top_begin, uint64_t* top_end, uint64_t* leaf_begin,
                               uint64_t* leaf_end) {
  return guarded([&] {
    if (!p || p->n_levels < 1) throw Error{TQSIM_EINVAL, "plan is NULL or empty"};
    const ShardRange r = shard_levels(*p, rank, world);
    if (top_begin) *top_begin = r.lo[0];
    if (top_end) *top_end = r.hi[0];
    if (leaf_begin) *leaf_begin = r.lo.back();
    if (leaf_end) *leaf_end = r.hi.back();
  });
}

tqsim_status tqsim_create(const tqsim_circuit* c, const tqsim_noise_model* nm, uint64_t n_shots,
                          const uint32_t* arities, uint32_t n_levels, const tqsim_options* o,
                          tqsim_handle** out) {
  return guarded([&] {
    if (!out) throw Error{TQSIM_EINVAL, "out is NULL"};
    *out = create_handle(c, nm, n_shots, arities, n_levels, o, true);
  });
}

tqsim_status tqsim_get_plan(const tqsim_handle* h, tqsim_plan* out) {
  return guarded([&] {
    if (!h || !out) throw Error{TQSIM_EINVAL, "NULL argument"};
    *out = h->cplan;
  });
}

tqsim_status tqsim_get_stats(const tqsim_handle* h, tqsim_stats* out) {
  return guarded([&] {
    if (!h || !out) throw Error{TQSIM_EINVAL, "NULL argument"};
    *out = h->stats;
  });
}

void tqsim_destroy(tqsim_handle* h) {
  if (!h) return;
  if (h->d_two) cudaFree(h->d_two);
  if (h->d_pass_of) cudaFree(h->d_pass_of);
  if (h->d_seed) cudaFree(h->d_seed);
  if (h->d_kgates) cudaFree(h->d_kgates);
  if (h->d_trail_asel) cudaFree(h->d_trail_asel);
  if (h->h_tables_pinned) cudaFreeHost(h->h_tables_pinned);
  if (h->graph_exec) cudaGraphExecDestroy(h->graph_exec);
  if (h->capture_stream) cudaStreamDestroy(h->capture_stream);
  if (h->leaf_stream) cudaStreamDestroy(h->leaf_stream);
  for (cudaEvent_t e : h->pipe_ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : h->map_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
  delete h;
}

tqsim_status tqsim_workspace_bytes(const tqsim_handle* h, uint32_t rank, uint32_t world,
                                   uint64_t* bytes) {
  return guarded([&] {
    if (!h || !bytes) throw Error{TQSIM_EINVAL, "NULL argument"};
    *bytes = layout(h, shard_levels(h->cplan, rank, world)).total;
  });
}

tqsim_status tqsim_execute(tqsim_handle* h, uint64_t seed, uint32_t rank, uint32_t world,
                           void* stream, void* d_workspace, uint64_t workspace_bytes,
                           uint32_t* d_leaf_outcomes) {
  return guarded([&] {
    execute(h, seed, rank, world, static_cast<cudaStream_t>(stream), d_workspace, workspace_bytes,
            d_leaf_outcomes);
  });
}

tqsim_status tqsim_profile_passes(tqsim_handle* h, uint64_t seed, uint32_t rank, uint32_t world,
                                  void* stream, void* d_workspace, uint64_t workspace_bytes,
                                  uint32_t* d_leaf_outcomes, uint32_t reps, tqsim_pass_timing* out,
                                  uint64_t cap, uint64_t* n_out) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  const tqsim_status r = guarded([&] {
    if (!h || !n_out || reps < 1) throw Error{TQSIM_EINVAL, "NULL argument or reps < 1"};
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    // one real run: every level buffer holds states of the tree (batch 0 of each level)
    execute(h, seed, rank, world, st, d_workspace, workspace_bytes, d_leaf_outcomes);
    ckc(cudaStreamSynchronize(st), "sync");
    const ShardRange sr = shard_levels(h->cplan, rank, world);
    Exec x = make_exec(h, seed, st, d_workspace, sr, d_leaf_outcomes);
    ckc(cudaEventCreate(&e0), "event");
    ckc(cudaEventCreate(&e1), "event");
    const int n = h->n_sim;
    uint64_t k = 0;
    for (size_t d = 0; d < h->pp.levels.size() && !h->kraus; ++d) {
      const uint64_t inst = sr.count(d);
      if (inst == 0) continue;
      const uint64_t cnt = std::min<uint64_t>(x.L.cap[d], inst);
      const uint64_t first = sr.lo[d];   // first instance of the shard
      const uint32_t slice_begin = (uint32_t)h->plan.bounds[d];
      const uint32_t slice_len = (uint32_t)(h->plan.bounds[d + 1] - slice_begin);
      const uint32_t row_bytes = noise_row_bytes(slice_len);
      // the level's first batch's noise rows (drawn by the run above)
      uint8_t* rows = reinterpret_cast<uint8_t*>(x.ws + x.L.rows_off + x.L.rows_lvl_off[d]);
      (void)slice_begin;
      // as in the tree, instances sharing a representative's state are skipped and a
      // fan-out reads a skipped parent's representative (the dedup maps the run above
      // built); count the computed instances and the distinct parent states they read
      const bool dd = !(h->debug && h->debug->n_dumps) && !h->opts.no_dedup;
      const uint64_t A = h->plan.arities[d];
      const uint64_t pcnt_batch = d > 0 ? std::min<uint64_t>(x.L.cap[d - 1], sr.count(d - 1)) : 0;
      const uint32_t* maps = reinterpret_cast<const uint32_t*>(x.ws + x.L.map_off);
      const uint32_t* rep_d = dd && cnt > 1 ? maps + x.L.map_lvl[d] : nullptr;
      const uint32_t* rep_p = dd && d > 0 && pcnt_batch > 1 ? maps + x.L.map_lvl[d - 1] : nullptr;
      uint64_t comp = cnt, comp_par = 0;
      {
        std::vector<uint32_t> hr(cnt), hp(pcnt_batch);
        for (uint64_t q = 0; q < cnt; ++q) hr[q] = (uint32_t)q;
        for (uint64_t q = 0; q < pcnt_batch; ++q) hp[q] = (uint32_t)q;
        if (rep_d) ckc(cudaMemcpy(hr.data(), rep_d, cnt * 4, cudaMemcpyDeviceToHost), "map D2H");
        if (rep_p) ckc(cudaMemcpy(hp.data(), rep_p, pcnt_batch * 4, cudaMemcpyDeviceToHost), "map D2H");
        const uint64_t pfirst = d > 0 ? first / A : 0;
        std::vector<char> seen(pcnt_batch, 0);
        comp = 0;
        for (uint64_t q = 0; q < cnt; ++q) {
          if (hr[q] != q) continue;
          ++comp;
          if (d > 0) {
            const uint64_t pq = hp[(first + q) / A - pfirst];
            if (!seen[pq]) {
              seen[pq] = 1;
              ++comp_par;
            }
          }
        }
      }
      for (size_t p = 0; p < h->pp.levels[d].size(); ++p) {
        PassLaunch pl{};
        pl.src_mode = p > 0 ? 2u : (d == 0 ? 0u : 1u);
        pl.src = d > 0 ? x.ws + x.L.off[d - 1] : nullptr;
        pl.dst = x.ws + x.L.off[d];
        pl.child_first = first;
        pl.parent_first = d > 0 ? first / h->plan.arities[d] : 0;
        pl.arity = h->plan.arities[d];
        pl.batch = (uint32_t)cnt;
        pl.seed = seed;
        pl.p1 = h->noise.p1;
        pl.p2 = h->noise.p2;
        pl.runsum = x.ws + x.L.runs_off;
        pl.rows = rows;
        pl.row_bytes = row_bytes;
        const PassDesc& pd = h->pp.levels[d][p];
        // as in the tree: the leaf's last pass stores run sums only
        pl.variant = pd.leaf_sums ? 1u : 0u;
        pl.xlout = reinterpret_cast<uint32_t*>(x.ws + x.L.sel_off + 2 * align_up(4 * x.L.cap.back()));
        pl.rep = rep_d;
        pl.prep = rep_p;
        ck(launch_jit_pass(h->jit[d][p], pd, pl, st), "gate pass launch");   // warm
        ckc(cudaEventRecord(e0, st), "record");
        for (uint32_t i = 0; i < reps; ++i) ck(launch_jit_pass(h->jit[d][p], pd, pl, st), "gate pass launch");
        ckc(cudaEventRecord(e1, st), "record");
        ckc(cudaEventSynchronize(e1), "sync");
        float ms = 0.f;
        ckc(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
        const uint64_t amps = comp << n;   // computed children only (leaf dedup)
        double bytes = pl.variant == 1 ? (double)amps : (double)amps * 16;
        if (pl.src_mode == 2) bytes += (double)amps * 16;
        else if (pl.src_mode == 1) bytes += (double)(comp_par << n) * 16;
        if (out && k < cap) {
          tqsim_pass_timing& o = out[k];
          o.level = (uint32_t)d;
          o.pass = (uint32_t)p;
          o.states_per_launch = (uint32_t)cnt;
          o.reserved = 0;
          o.launches_per_tree = (double)inst / (double)cnt;
          o.ms_per_launch = ms / reps;
          o.alg_bytes_per_launch = bytes;
        }
        ++k;
      }
    }
    *n_out = k;
  });
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  return r;
}

tqsim_status tqsim_shard_levels(const tqsim_plan* p, uint32_t rank, uint32_t world, uint32_t* split_level,
                                uint64_t* lo, uint64_t* hi) {
  return guarded([&] {
    if (!p || p->n_levels < 1) throw Error{TQSIM_EINVAL, "plan is NULL or empty"};
    const ShardRange r = shard_levels(*p, rank, world);
    if (split_level) *split_level = r.split;
    for (uint32_t d = 0; d < p->n_levels; ++d) {
      if (lo) lo[d] = r.lo[d];
      if (hi) hi[d] = r.hi[d];
    }
  });
}

tqsim_status tqsim_profile_tree(tqsim_handle* h, uint64_t seed, uint32_t rank, uint32_t world, void* stream,
                                void* d_workspace, uint64_t workspace_bytes, uint32_t* d_leaf_outcomes,
                                tqsim_kernel_timing* out, uint64_t cap, uint64_t* n_out) {
  uint32_t prof0 = 0;
  const tqsim_status r = guarded([&] {
    if (!h || !n_out) throw Error{TQSIM_EINVAL, "NULL argument"};
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    prof0 = h->opts.profile;
    h->opts.profile = 1;
    h->tag_launches = true;
    execute(h, seed, rank, world, st, d_workspace, workspace_bytes, d_leaf_outcomes);   // synchronizes
    const ShardRange sr = shard_levels(h->cplan, rank, world);
    const Layout lay = layout(h, sr);
    const bool dedup = !(h->debug && h->debug->n_dumps) && !h->opts.no_dedup && !h->kraus && !h->small;
    const WorkMap wm = computed_work(h, sr, lay, static_cast<const char*>(d_workspace), dedup);
    fill_computed(h, sr, lay, static_cast<const char*>(d_workspace));
    std::map<std::tuple<int, uint32_t, uint32_t>, tqsim_kernel_timing> agg;
    for (size_t i = 0; i + 1 < h->ev_marks.size(); i += 2) {
      const tqsim_handle::Tag& tg = h->ev_tags.at(i / 2);
      float ms = 0.f;
      ckc(cudaEventElapsedTime(&ms, h->ev_pool[h->ev_marks[i].second], h->ev_pool[h->ev_marks[i + 1].second]),
          "elapsed");
      tqsim_kernel_timing& k = agg[std::make_tuple(tg.kind, tg.level, tg.pass)];
      k.kind = (uint32_t)tg.kind;
      k.level = tg.level;
      k.pass = tg.pass;
      k.launches += 1;
      k.ms += ms;
      if (tg.kind != 0 && tg.kind != 3) continue;
      k.states += tg.cnt;
      auto it = wm.find({tg.level, tg.b});
      const BatchWork w = it != wm.end() ? it->second : BatchWork{tg.cnt, 0};
      if (tg.kind == 0 && tg.level + 1 == h->plan.arities.size() && trail_active(h)) {   // trail kernels
        const uint64_t A = h->plan.arities[tg.level];
        const uint64_t pall = it != wm.end() ? w.parents_all : (tg.b + tg.cnt - 1) / A - tg.b / A + 1;
        const uint64_t comp = tg.pass == 0 ? w.comp : tg.cnt;
        k.computed_states += comp;
        k.alg_bytes += trail_alg_bytes(h, tg.pass, tg.cnt, w.comp, w.parents, pall);
        const uint64_t pnom = (tg.b + tg.cnt - 1) / A - tg.b / A + 1;
        k.nominal_bytes += trail_alg_bytes(h, tg.pass, tg.cnt, tg.cnt, pnom, pnom);
        k.fp64_per_amp = tg.pass == 0 || tg.pass == 100 ? h->jit_trail.a.fp64_per_amp
                                                         : h->jit_trail.b[tg.pass - 101].fp64_per_amp;
        continue;
      }
      if (tg.kind == 0) k.fp64_per_amp = h->jit[tg.level][tg.pass].fp64_per_amp;
      k.computed_states += w.comp;
      k.alg_bytes += pass_alg_bytes(h, tg.level, tg.pass, w.comp, w.parents, !(h->debug && h->debug->n_dumps));
      const uint64_t A = h->plan.arities[tg.level];
      const uint64_t par = tg.level > 0 ? (tg.b + tg.cnt - 1) / A - tg.b / A + 1 : 0;
      k.nominal_bytes += pass_alg_bytes(h, tg.level, tg.pass, tg.cnt, par, !(h->debug && h->debug->n_dumps));
    }
    uint64_t k = 0;
    for (const auto& kv : agg) {
      if (out && k < cap) out[k] = kv.second;
      ++k;
    }
    *n_out = k;
  });
  if (h) {
    h->opts.profile = prof0;
    h->tag_launches = false;
  }
  return r;
}

tqsim_status tqsim_run_ex(const tqsim_circuit* c, const tqsim_noise_model* nm, uint64_t n_shots,
                          const uint32_t* arities, uint32_t n_levels, uint64_t seed,
                          const tqsim_options* o, const tqsim_debug* debug, tqsim_result** out) {
  return guarded([&] {
    if (!out) throw Error{TQSIM_EINVAL, "out is NULL"};
    const auto t_start = std::chrono::steady_clock::now();
    std::lock_guard<std::mutex> lock(g_arena_mu);
    // cache key: the exact bytes of every input that shapes the prepared handle
    std::string key;
    auto put = [&](const void* p, size_t n) { key.append(static_cast<const char*>(p), n); };
    if (!c || (!c->gates && c->n_gates)) throw Error{TQSIM_EINVAL, "circuit is NULL"};
    validate_noise(nm);
    put(&c->n_qubits, sizeof(c->n_qubits));
    put(&c->n_gates, sizeof(c->n_gates));
    put(c->gates, sizeof(tqsim_gate) * c->n_gates);
    put(nm, sizeof(*nm));
    put(&n_shots, sizeof(n_shots));
    put(&n_levels, sizeof(n_levels));
    if (arities) put(arities, sizeof(uint32_t) * n_levels);
    else key.push_back('A');
    if (o) put(o, sizeof(*o));
    else key.push_back('D');
    tqsim_handle* h = nullptr;
    for (auto& e : g_hcache)
      if (e.key == key) {
        h = e.h;
        e.last_use = ++g_hcache_clock;
      }
    if (!h) {
      h = create_handle(c, nm, n_shots, arities, n_levels, o, true);
      if (g_hcache.size() >= HCACHE_MAX) {
        auto lru = std::min_element(g_hcache.begin(), g_hcache.end(),
                                    [](const CachedHandle& a, const CachedHandle& b) { return a.last_use < b.last_use; });
        tqsim_destroy(lru->h);
        g_hcache.erase(lru);
      }
      g_hcache.push_back(CachedHandle{key, h, ++g_hcache_clock});
    }
    cudaStream_t st = nullptr;
    try {
      h->debug = debug;
      const ShardRange sr = shard_levels(h->cplan, 0, 1);
      const Layout lay = layout(h, sr);
      const uint64_t ws = lay.total;
      const uint64_t nout = h->cplan.n_outcomes;
      const uint64_t out_off = align_up(ws);
      // per-leaf sampler debug outputs (u53, total, boundary flag), when asked for
      const bool want_u = debug && (debug->leaf_u || debug->leaf_total || debug->leaf_flagged);
      const uint64_t dbg_off = align_up(out_off + nout * 4);
      const uint64_t arena_bytes = want_u ? dbg_off + align_up(nout * 8) * 2 + nout : out_off + nout * 4;
      char* base = static_cast<char*>(arena_get(arena_bytes));
      if (!g_stream) ckc(cudaStreamCreateWithFlags(&g_stream, cudaStreamNonBlocking), "cudaStreamCreate");
      st = g_stream;
      if (want_u) {
        h->d_dbg_u = reinterpret_cast<double*>(base + dbg_off);
        h->d_dbg_total = reinterpret_cast<double*>(base + dbg_off + align_up(nout * 8));
        h->d_dbg_flag = reinterpret_cast<uint8_t*>(base + dbg_off + 2 * align_up(nout * 8));
      }
      // this call's per-gate tables (2q flags, pass index) from the host circuit
      upload_gate_tables(h, st);
      uint32_t* d_out = reinterpret_cast<uint32_t*>(base + out_off);
      ckc(cudaMemsetAsync(d_out, 0, nout * 4, st), "memset outcomes");
      execute(h, seed, 0, 1, st, base, ws, d_out);
      if (g_pinned_size < nout * 4) {   // page-locked landing buffer of the outcomes
        if (g_pinned) cudaFreeHost(g_pinned);
        g_pinned = nullptr;
        g_pinned_size = 0;
        ckc(cudaMallocHost(&g_pinned, nout * 4), "cudaMallocHost outcomes");
        g_pinned_size = nout * 4;
      }
      ckc(cudaMemcpyAsync(g_pinned, d_out, nout * 4, cudaMemcpyDeviceToHost, st), "D2H outcomes");
      ckc(cudaStreamSynchronize(st), "stream sync");
      const uint32_t* po = static_cast<const uint32_t*>(g_pinned);
      std::vector<uint32_t> outs(po, po + nout);
      if (want_u) {
        if (debug->leaf_u) ckc(cudaMemcpy(debug->leaf_u, h->d_dbg_u, nout * 8, cudaMemcpyDeviceToHost), "D2H u");
        if (debug->leaf_total)
          ckc(cudaMemcpy(debug->leaf_total, h->d_dbg_total, nout * 8, cudaMemcpyDeviceToHost), "D2H total");
        if (debug->leaf_flagged)
          ckc(cudaMemcpy(debug->leaf_flagged, h->d_dbg_flag, nout, cudaMemcpyDeviceToHost), "D2H flags");
      }
      h->d_dbg_u = h->d_dbg_total = nullptr;
      h->d_dbg_flag = nullptr;
      if (debug || h->opts.profile)   // work executed (dedup representatives): maps read back
        fill_computed(h, sr, lay, base);
      h->debug = nullptr;
      const double wall =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
      build_result(h, outs, wall, out);
    } catch (...) {
      h->debug = nullptr;
      h->d_dbg_u = h->d_dbg_total = nullptr;
      h->d_dbg_flag = nullptr;
      for (size_t i = 0; i < g_hcache.size(); ++i)   // a failed handle is not reused
        if (g_hcache[i].h == h) g_hcache.erase(g_hcache.begin() + i);
      tqsim_destroy(h);
      throw;
    }
  });
}

tqsim_status tqsim_run(const tqsim_circuit* c, const tqsim_noise_model* nm, uint64_t n_shots,
                       const uint32_t* tree_arities, uint32_t n_levels, uint64_t seed,
                       tqsim_result** out) {
  return tqsim_run_ex(c, nm, n_shots, tree_arities, n_levels, seed, nullptr, nullptr, out);
}

void tqsim_release_run_cache(void) {
  std::lock_guard<std::mutex> lock(g_arena_mu);
  for (auto& e : g_hcache) tqsim_destroy(e.h);
  g_hcache.clear();
  if (g_arena) cudaFree(g_arena);
  g_arena = nullptr;
  g_arena_size = 0;
  if (g_pinned) cudaFreeHost(g_pinned);
  g_pinned = nullptr;
  g_pinned_size = 0;
}

void tqsim_result_free(tqsim_result* r) {
  if (!r) return;
  std::free(r->bitstrings);
  std::free(r->counts);
  std::free(r->leaf_outcomes);
  std::free(r);
}

// B200 analogue of the paper's state-copy cost measurement (§3.3,
// fig:copy-overhead): the time of copying a batch of states
// device-to-device, in units of the engine's time per gate application on the same
// batch (a seeded probe slice of random U and CX gates, noise-free, run as level 1 of
// a [1, B] tree so its passes are the engine's ordinary fused passes).
tqsim_status tqsim_profile_copy_cost(uint32_t n_qubits, uint32_t n_probe_gates, uint64_t seed,
                                     double* copy_cost_gates, double* copy_ms, double* gate_ms) {
  void* a = nullptr;
  void* b = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  tqsim_handle* h = nullptr;
  auto cleanup = [&] {
    if (h) tqsim_destroy(h);
    if (a) cudaFree(a);
    if (b) cudaFree(b);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (st) cudaStreamDestroy(st);
  };
  const tqsim_status r = guarded([&] {
    if (!copy_cost_gates) throw Error{TQSIM_EINVAL, "copy_cost_gates is NULL"};
    if (n_qubits < 4 || n_qubits > 28 || n_probe_gates < 1 || n_probe_gates > 4096)
      throw Error{TQSIM_EINVAL, "profile needs 4 <= n_qubits <= 28 and 1..4096 probe gates"};
    require_device();
    const uint64_t S = 16ull << n_qubits;
    const uint64_t B = std::max<uint64_t>(1, (1ull << 26) >> n_qubits);
    ckc(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    ckc(cudaEventCreate(&e0), "event");
    ckc(cudaEventCreate(&e1), "event");
    ckc(cudaMalloc(&a, B * S), "cudaMalloc copy source");
    ckc(cudaMalloc(&b, B * S), "cudaMalloc copy target");
    ckc(cudaMemsetAsync(a, 0, B * S, st), "memset");
    for (int i = 0; i < 2; ++i) ckc(cudaMemcpyAsync(b, a, B * S, cudaMemcpyDeviceToDevice, st), "copy");
    ckc(cudaEventRecord(e0, st), "record");
    const int reps = 5;
    for (int i = 0; i < reps; ++i) ckc(cudaMemcpyAsync(b, a, B * S, cudaMemcpyDeviceToDevice, st), "copy");
    ckc(cudaEventRecord(e1, st), "record");
    ckc(cudaEventSynchronize(e1), "sync");
    float cms = 0.f;
    ckc(cudaEventElapsedTime(&cms, e0, e1), "elapsed");
    const double t_copy = cms / reps;
    cudaFree(b);
    b = nullptr;
    // probe slice: seeded random U(theta, phi, lambda) and CX gates; level 0 repeats it
    // on the single root instance, level 1 runs it on the B-state batch
    uint64_t x = seed * 0x9E3779B97F4A7C15ull + 1;
    auto rnd = [&] {
      x ^= x << 13;
      x ^= x >> 7;
      x ^= x << 17;
      return x;
    };
    std::vector<tqsim_gate> probe;
    for (uint32_t i = 0; i < 2 * n_probe_gates; ++i) {
      tqsim_gate g{};
      if (rnd() % 3 == 0) {
        g.kind = TQ_CX;
        g.q0 = (uint32_t)(rnd() % n_qubits);
        g.q1 = (g.q0 + 1 + (uint32_t)(rnd() % (n_qubits - 1))) % n_qubits;
      } else {
        g.kind = TQ_U;
        g.q0 = (uint32_t)(rnd() % n_qubits);
        g.theta = (double)(rnd() % 1000000) * 6.283185307179586e-6;
        g.phi = (double)(rnd() % 1000000) * 6.283185307179586e-6;
        g.lambda = (double)(rnd() % 1000000) * 6.283185307179586e-6;
      }
      probe.push_back(g);
    }
    const tqsim_circuit c{n_qubits, 0, probe.size(), probe.data()};
    const tqsim_noise_model nm{0.0, 0.0, 0.0, 0.0};
    tqsim_options o;
    tqsim_default_options(&o);
    o.profile = 1;
    const uint32_t ar[2] = {1, (uint32_t)B};
    h = create_handle(&c, &nm, B, ar, 2, &o, true);
    const Layout L = layout(h, shard_levels(h->cplan, 0, 1));
    cudaFree(a);
    a = nullptr;
    ckc(cudaMalloc(&a, L.total + h->cplan.n_outcomes * 4 + ALIGN), "cudaMalloc workspace");
    uint32_t* d_out = reinterpret_cast<uint32_t*>(static_cast<char*>(a) + align_up(L.total));
    double best = 0.0;
    for (int i = 0; i < 3; ++i) {
      execute(h, 1 + i, 0, 1, st, a, L.total, d_out);
      if (i == 0 || h->stats.pass_ms < best) best = h->stats.pass_ms;
    }
    const double t_gate = best / n_probe_gates;   // level 0 (one state) is ~1/B of it
    *copy_cost_gates = t_copy / t_gate;
    if (copy_ms) *copy_ms = t_copy;
    if (gate_ms) *gate_ms = t_gate;
  });
  cleanup();
  return r;
}

tqsim_status tqsim_debug_philox(const uint32_t* in, uint64_t n, uint32_t* out) {
  return guarded([&] {
    if (!in || !out) throw Error{TQSIM_EINVAL, "NULL argument"};
    require_device();
    uint32_t *di = nullptr, *dout = nullptr;
    ckc(cudaMalloc(&di, std::max<uint64_t>(1, n) * 24), "cudaMalloc");
    ckc(cudaMalloc(&dout, std::max<uint64_t>(1, n) * 16), "cudaMalloc");
    cudaMemcpy(di, in, n * 24, cudaMemcpyHostToDevice);
    int e = launch_philox_debug(di, n, dout);
    if (e == 0) e = (int)cudaMemcpy(out, dout, n * 16, cudaMemcpyDeviceToHost);
    cudaFree(di);
    cudaFree(dout);
    ck(e, "philox debug");
  });
}

tqsim_status tqsim_debug_noise_table(tqsim_handle* h, uint64_t seed, uint32_t level,
                                     uint64_t inst_begin, uint64_t count, uint8_t* out) {
  return guarded([&] {
    if (!h || !out) throw Error{TQSIM_EINVAL, "NULL argument"};
    if (level >= h->plan.arities.size()) throw Error{TQSIM_EINVAL, "level out of range"};
    const uint32_t b0 = (uint32_t)h->plan.bounds[level];
    const uint32_t len = (uint32_t)(h->plan.bounds[level + 1] - b0);
    uint8_t* d = nullptr;
    const uint64_t bytes = std::max<uint64_t>(1, count * len);
    ckc(cudaMalloc(&d, bytes), "cudaMalloc");
    int e = launch_noise_table(h->d_two + b0, b0, len, inst_begin, count, seed, h->noise.p1,
                               h->noise.p2, d);
    if (e == 0) e = (int)cudaMemcpy(out, d, count * len, cudaMemcpyDeviceToHost);
    cudaFree(d);
    ck(e, "noise table");
  });
}

}  // extern "C"
