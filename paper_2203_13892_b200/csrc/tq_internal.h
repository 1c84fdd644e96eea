// Internal declarations of the TQSim B200 runtime (not part of the C ABI).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/tqsim.h"

namespace tq {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
struct Error {
  tqsim_status status;
  std::string msg;
};

// ---------------------------------------------------------------- IR
enum OpType : uint8_t { OP_GEN = 0, OP_DIAG = 1, OP_CX = 2, OP_CZ = 3 };

struct LGate {              // one lowered gate = one noise location (R1)
  uint32_t kind;            // tqsim_gate_kind of the primitive (1q kinds, CX, CZ)
  uint32_t q0, q1;          // q1 = q0 for 1q
  bool two;
  uint8_t op;               // OpType
  double m[8];              // 2x2 complex, row major (re,im) pairs: m00 m01 m10 m11
};

// Validates and lowers (R4).  Throws Error{TQSIM_EINVAL}.
std::vector<LGate> lower(const tqsim_circuit* c);

// ---------------------------------------------------------------- planner
struct Options {
  double copy_cost_gates = 10.0, z = 1.96, eps = 0.05;
  uint64_t mem_budget = 180000000000ull;
  uint32_t topup = 0, tile_qubits = 0, batch_log2_amps = 0, profile = 0, no_dedup = 0, trail_low = 0, small_tree = 0;
};
Options options_from(const tqsim_options* o);

struct Plan {
  std::vector<uint32_t> arities;
  std::vector<uint64_t> bounds;   // size L+1
  double p_hat = 0.0;
};

Plan make_plan(const std::vector<LGate>& gates, uint32_t n_qubits, const tqsim_noise_model* nm,
               uint64_t n_shots, const uint32_t* arities, uint32_t n_levels, const Options& o);
void fill_plan(const Plan& p, uint32_t n_qubits, uint64_t n_gates, uint64_t hbm_passes,
               tqsim_plan* out);
std::vector<uint64_t> instances(const Plan& p);   // Eq.2, per level

// ---------------------------------------------------------------- pass plan
constexpr int RBITS = 4;        // amplitudes per thread = 2^RBITS (register-resident qubits)
constexpr int MAX_K = 13;       // max tile qubits per HBM pass (2^13 * 16 B = 128 KiB smem)
constexpr int LOW_Q = 3;        // qubits 0..4 are in every tile (512 B contiguous segments)
constexpr int MAX_PASS_OPS = 192; // gates per pass kernel (code size / shared codes bound)
constexpr int RUN_Q = 3;          // leaf |a|^2 run sums cover 2^RUN_Q consecutive amplitudes

// Role of a gate in its pass (first pass of a level only for roles 1..3, passplan.cpp)
enum OpRole : uint8_t {
  ROLE_REG = 0,       // applied to amplitudes held in registers
  ROLE_DIAG = 1,      // part of a diagonal unit: phases from known index bits, no register
  ROLE_SWAP = 2,      // part of an absorbed SWAP: a relabeling of address bits at the store
  ROLE_STOREMAP = 3,  // an absorbed CX: a GF(2)-linear map of the store address
};

struct OpDesc {
  uint8_t type;                 // OpType
  uint8_t ra, rb;               // register bit(s) 0..3 (rb = target for CX)
  uint8_t two;                  // 2q noise location
  uint32_t gate;                // lowered gate index g (noise key + matrix)
  uint8_t role;                 // OpRole
};

struct PhaseDesc {              // 32 bytes, device-readable
  uint8_t rpos[RBITS];          // tile-local positions held in registers
  uint8_t tpos[MAX_K - RBITS];  // thread-index bit m -> tile-local position
  uint8_t pad[32 - RBITS - (MAX_K - RBITS) - 8];
  uint32_t op_begin, op_end;    // global op indices
};
static_assert(sizeof(PhaseDesc) == 32, "PhaseDesc layout");

struct PassDesc {
  int K = 0;                    // tile qubits
  uint8_t tile_q[MAX_K];        // tile-local position -> global qubit
  int n_out = 0;
  uint8_t out_q[32];            // non-tile qubits (ascending)
  uint32_t phase_begin = 0, phase_end = 0;
  uint32_t op_begin = 0, op_end = 0;
  uint64_t tile_mask = 0;
  bool leaf_sums = false;       // last pass of the leaf level: also writes |a|^2 run sums
  uint32_t slice_begin = 0;     // first lowered gate of the level's slice
  uint32_t pass_index = 0;      // index of this pass within its level
  uint32_t slice_len = 0;       // gates of the level's slice
  bool mask_any = false;        // take the careful path when any gate of the slice erred
                                // (trail passes: their gates' pass bits are not in the row mask)
};

// Fast projection of the conditional leaf sampling (kernels.cu trail_project_kernel): pass A
// = diagonal units (both qubits among the top bits, or both below) followed by 1q gates on
// the top bits, so psi(x) = D_x(x) sum_y c[y] phi(y, x) with c[y] = prod_j U_j[sel_j][y_j]
// * D_top(y) per leaf (a leaf with a Pauli inside a diagonal unit takes the generated kernel).
constexpr int PROJ_MAX_G = 48;
constexpr int PROJ_MAX_U = 24;
constexpr int PROJ_MAX_DG = 72;
struct ProjSpec {
  uint32_t m, n2, ng, nug, nux, ndg;
  uint32_t gbit[PROJ_MAX_G];        // top bit j (qubit n2 + j) of 1q gate i, slice order
  uint32_t goff[PROJ_MAX_G];        // its slice offset (noise code)
  double gmat[PROJ_MAX_G][8];       // its 2x2 (re, im row major)
  uint32_t ua[PROJ_MAX_U], ub[PROJ_MAX_U];   // units: [0, nug) top-bit indices, [nug, nug+nux) qubits < n2
  double uT[PROJ_MAX_U][8];         // phase by bit_a + 2 bit_b (complex)
  uint32_t dgoff[PROJ_MAX_DG];      // slice offsets of every diagonal-unit gate
  // each unit's gates (1, or 3 for CX.D.CX), for its effective operator under a leaf's Paulis:
  // kind 0 = 1q diagonal on ua, 1 = 1q diagonal on ub, 2 = CX(ua -> ub), 3 = CZ(ua, ub)
  uint8_t ugn[PROJ_MAX_U];
  uint8_t ugk[PROJ_MAX_U][3];
  uint32_t ugoff[PROJ_MAX_U][3];    // slice offsets (noise codes)
  double ugd[PROJ_MAX_U][3][4];     // kind 0/1: diag(d0, d1) as (re, im, re, im)
};

// Conditional leaf sampling through the trailing layer (passplan.cpp plan_trail)
struct TrailPlan {
  bool on = false;
  int m = 0, n2 = 0;            // G1 = the top m qubits; stage-2 width n2 = n - m
  PassDesc a;                   // pass A over {0..2} ∪ G1: run sums (variant 1) / projection (variant 3)
  std::vector<PassDesc> b;      // stage-2 passes on the projected n2-qubit states (last: run sums)
  bool fast = false;            // pass A fits ProjSpec: the hand-written projection
  ProjSpec proj{};
};
struct TrailProjLaunch {
  const void* src;              // parent level batch
  const uint32_t* prep;         // parent dedup map (or null)
  uint64_t child_first, parent_first;
  uint32_t arity, batch, n;
  const uint8_t* rows;
  uint32_t row_bytes;
  const uint32_t* hsel;         // per leaf: the chosen top bits
  void* psi;                    // per leaf: the projected 2^n2 state
  uint32_t* glist;              // leaves for the generated projection (a Pauli inside a unit)
  uint32_t* gcount;
};
int launch_trail_project(const ProjSpec& spec, const TrailProjLaunch& L, void* stream);

struct PassPlan {
  int n_sim = 0;                         // simulated width (>= RBITS)
  std::vector<std::vector<PassDesc>> levels;   // per level, its passes
  std::vector<PhaseDesc> phases;
  std::vector<OpDesc> ops;
  TrailPlan trail;                       // leaf level: conditional sampling (default path)
  uint64_t passes_total(const std::vector<uint64_t>& inst) const;
};

PassPlan make_pass_plan(const std::vector<LGate>& gates, uint32_t n_qubits, const Plan& plan,
                        const Options& o);

// ---------------------------------------------------------------- kernels (kernels.cu)
struct PassLaunch {
  const void* src;              // double2*; root synthesized when src_mode == 0
  void* dst;
  uint32_t src_mode;            // 0 root |0..0>, 1 fan-out from parent batch, 2 in place
  uint64_t child_first;         // global instance id of batch slot 0
  uint64_t parent_first;        // global instance id of parent slot 0 (mode 1)
  uint32_t arity;               // A_d (mode 1)
  uint32_t batch;
  uint64_t seed;
  double p1, p2;
  void* runsum;                 // leaf |a|^2 run sums (leaf_sums passes only)
  const void* rows;             // noise rows of the batch (launch_noise_rows), row_bytes each
  uint32_t row_bytes;
  uint32_t variant;             // leaf-sum passes: 0 store, 1 run sums only, 2 recompute
  const uint32_t* tiles;        // variant 2: tile index per leaf
  const uint32_t* runsel;       // variant 2: selected run per leaf
  void* scratch;                // variant 2: 8 amplitudes per leaf (double2)
  uint32_t* xlout;              // variant 1: store-address XOR per leaf
  const uint32_t* rep;          // dedup map of the batch (null: every instance computed)
  const uint32_t* prep;         // dedup map of the parent batch (fan-out reads prep[parent])
  const uint32_t* wlist;        // variant 3 with a work list: the leaves (slots) to project
  const uint32_t* wcount;       //   and their count (device); grid = persistent CTAs
  uint32_t clean;               // variant 1: the work list holds only items without an error in
                                //   the pass (the fast-code kernel, JitPass::kernel_clean)
};

// Noise rows of one level batch (row a3): per instance a row of row_bytes bytes,
// [0..4) = u32 bitmask of the level's passes with >= 1 drawn error (bit min(p, 31)),
// [4 + t] = Pauli code of slice gate t (0 = none).  One warp per instance.
inline uint32_t noise_row_bytes(uint32_t slice_len) { return (4u + slice_len + 15u) / 16u * 16u; }
int launch_noise_rows(const uint8_t* d_two, const uint8_t* d_pass_of, uint32_t slice_begin,
                      uint32_t slice_len, uint64_t inst_first, uint32_t count, const uint64_t* d_seed,
                      double p1, double p2, uint32_t row_bytes, uint8_t* d_rows, void* stream);
int launch_set_seed(uint64_t* d_seed, uint64_t seed, void* stream);
// the batch's computed instances (rep[s] == s) in slot order -> list, *count; xlout (leaf level,
// may be null) = 0 for the others
int launch_compact_reps(const uint8_t* d_err_sel, uint32_t slice_len,   // d_err_sel: as NoiseLevel::err_sel
                        const uint32_t* d_rep, uint32_t cnt, uint32_t* d_list, uint32_t* d_count, uint32_t* d_xlout,
                        const uint8_t* d_rows, uint32_t row_bytes, uint32_t emask, uint32_t* d_list2, uint32_t* d_count2,
                        void* stream);
// All noise rows of a shard in one launch (one warp per instance of every level).
struct NoiseLevel {
  uint64_t inst_first;   // global instance id of the shard's first instance at this level
  uint64_t count;        // the shard's instances at this level
  uint64_t rows_off;     // byte offset of the level's rows in the rows region
  uint32_t slice_begin, slice_len, row_bytes, pad;
  // dedup map (launch_dedup_map): entry offset of the level in the rep / pos arrays,
  // the level's batch cap and arity
  uint64_t map_off;
  uint64_t cap;
  uint32_t arity, pad2;
  // which gates' errors make an instance "not error-free" for the dedup map: null = any gate
  // of the slice (the row's pass bitmask); else a byte per slice gate (the conditional-sampling
  // leaf level: only pass A's gates -- the marginals are of pass A's state)
  const uint8_t* err_sel;
};
constexpr int NOISE_MAX_LEVELS = 64;
struct NoiseLevels {
  NoiseLevel lv[NOISE_MAX_LEVELS];
  uint32_t n_levels;
};
// Per instance of every level of the shard: rep = batch-relative index of the instance
// whose computed state it shares (itself unless it drew no error and an earlier instance of
// its batch with the same effective parent did not either), pos = its batch-relative index.
int launch_dedup_map(const uint8_t* d_rows, const NoiseLevels& L, uint32_t* d_rep, uint32_t* d_pos,
                     void* stream);
int launch_dedup_map_level(const uint8_t* d_rows, const NoiseLevels& L, uint32_t d, uint32_t* d_rep,
                           uint32_t* d_pos, void* stream);
int launch_noise_rows_all(const uint8_t* d_two, const uint8_t* d_pass_of, const NoiseLevels& L,
                          uint64_t total_instances, const uint64_t* d_seed, double p1, double p2,
                          uint8_t* d_rows, void* stream);

struct LeafSelect;
int launch_chunk_sums(const double* runsums, uint32_t batch, int n_sim, int chunk_log2,
                      double* sums, void* stream, const LeafSelect* sel = nullptr, uint64_t leaf_first = 0);
// leaf sampling without a stored leaf state (select -> recompute one tile -> finish)
struct LeafSelect {
  uint32_t* runsel;
  double* t3;
  uint32_t* tile;
  const uint32_t* xl;
  uint32_t n_out;
  uint32_t out_row[32];      // out-of-tile qubit i = parity(out_row[i] & stored address)
  // dedup map of the leaf batch: read the representative's sums (null: none)
  const uint32_t* rep = nullptr;
  // debug outputs by global leaf id (tqsim_debug leaf_u / leaf_total / leaf_flagged), or null
  double* dbg_u = nullptr;
  double* dbg_total = nullptr;
  uint8_t* dbg_flag = nullptr;
  // conditional leaf sampling: stage-1 outputs (chunk = top bits, residual target) /
  // stage-2 inputs (target override, top bits ORed into the outcome at hi_shift)
  uint32_t* hsel = nullptr;
  double* htarget = nullptr;
  const double* tgt = nullptr;
  const uint32_t* hi = nullptr;
  uint32_t hi_shift = 0;
};
int launch_sample_finish(const void* scratch, const uint32_t* runsel, const double* t3, uint32_t batch,
                         int n_user, uint64_t leaf_first, const uint64_t* d_seed, double p01, double p10,
                         uint32_t* d_out, void* stream, uint8_t* d_flag = nullptr,
                         const uint32_t* d_hi = nullptr, uint32_t hi_shift = 0);
int launch_sample(const void* states, const double* runsums, const double* sums, uint32_t batch,
                  int n_sim, int n_user, int chunk_log2, uint64_t leaf_first, const uint64_t* d_seed,
                  double p01, double p10, uint32_t* d_out, void* stream, const LeafSelect* sel = nullptr);
// n_sim - RUN_Q <= SMALL_SAMPLE_RUNS_LOG2: one kernel reads all run sums of a leaf
constexpr int SMALL_SAMPLE_RUNS_LOG2 = 14;
int launch_sample_small(const void* states, const double* runsums, uint32_t batch, int n_sim,
                        int n_user, uint64_t leaf_first, const uint64_t* d_seed, double p01, double p10,
                        uint32_t* d_out, void* stream, const LeafSelect* sel = nullptr);
int launch_philox_debug(const uint32_t* d_in, uint64_t n, uint32_t* d_out);
int launch_noise_table(const uint8_t* d_two, uint32_t slice_begin, uint32_t slice_len,
                       uint64_t inst_begin, uint64_t count, uint64_t seed, double p1, double p2,
                       uint8_t* d_out);
const char* cuda_error_string(int code);

// ---------------------------------------------------------------- Kraus engine (kraus.cu)
struct KGate {                  // a lowered gate for the Kraus engine (device table)
  uint32_t two, op, q0, q1;     // op: OpType (OP_CX / OP_CZ for 2q)
  double m[8];                  // 1q: 2x2 complex row major (re, im)
};
struct KrausArgs {
  const KGate* gates;
  const void* src;              // parent level batch (mode 1)
  void* dst;                    // this level batch (non-leaf)
  const uint8_t* src_flag;      // parent's path flag (R36)
  uint8_t* dst_flag;
  uint64_t child_first, parent_first;
  uint32_t arity, g0, g1, n, n_user, mode, leaf, ch_mask;   // ch_mask: 1 TR, 2 AD, 4 PD
  uint32_t store_leaf;          // leaf level: also store the state (state dumps)
  const uint64_t* seedp;
  double p1, p2, p01, p10;
  double trg[2], trl[2];        // TR amplitude / phase damping parameters per gate class (1q, 2q)
  double ad, pd;
  uint32_t* out;
  double* dbg_u;
  double* dbg_total;
  uint8_t* dbg_flag;
};
int launch_kraus_slice(const KrausArgs& a, uint32_t batch, void* stream);

// Small-state tree (small.cu): one warp per leaf recomputes its root-to-leaf
// path with the inherited keys, the state in shared memory (n_sim <= TQSIM_SMALL_MAX_QUBITS).
constexpr int SMALL_TREE_WARPS = 4;   // warps (leaves) per CTA
struct SmallTreeArgs {
  const KGate* gates;
  uint64_t leaf_first, leaf_count;      // the shard's leaf range
  uint32_t levels, n, n_user, reserved;
  uint32_t arity[TQSIM_MAX_LEVELS];
  uint32_t bounds[TQSIM_MAX_LEVELS + 1];
  const uint64_t* seedp;
  double p1, p2, p01, p10;
  uint32_t* out;
  double* dbg_u;
  double* dbg_total;
  uint8_t* dbg_flag;
};
int launch_small_tree(const SmallTreeArgs& a, void* stream);
inline bool kraus_enabled(const tqsim_noise_model& nm) {
  return nm.amp_damping > 0.0 || nm.phase_damping > 0.0 || nm.t1 > 0.0;
}

// ---------------------------------------------------------------- JIT pass kernels (jit.cpp)
// TMA staging of a pass's tiles (TQSIM_TMA, jit.cpp): the tile {0,1,2} ∪ H as one 5-D tensor-map
// box over the source batch.  Dims in order (innermost first): qubits 0..2 as 16 doubles, then
// runs of qubits alternately in the tile (box = 2^len) or out of it (box 1, coordinate = the
// tile index bits tbit..tbit+len-1), padded, and the state index (coordinate = the source slot).
struct TmaGeom {
  int ndims = 0;
  int kind[5] = {};     // 0 out-of-tile run, 1 in-tile run (incl. dim 0), 2 state index
  int qstart[5] = {};   // first qubit of the run
  int len[5] = {};      // qubits in the run
  int tbit[5] = {};     // out-of-tile runs: first bit in the tile index t
};
bool tma_geom(const PassDesc& pd, int n, TmaGeom* g);

struct JitPass {
  void* kernel = nullptr;   // cudaKernel_t
  void* kernel_nostore = nullptr;     // leaf-sum passes: run sums only (variant 1)
  void* kernel_recompute = nullptr;   // leaf-sum passes: one tile per leaf, 8 amps (variant 2)
  void* kernel_clean = nullptr;       // variant 1 for work-list items whose pass drew no error
  std::vector<uint32_t> out_row;   // per out-of-tile qubit: stored-address bits whose parity is its bit
  int threads = 0;
  size_t smem = 0;
  std::vector<double> coefs;      // by-value coefficient parameter (TQSIM_JIT_COEF=0 mode)
  double fp64_per_amp = 0.0;      // FP64 operations per amplitude of the fast path (cost model)
  bool tma_v[2] = {false, false};   // kernel (v0) / kernel_nostore (v1) take a tensor map (persistent CTAs)
  size_t smem_tma = 0;              // their dynamic shared memory (two tile buffers + mbarriers)
  TmaGeom geom;
  int n_sim = 0;                  // state width the kernel was generated for
  // trail pass A: the projection kernel (variant 3) and its launch parameters
  void* kernel_project = nullptr;
  int threads_project = 0;
  size_t smem_project = 0;
  std::vector<double> coefs_project;
};
struct JitTrail {                  // kernels of PassPlan::trail
  JitPass a;                       // kernel_nostore = run sums (v1), kernel_project = projection (v3)
  std::vector<JitPass> b;          // stage-2 passes (the last: kernel_nostore v1, kernel_recompute v2)
};
std::vector<std::vector<JitPass>> jit_build(const PassPlan& pp, const std::vector<LGate>& gates,
                                            double* compile_seconds, JitTrail* trail = nullptr);
void jit_compile_only(const PassPlan& pp, const std::vector<LGate>& gates, uint64_t* n_kernels,
                      uint64_t* cubin_bytes);
std::string jit_source(const PassPlan& pp, const std::vector<LGate>& gates, size_t level,
                       size_t pass, const std::string& name);
uint64_t jit_compile_count();
int launch_jit_pass(const JitPass& jp, const PassDesc& pd, const PassLaunch& L, void* stream);

}  // namespace tq
