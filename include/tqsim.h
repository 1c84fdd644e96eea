/*
 * tqsim.h -- C ABI of the B200-native TQSim hot path.
 *
 * TQSim (arXiv 2203.13892): multi-shot noisy statevector simulation that
 * reuses intermediate states through a tree.  Citations: "P:n" = line n of the
 * paper text with its section / equation; "S:n" = SPEC.md line n;
 * "R<k>" = reading k of DESIGN.md (the paper is silent / ambiguous there).
 *
 * Problem statement: given a circuit, a noise model and N
 * shots, return a histogram of >= N noisy measurement outcomes.
 *
 * Conventions shared by every entry point
 *   - Basis index x = sum_q bit_q * 2^q (little endian, R6).  Outcomes
 *     and bitstrings are such integers.
 *   - All pointers are plain host pointers unless the name starts with d_
 *     (device pointer, CUDA global memory of the current device) or the
 *     argument is a `void* stream` (a cudaStream_t, NULL = legacy default).
 *   - Ownership: the caller owns every input and may free it after the call
 *     returns (the library copies what it keeps).  Objects returned through
 *     `**out` are owned by the library and released with the matching
 *     *_free / tqsim_destroy call.  Device buffers passed in stay caller-owned.
 *   - Errors: every function returns a tqsim_status; on failure nothing is
 *     written to `*out` and tqsim_last_error() returns a thread-local message.
 *     No C++ exception ever crosses this boundary.
 *   - Functions marked [host] never touch the GPU and work without one.
 *   - Functions marked [gpu] need a CUDA device of compute capability 10.0
 *     (B200, sm_100a); without it they return TQSIM_ECUDA.  There is no CPU
 *     fallback.
 */
#ifndef TQSIM_H
#define TQSIM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TQSIM_MAX_LEVELS 64
#define TQSIM_MAX_QUBITS 30

typedef enum {
  TQSIM_OK = 0,
  TQSIM_EINVAL = 2,     /* bad circuit / noise / arity / argument (SPEC exit code 2) */
  TQSIM_ECAPACITY = 3,  /* memory budget or workspace too small (SPEC exit code 3)  */
  TQSIM_ECUDA = 4,      /* CUDA error or no sm_100 device                                    */
  TQSIM_ENCCL = 5,      /* reserved: collective failure (the allreduce runs in the caller)  */
  TQSIM_EINTERNAL = 6
} tqsim_status;

/* Gate kinds (S:33 set + P(U1)).  Matrices (R5, standard OpenQASM 2 forms):
 *   H=[[1,1],[1,-1]]/sqrt2, X, Y=[[0,-i],[i,0]], Z, S=diag(1,i), SDG, T=diag(1,e^{i pi/4}), TDG,
 *   RX(t)=[[c,-is],[-is,c]], RY(t)=[[c,-s],[s,c]], RZ(t)=diag(e^{-it/2},e^{it/2}),
 *   P(t)=diag(1,e^{it}), U(t,p,l)=[[c,-e^{il}s],[e^{ip}s,e^{i(p+l)}c]],  c=cos t/2, s=sin t/2.
 *   Single-angle gates (RX, RY, RZ, P, CP) take their angle in `theta`.
 *   CX(q0=control, q1=target); CZ(q0,q1); SWAP(q0,q1); CP(theta; q0=control, q1=target).
 * Lowering (R4): CP -> P(t/2)q0, CX, P(-t/2)q1, CX, P(t/2)q1;  SWAP -> CX(a,b) CX(b,a) CX(a,b).
 * Every LOWERED gate is one noise location (R1); gate index g counts lowered gates. */
typedef enum {
  TQ_X = 0, TQ_Y, TQ_Z, TQ_H, TQ_S, TQ_SDG, TQ_T, TQ_TDG,
  TQ_RX, TQ_RY, TQ_RZ, TQ_P, TQ_U, TQ_CX, TQ_CZ, TQ_SWAP, TQ_CP
} tqsim_gate_kind;

typedef struct {
  uint32_t kind;      /* tqsim_gate_kind */
  uint32_t q0, q1;    /* q1 used by 2q kinds only; must differ from q0 */
  uint32_t reserved;  /* 0 */
  double theta, phi, lambda;
} tqsim_gate;         /* 40 bytes */

typedef struct {
  uint32_t n_qubits;  /* 1 .. TQSIM_MAX_QUBITS */
  uint32_t reserved;
  uint64_t n_gates;   /* >= 1 */
  const tqsim_gate* gates;
} tqsim_circuit;

/* Depolarizing noise (R1/R2): after every lowered 1q gate, with
 * probability p1 one of X,Y,Z uniformly; after every 2q gate, with probability
 * p2 one of the 15 non-II Pauli pairs uniformly.  Readout error (R11):
 * each measured bit flips 0->1 with readout_p01 and 1->0 with readout_p10.
 * All in [0, 1].
 * Non-Pauli channels (§4.3.2, Table 2; readings R31-R37): after every lowered
 * gate and its depolarizing Pauli, on each qubit the gate acts on, thermal relaxation
 * (t1 > 0: amplitude damping with 1 - exp(-t/t1) then phase damping with
 * 1 - exp(-2t/t2 + t/t1), t = gate_time_1q / gate_time_2q, requires t2 <= 2 t1),
 * amplitude damping (amp_damping = gamma) and phase damping (phase_damping = lambda),
 * each unravelled as a keyed quantum trajectory (R34-R35).  Any of them enabled selects
 * the Kraus engine: the state of every trajectory resident in shared memory -- one CTA's
 * for n_qubits <= 13, a thread-block cluster of 2^(n-13) CTAs (distributed shared memory)
 * for 14..16; n_qubits <= 16 (TQSIM_EINVAL otherwise).  0 = off. */
typedef struct {
  double p1, p2, readout_p01, readout_p10;
  double amp_damping, phase_damping;
  double t1, t2, gate_time_1q, gate_time_2q;   /* seconds */
} tqsim_noise_model;

#define TQSIM_KRAUS_MAX_QUBITS 16

/* Small-state tree (SURVEY §8(a) kernel notes): a circuit of at most this
 * many qubits (Pauli noise only) may run the whole tree as ONE kernel -- one warp per leaf,
 * the state in shared memory, the root-to-leaf path recomputed with the inherited keys
 * (identical noise draws and outcomes to the tree; §3, R7). */
#define TQSIM_SMALL_MAX_QUBITS 10

typedef struct {
  double copy_cost_gates;     /* first-slice length m = round(.) (R14); default 10;
                                 -1 = this engine's fused fan-out cost: half the gates one HBM pass
                                 holds, from the pass planner on the whole circuit */
  double z;                   /* Eq.4 z-score (R12); default 1.96 */
  double eps;                 /* Eq.4 margin of error; default 0.05 */
  uint64_t mem_budget_bytes;  /* HBM budget for states (P:310 memory limit, R25); default 180e9 */
  uint32_t topup;             /* 0 = A_0 <- max(A_0, ceil(N/A_r^k)) (R18, default); 1 = round robin */
  uint32_t tile_qubits;       /* HBM-pass tile width K (4..13); 0 = auto (12) */
  uint32_t batch_log2_amps;   /* target amplitudes per level batch = 2^v; 0 = auto (26) */
  uint32_t profile;           /* 1 = time every kernel launch with CUDA events (tqsim_stats) */
  uint32_t no_dedup;          /* 0 (default) = an error-free instance whose effective parent
                                 state equals an earlier instance's of its batch shares that
                                 instance's computed state (bit-identical);
                                 1 = every node instance of the tree is computed */
  uint32_t trail_low;         /* conditional leaf sampling: the marginal pass's tile =
                                 qubits 0..trail_low-1 + the top K - trail_low qubits (3..K-1);
                                 0 = auto (4 when K >= 10, else 3) */
  uint32_t small_tree;        /* small-state tree kernel (n_qubits <= TQSIM_SMALL_MAX_QUBITS, Pauli
                                 noise, no state dumps): 0 = auto (when the per-leaf recompute is
                                 cheap: n_outcomes * lowered gates * 2^max(n,5) <= 2^24), 1 = on
                                 whenever eligible, 2 = off (the general tree engine) */
} tqsim_options;

/* The tree plan (§3.1): level d executes lowered gates
 * [boundaries[d], boundaries[d+1]) (subcircuit d) and has
 * instances_d = prod_{i<=d} arities[i] nodes (Eq.2).  n_outcomes = prod arities >= n_shots. */
typedef struct {
  uint32_t n_levels;
  uint32_t n_qubits;
  uint32_t arities[TQSIM_MAX_LEVELS];
  uint64_t boundaries[TQSIM_MAX_LEVELS + 1];
  double first_error_rate;          /* Eq.3 p_hat (0 for fixed / flat plans) */
  double predicted_speedup_nodes;   /* node ratio vs (N,1,..,1) (Table 3) */
  double predicted_speedup_gates;   /* flat gate-apps / tree gate-apps */
  uint64_t n_lowered_gates;
  uint64_t n_outcomes;
  uint64_t node_executions;         /* sum_d instances_d */
  uint64_t gate_amp_updates;        /* sum_d instances_d * |slice_d| * 2^n */
  uint64_t flat_gate_amp_updates;   /* n_outcomes * n_lowered_gates * 2^n */
  uint64_t hbm_passes;              /* sum_d instances_d * passes(slice d) */
  uint32_t tile_qubits;             /* K: amplitudes per gate-pass tile = 2^K (auto or options) */
  uint32_t trail_top_bits;          /* conditional leaf sampling: the leaf index's
                                       top bits selected first from marginals (0 = off) */
  uint32_t trail_fast;              /* 1: its projection is the streaming kernel (diagonal units
                                       + top-qubit 1q gates), 0: the generated pass kernel */
  uint32_t small_tree;              /* 1: the tree runs as the small-state kernel (options.small_tree) */
} tqsim_plan;

/* Execution statistics of the last tqsim_execute on a handle. */
typedef struct {
  uint64_t kernel_launches;         /* every kernel this library launched */
  uint64_t pass_launches;           /* gate-pass kernels (the hot loop) */
  uint64_t measure_launches;
  uint64_t node_executions;
  uint64_t gate_amp_updates;
  uint64_t pass_bytes;              /* algorithmic HBM bytes of gate passes: states*2^n*32 (16 if root-synthesized read) */
  uint64_t measure_bytes;           /* algorithmic HBM bytes of leaf measurement */
  double pass_ms;                   /* sum of gate-pass launch durations (profile=1 only) */
  double measure_ms;                /* sum of measurement launch durations (profile=1 only) */
  uint64_t leaves;                  /* leaves sampled by this shard */
  uint64_t noise_launches;          /* noise-row kernels (one per level batch) */
  double noise_ms;                  /* sum of noise-row launch durations (profile=1 only) */
  /* Work actually executed (error-free duplicates skipped, options.no_dedup = 0).  Filled by
   * tqsim_profile_tree, and by tqsim_run_ex when it is given a tqsim_debug or options.profile = 1
   * (the dedup maps are read back: a synchronous D2H + host walk); tqsim_run (the hot call) and
   * tqsim_execute (asynchronous) leave them 0. */
  uint64_t computed_node_executions;
  uint64_t computed_gate_amp_updates;
  uint64_t computed_pass_bytes;     /* algorithmic bytes of the computed instances' passes */
} tqsim_stats;

typedef struct {
  tqsim_plan plan;
  uint64_t n_distinct;
  uint64_t* bitstrings;             /* ascending, length n_distinct */
  uint64_t* counts;                 /* sum = plan.n_outcomes */
  uint32_t* leaf_outcomes;          /* length plan.n_outcomes, leaf order */
  double wall_s;
  tqsim_stats stats;
} tqsim_result;

/* Optional debug outputs for parity tests (§2.3 sampling, R9).
 * State dumps: the state of node (level, instance) after its subcircuit (after the last
 * gate and its Pauli, before measurement) is copied to dump_host + i * 2 * 2^n doubles
 * (interleaved re, im).  Requesting dumps switches the run to the stored-state path
 * (every instance computed, leaf states stored).
 * Per-leaf sampler outputs (host arrays of plan.n_outcomes entries, either may be NULL;
 * they do NOT change the execution path -- dedup maps and the no-store leaf sampler stay
 * on): leaf_u[l] = the u53 uniform of leaf l (R9), leaf_flagged[l] = 1 iff u*total lies
 * within 1e-9 of C(x-1) or C(x) for the sampled x (the draw a rounding difference could
 * move), leaf_total[l] = sum |a|^2 of the leaf state as the sampler summed it. */
typedef struct {
  uint32_t n_dumps;
  uint32_t reserved;
  const uint32_t* dump_levels;
  const uint64_t* dump_instances;
  double* dump_host;
  double* leaf_u;
  uint8_t* leaf_flagged;
  double* leaf_total;
} tqsim_debug;

/* Operation record of the pass plan (for host-side invariant tests). */
typedef struct {
  uint32_t level, pass, phase, gate;   /* gate = lowered gate index g */
  uint64_t tile_qubit_mask;            /* global qubits staged by the pass's tiles */
  uint64_t reg_qubit_mask;             /* global qubits held in registers in the phase */
  uint32_t role;                       /* 0 register op; first pass of a level only:
                                          1 part of a diagonal unit (no register),
                                          2 part of an absorbed SWAP (store relabeling),
                                          3 absorbed CX (GF(2)-linear store-address map) */
  uint32_t reserved;
} tqsim_op_record;

/* Timing of one gate-pass kernel (tqsim_profile_passes). */
typedef struct {
  uint32_t level, pass;
  uint32_t states_per_launch;        /* batch the kernel was timed on (a full level batch) */
  uint32_t reserved;
  double launches_per_tree;          /* this shard's launches of the kernel, in full-batch units */
  double ms_per_launch;              /* CUDA-event average over `reps` back-to-back launches */
  double alg_bytes_per_launch;       /* algorithmic HBM bytes of one launch */
} tqsim_pass_timing;

typedef struct tqsim_handle tqsim_handle;

/* [host] */
void tqsim_default_options(tqsim_options* opts);
const char* tqsim_last_error(void);
const char* tqsim_version(void);

/* [host] Lower a circuit (R4).  Writes up to `cap` gates; *n_out = lowered count. */
/* [host] Parse an OpenQASM 2.0 program (SPEC S:52-60, S:95 subset:
 * qreg/creg (several qregs concatenated in declaration order), x y z h s sdg t tdg id,
 * rx ry rz p u1 (1 angle), u2, u u3 U (3 angles), cx CX cz swap cp cu1, barrier,
 * terminal measure; angles are pi-expressions with + - * / and parentheses; a
 * register argument broadcasts the gate).  `id` becomes U(0,0,0) (a noise location).
 * out: capacity `cap` gates (NULL / 0 to query); *n_gates, *n_qubits: sizes;
 * *measured (may be NULL): 1 if a measure statement was seen.
 * Errors: TQSIM_EINVAL "line L col C: ..." (syntax, unsupported gate, index range,
 * more than TQSIM_MAX_QUBITS qubits). */
tqsim_status tqsim_parse_qasm(const char* text, tqsim_gate* out, uint64_t cap, uint64_t* n_gates,
                              uint32_t* n_qubits, uint32_t* measured);

tqsim_status tqsim_lower_circuit(const tqsim_circuit* circuit, tqsim_gate* out, uint64_t cap,
                                 uint64_t* n_out);

/* [host] Plan the tree: DCP (§3.2, Eqs.3-5, R12-R18) when arities ==
 * NULL, else the fixed-arity override split into n_levels near-equal slices
 * (R20; requires prod arities >= n_shots, every arity >= 1,
 * n_levels <= lowered gate count).  opts NULL = defaults. */
tqsim_status tqsim_plan_circuit(const tqsim_circuit* circuit, const tqsim_noise_model* noise,
                                uint64_t n_shots, const uint32_t* arities, uint32_t n_levels,
                                const tqsim_options* opts, tqsim_plan* out);

/* [host] The pass plan as op records (one per lowered gate). */
tqsim_status tqsim_describe_passes(const tqsim_circuit* circuit, const tqsim_noise_model* noise,
                                   uint64_t n_shots, const uint32_t* arities, uint32_t n_levels,
                                   const tqsim_options* opts, tqsim_op_record* out, uint64_t cap,
                                   uint64_t* n_out);

/* [host] Generate and compile (NVRTC, sm_100a; no GPU needed) every run-time
 * specialized gate-pass kernel of the plan: one kernel per (level, pass) whose
 * gate sequence, qubit positions and matrices are compile-time constants.
 * Outputs may be NULL.  Compile errors -> TQSIM_EINTERNAL with the NVRTC log. */
tqsim_status tqsim_compile_passes(const tqsim_circuit* circuit, const tqsim_noise_model* noise,
                                  uint64_t n_shots, const uint32_t* arities, uint32_t n_levels,
                                  const tqsim_options* opts, uint64_t* n_kernels,
                                  uint64_t* cubin_bytes, double* seconds);

/* [host] CUDA source of the specialized kernel of (level, pass): up to cap-1
 * characters + NUL are written to out; *n_out = full length. */
tqsim_status tqsim_pass_source(const tqsim_circuit* circuit, const tqsim_noise_model* noise,
                               uint64_t n_shots, const uint32_t* arities, uint32_t n_levels,
                               const tqsim_options* opts, uint32_t level, uint32_t pass, char* out,
                               uint64_t cap, uint64_t* n_out);

/* [host] Shard of rank/world (see tqsim_shard_levels): the level-0
 * instances [top_begin, top_end) the rank runs (ancestors of its split-level range,
 * recomputed when the split is below level 0) and its contiguous leaf range
 * [leaf_begin, leaf_end).  When world divides A_0 this is [A0*r/W, A0*(r+1)/W). */
tqsim_status tqsim_shard_range(const tqsim_plan* plan, uint32_t rank, uint32_t world,
                               uint64_t* top_begin, uint64_t* top_end, uint64_t* leaf_begin,
                               uint64_t* leaf_end);

/* [gpu] Create an execution handle on the current device: lowering, plan,
 * pass plan, gate tables uploaded to HBM. */
tqsim_status tqsim_create(const tqsim_circuit* circuit, const tqsim_noise_model* noise,
                          uint64_t n_shots, const uint32_t* arities, uint32_t n_levels,
                          const tqsim_options* opts, tqsim_handle** out);
tqsim_status tqsim_get_plan(const tqsim_handle* h, tqsim_plan* out);
tqsim_status tqsim_get_stats(const tqsim_handle* h, tqsim_stats* out);
void tqsim_destroy(tqsim_handle* h);

/* [host] Device workspace a shard needs (state batches of every level + leaf scratch). */
tqsim_status tqsim_workspace_bytes(const tqsim_handle* h, uint32_t rank, uint32_t world,
                                   uint64_t* bytes);

/* [gpu] Run the shard (rank, world) of the tree asynchronously on `stream`:
 * every leaf l of the shard gets d_leaf_outcomes[l] = its measured bitstring;
 * other entries are not touched (zero the array and allreduce(SUM) across
 * ranks to combine).  d_workspace: >= tqsim_workspace_bytes,
 * 256-byte aligned.  d_leaf_outcomes: plan.n_outcomes uint32.  The call
 * returns once all work is enqueued (profile=1: once it has finished). */
tqsim_status tqsim_execute(tqsim_handle* h, uint64_t seed, uint32_t rank, uint32_t world,
                           void* stream, void* d_workspace, uint64_t workspace_bytes,
                           uint32_t* d_leaf_outcomes);

/* [gpu] Live timing of every gate-pass kernel of the handle (the roofline input of
 * bench.py): runs the shard once (seed) to fill the workspace with real states, then
 * for each (level, pass) re-runs that level's first batch's noise rows and times `reps`
 * back-to-back launches of the pass on its in-tree operands with CUDA events on
 * `stream`.  Synchronous; out: capacity `cap` records (NULL / 0 to query *n_out). */
tqsim_status tqsim_profile_passes(tqsim_handle* h, uint64_t seed, uint32_t rank, uint32_t world,
                                  void* stream, void* d_workspace, uint64_t workspace_bytes,
                                  uint32_t* d_leaf_outcomes, uint32_t reps, tqsim_pass_timing* out,
                                  uint64_t cap, uint64_t* n_out);

/* In-tree timing of the tree's kernels, aggregated per (kind, level, pass) (tqsim_profile_tree). */
typedef struct {
  uint32_t kind;              /* 0 gate pass (tq_pass_l<level>_p<pass>), 1 leaf measurement of the
                                 level (select + leaf recompute + finish kernels), 2 noise rows */
  uint32_t level, pass;
  uint32_t reserved;
  uint64_t launches;
  uint64_t states;            /* node instances the launches covered (their grids) */
  uint64_t computed_states;   /* instances actually computed (dedup representatives) */
  double ms;                  /* sum of the launches' CUDA-event durations (serialised, in tree order) */
  double alg_bytes;           /* algorithmic HBM bytes of the computed instances */
  double nominal_bytes;       /* the same counted for every instance (SURVEY §8(d) per-unit figure) */
  double fp64_per_amp;        /* kind 0: FP64 operations per amplitude of the fast path (cost model) */
} tqsim_kernel_timing;

/* [gpu] Run the shard once with every launch bracketed by CUDA events on `stream` (no graph,
 * no pipelining: the kernels run in tree order, one at a time) and report each kernel
 * family's summed device time with the work it did (the roofline input of bench.py).
 * Synchronous.  out: capacity `cap` records (NULL / 0 to query *n_out). */
tqsim_status tqsim_profile_tree(tqsim_handle* h, uint64_t seed, uint32_t rank, uint32_t world,
                                void* stream, void* d_workspace, uint64_t workspace_bytes,
                                uint32_t* d_leaf_outcomes, tqsim_kernel_timing* out, uint64_t cap,
                                uint64_t* n_out);

/* [host] The shard's instance range at every level: the tree is split at
 * level *split_level, the first level whose instance count is a multiple of world (else
 * the first with >= 16 * world instances, else the leaf level); rank owns level-split
 * instances [I*rank/world, I*(rank+1)/world) and all their descendants, and recomputes
 * their ancestors.  lo, hi: arrays of plan->n_levels entries (host); the rank's level-d
 * instances are [lo[d], hi[d]). */
tqsim_status tqsim_shard_levels(const tqsim_plan* plan, uint32_t rank, uint32_t world,
                                uint32_t* split_level, uint64_t* lo, uint64_t* hi);

/* [gpu] The north_star call: host circuit in, host histogram out (allocates
 * its own workspace, synchronous).  tree_arities NULL = auto (DCP). */
tqsim_status tqsim_run(const tqsim_circuit* circuit, const tqsim_noise_model* noise,
                       uint64_t n_shots, const uint32_t* tree_arities, uint32_t n_levels,
                       uint64_t seed, tqsim_result** out);

/* [gpu] tqsim_run with options and optional state dumps (debug may be NULL). */
tqsim_status tqsim_run_ex(const tqsim_circuit* circuit, const tqsim_noise_model* noise,
                          uint64_t n_shots, const uint32_t* tree_arities, uint32_t n_levels,
                          uint64_t seed, const tqsim_options* opts, const tqsim_debug* debug,
                          tqsim_result** out);
void tqsim_result_free(tqsim_result* r);

/* [host] Release what tqsim_run / tqsim_run_ex keep between calls: the prepared-handle
 * (plan) cache, the device workspace arena and the page-locked outcome buffer.  The next
 * call plans and allocates again.  Not concurrent with a running tqsim_run. */
void tqsim_release_run_cache(void);

/* [gpu] B200 state-copy cost in gate units (§3.3, fig:copy-overhead; SURVEY
 * §8(f) #2): *copy_ms = device-to-device copy of a 1 GiB batch of n-qubit states,
 * *gate_ms = the engine's time per gate application on the same batch (seeded probe
 * slice of n_probe_gates random U / CX gates, noise-free), *copy_cost_gates = their
 * ratio -- the value to pass as tqsim_options.copy_cost_gates for a device-measured
 * DCP first-slice length (the default 10 is the paper's desktop-GPU figure, R14).
 * n_qubits in [4, 28]; copy_ms / gate_ms may be NULL. */
tqsim_status tqsim_profile_copy_cost(uint32_t n_qubits, uint32_t n_probe_gates, uint64_t seed,
                                     double* copy_cost_gates, double* copy_ms, double* gate_ms);

/* [gpu] Debug / parity hooks running the SAME device functions as the hot path.
 * Philox4x32-10 on n counters: in = n x {c0,c1,c2,c3,k0,k1}, out = n x 4 words. */
tqsim_status tqsim_debug_philox(const uint32_t* in, uint64_t n, uint32_t* out);
/* Noise codes of level `level`, instances [inst_begin, inst_begin+count):
 * out[i * slice_len + t] = code of gate boundaries[level]+t (0 none, 1..3 / 1..15). */
tqsim_status tqsim_debug_noise_table(tqsim_handle* h, uint64_t seed, uint32_t level,
                                     uint64_t inst_begin, uint64_t count, uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif /* TQSIM_H */
