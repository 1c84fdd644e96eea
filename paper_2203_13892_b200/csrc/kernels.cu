// Static sm_100a kernels of the TQSim hot path and the
// debug hooks.  The gate-pass kernels (row a5) are specialized per pass at run
// time (jit.cpp); both include the same device functions (tq_device_common.cuh).
//
//  chunk_sums       sums of 2^C-amplitude chunks from the 8-amplitude |a|^2 run
//                   sums the leaf's last gate pass writes (fused, jit.cpp)
//  sample_kernel    one CTA per leaf: warp-shuffle block scans -> chunk -> run ->
//                   amplitude: the smallest x with C(x) > u*total (§2.3
//                   "the final outcome is sampled", reading R9), then readout
//                   flips (R11).
#include <cuda_runtime.h>
#include <cstdlib>

#include "tq_device_common.cuh"
#include "tq_internal.h"

namespace tq {
namespace dev {

constexpr int MT = 256;   // threads of the measurement kernels

// Leaf sampling without a stored leaf state: the select phase writes, per leaf, the run
// holding u*total (runsel), the residual target inside the run (t3) and the tile the
// leaf pass must recompute to produce that run (tile); the finish phase walks the 8
// recomputed amplitudes (scratch).
struct SelectOut {
  uint32_t* runsel;
  double* t3;
  uint32_t* tile;
  const uint32_t* xl;         // the leaf pass's store-address XOR per leaf
  uint32_t n_out;
  uint32_t out_row[32];       // out-of-tile qubit i = parity(out_row[i] & stored address)
  const uint32_t* rep;        // dedup map of the leaf batch (null: every leaf computed)
  // debug outputs (tqsim_debug; null = not requested), indexed by global leaf id
  double* dbg_u;
  double* dbg_total;
  uint8_t* dbg_flag;
  // conditional leaf sampling: stage 1 writes the chosen chunk (the top bits)
  // and the residual target; stage 2 samples the rest with that target and ORs the top bits
  uint32_t* hsel;
  double* htarget;
  const double* tgt;
  const uint32_t* hi;
  uint32_t hi_shift;
};

// R9: the draw is flagged when u*total lies within 1e-9 of C(x-1) or C(x).  t = target
// relative to the run start, c0 / c1 = the run's cumulative sums before / after x.
__device__ __forceinline__ uint8_t tq_flag(double t, double c0, double c1) {
  return (uint8_t)((t - c0 < 1e-9) || (c1 - t < 1e-9));
}

// The leaf whose run sums leaf s reads (the dedup map: the gate passes computed only it)
__device__ __forceinline__ uint32_t tq_dedup_rep(const SelectOut& so, uint64_t leaf_first, uint32_t s) {
  (void)leaf_first;
  return so.rep ? so.rep[s] : s;
}

__device__ __forceinline__ uint32_t tile_of_run(uint64_t run, uint32_t xl, const SelectOut& so) {
  const uint64_t a = (run << RUN_Q) ^ (uint64_t)xl;   // source (physical) index, logical bits
  uint32_t t = 0;
  for (uint32_t i = 0; i < so.n_out; ++i) t |= (uint32_t)(__popcll(a & (uint64_t)so.out_row[i]) & 1) << i;
  return t;
}

struct __align__(16) cd {
  double x, y;
};

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double r = threadIdx.x < (MT >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    if (threadIdx.x == 0) red[0] = r;
  }
  __syncthreads();
  return red[0];
}

// Inclusive block scan of one double per thread (warp shuffles + per-warp totals).
__device__ __forceinline__ double block_incl_scan(double v, double* wsum) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double n = __shfl_up_sync(0xffffffffu, v, o);
    if (l >= o) v += n;
  }
  __syncthreads();
  if (l == 31) wsum[w] = v;
  __syncthreads();
  double before = 0.0;
  for (int i = 0; i < w; ++i) before += wsum[i];
  return before + v;
}

// index of the first thread whose predicate is true (MT if none)
__device__ __forceinline__ int block_first(bool pred, int* sh) {
  const unsigned bal = __ballot_sync(0xffffffffu, pred);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (threadIdx.x == 0) *sh = MT;
  __syncthreads();
  if (l == 0 && bal) atomicMin(sh, w * 32 + __ffs(bal) - 1);
  __syncthreads();
  return *sh;
}

// Chunk sums over the leaf's run sums (written by the fused last gate pass):
// chunk = 2^chunk_log2 amplitudes = 2^(chunk_log2 - RUN_Q) runs.
__global__ void __launch_bounds__(MT) chunk_sums_kernel(const double* __restrict__ runs, uint32_t n,
                                                        uint32_t chunk_log2,
                                                        double* __restrict__ sums, uint64_t leaf_first,
                                                        const __grid_constant__ SelectOut so) {
  __shared__ double red[MT / 32];
  const uint32_t rpc = 1u << (chunk_log2 - RUN_Q);   // runs per chunk
  const uint64_t bid = blockIdx.x;                   // = state * n_chunks + chunk
  const uint32_t st = (uint32_t)(bid >> (n - chunk_log2));
  if (tq_dedup_rep(so, leaf_first, st) != st) return;   // a duplicate: its representative's sums
  const double* p = runs + bid * rpc;
  double acc = 0.0;
  for (uint32_t i = threadIdx.x; i < rpc; i += MT) acc += p[i];
  const double tot = block_sum(acc, red);
  if (threadIdx.x == 0) sums[bid] = tot;
}

// First index i of v[0..len) whose running sum from `base` exceeds target, found by
// the whole block over per-thread contiguous ranges (block scan + ballot).  Returns
// len if none; *before = running sum before v[i].
__device__ __forceinline__ uint64_t block_search(const double* __restrict__ v, uint64_t len,
                                                 double target, double* before, double* wsum,
                                                 int* first_sh, uint64_t* pick_sh,
                                                 double* before_sh) {
  const uint64_t per = (len + MT - 1) / MT;
  const uint64_t c0 = per * threadIdx.x < len ? per * threadIdx.x : len;
  const uint64_t c1 = c0 + per < len ? c0 + per : len;
  double loc = 0.0;
  for (uint64_t c = c0; c < c1; ++c) loc += v[c];
  const double incl = block_incl_scan(loc, wsum);
  const int tsel = block_first(incl > target, first_sh);
  if (threadIdx.x == 0) {
    *pick_sh = len;
    *before_sh = 0.0;
  }
  __syncthreads();
  if ((int)threadIdx.x == tsel) {
    double acc = incl - loc;
    uint64_t pick = len;
    for (uint64_t c = c0; c < c1; ++c) {
      if (acc + v[c] > target) {
        pick = c;
        break;
      }
      acc += v[c];
    }
    if (pick == len) {   // rounding between the scan and the sequential walk: last non-empty
      acc = incl - loc;
      for (uint64_t c = c0; c < c1; ++c)
        if (v[c] > 0.0) pick = c;
      for (uint64_t c = c0; c < pick && pick < len; ++c) acc += v[c];
    }
    *pick_sh = pick;
    *before_sh = acc;
  }
  __syncthreads();
  if (*pick_sh == len) {   // target beyond the total (rounding): last non-empty entry
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t c = len;
      double acc = 0.0;
      for (uint64_t i = 0; i < len; ++i)
        if (v[i] > 0.0) c = i;
      if (c == len) c = len - 1;
      for (uint64_t i = 0; i < c; ++i) acc += v[i];
      *pick_sh = c;
      *before_sh = acc;
    }
    __syncthreads();
  }
  *before = *before_sh;
  const uint64_t r = *pick_sh;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(MT) sample_kernel(const cd* __restrict__ states,
                                                    const double* __restrict__ runs,
                                                    const double* __restrict__ sums, uint32_t n,
                                                    uint32_t n_user, uint32_t chunk_log2,
                                                    uint64_t leaf_first, const uint64_t* __restrict__ seedp,
                                                    double p01, double p10, uint32_t* __restrict__ out,
                                                    const __grid_constant__ SelectOut so) {
  const uint64_t seed = *seedp;
  __shared__ double wsum[MT / 32];
  __shared__ int first_sh;
  __shared__ uint64_t pick_sh;
  __shared__ double before_sh, total_sh;
  const uint32_t s = blockIdx.x;
  const uint64_t leaf = leaf_first + s;
  const uint64_t nc = 1ull << (n - chunk_log2);
  const uint32_t rpc = 1u << (chunk_log2 - RUN_Q);
  const uint32_t sr = tq_dedup_rep(so, leaf_first, s);   // whose run / chunk sums to read
  const double* cs = sums + (uint64_t)sr * nc;
  const double u = tq_measure_uniform(leaf, seed);

  // total = sum of chunk sums (block reduction in a fixed order)
  double loc = 0.0;
  for (uint64_t c = threadIdx.x; c < nc; c += MT) loc += cs[c];
  const double tot = block_sum(loc, wsum);
  if (threadIdx.x == 0) total_sh = tot;
  __syncthreads();
  const double target = so.tgt ? so.tgt[s] : u * total_sh;   // stage 2: the residual target
  if (threadIdx.x == 0 && so.dbg_u && !so.tgt) so.dbg_u[leaf] = u;
  if (threadIdx.x == 0 && so.dbg_total && !so.tgt) so.dbg_total[leaf] = total_sh;
  // level 1: chunk;  level 2: 8-amplitude run inside the chunk;  level 3: amplitude
  double before1 = 0.0, before2 = 0.0;
  const uint64_t chunk = block_search(cs, nc, target, &before1, wsum, &first_sh, &pick_sh, &before_sh);
  if (so.hsel) {   // stage 1 of the conditional sampling: the chunk = the leaf's top bits
    if (threadIdx.x == 0) {
      so.hsel[s] = (uint32_t)chunk;
      so.htarget[s] = target - before1;
    }
    return;
  }
  const double* rs = runs + ((uint64_t)sr << (n - RUN_Q)) + chunk * rpc;
  const uint64_t run = block_search(rs, rpc, target - before1, &before2, wsum, &first_sh, &pick_sh,
                                    &before_sh);
  if (threadIdx.x == 0 && so.runsel) {   // select phase only (the leaf state was not stored)
    const uint64_t r = chunk * rpc + run;
    so.runsel[s] = (uint32_t)r;
    so.t3[s] = target - before1 - before2;
    so.tile[s] = tile_of_run(r, so.xl[s], so);
    return;
  }
  if (threadIdx.x == 0) {
    const double t3 = target - before1 - before2;
    const uint64_t base = ((chunk * rpc + run) << RUN_Q);
    const cd* ap = states + ((uint64_t)s << n) + base;
    double acc = 0.0, c0 = 0.0, c1 = 0.0;
    int x = -1, lastnz = -1;
    for (int e = 0; e < (1 << RUN_Q); ++e) {
      const cd v = ap[e];
      const double pr = v.x * v.x + v.y * v.y;
      if (pr > 0.0) lastnz = e;
      if (x < 0) c0 = acc;
      acc += pr;
      if (x < 0 && acc > t3) {
        x = e;
        c1 = acc;
      }
    }
    uint8_t flag = x < 0 ? 1 : tq_flag(t3, c0, c1);
    if (x < 0) x = lastnz >= 0 ? lastnz : 0;   // rounding: the last non-zero amplitude of the run
    if (so.dbg_flag) so.dbg_flag[leaf] = flag;
    const uint32_t xi = (uint32_t)(base + (uint64_t)x);
    // readout (R11): bit b flips iff word (b&3) of Philox(ctr=(b>>2, leaf, 2, 0)) * 2^-32 < p
    uint32_t mask = 0;
    if (p01 > 0.0 || p10 > 0.0) {
      tq_w4 rw = {0, 0, 0, 0};
      for (uint32_t b = 0; b < n_user; ++b) {
        if ((b & 3u) == 0) rw = tq_philox_keyed(b >> 2, leaf, 2u, seed);
        const uint32_t wv = (b & 3u) == 0 ? rw.x : (b & 3u) == 1 ? rw.y : (b & 3u) == 2 ? rw.z : rw.w;
        const double p = ((xi >> b) & 1u) ? p10 : p01;
        if ((double)wv * 0x1p-32 < p) mask |= 1u << b;
      }
    }
    out[leaf] = xi ^ mask;
  }
}

// Small states (<= 2^17 amplitudes): one CTA per leaf reads all of the leaf's run sums
// (16-64 per thread, contiguous), block-scans the per-thread totals, and the thread
// whose range crosses u*total walks its runs; then the run's 8 amplitudes -> x and
// readout -- the chunk level (and its kernel) is not needed (§2.3, R9, R11).
__device__ __forceinline__ uint32_t readout_flips(uint32_t xi, uint32_t n_user, uint64_t leaf,
                                                  uint64_t seed, double p01, double p10) {
  uint32_t mask = 0;
  if (p01 > 0.0 || p10 > 0.0) {
    tq_w4 rw = {0, 0, 0, 0};
    for (uint32_t b = 0; b < n_user; ++b) {
      if ((b & 3u) == 0) rw = tq_philox_keyed(b >> 2, leaf, 2u, seed);
      const uint32_t wv = (b & 3u) == 0 ? rw.x : (b & 3u) == 1 ? rw.y : (b & 3u) == 2 ? rw.z : rw.w;
      const double p = ((xi >> b) & 1u) ? p10 : p01;
      if ((double)wv * 0x1p-32 < p) mask |= 1u << b;
    }
  }
  return mask;
}

__global__ void __launch_bounds__(MT) sample_small_kernel(const cd* __restrict__ states,
                                                          const double* __restrict__ runs,
                                                          uint32_t n, uint32_t n_user,
                                                          uint64_t leaf_first,
                                                          const uint64_t* __restrict__ seedp,
                                                          double p01, double p10,
                                                          uint32_t* __restrict__ out,
                                                          const __grid_constant__ SelectOut so) {
  // warp w owns the contiguous run segment [w*seg, (w+1)*seg); lanes read it coalesced
  constexpr uint32_t W = MT / 32;
  __shared__ double wtot[W];
  const uint64_t seed = *seedp;
  const uint32_t s = blockIdx.x, w = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const uint64_t leaf = leaf_first + s;
  const uint32_t R = 1u << (n - RUN_Q);
  const uint32_t seg = (R + W - 1) / W;
  const double* rs = runs + ((uint64_t)tq_dedup_rep(so, leaf_first, s) << (n - RUN_Q));
  const uint32_t s0 = w * seg, s1 = min(R, s0 + seg);
  double part = 0.0;
  for (uint32_t i = s0 + lane; i < s1; i += 32u) part += rs[i];
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) wtot[w] = part;
  __syncthreads();
  // every warp walks the W segment totals (identical order -> identical decision)
  double total = 0.0;
  for (uint32_t i = 0; i < W; ++i) total += wtot[i];
  const double u = tq_measure_uniform(leaf, seed);
  const double target = so.tgt ? so.tgt[s] : u * total;   // stage 2: the residual target
  if (threadIdx.x == 0 && so.dbg_u && !so.tgt) so.dbg_u[leaf] = u;
  if (threadIdx.x == 0 && so.dbg_total && !so.tgt) so.dbg_total[leaf] = total;
  double before = 0.0;
  int ws = -1, wlast = 0;
  for (uint32_t i = 0; i < W; ++i) {
    if (wtot[i] > 0.0) wlast = (int)i;
    if (ws < 0 && before + wtot[i] > target) ws = (int)i;
    if (ws < 0) before += wtot[i];
  }
  if (ws < 0) {   // rounding: target at the very top -> the last segment with mass
    ws = wlast;
    before = 0.0;
    for (int i = 0; i < ws; ++i) before += wtot[i];
  }
  if ((int)w != ws) return;
  // this warp: 32-run rounds, warp inclusive scan + ballot finds the first crossing
  const uint32_t a0 = ws * seg, a1 = min(R, a0 + seg);
  uint32_t run = a1 - 1, lastnz = a0;
  double acc = before;
  bool found = false;
  for (uint32_t base = a0; base < a1 && !found; base += 32u) {
    const uint32_t i = base + lane;
    const double v = i < a1 ? rs[i] : 0.0;
    double incl = v;
    for (int o = 1; o < 32; o <<= 1) {
      const double t = __shfl_up_sync(0xffffffffu, incl, o);
      if ((int)lane >= o) incl += t;
    }
    const unsigned nz = __ballot_sync(0xffffffffu, v > 0.0);
    if (nz) lastnz = base + 31u - __clz(nz);
    const unsigned hit = __ballot_sync(0xffffffffu, acc + incl > target);
    if (hit) {
      const int f = __ffs(hit) - 1;
      run = base + (uint32_t)f;
      acc += __shfl_sync(0xffffffffu, incl - v, f);
      found = true;
    } else {
      acc += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  if (!found) {   // rounding between the segment total and the walk: last run with mass
    run = lastnz;
    acc = before;
    for (uint32_t i = a0; i < run; ++i) acc += rs[i];
  }
  if (lane != 0) return;
  const double t3 = target - acc;
  if (so.runsel) {   // select phase only (the leaf state was not stored)
    so.runsel[s] = run;
    so.t3[s] = t3;
    so.tile[s] = tile_of_run(run, so.xl[s], so);
    return;
  }
  const uint64_t abase = (uint64_t)run << RUN_Q;
  const cd* ap = states + ((uint64_t)s << n) + abase;
  double c = 0.0, c0 = 0.0, c1 = 0.0;
  int x = -1, lastamp = -1;
  for (int e = 0; e < (1 << RUN_Q); ++e) {
    const cd v = ap[e];
    const double pr = v.x * v.x + v.y * v.y;
    if (pr > 0.0) lastamp = e;
    if (x < 0) c0 = c;
    c += pr;
    if (x < 0 && c > t3) {
      x = e;
      c1 = c;
    }
  }
  if (so.dbg_flag) so.dbg_flag[leaf] = x < 0 ? 1 : tq_flag(t3, c0, c1);
  if (x < 0) x = lastamp >= 0 ? lastamp : 0;
  uint32_t xi = (uint32_t)(abase + (uint64_t)x);
  if (so.hi) xi |= so.hi[s] << so.hi_shift;
  out[leaf] = xi ^ readout_flips(xi, n_user, leaf, seed, p01, p10);
}

// Finish phase: one thread per leaf walks the recomputed run (8 amplitudes) for the
// smallest x with C(x) > u*total (R9), then the readout flips (R11).
__global__ void __launch_bounds__(MT) sample_finish_kernel(const cd* __restrict__ scratch,
                                                           const uint32_t* __restrict__ runsel,
                                                           const double* __restrict__ t3s, uint32_t batch,
                                                           uint32_t n_user, uint64_t leaf_first,
                                                           const uint64_t* __restrict__ seedp, double p01,
                                                           double p10, uint32_t* __restrict__ out,
                                                           uint8_t* __restrict__ dbg_flag,
                                                           const uint32_t* __restrict__ hi, uint32_t hi_shift) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= batch) return;
  const uint64_t seed = *seedp;
  const uint64_t leaf = leaf_first + s;
  const double t3 = t3s[s];
  const cd* ap = scratch + ((uint64_t)s << RUN_Q);
  double c = 0.0, c0 = 0.0, c1 = 0.0;
  int x = -1, lastamp = -1;
  for (int e = 0; e < (1 << RUN_Q); ++e) {
    const cd v = ap[e];
    const double pr = v.x * v.x + v.y * v.y;
    if (pr > 0.0) lastamp = e;
    if (x < 0) c0 = c;
    c += pr;
    if (x < 0 && c > t3) {
      x = e;
      c1 = c;
    }
  }
  if (dbg_flag) dbg_flag[leaf] = x < 0 ? 1 : tq_flag(t3, c0, c1);
  if (x < 0) x = lastamp >= 0 ? lastamp : 0;
  uint32_t xi = (uint32_t)(((uint64_t)runsel[s] << RUN_Q) + (uint64_t)x);
  if (hi) xi |= hi[s] << hi_shift;   // conditional sampling: the stage-1 top bits
  out[leaf] = xi ^ readout_flips(xi, n_user, leaf, seed, p01, p10);
}

// ------------------------------------------------------------------ debug hooks
__global__ void philox_debug_kernel(const uint32_t* in, uint64_t n, uint32_t* out) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t* v = in + 6 * i;
  const tq_w4 r = tq_philox4x32_10(v[0], v[1], v[2], v[3], v[4], v[5]);
  out[4 * i + 0] = r.x;
  out[4 * i + 1] = r.y;
  out[4 * i + 2] = r.z;
  out[4 * i + 3] = r.w;
}

__global__ void noise_table_kernel(const uint8_t* two, uint32_t slice_begin, uint32_t slice_len,
                                   uint64_t inst_begin, uint64_t count, uint64_t seed, double p1,
                                   double p2, uint8_t* out) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= count * slice_len) return;
  const uint64_t inst = inst_begin + i / slice_len;
  const uint32_t t = (uint32_t)(i % slice_len);
  const bool tw = two[t] != 0;
  out[i] = (uint8_t)tq_noise_code(slice_begin + t, inst, seed, tw ? p2 : p1, tw);
}

// Noise rows (row a3, §2.5, "after each of the gates", R1/R7/R8): one
// warp per instance of a level batch draws the keyed Pauli code of every gate of
// the slice and ORs the pass bitmask the gate-pass kernels branch on (error-free
// instances take the fused fast path).  Drawn once per instance, not per tile.
__global__ void __launch_bounds__(256) noise_rows_kernel(
    const uint8_t* __restrict__ two, const uint8_t* __restrict__ pass_of, uint32_t slice_begin,
    uint32_t slice_len, uint64_t inst_first, uint32_t count, const uint64_t* __restrict__ seedp,
    double p1, double p2, uint32_t row_bytes, uint8_t* __restrict__ rows) {
  const uint64_t seed = *seedp;
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  if (w >= count) return;
  const uint64_t inst = inst_first + w;
  uint8_t* row = rows + w * row_bytes;
  uint32_t mask = 0;
  for (uint32_t t = lane; t < slice_len; t += 32u) {
    const uint32_t g = slice_begin + t;
    const bool tw = two[g] != 0;
    const uint32_t c = tq_noise_code(g, inst, seed, tw ? p2 : p1, tw);
    row[4 + t] = (uint8_t)c;
    if (c) mask |= 1u << pass_of[g];
  }
  mask = __reduce_or_sync(0xffffffffu, mask);
  if (lane == 0) *reinterpret_cast<uint32_t*>(row) = mask;
}

// Every noise row of a shard (all levels) in one launch: warp w -> (level, instance) by
// the levels' cumulative counts; the row as in noise_rows_kernel.
__global__ void __launch_bounds__(256) noise_rows_all_kernel(
    const uint8_t* __restrict__ two, const uint8_t* __restrict__ pass_of, const __grid_constant__ NoiseLevels L,
    uint64_t total, const uint64_t* __restrict__ seedp, double p1, double p2, uint8_t* __restrict__ rows) {
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  if (w >= total) return;
  uint64_t rem = w;
  uint32_t d = 0;
  while (d + 1 < L.n_levels && rem >= L.lv[d].count) rem -= L.lv[d].count, ++d;
  const NoiseLevel& lv = L.lv[d];
  const uint64_t seed = *seedp;
  const uint64_t inst = lv.inst_first + rem;
  uint8_t* row = rows + lv.rows_off + rem * lv.row_bytes;
  uint32_t mask = 0;
  for (uint32_t t = lane; t < lv.slice_len; t += 32u) {
    const uint32_t g = lv.slice_begin + t;
    const bool tw = two[g] != 0;
    const uint32_t c = tq_noise_code(g, inst, seed, tw ? p2 : p1, tw);
    row[4 + t] = (uint8_t)c;
    if (c) mask |= 1u << pass_of[g];
  }
  mask = __reduce_or_sync(0xffffffffu, mask);
  if (lane == 0) *reinterpret_cast<uint32_t*>(row) = mask;
}

// Dedup map of every level of the shard (one CTA, levels in order: a level's map reads its
// parent level's).  Batches are formed as run_level forms them: level 0 in caps from the
// shard's first instance, level d+1 in caps from (parent batch start) * arity.  An instance
// with an error in its slice is computed (rep = itself).  An error-free instance shares the
// state of the first error-free child, in its batch, of its parent's representative P*
// (different parents with the same representative hold the same state), else of the first
// error-free sibling in its batch, else it is computed; the chosen instance is computed by
// the same rule.
__device__ __forceinline__ void dedup_map_level(const uint8_t* __restrict__ rows, const NoiseLevels& L,
                                                uint32_t d, uint64_t idx0, uint64_t stride,
                                                uint32_t* __restrict__ rep, uint32_t* __restrict__ pos) {
  {
    const NoiseLevel& lv = L.lv[d];
    const uint8_t* rw = rows + lv.rows_off;
    // em(j) != 0: instance j drew an error that makes it "not error-free" (lv.err_sel: only those gates)
    auto em = [&](uint64_t j) -> uint32_t {
      const uint8_t* row = rw + (j - lv.inst_first) * lv.row_bytes;
      if (!lv.err_sel) return *reinterpret_cast<const uint32_t*>(row);
      for (uint32_t t = 0; t < lv.slice_len; ++t)
        if (lv.err_sel[t] && row[4 + t]) return 1u;
      return 0u;
    };
    const uint64_t A = lv.arity;
    for (uint64_t idx = idx0; idx < lv.count; idx += stride) {
      const uint64_t j = lv.inst_first + idx;
      uint64_t bs, P = 0, Ps = 0, cfirst;
      if (d == 0) {
        bs = lv.inst_first + ((j - lv.inst_first) / lv.cap) * lv.cap;
        cfirst = lv.inst_first;   // level-0 siblings: the shard's level-0 instances
      } else {
        const NoiseLevel& pl = L.lv[d - 1];
        P = j / A;
        const uint64_t pidx = P - pl.inst_first;
        const uint64_t pbs = P - pos[pl.map_off + pidx];
        // the parent batch's children start at pbs * A, clipped to the shard's first
        // instance of this level (a shard split below level 0 recomputes its ancestors)
        const uint64_t rs = pbs * A > lv.inst_first ? pbs * A : lv.inst_first;
        bs = rs + ((j - rs) / lv.cap) * lv.cap;
        Ps = pbs + rep[pl.map_off + pidx];
        cfirst = P * A;
      }
      pos[lv.map_off + idx] = (uint32_t)(j - bs);
      uint64_t r = j;
      if (em(j) == 0u) {
        bool found = false;
        if (d > 0 && Ps != P)   // children of the parent's representative
          for (uint64_t c = (Ps * A > bs ? Ps * A : bs); c < Ps * A + A && c < j; ++c)
            if (em(c) == 0u) {
              r = c;
              found = true;
              break;
            }
        if (!found)
          for (uint64_t c = (cfirst > bs ? cfirst : bs); c < j; ++c)
            if (em(c) == 0u) {
              r = c;
              break;
            }
      }
      rep[lv.map_off + idx] = (uint32_t)(r - bs);
    }
  }
}

// all levels, one CTA (levels in order)
__global__ void __launch_bounds__(1024) dedup_map_kernel(const uint8_t* __restrict__ rows,
                                                         const __grid_constant__ NoiseLevels L,
                                                         uint32_t* __restrict__ rep, uint32_t* __restrict__ pos) {
  for (uint32_t d = 0; d < L.n_levels; ++d) {
    dedup_map_level(rows, L, d, threadIdx.x, blockDim.x, rep, pos);
    __syncthreads();
  }
}

// one level, one thread per instance (a chain of these on a side stream runs ahead of
// the tree's levels)
__global__ void __launch_bounds__(256) dedup_map_level_kernel(const uint8_t* __restrict__ rows,
                                                              const __grid_constant__ NoiseLevels L, uint32_t d,
                                                              uint32_t* __restrict__ rep, uint32_t* __restrict__ pos) {
  dedup_map_level(rows, L, d, blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, (uint64_t)gridDim.x * blockDim.x,
                  rep, pos);
}

// A leaf whose Pauli falls inside a diagonal unit on the TOP bits keeps the streaming
// projection: the unit with its Paulis is monomial, U|idx> = D[idx] |idx ^ flip> (a Pauli pushed
// through CX / diagonal gates stays a Pauli), idx = bit ua + 2 bit ub of the top index.  Applied
// to the gates' basis states in slice order; returns the flip as a mask over the top bits.
// (Units on the low bits would move the rows read: those leaves go to the generated kernel.)
__device__ __forceinline__ void proj_pauli(uint32_t c, int& b, cd& amp) {
  if (c == 1u) {
    b ^= 1;
  } else if (c == 2u) {   // Y|0> = i|1>, Y|1> = -i|0>
    amp = b ? cd{amp.y, -amp.x} : cd{-amp.y, amp.x};
    b ^= 1;
  } else if (c == 3u && b) {
    amp = {-amp.x, -amp.y};
  }
}
__device__ uint32_t proj_unit_eff(const ProjSpec& sp, uint32_t u, const unsigned char* codes, cd* D) {
  const bool one = sp.ua[u] == sp.ub[u];
  uint32_t xm = 0;
  for (int idx = 0; idx < 4; ++idx) {
    if (one && (idx == 1 || idx == 2)) {
      D[idx] = {0.0, 0.0};
      continue;
    }
    int ba = idx & 1, bb = idx >> 1;
    cd amp = {1.0, 0.0};
    for (uint32_t g = 0; g < sp.ugn[u]; ++g) {
      const uint32_t k = sp.ugk[u][g], code = codes[4 + sp.ugoff[u][g]];
      uint32_t pa = 0, pb = 0;
      if (k <= 1u) {   // 1q diagonal
        const double* d = sp.ugd[u][g];
        const cd e = (k == 0u ? ba : bb) ? cd{d[2], d[3]} : cd{d[0], d[1]};
        amp = {amp.x * e.x - amp.y * e.y, amp.x * e.y + amp.y * e.x};
        (k == 0u ? pa : pb) = code;
      } else {         // CX(ua -> ub) / CZ(ua, ub), then the Pauli pair (q0 = code >> 2 on ua)
        if (k == 2u) {
          if (ba) bb ^= 1;
        } else if (ba && bb) {
          amp = {-amp.x, -amp.y};
        }
        pa = code >> 2;
        pb = code & 3u;
      }
      proj_pauli(pa, ba, amp);
      if (one) bb = ba;
      proj_pauli(pb, bb, amp);
      if (one) ba = bb;
    }
    const int f = idx ^ (ba | (bb << 1));
    if (f & 1) xm |= 1u << sp.ua[u];
    if (f & 2) xm |= 1u << sp.ub[u];
    D[idx] = amp;
  }
  return xm;
}
__device__ __forceinline__ bool proj_unit_erred(const ProjSpec& sp, uint32_t u, const unsigned char* codes) {
  bool e = false;
  for (uint32_t g = 0; g < sp.ugn[u]; ++g) e |= codes[4 + sp.ugoff[u][g]] != 0;
  return e;
}
// c[y] = prod_j U_j[sel_j][cur_j] * (the units' factors along the walk cur: y -> y ^ flips),
// E/X/on: the leaf's effective operators of the erred top units (else the planned tables)
__device__ __forceinline__ cd proj_coef(const ProjSpec& sp, const cd (*U)[4], uint32_t sel, uint32_t y,
                                        const cd (*E)[4], const uint32_t* X, const uint8_t* on) {
  uint32_t cur = y;
  for (uint32_t u = 0; u < sp.nug; ++u)
    if (on[u]) cur ^= X[u];
  cd v = {1.0, 0.0};
  for (uint32_t j = 0; j < sp.m; ++j) {
    const cd e = U[j][2 * ((sel >> j) & 1u) + ((cur >> j) & 1u)];
    v = {v.x * e.x - v.y * e.y, v.x * e.y + v.y * e.x};
  }
  cur = y;
  for (uint32_t u = 0; u < sp.nug; ++u) {
    const uint32_t idx = ((cur >> sp.ua[u]) & 1u) | (((cur >> sp.ub[u]) & 1u) << 1);
    const cd e = on[u] ? E[u][idx] : cd{sp.uT[u][2 * idx], sp.uT[u][2 * idx + 1]};
    v = {v.x * e.x - v.y * e.y, v.x * e.y + v.y * e.x};
    if (on[u]) cur ^= X[u];
  }
  return v;
}

// Conditional leaf sampling, projection onto the chosen top bits for pass A
// = diagonal units then 1q gates on the top bits (ProjSpec): per leaf s with top bits sel,
//   psi_s(x) = D_x(x) * sum_y c_s[y] * phi(y 2^n2 + x),  c_s[y] = prod_j U_j[sel_j][y_j] * D_top(y),
// U_j = the product (in slice order) of the keyed-Pauli-times-gate 2x2s of top qubit j.  A leaf
// whose noise row has a Pauli inside a diagonal unit is appended to glist (the generated
// projection kernel handles it).  One complex FMA per amplitude read: HBM-bound.
constexpr int PT = 256, PV = 2;   // threads, consecutive x per thread (one 32-byte access)
__global__ void __launch_bounds__(PT) trail_project_kernel(const __grid_constant__ ProjSpec sp,
                                                           const __grid_constant__ TrailProjLaunch L,
                                                           const uint64_t* __restrict__ seedp) {
  (void)seedp;
  __shared__ cd U[16][4];
  __shared__ cd coef[1 << 10];
  __shared__ cd UE[PROJ_MAX_U][4];
  __shared__ uint32_t UX[PROJ_MAX_U];
  __shared__ uint8_t UON[PROJ_MAX_U];
  __shared__ int skip;
  const uint32_t s = blockIdx.x % L.batch, c = blockIdx.x / L.batch;
  const unsigned char* codes = L.rows + (uint64_t)s * L.row_bytes;
  if (threadIdx.x == 0) {   // a Pauli inside a low-bit unit: the generated kernel
    bool e = false;
    for (uint32_t u = sp.nug; u < sp.nug + sp.nux; ++u) e |= proj_unit_erred(sp, u, codes);
    skip = e;
    if (e && c == 0) L.glist[atomicAdd(L.gcount, 1u)] = s;
  }
  if (threadIdx.x >= 32 && threadIdx.x < 32 + sp.nug) {   // the top units under this leaf's Paulis
    const uint32_t u = threadIdx.x - 32;
    UON[u] = proj_unit_erred(sp, u, codes);
    UX[u] = UON[u] ? proj_unit_eff(sp, u, codes, UE[u]) : 0u;
  }
  if (threadIdx.x < sp.m) {   // U_j: the top qubit's gates with their Paulis, in slice order
    cd u[4] = {{1.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {1.0, 0.0}};
    for (uint32_t i = 0; i < sp.ng; ++i) {
      if (sp.gbit[i] != threadIdx.x) continue;
      cd g[4] = {{sp.gmat[i][0], sp.gmat[i][1]}, {sp.gmat[i][2], sp.gmat[i][3]},
                 {sp.gmat[i][4], sp.gmat[i][5]}, {sp.gmat[i][6], sp.gmat[i][7]}};
      const uint32_t code = codes[4 + sp.goff[i]];
      if (code) {   // P g: X swaps the rows, Z negates row 1, Y = [[0,-i],[i,0]]
        cd r0 = g[0], r1 = g[1], r2 = g[2], r3 = g[3];
        if (code == 1) { g[0] = r2; g[1] = r3; g[2] = r0; g[3] = r1; }
        else if (code == 2) {
          g[0] = {r2.y, -r2.x}; g[1] = {r3.y, -r3.x}; g[2] = {-r0.y, r0.x}; g[3] = {-r1.y, r1.x};
        } else { g[2] = {-r2.x, -r2.y}; g[3] = {-r3.x, -r3.y}; }
      }
      cd v[4];   // u <- g u
      for (int r = 0; r < 2; ++r)
        for (int k = 0; k < 2; ++k) {
          const cd a = g[2 * r], b = g[2 * r + 1], x0 = u[k], x1 = u[2 + k];
          v[2 * r + k] = {a.x * x0.x - a.y * x0.y + b.x * x1.x - b.y * x1.y,
                          a.x * x0.y + a.y * x0.x + b.x * x1.y + b.y * x1.x};
        }
      for (int k = 0; k < 4; ++k) u[k] = v[k];
    }
    for (int k = 0; k < 4; ++k) U[threadIdx.x][k] = u[k];
  }
  __syncthreads();
  if (skip) return;
  const uint32_t sel = L.hsel[s];
  const uint32_t Y = 1u << sp.m;
  for (uint32_t y = threadIdx.x; y < Y; y += PT)   // c[y] = prod_j U_j[sel_j][y_j] * D_top(y)
    coef[y] = proj_coef(sp, U, sel, y, UE, UX, UON);
  __syncthreads();
  const uint64_t j = L.child_first + s;
  uint64_t pj = j / L.arity - L.parent_first;
  if (L.prep) pj = L.prep[pj];
  const cd* __restrict__ src = static_cast<const cd*>(L.src) + (pj << L.n);
  const uint32_t n2 = sp.n2;
  const uint64_t x0 = ((uint64_t)c * PT + threadIdx.x) * PV;
  if (x0 >= (1ull << n2)) return;
  double a0x = 0.0, a0y = 0.0, a1x = 0.0, a1y = 0.0;
#pragma unroll 4
  for (uint32_t y = 0; y < Y; ++y) {
    double px, py, qx, qy;
    asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(px), "=d"(py), "=d"(qx), "=d"(qy)
                 : "l"(src + (((uint64_t)y << n2) | x0)));
    const cd k = coef[y];
    a0x = fma(k.x, px, fma(-k.y, py, a0x));
    a0y = fma(k.x, py, fma(k.y, px, a0y));
    a1x = fma(k.x, qx, fma(-k.y, qy, a1x));
    a1y = fma(k.x, qy, fma(k.y, qx, a1y));
  }
  cd r0 = {a0x, a0y}, r1 = {a1x, a1y};
  for (uint32_t u = sp.nug; u < sp.nug + sp.nux; ++u) {   // D_x: units below the top bits
    for (int v = 0; v < PV; ++v) {
      const uint64_t x = x0 + v;
      const uint32_t idx = (uint32_t)((x >> sp.ua[u]) & 1u) | (uint32_t)(((x >> sp.ub[u]) & 1u) << 1);
      const cd e = {sp.uT[u][2 * idx], sp.uT[u][2 * idx + 1]};
      cd& r = v ? r1 : r0;
      r = {r.x * e.x - r.y * e.y, r.x * e.y + r.y * e.x};
    }
  }
  cd* dst = static_cast<cd*>(L.psi) + ((uint64_t)s << n2) + x0;
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst), "d"(r0.x), "d"(r0.y), "d"(r1.x), "d"(r1.y)
               : "memory");
}

// The same projection for sibling pairs (leaf arity 2, the DCP plans' leaf level): one CTA
// per (parent, chunk of x) reads the parent's amplitudes once for both children -- half the
// L2->SM traffic of one CTA per leaf -- with 8 row loads in flight per thread.
constexpr int QT = 256, QV = 2;
__device__ __forceinline__ void tq_bulk_prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <int MINB>
__global__ void __launch_bounds__(QT, MINB) trail_project_pair_kernel(const __grid_constant__ ProjSpec sp,
                                                                const __grid_constant__ TrailProjLaunch L,
                                                                uint32_t pf) {
  extern __shared__ cd pcoef[];   // [2][2^m]
  __shared__ cd U[2][16][4];
  __shared__ cd UE[2][PROJ_MAX_U][4];
  __shared__ uint32_t UX[2][PROJ_MAX_U];
  __shared__ uint8_t UON[2][PROJ_MAX_U];
  __shared__ int live[2];
  const uint64_t pfirst = L.child_first / 2;
  const uint32_t npar = (uint32_t)((L.child_first + L.batch - 1) / 2 - pfirst + 1);
  const uint32_t g = blockIdx.x % npar, c = blockIdx.x / npar;
  const uint64_t P = pfirst + g;
  // the CTA's rows: 2^m rows of (2^n2 amplitudes apart), its chunk of QT * QV of each; with
  // pf > 0 one thread streams the rows pf ahead into L2 (bulk prefetch: no registers held)
  const uint64_t xb = (uint64_t)c * QT * QV;
  const uint32_t rbytes = (uint32_t)(16 * ((1ull << sp.n2) - xb < (uint64_t)QT * QV ? (1ull << sp.n2) - xb
                                                                                    : (uint64_t)QT * QV));
  const cd* psrc = nullptr;
  if (pf && threadIdx.x == 0 && xb < (1ull << sp.n2)) {
    uint64_t pq = P - L.parent_first;
    if (L.prep) pq = L.prep[pq];
    psrc = static_cast<const cd*>(L.src) + (pq << L.n) + xb;
    for (uint32_t y = 0; y < pf && y < (1u << sp.m); ++y) tq_bulk_prefetch_l2(psrc + ((uint64_t)y << sp.n2), rbytes);
  }
  const uint64_t j0 = P * 2 > L.child_first ? P * 2 : L.child_first;
  const uint64_t j1 = P * 2 + 2 < L.child_first + L.batch ? P * 2 + 2 : L.child_first + L.batch;
  const uint32_t nc = (uint32_t)(j1 - j0), s0 = (uint32_t)(j0 - L.child_first);
  if (threadIdx.x < nc) {   // a child with a Pauli inside a low-bit unit -> the generated kernel
    const uint32_t sl = s0 + threadIdx.x;
    const unsigned char* codes = L.rows + (uint64_t)sl * L.row_bytes;
    bool e = false;
    for (uint32_t u = sp.nug; u < sp.nug + sp.nux; ++u) e |= proj_unit_erred(sp, u, codes);
    live[threadIdx.x] = !e;
    if (e && c == 0) L.glist[atomicAdd(L.gcount, 1u)] = sl;
  }
  if (threadIdx.x >= 64 && threadIdx.x < 64 + nc * sp.nug) {   // top units under each child's Paulis
    const uint32_t ci = (threadIdx.x - 64) / sp.nug, u = (threadIdx.x - 64) % sp.nug;
    const unsigned char* codes = L.rows + (uint64_t)(s0 + ci) * L.row_bytes;
    UON[ci][u] = proj_unit_erred(sp, u, codes);
    UX[ci][u] = UON[ci][u] ? proj_unit_eff(sp, u, codes, UE[ci][u]) : 0u;
  }
  if (threadIdx.x < nc * sp.m) {   // U_j of child ci: the top qubit's gates with their Paulis
    const uint32_t ci = threadIdx.x / sp.m, jb = threadIdx.x % sp.m;
    const unsigned char* codes = L.rows + (uint64_t)(s0 + ci) * L.row_bytes;
    cd u[4] = {{1.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {1.0, 0.0}};
    for (uint32_t i = 0; i < sp.ng; ++i) {
      if (sp.gbit[i] != jb) continue;
      cd gm[4] = {{sp.gmat[i][0], sp.gmat[i][1]}, {sp.gmat[i][2], sp.gmat[i][3]},
                  {sp.gmat[i][4], sp.gmat[i][5]}, {sp.gmat[i][6], sp.gmat[i][7]}};
      const uint32_t code = codes[4 + sp.goff[i]];
      if (code) {   // P g: X swaps the rows, Z negates row 1, Y = [[0,-i],[i,0]]
        const cd r0 = gm[0], r1 = gm[1], r2 = gm[2], r3 = gm[3];
        if (code == 1) { gm[0] = r2; gm[1] = r3; gm[2] = r0; gm[3] = r1; }
        else if (code == 2) {
          gm[0] = {r2.y, -r2.x}; gm[1] = {r3.y, -r3.x}; gm[2] = {-r0.y, r0.x}; gm[3] = {-r1.y, r1.x};
        } else { gm[2] = {-r2.x, -r2.y}; gm[3] = {-r3.x, -r3.y}; }
      }
      cd v[4];   // u <- g u
      for (int r = 0; r < 2; ++r)
        for (int k = 0; k < 2; ++k) {
          const cd a = gm[2 * r], b = gm[2 * r + 1], x0 = u[k], x1 = u[2 + k];
          v[2 * r + k] = {a.x * x0.x - a.y * x0.y + b.x * x1.x - b.y * x1.y,
                          a.x * x0.y + a.y * x0.x + b.x * x1.y + b.y * x1.x};
        }
      for (int k = 0; k < 4; ++k) u[k] = v[k];
    }
    for (int k = 0; k < 4; ++k) U[ci][jb][k] = u[k];
  }
  __syncthreads();
  const uint32_t Y = 1u << sp.m;
  for (uint32_t i = threadIdx.x; i < 2 * Y; i += QT) {   // c_ci[y] = prod_j U_j[sel_j][y_j] * D_top(y)
    const uint32_t ci = i / Y, y = i % Y;
    cd v = {0.0, 0.0};
    if (ci < nc) v = proj_coef(sp, U[ci], L.hsel[s0 + ci], y, UE[ci], UX[ci], UON[ci]);
    pcoef[i] = v;
  }
  __syncthreads();
  if (!live[0] && (nc < 2 || !live[1])) return;
  uint64_t pj = P - L.parent_first;
  if (L.prep) pj = L.prep[pj];
  const cd* __restrict__ src = static_cast<const cd*>(L.src) + (pj << L.n);
  const uint32_t n2 = sp.n2;
  const uint64_t x0 = ((uint64_t)c * QT + threadIdx.x) * QV;
  if (x0 >= (1ull << n2)) return;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
  // QR rows per step: every load of the step issued before the first use (QR x 32 B in flight)
  constexpr uint32_t QR = 8;
  const char* rp = reinterpret_cast<const char*>(src + x0);   // row y at rp + y * rstride
  const uint64_t rstride = (uint64_t)16 << n2;
  for (uint32_t y0 = 0; y0 < Y; y0 += QR) {
    if (psrc)
      for (uint32_t y = y0 + pf; y < y0 + pf + QR && y < Y; ++y) tq_bulk_prefetch_l2(psrc + ((uint64_t)y << n2), rbytes);
    double px[QR], py[QR], qx[QR], qy[QR];
#pragma unroll
    for (uint32_t i = 0; i < QR; ++i) {   // (Y is a multiple of QR: the launcher checks m >= 3)
      asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                   : "=d"(px[i]), "=d"(py[i]), "=d"(qx[i]), "=d"(qy[i])
                   : "l"(rp));
      rp += rstride;
    }
#pragma unroll
    for (uint32_t i = 0; i < QR; ++i) {
      const cd k = pcoef[y0 + i], h = pcoef[Y + y0 + i];
      a0 = fma(k.x, px[i], fma(-k.y, py[i], a0));
      a1 = fma(k.x, py[i], fma(k.y, px[i], a1));
      a2 = fma(k.x, qx[i], fma(-k.y, qy[i], a2));
      a3 = fma(k.x, qy[i], fma(k.y, qx[i], a3));
      b0 = fma(h.x, px[i], fma(-h.y, py[i], b0));
      b1 = fma(h.x, py[i], fma(h.y, px[i], b1));
      b2 = fma(h.x, qx[i], fma(-h.y, qy[i], b2));
      b3 = fma(h.x, qy[i], fma(h.y, qx[i], b3));
    }
  }
  for (uint32_t ci = 0; ci < nc; ++ci) {
    if (!live[ci]) continue;
    cd r0 = ci ? cd{b0, b1} : cd{a0, a1}, r1 = ci ? cd{b2, b3} : cd{a2, a3};
    for (uint32_t u = sp.nug; u < sp.nug + sp.nux; ++u) {   // D_x: units below the top bits
      for (int v = 0; v < QV; ++v) {
        const uint64_t x = x0 + v;
        const uint32_t idx = (uint32_t)((x >> sp.ua[u]) & 1u) | (uint32_t)(((x >> sp.ub[u]) & 1u) << 1);
        const cd e = {sp.uT[u][2 * idx], sp.uT[u][2 * idx + 1]};
        cd& r = v ? r1 : r0;
        r = {r.x * e.x - r.y * e.y, r.x * e.y + r.y * e.x};
      }
    }
    cd* dst = static_cast<cd*>(L.psi) + ((uint64_t)(s0 + ci) << n2) + x0;
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst), "d"(r0.x), "d"(r0.y), "d"(r1.x), "d"(r1.y)
                 : "memory");
  }
}

// The computed instances (dedup representatives) of a batch, in slot order: the work list of
// the batch's pass kernels (persistent CTAs, no empty CTAs for the shared instances).  The
// leaf level's skipped instances get store-address XOR 0 (their representative is error-free).
// With rows: the representatives whose noise row has no error in the pass (emask bits of the
// row's pass bitmask) go to list, the others to list2 (the clean kernel / the full kernel).
constexpr int CR_T = 1024;   // one CTA: a C2 leaf batch (2,048 slots) in two rounds
__global__ void __launch_bounds__(CR_T) compact_reps_kernel(const uint8_t* __restrict__ err_sel, uint32_t slice_len,
                                                           const uint32_t* __restrict__ rep, uint32_t cnt,
                                                           uint32_t* __restrict__ list, uint32_t* __restrict__ count,
                                                           uint32_t* __restrict__ xlout,
                                                           const uint8_t* __restrict__ rows, uint32_t row_bytes,
                                                           uint32_t emask, uint32_t* __restrict__ list2,
                                                           uint32_t* __restrict__ count2) {
  __shared__ uint32_t wsum[2][CR_T / 32];
  __shared__ uint32_t base[2];
  if (threadIdx.x < 2) base[threadIdx.x] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (uint32_t c0 = 0; c0 < cnt; c0 += blockDim.x) {
    const uint32_t s = c0 + threadIdx.x;
    const bool keep = s < cnt && (!rep || rep[s] == s);
    if (s < cnt && !keep && xlout) xlout[s] = 0u;
    bool err = false;
    if (keep && rows) {
      const uint8_t* row = rows + (uint64_t)s * row_bytes;
      if (err_sel) {   // only the selected gates' errors (the trail's pass A)
        for (uint32_t t = 0; t < slice_len && !err; ++t) err = err_sel[t] && row[4 + t];
      } else {
        err = (*reinterpret_cast<const uint32_t*>(row) & emask) != 0u;
      }
    }
    const bool k0 = keep && !err, k1 = keep && err;
    const unsigned b0 = __ballot_sync(0xffffffffu, k0), b1 = __ballot_sync(0xffffffffu, k1);
    if (lane == 0) {
      wsum[0][w] = __popc(b0);
      wsum[1][w] = __popc(b1);
    }
    __syncthreads();
    uint32_t o0 = base[0], o1 = base[1];
    for (int i = 0; i < w; ++i) {
      o0 += wsum[0][i];
      o1 += wsum[1][i];
    }
    const unsigned below = (1u << lane) - 1u;
    if (k0) list[o0 + __popc(b0 & below)] = s;
    if (k1) list2[o1 + __popc(b1 & below)] = s;
    __syncthreads();
    if (threadIdx.x < 2) {
      uint32_t t = 0;
      for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += wsum[threadIdx.x][i];
      base[threadIdx.x] += t;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *count = base[0];
    if (count2) *count2 = base[1];
  }
}

// The run's seed in device memory: the tree's launches (a replayed CUDA graph) read it
__global__ void set_seed_kernel(uint64_t* d_seed, uint64_t seed) { *d_seed = seed; }

}  // namespace dev

// ------------------------------------------------------------------ launchers
int launch_noise_rows_all(const uint8_t* d_two, const uint8_t* d_pass_of, const NoiseLevels& L,
                          uint64_t total_instances, const uint64_t* d_seed, double p1, double p2,
                          uint8_t* d_rows, void* stream) {
  if (total_instances == 0) return 0;
  const uint64_t threads = total_instances * 32;
  dev::noise_rows_all_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      d_two, d_pass_of, L, total_instances, d_seed, p1, p2, d_rows);
  return (int)cudaGetLastError();
}

int launch_dedup_map(const uint8_t* d_rows, const NoiseLevels& L, uint32_t* d_rep, uint32_t* d_pos,
                     void* stream) {
  dev::dedup_map_kernel<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(d_rows, L, d_rep, d_pos);
  return (int)cudaGetLastError();
}

int launch_dedup_map_level(const uint8_t* d_rows, const NoiseLevels& L, uint32_t d, uint32_t* d_rep,
                           uint32_t* d_pos, void* stream) {
  const uint64_t cnt = L.lv[d].count;
  if (cnt == 0) return 0;
  const unsigned grid = (unsigned)std::min<uint64_t>((cnt + 255) / 256, 4096);
  dev::dedup_map_level_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(d_rows, L, d, d_rep, d_pos);
  return (int)cudaGetLastError();
}

int launch_trail_project(const ProjSpec& spec, const TrailProjLaunch& L, void* stream) {
  static const bool pair = [] {
    const char* e = std::getenv("TQSIM_PROJ_PAIR");   // 0: one CTA per leaf also for arity 2
    return !(e && e[0] == '0');
  }();
  if (pair && L.arity == 2 && spec.m >= 3) {
    const uint64_t per_par = std::max<uint64_t>(1, (1ull << spec.n2) / (dev::QT * dev::QV));
    const uint64_t npar = L.batch ? (L.child_first + L.batch - 1) / 2 - L.child_first / 2 + 1 : 0;
    const uint64_t grid = per_par * npar;
    if (grid == 0) return 0;
    const size_t smem = (size_t)2 * sizeof(double) * 2 << spec.m;
    static const uint32_t pf = [] {   // rows prefetched ahead into L2 (0 = off)
      const char* e = std::getenv("TQSIM_PROJ_PF");
      return e ? (uint32_t)std::atoi(e) : 0u;
    }();
    static const int minb = [] {   // resident CTAs per SM the register budget targets
      const char* e = std::getenv("TQSIM_PROJ_MINB");
      return e ? std::atoi(e) : 3;
    }();
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (minb >= 5) dev::trail_project_pair_kernel<5><<<(unsigned)grid, dev::QT, smem, st>>>(spec, L, pf);
    else if (minb == 4) dev::trail_project_pair_kernel<4><<<(unsigned)grid, dev::QT, smem, st>>>(spec, L, pf);
    else dev::trail_project_pair_kernel<3><<<(unsigned)grid, dev::QT, smem, st>>>(spec, L, pf);
    return (int)cudaGetLastError();
  }
  const uint64_t per_leaf = std::max<uint64_t>(1, (1ull << spec.n2) / (dev::PT * dev::PV));
  const uint64_t grid = per_leaf * L.batch;
  if (grid == 0) return 0;
  dev::trail_project_kernel<<<(unsigned)grid, dev::PT, 0, static_cast<cudaStream_t>(stream)>>>(spec, L, nullptr);
  return (int)cudaGetLastError();
}

int launch_compact_reps(const uint8_t* d_err_sel, uint32_t slice_len,
                        const uint32_t* d_rep, uint32_t cnt, uint32_t* d_list, uint32_t* d_count, uint32_t* d_xlout,
                        const uint8_t* d_rows, uint32_t row_bytes, uint32_t emask, uint32_t* d_list2, uint32_t* d_count2,
                        void* stream) {
  dev::compact_reps_kernel<<<1, dev::CR_T, 0, static_cast<cudaStream_t>(stream)>>>(d_err_sel, slice_len, d_rep, cnt,
                                                                             d_list, d_count, d_xlout,
                                                                             d_rows, row_bytes, emask, d_list2,
                                                                             d_count2);
  return (int)cudaGetLastError();
}

int launch_set_seed(uint64_t* d_seed, uint64_t seed, void* stream) {
  dev::set_seed_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(d_seed, seed);
  return (int)cudaGetLastError();
}

int launch_noise_rows(const uint8_t* d_two, const uint8_t* d_pass_of, uint32_t slice_begin,
                      uint32_t slice_len, uint64_t inst_first, uint32_t count, const uint64_t* d_seed,
                      double p1, double p2, uint32_t row_bytes, uint8_t* d_rows, void* stream) {
  if (count == 0) return 0;
  const uint64_t threads = (uint64_t)count * 32;
  dev::noise_rows_kernel<<<(unsigned)((threads + 255) / 256), 256, 0,
                           static_cast<cudaStream_t>(stream)>>>(
      d_two, d_pass_of, slice_begin, slice_len, inst_first, count, d_seed, p1, p2, row_bytes, d_rows);
  return (int)cudaGetLastError();
}

static dev::SelectOut select_out(const LeafSelect* sel);
int launch_chunk_sums(const double* runsums, uint32_t batch, int n_sim, int chunk_log2,
                      double* sums, void* stream, const LeafSelect* sel, uint64_t leaf_first) {
  const uint64_t grid = (uint64_t)batch << (n_sim - chunk_log2);
  if (grid == 0) return 0;
  dev::chunk_sums_kernel<<<(unsigned)grid, dev::MT, 0, static_cast<cudaStream_t>(stream)>>>(
      runsums, (uint32_t)n_sim, (uint32_t)chunk_log2, sums, leaf_first, select_out(sel));
  return (int)cudaGetLastError();
}

static dev::SelectOut select_out(const LeafSelect* sel) {
  dev::SelectOut so{};
  if (!sel) return so;
  so.dbg_u = sel->dbg_u;
  so.dbg_total = sel->dbg_total;
  so.dbg_flag = sel->dbg_flag;
  so.hsel = sel->hsel;
  so.htarget = sel->htarget;
  so.tgt = sel->tgt;
  so.hi = sel->hi;
  so.hi_shift = sel->hi_shift;
  so.runsel = sel->runsel;
  so.t3 = sel->t3;
  so.tile = sel->tile;
  so.xl = sel->xl;
  so.n_out = sel->n_out;
  for (uint32_t i = 0; i < sel->n_out && i < 32; ++i) so.out_row[i] = sel->out_row[i];
  so.rep = sel->rep;
  return so;
}

int launch_sample(const void* states, const double* runsums, const double* sums, uint32_t batch,
                  int n_sim, int n_user, int chunk_log2, uint64_t leaf_first, const uint64_t* d_seed,
                  double p01, double p10, uint32_t* d_out, void* stream, const LeafSelect* sel) {
  if (batch == 0) return 0;
  dev::sample_kernel<<<batch, dev::MT, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const dev::cd*>(states), runsums, sums, (uint32_t)n_sim, (uint32_t)n_user,
      (uint32_t)chunk_log2, leaf_first, d_seed, p01, p10, d_out, select_out(sel));
  return (int)cudaGetLastError();
}

int launch_sample_finish(const void* scratch, const uint32_t* runsel, const double* t3, uint32_t batch,
                         int n_user, uint64_t leaf_first, const uint64_t* d_seed, double p01, double p10,
                         uint32_t* d_out, void* stream, uint8_t* d_flag, const uint32_t* d_hi, uint32_t hi_shift) {
  if (batch == 0) return 0;
  dev::sample_finish_kernel<<<(batch + dev::MT - 1) / dev::MT, dev::MT, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const dev::cd*>(scratch), runsel, t3, batch, (uint32_t)n_user, leaf_first, d_seed, p01, p10,
      d_out, d_flag, d_hi, hi_shift);
  return (int)cudaGetLastError();
}

int launch_sample_small(const void* states, const double* runsums, uint32_t batch, int n_sim,
                        int n_user, uint64_t leaf_first, const uint64_t* d_seed, double p01, double p10,
                        uint32_t* d_out, void* stream, const LeafSelect* sel) {
  if (batch == 0) return 0;
  dev::sample_small_kernel<<<batch, dev::MT, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const dev::cd*>(states), runsums, (uint32_t)n_sim, (uint32_t)n_user, leaf_first,
      d_seed, p01, p10, d_out, select_out(sel));
  return (int)cudaGetLastError();
}

int launch_philox_debug(const uint32_t* d_in, uint64_t n, uint32_t* d_out) {
  if (n == 0) return 0;
  dev::philox_debug_kernel<<<(unsigned)((n + 255) / 256), 256>>>(d_in, n, d_out);
  return (int)cudaGetLastError();
}

int launch_noise_table(const uint8_t* d_two, uint32_t slice_begin, uint32_t slice_len,
                       uint64_t inst_begin, uint64_t count, uint64_t seed, double p1, double p2,
                       uint8_t* d_out) {
  const uint64_t total = count * slice_len;
  if (total == 0) return 0;
  dev::noise_table_kernel<<<(unsigned)((total + 255) / 256), 256>>>(d_two, slice_begin, slice_len,
                                                                   inst_begin, count, seed, p1, p2,
                                                                   d_out);
  return (int)cudaGetLastError();
}

const char* cuda_error_string(int code) { return cudaGetErrorString((cudaError_t)code); }

}  // namespace tq
