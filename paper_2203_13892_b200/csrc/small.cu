// Small-state tree (SURVEY §8(a) kernel notes, "n <= 10 takes the small_state_tree path";
// DESIGN.md §6.4).  For a state of at most 2^10 amplitudes (16 KiB) the tree's HBM
// passes, noise rows, dedup maps and sampler launches cost more than the arithmetic, so
// one kernel runs the whole tree: one warp per leaf, its state resident in the warp's
// slice of shared memory, recomputing its root-to-leaf path with the INHERITED keys --
// slice d runs with the key j_d of the leaf's level-d ancestor (§3: a node's
// subcircuit with its own noise draws; R7 keying), so every leaf sees exactly the noise
// draws the tree gives it and the outcome is the tree's (oracle: tree.simulate_leaf_flat,
// "per-leaf flat recompute with inherited keys must equal the tree DFS").
//
// Per lowered gate g of slice d (§2.5: one noise location per lowered gate;
// R1 / R8 draw): the 32 lanes draw the keyed Pauli codes of 32 consecutive gates at once
// (one Philox each) and broadcast them by shuffle; a 1q gate runs as the one 2x2 P_g G_g
// (a Pauli is monomial: exact entries), a 2q gate as CX / CZ then the Pauli pair.  Leaf
// (§2.3, R9): lane l owns amplitudes [l C, (l+1) C), C = 2^n / 32; warp scan of the
// chunk sums; target = u53 * total; the smallest x with C(x) > target; readout flips (R11).
#include <cuda_runtime.h>

#include "tq_device_common.cuh"
#include "tq_internal.h"

namespace tq {
namespace dev {

struct __align__(16) sd2 {
  double x, y;
};

__device__ __forceinline__ sd2 smul(sd2 a, sd2 b) { return sd2{a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
__device__ __forceinline__ sd2 sadd(sd2 a, sd2 b) { return sd2{a.x + b.x, a.y + b.y}; }

// Pauli code 1..3 = X, Y, Z as a complex 2x2 (Y = [[0,-i],[i,0]])
__device__ __forceinline__ void s_pauli(uint32_t c, sd2* m) {
  const sd2 z{0.0, 0.0}, one{1.0, 0.0};
  if (c == 1) { m[0] = z; m[1] = one; m[2] = one; m[3] = z; }
  else if (c == 2) { m[0] = z; m[1] = sd2{0.0, -1.0}; m[2] = sd2{0.0, 1.0}; m[3] = z; }
  else { m[0] = one; m[1] = z; m[2] = z; m[3] = sd2{-1.0, 0.0}; }
}

// psi <- m psi on qubit q, by the warp (pairs i0 = i with bit q clear, i1 = i0 | 2^q)
__device__ __forceinline__ void s_apply_1q(sd2* psi, uint32_t half, uint32_t lane, int q, const sd2* m) {
  const uint32_t lowm = (1u << q) - 1u;
  for (uint32_t i = lane; i < half; i += 32u) {
    const uint32_t i0 = ((i >> q) << (q + 1)) | (i & lowm), i1 = i0 | (1u << q);
    const sd2 a = psi[i0], b = psi[i1];
    psi[i0] = sadd(smul(m[0], a), smul(m[1], b));
    psi[i1] = sadd(smul(m[2], a), smul(m[3], b));
  }
}

__device__ __forceinline__ uint32_t s_insert2(uint32_t i, int lo, int hi) {
  i = ((i >> lo) << (lo + 1)) | (i & ((1u << lo) - 1u));
  return ((i >> hi) << (hi + 1)) | (i & ((1u << hi) - 1u));
}

__global__ void __launch_bounds__(SMALL_TREE_WARPS * 32) small_tree_kernel(const __grid_constant__ SmallTreeArgs a) {
  extern __shared__ sd2 sm[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const uint64_t k = (uint64_t)blockIdx.x * SMALL_TREE_WARPS + warp;
  if (k >= a.leaf_count) return;   // whole warps exit; only __syncwarp below
  const uint64_t leaf = a.leaf_first + k;
  const int n = (int)a.n;
  const uint32_t N = 1u << n, half = N >> 1, quarter = N >> 2;
  sd2* psi = sm + ((size_t)warp << n);
  const uint64_t seed = *a.seedp;
  for (uint32_t i = lane; i < N; i += 32u) psi[i] = sd2{i == 0 ? 1.0 : 0.0, 0.0};   // |0..0>
  __syncwarp();
  const KGate* __restrict__ G = a.gates;
  for (uint32_t d = 0; d < a.levels; ++d) {
    uint64_t j = leaf;   // the level-d ancestor: j_d = leaf / prod_{e > d} A_e
    for (uint32_t e = a.levels - 1; e > d; --e) j /= a.arity[e];
    const uint32_t g0 = a.bounds[d], g1 = a.bounds[d + 1];
    for (uint32_t gb = g0; gb < g1; gb += 32u) {
      const uint32_t gl = gb + lane;
      uint32_t mycode = 0u;
      if (gl < g1) {
        const bool tw = G[gl].two != 0u;
        mycode = tq_noise_code(gl, j, seed, tw ? a.p2 : a.p1, tw);
      }
      const uint32_t cnt = min(32u, g1 - gb);
      for (uint32_t t = 0; t < cnt; ++t) {
        const uint32_t code = __shfl_sync(0xffffffffu, mycode, (int)t);
        const KGate& gt = G[gb + t];
        if (!gt.two) {   // P_g G_g as one 2x2
          sd2 m[4] = {sd2{gt.m[0], gt.m[1]}, sd2{gt.m[2], gt.m[3]}, sd2{gt.m[4], gt.m[5]}, sd2{gt.m[6], gt.m[7]}};
          if (code) {
            sd2 p[4];
            s_pauli(code, p);
            const sd2 r0 = sadd(smul(p[0], m[0]), smul(p[1], m[2])), r1 = sadd(smul(p[0], m[1]), smul(p[1], m[3]));
            const sd2 r2 = sadd(smul(p[2], m[0]), smul(p[3], m[2])), r3 = sadd(smul(p[2], m[1]), smul(p[3], m[3]));
            m[0] = r0; m[1] = r1; m[2] = r2; m[3] = r3;
          }
          s_apply_1q(psi, half, lane, (int)gt.q0, m);
        } else {
          const int c = (int)gt.q0, tq = (int)gt.q1;
          const int lo = c < tq ? c : tq, hi = c < tq ? tq : c;
          if (gt.op == OP_CX) {
            for (uint32_t i = lane; i < quarter; i += 32u) {
              const uint32_t b = s_insert2(i, lo, hi) | (1u << c), b1 = b | (1u << tq);
              const sd2 v = psi[b];
              psi[b] = psi[b1];
              psi[b1] = v;
            }
          } else {   // CZ
            for (uint32_t i = lane; i < quarter; i += 32u) {
              const uint32_t b = s_insert2(i, lo, hi) | (1u << c) | (1u << tq);
              psi[b] = sd2{-psi[b].x, -psi[b].y};
            }
          }
          if (code) {   // the Pauli pair after the gate: q0 = code >> 2, q1 = code & 3
            sd2 p[4];
            if (code >> 2) {
              __syncwarp();
              s_pauli(code >> 2, p);
              s_apply_1q(psi, half, lane, c, p);
            }
            if (code & 3u) {
              __syncwarp();
              s_pauli(code & 3u, p);
              s_apply_1q(psi, half, lane, tq, p);
            }
          }
        }
        __syncwarp();
      }
    }
  }
  // leaf sampling (R9): lane chunks of C amplitudes, warp inclusive scan of the chunk sums
  const uint32_t C = N >> 5;
  const uint32_t c0 = lane * C;
  double loc = 0.0;
  for (uint32_t i = c0; i < c0 + C; ++i) loc += psi[i].x * psi[i].x + psi[i].y * psi[i].y;
  double incl = loc;
  for (int o = 1; o < 32; o <<= 1) {
    const double v = __shfl_up_sync(0xffffffffu, incl, o);
    if ((int)lane >= o) incl += v;
  }
  const double total = __shfl_sync(0xffffffffu, incl, 31);
  const double u = tq_measure_uniform(leaf, seed);
  const double target = u * total;
  const uint32_t over = __ballot_sync(0xffffffffu, incl > target);
  uint32_t flag = 0u;
  uint32_t pick;
  if (over) {
    pick = (uint32_t)(__ffs(over) - 1);
  } else {   // rounding: the target at the very top -> the last chunk
    pick = 31u;
    flag = 1u;
  }
  if (lane != pick) return;
  double c = incl - loc, cb = c, ca = c;
  int x = -1, lastnz = -1;
  for (uint32_t i = c0; i < c0 + C; ++i) {
    const double p = psi[i].x * psi[i].x + psi[i].y * psi[i].y;
    if (p > 0.0) lastnz = (int)i;
    if (x < 0) cb = c;
    c += p;
    if (x < 0 && c > target) {
      x = (int)i;
      ca = c;
    }
  }
  if (x < 0) {
    x = lastnz >= 0 ? lastnz : (int)c0;
    flag = 1u;
  } else if (target - cb < 1e-9 || ca - target < 1e-9) {
    flag = 1u;
  }
  uint32_t mask = 0;
  if (a.p01 > 0.0 || a.p10 > 0.0) {
    tq_w4 rw = {0, 0, 0, 0};
    for (uint32_t b = 0; b < a.n_user; ++b) {
      if ((b & 3u) == 0) rw = tq_philox_keyed(b >> 2, leaf, 2u, seed);
      const uint32_t wv = (b & 3u) == 0 ? rw.x : (b & 3u) == 1 ? rw.y : (b & 3u) == 2 ? rw.z : rw.w;
      const double p = (((uint32_t)x >> b) & 1u) ? a.p10 : a.p01;
      if ((double)wv * 0x1p-32 < p) mask |= 1u << b;
    }
  }
  a.out[leaf] = (uint32_t)x ^ mask;
  if (a.dbg_u) a.dbg_u[leaf] = u;
  if (a.dbg_total) a.dbg_total[leaf] = total;
  if (a.dbg_flag) a.dbg_flag[leaf] = (uint8_t)flag;
}

}  // namespace dev

int launch_small_tree(const SmallTreeArgs& a, void* stream) {
  if (a.leaf_count == 0) return 0;
  if (a.n < 5 || a.n > TQSIM_SMALL_MAX_QUBITS) return (int)cudaErrorInvalidValue;
  const size_t smem = (size_t)SMALL_TREE_WARPS * ((size_t)16 << a.n);
  static bool attr = false;
  if (!attr) {
    const cudaError_t e =
        cudaFuncSetAttribute(dev::small_tree_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)((size_t)SMALL_TREE_WARPS * ((size_t)16 << TQSIM_SMALL_MAX_QUBITS)));
    if (e != cudaSuccess) return (int)e;
    attr = true;
  }
  const uint64_t blocks = (a.leaf_count + SMALL_TREE_WARPS - 1) / SMALL_TREE_WARPS;
  if (blocks > 0x7FFFFFFFull) return (int)cudaErrorInvalidConfiguration;
  dev::small_tree_kernel<<<(unsigned)blocks, SMALL_TREE_WARPS * 32, smem, static_cast<cudaStream_t>(stream)>>>(a);
  return (int)cudaGetLastError();
}

}  // namespace tq
