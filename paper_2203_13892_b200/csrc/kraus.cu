// Kraus engine: noisy trajectories with non-Pauli error channels --
// thermal relaxation, amplitude damping, phase damping (§4.3.2, Table 2
// P:479-498; readings R31-R37 in DESIGN.md) -- on top of the depolarizing Pauli draw.
//
// A Kraus choice depends on the trajectory's current state (p_k = ||K_k psi||^2, R35), so
// every noise location is a reduction over the whole state before the next gate may run.
// For the widths the paper studies these channels at (QFT_12, QPE_9, BV_10)
// a state is at most 2^13 complex128 = 128 KiB: it lives in ONE CTA's shared memory for a
// whole subcircuit, and each location costs one block reduction, not an HBM pass.
//
// One CTA = one tree-node instance j (§3): load the parent's state (fused fan-out,
// or |0..0> at the root), then per lowered gate g of the slice
//   1. psi <- (P_g G_g) psi        gate with its keyed depolarizing Pauli (R1, R8)
//   2. the joint |a|^2 table over the gate's qubits (block reduction, fixed order)
//   3. the R33 sequence of Kraus decisions run on that table (the Kraus operators of
//      AD / PD / TR are monomial on the computational basis, so the table after each
//      choice follows classically): r from Philox tag 3/4 (R34), k = smallest with
//      r < p_0 + .. + p_k (R35), each qubit's chosen operators multiplied into one real
//      2x2 M_i with the 1/sqrt(p_k) normalisations
//   4. psi <- (M_0 (x) M_1) psi
// and at the end store the state for the children (HBM), or, at a leaf, sample it in place
// (block scan of |a|^2, smallest x with C(x) > u*total, R9; readout flips, R11).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "tq_device_common.cuh"
#include "tq_internal.h"

namespace tq {
namespace dev {

struct __align__(16) kd2 {
  double x, y;
};

constexpr int KT = 256;   // threads per CTA

__device__ __forceinline__ kd2 kmul(kd2 a, kd2 b) { return kd2{a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
__device__ __forceinline__ kd2 kadd(kd2 a, kd2 b) { return kd2{a.x + b.x, a.y + b.y}; }

// psi <- m psi on qubit q (m row-major complex 2x2)
__device__ __forceinline__ void k_apply_1q(kd2* psi, int n, int q, const kd2 m0, const kd2 m1, const kd2 m2,
                                           const kd2 m3) {
  const uint32_t half = 1u << (n - 1), lowm = (1u << q) - 1u;
  for (uint32_t i = threadIdx.x; i < half; i += blockDim.x) {
    const uint32_t i0 = ((i >> q) << (q + 1)) | (i & lowm), i1 = i0 | (1u << q);
    const kd2 a = psi[i0], b = psi[i1];
    psi[i0] = kadd(kmul(m0, a), kmul(m1, b));
    psi[i1] = kadd(kmul(m2, a), kmul(m3, b));
  }
}

// psi <- m psi on qubit q, m real 2x2
__device__ __forceinline__ void k_apply_real(kd2* psi, int n, int q, double a00, double a01, double a10,
                                             double a11) {
  const uint32_t half = 1u << (n - 1), lowm = (1u << q) - 1u;
  for (uint32_t i = threadIdx.x; i < half; i += blockDim.x) {
    const uint32_t i0 = ((i >> q) << (q + 1)) | (i & lowm), i1 = i0 | (1u << q);
    const kd2 a = psi[i0], b = psi[i1];
    psi[i0] = kd2{a00 * a.x + a01 * b.x, a00 * a.y + a01 * b.y};
    psi[i1] = kd2{a10 * a.x + a11 * b.x, a10 * a.y + a11 * b.y};
  }
}

__device__ __forceinline__ uint32_t k_insert2(uint32_t i, int lo, int hi) {
  i = ((i >> lo) << (lo + 1)) | (i & ((1u << lo) - 1u));
  return ((i >> hi) << (hi + 1)) | (i & ((1u << hi) - 1u));
}

__device__ __forceinline__ void k_apply_cx(kd2* psi, int n, int c, int t) {
  const uint32_t quarter = 1u << (n - 2);
  const int lo = c < t ? c : t, hi = c < t ? t : c;
  for (uint32_t i = threadIdx.x; i < quarter; i += blockDim.x) {
    const uint32_t b = k_insert2(i, lo, hi) | (1u << c), b1 = b | (1u << t);
    const kd2 v = psi[b];
    psi[b] = psi[b1];
    psi[b1] = v;
  }
}

__device__ __forceinline__ void k_apply_cz(kd2* psi, int n, int c, int t) {
  const uint32_t quarter = 1u << (n - 2);
  const int lo = c < t ? c : t, hi = c < t ? t : c;
  for (uint32_t i = threadIdx.x; i < quarter; i += blockDim.x) {
    const uint32_t b = k_insert2(i, lo, hi) | (1u << c) | (1u << t);
    psi[b] = kd2{-psi[b].x, -psi[b].y};
  }
}

// Pauli code 1..3 = X, Y, Z as a complex 2x2 (Y = [[0,-i],[i,0]])
__device__ __forceinline__ void k_pauli(uint32_t c, kd2* m) {
  const kd2 z{0.0, 0.0}, one{1.0, 0.0};
  if (c == 1) { m[0] = z; m[1] = one; m[2] = one; m[3] = z; }
  else if (c == 2) { m[0] = z; m[1] = kd2{0.0, -1.0}; m[2] = kd2{0.0, 1.0}; m[3] = z; }
  else { m[0] = one; m[1] = z; m[2] = z; m[3] = kd2{-1.0, 0.0}; }
}

struct KrausShared {
  double red[KT / 32][4];
  double tbl[4];
  double M[2][4];      // per gate qubit: the chosen operators' product (real 2x2)
  uint32_t code;
  uint32_t flag;
  double scan[KT / 32];
  int pick;
  double before;
};

// Joint |a|^2 table over (bit q0, bit q1): tbl[b0 + 2 b1].  Fixed-order block reduction.
// (goff: the global index of psi[0] -- a cluster CTA's slice, see kraus_cluster_kernel)
__device__ __forceinline__ void k_joint_table(const kd2* psi, int n, int q0, int q1, KrausShared& sh,
                                              uint32_t goff = 0u) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const uint32_t N = 1u << n;
  for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
    const kd2 a = psi[i];
    const uint32_t gi = goff | i;
    const uint32_t k = ((gi >> q0) & 1u) | (((gi >> q1) & 1u) << 1);
    const double p = a.x * a.x + a.y * a.y;
#pragma unroll
    for (int t = 0; t < 4; ++t) acc[t] += (k == (uint32_t)t) ? p : 0.0;
  }
#pragma unroll
  for (int t = 0; t < 4; ++t)
    for (int o = 16; o > 0; o >>= 1) acc[t] += __shfl_xor_sync(0xffffffffu, acc[t], o);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int t = 0; t < 4; ++t) sh.red[w][t] = acc[t];
  __syncthreads();
  if (threadIdx.x < 4) {
    double s = 0.0;
    for (int v = 0; v < (int)(blockDim.x >> 5); ++v) s += sh.red[v][threadIdx.x];
    sh.tbl[threadIdx.x] = s;
  }
  __syncthreads();
}

// R33-R36 on the joint table (thread 0): channels in order TR-amplitude, TR-phase, AD, PD;
// within a channel q0 then q1.  type 0 = amplitude damping set, 1 = phase damping set.
__device__ void k_decide(const KrausArgs& a, uint32_t g, uint64_t j, uint64_t seed, bool two, KrausShared& sh) {
  double P[4] = {sh.tbl[0], sh.tbl[1], sh.tbl[2], sh.tbl[3]};
  double M[2][4] = {{1.0, 0.0, 0.0, 1.0}, {1.0, 0.0, 0.0, 1.0}};
  uint32_t flag = 0;
  const int nq = two ? 2 : 1;
  tq_w4 w[2];
  w[0] = tq_philox_keyed(g, j, 3u, seed);
  w[1] = tq_philox_keyed(g, j, 4u, seed);   // sub-locations 4..7 (AD, PD)
  for (int c = 0; c < 4; ++c) {
    double par;
    int type;
    if (c == 0) { if (!(a.ch_mask & 1u)) continue; par = a.trg[two]; type = 0; }
    else if (c == 1) { if (!(a.ch_mask & 1u)) continue; par = a.trl[two]; type = 1; }
    else if (c == 2) { if (!(a.ch_mask & 2u)) continue; par = a.ad; type = 0; }
    else { if (!(a.ch_mask & 4u)) continue; par = a.pd; type = 1; }
    for (int i = 0; i < nq; ++i) {
      const int s = 2 * c + i;
      const tq_w4& ww = w[s >> 2];
      const uint32_t wv = (s & 3) == 0 ? ww.x : (s & 3) == 1 ? ww.y : (s & 3) == 2 ? ww.z : ww.w;
      const double r = (double)wv * 0x1p-32;
      const int bit = 1 << i;
      double P0 = 0.0, P1 = 0.0;
      for (int k = 0; k < 4; ++k) (k & bit ? P1 : P0) += P[k];
      const double p0 = P0 + (1.0 - par) * P1, p1 = par * P1;
      int kk;
      if (r < p0) kk = 0;
      else if (r < p0 + p1) kk = 1;
      else {   // beyond the total (rounding): the last non-zero operator
        kk = p1 > 0.0 ? 1 : 0;
        flag = 1;
      }
      if (fabs(r - p0) < 1e-9 || fabs(r - (p0 + p1)) < 1e-9) flag = 1;
      const double pk = kk ? p1 : p0, inv = 1.0 / sqrt(pk);
      double K[4];   // the chosen Kraus operator / sqrt(p_k), real 2x2 row-major
      if (kk == 0) {
        K[0] = inv; K[1] = 0.0; K[2] = 0.0; K[3] = sqrt(1.0 - par) * inv;
        for (int k = 0; k < 4; ++k) P[k] = (k & bit ? (1.0 - par) * P[k] : P[k]) / pk;
      } else if (type == 0) {   // amplitude damping K1 = sqrt(g) |0><1|
        K[0] = 0.0; K[1] = sqrt(par) * inv; K[2] = 0.0; K[3] = 0.0;
        for (int k = 0; k < 4; ++k)
          if (k & bit) {
            P[k ^ bit] = par * P[k] / pk;
            P[k] = 0.0;
          }
      } else {                  // phase damping K1 = sqrt(l) |1><1|
        K[0] = 0.0; K[1] = 0.0; K[2] = 0.0; K[3] = sqrt(par) * inv;
        for (int k = 0; k < 4; ++k) P[k] = (k & bit ? par * P[k] : 0.0) / pk;
      }
      // M_i <- K M_i
      const double m0 = M[i][0], m1 = M[i][1], m2 = M[i][2], m3 = M[i][3];
      M[i][0] = K[0] * m0 + K[1] * m2;
      M[i][1] = K[0] * m1 + K[1] * m3;
      M[i][2] = K[2] * m0 + K[3] * m2;
      M[i][3] = K[2] * m1 + K[3] * m3;
    }
  }
  for (int i = 0; i < 2; ++i)
    for (int k = 0; k < 4; ++k) sh.M[i][k] = M[i][k];
  sh.flag |= flag;
}

__global__ void __launch_bounds__(KT) kraus_slice_kernel(const __grid_constant__ KrausArgs a) {
  extern __shared__ kd2 psi[];
  __shared__ KrausShared sh;
  const int n = (int)a.n;
  const uint32_t N = 1u << n;
  const uint32_t s = blockIdx.x;
  const uint64_t j = a.child_first + s;
  const uint64_t seed = *a.seedp;
  const kd2* __restrict__ gsrc = reinterpret_cast<const kd2*>(a.src);
  if (threadIdx.x == 0) sh.flag = 0u;
  // fan-out: the parent's state, or |0..0> at the root
  uint64_t pj = 0;
  if (a.mode == 1) {
    pj = j / a.arity - a.parent_first;
    for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) psi[i] = gsrc[(pj << n) + i];
  } else {
    for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) psi[i] = kd2{i == 0 ? 1.0 : 0.0, 0.0};
  }
  __syncthreads();
  if (threadIdx.x == 0 && a.mode == 1 && a.src_flag) sh.flag = a.src_flag[pj];
  const KGate* __restrict__ G = a.gates;
  for (uint32_t g = a.g0; g < a.g1; ++g) {
    const KGate gt = G[g];
    const bool two = gt.two != 0;
    const uint32_t code = tq_noise_code(g, j, seed, two ? a.p2 : a.p1, two);
    if (!two) {   // P_g G_g as one 2x2 (a Pauli is monomial: exact entries)
      kd2 m[4] = {kd2{gt.m[0], gt.m[1]}, kd2{gt.m[2], gt.m[3]}, kd2{gt.m[4], gt.m[5]}, kd2{gt.m[6], gt.m[7]}};
      if (code) {
        kd2 p[4];
        k_pauli(code, p);
        const kd2 r0 = kadd(kmul(p[0], m[0]), kmul(p[1], m[2])), r1 = kadd(kmul(p[0], m[1]), kmul(p[1], m[3]));
        const kd2 r2 = kadd(kmul(p[2], m[0]), kmul(p[3], m[2])), r3 = kadd(kmul(p[2], m[1]), kmul(p[3], m[3]));
        m[0] = r0; m[1] = r1; m[2] = r2; m[3] = r3;
      }
      k_apply_1q(psi, n, (int)gt.q0, m[0], m[1], m[2], m[3]);
    } else {
      if (gt.op == OP_CX) k_apply_cx(psi, n, (int)gt.q0, (int)gt.q1);
      else k_apply_cz(psi, n, (int)gt.q0, (int)gt.q1);
      if (code) {
        __syncthreads();
        kd2 p[4];
        if (code >> 2) {
          k_pauli(code >> 2, p);
          k_apply_1q(psi, n, (int)gt.q0, p[0], p[1], p[2], p[3]);
          __syncthreads();
        }
        if (code & 3u) {
          k_pauli(code & 3u, p);
          k_apply_1q(psi, n, (int)gt.q1, p[0], p[1], p[2], p[3]);
        }
      }
    }
    __syncthreads();
    // the gate's Kraus channels (R33): one joint table, the decisions, one sweep per qubit
    k_joint_table(psi, n, (int)gt.q0, two ? (int)gt.q1 : (int)gt.q0, sh);
    if (threadIdx.x == 0) k_decide(a, g, j, seed, two, sh);
    __syncthreads();
    k_apply_real(psi, n, (int)gt.q0, sh.M[0][0], sh.M[0][1], sh.M[0][2], sh.M[0][3]);
    if (two) {
      __syncthreads();
      k_apply_real(psi, n, (int)gt.q1, sh.M[1][0], sh.M[1][1], sh.M[1][2], sh.M[1][3]);
    }
    __syncthreads();
  }
  if (!a.leaf || a.store_leaf) {   // the node's state for its children (or a leaf's, for dumps)
    kd2* __restrict__ dst = reinterpret_cast<kd2*>(a.dst) + ((uint64_t)s << n);
    for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) dst[i] = psi[i];
    if (threadIdx.x == 0 && a.dst_flag) a.dst_flag[s] = (uint8_t)sh.flag;
    if (!a.leaf) return;
  }
  // leaf (§2.3, R9): thread t owns amplitudes [t C, (t+1) C); block scan of the chunk sums
  const uint32_t T = blockDim.x, C = (N + T - 1) / T;
  const uint32_t c0 = threadIdx.x * C < N ? threadIdx.x * C : N, c1 = c0 + C < N ? c0 + C : N;
  double loc = 0.0;
  for (uint32_t i = c0; i < c1; ++i) loc += psi[i].x * psi[i].x + psi[i].y * psi[i].y;
  double incl = loc;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    const double v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) sh.scan[w] = incl;
  if (threadIdx.x == 0) sh.pick = (int)T;
  __syncthreads();
  double before = 0.0, total = 0.0;
  for (int v = 0; v < (int)(T >> 5); ++v) {
    if (v < w) before += sh.scan[v];
    total += sh.scan[v];
  }
  incl += before;
  const uint64_t leaf = j;
  const double u = tq_measure_uniform(leaf, seed);
  const double target = u * total;
  if (incl > target) atomicMin(&sh.pick, (int)threadIdx.x);   // the first chunk whose scan exceeds it
  __syncthreads();
  if (threadIdx.x == 0 && sh.pick == (int)T) {   // rounding: the target at the very top -> the last chunk
    int t = 0;
    for (int v = 0; v < (int)T; ++v)
      if ((uint32_t)v * C < N) t = v;
    sh.pick = t;
    sh.flag = 1u;
  }
  __syncthreads();
  if ((int)threadIdx.x != sh.pick) return;
  double c = incl - loc, cb = c, ca = c;
  int x = -1, lastnz = -1;
  for (uint32_t i = c0; i < c1; ++i) {
    const double p = psi[i].x * psi[i].x + psi[i].y * psi[i].y;
    if (p > 0.0) lastnz = (int)i;
    if (x < 0) cb = c;
    c += p;
    if (x < 0 && c > target) {
      x = (int)i;
      ca = c;
    }
  }
  uint32_t flag = sh.flag;
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

// ---------------------------------------------------------------------------------------
// Widths 14..16: the state is spread over a thread-block CLUSTER of CL = 2^(n-13) CTAs, each
// holding a 2^13-amplitude slice (128 KiB) in its shared memory; global index i lives in rank
// i >> 13 at slot i & (2^13 - 1).  Gates on the slice's qubits stay in the CTA; gates on the
// top qubits pair amplitudes across CTAs through distributed shared memory (DSMEM,
// map_shared_rank).  Every gate / Kraus sweep enumerates its pairs globally, CTA r taking the
// r-th contiguous share (for a slice qubit that share is exactly its own slice), with a
// cluster barrier between sweeps.  The joint table: each CTA reduces its slice, then every CTA
// sums the CL partial tables in rank order, so all CTAs hold the same table and take the same
// R33 decisions.  The leaf sample: per-CTA totals summed in rank order, the CTA whose range
// holds u * total finishes the search (R9, R11) -- the same rules as kraus_slice_kernel.
constexpr int KCQ = 13;   // qubits per CTA slice

struct KrausClusterShared {
  KrausShared k;
  double tsum[4];
  double ctot;
  int found;
  kd2* rp[8];   // every rank's slice (generic DSMEM addresses)
};

__device__ __forceinline__ kd2* kc_at(const KrausClusterShared& sh, uint32_t i) {
  return sh.rp[i >> KCQ] + (i & ((1u << KCQ) - 1u));
}

// psi <- m psi on qubit q over the cluster's state (pairs p of CTA rank: [rank per, (rank+1) per))
__device__ __forceinline__ void kc_apply_1q(const KrausClusterShared& sh, int n, uint32_t rank, uint32_t CL, int q,
                                            const kd2 m0, const kd2 m1, const kd2 m2, const kd2 m3) {
  const uint32_t per = (1u << (n - 1)) / CL, lowm = (1u << q) - 1u;
#pragma unroll 4
  for (uint32_t p = rank * per + threadIdx.x; p < (rank + 1) * per; p += blockDim.x) {
    const uint32_t i0 = ((p >> q) << (q + 1)) | (p & lowm), i1 = i0 | (1u << q);
    kd2* A = kc_at(sh, i0);
    kd2* B = kc_at(sh, i1);
    const kd2 a = *A, b = *B;
    *A = kadd(kmul(m0, a), kmul(m1, b));
    *B = kadd(kmul(m2, a), kmul(m3, b));
  }
}

__device__ __forceinline__ void kc_apply_real(const KrausClusterShared& sh, int n, uint32_t rank, uint32_t CL, int q,
                                              double a00, double a01, double a10, double a11) {
  const uint32_t per = (1u << (n - 1)) / CL, lowm = (1u << q) - 1u;
#pragma unroll 4
  for (uint32_t p = rank * per + threadIdx.x; p < (rank + 1) * per; p += blockDim.x) {
    const uint32_t i0 = ((p >> q) << (q + 1)) | (p & lowm), i1 = i0 | (1u << q);
    kd2* A = kc_at(sh, i0);
    kd2* B = kc_at(sh, i1);
    const kd2 a = *A, b = *B;
    *A = kd2{a00 * a.x + a01 * b.x, a00 * a.y + a01 * b.y};
    *B = kd2{a10 * a.x + a11 * b.x, a10 * a.y + a11 * b.y};
  }
}

__device__ __forceinline__ void kc_apply_2q(const KrausClusterShared& sh, int n, uint32_t rank, uint32_t CL, bool cx,
                                            int c, int t) {
  const uint32_t per = (1u << (n - 2)) / CL;
  const int lo = c < t ? c : t, hi = c < t ? t : c;
  for (uint32_t p = rank * per + threadIdx.x; p < (rank + 1) * per; p += blockDim.x) {
    const uint32_t b = k_insert2(p, lo, hi) | (1u << c), b1 = b | (1u << t);
    if (cx) {
      kd2* A = kc_at(sh, b);
      kd2* B = kc_at(sh, b1);
      const kd2 v = *A;
      *A = *B;
      *B = v;
    } else {
      kd2* B = kc_at(sh, b1);
      *B = kd2{-B->x, -B->y};
    }
  }
}

// Dispatch: a sweep on a slice qubit (< 13) touches only the CTA's own slice -- the
// single-CTA sweeps on psi (plain shared-memory accesses); a top qubit goes through DSMEM.
__device__ __forceinline__ void kc_1q(kd2* psi, const KrausClusterShared& sh, int n, uint32_t rank, uint32_t CL, int q,
                                      const kd2 m0, const kd2 m1, const kd2 m2, const kd2 m3) {
  if (q < KCQ) k_apply_1q(psi, KCQ, q, m0, m1, m2, m3);
  else kc_apply_1q(sh, n, rank, CL, q, m0, m1, m2, m3);
}

__device__ __forceinline__ void kc_real(kd2* psi, const KrausClusterShared& sh, int n, uint32_t rank, uint32_t CL,
                                        int q, double a00, double a01, double a10, double a11) {
  if (q < KCQ) k_apply_real(psi, KCQ, q, a00, a01, a10, a11);
  else kc_apply_real(sh, n, rank, CL, q, a00, a01, a10, a11);
}

// CX / CZ: local unless the CX target is a top qubit.  A top control selects whole CTAs (the
// target flip is then a local X: exact, 0 a + 1 b = b); CZ is diagonal (a sign per amplitude).
__device__ __forceinline__ void kc_2q(kd2* psi, const KrausClusterShared& sh, int n, uint32_t rank, uint32_t CL,
                                      uint32_t goff, bool cx, int c, int t) {
  if (!cx) {
    const uint32_t m = (1u << c) | (1u << t);
    for (uint32_t i = threadIdx.x; i < (1u << KCQ); i += blockDim.x)
      if (((goff | i) & m) == m) psi[i] = kd2{-psi[i].x, -psi[i].y};
  } else if (t < KCQ) {
    if (c < KCQ) k_apply_cx(psi, KCQ, c, t);
    else if ((goff >> c) & 1u) k_apply_real(psi, KCQ, t, 0.0, 1.0, 1.0, 0.0);
  } else {
    kc_apply_2q(sh, n, rank, CL, true, c, t);
  }
}

__global__ void __launch_bounds__(KT) kraus_cluster_kernel(const __grid_constant__ KrausArgs a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ kd2 psi[];
  __shared__ KrausClusterShared sh;
  const int n = (int)a.n;
  const uint32_t CL = 1u << (n - KCQ), L = 1u << KCQ;
  const uint32_t rank = cl.block_rank();
  const uint32_t goff = rank << KCQ;
  const uint32_t s = blockIdx.x / CL;
  const uint64_t j = a.child_first + s;
  const uint64_t seed = *a.seedp;
  const kd2* __restrict__ gsrc = reinterpret_cast<const kd2*>(a.src);
  if (threadIdx.x < CL) sh.rp[threadIdx.x] = cl.map_shared_rank(psi, (int)threadIdx.x);
  if (threadIdx.x == 0) sh.k.flag = 0u;
  uint64_t pj = 0;
  if (a.mode == 1) {   // fan-out: this rank's slice of the parent's state
    pj = j / a.arity - a.parent_first;
    for (uint32_t i = threadIdx.x; i < L; i += blockDim.x) psi[i] = gsrc[(pj << n) + goff + i];
  } else {             // |0..0> at the root
    for (uint32_t i = threadIdx.x; i < L; i += blockDim.x) psi[i] = kd2{(goff | i) == 0 ? 1.0 : 0.0, 0.0};
  }
  if (threadIdx.x == 0 && a.mode == 1 && a.src_flag) sh.k.flag = a.src_flag[pj];
  cl.sync();
  const KGate* __restrict__ G = a.gates;
  for (uint32_t g = a.g0; g < a.g1; ++g) {
    const KGate gt = G[g];
    const bool two = gt.two != 0;
    const uint32_t code = tq_noise_code(g, j, seed, two ? a.p2 : a.p1, two);
    if (!two) {
      kd2 m[4] = {kd2{gt.m[0], gt.m[1]}, kd2{gt.m[2], gt.m[3]}, kd2{gt.m[4], gt.m[5]}, kd2{gt.m[6], gt.m[7]}};
      if (code) {
        kd2 p[4];
        k_pauli(code, p);
        const kd2 r0 = kadd(kmul(p[0], m[0]), kmul(p[1], m[2])), r1 = kadd(kmul(p[0], m[1]), kmul(p[1], m[3]));
        const kd2 r2 = kadd(kmul(p[2], m[0]), kmul(p[3], m[2])), r3 = kadd(kmul(p[2], m[1]), kmul(p[3], m[3]));
        m[0] = r0; m[1] = r1; m[2] = r2; m[3] = r3;
      }
      kc_1q(psi, sh, n, rank, CL, (int)gt.q0, m[0], m[1], m[2], m[3]);
    } else {
      kc_2q(psi, sh, n, rank, CL, goff, gt.op == OP_CX, (int)gt.q0, (int)gt.q1);
      if (code) {
        kd2 p[4];
        if (code >> 2) {
          cl.sync();
          k_pauli(code >> 2, p);
          kc_1q(psi, sh, n, rank, CL, (int)gt.q0, p[0], p[1], p[2], p[3]);
        }
        if (code & 3u) {
          cl.sync();
          k_pauli(code & 3u, p);
          kc_1q(psi, sh, n, rank, CL, (int)gt.q1, p[0], p[1], p[2], p[3]);
        }
      }
    }
    cl.sync();
    // the gate's Kraus channels (R33): this slice's partial table, the cluster's sum in rank
    // order (identical in every CTA), the decisions, one sweep per qubit
    k_joint_table(psi, KCQ, (int)gt.q0, two ? (int)gt.q1 : (int)gt.q0, sh.k, goff);
    cl.sync();
    if (threadIdx.x < 4) {
      double t = 0.0;
      for (uint32_t r = 0; r < CL; ++r) t += cl.map_shared_rank(&sh.k.tbl[0], (int)r)[threadIdx.x];
      sh.tsum[threadIdx.x] = t;
    }
    cl.sync();   // every rank has read every partial table
    if (threadIdx.x < 4) sh.k.tbl[threadIdx.x] = sh.tsum[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0) k_decide(a, g, j, seed, two, sh.k);
    __syncthreads();
    kc_real(psi, sh, n, rank, CL, (int)gt.q0, sh.k.M[0][0], sh.k.M[0][1], sh.k.M[0][2], sh.k.M[0][3]);
    if (two) {
      cl.sync();
      kc_real(psi, sh, n, rank, CL, (int)gt.q1, sh.k.M[1][0], sh.k.M[1][1], sh.k.M[1][2], sh.k.M[1][3]);
    }
    cl.sync();
  }
  if (!a.leaf || a.store_leaf) {
    kd2* __restrict__ dst = reinterpret_cast<kd2*>(a.dst) + ((uint64_t)s << n) + goff;
    for (uint32_t i = threadIdx.x; i < L; i += blockDim.x) dst[i] = psi[i];
    if (threadIdx.x == 0 && rank == 0 && a.dst_flag) a.dst_flag[s] = (uint8_t)sh.k.flag;
  }
  if (a.leaf) {
    // leaf (§2.3, R9): thread t of rank r owns global amplitudes goff + [t C, (t+1) C)
    const uint32_t T = blockDim.x, C = L / T;
    const uint32_t c0 = threadIdx.x * C, c1 = c0 + C;
    double loc = 0.0;
    for (uint32_t i = c0; i < c1; ++i) loc += psi[i].x * psi[i].x + psi[i].y * psi[i].y;
    double incl = loc;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      const double v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) sh.k.scan[w] = incl;
    if (threadIdx.x == 0) sh.k.pick = (int)T;
    __syncthreads();
    double before = 0.0, ctot = 0.0;
    for (int v = 0; v < (int)(T >> 5); ++v) {
      if (v < w) before += sh.k.scan[v];
      ctot += sh.k.scan[v];
    }
    if (threadIdx.x == 0) sh.ctot = ctot;
    cl.sync();
    double rbefore = 0.0, total = 0.0;
    for (uint32_t r = 0; r < CL; ++r) {
      const double v = *cl.map_shared_rank(&sh.ctot, (int)r);
      if (r < rank) rbefore += v;
      total += v;
    }
    incl += rbefore + before;
    const uint64_t leaf = j;
    const double u = tq_measure_uniform(leaf, seed);
    const double target = u * total;
    if (incl > target) atomicMin(&sh.k.pick, (int)threadIdx.x);   // this rank's first chunk past it
    __syncthreads();
    if (threadIdx.x == 0) sh.found = sh.k.pick < (int)T ? 1 : 0;
    cl.sync();
    uint32_t win = CL;   // the first rank holding the target
    for (uint32_t r = CL; r-- > 0;)
      if (*cl.map_shared_rank(&sh.found, (int)r)) win = r;
    uint32_t flag = sh.k.flag;
    int pick = sh.k.pick;
    if (win == CL) {   // rounding: the target at the very top -> the last chunk of the last rank
      win = CL - 1;
      pick = (int)T - 1;
      flag = 1u;
    }
    if (rank == win && (int)threadIdx.x == pick) {
      double c = incl - loc, cb = c, ca = c;
      int x = -1, lastnz = -1;
      for (uint32_t i = c0; i < c1; ++i) {
        const double p = psi[i].x * psi[i].x + psi[i].y * psi[i].y;
        if (p > 0.0) lastnz = (int)(goff | i);
        if (x < 0) cb = c;
        c += p;
        if (x < 0 && c > target) {
          x = (int)(goff | i);
          ca = c;
        }
      }
      if (x < 0) {
        x = lastnz >= 0 ? lastnz : (int)(goff | c0);
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
  }
  cl.sync();   // no CTA leaves while another may still read its shared memory
}

}  // namespace dev

int launch_kraus_slice(const KrausArgs& a, uint32_t batch, void* stream) {
  if (batch == 0) return 0;
  const size_t smem = (size_t)16 << a.n;
  static bool attr = false;
  if (!attr) {
    const cudaError_t e = cudaFuncSetAttribute(dev::kraus_slice_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)((size_t)16 << dev::KCQ));
    if (e != cudaSuccess) return (int)e;
    attr = true;
  }
  if (a.n <= (uint32_t)dev::KCQ) {
    dev::kraus_slice_kernel<<<batch, dev::KT, smem, static_cast<cudaStream_t>(stream)>>>(a);
    return (int)cudaGetLastError();
  }
  // 14..16 qubits: one cluster of 2^(n-13) CTAs per instance (state in distributed shared memory)
  const size_t csmem = (size_t)16 << dev::KCQ;
  static bool cattr = false;
  if (!cattr) {
    const cudaError_t e =
        cudaFuncSetAttribute(dev::kraus_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem);
    if (e != cudaSuccess) return (int)e;
    cattr = true;
  }
  const uint32_t CL = 1u << (a.n - dev::KCQ);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(batch * CL);
  cfg.blockDim = dim3(dev::KT);
  cfg.dynamicSmemBytes = csmem;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, dev::kraus_cluster_kernel, a);
  return e != cudaSuccess ? (int)e : (int)cudaGetLastError();
}

}  // namespace tq
