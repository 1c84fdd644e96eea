// sm_100a kernels of the TQSim hot path.
//
//  pass_kernel<K>   one HBM pass of a slice over a batch of complex128 states:
//                   stage a 2^K-amplitude tile (tile qubits = pass.tile_q),
//                   run the pass's register phases (16 amplitudes / thread,
//                   4 tile qubits in registers, re-shuffled through an
//                   XOR-swizzled shared-memory tile between phases), apply
//                   every gate of the pass with its keyed Pauli error folded in
//                   (§2.5; readings R1, R7, R8), write back.
//                   The first pass of a node reads its PARENT's state (fan-out
//                   fused with the copy, P:310 state copy) or synthesizes
//                   |0..0> for level 0 (the root).
//  chunk_sums       |a|^2 sums of 2^C-amplitude contiguous chunks (leaf states)
//  sample_kernel    one CTA per leaf: warp-shuffle block scan over the chunk
//                   sums -> chunk, re-read chunk, block scan -> smallest x with
//                   C(x) > u*total (§2.3, R9), readout flips (R11).
//
// No tensor cores: the work is not a dense contraction (BASELINE north_star).
#include <cuda_runtime.h>

#include "tq_internal.h"

namespace tq {
namespace dev {

// ------------------------------------------------------------------ Philox4x32-10
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k.x += W0;
      k.y += W1;
    }
    const uint32_t lo0 = M0 * c.x, hi0 = __umulhi(M0, c.x);
    const uint32_t lo1 = M1 * c.z, hi1 = __umulhi(M1, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

__device__ __forceinline__ uint2 seed_key(uint64_t seed) {
  return make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
}

// Keyed depolarizing draw of lowered gate g at node instance j (R1, R7, R8):
// 0 = no error, else Pauli code 1..3 (1q) / 1..15 (2q; q0 = code>>2, q1 = code&3).
__device__ __forceinline__ uint32_t noise_code(uint32_t g, uint64_t j, uint64_t seed, double p,
                                               bool two) {
  if (!(p > 0.0)) return 0;
  const uint4 w = philox4x32_10(make_uint4(g, (uint32_t)j, 0u, (uint32_t)(j >> 32)), seed_key(seed));
  if (!((double)w.x * 0x1p-32 < p)) return 0;
  return 1u + __umulhi(w.y, two ? 15u : 3u);
}

// ------------------------------------------------------------------ complex helpers
__device__ __forceinline__ double2 cmad2(double2 m0, double2 x, double2 m1, double2 y) {
  // m0*x + m1*y
  double2 r;
  r.x = fma(m0.x, x.x, fma(-m0.y, x.y, fma(m1.x, y.x, -m1.y * y.y)));
  r.y = fma(m0.x, x.y, fma(m0.y, x.x, fma(m1.x, y.y, m1.y * y.x)));
  return r;
}
__device__ __forceinline__ double2 cmul(double2 m, double2 x) {
  return make_double2(fma(m.x, x.x, -m.y * x.y), fma(m.x, x.y, m.y * x.x));
}
__device__ __forceinline__ double2 mul_i(double2 v) { return make_double2(-v.y, v.x); }
__device__ __forceinline__ double2 mul_mi(double2 v) { return make_double2(v.y, -v.x); }
__device__ __forceinline__ double2 neg(double2 v) { return make_double2(-v.x, -v.y); }

constexpr int NA = 1 << RBITS;   // amplitudes per thread

template <int B>
__device__ __forceinline__ void apply_gen(double2 (&a)[NA], double2 m00, double2 m01, double2 m10,
                                          double2 m11) {
#pragma unroll
  for (int k = 0; k < NA; ++k)
    if (!(k & (1 << B))) {
      const double2 x = a[k], y = a[k | (1 << B)];
      a[k] = cmad2(m00, x, m01, y);
      a[k | (1 << B)] = cmad2(m10, x, m11, y);
    }
}
template <int B>
__device__ __forceinline__ void apply_diag(double2 (&a)[NA], double2 d0, double2 d1, bool d0_one) {
#pragma unroll
  for (int k = 0; k < NA; ++k) {
    if (k & (1 << B)) a[k] = cmul(d1, a[k]);
    else if (!d0_one) a[k] = cmul(d0, a[k]);
  }
}
template <int C, int T>
__device__ __forceinline__ void apply_cx(double2 (&a)[NA]) {
#pragma unroll
  for (int k = 0; k < NA; ++k)
    if ((k & (1 << C)) && !(k & (1 << T))) {
      const double2 t = a[k];
      a[k] = a[k | (1 << T)];
      a[k | (1 << T)] = t;
    }
}
template <int C, int T>
__device__ __forceinline__ void apply_cz(double2 (&a)[NA]) {
#pragma unroll
  for (int k = 0; k < NA; ++k)
    if ((k & (1 << C)) && (k & (1 << T))) a[k] = neg(a[k]);
}
template <int B>
__device__ __forceinline__ void apply_pauli(double2 (&a)[NA], uint32_t p) {
  if (p == 0) return;
#pragma unroll
  for (int k = 0; k < NA; ++k)
    if (!(k & (1 << B))) {
      const double2 x = a[k], y = a[k | (1 << B)];
      if (p == 1) {            // X
        a[k] = y;
        a[k | (1 << B)] = x;
      } else if (p == 2) {     // Y = [[0,-i],[i,0]]
        a[k] = mul_mi(y);
        a[k | (1 << B)] = mul_i(x);
      } else {                 // Z
        a[k | (1 << B)] = neg(y);
      }
    }
}

__device__ __forceinline__ void gen_dispatch(double2 (&a)[NA], int b, double2 m00, double2 m01,
                                             double2 m10, double2 m11) {
  switch (b) {
    case 0: apply_gen<0>(a, m00, m01, m10, m11); break;
    case 1: apply_gen<1>(a, m00, m01, m10, m11); break;
    case 2: apply_gen<2>(a, m00, m01, m10, m11); break;
    default: apply_gen<3>(a, m00, m01, m10, m11); break;
  }
}
__device__ __forceinline__ void diag_dispatch(double2 (&a)[NA], int b, double2 d0, double2 d1) {
  const bool one = d0.x == 1.0 && d0.y == 0.0;
  switch (b) {
    case 0: apply_diag<0>(a, d0, d1, one); break;
    case 1: apply_diag<1>(a, d0, d1, one); break;
    case 2: apply_diag<2>(a, d0, d1, one); break;
    default: apply_diag<3>(a, d0, d1, one); break;
  }
}
__device__ __forceinline__ void pauli_dispatch(double2 (&a)[NA], int b, uint32_t p) {
  switch (b) {
    case 0: apply_pauli<0>(a, p); break;
    case 1: apply_pauli<1>(a, p); break;
    case 2: apply_pauli<2>(a, p); break;
    default: apply_pauli<3>(a, p); break;
  }
}
#define TQ_CASE2(F, C, T) case (C * 4 + T): F<C, T>(a); break;
__device__ __forceinline__ void cx_dispatch(double2 (&a)[NA], int c, int t) {
  switch (c * 4 + t) {
    TQ_CASE2(apply_cx, 0, 1) TQ_CASE2(apply_cx, 0, 2) TQ_CASE2(apply_cx, 0, 3)
    TQ_CASE2(apply_cx, 1, 0) TQ_CASE2(apply_cx, 1, 2) TQ_CASE2(apply_cx, 1, 3)
    TQ_CASE2(apply_cx, 2, 0) TQ_CASE2(apply_cx, 2, 1) TQ_CASE2(apply_cx, 2, 3)
    TQ_CASE2(apply_cx, 3, 0) TQ_CASE2(apply_cx, 3, 1) TQ_CASE2(apply_cx, 3, 2)
    default: break;
  }
}
__device__ __forceinline__ void cz_dispatch(double2 (&a)[NA], int c, int t) {
  if (c > t) { const int s = c; c = t; t = s; }
  switch (c * 4 + t) {
    TQ_CASE2(apply_cz, 0, 1) TQ_CASE2(apply_cz, 0, 2) TQ_CASE2(apply_cz, 0, 3)
    TQ_CASE2(apply_cz, 1, 2) TQ_CASE2(apply_cz, 1, 3) TQ_CASE2(apply_cz, 2, 3)
    default: break;
  }
}

// Apply one op (gate + its keyed Pauli error) to the register tile.
__device__ __forceinline__ void apply_op(double2 (&a)[NA], const OpDesc od, uint32_t code,
                                         const double2* __restrict__ mats) {
  if (od.type == OP_CX || od.type == OP_CZ) {
    if (od.type == OP_CX) cx_dispatch(a, od.ra, od.rb);
    else cz_dispatch(a, od.ra, od.rb);
    if (code) {
      pauli_dispatch(a, od.ra, code >> 2);
      pauli_dispatch(a, od.rb, code & 3u);
    }
    return;
  }
  const double2* m = mats + 4ull * od.gate;
  double2 m00 = __ldg(m), m01 = __ldg(m + 1), m10 = __ldg(m + 2), m11 = __ldg(m + 3);
  if (od.type == OP_DIAG && code == 0) {
    diag_dispatch(a, od.ra, m00, m11);
    return;
  }
  // P . M: X swaps rows, Z negates row 1, Y: row0 <- -i row1, row1 <- i row0 (exact)
  if (code == 1) {
    double2 t0 = m00, t1 = m01;
    m00 = m10; m01 = m11; m10 = t0; m11 = t1;
  } else if (code == 2) {
    double2 t0 = m00, t1 = m01;
    m00 = mul_mi(m10); m01 = mul_mi(m11); m10 = mul_i(t0); m11 = mul_i(t1);
  } else if (code == 3) {
    m10 = neg(m10); m11 = neg(m11);
  }
  gen_dispatch(a, od.ra, m00, m01, m10, m11);
}

// XOR swizzle of a tile-local index: bank group (low 3 bits, 16-byte units)
// ^= XOR of the higher 3-bit groups.  Linear over GF(2).
__device__ __forceinline__ uint32_t swz(uint32_t i) {
  return i ^ (((i >> 3) ^ (i >> 6) ^ (i >> 9) ^ (i >> 12)) & 7u);
}

struct KArgs {
  const double2* src;
  double2* dst;
  const OpDesc* ops;
  const PhaseDesc* phases;
  const double2* mats;
  uint64_t seed;
  double p1, p2;
  uint64_t child_first, parent_first;
  uint32_t arity, batch, src_mode, n, n_out;
  uint32_t phase_begin, phase_end, op_begin, op_end;
  uint8_t tile_q[MAX_K];
  uint8_t out_q[32];
};

#ifndef TQ_PASS_MINB
#define TQ_PASS_MINB(K) 1
#endif

template <int K>
__global__ void __launch_bounds__(1 << (K - RBITS), TQ_PASS_MINB(K)) pass_kernel(const KArgs a) {
  constexpr int T = 1 << (K - RBITS);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* tile = reinterpret_cast<double2*>(smem_raw);
  uint8_t* codes = smem_raw + (sizeof(double2) << K);

  const uint32_t tid = threadIdx.x;
  const uint64_t bid = blockIdx.x;
  const uint32_t s = (uint32_t)(bid % a.batch);
  const uint64_t t = bid / a.batch;
  const uint64_t inst = a.child_first + s;

  uint32_t gtile = 0;
  for (uint32_t i = 0; i < a.n_out; ++i) gtile |= (uint32_t)((t >> i) & 1u) << a.out_q[i];

  const uint32_t nops = a.op_end - a.op_begin;
  for (uint32_t i = tid; i < nops; i += T) {
    const OpDesc od = a.ops[a.op_begin + i];
    codes[i] = (uint8_t)noise_code(od.gate, inst, a.seed, od.two ? a.p2 : a.p1, od.two != 0);
  }

  double2* dst = a.dst + ((uint64_t)s << a.n);
  const double2* src = dst;
  if (a.src_mode == 1) src = a.src + ((inst / a.arity - a.parent_first) << a.n);
  __syncthreads();

  double2 amp[NA];
  for (uint32_t ph = a.phase_begin; ph < a.phase_end; ++ph) {
    const PhaseDesc P = a.phases[ph];
    const bool first = ph == a.phase_begin, last = ph + 1 == a.phase_end;
    uint32_t lb = 0;
#pragma unroll
    for (int m = 0; m < K - RBITS; ++m) lb |= ((tid >> m) & 1u) << P.tpos[m];
    if (first) {
      uint32_t gb = gtile;
#pragma unroll
      for (int m = 0; m < K - RBITS; ++m) gb |= ((tid >> m) & 1u) << a.tile_q[P.tpos[m]];
      uint32_t gr[RBITS];
#pragma unroll
      for (int b = 0; b < RBITS; ++b) gr[b] = 1u << a.tile_q[P.rpos[b]];
#pragma unroll
      for (int k = 0; k < NA; ++k) {
        uint32_t g = gb;
#pragma unroll
        for (int b = 0; b < RBITS; ++b)
          if (k & (1 << b)) g |= gr[b];
        if (a.src_mode == 0) amp[k] = make_double2(g == 0 ? 1.0 : 0.0, 0.0);
        else amp[k] = src[g];
      }
    } else {
      __syncthreads();
      const uint32_t sb = swz(lb);
      uint32_t sr[RBITS];
#pragma unroll
      for (int b = 0; b < RBITS; ++b) sr[b] = swz(1u << P.rpos[b]);
#pragma unroll
      for (int k = 0; k < NA; ++k) {
        uint32_t o = sb;
#pragma unroll
        for (int b = 0; b < RBITS; ++b)
          if (k & (1 << b)) o ^= sr[b];
        amp[k] = tile[o];
      }
      __syncthreads();
    }
    for (uint32_t i = P.op_begin; i < P.op_end; ++i)
      apply_op(amp, a.ops[i], codes[i - a.op_begin], a.mats);
    if (last) {
      uint32_t gb = gtile;
#pragma unroll
      for (int m = 0; m < K - RBITS; ++m) gb |= ((tid >> m) & 1u) << a.tile_q[P.tpos[m]];
      uint32_t gr[RBITS];
#pragma unroll
      for (int b = 0; b < RBITS; ++b) gr[b] = 1u << a.tile_q[P.rpos[b]];
#pragma unroll
      for (int k = 0; k < NA; ++k) {
        uint32_t g = gb;
#pragma unroll
        for (int b = 0; b < RBITS; ++b)
          if (k & (1 << b)) g |= gr[b];
        dst[g] = amp[k];
      }
    } else {
      const uint32_t sb = swz(lb);
      uint32_t sr[RBITS];
#pragma unroll
      for (int b = 0; b < RBITS; ++b) sr[b] = swz(1u << P.rpos[b]);
#pragma unroll
      for (int k = 0; k < NA; ++k) {
        uint32_t o = sb;
#pragma unroll
        for (int b = 0; b < RBITS; ++b)
          if (k & (1 << b)) o ^= sr[b];
        tile[o] = amp[k];
      }
    }
  }
}

// ------------------------------------------------------------------ measurement
constexpr int MT = 256;   // threads of the measurement kernels

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = threadIdx.x < (MT >> 5) ? red[threadIdx.x] : 0.0;
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

__global__ void __launch_bounds__(MT) chunk_sums_kernel(const double2* __restrict__ states,
                                                        uint32_t n, uint32_t chunk_log2,
                                                        double* __restrict__ sums) {
  __shared__ double red[MT / 32];
  const uint64_t n_chunks = 1ull << (n - chunk_log2);
  const uint64_t bid = blockIdx.x;
  const uint64_t s = bid >> (n - chunk_log2), c = bid & (n_chunks - 1);
  const double2* p = states + (s << n) + (c << chunk_log2);
  double acc = 0.0;
  for (uint32_t i = threadIdx.x; i < (1u << chunk_log2); i += MT) {
    const double2 v = p[i];
    acc = fma(v.x, v.x, fma(v.y, v.y, acc));
  }
  const double tot = block_sum(acc, red);
  if (threadIdx.x == 0) sums[bid] = tot;
}

__global__ void __launch_bounds__(MT) sample_kernel(const double2* __restrict__ states,
                                                    const double* __restrict__ sums, uint32_t n,
                                                    uint32_t n_user, uint32_t chunk_log2,
                                                    uint64_t leaf_first, uint64_t seed, double p01,
                                                    double p10, uint32_t* __restrict__ out) {
  __shared__ double wsum[MT / 32];
  __shared__ int first_sh;
  __shared__ uint64_t pick_sh;
  __shared__ double before_sh;
  const uint32_t s = blockIdx.x;
  const uint64_t leaf = leaf_first + s;
  const uint64_t nc = 1ull << (n - chunk_log2);
  const double* cs = sums + (uint64_t)s * nc;
  const double2* st = states + ((uint64_t)s << n);

  // u53 (R9): ((w0 >> 5) 2^26 + (w1 >> 6)) 2^-53 from Philox(ctr = (0, leaf, 1, 0))
  const uint4 w = philox4x32_10(make_uint4(0u, (uint32_t)leaf, 1u, (uint32_t)(leaf >> 32)),
                                seed_key(seed));
  const double u = ((double)(w.x >> 5) * 67108864.0 + (double)(w.y >> 6)) * 0x1p-53;

  // (a) chunk selection over contiguous per-thread ranges of chunk sums
  const uint64_t per = (nc + MT - 1) / MT;
  const uint64_t c0 = per * threadIdx.x < nc ? per * threadIdx.x : nc;
  const uint64_t c1 = c0 + per < nc ? c0 + per : nc;
  double loc = 0.0;
  for (uint64_t c = c0; c < c1; ++c) loc += cs[c];
  double incl = block_incl_scan(loc, wsum);
  __shared__ double total_sh;
  if (threadIdx.x == MT - 1) total_sh = incl;
  __syncthreads();
  const double target = u * total_sh;
  int tsel = block_first(incl > target, &first_sh);
  if (threadIdx.x == 0) { pick_sh = ~0ull; before_sh = 0.0; }
  __syncthreads();
  if ((int)threadIdx.x == tsel) {
    double acc = incl - loc;
    uint64_t pick = ~0ull;
    for (uint64_t c = c0; c < c1; ++c) {
      if (acc + cs[c] > target) { pick = c; break; }
      acc += cs[c];
    }
    if (pick == ~0ull) {   // rounding: take the last non-empty chunk of the range
      acc = incl - loc;
      for (uint64_t c = c0; c < c1; ++c)
        if (cs[c] > 0.0) pick = c;
      for (uint64_t c = c0; c < pick; ++c) acc += cs[c];
    }
    pick_sh = pick;
    before_sh = acc;
  }
  __syncthreads();
  uint64_t chunk = pick_sh;
  if (chunk == ~0ull) {   // target beyond total (rounding): last non-empty chunk
    if (threadIdx.x == 0) {
      uint64_t c = nc;
      double acc = 0.0;
      for (uint64_t i = 0; i < nc; ++i)
        if (cs[i] > 0.0) c = i;
      for (uint64_t i = 0; i < c && c < nc; ++i) acc += cs[i];
      pick_sh = c < nc ? c : nc - 1;
      before_sh = acc;
    }
    __syncthreads();
    chunk = pick_sh;
  }
  const double target2 = target - before_sh;

  // (b) within the chunk: per-thread contiguous runs of |a|^2
  const uint32_t clen = 1u << chunk_log2;
  const uint32_t per2 = (clen + MT - 1) / MT;
  const uint32_t e0 = min(clen, per2 * threadIdx.x), e1 = min(clen, e0 + per2);
  const double2* cp = st + (chunk << chunk_log2);
  double loc2 = 0.0;
  for (uint32_t e = e0; e < e1; ++e) {
    const double2 v = cp[e];
    loc2 += v.x * v.x + v.y * v.y;
  }
  const double incl2 = block_incl_scan(loc2, wsum);
  const int tsel2 = block_first(incl2 > target2, &first_sh);
  __shared__ int64_t x_sh;
  if (threadIdx.x == 0) x_sh = -1;
  __syncthreads();
  if ((int)threadIdx.x == (tsel2 < MT ? tsel2 : -1)) {
    double acc = incl2 - loc2;
    int64_t x = -1;
    for (uint32_t e = e0; e < e1; ++e) {
      const double2 v = cp[e];
      acc += v.x * v.x + v.y * v.y;
      if (acc > target2) { x = e; break; }
    }
    if (x < 0)
      for (uint32_t e = e0; e < e1; ++e) {
        const double2 v = cp[e];
        if (v.x * v.x + v.y * v.y > 0.0) x = e;
      }
    x_sh = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t x = x_sh;
    if (x < 0) {   // fall back to the last non-zero amplitude of the chunk
      for (uint32_t e = 0; e < clen; ++e) {
        const double2 v = cp[e];
        if (v.x * v.x + v.y * v.y > 0.0) x = e;
      }
      if (x < 0) x = 0;
    }
    const uint32_t xi = (uint32_t)((chunk << chunk_log2) + (uint64_t)x);
    // readout (R11): bit b flips iff word (b&3) of Philox(ctr=(b>>2, leaf, 2, 0)) * 2^-32 < p
    uint32_t mask = 0;
    if (p01 > 0.0 || p10 > 0.0) {
      uint4 rw = make_uint4(0, 0, 0, 0);
      for (uint32_t b = 0; b < n_user; ++b) {
        if ((b & 3u) == 0)
          rw = philox4x32_10(make_uint4(b >> 2, (uint32_t)leaf, 2u, (uint32_t)(leaf >> 32)),
                             seed_key(seed));
        const uint32_t wv = (b & 3u) == 0 ? rw.x : (b & 3u) == 1 ? rw.y : (b & 3u) == 2 ? rw.z : rw.w;
        const double p = ((xi >> b) & 1u) ? p10 : p01;
        if ((double)wv * 0x1p-32 < p) mask |= 1u << b;
      }
    }
    out[leaf] = xi ^ mask;
  }
}

// ------------------------------------------------------------------ debug hooks
__global__ void philox_debug_kernel(const uint32_t* in, uint64_t n, uint32_t* out) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t* v = in + 6 * i;
  const uint4 r = philox4x32_10(make_uint4(v[0], v[1], v[2], v[3]), make_uint2(v[4], v[5]));
  out[4 * i + 0] = r.x; out[4 * i + 1] = r.y; out[4 * i + 2] = r.z; out[4 * i + 3] = r.w;
}

__global__ void noise_table_kernel(const uint8_t* two, uint32_t slice_begin, uint32_t slice_len,
                                   uint64_t inst_begin, uint64_t count, uint64_t seed, double p1,
                                   double p2, uint8_t* out) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= count * slice_len) return;
  const uint64_t inst = inst_begin + i / slice_len;
  const uint32_t t = (uint32_t)(i % slice_len);
  const bool tw = two[t] != 0;
  out[i] = (uint8_t)noise_code(slice_begin + t, inst, seed, tw ? p2 : p1, tw);
}

}  // namespace dev

// ------------------------------------------------------------------ launchers
namespace {

template <int K>
int launch_pass_k(const dev::KArgs& ka, uint64_t grid, size_t smem, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(dev::pass_kernel<K>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return (int)e;
    attr_set = true;
  }
  dev::pass_kernel<K><<<(unsigned)grid, 1 << (K - RBITS), smem, st>>>(ka);
  return (int)cudaGetLastError();
}

}  // namespace

int launch_pass(const PassDesc& pd, int n_sim, const DeviceTables& t, const PassLaunch& L,
                void* stream) {
  dev::KArgs ka{};
  ka.src = static_cast<const double2*>(L.src);
  ka.dst = static_cast<double2*>(L.dst);
  ka.ops = t.ops;
  ka.phases = t.phases;
  ka.mats = reinterpret_cast<const double2*>(t.mats);
  ka.seed = L.seed;
  ka.p1 = L.p1;
  ka.p2 = L.p2;
  ka.child_first = L.child_first;
  ka.parent_first = L.parent_first;
  ka.arity = L.arity ? L.arity : 1;
  ka.batch = L.batch;
  ka.src_mode = L.src_mode;
  ka.n = (uint32_t)n_sim;
  ka.n_out = (uint32_t)pd.n_out;
  ka.phase_begin = pd.phase_begin;
  ka.phase_end = pd.phase_end;
  ka.op_begin = pd.op_begin;
  ka.op_end = pd.op_end;
  for (int i = 0; i < MAX_K; ++i) ka.tile_q[i] = i < pd.K ? pd.tile_q[i] : 0;
  for (int i = 0; i < 32; ++i) ka.out_q[i] = i < pd.n_out ? pd.out_q[i] : 0;
  const uint64_t grid = (uint64_t)L.batch << pd.n_out;
  if (grid == 0) return 0;
  if (grid > 0x7FFFFFFFull) return (int)cudaErrorInvalidConfiguration;
  const size_t smem = (sizeof(double2) << pd.K) + ((pd.op_end - pd.op_begin + 15) & ~15u);
  if (smem > 200 * 1024) return (int)cudaErrorInvalidConfiguration;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (pd.K) {
    case 4: return launch_pass_k<4>(ka, grid, smem, st);
    case 5: return launch_pass_k<5>(ka, grid, smem, st);
    case 6: return launch_pass_k<6>(ka, grid, smem, st);
    case 7: return launch_pass_k<7>(ka, grid, smem, st);
    case 8: return launch_pass_k<8>(ka, grid, smem, st);
    case 9: return launch_pass_k<9>(ka, grid, smem, st);
    case 10: return launch_pass_k<10>(ka, grid, smem, st);
    case 11: return launch_pass_k<11>(ka, grid, smem, st);
    case 12: return launch_pass_k<12>(ka, grid, smem, st);
    case 13: return launch_pass_k<13>(ka, grid, smem, st);
    default: return (int)cudaErrorInvalidValue;
  }
}

int launch_chunk_sums(const void* states, uint32_t batch, int n_sim, int chunk_log2, double* sums,
                      void* stream) {
  const uint64_t grid = (uint64_t)batch << (n_sim - chunk_log2);
  if (grid == 0) return 0;
  dev::chunk_sums_kernel<<<(unsigned)grid, dev::MT, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const double2*>(states), (uint32_t)n_sim, (uint32_t)chunk_log2, sums);
  return (int)cudaGetLastError();
}

int launch_sample(const void* states, const double* sums, uint32_t batch, int n_sim, int n_user,
                  int chunk_log2, uint64_t leaf_first, uint64_t seed, double p01, double p10,
                  uint32_t* d_out, void* stream) {
  if (batch == 0) return 0;
  dev::sample_kernel<<<batch, dev::MT, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const double2*>(states), sums, (uint32_t)n_sim, (uint32_t)n_user,
      (uint32_t)chunk_log2, leaf_first, seed, p01, p10, d_out);
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
