// Device functions shared VERBATIM by the static kernels (kernels.cu includes
// this file) and by every run-time specialized gate-pass kernel (jit.cpp embeds
// this file's text as the NVRTC prelude), so the noise draws of the hot path
// and of the debug hooks are the same code.
//
// Philox4x32-10 (Salmon et al., SC'11) keyed per BASELINE north_star
// "(seed, tree node, branch, gate index)", reading R7:
//   counter = (g, j mod 2^32, tag, j >> 32), key = (seed mod 2^32, seed >> 32),
//   tag 0 = gate noise, 1 = measurement uniform, 2 = readout.
// Depolarizing draw (§2.5; readings R1, R8):
//   error iff w0 * 2^-32 < p; code = 1 + ((w1 * 3) >> 32) (1q) / 1 + ((w1 * 15) >> 32) (2q).
#pragma once

typedef unsigned int tq_u32;
typedef unsigned long long tq_u64;

struct tq_w4 {
  tq_u32 x, y, z, w;
};

__device__ __forceinline__ tq_w4 tq_philox4x32_10(tq_u32 c0, tq_u32 c1, tq_u32 c2, tq_u32 c3,
                                                 tq_u32 k0, tq_u32 k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const tq_u32 lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const tq_u32 lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const tq_u32 n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  tq_w4 o;
  o.x = c0; o.y = c1; o.z = c2; o.w = c3;
  return o;
}

__device__ __forceinline__ tq_w4 tq_philox_keyed(tq_u32 c0, tq_u64 j, tq_u32 tag, tq_u64 seed) {
  return tq_philox4x32_10(c0, (tq_u32)j, tag, (tq_u32)(j >> 32), (tq_u32)seed, (tq_u32)(seed >> 32));
}

// 0 = no error, else the Pauli code (1..3 for 1q; 1..15 for 2q with q0 = code>>2, q1 = code&3)
__device__ __forceinline__ tq_u32 tq_noise_code(tq_u32 g, tq_u64 j, tq_u64 seed, double p, bool two) {
  if (!(p > 0.0)) return 0u;
  const tq_w4 w = tq_philox_keyed(g, j, 0u, seed);
  if (!((double)w.x * 0x1p-32 < p)) return 0u;
  return 1u + __umulhi(w.y, two ? 15u : 3u);
}

// u53 of the leaf measurement (reading R9): ((w0 >> 5) 2^26 + (w1 >> 6)) 2^-53
__device__ __forceinline__ double tq_measure_uniform(tq_u64 leaf, tq_u64 seed) {
  const tq_w4 w = tq_philox_keyed(0u, leaf, 1u, seed);
  return ((double)(w.x >> 5) * 67108864.0 + (double)(w.y >> 6)) * 0x1p-53;
}

// XOR swizzle of a tile-local amplitude index (16-byte units): the bank group
// (low 3 bits) is XORed with the higher 3-bit groups.  Linear over GF(2).
__device__ __forceinline__ tq_u32 tq_swz(tq_u32 i) {
  return i ^ (((i >> 3) ^ (i >> 6) ^ (i >> 9) ^ (i >> 12)) & 7u);
}
