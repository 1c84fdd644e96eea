// Static sm_100a kernels of the TQSim hot path and the
// debug hooks.  The gate-pass kernels (row a5) are specialized per pass at run
// time (jit.cpp); both include the same device functions (tq_device_common.cuh).
//
//  chunk_sums       |a|^2 sums of 2^C-amplitude contiguous chunks of leaf states
//  sample_kernel    one CTA per leaf: warp-shuffle block scan over the chunk
//                   sums -> chunk, re-read the chunk, block scan -> the smallest
//                   x with C(x) > u*total (§2.3 "the final outcome is
//                   sampled", reading R9), readout flips (R11).
#include <cuda_runtime.h>

#include "tq_device_common.cuh"
#include "tq_internal.h"

namespace tq {
namespace dev {

constexpr int MT = 256;   // threads of the measurement kernels

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

__global__ void __launch_bounds__(MT) chunk_sums_kernel(const cd* __restrict__ states, uint32_t n,
                                                        uint32_t chunk_log2,
                                                        double* __restrict__ sums) {
  __shared__ double red[MT / 32];
  const uint64_t n_chunks = 1ull << (n - chunk_log2);
  const uint64_t bid = blockIdx.x;
  const uint64_t s = bid >> (n - chunk_log2), c = bid & (n_chunks - 1);
  const cd* p = states + (s << n) + (c << chunk_log2);
  double acc = 0.0;
  for (uint32_t i = threadIdx.x; i < (1u << chunk_log2); i += MT) {
    const cd v = p[i];
    acc = fma(v.x, v.x, fma(v.y, v.y, acc));
  }
  const double tot = block_sum(acc, red);
  if (threadIdx.x == 0) sums[bid] = tot;
}

__global__ void __launch_bounds__(MT) sample_kernel(const cd* __restrict__ states,
                                                    const double* __restrict__ sums, uint32_t n,
                                                    uint32_t n_user, uint32_t chunk_log2,
                                                    uint64_t leaf_first, uint64_t seed, double p01,
                                                    double p10, uint32_t* __restrict__ out) {
  __shared__ double wsum[MT / 32];
  __shared__ int first_sh;
  __shared__ uint64_t pick_sh;
  __shared__ double before_sh, total_sh;
  __shared__ int64_t x_sh;
  const uint32_t s = blockIdx.x;
  const uint64_t leaf = leaf_first + s;
  const uint64_t nc = 1ull << (n - chunk_log2);
  const double* cs = sums + (uint64_t)s * nc;
  const cd* st = states + ((uint64_t)s << n);
  const double u = tq_measure_uniform(leaf, seed);

  // (a) chunk selection over contiguous per-thread ranges of chunk sums
  const uint64_t per = (nc + MT - 1) / MT;
  const uint64_t c0 = per * threadIdx.x < nc ? per * threadIdx.x : nc;
  const uint64_t c1 = c0 + per < nc ? c0 + per : nc;
  double loc = 0.0;
  for (uint64_t c = c0; c < c1; ++c) loc += cs[c];
  const double incl = block_incl_scan(loc, wsum);
  if (threadIdx.x == MT - 1) total_sh = incl;
  __syncthreads();
  const double target = u * total_sh;
  const int tsel = block_first(incl > target, &first_sh);
  if (threadIdx.x == 0) {
    pick_sh = ~0ull;
    before_sh = 0.0;
  }
  __syncthreads();
  if ((int)threadIdx.x == tsel) {
    double acc = incl - loc;
    uint64_t pick = ~0ull;
    for (uint64_t c = c0; c < c1; ++c) {
      if (acc + cs[c] > target) {
        pick = c;
        break;
      }
      acc += cs[c];
    }
    if (pick == ~0ull) {   // rounding: the last non-empty chunk of the range
      acc = incl - loc;
      for (uint64_t c = c0; c < c1; ++c)
        if (cs[c] > 0.0) pick = c;
      for (uint64_t c = c0; c < pick; ++c) acc += cs[c];
    }
    pick_sh = pick;
    before_sh = acc;
  }
  __syncthreads();
  if (pick_sh == ~0ull) {   // target beyond the total (rounding): last non-empty chunk
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t c = nc;
      double acc = 0.0;
      for (uint64_t i = 0; i < nc; ++i)
        if (cs[i] > 0.0) c = i;
      if (c == nc) c = nc - 1;
      for (uint64_t i = 0; i < c; ++i) acc += cs[i];
      pick_sh = c;
      before_sh = acc;
    }
    __syncthreads();
  }
  const uint64_t chunk = pick_sh;
  const double target2 = target - before_sh;

  // (b) within the chunk: per-thread contiguous runs of |a|^2
  const uint32_t clen = 1u << chunk_log2;
  const uint32_t per2 = (clen + MT - 1) / MT;
  const uint32_t e0 = min(clen, per2 * threadIdx.x), e1 = min(clen, e0 + per2);
  const cd* cp = st + (chunk << chunk_log2);
  double loc2 = 0.0;
  for (uint32_t e = e0; e < e1; ++e) {
    const cd v = cp[e];
    loc2 += v.x * v.x + v.y * v.y;
  }
  const double incl2 = block_incl_scan(loc2, wsum);
  const int tsel2 = block_first(incl2 > target2, &first_sh);
  if (threadIdx.x == 0) x_sh = -1;
  __syncthreads();
  if (tsel2 < MT && (int)threadIdx.x == tsel2) {
    double acc = incl2 - loc2;
    int64_t x = -1;
    for (uint32_t e = e0; e < e1; ++e) {
      const cd v = cp[e];
      acc += v.x * v.x + v.y * v.y;
      if (acc > target2) {
        x = e;
        break;
      }
    }
    if (x < 0)
      for (uint32_t e = e0; e < e1; ++e) {
        const cd v = cp[e];
        if (v.x * v.x + v.y * v.y > 0.0) x = e;
      }
    x_sh = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t x = x_sh;
    if (x < 0) {   // fall back to the last non-zero amplitude of the chunk
      for (uint32_t e = 0; e < clen; ++e) {
        const cd v = cp[e];
        if (v.x * v.x + v.y * v.y > 0.0) x = e;
      }
      if (x < 0) x = 0;
    }
    const uint32_t xi = (uint32_t)((chunk << chunk_log2) + (uint64_t)x);
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

}  // namespace dev

// ------------------------------------------------------------------ launchers
int launch_chunk_sums(const void* states, uint32_t batch, int n_sim, int chunk_log2, double* sums,
                      void* stream) {
  const uint64_t grid = (uint64_t)batch << (n_sim - chunk_log2);
  if (grid == 0) return 0;
  dev::chunk_sums_kernel<<<(unsigned)grid, dev::MT, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const dev::cd*>(states), (uint32_t)n_sim, (uint32_t)chunk_log2, sums);
  return (int)cudaGetLastError();
}

int launch_sample(const void* states, const double* sums, uint32_t batch, int n_sim, int n_user,
                  int chunk_log2, uint64_t leaf_first, uint64_t seed, double p01, double p10,
                  uint32_t* d_out, void* stream) {
  if (batch == 0) return 0;
  dev::sample_kernel<<<batch, dev::MT, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const dev::cd*>(states), sums, (uint32_t)n_sim, (uint32_t)n_user,
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
