// Microbenchmark: how to stream 2^12-amplitude complex128 tiles through an SM at
// HBM rate on B200 (design input for the gate-pass kernels).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o stream_bench stream_bench.cu
//   ./stream_bench
//
// Every variant reads a 1 GiB batch of tiles and writes it back (in place), with
// X smem exchanges ("phases") and F complex multiplies per amplitude per phase.
//   A  direct: 2 CTAs x 256 threads per SM, 16 LDG.128 -> registers -> STG (coalesced)
//   B  direct, lanes on scattered tile positions (uncoalesced, like v1 phase 0)
//   C  persistent LDGSTS ring (3 x 64 KiB stages, 1 CTA x 256 threads per SM)
//   D  persistent cp.async.bulk ring (3 stages, run = 2^RUNQ amplitudes per bulk op)
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

struct __align__(16) d2 { double x, y; };
constexpr int K = 12, TILE = 1 << K, T = 256, NS = 3;

__device__ __forceinline__ unsigned swz(unsigned i) { return i ^ (((i >> 3) ^ (i >> 6) ^ (i >> 9) ^ (i >> 12)) & 7u); }

template <int F>
__device__ __forceinline__ void compute(d2 (&r)[16], double c, double s) {
#pragma unroll
  for (int f = 0; f < F; ++f)
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const d2 x = r[k];
      r[k].x = fma(c, x.x, -s * x.y);
      r[k].y = fma(c, x.y, s * x.x);
    }
}

// lane -> tile position map: coalesced = identity (positions 0..7 on thread bits)
template <bool COAL>
__device__ __forceinline__ unsigned tpos_off(unsigned tid, int k) {
  if (COAL) return tid | ((unsigned)k << 8);
  // registers on positions 0,1,3,4, threads on 2,5..11 (the v1 l9_p0 layout)
  unsigned o = 0;
  o |= ((unsigned)k & 1u) << 0; o |= (((unsigned)k >> 1) & 1u) << 1;
  o |= (((unsigned)k >> 2) & 1u) << 3; o |= (((unsigned)k >> 3) & 1u) << 4;
  o |= (tid & 1u) << 2;
  o |= (tid >> 1) << 5;
  return o;
}

template <bool COAL, int X, int F>
__global__ void __launch_bounds__(T, 2) direct_kernel(d2* __restrict__ st, double c, double s) {
  extern __shared__ d2 tile[];
  const unsigned tid = threadIdx.x;
  d2* base = st + ((size_t)blockIdx.x << K);
  d2 r[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) r[k] = base[tpos_off<COAL>(tid, k)];
  compute<F>(r, c, s);
#pragma unroll
  for (int x = 0; x < X; ++x) {
#pragma unroll
    for (int k = 0; k < 16; ++k) tile[swz(tid * 16 + k)] = r[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) r[k] = tile[swz(tid + 256 * k)];
    __syncthreads();
    compute<F>(r, c, s);
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) base[tpos_off<COAL>(tid, k)] = r[k];
}

__device__ __forceinline__ void cp16(void* sdst, const void* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" :: "n"(N) : "memory"); }

template <int X, int F>
__global__ void __launch_bounds__(T, 1) ldgsts_kernel(d2* __restrict__ st, unsigned long long ntiles, double c, double s) {
  extern __shared__ __align__(16) d2 stages[];
  const unsigned tid = threadIdx.x;
  auto issue = [&](unsigned long long t, unsigned sidx) {
    const d2* src = st + (t << K);
    d2* sb = stages + ((size_t)sidx << K);
#pragma unroll
    for (int k = 0; k < 16; ++k) cp16(sb + swz(tid + 256 * k), src + tid + 256 * k);
  };
  for (unsigned j = 0; j < NS - 1; ++j) {
    const unsigned long long t = blockIdx.x + (unsigned long long)j * gridDim.x;
    if (t < ntiles) issue(t, j);
    cp_commit();
  }
  unsigned sidx = 0;
  for (unsigned long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const unsigned long long t2 = t + (unsigned long long)(NS - 1) * gridDim.x;
    if (t2 < ntiles) issue(t2, sidx == 0 ? NS - 1 : sidx - 1);
    cp_commit();
    cp_wait<NS - 1>();
    __syncthreads();
    d2* tile = stages + ((size_t)sidx << K);
    d2 r[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) r[k] = tile[swz(tid * 16 + k)];
    compute<F>(r, c, s);
#pragma unroll
    for (int x = 0; x < X; ++x) {
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k) tile[swz(tid * 16 + k)] = r[k];
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k) r[k] = tile[swz(tid + 256 * k)];
      compute<F>(r, c, s);
    }
    d2* dst = st + (t << K);
#pragma unroll
    for (int k = 0; k < 16; ++k) dst[tid + 256 * k] = r[k];
    __syncthreads();
    sidx = sidx + 1 == NS ? 0 : sidx + 1;
  }
  cp_wait<0>();
}

// ---- bulk copies + mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" :: "r"((unsigned)__cvta_generic_to_shared(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" :: "r"((unsigned)__cvta_generic_to_shared(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT;\n}\n" :: "r"((unsigned)__cvta_generic_to_shared(b)), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               :: "r"((unsigned)__cvta_generic_to_shared(sdst)), "l"(gsrc), "r"(bytes),
                  "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}

template <int RUNQ, int X, int F>
__global__ void __launch_bounds__(T, 1) bulk_kernel(d2* __restrict__ st, unsigned long long ntiles, double c, double s) {
  extern __shared__ __align__(128) d2 stages[];
  __shared__ __align__(8) uint64_t bars[NS];
  const unsigned tid = threadIdx.x;
  constexpr int NRUN = TILE >> RUNQ;   // bulk ops per tile
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](unsigned long long t, unsigned sidx) {
    // threads 0..NRUN-1 each issue one run; thread 0 arms the barrier first
    if (tid == 0) mbar_expect_tx(&bars[sidx], TILE * 16);
    __syncwarp();
    const d2* src = st + (t << K);
    d2* sb = stages + ((size_t)sidx << K);
    for (int r = tid; r < NRUN; r += T)
      bulk_g2s(sb + (r << RUNQ), src + (r << RUNQ), 16u << RUNQ, &bars[sidx]);
  };
  for (unsigned j = 0; j < NS - 1; ++j) {
    const unsigned long long t = blockIdx.x + (unsigned long long)j * gridDim.x;
    if (t < ntiles) issue(t, j);
  }
  unsigned sidx = 0, phase = 0;
  for (unsigned long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const unsigned long long t2 = t + (unsigned long long)(NS - 1) * gridDim.x;
    if (t2 < ntiles) issue(t2, sidx == 0 ? NS - 1 : sidx - 1);
    mbar_wait(&bars[sidx], phase);
    d2* tile = stages + ((size_t)sidx << K);
    d2 r[16];   // unswizzled stage: read the thread's 16 contiguous amplitudes
#pragma unroll
    for (int k = 0; k < 16; ++k) r[k] = tile[tid + 256 * k];
    compute<F>(r, c, s);
#pragma unroll
    for (int x = 0; x < X; ++x) {
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k) tile[swz(tid * 16 + k)] = r[k];
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k) r[k] = tile[swz(tid + 256 * k)];
      compute<F>(r, c, s);
    }
    d2* dst = st + (t << K);
#pragma unroll
    for (int k = 0; k < 16; ++k) dst[tid + 256 * k] = r[k];
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic smem writes before TMA refill
    __syncthreads();
    if (++sidx == NS) { sidx = 0; phase ^= 1; }
  }
}

template <class Fn>
float time_it(Fn fn, int reps = 10) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  fn(); fn();
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int i = 0; i < reps; ++i) fn();
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b));
  CK(cudaGetLastError());
  return ms / reps;
}

int main(int argc, char** argv) {
  const size_t bytes = 1ull << 30, ntiles = bytes / (16 * TILE);
  d2* st; CK(cudaMalloc(&st, bytes)); CK(cudaMemset(st, 0, bytes));
  int nsm = 0; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const double c = 0.8, s = 0.6;
  auto report = [&](const char* name, float ms) {
    printf("%-34s %8.3f ms  %7.0f GB/s\n", name, ms, 2.0 * bytes / (ms * 1e-3) / 1e9); fflush(stdout);
  };
#define DIRECT(COAL, X, F) { auto k = direct_kernel<COAL, X, F>; CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536)); \
    report("direct coal=" #COAL " X=" #X " F=" #F, time_it([&] { k<<<ntiles, T, X ? 65536 : 0>>>(st, c, s); })); }
#define LDGSTS(X, F) { auto k = ldgsts_kernel<X, F>; size_t sm = NS * TILE * 16; CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    report("ldgsts X=" #X " F=" #F, time_it([&] { k<<<nsm, T, sm>>>(st, ntiles, c, s); })); }
#define BULK(R, X, F) { auto k = bulk_kernel<R, X, F>; size_t sm = NS * TILE * 16; CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    report("bulk run=2^" #R " X=" #X " F=" #F, time_it([&] { k<<<nsm, T, sm>>>(st, ntiles, c, s); })); }
  if (argc > 1) {   // compute-heavy sweep: does prefetching the next tile pay?
    DIRECT(true, 1, 8) DIRECT(true, 1, 16) DIRECT(true, 1, 32) DIRECT(true, 2, 16)
    LDGSTS(1, 8) LDGSTS(1, 16) LDGSTS(1, 32) LDGSTS(2, 16)
    BULK(6, 1, 8) BULK(6, 1, 16) BULK(6, 1, 32) BULK(6, 2, 16)
    return 0;
  }
  DIRECT(true, 0, 0) DIRECT(false, 0, 0) DIRECT(true, 1, 0) DIRECT(false, 1, 0) DIRECT(true, 1, 4) DIRECT(true, 3, 2)
  LDGSTS(0, 0) LDGSTS(1, 0) LDGSTS(1, 4) LDGSTS(3, 2)
  BULK(3, 0, 0) BULK(6, 0, 0) BULK(12, 0, 0) BULK(6, 1, 0) BULK(6, 1, 4) BULK(6, 3, 2) BULK(3, 1, 0)
  return 0;
}
