// Microbenchmark: HBM read+write throughput of 2^11-amplitude complex128 tiles under
// different thread layouts (design input for the load/store phases).
// A layout = the 4 tile positions held in registers (rpos) and the 7 on thread bits
// (tpos, lane bits first).  V256: registers k, k|1 with rpos[0] = 0 (qubit 0) move as one
// 32-byte LDG/STG.256 (sm_100), so a lane's access covers a whole 32-byte sector.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o io_layout_bench io_layout_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

struct __align__(16) d2 { double x, y; };
constexpr int K = 11, T = 128;

struct Layout { int rpos[4]; int tpos[7]; };
__constant__ Layout L, LS;   // load layout, store layout (mixed variants)

__device__ __forceinline__ unsigned off_l(const Layout& l, unsigned tid, int k) {
  unsigned o = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) o |= ((unsigned)(k >> b) & 1u) << l.rpos[b];
#pragma unroll
  for (int m = 0; m < 7; ++m) o |= ((tid >> m) & 1u) << l.tpos[m];
  return o;
}
__device__ __forceinline__ unsigned off(unsigned tid, int k) { return off_l(L, tid, k); }

// load with L (16-byte), store with LS (32-byte pairs): the data lands permuted
// (timing only), as in a pass whose last phase has a different layout
__global__ void __launch_bounds__(T, 4) kern_mixed(d2* __restrict__ st, double c, double s) {
  const unsigned tid = threadIdx.x;
  d2* base = st + ((size_t)blockIdx.x << K);
  d2 r[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) r[k] = base[off(tid, k)];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const d2 x = r[k];
    r[k].x = fma(c, x.x, -s * x.y);
    r[k].y = fma(c, x.y, s * x.x);
  }
#pragma unroll
  for (int k = 0; k < 16; k += 2) {
    d2* p = base + off_l(LS, tid, k);
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" :: "l"(p), "d"(r[k].x), "d"(r[k].y), "d"(r[k + 1].x), "d"(r[k + 1].y) : "memory");
  }
}

template <bool V256>
__global__ void __launch_bounds__(T, 4) kern(d2* __restrict__ st, double c, double s) {
  const unsigned tid = threadIdx.x;
  d2* base = st + ((size_t)blockIdx.x << K);
  d2 r[16];
  if (V256) {
#pragma unroll
    for (int k = 0; k < 16; k += 2) {
      const d2* p = base + off(tid, k);
      asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r[k].x), "=d"(r[k].y), "=d"(r[k + 1].x), "=d"(r[k + 1].y) : "l"(p));
    }
  } else {
#pragma unroll
    for (int k = 0; k < 16; ++k) r[k] = base[off(tid, k)];
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const d2 x = r[k];
    r[k].x = fma(c, x.x, -s * x.y);
    r[k].y = fma(c, x.y, s * x.x);
  }
  if (V256) {
#pragma unroll
    for (int k = 0; k < 16; k += 2) {
      d2* p = base + off(tid, k);
      asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" :: "l"(p), "d"(r[k].x), "d"(r[k].y), "d"(r[k + 1].x), "d"(r[k + 1].y) : "memory");
    }
  } else {
#pragma unroll
    for (int k = 0; k < 16; ++k) base[off(tid, k)] = r[k];
  }
}

int main() {
  const size_t bytes = 1ull << 30, amps = bytes / 16, tiles = amps >> K;
  d2* st;
  CK(cudaMalloc(&st, bytes));
  CK(cudaMemset(st, 0, bytes));
  struct V { const char* name; Layout l; bool v256; };
  V vs[] = {
      {"lanes 0..6 on q0..6 (current coalesced)", {{7, 8, 9, 10}, {0, 1, 2, 3, 4, 5, 6}}, false},
      {"lane0 q0, lanes on q4..9, regs q1,2,3,10", {{1, 2, 3, 10}, {0, 4, 5, 6, 7, 8, 9}}, false},
      {"lanes q3..9, regs q0,1,2,10 (16B, scattered)", {{0, 1, 2, 10}, {3, 4, 5, 6, 7, 8, 9}}, false},
      {"lanes q3..9, regs q0,1,2,10 (V256)", {{0, 1, 2, 10}, {3, 4, 5, 6, 7, 8, 9}}, true},
      {"lanes q2..8, regs q0,1,9,10 (V256)", {{0, 1, 9, 10}, {2, 3, 4, 5, 6, 7, 8}}, true},
      {"lanes q1..7, regs q0,8,9,10 (V256)", {{0, 8, 9, 10}, {1, 2, 3, 4, 5, 6, 7}}, true},
      {"lanes q5..10,q1 regs q0,2,3,4 (V256)", {{0, 2, 3, 4}, {5, 6, 7, 8, 9, 10, 1}}, true},
      {"regs q0,1,3,4; lanes q2,5..10 (old v1 l9)", {{0, 1, 3, 4}, {2, 5, 6, 7, 8, 9, 10}}, false},
      {"regs q0,1,4,5 lanes q2,3,6..10 (V256)", {{0, 1, 4, 5}, {2, 3, 6, 7, 8, 9, 10}}, true},
      {"regs q0,1,4,5 lanes q2,3,7,6,8..10 (V256)", {{0, 1, 4, 5}, {2, 3, 7, 6, 8, 9, 10}}, true},
      {"regs q5..8 lanes q0..4,9,10", {{5, 6, 7, 8}, {0, 1, 2, 3, 4, 9, 10}}, false},
      {"regs q0,1,9,10 lanes q2..8 (16B)", {{0, 1, 9, 10}, {2, 3, 4, 5, 6, 7, 8}}, false},
  };
  {
    Layout ld = {{7, 8, 9, 10}, {0, 1, 2, 3, 4, 5, 6}}, stl = {{0, 1, 4, 5}, {2, 3, 7, 6, 8, 9, 10}};
    CK(cudaMemcpyToSymbol(L, &ld, sizeof(Layout)));
    CK(cudaMemcpyToSymbol(LS, &stl, sizeof(Layout)));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int i = 0; i < 3; ++i) kern_mixed<<<(unsigned)tiles, T>>>(st, 0.6, 0.8);
    CK(cudaEventRecord(a));
    for (int i = 0; i < 20; ++i) kern_mixed<<<(unsigned)tiles, T>>>(st, 0.6, 0.8);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    ms /= 20;
    printf("%-48s %8.4f ms  %7.0f GB/s\n", "load coalesced 16B, store V256 q0,1,4,5", ms, 2.0 * bytes / (ms * 1e-3) / 1e9);
  }
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (auto& v : vs) {
    CK(cudaMemcpyToSymbol(L, &v.l, sizeof(Layout)));
    auto launch = [&]() {
      if (v.v256) kern<true><<<(unsigned)tiles, T>>>(st, 0.6, 0.8);
      else kern<false><<<(unsigned)tiles, T>>>(st, 0.6, 0.8);
    };
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    const int reps = 20;
    for (int i = 0; i < reps; ++i) launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= reps;
    printf("%-48s %8.4f ms  %7.0f GB/s\n", v.name, ms, 2.0 * bytes / (ms * 1e-3) / 1e9);
  }
  return 0;
}
