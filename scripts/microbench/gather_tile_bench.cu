// Microbenchmark: HBM read+write throughput of gate-pass tiles whose qubit set has only r
// contiguous low qubits (runs of 2^r amplitudes = 16 * 2^r bytes), the rest high qubits
// (design input: a pass over tile {0, 1} + 11 high qubits covers 2 more qubits than the
// standard {0, 1, 2} + 10 and can save a whole pass of C4's 24-qubit leaf level).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gather_tile_bench gather_tile_bench.cu
//
// Batch of 8 states x 2^24 amplitudes (2 GiB), tile of 2^12 amplitudes, 256 threads x 16
// registers; tile position p -> qubit Q[p] with Q = {0..r-1} U {24-12+r .. 23}; lanes on
// positions 0..4, registers on 8..11, warps on 5..7 (a typical pass's load phase).
// V256: registers k, k|1 on position 0 moved as one 32-byte access.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

struct __align__(16) d2 { double x, y; };
constexpr int N = 24, K = 12, T = 256;

struct Map { unsigned col[K]; unsigned out[N - K]; int rpos[4]; int tpos[8]; };
__constant__ Map M;

__device__ __forceinline__ unsigned long long addr(unsigned t, unsigned tid, int k) {
  unsigned long long a = 0;
#pragma unroll
  for (int i = 0; i < N - K; ++i) a |= (unsigned long long)((t >> i) & 1u) << M.out[i];
#pragma unroll
  for (int b = 0; b < 4; ++b) a |= (unsigned long long)((k >> b) & 1) << M.col[M.rpos[b]];
#pragma unroll
  for (int m = 0; m < 8; ++m) a |= (unsigned long long)((tid >> m) & 1u) << M.col[M.tpos[m]];
  return a;
}

template <bool V256>
__global__ void __launch_bounds__(T, 2) kern(d2* __restrict__ st, double c, double s) {
  const unsigned tid = threadIdx.x;
  const unsigned long long sidx = blockIdx.x >> (N - K);
  const unsigned t = blockIdx.x & ((1u << (N - K)) - 1);
  d2* base = st + (sidx << N);
  d2 r[16];
  if (V256) {
#pragma unroll
    for (int k = 0; k < 16; k += 2) {
      const d2* p = base + addr(t, tid, k);
      asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r[k].x), "=d"(r[k].y), "=d"(r[k + 1].x), "=d"(r[k + 1].y) : "l"(p));
    }
  } else {
#pragma unroll
    for (int k = 0; k < 16; ++k) r[k] = base[addr(t, tid, k)];
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
      d2* p = base + addr(t, tid, k);
      asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" :: "l"(p), "d"(r[k].x), "d"(r[k].y), "d"(r[k + 1].x), "d"(r[k + 1].y) : "memory");
    }
  } else {
#pragma unroll
    for (int k = 0; k < 16; ++k) base[addr(t, tid, k)] = r[k];
  }
}

int main() {
  const size_t states = 8, bytes = states << (N + 4);
  d2* st;
  CK(cudaMalloc(&st, bytes));
  CK(cudaMemset(st, 0, bytes));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int r = 0; r <= 4; ++r) {
    for (int v = 0; v < 3; ++v) {
      Map m{};
      // tile qubits: 0..r-1 then the top K-r qubits
      for (int p = 0; p < K; ++p) m.col[p] = p < r ? p : (N - K + p);
      int o = 0;
      for (int q = 0; q < N; ++q) {
        bool in = false;
        for (int p = 0; p < K; ++p) in |= (int)m.col[p] == q;
        if (!in) m.out[o++] = q;
      }
      // v0: lanes on positions 0..4, warps 5..7, regs 8..11;  v1: V256 (regs 0, 8, 9, 10), lanes 1..5;
      // v2: lanes on 0..4, tile walked "warp-major": regs on 5, 6, 7, 8, warps 9..11
      int rp0[4] = {8, 9, 10, 11}, tp0[8] = {0, 1, 2, 3, 4, 5, 6, 7};
      int rp1[4] = {0, 9, 10, 11}, tp1[8] = {1, 2, 3, 4, 5, 6, 7, 8};
      int rp2[4] = {5, 6, 7, 8}, tp2[8] = {0, 1, 2, 3, 4, 9, 10, 11};
      int* rp = v == 0 ? rp0 : v == 1 ? rp1 : rp2;
      int* tp = v == 0 ? tp0 : v == 1 ? tp1 : tp2;
      for (int i = 0; i < 4; ++i) m.rpos[i] = rp[i];
      for (int i = 0; i < 8; ++i) m.tpos[i] = tp[i];
      if (v == 1 && r == 0) continue;
      CK(cudaMemcpyToSymbol(M, &m, sizeof(Map)));
      const unsigned grid = (unsigned)(states << (N - K));
      auto launch = [&]() {
        if (v == 1) kern<true><<<grid, T>>>(st, 0.6, 0.8);
        else kern<false><<<grid, T>>>(st, 0.6, 0.8);
      };
      for (int i = 0; i < 3; ++i) launch();
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      const int reps = 10;
      for (int i = 0; i < reps; ++i) launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      ms /= reps;
      printf("runs of 2^%d amps (%4d B)  %-28s %8.3f ms  %7.0f GB/s\n", r, 16 << r,
             v == 0 ? "lanes 0..4, regs 8..11" : v == 1 ? "V256 regs 0,9..11" : "lanes 0..4, regs 5..8",
             ms, 2.0 * bytes / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
