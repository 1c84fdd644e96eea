// Microbenchmark: read throughput of the leaf-level access pattern (design input for the
// trail marginal pass and the streaming projection).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o row_stride_bench row_stride_bench.cu
//
// 16 states x 2^24 complex128 (4 GiB).  Each CTA (256 threads, 32 B per thread per row)
// reads 256 "rows" of 8 KiB and reduces them (a sum, kept live):
//   strided:    row y of the CTA's chunk at  state + y * 1 MiB + chunk * 8 KiB   (the projection:
//               top-bit pattern y, 2^16 amplitudes per pattern; one CTA spans the whole 256 MiB)
//   contiguous: row y at state + chunk * 2 MiB + y * 8 KiB                         (one 2 MiB page)
//   strided_g:  strided, but the 128 chunks of a state's row run on consecutive CTAs
//               (grid order chunk-fastest instead of state-fastest)
// Same bytes, same loads in flight (unroll 8); the difference is the address spread per CTA.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int T = 256, ROWS = 256, STATES = 16;
constexpr size_t STATE_BYTES = size_t(16) << 24, ROW_STRIDE = size_t(1) << 20, CHUNK = size_t(8) << 10;

template <int MODE>
__global__ void __launch_bounds__(T) kern(const char* __restrict__ base, double* out) {
  unsigned st, ch;
  if (MODE == 2) { ch = blockIdx.x % 128; st = blockIdx.x / 128; }
  else { st = blockIdx.x % STATES; ch = blockIdx.x / STATES; }
  const char* s = base + st * STATE_BYTES;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll 8
  for (int y = 0; y < ROWS; ++y) {
    const size_t off = MODE == 1 ? ch * (ROWS * CHUNK) + y * CHUNK : y * ROW_STRIDE + ch * CHUNK;
    double px, py, qx, qy;
    asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(px), "=d"(py), "=d"(qx), "=d"(qy) : "l"(s + off + threadIdx.x * 32));
    a0 = fma(px, 1.0000001, a0); a1 = fma(py, 1.0000001, a1); a2 = fma(qx, 1.0000001, a2); a3 = fma(qy, 1.0000001, a3);
  }
  if (a0 + a1 + a2 + a3 == 12345.0) out[blockIdx.x] = a0;
}

int main() {
  const size_t bytes = STATES * STATE_BYTES;
  char* d;
  double* o;
  CK(cudaMalloc(&d, bytes));
  CK(cudaMalloc(&o, 1 << 20));
  CK(cudaMemset(d, 0, bytes));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const unsigned grid = STATES * 128;
  const char* names[3] = {"strided (1 MiB rows, state-fastest grid)", "contiguous (2 MiB per CTA)",
                          "strided (1 MiB rows, chunk-fastest grid)"};
  for (int mode = 0; mode < 3; ++mode) {
    auto launch = [&]() {
      if (mode == 0) kern<0><<<grid, T>>>(d, o);
      else if (mode == 1) kern<1><<<grid, T>>>(d, o);
      else kern<2><<<grid, T>>>(d, o);
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
    printf("%-44s %8.3f ms  %7.0f GB/s\n", names[mode], ms, bytes / (ms * 1e-3) / 1e9);
  }
  return 0;
}
