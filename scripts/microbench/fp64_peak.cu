// Microbenchmark: the FP64 FMA (DFMA) throughput of this B200 -- the `alu` roofline
// denominator of the FP64-bound gate passes.  The guides carry no FP64
// figure for sm_100a; the derivation 148 SMs x 64 DFMA/clk x f_clk is checked here.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu && ./fp64_peak
//
// Each thread runs 8 independent DFMA chains (enough ILP to cover the pipe latency) for
// ITER iterations; grid = 148 x 8 CTAs x 256 threads.  Reports DFMA/s (best of 5, CUDA
// events) and the implied DFMA/clk/SM at the clock sampled by nvidia-smi.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

constexpr int ITER = 4096, CH = 8;

__global__ void __launch_bounds__(256) dfma_kernel(double* out, double a, double b) {
  double r[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) r[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < ITER; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) r[c] = fma(r[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += r[c];
  if (s == 123.456) out[blockIdx.x] = s;   // keeps the chains alive
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
  double* out;
  CK(cudaMalloc(&out, 1 << 20));
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    CK(cudaEventRecord(e0));
    dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  const double dfma = (double)blocks * threads * ITER * CH;
  const double rate = dfma / (best * 1e-3);
  printf("{\"sms\": %d, \"attr_clock_mhz\": %.0f, \"ms\": %.4f, \"dfma_per_s\": %.4e, "
         "\"dfma_per_clk_sm_at_attr_clock\": %.2f, \"tflops_fp64\": %.2f}\n",
         sms, clk_khz / 1e3, best, rate, rate / (sms * clk_khz * 1e3), 2 * rate / 1e12);
  return 0;
}
