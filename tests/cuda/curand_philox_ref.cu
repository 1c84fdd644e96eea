// TEST-ONLY reference: cuRAND's stateless Philox4x32-10
// (/usr/local/cuda/include/curand_philox4x32_x.h, curand_Philox4x32_10) as an
// implementation independent of both the oracle and libtqsim's device Philox.
#include <cuda_runtime.h>
#include <curand_philox4x32_x.h>
#include <cstdint>

__global__ void curand_philox_kernel(const uint32_t* in, uint64_t n, uint32_t* out) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t* v = in + 6 * i;
  uint4 r = curand_Philox4x32_10(make_uint4(v[0], v[1], v[2], v[3]), make_uint2(v[4], v[5]));
  out[4 * i] = r.x; out[4 * i + 1] = r.y; out[4 * i + 2] = r.z; out[4 * i + 3] = r.w;
}

extern "C" int curand_philox_ref(const uint32_t* in, uint64_t n, uint32_t* out) {
  uint32_t *di = nullptr, *dout = nullptr;
  if (cudaMalloc(&di, n * 24 + 24) != cudaSuccess) return 1;
  if (cudaMalloc(&dout, n * 16 + 16) != cudaSuccess) return 1;
  cudaMemcpy(di, in, n * 24, cudaMemcpyHostToDevice);
  curand_philox_kernel<<<(unsigned)((n + 255) / 256), 256>>>(di, n, dout);
  cudaError_t e = cudaMemcpy(out, dout, n * 16, cudaMemcpyDeviceToHost);
  cudaFree(di);
  cudaFree(dout);
  return e == cudaSuccess ? 0 : 2;
}
