#include <cstdio>
__global__ void __launch_bounds__(128, 4) k(const unsigned* rep, unsigned batch, int* out) {
  const unsigned s = blockIdx.x % batch;
  if (rep[s] != s) return;
  if (threadIdx.x == 0 && rep[s] == 0xffffffffu) out[0] = 1;
}
int main() {
  unsigned* rep; int* out; const unsigned batch = 2048;
  cudaMalloc(&rep, batch * 4); cudaMalloc(&out, 4);
  unsigned h[2048]; for (unsigned i = 0; i < batch; ++i) h[i] = i ^ 1;   // all skip
  cudaMemcpy(rep, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (unsigned grid : {32768u, 13000u, 65536u}) {
    for (int i = 0; i < 3; ++i) k<<<grid, 128>>>(rep, batch, out);
    cudaEventRecord(a);
    for (int i = 0; i < 20; ++i) k<<<grid, 128>>>(rep, batch, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("grid %u: %.2f us per launch (all CTAs exit)\n", grid, ms * 1000 / 20);
  }
  return 0;
}
