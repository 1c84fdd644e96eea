"""Are per-launch CUDA events accurate for kernels launched the way libtqsim launches
them (cudaLibraryLoadData + cudaLibraryGetKernel + cudaLaunchKernel(cudaKernel_t))?
Same kernel through a static __global__ vs through the library path, events per launch
vs total.   python scripts/microbench/lib_launch_harness.py <config> <level> <pass>
"""
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

MAIN = r'''
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <fstream>
#include <sstream>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("cuda %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)
struct __align__(16) tq_d2 { double x, y; };
typedef unsigned int tq_u32; typedef unsigned long long tq_u64;
struct TqJitArgs { const tq_d2* src; tq_d2* dst; tq_u64 seed; double p1, p2; tq_u64 child_first, parent_first; tq_u32 arity, batch;
  double* runsum; const unsigned char* rows; tq_u32 row_bytes; };
int main(int argc, char** argv) {
  std::ifstream f(argv[1], std::ios::binary); std::stringstream ss; ss << f.rdbuf(); std::string cubin = ss.str();
  cudaLibrary_t lib; cudaKernel_t k;
  CK(cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
  CK(cudaLibraryGetKernel(&k, lib, "tq_pass"));
  const int n = N_QUBITS, K = K_TILE, T = THREADS; const unsigned batch = BATCH;
  const size_t S = (size_t)1 << n; const size_t smem = SMEM;
  if (smem > 48 * 1024) CK(cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  tq_d2 *src, *dst; unsigned char* rows; double* runsum;
  CK(cudaMalloc(&src, batch * S * 16)); CK(cudaMalloc(&dst, batch * S * 16));
  CK(cudaMalloc(&rows, (size_t)batch * 1024)); CK(cudaMalloc(&runsum, batch * (S / 8) * 8));
  // random data (not zeros)
  std::vector<double> h(batch * S * 2); for (size_t i = 0; i < h.size(); ++i) h[i] = (double)((i * 2654435761u) % 1000) * 1e-3;
  CK(cudaMemcpy(src, h.data(), batch * S * 16, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dst, h.data(), batch * S * 16, cudaMemcpyHostToDevice));
  CK(cudaMemset(rows, 0, (size_t)batch * 1024));
  TqJitArgs a; a.src = src; a.dst = dst; a.seed = 1; a.p1 = 0; a.p2 = 0; a.child_first = 0; a.parent_first = 0;
  a.arity = 2; a.batch = batch; a.runsum = runsum; a.rows = rows; a.row_bytes = CROW;
  double coef = 0.0; void* args[] = {&a, &coef};
  const unsigned grid = batch << (n - K);
  const int R = 40; cudaEvent_t ev[R + 1]; for (auto& evx : ev) CK(cudaEventCreate(&evx));
  for (int i = 0; i < 3; ++i) CK(cudaLaunchKernel((const void*)k, dim3(grid), dim3(T), args, smem, 0));
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(ev[0], 0));
  for (int i = 0; i < R; ++i) { CK(cudaLaunchKernel((const void*)k, dim3(grid), dim3(T), args, smem, 0)); CK(cudaEventRecord(ev[i + 1], 0)); }
  CK(cudaEventSynchronize(ev[R]));
  float tot; CK(cudaEventElapsedTime(&tot, ev[0], ev[R]));
  double sum = 0; for (int i = 0; i < R; ++i) { float m; CK(cudaEventElapsedTime(&m, ev[i], ev[i + 1])); sum += m; }
  // events only around kernels, with an extra event pair per launch (library's profile mode)
  cudaEvent_t e2[2 * R]; for (auto& evx : e2) CK(cudaEventCreate(&evx));
  cudaEvent_t t0, t1; CK(cudaEventCreate(&t0)); CK(cudaEventCreate(&t1));
  CK(cudaEventRecord(t0, 0));
  for (int i = 0; i < R; ++i) { CK(cudaEventRecord(e2[2 * i], 0)); CK(cudaLaunchKernel((const void*)k, dim3(grid), dim3(T), args, smem, 0)); CK(cudaEventRecord(e2[2 * i + 1], 0)); }
  CK(cudaEventRecord(t1, 0)); CK(cudaEventSynchronize(t1));
  float tot2; CK(cudaEventElapsedTime(&tot2, t0, t1));
  double ks = 0; for (int i = 0; i < R; ++i) { float m; CK(cudaEventElapsedTime(&m, e2[2 * i], e2[2 * i + 1])); ks += m; }
  printf("library-path launch: back-to-back total %.3f ms (%.4f / launch), event-interval sum %.3f; bracketed: total %.3f kernel-sum %.3f (%.4f / launch)\n",
         tot, tot / R, sum, tot2, ks, ks / R);
  return 0;
}
'''


def main():
    cfg, lv, ps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    import paper_2203_13892_b200.tqsim as T
    from workloads import load_config
    w = load_config(cfg)
    n, gates, noise, shots, ar = T.workload_args(w)
    s = T.tqsim_pass_source(n, gates, noise, shots, ar, None, lv, ps)
    thr = int(re.search(r"__launch_bounds__\((\d+),", s).group(1))
    K = thr.bit_length() - 1 + 4
    smem = (16 << K) if "extern __shared__ tq_d2 tile[]" in s else 0
    crow = int(re.search(r"a\.rows \+ \(tq_u64\)s \* (\d+)u", s).group(1))
    d = tempfile.mkdtemp()
    cu, cub = os.path.join(d, "k.cu"), os.path.join(d, "k.cubin")
    open(cu, "w").write(s)
    r = subprocess.run(["nvcc", "-arch=sm_100a", "-cubin", "-std=c++17", "-o", cub, cu], capture_output=True, text=True)
    if r.returncode:
        print(r.stderr[:2000]); sys.exit(1)
    m = (MAIN.replace("N_QUBITS", str(n)).replace("K_TILE", str(K)).replace("THREADS", str(thr))
         .replace("BATCH", str(max(1, (1 << 26) >> n))).replace("SMEM", str(smem)).replace("CROW", str(crow)))
    hc, exe = os.path.join(d, "h.cu"), os.path.join(d, "h")
    open(hc, "w").write(m)
    r = subprocess.run(["nvcc", "-O2", "-std=c++17", "-o", exe, hc], capture_output=True, text=True)
    if r.returncode:
        print(r.stderr[:2000]); sys.exit(1)
    if os.environ.get("HARNESS_COMPILE_ONLY"):
        print("compiled", exe); return
    subprocess.run([exe, cub], check=True)


if __name__ == "__main__":
    main()
