"""Standalone timing of ONE generated gate-pass kernel (design experiments).

    python scripts/microbench/pass_harness.py <config> <level> <pass> [--variant NAME] [--tile K]

Generates the pass's CUDA source through the C ABI (tqsim_pass_source), appends a
main() that launches it on a synthetic 1 GiB batch (noise rows all zero: the fast
path; --careful sets every row's error mask: the careful path), compiles it with nvcc
for sm_100a and prints ms and algorithmic GB/s.  --variant applies a source edit
(see VARIANTS) to measure what a piece of the kernel costs.
"""
import argparse
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
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("cuda %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)
int main() {
  const int n = N_QUBITS, K = K_TILE, T = THREADS, mode = MODE;
  const unsigned batch = BATCH, arity = 2, crow = CROW;
  const size_t S = (size_t)1 << n;
  tq_d2 *src, *dst; unsigned char* rows; double* runsum;
  const size_t nparent = mode == 1 ? (batch + arity - 1) / arity : batch;
  CK(cudaMalloc(&src, nparent * S * 16)); CK(cudaMalloc(&dst, batch * S * 16));
  CK(cudaMalloc(&rows, (size_t)batch * crow)); CK(cudaMalloc(&runsum, batch * (S / 8) * 8));
  CK(cudaMemset(src, 0, nparent * S * 16)); CK(cudaMemset(dst, 0, batch * S * 16));
  CK(cudaMemset(rows, CAREFUL ? 0xff : 0, (size_t)batch * crow));
  if (CAREFUL) {  // error mask set; codes 0 except the first gate of the pass
    unsigned char* h = (unsigned char*)calloc((size_t)batch * crow, 1);
    for (unsigned s = 0; s < batch; ++s) { h[s * crow + 0] = 0xff; h[s * crow + 1] = 0xff; h[s * crow + 2] = 0xff; h[s * crow + 3] = 0xff; h[s * crow + 4 + GOFF0] = 1; }
    CK(cudaMemcpy(rows, h, (size_t)batch * crow, cudaMemcpyHostToDevice));
  }
  TqJitArgs a;
  a.src = mode == 1 ? src : dst; a.dst = dst; a.seed = 1; a.p1 = 0; a.p2 = 0;
  a.child_first = 0; a.parent_first = 0; a.arity = mode == 1 ? arity : 1; a.batch = batch;
  a.runsum = runsum; a.rows = rows; a.row_bytes = crow;
  unsigned* xlout; CK(cudaMalloc(&xlout, batch * 4)); a.xlout = xlout; a.tiles = nullptr; a.runsel = nullptr; a.scratch = nullptr;
  a.rep = nullptr; a.prep = nullptr;
  TqCoef cf = {};
  const size_t smem = SMEM;
  if (smem > 48 * 1024) CK(cudaFuncSetAttribute(tq_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const unsigned grid = batch << (n - K);
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  for (int i = 0; i < 3; ++i) tq_pass<<<grid, T, smem>>>(a, cf);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  const int reps = 10;
  for (int i = 0; i < reps; ++i) tq_pass<<<grid, T, smem>>>(a, cf);
  CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); ms /= reps;
  const double bytes = (getenv("TQSIM_JIT_VARIANT") ? (double)batch * S : (double)batch * S * 16) + (double)(mode == 0 ? 0 : (mode == 1 ? nparent : batch)) * S * 16;
  printf("%-28s %8.4f ms  %7.0f GB/s(alg)  grid %u x %d  smem %zu\n", "VARIANT", ms, bytes / (ms * 1e-3) / 1e9, grid, T, smem);
  return 0;
}
'''

VARIANTS = {
    "base": lambda s: s,
    # no phase-exchange barriers' work: drop every fast-path op block (keeps loads/stores/exchanges)
    "nocompute": lambda s: re.sub(r"\n    \{\n(?:      [^\n]*\n)+    \}\n", "\n", s),
    # the store ignores relabelings of out-of-tile qubits (wrong results; timing only)
    "norelabel": lambda s: re.sub(r"gtile_st \|= \(tq_u32\)\(\(t >> (\d+)\) & 1ull\) << \d+;", "", s).replace(
        "  tq_d2* __restrict__ dst =", "  gtile_st = gtile;\n  tq_d2* __restrict__ dst =", 1),
    # no leaf run sums (timing only)
    "nosums": lambda s: re.sub(r"\n    a\.runsum\[[^\n]*", "", s),
    # run sums computed, stores predicated off (never taken)
    "sumsnostore": lambda s: re.sub(r"\n    a\.runsum\[[^\n]*\] = ([^;]*);", r"\n    if (\1 < -1.0) a.runsum[0] = \1;", s),
    # run sums stored to a contiguous per-thread slot (address pattern only)
    "sumsflat": lambda s: re.sub(r"\n    a\.runsum\[[^\n]*\+ (\d+)u\][^\n]*\] = ([^;]*);",
                                 r"\n    a.runsum[((tq_u64)bid * blockDim.x + tid) * 2 + \1] = \2;", s),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("level", type=int)
    ap.add_argument("pass_", type=int)
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--variant", default="base")
    ap.add_argument("--careful", action="store_true")
    ap.add_argument("--src-out", default="")
    ap.add_argument("--src-in", default="", help="use this (edited) kernel source instead")
    args = ap.parse_args()
    import paper_2203_13892_b200.tqsim as T
    from workloads import load_config
    w = load_config(args.config)
    n, gates, noise, shots, ar = T.workload_args(w)
    opts = T.default_options(tile_qubits=args.tile)
    plan = T.tqsim_plan_circuit(n, gates, noise, shots, ar, opts)
    if args.src_in:
        src = open(args.src_in).read()
    else:
        src = T.tqsim_pass_source(n, gates, noise, shots, ar, opts, args.level, args.pass_)
    src = VARIANTS[args.variant](src)
    if args.src_out:
        open(args.src_out, "w").write(src)
    thr = int(re.search(r"__launch_bounds__\((\d+),", src).group(1))
    K = thr.bit_length() - 1 + 4
    mode = 1 if "tq_u64 pj = " in src or "/ a.arity - a.parent_first" in src else (2 if "const tq_d2* src = dst;" in src else 0)
    smem = (16 << K) if "extern __shared__ tq_d2 tile[]" in src else 0
    crow = int(re.search(r"a\.rows \+ \(tq_u64\)s \* (\d+)u", src).group(1))
    goff0 = int(re.search(r"GOFF\[\d+\] = \{(\d+)", src).group(1))
    batch = max(1, (1 << 26) >> n)
    body = (MAIN.replace("N_QUBITS", str(n)).replace("K_TILE", str(K)).replace("THREADS", str(thr))
            .replace("MODE", str(mode)).replace("BATCH", str(batch)).replace("CROW", str(crow))
            .replace("SMEM", str(smem)).replace("CAREFUL", "1" if args.careful else "0")
            .replace("GOFF0", str(goff0))
            .replace("VARIANT", "%s l%d p%d %s%s" % (args.config, args.level, args.pass_, args.variant,
                                                     " careful" if args.careful else "")))
    d = tempfile.mkdtemp()
    cu = os.path.join(d, "h.cu")
    open(cu, "w").write(src.replace('extern "C" __global__', '__global__') + body)
    exe = os.path.join(d, "h")
    r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                        "-o", exe, cu], capture_output=True, text=True)
    if r.returncode:
        print(r.stderr[:3000])
        sys.exit(1)
    if os.environ.get("HARNESS_COMPILE_ONLY"):
        print("compiled", exe)
        return
    if os.environ.get("HARNESS_NCU"):   # --set full capture of one launch of the kernel
        subprocess.run(["ncu", "--set", "full", "--clock-control", "none", "-s", "3", "-c", "1", "-o",
                        os.environ["HARNESS_NCU"], "-f", exe], check=True)
        return
    subprocess.run([exe], check=True)


if __name__ == "__main__":
    main()
