"""Do per-launch CUDA events account for a tree's time?  Launch two generated pass
kernels (from different modules / sources) back to back, alternating, on a 1 GiB
batch; compare the sum of per-launch event intervals with the total, and with the
same kernel repeated.  python scripts/microbench/switch_harness.py <config> lA pA lB pB
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
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("cuda %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)
template <class Kern> void setsm(Kern k, size_t smem) { if (smem > 48 * 1024) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); }
int main() {
  const size_t S = (size_t)1 << NQ; const unsigned batch = BATCH;
  tq_d2 *src, *dst; unsigned char* rows; double* runsum;
  CK(cudaMalloc(&src, batch * S * 16)); CK(cudaMalloc(&dst, batch * S * 16));
  CK(cudaMalloc(&rows, (size_t)batch * 1024)); CK(cudaMalloc(&runsum, batch * (S / 8) * 8));
  CK(cudaMemset(src, 0, batch * S * 16)); CK(cudaMemset(dst, 0, batch * S * 16)); CK(cudaMemset(rows, 0, (size_t)batch * 1024));
  TqJitArgs a; a.src = src; a.dst = dst; a.seed = 1; a.p1 = 0; a.p2 = 0; a.child_first = 0; a.parent_first = 0;
  a.arity = 2; a.batch = batch; a.runsum = runsum; a.rows = rows; a.row_bytes = CROWA;
  TqJitArgs b = a; b.row_bytes = CROWB; b.arity = 2;
  TqCoef_A ca = {}; TqCoef_B cb = {};
  setsm(tq_passA, SMEMA); setsm(tq_passB, SMEMB);
  const unsigned ga = batch << (NQ - KA), gb = batch << (NQ - KB);
  const int R = 20;
  cudaEvent_t ev[2 * R + 1]; for (auto& evx : ev) CK(cudaEventCreate(&evx));
  for (int mode = 0; mode < 3; ++mode) {   // 0: A A A..., 1: B B B..., 2: A B A B ...
    for (int i = 0; i < 4; ++i) { tq_passA<<<ga, TA, SMEMA>>>(a, ca); tq_passB<<<gb, TB, SMEMB>>>(b, cb); }
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(ev[0]));
    for (int i = 0; i < 2 * R; ++i) {
      const bool useA = mode == 0 || (mode == 2 && (i & 1) == 0);
      if (useA) tq_passA<<<ga, TA, SMEMA>>>(a, ca); else tq_passB<<<gb, TB, SMEMB>>>(b, cb);
      CK(cudaEventRecord(ev[i + 1]));
    }
    CK(cudaEventSynchronize(ev[2 * R])); CK(cudaGetLastError());
    float tot; CK(cudaEventElapsedTime(&tot, ev[0], ev[2 * R]));
    double sa = 0, sb = 0; int na = 0, nb = 0;
    for (int i = 0; i < 2 * R; ++i) { float m; CK(cudaEventElapsedTime(&m, ev[i], ev[i + 1]));
      const bool useA = mode == 0 || (mode == 2 && (i & 1) == 0); if (useA) { sa += m; ++na; } else { sb += m; ++nb; } }
    printf("mode %s: total %.3f ms for %d launches; mean event interval A %.4f B %.4f ms\n",
           mode == 0 ? "A-only" : mode == 1 ? "B-only" : "A/B alternating", tot, 2 * R, na ? sa / na : 0, nb ? sb / nb : 0);
  }
  return 0;
}
'''


def main():
    cfg, la, pa, lb, pb = sys.argv[1], *map(int, sys.argv[2:6])
    import paper_2203_13892_b200.tqsim as T
    from workloads import load_config
    w = load_config(cfg)
    n, gates, noise, shots, ar = T.workload_args(w)
    srcs = []
    info = []
    for tag, (l, p) in (("A", (la, pa)), ("B", (lb, pb))):
        s = T.tqsim_pass_source(n, gates, noise, shots, ar, None, l, p)
        thr = int(re.search(r"__launch_bounds__\((\d+),", s).group(1))
        K = thr.bit_length() - 1 + 4
        smem = (16 << K) if "extern __shared__ tq_d2 tile[]" in s else 0
        crow = int(re.search(r"a\.rows \+ \(tq_u64\)s \* (\d+)u", s).group(1))
        body = s[s.index("struct TqCoef"):]
        body = (body.replace("struct TqCoef", "struct TqCoef_" + tag).replace("const TqCoef cf", "const TqCoef_%s cf" % tag)
                .replace('extern "C" __global__', "__global__").replace(" tq_pass(", " tq_pass%s(" % tag)
                .replace("GOFF", "GOFF_" + tag).replace("ERRX", "ERRX_" + tag).replace("ERRZ", "ERRZ_" + tag)
                .replace("GD[", "GD_%s[" % tag).replace("GD +", "GD_%s +" % tag))
        prelude = s[:s.index("struct TqCoef")]
        srcs.append(body)
        info.append((thr, K, smem, crow))
    batch = max(1, (1 << 26) >> n)
    m = (MAIN.replace("NQ", str(n)).replace("BATCH", str(batch)).replace("CROWA", str(info[0][3]))
         .replace("CROWB", str(info[1][3])).replace("SMEMA", str(info[0][2])).replace("SMEMB", str(info[1][2]))
         .replace("KA", str(info[0][1])).replace("KB", str(info[1][1])).replace("TA", str(info[0][0]))
         .replace("TB", str(info[1][0])))
    d = tempfile.mkdtemp()
    cu = os.path.join(d, "s.cu")
    open(cu, "w").write(prelude + srcs[0] + srcs[1] + m)
    exe = os.path.join(d, "s")
    r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-o", exe, cu],
                       capture_output=True, text=True)
    if r.returncode:
        print(r.stderr[:3000])
        sys.exit(1)
    if os.environ.get("HARNESS_COMPILE_ONLY"):
        print("compiled", exe)
        return
    subprocess.run([exe], check=True)


if __name__ == "__main__":
    main()
