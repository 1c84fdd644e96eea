"""Predict a tree's device time from isolated per-pass kernel times (pass_harness) x the
number of launches of each pass (plan instances / batch), to cross-check in-app timing.
    python scripts/microbench/tree_from_harness.py c4_qaoa24
"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2203_13892_b200.tqsim as T  # noqa: E402
from workloads import load_config  # noqa: E402

cfg = sys.argv[1]
w = load_config(cfg)
n, gates, noise, shots, ar = T.workload_args(w)
p = T.tqsim_plan_circuit(n, gates, noise, shots, ar)
inst = 1
batch = max(1, (1 << 26) >> n)
total = 0.0
for d in range(p.n_levels):
    inst = inst * p.arities[d]
    launches = -(-inst // batch)
    frac_last = (inst - (launches - 1) * batch) / batch
    q = 0
    while True:
        try:
            T.tqsim_pass_source(n, gates, noise, shots, ar, None, d, q)
        except T.TqsimError:
            break
        out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts/microbench/pass_harness.py"), cfg, str(d), str(q)],
                             capture_output=True, text=True).stdout
        ms = float(re.search(r"\s([0-9.]+) ms", out).group(1))
        t = ms * ((launches - 1) + frac_last)
        total += t
        print("level %d pass %d: %.4f ms x %d launches -> %.1f ms" % (d, q, ms, launches, t), flush=True)
        q += 1
print("predicted pass time per tree: %.1f ms" % total)
