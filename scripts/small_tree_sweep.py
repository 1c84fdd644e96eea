"""Small-state tree kernel vs the general tree engine: device time per tree
(CUDA events around K replays of tqsim_execute on one stream) for a sweep of widths and
shot counts; one JSON line per case.  Calibrates options.small_tree's auto threshold.
    python scripts/small_tree_sweep.py > gpurun_out/small_sweep.jsonl
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_13892_b200.tqsim as T  # noqa: E402
from workloads import load_config, qft_gates, random_circuit  # noqa: E402


def time_tree(n, gates, noise, shots, ar, small, steps=20):
    h = T.tqsim_create(n, gates, noise, shots, ar, T.default_options(small_tree=small))
    N = int(h.plan.n_outcomes)
    ws = torch.empty(max(1, h.workspace_bytes(0, 1)), dtype=torch.uint8, device="cuda")
    out = torch.zeros(N, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream()
    for i in range(3):
        h.execute(100 + i, 0, 1, st.cuda_stream, ws.data_ptr(), ws.numel(), out.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(steps):
        h.execute(i, 0, 1, st.cuda_stream, ws.data_ptr(), ws.numel(), out.data_ptr())
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    plan = h.plan
    launches = int(h.stats().kernel_launches)
    h.close()
    return ms, plan, launches


cases = []
w = load_config("c1_qft5")
n, gates, noise, shots, ar = T.workload_args(w)
cases.append(("c1_qft5", n, gates, noise, shots, ar))
rng = np.random.default_rng(1)
for n in (6, 8, 10):
    g = qft_gates(n)
    for shots, ar in ((1000, [10, 100]), (10000, [20, 500]), (100000, [100, 1000])):
        cases.append(("qft%d_%d" % (n, shots), n, g, T.noise_arg(0.001, 0.01, 0.01, 0.01), shots, ar))
    g = random_circuit(n, 200, rng)
    cases.append(("rand%d_200g_10k" % n, n, g, T.noise_arg(0.001, 0.01, 0.01, 0.01), 10000, [20, 500]))
for name, n, g, nz, shots, ar in cases:
    ms1, p1, l1 = time_tree(n, g, nz, shots, ar, 1)
    ms2, p2, l2 = time_tree(n, g, nz, shots, ar, 2)
    flat = int(p1.n_outcomes) * int(p1.n_lowered_gates) * (1 << max(n, 5))
    print(json.dumps({"case": name, "n": n, "outcomes": int(p1.n_outcomes), "lowered_gates": int(p1.n_lowered_gates),
                      "arities": p1.arity_list, "flat_work": flat, "log2_flat_work": round(float(np.log2(flat)), 2),
                      "small_ms": round(ms1, 4), "general_ms": round(ms2, 4), "small_launches": l1,
                      "general_launches": l2, "speedup_small": round(ms2 / ms1, 3)}), flush=True)
