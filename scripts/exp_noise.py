"""Experiment: gate-pass time vs noise level at a FIXED plan (fast vs careful CTA paths).

    python scripts/exp_noise.py c2_qft15
"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_13892_b200.tqsim as T
from workloads import load_config

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2_qft15"
w = load_config(cfg)
n, gates, noise, shots, ar = T.workload_args(w)
h0 = T.tqsim_create(n, gates, noise, shots, ar, T.default_options())
arities = h0.plan.arity_list
h0.close()
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
for scale in [0.0, 1.0, 2.0, 1000.0]:
    nz = T.noise_arg(min(1.0, w.p1 * scale), min(1.0, w.p2 * scale), w.readout_p01, w.readout_p10)
    h = T.tqsim_create(n, gates, nz, shots, arities, T.default_options(profile=1))
    ws = torch.empty(h.workspace_bytes(0, 1), dtype=torch.uint8, device=dev)
    out = torch.zeros(h.plan.n_outcomes, dtype=torch.int32, device=dev)
    for i in range(2):
        h.execute(i, 0, 1, st.cuda_stream, ws.data_ptr(), ws.numel(), out.data_ptr())
    tot = 0.0
    for i in range(3):
        h.execute(10 + i, 0, 1, st.cuda_stream, ws.data_ptr(), ws.numel(), out.data_ptr())
        s = h.stats()
        tot += s.pass_ms
    s = h.stats()
    print("%s scale %g: pass_ms %.3f  alg GB/s %.0f  measure_ms %.3f" % (cfg, scale, tot / 3, s.pass_bytes / (tot / 3 * 1e-3) / 1e9, s.measure_ms), flush=True)
    h.close()
