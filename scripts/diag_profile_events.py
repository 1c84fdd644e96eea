import sys, os
sys.path.insert(0, "/root/repo")
import torch
import paper_2203_13892_b200.tqsim as T
from workloads import load_config
for cfg in ["c2_qft15", "c4_qaoa24"]:
    w = load_config(cfg)
    n, gates, noise, shots, ar = T.workload_args(w)
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    for prof in (1, 0):
        h = T.tqsim_create(n, gates, noise, shots, ar, T.default_options(profile=prof))
        ws = torch.empty(h.workspace_bytes(0, 1), dtype=torch.uint8, device=dev)
        out = torch.zeros(h.plan.n_outcomes, dtype=torch.int32, device=dev)
        h.execute(0, 0, 1, st.cuda_stream, ws.data_ptr(), ws.numel(), out.data_ptr())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        h.execute(1, 0, 1, st.cuda_stream, ws.data_ptr(), ws.numel(), out.data_ptr())
        e1.record(st)
        torch.cuda.synchronize()
        s = h.stats()
        print(cfg, "profile", prof, "total %.3f ms" % e0.elapsed_time(e1), "pass %.3f meas %.3f noise %.3f" % (s.pass_ms, s.measure_ms, s.noise_ms),
              "launches", s.kernel_launches, "pass GB/s %.0f" % (s.pass_bytes / (s.pass_ms * 1e-3) / 1e9 if s.pass_ms else 0), flush=True)
        h.close()
