"""Host enqueue time of tqsim_execute vs device time (is the tree launch-bound?)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_13892_b200.tqsim as T
from workloads import load_config
for cfg in sys.argv[1:] or ["c2_qft15", "c4_qaoa24"]:
    w = load_config(cfg)
    n, gates, noise, shots, ar = T.workload_args(w)
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    h = T.tqsim_create(n, gates, noise, shots, ar, T.default_options())
    ws = torch.empty(h.workspace_bytes(0, 1), dtype=torch.uint8, device=dev)
    out = torch.zeros(h.plan.n_outcomes, dtype=torch.int32, device=dev)
    for i in range(2):
        h.execute(i, 0, 1, st.cuda_stream, ws.data_ptr(), ws.numel(), out.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    t0 = time.perf_counter()
    h.execute(7, 0, 1, st.cuda_stream, ws.data_ptr(), ws.numel(), out.data_ptr())
    t_enq = time.perf_counter() - t0
    e1.record(st)
    torch.cuda.synchronize()
    t_all = time.perf_counter() - t0
    print(cfg, "GRAPH=%s" % os.environ.get("TQSIM_GRAPH", "1"), "enqueue %.3f ms" % (t_enq * 1e3),
          "device %.3f ms" % e0.elapsed_time(e1), "wall %.3f ms" % (t_all * 1e3), "launches", h.stats().kernel_launches, flush=True)
    h.close()
