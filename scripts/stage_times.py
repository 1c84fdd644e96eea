"""Device time per stage of one tree (profile mode: CUDA events around every pass /
measurement / noise launch, serialised, no graph): pass_ms, measure_ms, noise_ms.

    python scripts/stage_times.py c4_qaoa24
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2203_13892_b200.tqsim as T
    from workloads import load_config
    w = load_config(sys.argv[1])
    n, gates, noise, shots, ar = T.workload_args(w)
    h = T.tqsim_create(n, gates, noise, shots, ar, T.default_options(profile=1))
    ws = torch.empty(h.workspace_bytes(), dtype=torch.uint8, device="cuda")
    out = torch.zeros(h.plan.n_outcomes, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for seed in (1, 2):
        h.execute(seed, 0, 1, st, ws.data_ptr(), ws.numel(), out.data_ptr())
        torch.cuda.synchronize()
        s = h.stats()
        print("%s seed %d: pass_ms %.3f measure_ms %.3f noise_ms %.3f launches %d" %
              (sys.argv[1], seed, s.pass_ms, s.measure_ms, s.noise_ms, s.kernel_launches))
    h.close()


if __name__ == "__main__":
    main()
