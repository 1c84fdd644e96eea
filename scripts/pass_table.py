"""Per-pass table of one config (tqsim_profile_passes): level, pass, states per launch,
launches per tree, ms per launch, algorithmic GB/s, ms per tree.

    python scripts/pass_table.py c4_qaoa24 [--tile K]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--shard", default="0/1", help="r/w: this shard of the tree only")
    args = ap.parse_args()
    import torch
    import paper_2203_13892_b200.tqsim as T
    from workloads import load_config
    w = load_config(args.config)
    n, gates, noise, shots, ar = T.workload_args(w)
    h = T.tqsim_create(n, gates, noise, shots, ar, T.default_options(tile_qubits=args.tile))
    rk, wd = (int(v) for v in args.shard.split("/"))
    ws = torch.empty(h.workspace_bytes(rk, wd), dtype=torch.uint8, device="cuda")
    out = torch.zeros(h.plan.n_outcomes, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    h.execute(1, rk, wd, st, ws.data_ptr(), ws.numel(), out.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in range(1 if wd > 1 else 3):
        h.execute(2 + s, rk, wd, st, ws.data_ptr(), ws.numel(), out.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    step = e0.elapsed_time(e1) / (1 if wd > 1 else 3)
    rows = h.profile_passes(1, rk, wd, st, ws.data_ptr(), ws.numel(), out.data_ptr())
    tot = 0.0
    print("%-5s %-4s %6s %10s %10s %8s %9s" % ("level", "pass", "states", "launch/tr", "ms/launch", "GB/s", "ms/tree"))
    for r in rows:
        mt = r.launches_per_tree * r.ms_per_launch
        tot += mt
        print("%-5d %-4d %6d %10.2f %10.4f %8.0f %9.3f" % (r.level, r.pass_, r.states_per_launch, r.launches_per_tree,
                                                        r.ms_per_launch, r.alg_bytes_per_launch / r.ms_per_launch / 1e6, mt))
    print("passes %.3f ms/tree of step %.3f ms (%.3f)" % (tot, step, tot / step))
    h.close()


if __name__ == "__main__":
    main()
