#!/usr/bin/env python3
"""One tree of a config through tqsim_profile_tree (every launch in tree order, no graph) --
the command the ncu launch lists / full captures of round 2 wrap (scripts/ncu_call.sh).

    python scripts/ncu_tree.py <config> <out.json> [--shard r/w]

Writes the per-kernel-family in-tree record (launches, states, computed states, CUDA-event
ms, algorithmic bytes) so profiles/ncu_join.py can divide ncu's per-launch DRAM bytes and
FP64 instruction counts by the work the same launches did (seed 0, as bench.py profiles)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2203_13892_b200.tqsim as T  # noqa: E402
from workloads import load_config  # noqa: E402


def main():
    cfg, out_path = sys.argv[1], sys.argv[2]
    r, w = 0, 1
    if len(sys.argv) > 4 and sys.argv[3] == "--shard":
        r, w = (int(v) for v in sys.argv[4].split("/"))
    wl = load_config(cfg)
    n, gates, noise, shots, ar = T.workload_args(wl)
    h = T.tqsim_create(n, gates, noise, shots, ar)
    ws = torch.empty(h.workspace_bytes(r, w), dtype=torch.uint8, device="cuda")
    out = torch.zeros(int(h.plan.n_outcomes), dtype=torch.int32, device="cuda")
    prof = h.profile_tree(0, r, w, torch.cuda.current_stream().cuda_stream, ws.data_ptr(), ws.numel(),
                          out.data_ptr())
    recs = [{"kind": k.kind, "level": k.level, "pass": k.pass_, "launches": k.launches, "states": k.states,
             "computed_states": k.computed_states, "ms": k.ms, "alg_bytes": k.alg_bytes,
             "nominal_bytes": k.nominal_bytes, "fp64_per_amp_model": k.fp64_per_amp} for k in prof]
    json.dump({"config": cfg, "n_qubits": n, "shard": [r, w], "families": recs}, open(out_path, "w"), indent=1)
    print("ok", len(recs), "families", sum(k.launches for k in prof), "launches")


if __name__ == "__main__":
    main()
