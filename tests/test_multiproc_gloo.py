"""N>1 host path on CPU (gloo, world_size 2 and 3): shard ranges from the C ABI,
per-rank leaf outcomes (the oracle stands in for each rank's GPU shard, as no
GPU is available here), the product's all_reduce(SUM) combine and histogram.
The combined array must equal the single-process oracle run bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, arities, result_q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2203_13892_b200.tqsim as T
        from paper_2203_13892_b200.distributed import combine, histogram
        from oracle import gates as OG
        from oracle.planner import Plan
        from oracle.tree import NoiseModel, simulate_tree
        from workloads import load_config

        w = load_config("c1_qft5")
        n, gates, noise, shots, _ = T.workload_args(w)
        plan = T.tqsim_plan_circuit(n, gates, noise, 60, arities)
        t0, t1, l0, l1 = T.tqsim_shard_range(plan, rank, world)
        oplan = Plan(plan.arity_list, plan.boundary_list)
        nm = NoiseModel(0.03, 0.08, 0.02, 0.02)
        low = OG.lower(gates)
        res = simulate_tree(n, low, oplan, nm, 5, top_range=(t0, t1))
        out = torch.zeros(int(plan.n_outcomes), dtype=torch.int32)
        for l, r in res.leaves.items():
            assert l0 <= l < l1
            out[l] = r.outcome
        combine(out)
        if rank == 0:
            full = simulate_tree(n, low, oplan, nm, 5)
            want = full.outcome_array(int(plan.n_outcomes))
            ok = np.array_equal(out.numpy().astype(np.uint32), want)
            h = histogram(out.numpy())
            hw = {}
            for v in want:
                hw[int(v)] = hw.get(int(v), 0) + 1
            result_q.put((ok, h == hw, int(plan.n_outcomes)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,arities", [(2, [6, 10]), (3, [5, 3, 4]), (2, [1, 60])])
def test_gloo_sharded_combine_equals_single_run(world, arities):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_worker, args=(world, _free_port(), arities, q), nprocs=world, join=True)
    ok, hist_ok, n_out = q.get(timeout=60)
    assert ok and hist_ok and n_out == int(np.prod(arities))
