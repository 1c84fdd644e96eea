"""N>1 host path on CPU (gloo, world_size 2, 3 and 8): shard ranges from the C ABI
(tqsim_shard_range / tqsim_shard_levels: split at the first level whose
instance count the world divides, ancestors recomputed), per-rank leaf outcomes (the
oracle stands in for each rank's GPU shard, as no GPU is available here), the
product's all_reduce(SUM) combine and histogram.  The combined array must equal the
single-process oracle run bit for bit."""
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
        split, lo, hi = T.tqsim_shard_levels(plan, rank, world)
        assert (lo[0], hi[0], lo[-1], hi[-1]) == (t0, t1, l0, l1)
        res = simulate_tree(n, low, oplan, nm, 5, top_range=(t0, t1))
        out = torch.zeros(int(plan.n_outcomes), dtype=torch.int32)
        mine = {l: r for l, r in res.leaves.items() if l0 <= l < l1}
        assert sorted(mine) == list(range(l0, l1))
        for l, r in mine.items():
            out[l] = r.outcome
        cnt = torch.tensor([l1 - l0], dtype=torch.int64)
        dist.all_reduce(cnt, op=dist.ReduceOp.MAX)       # balance: the largest shard
        top = int(cnt.item())
        combine(out)
        if rank == 0:
            full = simulate_tree(n, low, oplan, nm, 5)
            want = full.outcome_array(int(plan.n_outcomes))
            ok = np.array_equal(out.numpy().astype(np.uint32), want)
            h = histogram(out.numpy())
            hw = {}
            for v in want:
                hw[int(v)] = hw.get(int(v), 0) + 1
            result_q.put((ok, h == hw, int(plan.n_outcomes), split, top))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,arities,split", [(2, [6, 10], 0), (3, [5, 3, 4], 1), (2, [1, 60], 1),
                                                (8, [20, 2, 2], 1), (3, [20, 2, 2], 2)])
def test_gloo_sharded_combine_equals_single_run(world, arities, split):
    """A_0 = 20 at W = 8 (C2/C3's top level): split at level 1 (40 instances, 5 per rank),
    so every rank gets exactly 1/8 of the leaves; W = 3 splits where >= 16 W instances."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_worker, args=(world, _free_port(), arities, q), nprocs=world, join=True)
    ok, hist_ok, n_out, got_split, largest = q.get(timeout=120)
    assert ok and hist_ok and n_out == int(np.prod(arities))
    assert got_split == split
    if n_out % world == 0 and split < len(arities):
        per = int(np.prod(arities[:split + 1]))
        if per % world == 0:
            assert largest == n_out // world          # perfect balance
