#!/usr/bin/env python3
"""Throughput bench of the TQSim B200 hot path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2_qft15] [--impl tqsim|reference]

A step = one whole tree run (every §8(a) row: noise draws, fan-out, gate
passes, leaf measurement, readout; + the NCCL allreduce of leaf outcomes when
N > 1) of BASELINE.json's config (default configs[1] = C2 qft15, 10,000 shots ->
10,240 outcomes).  Top-level branches are sharded over ranks (weak scaling of
the number of trees: every rank runs its shard of one tree per step, so the
job does one tree per step; "scaling": "strong").

value     noisy shots/s = outcomes per tree * K / (max over ranks of the CUDA-event
          time of K steps), inputs (gate tables) resident in HBM.
e2e       the same metric through the C-ABI call a user makes (tqsim_run for N=1:
          host circuit in, host histogram out; planning, H2D of the gate tables,
          D2H of the outcomes and the histogram inside the timed region).
roofline  gate-pass kernels: algorithmic bytes / CUDA-event time of every distinct pass
          kernel (5 back-to-back launches on its in-tree operands, tqsim_profile_passes),
          weighted by its launches per tree, vs MEASURED_PEAKS.json hbm_gbs.
cpu_baseline  the oracle (oracle/, numpy, 1 thread) on a bounded sample of the
          same workload (the first leaves of its DFS, ~20 s), rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "noisy shots/sec and gate-amp updates/s; gate-kernel HBM GB/s vs B200 peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2_qft15")
    ap.add_argument("--impl", default="tqsim", choices=["tqsim", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--batch-log2", type=int, default=0)
    ap.add_argument("--shard", default="", help="r/w: time only shard r of w (single-GPU experiments)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + q,
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        self.f.flush()
        rows = []
        try:
            with open(self.f.name) as fh:
                for line in fh:
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) >= 9 and parts[1].replace(".", "").isdigit():
                        rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][2]),
                "reasons": reasons, "samples": len(rows)}


def cpu_baseline(w, budget_s: float = 20.0):
    """The oracle as it stands (numpy, 1 thread) on a bounded sample of the workload: the
    oracle's own slice / leaf functions (oracle/tree.py) driven in the same DFS order as
    oracle.tree.simulate_tree (state reuse), stopped at the first leaf after `budget_s`
    seconds.  Widths above 22 qubits are not sampled (one oracle slice takes minutes)."""
    from threadpoolctl import threadpool_limits

    from oracle import gates as OG
    from oracle.planner import dcp_plan, fixed_plan
    from oracle.statevector import zero_state
    from oracle.tree import NoiseModel, error_rates, run_slice, sample_leaf

    n = w.circuit.n_qubits
    if n > 22:
        return {"value": None, "unit": "shots/s", "cores": 1, "kind": "oracle",
                "sample": "not sampled: %d qubits (one oracle slice takes minutes on one core)" % n}
    low = OG.lower(w.circuit.gates)
    nm = NoiseModel(w.p1, w.p2, w.readout_p01, w.readout_p10)
    if w.arities:
        plan = fixed_plan(len(low), w.arities)
    else:
        plan = dcp_plan(error_rates(low, nm), w.shots, n, w.copy_cost_gates)
    A, B, L = plan.arities, plan.boundaries, len(plan.arities)
    leaves = 0

    class Done(Exception):
        pass

    with threadpool_limits(1):
        t0 = time.perf_counter()

        def node(d, j, parent):
            nonlocal leaves
            psi = run_slice(parent.copy(), n, low, B[d], B[d + 1], j, w.seed, nm)
            if d == L - 1:
                sample_leaf(psi, n, j, w.seed, nm)
                leaves += 1
                if time.perf_counter() - t0 > budget_s:
                    raise Done
                return
            for br in range(A[d + 1]):
                node(d + 1, j * A[d + 1] + br, psi)

        try:
            for j0 in range(A[0]):
                node(0, j0, zero_state(n))
        except Done:
            pass
        dt = time.perf_counter() - t0
    return {"value": leaves / dt, "unit": "shots/s", "cores": 1, "kind": "oracle",
            "sample": "first %d leaves (DFS order, state reuse) of the %d-leaf tree of %s, %.1f s"
                      % (leaves, plan.n_outcomes, w.name, dt)}


def run_reference(args, w, rank, world):
    if rank != 0:
        return
    for _ in range(args.warmup if args.warmup < 1 else 1):
        pass
    vals = []
    cb = None
    for s in range(args.steps):
        cb = cpu_baseline(w, budget_s=10.0)
        if cb["value"] is None:
            print(json.dumps({"impl": "reference", "unavailable": cb["sample"]}), flush=True)
            return
        vals.append(cb["value"])
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "shots/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": None, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "shots": w.shots},
            "cpu_baseline": {"value": v, "unit": "shots/s", "cores": 1, "kind": "oracle",
                             "sample": cb["sample"]},
            "e2e": {"value": v, "unit": "shots/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    from workloads import load_config
    w = load_config(args.config)
    if args.impl == "reference":
        return run_reference(args, w, rank, world)

    import torch
    import torch.distributed as dist
    import paper_2203_13892_b200.tqsim as T

    if args.shard and world == 1:
        rank, world_override = (int(v) for v in args.shard.split("/"))
    else:
        world_override = None
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    n, gates, noise, shots, ar = T.workload_args(w)
    opts = T.default_options(tile_qubits=args.tile, batch_log2_amps=args.batch_log2)
    h = T.tqsim_create(n, gates, noise, shots, ar, opts)
    plan = h.plan
    N = int(plan.n_outcomes)
    xw = world_override or world          # shards the tree is cut into
    ws = torch.empty(h.workspace_bytes(rank, xw), dtype=torch.uint8, device=dev)
    out = torch.zeros(N, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream(dev)

    def step(seed):
        out.zero_()
        h.execute(seed, rank, xw, st.cuda_stream, ws.data_ptr(), ws.numel(), out.data_ptr())
        if world > 1:
            dist.all_reduce(out, op=dist.ReduceOp.SUM)

    for i in range(args.warmup):
        step(1000 + i)
    torch.cuda.synchronize(dev)
    stats1 = h.stats()
    launches_per_step = int(stats1.kernel_launches)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(st)
        for i in range(args.steps):
            step(i)
        e1.record(st)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    clocks = clk.summary()

    # roofline of the gate-pass kernel family: every distinct pass kernel timed live with
    # CUDA events on this stream over back-to-back launches on its in-tree operands
    # (tqsim_profile_passes), weighted by its launches per tree.  (Per-launch events
    # around every kernel of the tree under-measured the kernels by ~25% on B200 --
    # their sum disagreed with the step time and the ncu launch list -- so they are not used.)
    timings = h.profile_passes(0, rank, xw, st.cuda_stream, ws.data_ptr(), ws.numel(), out.data_ptr(), reps=5)
    pass_ms = sum(t.ms_per_launch * t.launches_per_tree for t in timings)
    pass_bytes = sum(t.alg_bytes_per_launch * t.launches_per_tree for t in timings)
    pass_launches = sum(t.launches_per_tree for t in timings)
    top = max(timings, key=lambda t: t.ms_per_launch * t.launches_per_tree)
    hbm_peak, peak_src = peaks()
    achieved = pass_bytes / (pass_ms * 1e-3) / 1e9 if pass_ms > 0 else 0.0
    top_achieved = top.alg_bytes_per_launch / (top.ms_per_launch * 1e-3) / 1e9

    # end to end through the public API with HOST buffers: N=1 the north_star call
    # tqsim_run (host circuit in -> lowering, planning, kernel-cache lookup, tree, D2H of
    # the outcomes, host histogram); N>1 each rank: tqsim_create + tqsim_execute of its
    # shard + all_reduce + D2H + histogram on rank 0.
    e2e = None
    if not args.no_e2e and not args.shard:
        from paper_2203_13892_b200.distributed import histogram
        if world == 1:
            ca = T.CircuitArg(n, gates)                     # the user's circuit, marshalled once
            tc = time.perf_counter()
            T.tqsim_run(n, ca, noise, shots, ar, 0)         # first call: plan + codegen + arena
            first_call_s = time.perf_counter() - tc
            t0 = time.perf_counter()
            for i in range(args.steps):
                T.tqsim_run(n, ca, noise, shots, ar, i)
            dt = time.perf_counter() - t0
        else:
            from paper_2203_13892_b200.distributed import ShardRunner
            host = torch.empty(N, dtype=torch.int32, pin_memory=True)
            runner = ShardRunner(h, rank, world, dev)      # the multi-GPU public API

            def e2e_step(seed):
                res = runner.run(seed, stream=st)              # shard + NCCL all_reduce(SUM)
                host.copy_(res)                                # D2H of the combined outcomes
                if rank == 0:
                    histogram(host.numpy())

            e2e_step(0)
            dist.barrier()
            t0 = time.perf_counter()
            for i in range(args.steps):
                e2e_step(i)
            dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            dt = float(dt.item())
        n_low = len(T.tqsim_lower_circuit(n, gates))
        if world > 1:
            first_call_s = None
        if world == 1:
            note = ("tqsim_run per step: host circuit in (validated, hashed; the prepared plan and its "
                    "specialized kernels are reused from the library's plan cache after the first call), "
                    "h2d = per-gate noise-class and pass tables (2 B / lowered gate) + kernel parameters, "
                    "d2h = leaf outcomes (uint32) into page-locked memory, host histogram (C; returned as arrays, the dict view of Result.counts is built on first access)")
            h2d = 2 * n_low + 96 * launches_per_step
        else:
            note = ("distributed.ShardRunner per step on every rank: the shard (replayed CUDA graph), "
                    "NCCL all_reduce(SUM) of the leaf outcomes, D2H, histogram on rank 0; h2d = kernel "
                    "parameters (seed); max over ranks")
            h2d = 96
        e2e = {"value": N * args.steps / dt, "unit": "shots/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": N * 4, "note": note,
               "first_call_s": first_call_s}
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic_%s.json" % w.name)
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(w)

    if rank == 0:
        shots_s = N * args.steps / (ms * 1e-3)
        gau = plan.gate_amp_updates * args.steps / (ms * 1e-3)
        line = {
            "metric": METRIC, "value": shots_s, "unit": "shots/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "n_qubits": n, "shots": shots, "outcomes": N,
                       "arities": plan.arity_list, "lowered_gates": int(plan.n_lowered_gates),
                       "tile_qubits": int(plan.tile_qubits),
                       "l2": "inputs larger than L2 (state batches >= 1 GiB per launch group)",
                       "parallelism": "top-level branch sharding x%d" % world},
            "gate_amp_updates_per_s": gau,
            "tree_vs_flat_gate_ratio": plan.flat_gate_amp_updates / plan.gate_amp_updates,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak if hbm_peak else None,
                         "traffic": traffic["dram_bytes_per_launch"] if traffic else None,
                         "traffic_source": traffic["source"] if traffic else None,
                         "alg_bytes_same_launch": traffic["alg_bytes_per_launch"] if traffic else None,
                         "peak_source": peak_src,
                         "kernel": "tq_pass_l*_p* (run-time specialized gate pass, all launches, "
                                   "weighted by launches per tree)",
                         "method": "per-kernel CUDA events over 5 back-to-back launches on in-tree operands",
                         "pass_ms_per_step": pass_ms,
                         "pass_share_of_step": pass_ms / (ms / args.steps),
                         "alg_bytes_per_launch": pass_bytes / pass_launches if pass_launches else None,
                         "pass_launches_per_step": pass_launches,
                         "top_kernel": {"name": "tq_pass_l%d_p%d" % (top.level, top.pass_),
                                        "ms_per_launch": top.ms_per_launch,
                                        "launches_per_step": top.launches_per_tree,
                                        "achieved_gbs": top_achieved, "frac": top_achieved / hbm_peak}},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    h.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
