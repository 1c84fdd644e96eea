#!/usr/bin/env python3
"""Throughput bench of the TQSim B200 hot path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4_qaoa24] [--impl tqsim|reference]

A step = one whole tree run (every §8(a) row: noise draws, fan-out, gate passes, leaf
measurement, readout; + the NCCL allreduce of leaf outcomes when N > 1) of the workload.
Default workload: C4 (QAOA-24 MaxCut, 8,192 shots -> 8,192 outcomes, BASELINE.json
configs[3]) -- the largest config whose whole tree runs on one GPU in a step (C5's tree
is 4 GiB states x 65,408 node executions; it runs as shards, `--config c5_hea28 --shard r/w`).
N > 1: the tree is split over the ranks at the first level whose instance count N divides
(tqsim_shard_levels); every rank runs its shard of one tree per step, the job one tree per
step ("scaling": "strong").  Without WORLD_SIZE in the environment, --gpus N > 1 re-launches
itself under torch.distributed.run with N processes (one per GPU).

value     noisy shots/s = outcomes per tree * K / (max over ranks of the CUDA-event time
          of K steps), inputs (gate tables) resident in HBM.
e2e       the same metric through the C-ABI call a user makes (tqsim_run for N=1: host
          circuit in, host histogram out; validation, plan-cache lookup, H2D of the gate
          tables, the tree, D2H of the outcomes and the histogram in the timed region).
roofline  the dominant kernel (the gate-pass kernel family (level, pass) with the largest
          in-tree device time): algorithmic bytes of the instances it computed / its summed
          CUDA-event time, every launch of one tree timed in tree order (tqsim_profile_tree),
          vs MEASURED_PEAKS.json hbm_gbs; an FP64 view beside it.
cpu_baseline  the oracle (oracle/, numpy) on os.cpu_count() processes over disjoint top-level
          subtrees, ~20 s, rank 0 only; widths whose single leaf takes longer than the budget
          report the measured oracle gate-amplitude rate extrapolated to shots/s.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "noisy shots/sec and gate-amp updates/s; gate-kernel HBM GB/s vs B200 peak"
DEFAULT_CONFIG = "c4_qaoa24"
# FP64 ALU ceiling: 148 SMs x 64 DFMA/clk/SM (sm_100 FP64 pipe) x clock
FP64_DFMA_PER_CLK_SM = 64
N_SM = 148


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--impl", default="tqsim", choices=["tqsim", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-dedup-steps", type=int, default=2,
                    help="also time this many steps with options.no_dedup=1 (0 = skip)")
    ap.add_argument("--flat-shots", type=int, default=0,
                    help="time the flat baseline on this many shots (0 = auto: all for n <= 16, else "
                         "min(shots, 1024); -1 = skip)")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--batch-log2", type=int, default=0)
    ap.add_argument("--copy-cost", type=float, default=10.0,
                    help="DCP first-slice length (copy cost in gates, R14); -1 = the fused fan-out's cost")
    ap.add_argument("--small-tree", type=int, default=0,
                    help="options.small_tree: 0 auto, 1 on (n <= 10), 2 off (DESIGN.md §6.4)")
    ap.add_argument("--shard", default="", help="r/w: time only shard r of w (single-GPU experiments)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", float(d.get("sm_max_mhz", 1965.0))
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)", 1965.0


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


# ------------------------------------------------------------------ oracle timing (CPU)
def _cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _oracle_worker(args):
    """One process of the oracle sample: DFS (state reuse, oracle/tree.py's order) over the
    subtrees of the given level-1 nodes until `budget_s`; returns (leaves, gate-amp updates,
    seconds).  Runs the oracle as it stands (numpy, one thread per process)."""
    name, nodes, budget_s = args
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"
    from threadpoolctl import threadpool_limits

    from oracle import gates as OG
    from oracle.planner import dcp_plan, fixed_plan
    from oracle.statevector import zero_state
    from oracle.tree import NoiseModel, error_rates, run_slice, sample_leaf
    from workloads import load_config

    w = load_config(name)
    n = w.circuit.n_qubits
    low = OG.lower(w.circuit.gates)
    nm = NoiseModel(w.p1, w.p2, w.readout_p01, w.readout_p10)
    plan = fixed_plan(len(low), w.arities) if w.arities else dcp_plan(error_rates(low, nm), w.shots, n,
                                                                       w.copy_cost_gates)
    A, B, L = plan.arities, plan.boundaries, len(plan.arities)
    leaves = 0
    gau = 0

    class Done(Exception):
        pass

    with threadpool_limits(1):
        t0 = time.perf_counter()

        def node(d, j, parent):
            nonlocal leaves, gau
            psi = parent
            for g in range(B[d], B[d + 1]):           # gate by gate so the budget is honoured
                psi = run_slice(psi if g > B[d] else psi.copy(), n, low, g, g + 1, j, w.seed, nm)
                gau += 2 ** n
                if time.perf_counter() - t0 > budget_s:
                    raise Done
            if d == L - 1:
                sample_leaf(psi, n, j, w.seed, nm)
                leaves += 1
                return
            for br in range(A[d + 1]):
                node(d + 1, j * A[d + 1] + br, psi)

        try:
            for (d, j) in nodes:
                anc, x = [], j
                for dd in range(d, -1, -1):
                    anc.append((dd, x))
                    x //= A[dd]
                psi = zero_state(n)
                for (dd, jj) in reversed(anc[1:]):      # the node's ancestors, flat
                    psi = run_slice(psi, n, low, B[dd], B[dd + 1], jj, w.seed, nm)
                    gau += (B[dd + 1] - B[dd]) * 2 ** n
                node(d, j, psi)
        except Done:
            pass
        dt = time.perf_counter() - t0
    return leaves, gau, dt


def cpu_baseline(w, plan, budget_s: float = 20.0, procs: int = 0):
    """The oracle on os.cpu_count() processes, each over its own level-1 subtrees, bounded
    by `budget_s`.  value = leaves / s when the sample completed leaves in every process;
    otherwise (wide states) the measured oracle gate-amp rate / (tree gate-amps per outcome)
    = shots/s, labelled extrapolated."""
    import multiprocessing as mp
    procs = procs or os.cpu_count() or 1
    A = plan.arity_list
    lvl1 = A[0] * (A[1] if len(A) > 1 else 1)
    d1 = 1 if len(A) > 1 else 0
    tasks = []
    for p in range(procs):
        nodes = [(d1, j) for j in range(p, lvl1, procs)]
        if nodes:
            tasks.append((w.name, nodes, budget_s))
    ctx = mp.get_context("spawn")       # the parent may hold a CUDA context: no fork
    with ctx.Pool(len(tasks)) as pool:
        res = pool.map(_oracle_worker, tasks)
    leaves = sum(r[0] for r in res)
    gau = sum(r[1] for r in res)
    dt = max(r[2] for r in res)
    per_out = plan.gate_amp_updates / plan.n_outcomes       # tree gate-amps per outcome
    gau_rate = gau / dt
    extrap = min(r[0] for r in res) == 0
    value = gau_rate / per_out if extrap else leaves / dt
    return {"value": value, "unit": "shots/s", "cores": len(tasks), "kind": "oracle",
            "cpu_model": _cpu_model(),
            "oracle_gate_amp_updates_per_s": gau_rate,
            "extrapolated": extrap,
            "sample": ("%d processes x %.0f s of the oracle's DFS (oracle/tree.py run_slice / sample_leaf, "
                       "numpy complex128, 1 thread each) over disjoint level-1 subtrees of the %d-leaf %s tree: "
                       "%d leaves, %.3g gate-amp updates%s"
                       % (len(tasks), dt, plan.n_outcomes, w.name, leaves, gau,
                          "; shots/s = oracle gate-amp rate / tree gate-amps per outcome (extrapolated)"
                          if extrap else ""))}


def run_reference(args, w, rank, world):
    """--impl reference: the oracle, as it stands, on the host cores (rank 0 only)."""
    if rank != 0:
        return
    import paper_2203_13892_b200.tqsim as T
    n, gates, noise, shots, ar = T.workload_args(w)
    plan = T.tqsim_plan_circuit(n, gates, noise, shots, ar)
    budget = max(2.0, min(10.0, 150.0 / max(1, args.steps + args.warmup)))
    vals = []
    cb = None
    for s in range(args.warmup + args.steps):
        cb = cpu_baseline(w, plan, budget_s=budget)
        if s >= args.warmup:
            vals.append(cb["value"])
    v = statistics.median(vals)
    cb["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "shots/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": budget * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "shots": w.shots, "outcomes": int(plan.n_outcomes),
                       "arities": plan.arity_list},
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "shots/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ launcher
def _relaunch_distributed(args):
    """--gpus N > 1 without a torchrun environment: run this script under
    torch.distributed.run, one process per GPU (rendezvous on 127.0.0.1)."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"error": "--gpus %d needs %d GPUs, this node has %d" % (args.gpus, args.gpus, have)}),
              flush=True)
        sys.exit(2)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl != "reference":
        return _relaunch_distributed(args)
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

    shard_r, shard_w = None, None
    if args.shard and world == 1:
        shard_r, shard_w = (int(v) for v in args.shard.split("/"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        dist.init_process_group("nccl", device_id=dev)
    n, gates, noise, shots, ar = T.workload_args(w)

    # cold first call of the public API (plan + NVRTC compile of every pass kernel + arena):
    # measured first, in a process that has compiled nothing yet; its arena is then released
    first_call_s = None
    if world == 1 and not args.no_e2e and not args.shard:
        ca = T.CircuitArg(n, gates)
        tc = time.perf_counter()
        T.tqsim_run(n, ca, noise, shots, ar, 0)
        first_call_s = time.perf_counter() - tc
        T.tqsim_release_run_cache()

    opts = T.default_options(tile_qubits=args.tile, batch_log2_amps=args.batch_log2, copy_cost_gates=args.copy_cost,
                             small_tree=args.small_tree)
    h = T.tqsim_create(n, gates, noise, shots, ar, opts)
    plan = h.plan
    N = int(plan.n_outcomes)
    xr, xw = (shard_r, shard_w) if shard_w else (rank, world)
    ws = torch.empty(h.workspace_bytes(xr, xw), dtype=torch.uint8, device=dev)
    out = torch.zeros(N, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream(dev)
    _, _, leaf0, leaf1 = T.tqsim_shard_range(plan, xr, xw)
    step_outcomes = N if not shard_w else leaf1 - leaf0      # outcomes one step produces

    def step(seed):
        out.zero_()
        h.execute(seed, xr, xw, st.cuda_stream, ws.data_ptr(), ws.numel(), out.data_ptr())
        if world > 1:
            dist.all_reduce(out, op=dist.ReduceOp.SUM)

    for i in range(args.warmup):
        step(1000 + i)
    torch.cuda.synchronize(dev)
    launches_per_step = int(h.stats().kernel_launches)
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
    ms_step = ms / args.steps

    # in-tree timing of every kernel family of one tree (events around every launch, tree
    # order, no graph) + the work each launch computed (dedup maps read back)
    prof = h.profile_tree(0, xr, xw, st.cuda_stream, ws.data_ptr(), ws.numel(), out.data_ptr())
    stats = h.stats()
    passes = [k for k in prof if k.kind == 0]
    tree_ms = sum(k.ms for k in prof)
    pass_ms = sum(k.ms for k in passes)
    pass_bytes = sum(k.alg_bytes for k in passes)
    pass_nominal = sum(k.nominal_bytes for k in passes)
    top = max(passes, key=lambda k: k.ms)
    hbm_peak, peak_src, sm_max = peaks()
    fp64_peak = N_SM * FP64_DFMA_PER_CLK_SM * sm_max * 1e6 / 1e12          # T DFMA/s
    amps = 1 << n
    top_name = "tq_pass_l%d_p%d" % (top.level, top.pass_)
    # ncu evidence of the same tree (profiles/ncu_<workload>.json, profiles/ncu_join.py):
    # DRAM bytes per launch and FP64 pipe instructions (DFMA + DADD + DMUL) per computed
    # amplitude of each kernel family; without it the FP64 work is the code generator's model
    ncu = None
    npath = os.path.join(ROOT, "profiles", "ncu_%s.json" % w.name)
    if os.path.exists(npath):
        with open(npath) as f:
            ncu = {r["kernel"]: r for r in json.load(f)["families"]}
    top_ncu = ncu.get(top_name) if ncu else None
    fp64_per_amp = top_ncu["fp64_inst_per_computed_amp"] if top_ncu and top_ncu.get(
        "fp64_inst_per_computed_amp") else top.fp64_per_amp
    fp64_src = ("ncu-measured FP64 thread instructions per computed amplitude (%s)" % os.path.basename(npath)
                if top_ncu else "code-generator cost model (FP64 ops per amplitude, fast path)")
    top_gbs = top.alg_bytes / (top.ms * 1e-3) / 1e9
    top_fp64 = fp64_per_amp * top.computed_states * amps / (top.ms * 1e-3) / 1e12
    fam_gbs = pass_bytes / (pass_ms * 1e-3) / 1e9
    # which roof binds the top kernel: the larger of its time at the HBM peak and at the FP64 peak
    t_hbm = top.alg_bytes / (hbm_peak * 1e9)
    t_fp64 = fp64_per_amp * top.computed_states * amps / (fp64_peak * 1e12)
    bound = "hbm" if t_hbm >= t_fp64 else "alu"
    traffic = {"dram_bytes_per_launch": top_ncu["dram_bytes_per_launch"],
               "source": "ncu launch list of one tree, %s family (%s)" % (top_name, os.path.basename(npath))} \
        if top_ncu and top_ncu.get("dram_bytes_per_launch") else None
    roofline = {
        "bound": bound,
        "achieved": top_gbs if bound == "hbm" else top_fp64,
        "peak": hbm_peak if bound == "hbm" else fp64_peak,
        "unit": "GB/s" if bound == "hbm" else "T DFMA/s",
        "frac": (top_gbs / hbm_peak) if bound == "hbm" else (top_fp64 / fp64_peak),
        "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
        "traffic_source": traffic.get("source") if traffic else None,
        "kernel": top_name,
        "peak_source": peak_src if bound == "hbm" else
        "derived: 148 SMs x 64 DFMA/clk x %.0f MHz (DESIGN.md §6.1)" % sm_max,
        "method": "tqsim_profile_tree: every launch of one tree bracketed by CUDA events on the launching "
                  "stream, tree order, no graph; bytes = algorithmic bytes of the instances computed",
        "launches_per_step": top.launches,
        "ms_per_step": top.ms,
        "alg_bytes_per_launch": top.alg_bytes / top.launches,
        "nominal_bytes_per_launch": top.nominal_bytes / top.launches,
        "computed_states": top.computed_states, "states": top.states,
        "hbm_gbs": top_gbs, "hbm_frac": top_gbs / hbm_peak,
        "fp64_tdfma_s": top_fp64, "fp64_frac": top_fp64 / fp64_peak, "fp64_peak_tdfma_s": fp64_peak,
        "fp64_work_source": fp64_src, "fp64_inst_per_computed_amp": fp64_per_amp,
        "share_of_tree": top.ms / tree_ms if tree_ms else None,
        "pass_family": {"ms_per_step": pass_ms, "alg_gbs": fam_gbs, "frac": fam_gbs / hbm_peak,
                        "alg_bytes": pass_bytes, "nominal_bytes": pass_nominal,
                        "nominal_gbs": pass_nominal / (pass_ms * 1e-3) / 1e9,
                        "share_of_tree": pass_ms / tree_ms if tree_ms else None},
        "profiled_tree_ms": tree_ms,
        "graph_step_ms": ms_step,
        "kernels": sorted(({"k": ("pass_l%d_p%d" % (k.level, k.pass_)) if k.kind == 0 else
                            ("measure_l%d" % k.level if k.kind == 1 else "noise"),
                            "ms": round(k.ms, 4), "launches": k.launches,
                            "gbs": round(k.alg_bytes / (k.ms * 1e-3) / 1e9, 1) if k.kind == 0 and k.ms else None}
                           for k in prof), key=lambda r: -r["ms"])[:12],
    }

    # the same tree with every instance computed (options.no_dedup = 1)
    no_dedup = None
    if args.no_dedup_steps > 0 and not shard_w:
        del ws
        torch.cuda.empty_cache()
        h2 = T.tqsim_create(n, gates, noise, shots, ar,
                            T.default_options(tile_qubits=args.tile, batch_log2_amps=args.batch_log2, no_dedup=1,
                                              copy_cost_gates=args.copy_cost))
        ws2 = torch.empty(h2.workspace_bytes(xr, xw), dtype=torch.uint8, device=dev)
        for i in range(1):
            h2.execute(2000 + i, xr, xw, st.cuda_stream, ws2.data_ptr(), ws2.numel(), out.data_ptr())
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0.record(st)
        for i in range(args.no_dedup_steps):
            out.zero_()
            h2.execute(i, xr, xw, st.cuda_stream, ws2.data_ptr(), ws2.numel(), out.data_ptr())
            if world > 1:
                dist.all_reduce(out, op=dist.ReduceOp.SUM)
        e1.record(st)
        torch.cuda.synchronize(dev)
        ms2 = e0.elapsed_time(e1) / args.no_dedup_steps
        t2 = torch.tensor([ms2], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        ms2 = float(t2.item())
        no_dedup = {"ms_per_step": ms2, "shots_per_s": step_outcomes / (ms2 * 1e-3),
                    "gate_amp_updates_per_s": plan.gate_amp_updates / (ms2 * 1e-3),
                    "steps": args.no_dedup_steps,
                    "note": "options.no_dedup = 1: every node instance of the tree computed (TQSim's "
                            "own reuse only; error-free duplicates not shared)"}
        h2.close()
        del ws2
        torch.cuda.empty_cache()

    # the paper's baseline: every shot simulated on its own (the flat plan (F),
    # options.no_dedup = 1), timed on F shots of the same circuit and noise; flat work is
    # linear in shots, so ms per N shots = ms(F) * N / F
    flat = None
    if args.flat_shots >= 0 and not shard_w and world == 1:
        F = args.flat_shots or (N if n <= 16 else min(N, 1024))
        try:
            del ws
        except NameError:
            pass
        torch.cuda.empty_cache()
        h3 = T.tqsim_create(n, gates, noise, F, [F],
                            T.default_options(tile_qubits=args.tile, batch_log2_amps=args.batch_log2, no_dedup=1))
        assert list(h3.plan.arity_list) == [F]
        ws3 = torch.empty(h3.workspace_bytes(0, 1), dtype=torch.uint8, device=dev)
        out3 = torch.zeros(F, dtype=torch.int32, device=dev)
        h3.execute(3000, 0, 1, st.cuda_stream, ws3.data_ptr(), ws3.numel(), out3.data_ptr())
        torch.cuda.synchronize(dev)
        fsteps = 2
        e0.record(st)
        for i in range(fsteps):
            h3.execute(3100 + i, 0, 1, st.cuda_stream, ws3.data_ptr(), ws3.numel(), out3.data_ptr())
        e1.record(st)
        torch.cuda.synchronize(dev)
        ms3 = e0.elapsed_time(e1) / fsteps
        per_n = ms3 * N / F
        flat = {"shots_timed": F, "ms_per_timed_step": ms3, "ms_per_n_shots": per_n,
                "shots_per_s": F / (ms3 * 1e-3), "steps": fsteps,
                "speedup_tree_vs_flat": per_n / ms_step,
                "speedup_tree_no_dedup_vs_flat": (per_n / no_dedup["ms_per_step"]) if no_dedup else None,
                "note": "flat plan (F) with options.no_dedup = 1: each shot runs the whole circuit on its own "
                        "state (the paper's baseline); ms_per_n_shots scales the F-shot time to this config's "
                        "%d shots (flat work is linear in shots)" % N}
        h3.close()
        del ws3, out3
        torch.cuda.empty_cache()

    # end to end through the public API with HOST buffers
    e2e = None
    if not args.no_e2e and not args.shard:
        from paper_2203_13892_b200.distributed import histogram
        n_low = int(plan.n_lowered_gates)
        if world == 1:
            ca = T.CircuitArg(n, gates)                     # the user's circuit, marshalled once
            T.tqsim_run(n, ca, noise, shots, ar, 0)         # warm (plan cache + arena)
            t0 = time.perf_counter()
            for i in range(args.steps):
                T.tqsim_run(n, ca, noise, shots, ar, i)
            dt = time.perf_counter() - t0
            T.tqsim_release_run_cache()
            note = ("tqsim_run per step: host circuit in (validated, hashed; the prepared plan and its "
                    "specialized kernels are reused from the library's plan cache after the first call), "
                    "h2d = per-gate noise-class and pass tables (2 B / lowered gate) + the seed (the tree is a "
                    "replayed CUDA graph: no per-kernel parameters cross PCIe), "
                    "d2h = leaf outcomes (uint32) into page-locked memory, host histogram (C)")
            h2d = 2 * n_low + 8
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
            note = ("distributed.ShardRunner per step on every rank: the shard (replayed CUDA graph), "
                    "NCCL all_reduce(SUM) of the leaf outcomes, D2H, histogram on rank 0; max over ranks")
            h2d = 96
        e2e = {"value": N * args.steps / dt, "unit": "shots/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": N * 4, "note": note,
               "first_call_s": first_call_s,
               "first_call_note": "cold: the process's first tqsim_run (DCP + pass plan + NVRTC compile of "
                                  "every specialized kernel + workspace allocation + the tree)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(w, plan, budget_s=args.cpu_budget)

    if rank == 0:
        shots_s = step_outcomes * args.steps / (ms * 1e-3)
        frac_tree = step_outcomes / N
        gau = plan.gate_amp_updates * frac_tree * args.steps / (ms * 1e-3)
        cgau = stats.computed_gate_amp_updates * args.steps / (ms * 1e-3)
        line = {
            "metric": METRIC, "value": shots_s, "unit": "shots/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "n_qubits": n, "shots": shots, "outcomes": N,
                       "outcomes_per_step": step_outcomes,
                       "shard": args.shard or None,
                       "arities": plan.arity_list, "small_tree": int(plan.small_tree), "lowered_gates": int(plan.n_lowered_gates),
                       "tile_qubits": int(plan.tile_qubits),
                       "l2": "inputs larger than L2 (state batches >= 1 GiB per launch group)",
                       "parallelism": "tree sharding x%d (tqsim_shard_levels)" % world},
            "gate_amp_updates_per_s": gau,
            "computed_gate_amp_updates_per_s": cgau,
            "gate_amp_note": "gate_amp_updates_per_s counts the tree's nominal work (every node instance); "
                             "computed_... counts the instances executed (error-free duplicates are "
                             "computed once, DESIGN.md §7); no_dedup times the tree with every instance "
                             "computed",
            "tree_vs_flat_gate_ratio": plan.flat_gate_amp_updates / plan.gate_amp_updates,
            "no_dedup": no_dedup,
            "flat": flat,
            "roofline": roofline,
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
