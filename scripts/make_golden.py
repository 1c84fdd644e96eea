#!/usr/bin/env python3
"""Write the oracle-computed parity fixtures under tests/golden/ (test infrastructure).

    python scripts/make_golden.py c2_full|c3_full|c4_sub|c5_pairs|c4_beta0 [--procs P]

Imports ONLY `oracle/` (the plain numpy CPU simulator) and `workloads/` (seeded
inputs): no value here comes from the CUDA path.  The plan is the oracle's own
(oracle.planner.dcp_plan, the reading of P:265-294 §3.2 in DESIGN.md R12-R18); the
GPU tests assert the library plans the same tree before comparing.

Each fixture is a compressed .npz holding, per golden leaf l (
P:139 §2.3 sampling, P:173/P:277 noise after every gate, P:475 readout):
  leaf[l], x (sampled index before readout), outcome (after readout),
  flagged (draw within 1e-9 of a CDF boundary, reading R9), u (the u53 uniform),
  total (sum |a|^2 of the leaf state),
  chk_leaf[c], chk_idx[c, K], chk_amp[c, K]  for a subset of the leaves (every leaf of
          c4_sub / c5_pairs, every 331st of the full trees): amplitudes of the leaf state at
          K seeded indices plus the 8-amplitude run holding x (amplitude parity),
plus plan_arities, plan_boundaries, config name, seed and the command that wrote it.

Targets (SURVEY §8(c) "What pins each part"; VERDICT r1 "Next round" #1):
  c2_full   every leaf of the C2 (QFT-15) tree (10,240), DFS with reuse, parallel
            over top-level subtrees
  c3_full   every leaf of the C3 (brickwork-20) tree (10,240), same
  c4_sub    C4 (QAOA-24): the complete subtree under one level-4 node in 4 different
            top-level subtrees (4 x 32 leaves: whole sibling / cousin groups) and one
            isolated leaf in each of the 16 top-level subtrees
  c5_pairs  C5 (HEA-28): two sibling pairs of leaves in two different 8-GPU shards
            (top-level instances 3 and 83), prefix shared like the tree's DFS
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import gates as OG                                  # noqa: E402
from oracle.planner import dcp_plan, fixed_plan                 # noqa: E402
from oracle.statevector import zero_state                       # noqa: E402
from oracle.tree import (NoiseModel, error_rates, leaf_ancestors, run_slice,  # noqa: E402
                         sample_leaf)
from workloads import load_config, make_variant                 # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
N_CHK = 24          # seeded check indices per leaf (+ the 8-amplitude run of x)


def _single_thread():
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


def workload(name):
    w = make_variant(name) if name.endswith(("_beta0", "_ry0", "_monomial")) else load_config(name)
    low = OG.lower(w.circuit.gates)
    nm = NoiseModel(w.p1, w.p2, w.readout_p01, w.readout_p10)
    if w.arities:
        plan = fixed_plan(len(low), w.arities)
    else:
        plan = dcp_plan(error_rates(low, nm), w.shots, w.circuit.n_qubits, w.copy_cost_gates)
    return w, low, nm, plan


def leaf_record(psi, n, leaf, w, nm, chk_every):
    r = sample_leaf(psi, n, leaf, w.seed, nm)
    total = float(np.sum(psi.real ** 2 + psi.imag ** 2))
    rec = dict(leaf=leaf, x=r.x, outcome=r.outcome, flagged=r.flagged, u=r.u, total=total)
    if leaf % chk_every == 0:
        rng = np.random.default_rng(leaf + 7919 * n)
        idx = np.concatenate([rng.integers(0, 2 ** n, N_CHK), (r.x & ~7) + np.arange(8)]).astype(np.int64)
        rec.update(chk_idx=idx, chk_amp=psi[idx].copy())
    return rec


def subtree(args):
    """DFS (state reuse, as oracle.tree.simulate_tree) below node (d0, j0); the path to it
    is recomputed flat with inherited keys (oracle.tree.simulate_leaf_flat's rule)."""
    name, d0, j0, chk_every = args
    _single_thread()
    w, low, nm, plan = workload(name)
    n = w.circuit.n_qubits
    A, B, L = plan.arities, plan.boundaries, len(plan.arities)
    # ancestors of (d0, j0): j_d = j_{d+1} // A_{d+1}
    anc = [0] * (d0 + 1)
    j = j0
    for d in range(d0, -1, -1):
        anc[d] = j
        j //= A[d]
    psi = zero_state(n)
    for d in range(d0 + 1):
        psi = run_slice(psi, n, low, B[d], B[d + 1], anc[d], w.seed, nm)
    out = []

    def node(d, j, st):
        if d == L - 1:
            out.append(leaf_record(st, n, j, w, nm, chk_every))
            return
        for br in range(A[d + 1]):
            c = j * A[d + 1] + br
            node(d + 1, c, run_slice(st.copy(), n, low, B[d + 1], B[d + 2], c, w.seed, nm))

    node(d0, j0, psi)
    return out


def save(tag, name, plan, w, recs, extra):
    recs = sorted(recs, key=lambda r: r["leaf"])
    chk = [r for r in recs if "chk_idx" in r]
    arr = lambda k, dt: np.array([r[k] for r in recs], dtype=dt)
    meta = {"config": name, "seed": w.seed, "writer": "scripts/make_golden.py " + " ".join(sys.argv[1:]),
            "oracle": "oracle.tree run_slice / sample_leaf (numpy complex128)", **extra}
    path = os.path.join(GOLDEN, "%s.npz" % tag)
    np.savez_compressed(path, leaf=arr("leaf", np.int64), x=arr("x", np.uint32),
                        outcome=arr("outcome", np.uint32), flagged=arr("flagged", bool),
                        u=arr("u", np.float64), total=arr("total", np.float64),
                        chk_leaf=np.array([r["leaf"] for r in chk], dtype=np.int64),
                        chk_idx=np.stack([r["chk_idx"] for r in chk]),
                        chk_amp=np.stack([r["chk_amp"] for r in chk]),
                        plan_arities=np.array(plan.arities, dtype=np.int64),
                        plan_boundaries=np.array(plan.boundaries, dtype=np.int64),
                        meta=np.array(json.dumps(meta)))
    print("wrote %s: %d leaves, %d flagged" % (path, len(recs), int(arr("flagged", bool).sum())), flush=True)


def run_tasks(tasks, procs):
    ctx = mp.get_context("fork")
    recs = []
    with ctx.Pool(procs) as pool:
        for part in pool.imap_unordered(subtree, tasks):
            recs.extend(part)
            print("  %d leaves done" % len(recs), flush=True)
    return recs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("target", choices=["c2_full", "c3_full", "c4_sub", "c5_pairs"])
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    a = ap.parse_args()
    t0 = time.time()
    if a.target in ("c2_full", "c3_full"):
        name = {"c2_full": "c2_qft15", "c3_full": "c3_brick20"}[a.target]
        w, low, nm, plan = workload(name)
        # level-1 nodes as tasks (finer than top-level subtrees: better balance)
        tasks = [(name, 1, j, 331) for j in range(plan.arities[0] * plan.arities[1])]
        recs = run_tasks(tasks, a.procs)
        assert len(recs) == int(np.prod(plan.arities))
        save(a.target.replace("_full", "") + "_tree", name, plan, w, recs, {"coverage": "all leaves"})
    elif a.target == "c4_sub":
        name = "c4_qaoa24"
        w, low, nm, plan = workload(name)
        A = plan.arities
        per_top = int(np.prod(A[1:]))
        below4 = int(np.prod(A[5:]))          # leaves under one level-4 node
        tasks = []
        for t, k in ((0, 0), (5, 3), (10, 9), (15, 14)):   # level-4 node k of top-level subtree t
            tasks.append((name, 4, t * int(np.prod(A[1:5])) + k, 1))
        for t in range(A[0]):                              # one isolated leaf per top-level subtree
            tasks.append((name, len(A) - 1, t * per_top + (t * 97 + 13) % per_top, 1))
        recs = run_tasks(tasks, a.procs)
        assert len(recs) == 4 * below4 + A[0]
        save("c4_subtrees", name, plan, w, recs,
             {"coverage": "4 complete level-4 subtrees (32 leaves each) + 1 leaf per top-level subtree"})
    elif a.target == "c5_pairs":
        name = "c5_hea28"
        w, low, nm, plan = workload(name)
        A = plan.arities
        per_top = int(np.prod(A[1:]))
        L = len(A)
        tasks = []
        for t, off in ((3, 41), (83, 170)):               # shards 0 and 5 of 8 (16 tops each)
            leaf = t * per_top + off
            tasks.append((name, L - 2, leaf // A[-1], 1))      # a penultimate node: its 2 leaves
        recs = run_tasks(tasks, min(a.procs, 2))
        save("c5_pairs", name, plan, w, recs,
             {"coverage": "2 sibling pairs (top-level subtrees 3 and 83)"})
    print("%.0f s" % (time.time() - t0), flush=True)


if __name__ == "__main__":
    main()
