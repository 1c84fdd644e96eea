"""Randomised parity stress run (GPU box): many random circuits / trees / options through the
default path (dedup, work lists, conditional leaf sampling, small-state tree) against the
oracle's tree DFS; every non-flagged leaf outcome must match.  Test infrastructure (imports
oracle/), not part of the product.

    python scripts/stress_parity.py [seconds] [seed] [nmin nmax] > gpurun_out/stress.jsonl
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("TQSIM_SMALL", "0")
import paper_2203_13892_b200.tqsim as T  # noqa: E402
from oracle import gates as OG  # noqa: E402
from oracle.planner import Plan  # noqa: E402
from oracle.tree import NoiseModel, simulate_tree  # noqa: E402
from workloads import qft_gates, random_circuit  # noqa: E402
from workloads.generators import qaoa_gates, random_3_regular_edges  # noqa: E402


def kraus_case(rng, k):
    """Non-Pauli channels (the shared-memory Kraus engine) vs oracle/kraus.py."""
    from oracle import kraus as K
    n = int(rng.integers(KN[0], KN[1] + 1))
    gates = random_circuit(n, int(rng.integers(10, 60)), rng)
    if not gates:
        gates = random_circuit(n, 5, rng, kinds=["h", "rx"])
    L = int(rng.integers(1, 4))
    ar = [int(rng.integers(1, 5)) for _ in range(L)]
    shots = int(np.prod(ar))
    ad = float(rng.choice([0.0, 0.02, 0.2]))
    pdp = float(rng.choice([0.0, 0.02, 0.2]))
    t1 = float(rng.choice([0.0, 50e-6]))
    km = K.KrausModel(amp_damping=ad, phase_damping=pdp, t1=t1, t2=70e-6 if t1 else 0.0,
                      gate_time_1q=5e-6 if t1 else 0.0, gate_time_2q=30e-6 if t1 else 0.0)
    if not km.enabled:
        km = K.KrausModel(amp_damping=0.05)
    p = float(rng.choice([0.0, 0.01, 0.1]))
    nm = NoiseModel(p, 2 * p, float(rng.choice([0.0, 0.02])), 0.0)
    seed = int(rng.integers(0, 2 ** 40))
    noise = T.noise_arg(nm.p1, nm.p2, nm.readout_p01, nm.readout_p10, km.amp_damping, km.phase_damping, km.t1,
                        km.t2, km.gate_time_1q, km.gate_time_2q)
    res = T.tqsim_run_ex(n, gates, noise, shots, ar, seed, None, leaf_debug=True)
    plan = Plan(res.plan.arity_list, res.plan.boundary_list)
    ref = K.simulate_tree(n, OG.lower(gates), plan, nm, km, seed)
    bad, flagged = [], 0
    for l, r in ref.leaves.items():
        if r.flagged:
            flagged += 1
            continue
        if int(res.leaf_outcomes[l]) != r.outcome:
            bad.append(l)
    return {"case": k, "kind": "kraus", "n": n, "arities": ar, "p": p, "ad": ad, "pd": pdp, "t1": t1, "seed": seed,
            "leaves": len(ref.leaves), "flagged": flagged, "bad": bad[:8], "ok": not bad}


NMIN, NMAX = 4, 15   # qubit range of the Pauli cases (argv 3, 4)
# STRESS_KRAUS_N="lo,hi": Kraus cases only, n in [lo, hi] (10-13: one CTA, 14-16: the cluster engine)
KN = (1, 9)
KRAUS_ONLY = False
if os.environ.get("STRESS_KRAUS_N"):
    KN = tuple(int(x) for x in os.environ["STRESS_KRAUS_N"].split(","))
    KRAUS_ONLY = True


def one_case(rng, k):
    if KRAUS_ONLY or (NMAX <= 15 and rng.random() < 0.15):
        return kraus_case(rng, k)
    kind = rng.choice(["random", "qaoa", "qft"], p=[0.6, 0.3, 0.1])
    n = int(rng.integers(NMIN, NMAX))
    if kind == "qaoa" and n % 2:
        n += 1
    if kind == "random":
        gates = random_circuit(n, int(rng.integers(20, 120)), rng)
    elif kind == "qaoa":
        gates = qaoa_gates(n, random_3_regular_edges(n, rng), list(rng.uniform(0, 3, 2)), list(rng.uniform(0, 3, 2)))
    else:
        gates = qft_gates(n)
    L = int(rng.integers(1, 5))
    ar = [int(rng.integers(1, 5)) for _ in range(L)]
    shots = int(np.prod(ar))
    p = float(rng.choice([0.0, 0.01, 0.05, 0.2, 1.0]))
    nm = NoiseModel(p, min(1.0, 2 * p), float(rng.choice([0.0, 0.02])), float(rng.choice([0.0, 0.03])))
    tile = int(rng.choice([0, 4, 6, 8, 10, 12]))
    opts = T.default_options(tile_qubits=tile if tile <= n else 0,
                             batch_log2_amps=int(rng.choice([0, n, n + 1, n + 3])),
                             trail_low=int(rng.choice([0, 3, 4])) if tile == 0 or tile >= 8 else 0,
                             small_tree=int(rng.choice([0, 1, 2])), no_dedup=int(rng.random() < 0.2))
    seed = int(rng.integers(0, 2 ** 40))
    noise = T.noise_arg(nm.p1, nm.p2, nm.readout_p01, nm.readout_p10)
    res = T.tqsim_run_ex(n, gates, noise, shots, ar, seed, opts, leaf_debug=True)
    plan = Plan(res.plan.arity_list, res.plan.boundary_list)
    ref = simulate_tree(n, OG.lower(gates), plan, nm, seed)
    bad, flagged = [], 0
    for l, r in ref.leaves.items():
        if r.flagged:
            flagged += 1
            continue
        if int(res.leaf_outcomes[l]) != r.outcome or res.leaf_u[l] != r.u:
            bad.append(l)
    return {"case": k, "kind": kind, "n": n, "arities": ar, "p": p, "tile": tile,
            "trail": int(res.plan.trail_top_bits), "small": int(res.plan.small_tree),
            "no_dedup": int(opts.no_dedup), "batch_log2": int(opts.batch_log2_amps), "seed": seed,
            "leaves": len(ref.leaves), "flagged": flagged, "bad": bad[:8], "ok": not bad}


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    global NMIN, NMAX
    if len(sys.argv) > 4:
        NMIN, NMAX = int(sys.argv[3]), int(sys.argv[4])
    t0 = time.time()
    k = nbad = 0
    while time.time() - t0 < budget:
        try:
            r = one_case(rng, k)
        except T.TqsimError as e:
            r = {"case": k, "error": str(e), "ok": False}
        nbad += not r["ok"]
        print(json.dumps(r), flush=True)
        k += 1
    print(json.dumps({"cases": k, "failed": nbad, "seconds": round(time.time() - t0, 1)}), flush=True)


if __name__ == "__main__":
    main()
