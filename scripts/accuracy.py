"""Accuracy study (the paper's §4.1 / §5.2 methodology): normalized
fidelity (Eq.7) of the tree method vs the flat per-shot baseline run through the same
engine, over seeds, plus the speedup; JSON lines.

    python scripts/accuracy.py [--shots 32000] [--seeds 10] [--circuits qft12h,ghz16,brick12,qaoa12]

The paper reports |F_tree - F_flat| <= 0.016 (max), 0.006 (mean) over 48 circuits at
32,000 shots.  Ideal distributions come from a noise-free run of the same
engine (state dump), so only the noise treatment differs.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_13892_b200.tqsim as T  # noqa: E402
from paper_2203_13892_b200 import metrics as M  # noqa: E402
from workloads import generators as G  # noqa: E402


def circuit(name):
    rng = np.random.default_rng(0)
    if name.startswith("qft") and name.endswith("h"):   # QFT_n with an H prelude
        n = int(name[3:-1])
        return n, [G.g1("h", q) for q in range(n)] + G.qft_gates(n)
    if name.startswith("ghz"):
        n = int(name[3:])
        return n, G.ghz_gates(n)
    if name.startswith("brick"):
        n = int(name[5:])
        return n, G.brickwork_gates(n, 10, rng)
    if name.startswith("qaoa"):
        n = int(name[4:])
        edges = G.random_3_regular_edges(n, rng)
        gb = rng.uniform(0, np.pi, 4)
        return n, G.qaoa_gates(n, edges, gb[0::2], gb[1::2])
    raise ValueError(name)


def study(name, shots, seeds, noise):
    n, gates = circuit(name)
    ca = T.CircuitArg(n, gates)
    ideal = T.tqsim_run_ex(n, gates, T.noise_arg(0, 0), 1, [1], 0, None, [(0, 0)]).dumps[0]
    p_ideal = np.abs(ideal) ** 2
    ft, ff, tt, tf = [], [], [], []
    plan = None
    for s in range(seeds):
        t0 = time.perf_counter()
        tree = T.tqsim_run(n, ca, noise, shots, None, s)
        tt.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        flat = T.tqsim_run(n, ca, noise, shots, [shots], s)
        tf.append(time.perf_counter() - t0)
        plan = tree.plan.arity_list
        ft.append(M.normalized_fidelity(p_ideal, M.distribution(tree.counts, n)))
        ff.append(M.normalized_fidelity(p_ideal, M.distribution(flat.counts, n)))
    d = np.abs(np.array(ft) - np.array(ff))
    return {"circuit": name, "n_qubits": n, "shots": shots, "seeds": seeds, "tree_arities": plan,
            "F_tree_mean": float(np.mean(ft)), "F_flat_mean": float(np.mean(ff)),
            "absdiff_mean": float(d.mean()), "absdiff_max": float(d.max()),
            "diff_of_means": float(abs(np.mean(ft) - np.mean(ff))),
            "speedup_wall": float(np.median(tf[1:] or tf) / np.median(tt[1:] or tt))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shots", type=int, default=32000)
    ap.add_argument("--seeds", type=int, default=10)
    ap.add_argument("--circuits", default="qft12h,ghz16,brick12,qaoa12")
    ap.add_argument("--p1", type=float, default=1e-3)
    ap.add_argument("--p2", type=float, default=1e-2)
    ap.add_argument("--readout", type=float, default=1e-2)
    a = ap.parse_args()
    noise = T.noise_arg(a.p1, a.p2, a.readout, a.readout)
    for name in a.circuits.split(","):
        print(json.dumps(study(name, a.shots, a.seeds, noise)), flush=True)


if __name__ == "__main__":
    main()
