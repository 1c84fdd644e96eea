"""Accuracy studies (the paper's §4.1 / §5.2-5.4 methodology), run through the
product (tqsim_run on the GPU) with the host metrics of paper_2203_13892_b200/metrics.py.

    python scripts/accuracy.py fidelity  [--shots 32000] [--seeds 10] [--circuits qft12h,ghz16,brick12,qaoa12]
    python scripts/accuracy.py table3    [--seeds 10]                  # QPE_9 structures (Table 3)
    python scripts/accuracy.py errfreq   [--shots 32000]               # QFT_12 qubit error frequency
    python scripts/accuracy.py shots     [--seeds 10]                  # QPE_9 shots sensitivity
    python scripts/accuracy.py noisemodels [--seeds 10] [--shots 3200] # Table 2 models

Normalized fidelity Eq.7 of the tree output and of the flat per-shot baseline
(plan (N): the same engine without reuse) against the ideal distribution of a
noise-free run (state dump).  Tree and flat runs use INDEPENDENT seeds (s and 10^6 + s), so
their noise realisations are uncorrelated, as two simulators' would be.  Speedups are
wall-clock ratios of the two tqsim_run calls (medians over seeds).  JSON lines.
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

FLAT_SEED = 1_000_000
# Table 2 channels at the paper's rates and reading R32's TR parameters
AD = PD = 0.01
TR = dict(t1=50e-6, t2=70e-6, gate_time_1q=50e-9, gate_time_2q=300e-9)


def circuit(name):
    rng = np.random.default_rng(0)
    if name.startswith("qft") and name.endswith("h"):   # QFT_n with an H prelude
        n = int(name[3:-1])
        return n, [G.g1("h", q) for q in range(n)] + G.qft_gates(n)
    if name.startswith("qpe"):                           # QPE_n, phase 1/3
        n = int(name[3:])
        return n, G.qpe_gates(n - 1, 1.0 / 3.0)
    if name.startswith("bv"):                            # BV_n, hidden string all ones
        n = int(name[2:])
        return n, G.bv_gates(n, (1 << (n - 1)) - 1)
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


def ideal_distribution(n, gates):
    st = T.tqsim_run_ex(n, gates, T.noise_arg(0, 0), 1, [1], 0, None, [(0, 0)]).dumps[0]
    return np.abs(st) ** 2


def timed_run(n, ca, noise, shots, arities, seed):
    t0 = time.perf_counter()
    r = T.tqsim_run(n, ca, noise, shots, arities, seed)
    return r, time.perf_counter() - t0


def compare(n, gates, noise, shots, seeds, arities=None, p_ideal=None):
    """Tree (arities or DCP) vs flat, `seeds` repeats: normalized fidelities, speedup."""
    ca = T.CircuitArg(n, gates)
    if p_ideal is None:
        p_ideal = ideal_distribution(n, gates)
    timed_run(n, ca, noise, shots, arities, 0)          # warm: plan cache, kernels
    timed_run(n, ca, noise, shots, [shots], 0)
    ft, ff, tt, tf = [], [], [], []
    plan = None
    for s in range(seeds):
        tree, dt = timed_run(n, ca, noise, shots, arities, s)
        flat, df = timed_run(n, ca, noise, shots, [shots], FLAT_SEED + s)
        tt.append(dt)
        tf.append(df)
        plan = tree.plan
        ft.append(M.normalized_fidelity(p_ideal, M.distribution(tree.counts, n)))
        ff.append(M.normalized_fidelity(p_ideal, M.distribution(flat.counts, n)))
    ft, ff = np.array(ft), np.array(ff)
    # statistical margin of the difference of means: 3 sigma from the per-seed spreads
    sig = float(np.sqrt(ft.var(ddof=1) / seeds + ff.var(ddof=1) / seeds)) if seeds > 1 else None
    return {"n_qubits": n, "shots": shots, "seeds": seeds, "tree_arities": plan.arity_list,
            "outcomes": int(plan.n_outcomes), "node_ratio_speedup": float(plan.predicted_speedup_nodes),
            "F_tree_mean": float(ft.mean()), "F_flat_mean": float(ff.mean()),
            "diff_of_means": float(abs(ft.mean() - ff.mean())), "sigma_diff": sig,
            "F_tree": ft.round(4).tolist(), "F_flat": ff.round(4).tolist(),
            "speedup_wall": float(np.median(tf) / np.median(tt)),
            "tree_ms": 1e3 * float(np.median(tt)), "flat_ms": 1e3 * float(np.median(tf))}


def dep_noise(p1=1e-3, p2=1e-2, ro=1e-2):
    return T.noise_arg(p1, p2, ro, ro)


def study_fidelity(a):
    for name in a.circuits.split(","):
        n, gates = circuit(name)
        r = compare(n, gates, dep_noise(), a.shots, a.seeds)
        print(json.dumps({"study": "fidelity", "circuit": name, **r}), flush=True)


def study_table3(a):
    """Table 3: QPE_9, 1000 shots, the five manual structures on one 3-slice
    partition plus DCP's own, 10 repeats; max speedup (node ratio) vs measured, and the
    normalized-fidelity difference to the flat baseline."""
    n, gates = circuit("qpe9")
    p = ideal_distribution(n, gates)
    structs = [None, [250, 2, 2], [20, 10, 5], [10, 10, 10], [5, 10, 20], [2, 2, 250]]
    for ar in structs:
        r = compare(n, gates, dep_noise(), 1000, a.seeds, ar, p)
        print(json.dumps({"study": "table3", "circuit": "qpe9", "structure": ar or "DCP", **r}), flush=True)


def study_errfreq(a):
    """Qubit error frequency: QFT_12 on the equal superposition (H prelude); the
    ideal output is |0..0>, so a measured 1 on qubit q is an error of q.  Three flat
    baseline runs (seeds) and the tree run."""
    n, gates = circuit("qft12h")
    ca = T.CircuitArg(n, gates)
    runs = {}
    for tag, ar, seed in (("flat_a", [a.shots], FLAT_SEED), ("flat_b", [a.shots], FLAT_SEED + 1),
                          ("flat_c", [a.shots], FLAT_SEED + 2), ("tree", None, 0)):
        r = T.tqsim_run(n, ca, dep_noise(), a.shots, ar, seed)
        outs = r.leaf_outcomes[: a.shots].astype(np.uint64)
        freq = [float(((outs >> np.uint64(q)) & np.uint64(1)).mean()) for q in range(n)]
        runs[tag] = {"arities": r.plan.arity_list, "freq": [round(f, 5) for f in freq]}
    fl = np.array([runs[k]["freq"] for k in ("flat_a", "flat_b", "flat_c")])
    tr = np.array(runs["tree"]["freq"])
    out = {"study": "errfreq", "circuit": "qft12h", "shots": a.shots, "runs": runs,
           "max_abs_tree_minus_flat_mean": float(np.max(np.abs(tr - fl.mean(0)))),
           "max_flat_spread": float(np.max(fl.max(0) - fl.min(0))),
           "binomial_sigma_max": float(np.sqrt(fl.mean(0) * (1 - fl.mean(0)) / a.shots).max())}
    print(json.dumps(out), flush=True)


def study_shots(a):
    """Shots sensitivity: QPE_9 from 1k to 32k shots, DCP structure."""
    n, gates = circuit("qpe9")
    p = ideal_distribution(n, gates)
    for shots in (1000, 3000, 7000, 9000, 16000, 32000):
        r = compare(n, gates, dep_noise(), shots, a.seeds, None, p)
        print(json.dumps({"study": "shots", "circuit": "qpe9", **r}), flush=True)


def table2():
    tr = dict(t1=TR["t1"], t2=TR["t2"], gate_time_1q=TR["gate_time_1q"], gate_time_2q=TR["gate_time_2q"])
    ro = 1e-2
    return {"DC": dict(p1=1e-3, p2=1e-2), "DCR": dict(p1=1e-3, p2=1e-2, p01=ro, p10=ro),
            "TR": dict(**tr), "TRR": dict(p01=ro, p10=ro, **tr),
            "AD": dict(amp_damping=AD), "ADR": dict(amp_damping=AD, p01=ro, p10=ro),
            "PD": dict(phase_damping=PD), "PDR": dict(phase_damping=PD, p01=ro, p10=ro),
            "ALL": dict(p1=1e-3, p2=1e-2, p01=ro, p10=ro, amp_damping=AD, phase_damping=PD, **tr)}


def study_noisemodels(a):
    """Table 2's nine models on QFT_12 (H prelude), QPE_9, BV_10; the tree
    structure comes from DCP on the depolarizing parameters and is used for every model
    (P:636-637)."""
    for name in a.circuits.split(","):
        n, gates = circuit(name)
        p = ideal_distribution(n, gates)
        ar = T.tqsim_plan_circuit(n, gates, dep_noise(), a.shots).arity_list
        for model, kw in table2().items():
            kw = dict(kw)
            noise = T.noise_arg(kw.pop("p1", 0.0), kw.pop("p2", 0.0), kw.pop("p01", 0.0), kw.pop("p10", 0.0), **kw)
            r = compare(n, gates, noise, a.shots, a.seeds, ar, p)
            print(json.dumps({"study": "noisemodels", "circuit": name, "model": model, **r}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("study", choices=["fidelity", "table3", "errfreq", "shots", "noisemodels"])
    ap.add_argument("--shots", type=int, default=0)
    ap.add_argument("--seeds", type=int, default=10)
    ap.add_argument("--circuits", default="")
    a = ap.parse_args()
    if a.study == "fidelity":
        a.shots = a.shots or 32000
        a.circuits = a.circuits or "qft12h,ghz16,brick12,qaoa12"
        study_fidelity(a)
    elif a.study == "table3":
        study_table3(a)
    elif a.study == "errfreq":
        a.shots = a.shots or 32000
        study_errfreq(a)
    elif a.study == "shots":
        study_shots(a)
    else:
        a.shots = a.shots or 3200
        a.circuits = a.circuits or "qft12h,qpe9,bv10"
        study_noisemodels(a)


if __name__ == "__main__":
    main()
