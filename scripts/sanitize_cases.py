#!/usr/bin/env python3
"""Small cases for compute-sanitizer (racecheck / synccheck / memcheck), one tool per call:

    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py

Covers every kernel family on small inputs: C1 (QFT-5 tree, arities [10, 100]) and C2-shaped
(QFT-15, 40 shots) trees through the default path (dedup maps, no-store leaf sampler) and the
stored-state path (dumps), tiles K = 4..12 with p = 1 (every gate errs: the careful Pauli-frame
path, store maps, off-tile diagonal units), the chunk-sum sampler (n = 19), and the Kraus
engine.  Prints one line per case; exits non-zero on any failed check (the sanitizer's own
report is what is judged)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2203_13892_b200.tqsim as T  # noqa: E402
from workloads import load_config, qft_gates, random_circuit  # noqa: E402
from workloads.generators import hea_gates, qaoa_gates, random_3_regular_edges  # noqa: E402


def main():
    w = load_config("c1_qft5")
    n, gates, noise, shots, ar = T.workload_args(w)
    a = T.tqsim_run(n, gates, noise, shots, ar, 0)
    b = T.tqsim_run_ex(n, gates, noise, shots, ar, 0, None, [(1, 3)])
    assert np.array_equal(a.leaf_outcomes, b.leaf_outcomes)
    print("c1 tree ok")
    r = T.tqsim_run_ex(15, qft_gates(15), T.noise_arg(0.01, 0.05, 0.02, 0.02), 40, [4, 2, 5], 1)
    print("qft15 small tree ok", len(r.counts))
    rng = np.random.default_rng(0)
    for K in (4, 6, 8, 10, 12):
        n = 12
        g = random_circuit(n, 40, rng) + qaoa_gates(n, random_3_regular_edges(n, rng), [0.3], [0.4]) + \
            hea_gates(n, 1, rng.uniform(0, 6, (1, n)))
        opts = T.default_options(tile_qubits=K, batch_log2_amps=n + 2)
        for p in (0.0, 1.0):
            x = T.tqsim_run_ex(n, g, T.noise_arg(p, p, 0.02, 0.02), 24, [3, 2, 4], 7, opts)
            y = T.tqsim_run_ex(n, g, T.noise_arg(p, p, 0.02, 0.02), 24, [3, 2, 4], 7, opts, [(2, 5)])
            assert np.array_equal(x.leaf_outcomes, y.leaf_outcomes), (K, p)
        print("tile", K, "ok")
    g = random_circuit(19, 30, rng)
    r = T.tqsim_run_ex(19, g, T.noise_arg(0.003, 0.01, 0.02, 0.02), 12, [2, 6], 3)
    print("chunk-sum sampler ok", len(r.counts))
    r = T.tqsim_run(8, random_circuit(8, 30, rng), T.noise_arg(0.01, 0.05, 0.02, 0.02, amp_damping=0.1,
                                                               phase_damping=0.1, t1=5e-6, t2=6e-6,
                                                               gate_time_1q=1e-7, gate_time_2q=3e-7), 24, [4, 6], 2)
    print("kraus engine ok", len(r.counts))


if __name__ == "__main__":
    main()
