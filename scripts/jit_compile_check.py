"""Compile every generated pass kernel (all variants) of the BASELINE configs and of
random circuits with NVRTC on the host (no GPU needed): a CPU-side check of the
code generator.   python scripts/jit_compile_check.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_13892_b200.tqsim as T  # noqa: E402
from workloads import config_names, load_config, random_circuit  # noqa: E402

total = 0
for name in config_names():
    w = load_config(name)
    n, gates, noise, shots, ar = T.workload_args(w)
    k, b, sec = T.tqsim_compile_passes(n, gates, noise, shots, ar)
    total += k
    print(name, k, "kernels", round(sec, 1), "s", flush=True)
rng = np.random.default_rng(5)
for it in range(6):
    n = int(rng.integers(4, 16))
    gates = random_circuit(n, 60, rng)
    k, b, sec = T.tqsim_compile_passes(n, gates, T.noise_arg(0.1, 0.2), 50, [5, 10],
                                       T.default_options(tile_qubits=int(rng.choice([0, 7, 9, 12]))))
    total += k
print("ok", total, "kernels")
