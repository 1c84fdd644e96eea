"""B200 analogue of the paper's fig:copy-overhead: state-copy cost in gate
units for several widths, measured with tqsim_profile_copy_cost; JSON lines.

    python scripts/copy_cost_table.py [n ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_13892_b200.tqsim as T  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [12, 15, 20, 24, 28]:
    c, cm, gm = T.tqsim_profile_copy_cost(n, 64, 0)
    print(json.dumps({"n_qubits": n, "copy_cost_gates": round(c, 2), "copy_ms_per_GiB_batch": round(cm, 4),
                      "gate_ms_per_GiB_batch": round(gm, 5), "dcp_first_slice": max(1, int(c + 0.5))}),
          flush=True)
