#!/bin/bash
# After the non-monomial-run fix: the parity files, a replay of the stress seed that found it, C4/C2 bench lines.
set -u
O=gpurun_out/s5; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_small.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest_rc=$?" >> $O/pytest.log
timeout 300 python scripts/stress_parity.py 200 19 > $O/stress_pauli_seed19.jsonl 2> $O/stress.err; echo "rc=$?" >> $O/stress.err
timeout 600 python bench.py --steps 5 > $O/bench_c4.json 2> $O/bench_c4.err; echo "rc=$?" >> $O/bench_c4.err
timeout 300 python bench.py --config c2_qft15 > $O/bench_c2.json 2> $O/bench_c2.err; echo "rc=$?" >> $O/bench_c2.err
