#!/bin/bash
# One gpurun call: GPU tests, bench, microbenchmarks (usage: bash scripts/gpu_call.sh TAG "PYTEST -k EXPR" [bench args])
TAG=${1:-run}; KEXPR=${2:-}; shift 2; BARGS="$@"
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
if [ -n "$KEXPR" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$KEXPR" > $O/pytest.log 2>&1; echo "pytest_rc=$?" >> $O/pytest.log
fi
timeout 600 python bench.py $BARGS > $O/bench.log 2>&1; echo "bench_rc=$?" >> $O/bench.log
