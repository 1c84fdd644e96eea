#!/bin/bash
# GPU tests (all, or -k EXPR) + quick device-time lines of configs:  bash scripts/gpu_test_and_quick.sh TAG "KEXPR|all|none" cfg...
TAG=$1; K=$2; shift 2
O=gpurun_out/$TAG; mkdir -p $O
if [ "$K" = "all" ]; then timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest_rc=$?" >> $O/pytest.log
elif [ "$K" != "none" ]; then timeout 2400 python -m pytest tests -m gpu -x -q -k "$K" > $O/pytest.log 2>&1; echo "pytest_rc=$?" >> $O/pytest.log; fi
for c in "$@"; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e --no-dedup-steps 0 > $O/b_$c.json 2> $O/b_$c.err
  python - "$c" $O/b_$c.json >> $O/quick.txt <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[2]) if l.startswith("{")][-1])
r = d["roofline"]
top = sorted(r["kernels"], key=lambda k: -k["ms"])[:4]
print(sys.argv[1], "ms/step %.3f" % d["ms_per_step"], "clk", d["clocks"]["sm_mhz"], "top", r["kernel"],
      "frac %.3f" % r["frac"], " ".join("%s=%.3f" % (k["k"], k["ms"]) for k in top))
PY
done
