#!/bin/bash
# A/B of an environment knob on device time per tree (under gpurun, ONE GPU):
#   bash scripts/ab_env.sh TAG "ENV=VAL" config...   -> gpurun_out/TAG/ab.txt
TAG=$1; ENVKV=$2; shift 2
O=gpurun_out/$TAG; mkdir -p $O
for c in "$@"; do
  for e in "" "$ENVKV"; do
    env $e timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e --no-dedup-steps 0 --flat-shots -1 > $O/b.json 2> $O/b.err
    python - "$c" "${e:-base}" $O/b.json >> $O/ab.txt <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[3]) if l.startswith("{")][-1])
r = d["roofline"]
top = sorted(r["kernels"], key=lambda k: -k["ms"])[:4]
print(sys.argv[1], sys.argv[2], "ms/step %.3f" % d["ms_per_step"], "clk", d["clocks"]["sm_mhz"],
      "top", r["kernel"], "frac %.3f" % r["frac"], " ".join("%s=%.2f" % (k["k"], k["ms"]) for k in top))
PY
  done
done
