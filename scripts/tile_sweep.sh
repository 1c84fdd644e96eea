#!/bin/bash
# device ms/step per tile width: scripts/tile_sweep.sh <config> <tiles...>
c=$1; shift
for t in "$@"; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e --tile $t | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c tile $t', 'ms/step %.3f' % d['ms_per_step'], 'pass GB/s %.0f' % d['roofline']['achieved'])"
done
