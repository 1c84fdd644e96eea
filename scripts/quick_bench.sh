#!/bin/bash
# quick device-time comparison: ms/step and pass-kernel GB/s for the given configs
for c in "$@"; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', 'ms/step %.3f' % d['ms_per_step'], 'pass GB/s %.0f' % d['roofline']['achieved'], 'pass share %.3f' % d['roofline']['pass_share_of_step'], 'top', d['roofline']['top_kernel']['name'], '%.0f GB/s' % d['roofline']['top_kernel']['achieved_gbs'], 'launches', d['gpu_launches'])"
done
