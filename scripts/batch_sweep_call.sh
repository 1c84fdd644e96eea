O=gpurun_out/r02d_batch; mkdir -p $O
for spec in "c2_qft15 0" "c2_qft15 25" "c2_qft15 27" "c2_qft15 28" "c3_brick20 0" "c3_brick20 29" "c3_brick20 30"; do
  set -- $spec
  timeout 600 python bench.py --config $1 --batch-log2 $2 --steps 5 --warmup 3 --no-cpu --no-e2e --no-dedup-steps 0 > $O/b.json 2>/dev/null
  python -c "
import json
d=json.loads([l for l in open('$O/b.json') if l.startswith('{')][-1])
print('$1 batch_log2=$2', 'ms/step %.3f' % d['ms_per_step'], 'launches', d['gpu_launches'])" >> $O/sweep.txt
done
