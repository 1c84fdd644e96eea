#!/bin/bash
# Round-end evidence (under gpurun, ONE GPU): bench lines, ncu launch lists (C4, C2), FP64 counts
# of the top families, one --set full capture of the C4 top kernel.   bash scripts/gpu_final_evidence.sh TAG
TAG=$1; O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest_rc=$?" >> $O/pytest.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1; echo "smoke_rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo "rc=$?" >> $O/bench_c4.err
timeout 600 python bench.py --config c2_qft15 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --config c3_brick20 --steps 5 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --config c5_hea28 --shard 0/16 --steps 3 --no-e2e --no-dedup-steps 0 --no-cpu > $O/bench_c5s.json 2> $O/bench_c5s.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err
bash scripts/ncu_ll.sh c4_qaoa24 $TAG/c4ll
bash scripts/ncu_fp64.sh c4_qaoa24 $TAG/c4fp "tq_trail_a_v1|tq_pass_l[5-8]" 400
bash scripts/ncu_ll.sh c2_qft15 $TAG/c2ll
bash scripts/ncu_fp64.sh c2_qft15 $TAG/c2fp "tq_pass_l9|tq_pass_l8" 40
export TQSIM_JIT_LINEINFO=1
ncu --set full --clock-control none --import-source on -k regex:tq_trail_a_v1c -c 2 -o $O/c4full -f python scripts/ncu_tree.py c4_qaoa24 $O/c4full_tree.json > $O/c4full.log 2>&1; echo "rc=$?" >> $O/c4full.log
