#!/bin/bash
# ncu evidence for one config (run under gpurun on ONE B200):
#   scripts/profile_gpu.sh <config> <tag> [<full-capture kernel regex> <skip> <count>]
# 1) plain run of the exact command (must exit 0 before any ncu)
# 2) launch list: gpu__time_duration.sum of every launch (cold-cache, serialised)
# 3) optional: --set full capture of the top kernel (DRAM bytes, stalls, source)
set -u
CFG=$1; TAG=$2; RE=${3:-}; SKIP=${4:-0}; CNT=${5:-2}
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu"
export TQSIM_JIT_LINEINFO=1
mkdir -p gpurun_out
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_ll.log 2>&1
if [ -n "$RE" ]; then
  ncu --set full --clock-control none --import-source on -k regex:$RE -s $SKIP -c $CNT \
      -o gpurun_out/${TAG}_full -f $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
fi
