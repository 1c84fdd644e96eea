#!/bin/bash
# ncu evidence of one config (under gpurun, ONE GPU):  bash scripts/ncu_call.sh <config> <tag> [full-capture regex] [count]
# 1) the plain command must exit 0 first; 2) launch list of one tree: time, DRAM bytes, FP64
# thread instructions per launch; 3) optional --set full capture of the top kernel(s).
set -u
CFG=$1; TAG=$2; RE=${3:-}; CNT=${4:-2}
O=gpurun_out/$TAG; mkdir -p $O
export TQSIM_JIT_LINEINFO=1
CMD="python scripts/ncu_tree.py $CFG $O/tree.json"
$CMD > $O/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
ncu --metrics $M --clock-control none -c 20000 --csv --log-file $O/launches.csv python scripts/ncu_tree.py $CFG $O/tree_ncu.json > $O/ncu_ll.log 2>&1
echo "ll_rc=$?" >> $O/ncu_ll.log
if [ -n "$RE" ]; then
  ncu --set full --clock-control none --import-source on -k regex:$RE -c $CNT -o $O/full -f $CMD > $O/ncu_full.log 2>&1
  echo "full_rc=$?" >> $O/ncu_full.log
fi
