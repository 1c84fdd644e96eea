#!/bin/bash
# FP64 instruction counts + DRAM bytes of the launches of the kernels matching REGEX in one tree
#   bash scripts/ncu_fp64.sh <config> <tag> <regex> [count]
set -u
CFG=$1; TAG=$2; RE=$3; CNT=${4:-64}
O=gpurun_out/$TAG; mkdir -p $O
CMD="python scripts/ncu_tree.py $CFG $O/tree.json"
$CMD > $O/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
ncu --metrics $M --clock-control none -k regex:$RE -c $CNT --csv --log-file $O/fp64.csv python scripts/ncu_tree.py $CFG $O/tree_ncu.json > $O/ncu_fp64.log 2>&1
echo "rc=$?" >> $O/ncu_fp64.log
