#!/bin/bash
# --set full capture of the kernels matching REGEX in one C4-like tree (under gpurun, ONE GPU):
#   bash scripts/ncu_full.sh <config> <tag> <regex> [count]
set -u
CFG=$1; TAG=$2; RE=$3; CNT=${4:-2}
O=gpurun_out/$TAG; mkdir -p $O
export TQSIM_JIT_LINEINFO=1
CMD="python scripts/ncu_tree.py $CFG $O/tree.json"
$CMD > $O/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:$RE -c $CNT -o $O/full -f $CMD > $O/ncu_full.log 2>&1
echo "full_rc=$?" >> $O/ncu_full.log
