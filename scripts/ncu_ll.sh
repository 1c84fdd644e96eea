#!/bin/bash
# ncu launch list (time + DRAM bytes) of one tree of a config (under gpurun, ONE GPU):
#   bash scripts/ncu_ll.sh <config> <tag>
set -u
CFG=$1; TAG=$2
O=gpurun_out/$TAG; mkdir -p $O
CMD="python scripts/ncu_tree.py $CFG $O/tree.json"
$CMD > $O/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 20000 --csv \
    --log-file $O/launches.csv python scripts/ncu_tree.py $CFG $O/tree_ncu.json > $O/ncu_ll.log 2>&1
echo "ll_rc=$?" >> $O/ncu_ll.log
