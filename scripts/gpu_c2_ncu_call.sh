bash scripts/ncu_ll.sh c2_qft15 r02b_c2ll
export TQSIM_JIT_LINEINFO=1
O=gpurun_out/r02b_c2full; mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:tq_pass_l9_p0 -c 4 -o $O/full -f python scripts/ncu_tree.py c2_qft15 $O/tree.json > $O/ncu_full.log 2>&1; echo "rc=$?" >> $O/ncu_full.log
