set -u
O=gpurun_out/s3a; mkdir -p $O/dump_c2 $O/dump_c4
TQSIM_JIT_DUMP=$O/dump_c2 timeout 300 python scripts/ncu_tree.py c2_qft15 $O/c2_tree.json > $O/c2dump.log 2>&1
TQSIM_JIT_DUMP=$O/dump_c4 timeout 600 python scripts/ncu_tree.py c4_qaoa24 $O/c4_tree.json > $O/c4dump.log 2>&1
for f in $O/dump_c2/*.cubin $O/dump_c4/*trail_a*.cubin; do cuobjdump -res-usage $f 2>/dev/null | grep -E "Function|REG" ; done > $O/resusage.txt 2>&1
export TQSIM_JIT_LINEINFO=1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:tq_pass_l9_p0_v1$' -c 2 -o $O/c2v1 -f python scripts/ncu_tree.py c2_qft15 $O/c2b.json > $O/ncu_c2v1.log 2>&1; echo "rc=$?" >> $O/ncu_c2v1.log
du -sh $O
