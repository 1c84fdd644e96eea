#!/bin/bash
# Round-2 closing call (under gpurun, ONE GPU): randomised parity of the Kraus engines at 10-16
# qubits (single CTA and thread-block cluster) and of the default Pauli path at a new seed, then the
# C4 ncu launch list and one --set full capture of the top kernel at HEAD.
set -u
O=gpurun_out/s4; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
STRESS_KRAUS_N=10,16 timeout 560 python scripts/stress_parity.py 480 17 > $O/stress_kraus_10_16.jsonl 2> $O/stress_kraus.err; echo "rc=$?" >> $O/stress_kraus.err
timeout 400 python scripts/stress_parity.py 300 19 > $O/stress_pauli.jsonl 2> $O/stress_pauli.err; echo "rc=$?" >> $O/stress_pauli.err
timeout 900 bash scripts/ncu_ll.sh c4_qaoa24 s4/c4ll
export TQSIM_JIT_LINEINFO=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tq_trail_a_v1c -c 2 -o $O/c4full -f python scripts/ncu_tree.py c4_qaoa24 $O/c4full_tree.json > $O/c4full.log 2>&1; echo "rc=$?" >> $O/c4full.log
