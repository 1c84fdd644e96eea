#!/bin/bash
# a set of pass-harness experiments (run under gpurun)
H="python scripts/microbench/pass_harness.py"
for lp in "9 0" "9 1" "8 0" "5 0" "5 1"; do
  $H c2_qft15 $lp
  $H c2_qft15 $lp --variant nocompute
done
$H c2_qft15 9 0 --careful
$H c2_qft15 8 0 --careful
$H c2_qft15 9 0 --tile 12
$H c2_qft15 8 0 --tile 12
$H c3_brick20 5 0
$H c3_brick20 5 0 --variant nocompute
$H c4_qaoa24 3 0
