set -u
bash scripts/ab_env.sh s3c "TQSIM_ITEM_ORDER=1" c4_qaoa24 c2_qft15 c3_brick20
bash scripts/ab_env.sh s3d "TQSIM_PERSIST_WAVES=1" c4_qaoa24 c2_qft15
TQSIM_ITEM_ORDER=1 timeout 900 python -m pytest tests/test_gpu_golden.py -q -x > gpurun_out/s3c/golden_order1.log 2>&1; echo "rc=$?" >> gpurun_out/s3c/golden_order1.log
