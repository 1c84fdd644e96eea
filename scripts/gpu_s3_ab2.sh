set -u
bash scripts/ab_env.sh s3e "TQSIM_ITEM_ORDER=1" c2_qft15 c4_qaoa24 c2_qft15
bash scripts/ab_env.sh s3f "TQSIM_PERSIST_WAVES=4" c2_qft15 c4_qaoa24
