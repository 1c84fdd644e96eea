set -u
O=gpurun_out/s3i; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kraus.py -q -x > $O/kraus.log 2>&1; echo "rc=$?" >> $O/kraus.log
timeout 900 python scripts/accuracy.py noisemodels --circuits qft15h --shots 3200 --seeds 3 > $O/noisemodels_qft15h.jsonl 2> $O/nm.err; echo "rc=$?" >> $O/nm.err
