set -u
O=gpurun_out/s3h; mkdir -p $O
timeout 900 python scripts/accuracy.py noisemodels --circuits qft15h --shots 3200 --seeds 3 > $O/noisemodels_qft15h.jsonl 2> $O/nm.err; echo "rc=$?" >> $O/nm.err
