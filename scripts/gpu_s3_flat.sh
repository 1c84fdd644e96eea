set -u
O=gpurun_out/s3b; mkdir -p $O
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo "rc=$?" >> $O/bench_c4.err
timeout 600 python bench.py --config c2_qft15 > $O/bench_c2.json 2> $O/bench_c2.err; echo "rc=$?" >> $O/bench_c2.err
timeout 900 python bench.py --config c3_brick20 --steps 5 --no-cpu > $O/bench_c3.json 2> $O/bench_c3.err; echo "rc=$?" >> $O/bench_c3.err
