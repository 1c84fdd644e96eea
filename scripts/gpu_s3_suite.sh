set -u
O=gpurun_out/s3g; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kraus.py -q -x > $O/kraus.log 2>&1; echo "rc=$?" >> $O/kraus.log
timeout 1800 python -m pytest tests -m gpu -q --deselect tests/test_gpu_kraus.py > $O/pytest.log 2>&1; echo "pytest_rc=$?" >> $O/pytest.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1; echo "smoke_rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo "rc=$?" >> $O/bench_c4.err
timeout 600 python bench.py --config c2_qft15 > $O/bench_c2.json 2> $O/bench_c2.err; echo "rc=$?" >> $O/bench_c2.err
