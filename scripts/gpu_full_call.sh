O=gpurun_out/${1:-r02b_full}; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
( time timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 ) > $O/pytest.log 2>&1; echo "pytest_rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke_rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench_rc=$?" >> $O/bench.log
