O=gpurun_out/r02b_small; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_small.py -x -q > $O/pytest.log 2>&1; echo "pytest_rc=$?" >> $O/pytest.log
timeout 900 python scripts/small_tree_sweep.py > $O/sweep.jsonl 2> $O/sweep.err; echo "sweep_rc=$?" >> $O/sweep.err
