O=gpurun_out/r02c; mkdir -p $O
(cd scripts/microbench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/gtb gather_tile_bench.cu && /tmp/gtb > ../../$O/gather_tile_bench.txt 2>&1)
timeout 1200 python -m pytest tests -m gpu -x -q -k "kraus or c5_full or accuracy or split_level or all_instance or all_leaf or beta0" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for st in table3 errfreq shots; do timeout 600 python scripts/accuracy.py $st > $O/acc_$st.jsonl 2> $O/acc_$st.err; done
timeout 900 python scripts/accuracy.py noisemodels > $O/acc_noisemodels.jsonl 2> $O/acc_noisemodels.err
timeout 600 python scripts/accuracy.py fidelity > $O/acc_fidelity.jsonl 2> $O/acc_fidelity.err
