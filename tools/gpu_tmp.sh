mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "fused_leaf or fused_small or sparse_charges or tree_and_matmat" > gpurun_out/t_leaf.log 2>&1; echo "rc=$?" >> gpurun_out/t_leaf.log
python tools/qht_time.py cfg4 > gpurun_out/qht_fused.log 2>&1
HIKF_LEAF_FUSED=0 python tools/qht_time.py cfg4 > gpurun_out/qht_unfused.log 2>&1
HIKF_NN_TRACE=12 timeout 300 python bench.py --config cfg1 --steps 2 --warmup 3 --no-cpu-baseline --no-factored > gpurun_out/trace_cfg1.log 2>&1
HIKF_NN_TRACE=12 timeout 300 python bench.py --config cfg2 --steps 2 --warmup 3 --no-cpu-baseline --no-factored > gpurun_out/trace_cfg2.log 2>&1
timeout 600 ncu --set full --import-source on --kernel-name-base demangled -k regex:leaf_down -c 1 -f -o gpurun_out/leaf python tools/qht_time.py cfg4 > gpurun_out/ncu_leaf.log 2>&1
python tools/ncu_summary.py gpurun_out/leaf.ncu-rep > gpurun_out/leaf_summary.txt 2>&1
