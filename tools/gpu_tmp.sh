mkdir -p gpurun_out
python tools/qht_time.py cfg4 > gpurun_out/qht_m2lt.log 2>&1
HIKF_M2L_TARGET=0 python tools/qht_time.py cfg4 > gpurun_out/qht_m2lp.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "target_stationary or fused_leaf or sharded or tree_and_matmat or sparse_charges or filter_cfg2" > gpurun_out/t_m2l.log 2>&1; echo "rc=$?" >> gpurun_out/t_m2l.log
