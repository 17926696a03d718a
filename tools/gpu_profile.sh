#!/bin/bash
# Round evidence: the default bench line, the ncu launch list of the same command,
# ncu --set full of the K-GEMM (inside the NVTX "update" range of tools/prof_update.py)
# and of the fused leaf kernel of Q H^T; summaries land in gpurun_out/.
mkdir -p gpurun_out
python tools/qht_time.py cfg4 > gpurun_out/qht_time.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "fused_leaf or sharded" > gpurun_out/t_pre.log 2>&1 || exit 1
python bench.py --mode sharded --steps 3 --warmup 3 > gpurun_out/bench_sharded_n1.json 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-factored > gpurun_out/ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 40 > gpurun_out/launches_summary.txt 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "update/" --kernel-name-base demangled -k "regex:dgemm_rm_kernel.*bool.1" -c 1 -f \
  -o gpurun_out/kgemm python tools/prof_update.py > gpurun_out/ncu_kgemm.log 2>&1
python tools/ncu_summary.py gpurun_out/kgemm.ncu-rep > gpurun_out/kgemm_summary.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:leaf_down -c 1 -f \
  -o gpurun_out/leaf python tools/qht_time.py cfg4 > gpurun_out/ncu_leaf.log 2>&1
python tools/ncu_summary.py gpurun_out/leaf.ncu-rep > gpurun_out/leaf_summary.txt 2>&1
