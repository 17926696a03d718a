#!/bin/bash
# One GPU session: GPU tests, the default bench line, the launch list and one
# ncu --set full capture of the K-GEMM (each only after its command exits 0).
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-factored > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:dgemm_rm -c 1 -f \
  -o gpurun_out/kgemm python tools/prof_cfg4.py --steps 2 > gpurun_out/ncu_kgemm.log 2>&1
python tools/ncu_summary.py gpurun_out/kgemm.ncu-rep > gpurun_out/kgemm_summary.txt 2>&1
