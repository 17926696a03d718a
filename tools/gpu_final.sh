#!/bin/bash
# Round-end evidence on one B200: GPU tests, smoke, every config's bench line (clocked),
# the reference arm, the launch list and ncu summaries of the top kernels, cold start.
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 1800 python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 900 python bench.py --config cfg1 --steps 3000 --warmup 20 > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 900 python bench.py --config cfg2 --steps 80 --warmup 20 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 1200 python bench.py --config cfg3 --steps 200 --warmup 5 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 1500 python bench.py --config cfg5 --steps 10 --warmup 3 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 900 python bench.py --mode sharded --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg4_sharded_n1.json 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 2 > $O/reference_arm.json 2> $O/reference_arm.err
python tools/cold_start.py cfg4 > $O/cold.json 2>&1
python tools/cold_start.py cfg4 --warmup > $O/cold_warmup.json 2>&1
HIKF_QHT_TIMELINE=1 python tools/qht_time.py cfg4 > $O/qht_timeline.log 2>&1
python tools/qht_time.py cfg4 15 > $O/qht_time.log 2>&1; python tools/qht_time.py cfg2 15 >> $O/qht_time.log 2>&1; python tools/qht_time.py cfg1 15 >> $O/qht_time.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_qht.csv python tools/qht_time.py cfg4 > /dev/null 2>&1
python tools/launch_summary.py $O/launches_qht.csv 40 > $O/launches_qht_summary.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-factored > $O/ncu_launch.log 2>&1
python tools/launch_summary.py $O/launches.csv 40 > $O/launches_summary.txt 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "update/" --kernel-name-base demangled \
  -k "regex:dgemm_rm_kernel.*bool.1" -c 1 -f -o $O/kgemm python tools/prof_update.py > $O/ncu_kgemm.log 2>&1
python tools/ncu_summary.py $O/kgemm.ncu-rep > $O/kgemm_summary.txt 2>&1
ncu --set full --clock-control none --import-source on -k "regex:leaf_down|m2l_prod|m2l_reduce|p2p_sparse|l2l_child|spmm_rows|m2m_pairs" -c 26 -f \
  -o $O/qht python tools/qht_time.py cfg4 > $O/ncu_qht.log 2>&1
python tools/ncu_summary.py $O/qht.ncu-rep > $O/qht_summary.txt 2>&1
rm -f $O/*.ncu-rep
