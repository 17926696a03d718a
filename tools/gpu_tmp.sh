mkdir -p gpurun_out
python tools/qht_time.py cfg4 > gpurun_out/qht_compact.log 2>&1
python tools/cold_start.py cfg4 > gpurun_out/cold.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/gputest.log
