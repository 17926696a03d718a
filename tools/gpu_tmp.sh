mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/gputest.log
for c in cfg1 cfg2; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-factored > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
python tools/host_overhead.py cfg1 > gpurun_out/host_cfg1.log 2>&1
