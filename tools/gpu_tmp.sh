mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py -q -x > gpurun_out/t_sharded.log 2>&1; echo "rc=$?" >> gpurun_out/t_sharded.log
python tools/cold_start.py cfg4 > gpurun_out/cold.json 2>&1
CUDA_MODULE_LOADING=EAGER python tools/cold_start.py cfg4 > gpurun_out/cold_eager.json 2>&1
