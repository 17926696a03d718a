for g in 32 16 8; do HIKF_NN_POST_GRID=$g python bench.py --config cfg2 --steps 80 --warmup 20 --no-cpu-baseline --no-factored > gpurun_out/b2_$g.json 2>&1; done
for g in 32 8; do HIKF_NN_POST_GRID=$g python bench.py --config cfg1 --steps 2000 --warmup 20 --no-cpu-baseline --no-factored > gpurun_out/b1_$g.json 2>&1; done
python bench.py --config cfg3 --steps 60 --warmup 5 --no-cpu-baseline --no-factored > gpurun_out/b3.json 2>&1
