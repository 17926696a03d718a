# ncu captures of the Q H^T precompute kernels (run under gpurun, 1 GPU)
python tools/prof_cfg4.py > gpurun_out/prof_plain.log 2>&1 || exit 1
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
$N -k regex:box_stream -s 4 -c 2 -o gpurun_out/r01_box python tools/prof_cfg4.py > /dev/null 2>&1
$N -k regex:chol_inv_base -c 1 -o gpurun_out/r01_chol python tools/prof_cfg4.py > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
