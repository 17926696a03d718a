# ncu captures of the Q H^T precompute kernels (run under gpurun, 1 GPU)
python tools/prof_cfg4.py > gpurun_out/prof_plain.log 2>&1 || exit 1
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
$N -k regex:m2l_pairs -s 210 -c 1 -o gpurun_out/r01_m2l python tools/prof_cfg4.py > /dev/null 2>&1
$N -k regex:L2PProv -c 1 -o gpurun_out/r01_l2p python tools/prof_cfg4.py > /dev/null 2>&1
$N -k regex:L2LParent -s 4 -c 1 -o gpurun_out/r01_l2l python tools/prof_cfg4.py > /dev/null 2>&1
$N -k regex:pair_to_box -s 5 -c 1 -o gpurun_out/r01_p2b python tools/prof_cfg4.py > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
