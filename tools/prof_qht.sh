N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
$N -k regex:box_warp_kernel -c 8 -f -o /tmp/q1 python tools/prof_cfg4.py --steps 0 > gpurun_out/q1.log 2>&1
$N -k "regex:p2p_sparse|spmm_rows|p2p_scatter|m2m_pairs|p2m|sparse_build|regroup" -c 10 -f -o /tmp/q2 python tools/prof_cfg4.py --steps 0 > gpurun_out/q2.log 2>&1
$N -k regex:m2l_pairs -s 150 -c 6 -f -o /tmp/q3 python tools/prof_cfg4.py --steps 0 > gpurun_out/q3.log 2>&1
for q in q1 q2 q3; do python tools/ncu_summary.py /tmp/$q.ncu-rep > gpurun_out/${q}_summary.txt; ncu -i /tmp/$q.ncu-rep --page details --csv > gpurun_out/${q}_details.csv; done
cat gpurun_out/q*_summary.txt
