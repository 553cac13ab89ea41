# round-2 ncu captures of the exact-solve kernels (cluster, tile-level SPIKE, member-resident)
set -x
timeout 600 ncu --set full --import-source on --clock-control none -k regex:cl_stage -c 2 -o gpurun_out/r02_cluster python tools/cl_probe.py 512 4 1 > gpurun_out/r02_ncu_cluster.log 2>&1; echo "cluster rc $?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:cl_multi -c 1 -o gpurun_out/r02_resident python tools/res_prof.py > gpurun_out/r02_ncu_resident.log 2>&1; echo "resident rc $?"
timeout 600 ncu --set full --clock-control none -k "regex:cl_stage|sep_solve|filter_fix" -c 4 -o /tmp/r02_spike python tools/cl_probe.py 512 4 3 > gpurun_out/r02_ncu_spike.log 2>&1; echo "spike rc $?"
ncu -i /tmp/r02_spike.ncu-rep --page raw --csv > gpurun_out/r02_spike_raw.csv 2>&1
