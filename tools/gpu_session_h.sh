# round-2 session h: source-level ncu capture of the default stage kernels (hot spots)
set -x
timeout 600 python tools/geom_probe.py 0 0 20 > gpurun_out/r02h_geom.txt 2>&1; echo "geom rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stage_kernel -c 2 -o gpurun_out/r02h_tiles python tools/cl_probe.py 512 4 0 > gpurun_out/r02h_ncu_tiles.log 2>&1; echo "tiles rc $?"
cat gpurun_out/r02h_geom.txt
