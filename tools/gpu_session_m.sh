# round-2 session m: cfg5 (2^28 cells, bathymetry) launch list with DRAM bytes, and ncu --set full of its
# two stage kernels on a 2^24-cell domain of the same recipe
set -x
timeout 900 python bench.py --config cfg5 --steps 4 --warmup 3 --no-e2e --no-cpu --no-sub > gpurun_out/r02m_cfg5_plain.json 2> gpurun_out/r02m_cfg5_plain.err; echo "plain rc $?"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02m_cfg5_launches.csv python bench.py --config cfg5 --steps 4 --warmup 3 --no-e2e --no-cpu --no-sub > gpurun_out/r02m_cfg5_ll.log 2>&1; echo "ll rc $?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:stage_kernel -c 2 -o gpurun_out/r02m_cfg5_tiles python bench.py --config cfg5 --cells5 16777216 --steps 1 --warmup 3 --no-e2e --no-cpu --no-sub > gpurun_out/r02m_cfg5_full.log 2>&1; echo "full rc $?"
tail -c 300 gpurun_out/r02m_cfg5_plain.json
