# round-2 session j: final state of the tree -- GPU tests, smoke, bench line, reference arm, launch list, ncu --set full
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02j_gpu_tests.txt 2>&1; echo "tests rc $?"
tail -3 gpurun_out/r02j_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02j_smoke.txt 2>&1; echo "smoke rc $?"
timeout 900 python bench.py > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err; echo "bench rc $?"
timeout 900 python bench.py --impl reference > gpurun_out/r02j_bench_ref.json 2> gpurun_out/r02j_bench_ref.err; echo "ref rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02j_launches.csv python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu --no-sub > gpurun_out/r02j_ncu_ll.log 2>&1; echo "ll rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stage_kernel -c 2 -o gpurun_out/r02j_tiles python tools/cl_probe.py 512 4 0 > gpurun_out/r02j_ncu_tiles.log 2>&1; echo "tiles rc $?"
tail -c 400 gpurun_out/r02j_bench.json
