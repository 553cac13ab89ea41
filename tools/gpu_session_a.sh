set -x
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02_gpu_tests.log 2>&1; echo "tests rc $?"
tail -3 gpurun_out/r02_gpu_tests.log
timeout 900 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc $?"
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err; echo "ref rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu --no-sub > gpurun_out/r02_ncu_ll.log 2>&1; echo "ll rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stage_kernel -c 2 -o gpurun_out/r02_tiles python tools/cl_probe.py 512 4 0 > gpurun_out/r02_ncu_tiles.log 2>&1; echo "tiles rc $?"
