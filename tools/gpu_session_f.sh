# round-2 session f: bench line, reference arm, launch list and ncu --set full of the default path
set -x
timeout 900 python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err; echo "bench rc $?"
timeout 900 python bench.py --impl reference > gpurun_out/r02f_bench_ref.json 2> gpurun_out/r02f_bench_ref.err; echo "ref rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02f_launches.csv python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu --no-sub > gpurun_out/r02f_ncu_ll.log 2>&1; echo "ll rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stage_kernel -c 2 -o gpurun_out/r02f_tiles python tools/cl_probe.py 512 4 0 > gpurun_out/r02f_ncu_tiles.log 2>&1; echo "tiles rc $?"
timeout 900 python bench.py --config cfg5 --steps 20 --warmup 3 --no-sub --no-cpu 2>/dev/null | tail -1 > gpurun_out/r02f_bench_cfg5.json; echo "cfg5 rc $?"
for a in "--scheme explicit" "--scheme sgn" "--si-order 1" "--cluster 1" "--cluster 3"; do
  timeout 600 python bench.py $a --steps 20 --warmup 3 --no-sub --no-cpu 2>/dev/null | tail -1 >> gpurun_out/r02f_variants.jsonl
done
