# round-2 session o: final check after the bench.py changes (watchdog, cfg5 traffic): GPU tests, smoke, default bench line
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02o_gpu_tests.txt 2>&1; echo "tests rc $?"
tail -3 gpurun_out/r02o_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02o_smoke.txt 2>&1; echo "smoke rc $?"
timeout 900 python bench.py > gpurun_out/r02o_bench.json 2> gpurun_out/r02o_bench.err; echo "bench rc $?"
timeout 900 python bench.py --config cfg5 --steps 20 --warmup 3 --no-sub --no-cpu 2>/dev/null | tail -1 > gpurun_out/r02o_bench_cfg5.json; echo "cfg5 rc $?"
for a in "--scheme explicit" "--scheme sgn" "--si-order 1" "--cluster 1" "--cluster 3"; do
  timeout 600 python bench.py $a --steps 20 --warmup 3 --no-sub --no-cpu 2>/dev/null | tail -1 >> gpurun_out/r02o_variants.jsonl
done
tail -c 300 gpurun_out/r02o_bench.json
