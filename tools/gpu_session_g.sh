# round-2 session g: sanity of the restored tree (GPU tests, smoke, bench line)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02g_gpu_tests.txt 2>&1; echo "tests rc $?"
tail -3 gpurun_out/r02g_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g_smoke.txt 2>&1; echo "smoke rc $?"
timeout 900 python bench.py > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err; echo "bench rc $?"
tail -c 600 gpurun_out/r02g_bench.json
