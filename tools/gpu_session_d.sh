# round-2 bench variants (one JSON line each) and a members sweep of the default path
set -x
for args in "--scheme explicit" "--scheme sgn" "--si-order 1" "--picard 1" "--wb" "--config cfg5" "--cluster 1" "--cluster 3"; do
  timeout 600 python bench.py $args --steps 20 --warmup 3 --no-sub --no-cpu 2>/dev/null | tail -1 >> gpurun_out/r02_variants.jsonl
done
for m in 512 1024 2048 4096 8192; do
  echo "== members $m"; timeout 300 python tools/cl_probe.py $m 20 0
done > gpurun_out/r02_members.log 2>&1
