# round-2 session i: staged outputs at row index (no masks) vs the previous kernels, A/B on one box
set -x
for k in 1 2; do
  HSGN_LIB=paper_2510_07539_b200/lib/variants/base.so timeout 300 python tools/geom_probe.py 0 0 20 >> gpurun_out/r02i_geom.txt 2>&1
  timeout 300 python tools/geom_probe.py 0 0 20 >> gpurun_out/r02i_geom.txt 2>&1
done
cat gpurun_out/r02i_geom.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02i_gpu_tests.txt 2>&1; echo "tests rc $?"
tail -3 gpurun_out/r02i_gpu_tests.txt
