# round-2 session k: tile shape A/B on one box -- 128 x 5 rows at 5 CTAs per SM (default) against
# 160 x 5 at 4, 192 x 5 at 3 and 96 x 5 at 7 (variant builds of the same source)
set -x
V=paper_2510_07539_b200/lib/variants
for k in 1 2; do
  timeout 300 python tools/geom_probe.py 0 0 20 >> gpurun_out/r02k_geom.txt 2>&1
  for v in nt160 nt192 nt96; do
    HSGN_LIB=$V/$v.so timeout 300 python tools/geom_probe.py 0 0 20 >> gpurun_out/r02k_geom.txt 2>&1
  done
done
cat gpurun_out/r02k_geom.txt
HSGN_LIB=$V/nt160.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_diag.py -m gpu -x -q > gpurun_out/r02k_nt160_tests.txt 2>&1; echo "nt160 tests rc $?"
tail -5 gpurun_out/r02k_nt160_tests.txt
