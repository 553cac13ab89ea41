set -x
L=paper_2510_07539_b200/lib
for v in var_c51; do
  HSGN_LIB=$L/$v.so timeout 300 python tools/cl_probe.py 4096 20 1
  HSGN_LIB=$L/$v.so timeout 300 python tools/cl_probe.py 4096 20 3
done
timeout 300 python tools/geom_probe.py 0 0 20
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
