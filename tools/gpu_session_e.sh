set -x
L=paper_2510_07539_b200/lib
for v in var_g var_h; do HSGN_LIB=$L/$v.so timeout 300 python tools/geom_probe.py 0 0 20; done
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -25
