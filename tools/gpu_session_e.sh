set -x
L=paper_2510_07539_b200/lib
for v in var_cur var_wa var_hb; do HSGN_LIB=$L/$v.so timeout 300 python tools/geom_probe.py 0 0 20; done
