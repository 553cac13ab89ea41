set -x
for a in cfg2 cfg2lat 4096; do HSGN_LIB=paper_2510_07539_b200/lib/var_timing.so timeout 300 python tools/tile_timing.py $a; done
