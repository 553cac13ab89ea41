set -x
L=paper_2510_07539_b200/lib
HSGN_LIB=$L/var_l.so timeout 300 python tools/geom_probe.py 0 0 20
timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 --no-sub --no-cpu --no-e2e 2>/dev/null | tail -1 | cut -c1-200
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -5
