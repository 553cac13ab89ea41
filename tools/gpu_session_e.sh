set -x
for i in 1 2; do timeout 300 python tools/geom_probe.py 0 0 20; done
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
