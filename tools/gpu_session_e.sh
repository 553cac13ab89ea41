set -x
timeout 300 python tools/geom_probe.py 0 0 20
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
