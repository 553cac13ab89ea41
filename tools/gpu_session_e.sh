set -x
timeout 300 python tools/geom_probe.py 0 0 20
timeout 600 python -c "
import json, bench
r = bench.tend_records()
print(json.dumps({k: (round(v['seconds'], 5) if isinstance(v, dict) else v) for k, v in r.items()}))
"
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
