"""Dev probe: cfg3 (4096 x 4096) on the overlapped tiles with a caller-fixed
overlap / tile size, K timed SI steps (one graph with event nodes); per-stage
device us, HBM roofline fractions, observed rho_max.  HSGN_LIB selects a variant
build.  Usage: python tools/geom_probe.py [overlap] [tile_cells] [steps] [members]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_07539_b200 import hsgn as hs          # noqa: E402
from paper_2510_07539_b200 import workloads as W      # noqa: E402

ov = int(sys.argv[1]) if len(sys.argv) > 1 else 0
tc = int(sys.argv[2]) if len(sys.argv) > 2 else 0
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
members = int(sys.argv[4]) if len(sys.argv) > 4 else 4096
w = W.cfg3(members=members, n=4096)
s = hs.solver_for(w, overlap=ov, tile_cells=tc)
s.set_cluster(0)
s.run_steps(3)
s.sync()
ms1, ms2, tot = s.run_steps_timed(steps, total=True)
N = 4096 * members
peak = 6548.2e9
t1, t2 = ms1 / steps * 1e-3, ms2 / steps * 1e-3
d = s.diagnostics()
print(f"{os.path.basename(os.environ.get('HSGN_LIB', 'default'))} ov={ov} tc={tc} geom=({s.geometry.tile_cells},{s.geometry.overlap}): "
      f"stage1 {t1*1e6:.1f} us ({64*N/t1/peak:.3f}), stage2 {t2*1e6:.1f} us ({96*N/t2/peak:.3f}), "
      f"step {tot/steps*1e3:.1f} us, {2*N*steps/(tot*1e-3)/1e9:.2f} G cell-stage/s, rho_max {d['rho_max']:.3g}, "
      f"err {d.get('err', '?')}", flush=True)
