"""Dev: one member-resident launch for ncu (cfg3 shape, 512 members, K steps)."""
import sys
sys.path.insert(0, "/root/repo")
from paper_2510_07539_b200 import hsgn as hs
from paper_2510_07539_b200 import workloads as W
K = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = W.cfg3(members=512)
s = hs.solver_for(w)
s.set_cluster(1)
s.run_resident(K)
print("ok")
