import sys
sys.path.insert(0, "/root/repo")
from paper_2510_07539_b200 import hsgn as hs
from paper_2510_07539_b200 import workloads as W
w = W.cfg3(members=512)
s = hs.solver_for(w)
s.set_cluster(1)
s.run_resident(2)
s.run_resident(4)
print("ok")
