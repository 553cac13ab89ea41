"""Dev probe: one cfg5-recipe domain of n cells on one GPU -- single context vs
a loopback group of P slabs, overlapped tiles vs SPIKE (device ms per step).
Usage: python tools/slab_probe.py [log2 n] [P] [steps]"""
import sys; sys.path.insert(0, "/root/repo")
import torch
from paper_2510_07539_b200 import workloads as W, hsgn as hs
from tests.test_gpu_parity import gpu_solver
ln = int(sys.argv[1]) if len(sys.argv) > 1 else 24
P = int(sys.argv[2]) if len(sys.argv) > 2 else 4
K = int(sys.argv[3]) if len(sys.argv) > 3 else 10
w = W.cfg5_workload(1 << ln)


def timed(run, stream):
    run(2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    run(K)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K


for mode in (0, 3):
    s = gpu_solver(w)
    s.set_cluster(mode)
    ms = timed(s.run_steps, s.stream)
    print(f"single, mode {mode}: {ms:.3f} ms/step, {2 * w.n / (ms * 1e-3) / 1e9:.2f} G cell-stage/s")
    del s
    solvers, _ = hs.slab_solvers(w, P, align=4)
    for sv in solvers:
        sv.set_cluster(mode)
    g = hs.Group(solvers)
    ms = timed(g.run_steps, solvers[0].stream)
    print(f"{P} slabs, mode {mode}: {ms:.3f} ms/step, {2 * w.n / (ms * 1e-3) / 1e9:.2f} G cell-stage/s")
    del g, solvers
    torch.cuda.empty_cache()
