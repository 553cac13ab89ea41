"""Dev probe for the hsgn_run_host pipeline (numbers for DESIGN.md section 7):
pinned H2D / D2H bandwidth of the cfg3 state, device time of K steps, and the
wall time of run_host at several chunk counts.

    python tools/e2e_probe.py [members] [steps]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2510_07539_b200 import hsgn  # noqa: E402
from paper_2510_07539_b200 import workloads as W  # noqa: E402


def wall(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


def main():
    members = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    w = W.cfg3(members=members)
    N = w.n * members
    pin = [torch.from_numpy(np.ascontiguousarray(f.reshape(-1))).pin_memory() for f in (w.h, w.q, w.K, w.W)]
    outp = [torch.empty(N, dtype=torch.float64).pin_memory() for _ in range(4)]
    dev = [torch.empty(N, dtype=torch.float64, device="cuda") for _ in range(4)]
    _, th = wall(lambda: [d.copy_(p, non_blocking=True) for d, p in zip(dev, pin)])
    _, td = wall(lambda: [p.copy_(d, non_blocking=True) for d, p in zip(dev, outp)])
    gb = 4 * N * 8 / 1e9
    print(f"state {gb:.3f} GB: H2D {th * 1e3:.1f} ms ({gb / th:.1f} GB/s), D2H {td * 1e3:.1f} ms ({gb / td:.1f} GB/s)")
    s = hsgn.solver_for(w)
    s.run_steps(18)
    _, tc = wall(lambda: s.run_steps(steps))
    print(f"{steps} steps on the device: {tc * 1e3:.1f} ms")
    for ch in ([int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else (1, 2, 4, 8, 16)):
        s.run_host(*pin, steps, out=outp, chunks=ch)
        _, tr = wall(lambda: s.run_host(*pin, steps, out=outp, chunks=ch))
        print(f"run_host chunks {ch:2d}: {tr * 1e3:.1f} ms  ({2 * N * steps / tr / 1e9:.1f} G cell-stage/s)")
    s.set_state(*pin)
    _, tp = wall(lambda: (s.set_state(*pin), s.run_steps(steps), s.get_state(device=False)))
    print(f"set_state + run_steps + get_state(numpy): {tp * 1e3:.1f} ms")


if __name__ == "__main__":
    main()
