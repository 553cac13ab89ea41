#!/usr/bin/env python
"""Benchmark of the SI-IMEX hSGN hot path (BASELINE.json metric:
"fp64 cell-stage updates/s per GPU and whole box; % of HBM roofline").

Workload: BASELINE configs[2] = cfg3, the batched
ensemble of 4096 periodic domains x 4096 cells (seeded synthetic solitary
waves, lambda log-uniform in [1e2, 1e4], CFL_IMEX 2, MCFL 0.5).  It is the
largest single-GPU throughput config whose roofline is meaningful (state
512 MiB > L2, so no L2 flush is needed between steps).  One bench "step" = one
SI-IMEX step (2 stages) over the whole batch.  Multi-GPU: one process per GPU,
each runs its own 4096-member shard of a 4096*N-member ensemble (weak scaling,
no data-path collective: members are independent).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl hsgn|reference]

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 cell-stage updates/s (whole job)"
UNIT = "cell-stage/s"
CFL_EX = 0.4          # explicit scheme CFL
CFL_SGN = 0.9         # classical SGN scheme CFL
B_STAGE1 = 64   # algorithmic bytes per cell: read U^n (32), write U1 (32)
B_STAGE2 = 96   # read U^n + U1 (64), write U^{n+1} (32)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="hsgn", choices=["hsgn", "reference"])
    p.add_argument("--members", type=int, default=4096)
    p.add_argument("--cells", type=int, default=4096)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--e2e-chunks", type=int, default=8,
                   help="member chunks of the e2e job (hsgn_run_host copy/compute pipeline)")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--si-order", type=int, default=2, choices=[1, 2],
                   help="2: the paper's second-order SI step (headline); 1: first-order SI "
                        "(one implicit stage tau = dt, order-1 faces; SURVEY row f2)")
    p.add_argument("--picard", type=int, default=0,
                   help="Picard passes of the SI depth solve (reading A24, SURVEY row f4); 0: the paper's")
    p.add_argument("--wb", action="store_true",
                   help="exactly well-balanced face form of the SI stage (reading A25, SURVEY row f4)")
    p.add_argument("--scheme", default="si", choices=["si", "explicit", "sgn"],
                   help="si: the SI-IMEX step (headline); explicit: the explicit hSGN scheme "
                        "(Heun, CFL_EX 0.4); sgn: the classical SGN scheme (Heun, CFL_SGN 0.9) "
                        "on the same workload")
    p.add_argument("--cluster", type=int, default=-1,
                   help="1: cluster stage kernels (exact cross-CTA depth solve) whenever the member fits, "
                        "0: overlapped tiles, -1: library default (auto)")
    p.add_argument("--config", default="cfg3", choices=["cfg3", "cfg5"],
                   help="cfg3: ensemble (default, headline); cfg5: single 2^28-cell domain with bathymetry")
    p.add_argument("--cells5", type=int, default=1 << 28)
    p.add_argument("--no-sub", action="store_true",
                   help="skip the cfg5 and time-to-t_end sub-records of the default (cfg3) line")
    return p.parse_args()


def config_dict(a, world):
    d = _config_dict(a, world)
    if a.picard > 0:
        d["picard_passes"] = a.picard
    if a.wb:
        d["well_balanced"] = "A25 face form"
    if a.si_order == 1:
        d["scheme"] = "first-order SI (P:500-517: one implicit stage, tau = dt, order-1 faces)"
        d["order"] = 1
        d["tableau"] = "SI Euler (a_11 = 1)"
    if a.scheme == "sgn":
        d["scheme"] = "classical SGN (P:519-600): Heun, CFL_SGN 0.9, MUSCL + Rusanov, phi tridiagonal"
        d.pop("cfl_imex", None)
        d.pop("mcfl", None)
        d.pop("tableau", None)
        d["filter"] = "none"
    if a.scheme == "explicit":
        d["scheme"] = "explicit hSGN (P:442-480): Heun, CFL_EX 0.4, MUSCL + Rusanov, A19 filter"
        d.pop("cfl_imex", None)
        d.pop("mcfl", None)
        d.pop("tableau", None)
    return d


def _config_dict(a, world):
    if a.config == "cfg5":
        return {"workload": "cfg5_large_domain: %d cells, periodic, bathymetry 0.2 sin, lambda 1e4, "
                            "100-step config, A19 filter" % a.cells5, "cells": a.cells5,
                "cfl_imex": 2.0, "mcfl": 0.5, "order": 2,
                "parallelism": f"slabs x{world} (NCCL halo exchange + dt all-reduce)" if world > 1 else "single GPU",
                "l2": "inputs (8 GiB state) larger than L2: no flush"}
    return {"workload": "cfg3_ensemble: %d members x %d cells per GPU, periodic, 200-step config"
                        % (a.members, a.cells),
            "members_per_gpu": a.members, "cells_per_member": a.cells,
            "global_members": a.members * world, "lambda": "log-uniform [1e2, 1e4] per member",
            "cfl_imex": 2.0, "mcfl": 0.5, "order": 2, "tableau": "P:371-386 (gamma = 1 - 1/sqrt2)",
            "filter": "A19, sigma 0.25 on q and W", "parallelism": f"ensemble-sharded x{world}",
            "l2": "inputs (512 MiB state) larger than L2 (126 MB): no flush"}


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


def profile_fp64():
    """fp64 arithmetic of the stage-2 kernel from the committed ncu capture
    (profiles/ncu_summary.json: DADD + DMUL + 2 DFMA per cycle) against the
    measured DFMA peak (profiles/r01_dfma_peak.json, tools/dfma_peak.cu): the kernels are issue /
    latency-bound, neither HBM- nor fp64-bound."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        k = [x for x in d["full"] if "S2=1" in x["kernel"]][0]
        pk = d["fp64_peak_tflops"]
        return {"achieved": k["fp64_tflops"], "peak": pk, "unit": "TFLOP/s", "frac": k["fp64_tflops"] / pk,
                "pipe_active_pct": k["fp64_pipe_pct"], "issue_active_pct": k["issue_active_pct"],
                "source": d.get("summary", "profiles/r01_ncu_summary.md") + " (ncu --set full, 512 x 4096 cells)"}
    except Exception:
        return None


def profile_traffic(cells, bathy=False):
    """dram__bytes_read.sum + dram__bytes_write.sum per stage-2 launch, from the
    committed ncu launch list of the same workload (profiles/ncu_summary.json:
    cfg3, or cfg5 for the kernels with bathymetry), scaled to this run's cells
    per launch."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        b = (d.get("cfg5") or {}).get("stage2_dram_bytes_per_cell") if bathy else d.get("stage2_dram_bytes_per_cell")
        return None if b is None else b * cells
    except Exception:
        return None


# ---------------------------------------------------------------------------
# CPU oracle baseline (test infrastructure; timed only here, never on the product path)
# ---------------------------------------------------------------------------
def cpu_oracle_rate(w, members, steps, threads, min_seconds=0.0, explicit=False, si_order=2, picard=0,
                    wb=False):
    """Oracle cell-stage/s on the host cores (one member per thread), repeated
    until at least min_seconds of wall time; returns (rate, seconds, repeats)."""
    from oracle import oracle as O
    tab = O.euler_tableau() if si_order == 1 else None
    sig = 0.0 if explicit == "sgn" else w.filter_sigma
    jobs = [(O.Oracle(w.n, w.dx, g=w.g, lam=float(w.lam[m]), bc=w.bc, b=w.b, order=si_order,
                      filter_sigma=sig, tableau=tab, picard=picard, wb=wb), w.state(m)) for m in members]
    t0 = time.perf_counter()
    reps = 0
    while True:
        if explicit == "sgn":
            O.run_members(jobs, threads=threads, sgn=True, cfl=CFL_SGN, steps=steps)
        elif explicit:
            O.run_members(jobs, threads=threads, explicit=True, cfl=CFL_EX, steps=steps)
        else:
            O.run_members(jobs, threads=threads, cfl=w.cfl, mcfl=w.mcfl, steps=steps)
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= min_seconds:
            break
    return (1.0 if si_order == 1 and not explicit else 2.0) * w.n * len(members) * steps * reps / dt, dt, reps


def run_reference(a, rank, world):
    """--impl reference: the oracle (plain fp64 C, -O2, no FMA) on the host cores,
    each step a bounded sample of the same workload."""
    if rank != 0:
        return
    from paper_2510_07539_b200 import workloads as W
    threads = os.cpu_count() or 1
    sample_members = max(16 * threads, 64)
    w = W.cfg3(members=sample_members, n=a.cells)
    cpu_oracle_rate(w, range(sample_members), max(1, a.warmup), threads)
    rate, secs, _ = cpu_oracle_rate(w, range(sample_members), a.steps, threads)
    ms = secs / a.steps * 1e3
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(a, world),
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": f"{sample_members} cfg3 members x {a.steps} SI steps per run "
                                       f"(each bench step = 1 SI step over {sample_members} members)"},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        run_reference(a, rank, world)
        return
    import torch
    import torch.distributed as dist
    from paper_2510_07539_b200 import hsgn
    from paper_2510_07539_b200 import workloads as W

    backend = os.environ.get("HSGN_BENCH_BACKEND", "nccl") if world > 1 else "none"
    ngpu = max(torch.cuda.device_count(), 1)
    if backend != "nccl":
        local = local % ngpu          # (gloo: several ranks may share a GPU)
    elif local >= ngpu:
        raise SystemExit(f"LOCAL_RANK {local} but only {ngpu} GPUs visible (NCCL needs one GPU per rank)")
    phys_gpus = min(world, ngpu) if backend != "nccl" else world
    if a.config == "cfg5" and world > 1 and backend != "nccl":
        raise SystemExit("--config cfg5 over several ranks needs the NCCL slab transport (one GPU per rank)")
    torch.cuda.set_device(local)
    if world > 1 and backend == "nccl":
        # NCCL's communicator set-up (rings / NVLS) visible on stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if world > 1:
        # HSGN_BENCH_BACKEND=gloo: host-side collectives only (exercises the
        # multi-rank path with several ranks on one GPU; the ranks' kernels never
        # wait on each other: the ensemble shards need no data-path exchange)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    coll_dev = "cuda" if (world == 1 or os.environ.get("HSGN_BENCH_BACKEND", "nccl") == "nccl") else "cpu"

    bathy = False
    slab = a.config == "cfg5" and world > 1
    if a.config == "cfg5":
        # one large periodic domain with bathymetry, generated on the device; on
        # N GPUs each rank owns a contiguous slab (halo exchange + dt all-reduce
        # over NCCL inside libhsgn): strong scaling
        from paper_2510_07539_b200 import dist as D
        lo, hi = D.slab_range(a.cells5, rank, world)
        (h, q, K, Wf, b), meta = W.cfg5(a.cells5, device="cuda", first=lo, count=hi - lo)
        dx = meta["L"] / meta["n"]
        s = hsgn.Solver(hi - lo, 1, lo * dx, hi * dx,
                        bc=("halo", "halo") if slab else ("periodic", "periodic"))
        s.set_params(9.81, meta["lam"], meta["cfl"], meta["mcfl"])
        s.set_bathymetry(b)
        s.set_filter(0.25)
        s.set_state(h, q, K, Wf)
        if slab:
            D.attach_slab(s, rank, world)
        host_state = [x.cpu() for x in (h, q, K, Wf)] if not a.no_e2e else None
        del h, q, K, Wf
        Ntot = hi - lo
        bathy = True

        class _W:   # minimal stand-in for the e2e/cpu legs
            members = 1
            n = hi - lo
        w = _W()
    else:
        w = W.cfg3(members=a.members, n=a.cells, first_member=rank * a.members)
        s = hsgn.solver_for(w)
        Ntot = w.n * w.members
        host_state = None
    if a.si_order == 1:
        if a.config != "cfg3" or a.scheme != "si":
            raise SystemExit("--si-order 1: cfg3 SI only")
        s.close()
        s = hsgn.Solver(w.n, w.members, w.x_min, w.x_max, bc=w.bc, order=1)
        s.set_params(w.g, w.lam, w.cfl, w.mcfl)
        s.set_tableau(hsgn.euler_tableau())
        s.set_filter(w.filter_sigma)
        s.set_state(w.h.reshape(-1), w.q.reshape(-1), w.K.reshape(-1), w.W.reshape(-1))
    if a.picard > 0:
        s.set_picard(a.picard)
    if a.wb:
        if a.scheme != "si" or a.picard > 0:
            raise SystemExit("--wb: SI scheme without Picard passes")
        s.set_well_balanced(True)
    if a.scheme == "explicit":
        if a.config != "cfg3":
            raise SystemExit("--scheme explicit: cfg3 only (the explicit scheme needs a flat bottom)")
        s.set_params(w.g, w.lam, CFL_EX, 0.0)
        s.set_scheme("explicit", 2)
    if a.scheme == "sgn":
        if a.config != "cfg3":
            raise SystemExit("--scheme sgn: cfg3 only (flat bottom)")
        s.set_filter(0.0)
        s.set_params(w.g, w.lam, CFL_SGN, 0.0)
        s.set_scheme("sgn", 2)
    if a.cluster >= 0:
        s.set_cluster(a.cluster)
    state_bytes = 4 * 8 * Ntot

    def barrier():
        if world > 1:
            dist.barrier()

    # warm-up (also captures the CUDA graph)
    s.run_steps(max(a.warmup, 3))
    s.sync()
    torch.cuda.synchronize()

    stream = s.stream
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    l0 = s.launches
    barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    if slab:
        s.run_steps(a.steps)       # per-stage events are not recorded for slab contexts
        ms1 = ms2 = None
    else:
        # the K steps as one CUDA graph with event nodes between the kernels
        # (hsgn_run_steps_timed): device time of the steps and of each stage kernel
        ms1, ms2, ms_steps = s.run_steps_timed(a.steps, total=True)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ck = clocks.stop()
    launches = s.launches - l0
    elapsed = ev0.elapsed_time(ev1) if slab else ms_steps
    if slab:
        ms1 = ms2 = 0.5 * elapsed        # step-average model below
    t = torch.tensor([elapsed, ms1, ms2], device=coll_dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed, ms1, ms2 = [float(x) for x in t.tolist()]
    diag = s.diagnostics()

    nst = 1 if a.si_order == 1 else 2                         # cell-stages per cell and step
    value = nst * Ntot * a.steps * world / (elapsed / 1e3)    # Ntot = cells of this rank
    peaks, peak_src = measured_peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))
    if nst == 1:
        ms2 = ms1                      # the one (final) stage: U^n -> U^{n+1}, 64 B/cell
    t2 = ms2 / a.steps / 1e3
    t1 = ms1 / a.steps / 1e3
    bs1 = B_STAGE1 + (8 if bathy else 0)    # + b read per stage
    bs2 = (B_STAGE1 if nst == 1 else B_STAGE2) + (8 if bathy else 0)
    if a.scheme == "sgn":
        # (h, q) only: stage 1 reads X, writes U1 (32 B); stage 2 reads U1, U^n,
        # writes U^{n+1} (48 B) + carries K, W (32 B)
        bs1, bs2 = 32, 80
    ach2 = bs2 * Ntot / t2 / 1e9
    ach1 = bs1 * Ntot / t1 / 1e9
    # which depth-solve organisation ran (auto mode: DESIGN.md section 6); the
    # committed ncu traffic belongs to the overlapped-tile stage kernels
    org = ("cluster" if (a.scheme == "si" and s.cluster) else "spike" if (a.scheme == "si" and s.spike)
           else "tiles")
    traffic = profile_traffic(Ntot, bathy=bathy) if org == "tiles" and a.scheme == "si" and nst == 2 else None

    # e2e through the public API with host buffers: pinned host state in, K steps,
    # final state and per-member times out (hsgn_run_host; after the device-timed
    # region and the diagnostics, since the job leaves the solver without a state)
    e2e = None
    if not a.no_e2e:
        if host_state is not None:
            pin = [x.pin_memory() for x in host_state]
        else:
            pin = [torch.from_numpy(np.ascontiguousarray(f.reshape(-1))).pin_memory() for f in (w.h, w.q, w.K, w.W)]
        outp = [torch.empty(Ntot, dtype=torch.float64).pin_memory() for _ in range(4)]
        plain_e2e = slab or a.scheme == "sgn"
        if plain_e2e:
            # slab contexts (cfg5 over N GPUs) exchange halos every stage, and the SGN
            # tile geometry depends on the whole state: no member chunks to pipeline;
            # set_state + run_steps + get_state through pinned buffers
            import ctypes as C
            barrier()
            torch.cuda.synchronize()
            te0 = time.perf_counter()
            s.set_state(*pin)
            s.run_steps(a.steps)
            tt = np.empty(w.members)
            s._chk(s.L.hsgn_get_state(s.ctx, *[C.c_void_p(x.data_ptr()) for x in outp], C.c_void_p(tt.ctypes.data)))
            te = time.perf_counter() - te0
        else:
            # one untimed job first (the chunk views capture their step graphs), then the timed one
            s.run_host(*pin, a.steps, out=outp, chunks=a.e2e_chunks)
            barrier()
            torch.cuda.synchronize()
            te0 = time.perf_counter()
            _, tt = s.run_host(*pin, a.steps, out=outp, chunks=a.e2e_chunks)
            te = time.perf_counter() - te0
        tt_ = torch.tensor([te], device=coll_dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tt_, op=dist.ReduceOp.MAX)
        te = float(tt_.item())
        e2e = {"value": nst * Ntot * a.steps * world / te, "unit": UNIT,
               "h2d_bytes_per_step": state_bytes / a.steps,
               "d2h_bytes_per_step": (state_bytes + 8 * w.members) / a.steps,
               "what": ("Solver.set_state(pinned) + run_steps(K) + get_state(pinned); wall clock, max over ranks"
                        if plain_e2e else
                        f"Solver.run_host (hsgn_run_host): pinned host state in, K steps, final state and "
                        f"times out, pipelined over {a.e2e_chunks} member chunks; wall clock, max over ranks")}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu and a.config == "cfg3":   # N = 1 only
        threads = os.cpu_count() or 1
        nm = max(4 * threads, 16)
        rate, secs, reps = cpu_oracle_rate(w.subset(range(nm)), range(nm), 10, threads, min_seconds=10.0,
                                           explicit="sgn" if a.scheme == "sgn" else a.scheme == "explicit",
                                           si_order=a.si_order, picard=a.picard, wb=a.wb)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": f"first {nm} cfg3 members x 10 "
                         f"{ {'explicit': 'explicit Heun', 'sgn': 'classical SGN Heun'}.get(a.scheme, 'SI')} "
                         f"steps, repeated {reps}x ({secs:.1f} s wall)"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": elapsed / a.steps, "higher_is_better": True,
        "scaling": "strong" if a.config == "cfg5" else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(a, world),
        "per_gpu": value / world,
        "roofline": {"bound": "hbm", "achieved": ach2, "peak": peak, "unit": "GB/s",
                     "frac": ach2 / peak, "traffic": traffic,
                     "kernel": ("sgn_kernel<HEUN2,FINAL> (Heun stage 2)" if a.scheme == "sgn"
                                else "explicit_kernel<HEUN2,FINAL> (Heun stage 2)" if a.scheme == "explicit"
                                else ("cl_stage_kernel (cluster, exact solve)" if org == "cluster" else
                                      "cl_stage_kernel TIPS + sep_solve + FINISH (tile-level SPIKE)" if org == "spike"
                                      else "stage_kernel") +
                                     (" <FINAL> (the one SI stage)" if nst == 1 else " <STAGE2,FINAL> (stage 2)")),
                     "bytes_model": (f"{bs2} B/cell per launch (read U^n; write U^{{n+1}})" if nst == 1 else
                                     f"{bs2} B/cell per stage-2 launch (read U^n, U1{', b' if bathy else ''}; write U^{{n+1}})"),
                     "peak_source": peak_src,
                     "stage1": {"achieved": ach1, "frac": ach1 / peak, "bytes_model": f"{bs1} B/cell"},
                     "step_avg_frac": ((ach2 / peak) if nst == 1 else
                                       (0.5 * (bs1 + bs2) * 2 * Ntot / ((ms1 + ms2) / a.steps / 1e3) / 1e9) / peak),
                     "fp64": profile_fp64() if a.scheme == "si" and a.config == "cfg3" and nst == 2 else None},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches * world,
        "clocks": ck,
        "diag": {"steps": diag["steps"], "mass": diag["mass"], "min_h": diag["min_h"],
                 "t_max": diag["t_max"], "dt_last_min": diag["dt_last_min"]},
    }
    if phys_gpus != world:
        line["shared_gpu"] = f"{world} ranks on {phys_gpus} GPU(s) (gloo test mode)"
    sub_failed = False
    # sub-records: cfg5 (the largest single-GPU config; over NCCL slabs at N > 1,
    # strong scaling) and the times to t_end of the other configs (rank 0)
    if not a.no_sub and a.config == "cfg3" and a.scheme == "si" and a.si_order == 2 and a.picard == 0 \
            and not a.wb:
        del s
        torch.cuda.empty_cache()
        subs = {}
        # N > 1: the cfg5 sub-record is the one leg with a data-path collective (NCCL
        # inside libhsgn).  A failure or a hang there must not cost the headline line:
        # errors are recorded in the sub-record, and a watchdog thread on every rank
        # prints the line as it stands (rank 0) and leaves after SUB_TIMEOUT_S.
        done = _watchdog(line, subs, rank) if world > 1 else None
        if backend in ("none", "nccl"):
            try:
                subs["cfg5"] = cfg5_record(a, rank, world, dist, coll_dev, peak, peak_src)
            except Exception as e:          # noqa: BLE001 (reported, not swallowed)
                if world == 1:
                    raise
                subs["cfg5"] = {"error": f"{type(e).__name__}: {e}"[:400]}
                sub_failed = True
        if rank == 0 and not sub_failed:     # (after a failed leg the CUDA context may be unusable)
            subs["cfg3_resident"] = resident_record(a)
            subs["time_to_t_end"] = tend_records()
        if rank == 0:
            line["sub_records"] = subs
        if done is not None:
            done.set()
    if rank == 0:
        with _PRINT_LOCK:
            if not _PRINTED:
                _PRINTED.append(1)
                print(json.dumps(line), flush=True)
    if world > 1:
        # (a rank whose cfg5 leg failed may have left its peers inside a collective:
        # they leave through their watchdogs; do not wait for them here)
        if not sub_failed:
            dist.destroy_process_group()
        else:
            sys.stdout.flush()
            os._exit(0)


SUB_TIMEOUT_S = float(os.environ.get("HSGN_BENCH_SUB_TIMEOUT", "300"))
_PRINT_LOCK = threading.Lock()
_PRINTED = []


def _watchdog(line, subs, rank):
    """Multi-rank runs: if the sub-records have not finished after SUB_TIMEOUT_S
    (a rank stuck in a collective), rank 0 prints the headline line with what it
    has and every rank exits 0."""
    done = threading.Event()

    def run():
        if done.wait(SUB_TIMEOUT_S):
            return
        if rank == 0:
            with _PRINT_LOCK:
                if not _PRINTED:
                    _PRINTED.append(1)
                    part = dict(subs)
                    part.setdefault("cfg5", {"error": f"sub-records timed out after {SUB_TIMEOUT_S:g} s"})
                    out = dict(line)
                    out["sub_records"] = part
                    print(json.dumps(out), flush=True)
        sys.stdout.flush()
        os._exit(0)

    threading.Thread(target=run, daemon=True).start()
    return done


def _timed(stream, fn):
    """device seconds (CUDA events on the solver's stream) and wall seconds of fn()"""
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e0.record(stream)
    out = fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1) / 1e3, time.perf_counter() - w0


def cfg5_record(a, rank, world, dist, coll_dev, peak, peak_src):
    """BASELINE configs[4]: one periodic domain of a.cells5 cells with bathymetry,
    its 100-step configuration.  N = 1: one context; N > 1: contiguous slabs,
    one per rank, halo exchange + dt all-reduce over NCCL inside libhsgn
    (strong scaling).  Device time of the 100 steps (max over ranks), the
    stage-2 roofline (104 B/cell: U^n, U1, b read, U^{n+1} written; N = 1) and
    the end-to-end job through the public API: set_state from pinned host
    memory, the 100 steps, get_state into pinned host memory (wall clock)."""
    import ctypes as C
    import torch
    from paper_2510_07539_b200 import dist as D
    from paper_2510_07539_b200 import hsgn
    from paper_2510_07539_b200 import workloads as W
    n = a.cells5
    lo, hi = D.slab_range(n, rank, world)
    (h, q, K, Wf, b), meta = W.cfg5(n, device="cuda", first=lo, count=hi - lo)
    dx = meta["L"] / meta["n"]
    slab = world > 1
    s = hsgn.Solver(hi - lo, 1, lo * dx, hi * dx, bc=("halo", "halo") if slab else ("periodic", "periodic"))
    s.set_params(9.81, meta["lam"], meta["cfl"], meta["mcfl"])
    s.set_bathymetry(b)
    s.set_filter(0.25)
    s.set_state(h, q, K, Wf)
    if slab:
        D.attach_slab(s, rank, world)
    steps = int(meta["steps"])
    s.run_steps(6)
    s.sync()
    if world > 1:
        dist.barrier()
    if slab:
        _, dev, _ = _timed(s.stream, lambda: s.run_steps(steps))
        ms1 = ms2 = None
    else:
        ms1, ms2, tot = s.run_steps_timed(steps, total=True)
        dev = tot / 1e3
    t = torch.tensor([dev], device=coll_dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev = float(t.item())
    cells = hi - lo
    rec = {"workload": f"cfg5_large_domain: {n} cells, periodic, bathymetry 0.2 sin, lambda 1e4, "
                       f"{steps}-step config, A19 filter",
           "value": 2.0 * n * steps / dev, "unit": UNIT, "n_gpus": world, "steps": steps,
           "ms_per_step": dev / steps * 1e3, "time_to_end_s": dev,
           "scaling": "strong", "parallelism": (f"slabs x{world} (NCCL send/recv halos + all-reduce max)"
                                                if slab else "single GPU")}
    if not slab:
        ach = 104.0 * cells / (ms2 / steps / 1e3) / 1e9
        rec["roofline"] = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                           "kernel": "stage_kernel<STAGE2,FINAL,BATHY> (stage 2)",
                           "bytes_model": "104 B/cell per stage-2 launch (read U^n, U1, b; write U^{n+1})",
                           "peak_source": peak_src, "traffic": profile_traffic(cells, bathy=True),
                           "stage1_frac": 72.0 * cells / (ms1 / steps / 1e3) / 1e9 / peak}
    if not a.no_e2e:
        pin = [x.cpu().pin_memory() for x in (h, q, K, Wf)]
        del h, q, K, Wf
        outp = [torch.empty(cells, dtype=torch.float64).pin_memory() for _ in range(4)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        te0 = time.perf_counter()
        s.set_state(*pin)
        s.run_steps(steps)
        tt = np.empty(1)
        s._chk(s.L.hsgn_get_state(s.ctx, *[C.c_void_p(x.data_ptr()) for x in outp], C.c_void_p(tt.ctypes.data)))
        te = time.perf_counter() - te0
        t = torch.tensor([te], device=coll_dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        te = float(t.item())
        rec["e2e"] = {"value": 2.0 * n * steps / te, "unit": UNIT, "seconds": te,
                      "h2d_bytes": 32 * cells * world, "d2h_bytes": 32 * cells * world + 8,
                      "what": "Solver.set_state(pinned host) + run_steps(100) + get_state(pinned host) of the "
                              "whole 100-step job; wall clock, max over ranks (a single coupled domain: the "
                              "first step needs the global dt of the whole uploaded state)"}
    else:
        del h, q, K, Wf
    s.close()
    del s
    torch.cuda.empty_cache()
    return rec


def resident_record(a):
    """cfg3 on the member-resident kernel (hsgn_run_resident, one launch of
    a.steps steps; every member's state, stage inputs and intermediates stay in
    its cluster's shared memory, so HBM sees 64 B/cell per launch, not per
    stage): device time with CUDA events inside the call."""
    from paper_2510_07539_b200 import hsgn
    from paper_2510_07539_b200 import workloads as W
    w = W.cfg3(members=a.members, n=a.cells)
    s = hsgn.solver_for(w)
    s.run_resident(max(a.warmup, 3))
    k = max(a.steps, 10)
    ms = s.run_resident(k)
    d = s.diagnostics()
    s.set_cluster(1)                                # (only to read the cluster shape back)
    cl = list(s.cluster) if s.cluster else None
    cs = 2.0 * w.n * w.members * k
    rec = {"value": cs / (ms * 1e-3), "unit": "cell-stage/s", "steps": k, "ms_per_step": ms / k,
           "launches": 1, "cluster_ctas_x_rows": cl,
           "hbm_bytes_per_launch": 64 * w.n * w.members,
           "bound": "latency of the in-cluster exchanges and fp64 issue (no per-step HBM traffic)",
           "mass": d["mass"], "steps_done": d["steps"]}
    del s
    return rec


def _steps_to(w, t_end):
    """steps the dt rule takes to t_end (hsgn_step with return_dt on the
    overlapped tiles; not timed)"""
    from paper_2510_07539_b200 import hsgn
    s = hsgn.solver_for(w)
    t, k = 0.0, 0
    while t < t_end and k < 100000:
        d = float(s.step(return_dt=True)[0])
        if d <= 0.0:
            break
        t += d
        k += 1
    return k


def tend_records():
    """Times to t_end (device time of advance_to / run_steps, CUDA events) of
    the other BASELINE configs on one GPU: cfg1 soliton to t = 20, cfg2 dam
    break to t = 48 at lambda 1e2 / 1e3 / 1e4, cfg4 bar (4 lambdas) 200 steps."""
    from paper_2510_07539_b200 import hsgn
    from paper_2510_07539_b200 import workloads as W
    out = {}
    w = W.cfg1()
    s = hsgn.solver_for(w)
    s.advance_to(1.0)                               # warm-up (graph capture)
    s = hsgn.solver_for(w)
    _, dev, wall = _timed(s.stream, lambda: s.advance_to(w.t_end))
    st = s.diagnostics()["steps"]
    st1 = _steps_to(w, w.t_end)
    out["cfg1_soliton_t20"] = {"seconds": dev, "wall_s": wall, "steps": st1, "steps_launched": st,
                               "us_per_step": dev / st1 * 1e6, "cells": w.n}
    # the same run member-resident (hsgn_run_resident: one launch, the member in
    # its 2-CTA cluster's shared memory, steps after t_end carried at no cost)
    s = hsgn.solver_for(w)
    s.run_resident(8, t_end=1.0)                   # warm-up (module load)
    s = hsgn.solver_for(w)
    dev, calls = 0.0, 0
    while True:
        dev += s.run_resident(1024, t_end=w.t_end) * 1e-3
        calls += 1
        if s.get_state(device=False)[1][0] >= w.t_end or calls >= 8:
            break
    st = st1
    out["cfg1_soliton_t20_resident"] = {"seconds": dev, "launches": calls, "steps": st,
                                        "us_per_step": dev / st * 1e6, "cells": w.n,
                                        "t_reached": float(s.get_state(device=False)[1][0])}
    for lam in (1e2, 1e3, 1e4):
        w = W.cfg2(lam)
        s = hsgn.solver_for(w)
        _, dev, wall = _timed(s.stream, lambda: s.advance_to(w.t_end))
        st = s.diagnostics()["steps"]          # launched: the last poll of advance_to may carry
        out[f"cfg2_dambreak_lam{lam:g}_t48"] = {"seconds": dev, "wall_s": wall, "steps_launched": st,
                                                "us_per_launched_step": dev / st * 1e6, "cells": w.n}
    # the three lambdas as one 3-member ensemble (per-member dt and t_end): one
    # launch sequence serves all three, to the slowest member's t_end
    w = W.cfg2_lambdas()
    s = hsgn.solver_for(w)
    _, dev, wall = _timed(s.stream, lambda: s.advance_to(w.t_end))
    tt = s.get_state(device=False)[1]
    out["cfg2_dambreak_3lambdas_one_ensemble_t48"] = {"seconds": dev, "wall_s": wall,
                                                      "steps_launched": s.diagnostics()["steps"],
                                                      "t_reached": [float(x) for x in tt], "cells": 3 * w.n}
    w = W.cfg4()
    s = hsgn.solver_for(w)
    s.run_steps(18)
    s.sync()
    _, dev, wall = _timed(s.stream, lambda: s.run_steps(200))
    out["cfg4_bar_4lambdas_200steps"] = {"seconds": dev, "wall_s": wall, "steps": 200,
                                         "cells": w.n * w.members, "value": 2.0 * w.n * w.members * 200 / dev}
    out["unit"] = "seconds of device time (value: cell-stage/s)"
    return out


if __name__ == "__main__":
    main()
