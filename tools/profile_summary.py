"""Summarise ncu output into profiles/ (dev tool; run here, on the CPU box).

    python tools/profile_summary.py --round 1 --cells-full 16777216 --cells-prof 2097152 \
        gpurun_out/launches.csv gpurun_out/prof.ncu-rep

Writes profiles/r<NN>_launches.csv (copy of the launch list),
profiles/r<NN>_ncu_summary.md (human summary) and profiles/ncu_summary.json
(machine summary read by bench.py for roofline.traffic).
"""
import argparse
import collections
import csv
import io
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name):
    if "cl_stage_kernel" in name or "cl_multi_kernel" in name:
        return name.split("(")[0].replace("void ", "").replace("hsgn::", "").replace("(bool)", "")
    if "stage_kernel" in name:
        t = name.split("<")[1].split(">")[0].replace("(bool)", "")
        f = [x.strip() for x in t.split(",")]
        return "stage_kernel<S2=%s,FINAL=%s,BATHY=%s>" % tuple(f[:3])
    return name.split("(")[0]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    per = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[1:]:
        k = short(r[ix["Kernel Name"]])
        per[k][r[ix["Metric Name"]]].append(float(r[ix["Metric Value"]].replace(",", "")))
    out = {}
    for k, d in per.items():
        t = d.get("gpu__time_duration.sum", [])
        out[k] = {"launches": len(t),
                  "mean_us": (sum(t) / len(t) / 1e3) if t else None,
                  "total_us": sum(t) / 1e3 if t else None,
                  "dram_read_per_launch": (sum(d["dram__bytes_read.sum"]) / len(t)) if t and d.get("dram__bytes_read.sum") else None,
                  "dram_write_per_launch": (sum(d["dram__bytes_write.sum"]) / len(t)) if t and d.get("dram__bytes_write.sum") else None}
    return out


def full(rep):
    """per-launch metrics of an ncu report (or of its `--page raw --csv` export)"""
    if rep.endswith(".csv"):
        txt = open(rep).read()
        txt = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    want = {
        "gpu__time_duration.sum": "duration",
        "dram__bytes_read.sum": "dram_read",
        "dram__bytes_write.sum": "dram_write",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
        "sm__inst_executed.avg.per_cycle_active": "ipc_per_sm",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
        "launch__registers_per_thread": "registers",
        "launch__shared_mem_per_block_dynamic": "dyn_smem",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
        "smsp__inst_executed.sum": "warp_inst",
        "launch__grid_size": "grid",
        "launch__occupancy_limit_registers": "occ_limit_regs",
        "launch__occupancy_limit_shared_mem": "occ_limit_smem",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed": "dadd_per_cycle",
        "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed": "dmul_per_cycle",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed": "dfma_per_cycle",
        "sm__cycles_elapsed.avg.per_second": "clock_hz",
    }
    out = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for k, v in want.items():
            if k in hdr:
                i = hdr.index(k)
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                         "nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
                         "Ghz": 1e9, "Mhz": 1e6, "hz": 1}.get(units[i], 1)
                try:
                    d[v] = float(r[i].replace(",", "")) * scale      # bytes, ns
                except ValueError:
                    d[v] = r[i]
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        d["top_stalls"] = [(n, round(v, 3)) for v, n in sorted(st, reverse=True)[:6]]
        out.append(d)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", type=int, required=True)
    ap.add_argument("--cells-full", type=float, required=True, help="cells per launch in the launch list run")
    ap.add_argument("--cells-prof", type=float, required=True, help="cells per launch in the --set full run")
    ap.add_argument("--cfg5-launches", help="launch list of `bench.py --config cfg5` (2^28 cells)")
    ap.add_argument("--cfg5-rep", help="--set full capture of the cfg5 stage kernels")
    ap.add_argument("--cfg5-cells-full", type=float, default=float(1 << 28))
    ap.add_argument("--cfg5-cells-prof", type=float, default=float(1 << 24))
    ap.add_argument("launches")
    ap.add_argument("rep")
    a = ap.parse_args()
    tag = "r%02d" % a.round
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    shutil.copy(a.launches, os.path.join(prof, f"{tag}_launches.csv"))
    L = launches(a.launches)
    F = full(a.rep)
    tot = sum(v["total_us"] or 0 for v in L.values())
    md = [f"# ncu summary, round {a.round}", "",
          "Launch list: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
          "--clock-control none` over `python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu` "
          "(cfg3, 4096 x 4096 cells; cold-cache serialised launches: compare shares).", "",
          "| kernel | launches | mean us | share of time | DRAM B/cell read | DRAM B/cell write |",
          "|---|---|---|---|---|---|"]
    js = {"round": a.round, "summary": f"profiles/{tag}_ncu_summary.md", "launch_list": {}, "full": []}
    for k, v in sorted(L.items(), key=lambda kv: -(kv[1]["total_us"] or 0)):
        rd = (v["dram_read_per_launch"] or 0) / a.cells_full
        wr = (v["dram_write_per_launch"] or 0) / a.cells_full
        md.append(f"| {k} | {v['launches']} | {v['mean_us']:.1f} | {100 * (v['total_us'] or 0) / tot:.1f}% | {rd:.1f} | {wr:.1f} |")
        js["launch_list"][k] = dict(v, dram_read_per_cell=rd, dram_write_per_cell=wr)
    md += ["", "Full set (`ncu --set full --import-source on`, 512 members x 4096 cells, one launch each):", "",
           "| kernel | us | DRAM B/cell | occupancy % | issue active % | fp64 pipe % | IPC/SM | regs | top stalls (warps per issue) |",
           "|---|---|---|---|---|---|---|---|---|"]
    for d in F:
        b = (d.get("dram_read", 0) + d.get("dram_write", 0)) / a.cells_prof
        md.append("| %s | %.1f | %.1f | %.1f | %.1f | %.1f | %.2f | %d | %s |" % (
            d["kernel"], d.get("duration", 0) / 1e3, b, d.get("achieved_occupancy_pct", 0),
            d.get("issue_active_pct", 0), d.get("fp64_pipe_pct", 0), d.get("ipc_per_sm", 0),
            d.get("registers", 0), ", ".join(f"{n} {v}" for n, v in d["top_stalls"])))
        js["full"].append(dict(d, dram_bytes_per_cell=b))
    s2 = [v for k, v in js["launch_list"].items() if "S2=1" in k]
    if s2:
        js["stage2_dram_bytes_per_cell"] = s2[0]["dram_read_per_cell"] + s2[0]["dram_write_per_cell"]
    s1 = [v for k, v in js["launch_list"].items() if "S2=0" in k and "FINAL=0" in k]
    if s1:
        js["stage1_dram_bytes_per_cell"] = s1[0]["dram_read_per_cell"] + s1[0]["dram_write_per_cell"]
    # fp64 arithmetic rate against the measured DFMA peak (profiles/rNN_dfma_peak.json)
    pks = sorted(f for f in os.listdir(prof) if f.endswith("_dfma_peak.json") and f <= f"{tag}_dfma_peak.json")
    pk = os.path.join(prof, pks[-1]) if pks else ""
    if pk:
        peak = json.load(open(pk))
        ptf = peak["fp64_tflops"]
        md += ["", f"fp64 arithmetic (DADD + DMUL + 2 DFMA per cycle, ncu) against the measured DFMA peak "
                   f"{ptf:.1f} TFLOP/s (`tools/dfma_peak.cu`, {peak['dfma_per_clk_per_sm_at_max_clock']:.1f} "
                   f"DFMA/clk/SM, profiles/{os.path.basename(pk)}):", "", "| kernel | fp64 TFLOP/s | of peak | fp64 pipe active % |", "|---|---|---|---|"]
        js["fp64_peak_tflops"] = ptf
        for d in js["full"]:
            try:
                clk = float(d.get("clock_hz", 0)) or 1.965e9
                tf = (d["dadd_per_cycle"] + d["dmul_per_cycle"] + 2 * d["dfma_per_cycle"]) * clk / 1e12
            except (KeyError, TypeError):
                continue
            d["fp64_tflops"] = tf
            md.append(f"| {d['kernel']} | {tf:.2f} | {tf / ptf:.2f} | {d.get('fp64_pipe_pct', 0):.1f} |")
    if a.cfg5_launches:
        # cfg5 (one domain with bathymetry): the BATHY instantiations, 104 / 72 B/cell models
        rows = [r for r in csv.reader(open(a.cfg5_launches)) if len(r) > 10]
        keep = [rows[0]] + [r for r in rows[1:] if "hsgn::" in ",".join(r)]
        with open(os.path.join(prof, f"{tag}_cfg5_launches.csv"), "w", newline="") as f:
            csv.writer(f, quoting=csv.QUOTE_ALL).writerows(keep)
        L5 = {k: v for k, v in launches(os.path.join(prof, f"{tag}_cfg5_launches.csv")).items()}
        tot5 = sum(v["total_us"] or 0 for v in L5.values())
        md += ["", "cfg5 launch list (same ncu metrics over `python bench.py --config cfg5 --steps 4 --warmup 3 --no-e2e "
                   "--no-cpu --no-sub`, 2^28 cells with bathymetry; the library's kernels only, torch's input "
                   "generation dropped; algorithmic bytes: stage 2 104 B/cell, stage 1 72 B/cell):", "",
               "| kernel | launches | mean us | share of time | DRAM B/cell read | DRAM B/cell write |", "|---|---|---|---|---|---|"]
        js["cfg5"] = {"launch_list": {}, "full": []}
        for k, v in sorted(L5.items(), key=lambda kv: -(kv[1]["total_us"] or 0)):
            rd = (v["dram_read_per_launch"] or 0) / a.cfg5_cells_full
            wr = (v["dram_write_per_launch"] or 0) / a.cfg5_cells_full
            md.append(f"| {k} | {v['launches']} | {v['mean_us']:.1f} | {100 * (v['total_us'] or 0) / tot5:.1f}% | {rd:.1f} | {wr:.1f} |")
            js["cfg5"]["launch_list"][k] = dict(v, dram_read_per_cell=rd, dram_write_per_cell=wr)
            if "S2=1" in k and "BATHY=1" in k:
                js["cfg5"]["stage2_dram_bytes_per_cell"] = rd + wr
            if "S2=0" in k and "BATHY=1" in k:
                js["cfg5"]["stage1_dram_bytes_per_cell"] = rd + wr
        if a.cfg5_rep:
            md += ["", "cfg5 full set (`ncu --set full --import-source on`, one 2^24-cell domain of the cfg5 recipe):", "",
                   "| kernel | us | DRAM B/cell | occupancy % | issue active % | fp64 pipe % | IPC/SM | regs | top stalls (warps per issue) |",
                   "|---|---|---|---|---|---|---|---|---|"]
            for d in full(a.cfg5_rep):
                b = (d.get("dram_read", 0) + d.get("dram_write", 0)) / a.cfg5_cells_prof
                md.append("| %s | %.1f | %.1f | %.1f | %.1f | %.1f | %.2f | %d | %s |" % (
                    d["kernel"], d.get("duration", 0) / 1e3, b, d.get("achieved_occupancy_pct", 0),
                    d.get("issue_active_pct", 0), d.get("fp64_pipe_pct", 0), d.get("ipc_per_sm", 0),
                    d.get("registers", 0), ", ".join(f"{n} {v}" for n, v in d["top_stalls"])))
                js["cfg5"]["full"].append(dict(d, dram_bytes_per_cell=b))
    open(os.path.join(prof, f"{tag}_ncu_summary.md"), "w").write("\n".join(md) + "\n")
    json.dump(js, open(os.path.join(prof, "ncu_summary.json"), "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
