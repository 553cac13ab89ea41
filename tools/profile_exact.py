"""Summarise the round's ncu captures of the exact-solve kernels (cluster stage
kernels, tile-level SPIKE, member-resident multi-step) into
profiles/r<NN>_exact_kernels.md, with the static SASS evidence of the cluster /
DSMEM / mbarrier instructions (cuobjdump of the built library).  Dev tool.

    python tools/profile_exact.py --round 2 --cells-prof 2097152 \
        gpurun_out/r02_cluster.ncu-rep gpurun_out/r02_spike_raw.csv gpurun_out/r02_resident.ncu-rep
"""
import argparse
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from profile_summary import full  # noqa: E402

LIB = os.path.join(ROOT, "paper_2510_07539_b200", "lib", "libhsgn.so")
CLUSTER_OPS = ("UBLKCP", "LDGSTS", "UCGABAR_ARV", "UCGABAR_WAIT", "SYNCS", "STAS", "MEMBAR", "FENCE", "REDUX",
               "CREDUX", "MUFU")


def sass_ops(kernel_re):
    """static opcode counts of the kernels whose mangled name matches kernel_re"""
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    res, cur = collections.defaultdict(collections.Counter), None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1) if re.search(kernel_re, m.group(1)) else None
            continue
        if cur is None:
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", line)
        if m:
            res[cur][m.group(2) + (m.group(3) or "")] += 1
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", type=int, required=True)
    ap.add_argument("--cells-prof", type=float, required=True)
    ap.add_argument("reps", nargs="+")
    a = ap.parse_args()
    tag = "r%02d" % a.round
    md = [f"# Exact-solve kernels, ncu, round {a.round}", "",
          "`ncu --set full --clock-control none` on 512 cfg3 members x 4096 cells (2^21 cells per launch); "
          "sources: " + ", ".join(f"`{os.path.basename(r)}`" for r in a.reps) + ".  Captured by "
          "`tools/gpu_session_b.sh`; timings under ncu are serialised and not bench numbers.", "",
          "| kernel | us | DRAM B/cell | occupancy % | issue active % | fp64 pipe % | IPC/SM | regs | top stalls (warps per issue) |",
          "|---|---|---|---|---|---|---|---|---|"]
    for rep in a.reps:
        for d in full(rep):
            b = (d.get("dram_read", 0) + d.get("dram_write", 0)) / a.cells_prof
            md.append("| %s | %.1f | %.1f | %.1f | %.1f | %.1f | %.2f | %d | %s |" % (
                d["kernel"], d.get("duration", 0) / 1e3, b, d.get("achieved_occupancy_pct", 0),
                d.get("issue_active_pct", 0), d.get("fp64_pipe_pct", 0), d.get("ipc_per_sm", 0),
                d.get("registers", 0), ", ".join(f"{n} {v}" for n, v in d["top_stalls"])))
    md += ["", "Static SASS (cuobjdump -sass of the built library): TMA bulk copies (UBLKCP), cp.async "
               "(LDGSTS), cluster barrier (UCGABAR), mbarrier (SYNCS), remote shared stores with transaction "
               "completion (STAS = st.async ... mbarrier::complete_tx), warp reductions (REDUX / CREDUX), "
               "reciprocal / rsqrt seeds (MUFU.RCP64H / RSQ64H).  One row per kernel instantiation without "
               "bathymetry; the overlapped-tile stage kernels (default path) for comparison.", "",
           "| kernel | instructions | " + " | ".join(CLUSTER_OPS) + " |", "|---|---|" + "---|" * len(CLUSTER_OPS)]
    ops = sass_ops(r"stage_kernelILb[01]ELb[01]ELb0ELb0ELb0ELb0E|cl_stage_kernelILb[01]ELb[01]ELb0E|"
                   r"cl_multi_kernelILb0E|sep_solve|sep_coef|filter_fix|slab_iface")
    for k in sorted(ops):
        c = ops[k]
        tot = sum(c.values())
        row = [sum(v for op, v in c.items() if op.split(".")[0] == want) for want in CLUSTER_OPS]
        md.append(f"| `{k}` | {tot} | " + " | ".join(str(x) for x in row) + " |")
    path = os.path.join(ROOT, "profiles", f"{tag}_exact_kernels.md")
    open(path, "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
