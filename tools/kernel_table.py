"""Summary table of ncu --set full captures (dev tool; run here):
    python tools/kernel_table.py <cells per launch> rep1.ncu-rep [rep2 ...]"""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0] + "/tools")
from profile_summary import full  # noqa: E402

cells = float(sys.argv[1])
print("| kernel | us | DRAM B/cell | occupancy % | issue active % | fp64 pipe % | IPC/SM | regs | top stalls (warps per issue) |")
print("|---|---|---|---|---|---|---|---|---|")
for rep in sys.argv[2:]:
    for d in full(rep):
        b = (d.get("dram_read", 0) + d.get("dram_write", 0)) / cells
        print("| %s | %.1f | %.1f | %.1f | %.1f | %.1f | %.2f | %d | %s |" % (
            d["kernel"], d.get("duration", 0) / 1e3, b, d.get("achieved_occupancy_pct", 0),
            d.get("issue_active_pct", 0), d.get("fp64_pipe_pct", 0), d.get("ipc_per_sm", 0),
            d.get("registers", 0), ", ".join(f"{n} {v}" for n, v in d["top_stalls"])))
