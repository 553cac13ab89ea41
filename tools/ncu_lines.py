"""Dev tool: warp instructions executed and stall samples per CUDA source line
(and per SASS opcode) of one kernel in an ncu report, from
`ncu -i REP --page source --csv --print-source cuda,sass`.
Usage: python tools/ncu_lines.py REP kernel-substring [N]"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep, ksub = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
lines = defaultdict(lambda: [0, 0, ""])
ops = defaultdict(lambda: [0, 0])
fname, func, hdr = None, None, None
tot_i = tot_s = 0
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Function Name":
        func = row[1]
        continue
    if row[0] == "Line No":
        hdr = {h: i for i, h in enumerate(row)}
        hdr["_sass"] = 3                      # columns: line, cuda source, address, sass source, ...
        continue
    if func is None or ksub not in func or hdr is None:
        continue
    try:
        ie = int(row[hdr["Instructions Executed"]] or 0)
        sm = int(row[hdr["# Samples"]] or 0)
    except (ValueError, IndexError):
        continue
    key = (fname, int(row[0]) if row[0].isdigit() else -1)
    if row[2] == "-":                         # a CUDA line's aggregate row
        lines[key][0] += ie
        lines[key][1] += sm
        lines[key][2] = row[1].strip()[:70]
        continue
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", row[3])
    op = m.group(2) if m else "?"
    ops[op][0] += ie
    ops[op][1] += sm
    tot_i += ie
    tot_s += sm
print(f"warp instructions {tot_i}, samples {tot_s}")
print("by opcode:", ", ".join(f"{k} {v[0] / tot_i:.3f}" for k, v in sorted(ops.items(), key=lambda x: -x[1][0])[:25]))
print(f"{'file:line':28s} {'instr%':>7s} {'samp%':>6s}  source")
for k, v in sorted(lines.items(), key=lambda x: -x[1][0])[:N]:
    print(f"{k[0] + ':' + str(k[1]):28s} {100 * v[0] / tot_i:7.2f} {100 * v[1] / max(tot_s, 1):6.2f}  {v[2]}")
print("per file:", {f: round(100 * sum(v[0] for k, v in lines.items() if k[0] == f) / tot_i, 1)
                    for f in sorted({k[0] for k in lines})})
