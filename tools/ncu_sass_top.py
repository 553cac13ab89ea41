"""Dev tool: top SASS instructions by warp-stall samples from an ncu report
(ncu -i REP --page source --csv --print-source sass), per kernel, with the
dominant stall reasons, plus the samples of the instructions around each hot
spot.  Usage: python tools/ncu_sass_top.py REP [kernel-substring] [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ksub = sys.argv[2] if len(sys.argv) > 2 else ""
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for line in out.splitlines():
    if line.startswith('"Kernel Name"'):
        cur = [line.split(",", 1)[1], []]
        blocks.append(cur)
    elif cur is not None:
        cur[1].append(line)
for name, lines in blocks:
    if ksub not in name:
        continue
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr, rows = rows[0], rows[1:]
    ix = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(int(r[ix["# Samples"]] or 0) for r in rows)
    print(f"== {name}  samples {tot}, instructions {len(rows)}")
    agg = {}
    for r in rows:
        for h in stalls:
            agg[h] = agg.get(h, 0) + int(r[ix[h]] or 0)
    print("   " + ", ".join(f"{k[6:]} {v}" for k, v in sorted(agg.items(), key=lambda x: -x[1]) if v))
    order = sorted(range(len(rows)), key=lambda i: -int(rows[i][ix["# Samples"]] or 0))[:N]
    for i in sorted(order):
        r = rows[i]
        s = int(r[ix["# Samples"]] or 0)
        top = sorted(((int(r[ix[h]] or 0), h[6:]) for h in stalls), reverse=True)[:3]
        print(f"{i:6d} {s:5d} {r[ix['Source']].strip()[:60]:60s} " + " ".join(f"{h}:{v}" for v, h in top if v))
