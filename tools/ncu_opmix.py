"""Dev tool: executed warp-instructions by SASS opcode (and by address range
buckets) from an ncu report's source page.  python tools/ncu_opmix.py REP [kernel-substring]"""
import csv, io, subprocess, sys, re, collections
rep = sys.argv[1]; ksub = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for line in out.splitlines():
    if line.startswith('"Kernel Name"'):
        cur = [line.split(",", 1)[1], []]; blocks.append(cur)
    elif cur is not None:
        cur[1].append(line)
seen = set()
for name, lines in blocks:
    if ksub not in name or name in seen:
        continue
    seen.add(name)
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr, rows = rows[0], rows[1:]
    ix = {h: i for i, h in enumerate(hdr)}
    ops = collections.Counter()
    tot = 0
    for r in rows:
        src = r[ix["Source"]].strip()
        n = int(r[ix["Instructions Executed"]] or 0)
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0].split(".")[0]
        ops[op] += n; tot += n
    print(f"== {name} total {tot}")
    for op, n in ops.most_common(40):
        print(f"  {op:14s} {n:10d} {100*n/tot:5.1f}%")
