"""Attribute ncu SASS-level stall samples to CUDA source lines (dev tool).

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep paper_2510_07539_b200/lib/libhsgn.so

Uses nvdisasm line info (-lineinfo builds) to map each SASS offset to a line of
hsgn_kernels.cuh, then sums 'Warp Stall Sampling (All Samples)' per line."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def sass_lines(so):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True, check=True)
    cub = [os.path.join(d, f) for f in os.listdir(d) if f.endswith(".cubin")][0]
    out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    funcs = {}
    cur = None
    line = None
    for ln in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            cur = m.group(1)
            funcs[cur] = {}
            continue
        m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', ln)
        if m:
            line = (m.group(1), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur is not None and line is not None:
            funcs[cur][int(m.group(1), 16)] = line
    return funcs


def main(rep, so):
    funcs = sass_lines(so)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks = txt.split('"Kernel Name"')[1:]
    for b in blocks:
        name = b.split("\n", 1)[0]
        rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
        hdr = rows[0]
        ia, iss, iex = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        base = int(rows[1][ia], 16)
        # pick the mangled function whose size matches
        n = len(rows) - 1
        kb = re.search(r"hsgn::(\w+)<", name)
        kb = kb.group(1) if kb else "stage_kernel"
        cand = [f for f, m in funcs.items() if abs(len(m) - n) <= 2 and kb in f]
        key = None
        tag = re.findall(r"\(bool\)(\d)", name.split(">(")[0])
        if tag:
            t = kb + "I" + "".join("Lb%sE" % x for x in tag) + "E"
            for f in funcs:
                if t in f:
                    key = f
        if key is None and cand:
            key = cand[0]
        agg = collections.Counter()
        inst = collections.Counter()
        ops = collections.Counter()
        isrc = hdr.index("Source")
        tot = 0
        for r in rows[1:]:
            off = int(r[ia], 16) - base
            li = funcs.get(key, {}).get(off, ("?", 0))
            s = int(r[iss] or 0)
            agg[li] += s
            inst[li] += int(r[iex] or 0)
            op = r[isrc].split()
            op = [t for t in op if not t.startswith("@")]
            if op:
                ops[op[0].split(".")[0]] += int(r[iex] or 0)
            tot += s
        print("=== %s  (%s) total samples %d" % (name[:60], key, tot))
        for li, s in agg.most_common(int(os.environ.get("TOPN", "40"))):
            print("%6.2f%%  %-22s line %4d   inst %d" % (100.0 * s / max(tot, 1), li[0], li[1], inst[li]))
        cells = float(os.environ.get("CELLS", "0"))
        if cells:
            print("--- dynamic SASS opcodes, thread-inst per cell (x32 warp)")
            for op, c in ops.most_common(30):
                print("   %-10s %7.1f" % (op, 32.0 * c / cells))
            print("   total      %7.1f" % (32.0 * sum(ops.values()) / cells))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
