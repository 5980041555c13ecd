"""Join an ncu `--page source --csv` SASS dump with `nvdisasm -g` line info:
executed warp instructions (and stall samples) per CUDA source line.

  python tools/sass_lines.py <source.csv[.gz]> <kernel substring> <cubin> [top]
"""
import csv
import gzip
import io
import re
import subprocess
import sys
from collections import defaultdict


def sections(path):
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt") as f:
        txt = f.read()
    out, cur, name = {}, [], None
    for line in txt.splitlines():
        if line.startswith('"Kernel Name"'):
            if name:
                out[name] = cur
            name, cur = line.split(",", 1)[1].strip('",'), []
        elif name:
            cur.append(line)
    if name:
        out[name] = cur
    return out


def main():
    path, kern, cubin = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    secs = sections(path)
    name = next(k for k in secs if kern in k)
    kern = name
    rows = list(csv.reader(io.StringIO("\n".join(secs[name]))))
    hdr, rows = rows[0], rows[1:]
    ia, ie, iss = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index(
        "Warp Stall Sampling (All Samples)")
    base = int(rows[0][ia], 16)
    per_off = {int(r[ia], 16) - base: (int(r[ie] or 0), int(r[iss] or 0), r[1]) for r in rows}
    # nvdisasm line map for the matching function
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    mangled = re.search(r"k_project|k_deflate|k_stage1", kern)
    funcs = re.split(r"//-+ \.text\.", dis)
    want = None
    short = re.search(r"(k_\w+)", kern).group(1)
    tmpl = ("ILb1E" if re.search(r"<\(bool\)1>|<1>|<true>", kern) else
            "ILb0E" if re.search(r"<\(bool\)0>|<0>|<false>", kern) else "")
    mi = re.search(r"\(int\)(\d+)>", kern)
    if mi:
        tmpl += f"Li{mi.group(1)}E"
    for fblk in funcs:
        head = fblk.split("\n", 1)[0]
        if short in head and (not tmpl or tmpl in head):
            want = fblk
            break
    line_of, cur = {}, None
    for ln in want.splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m:
            line_of[int(m.group(1), 16)] = cur
    agg = defaultdict(lambda: [0, 0])
    tot_i = tot_s = 0
    for off, (ins, st, _) in per_off.items():
        key = line_of.get(off, "?")
        agg[key][0] += ins
        agg[key][1] += st
        tot_i += ins
        tot_s += st
    print(f"{name[:90]}\ntotal warp inst {tot_i:,}  stall samples {tot_s:,}")
    for k, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{k:28s} {i:>14,} {100*i/tot_i:6.2f}%  stall {100*s/max(tot_s,1):6.2f}%")


if __name__ == "__main__":
    main()
