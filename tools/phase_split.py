"""Group tools/sass_lines.py output (per source line) into phases delimited by
marker substrings of the source file: python tools/phase_split.py lines.txt
src.cu n_units 'name=marker' ..."""
import sys

lines_txt, src, units = sys.argv[1], sys.argv[2], float(sys.argv[3])
marks = []
text = open(src).read().splitlines()
for spec in sys.argv[4:]:
    name, pat = spec.split("=", 1)
    ln = next(i + 1 for i, l in enumerate(text) if pat in l)
    marks.append((ln, name))
marks.sort()
fname = src.split("/")[-1]
agg, tot = {}, 0
for l in open(lines_txt).read().splitlines()[2:]:
    p = l.split()
    f, _, ln = p[0].rpartition(":")
    n = int(p[1].replace(",", ""))
    tot += n
    if f == fname:
        ln = int(ln)
        k = "pre"
        for m, name in marks:
            if ln >= m:
                k = name
    else:
        k = f
    agg[k] = agg.get(k, 0) + n
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{k:28s} {v / units:9.0f}/unit {100 * v / tot:5.1f}%")
