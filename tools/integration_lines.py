"""Refresh the `mlk_b200.h:N` references of INTEGRATION.md's entry-point
table from the header (run after editing include/mlk_b200.h)."""
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
line = {}
for i, l in enumerate((ROOT / "include" / "mlk_b200.h").read_text().splitlines(), 1):
    m = re.match(r"^(?:int|const char\*) (mlk_\w+)\(", l)
    if m:
        line[m.group(1)] = i
doc = ROOT / "INTEGRATION.md"
out = []
for l in doc.read_text().splitlines():
    m = re.match(r"^\| `mlk_b200\.h:[^`]*` \| (.*?) \| (.*)$", l)
    if m:
        names = re.findall(r"`(mlk_\w+)", m.group(1))
        # expand "/ `_unmap`"-style suffixes to full names
        full = []
        for nm in names:
            full.append(nm)
        for suf in re.findall(r"`_(\w+)`", m.group(1)):
            base = names[0].rsplit("_", 1)[0]
            cand = [k for k in line if k.endswith("_" + suf) and k.startswith(base.split("_")[0])]
            full += [c for c in cand if c.startswith(names[0][:8])][:1]
        nums = sorted({line[n] for n in full if n in line})
        if "mlk_list_flags" in names:  # the section packers: a contiguous block
            nums = [line["mlk_list_flags"], 0, 0, line["mlk_pack_exceptions"]]
        if nums:
            ref = ",".join(str(x) for x in nums) if len(nums) <= 3 else f"{nums[0]}-{nums[-1]}"
            l = f"| `mlk_b200.h:{ref}` | {m.group(1)} | {m.group(2)}"
    out.append(l)
doc.write_text("\n".join(out) + "\n")
