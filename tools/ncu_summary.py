"""Summarise ncu captures and launch lists into profiles/ (run here, no GPU).

  python tools/ncu_summary.py REPORT.ncu-rep [...] --launches LAUNCHES.csv --out profiles/rN
writes <out>_kernels.json (per-launch key metrics, stall mix, DRAM bytes) and
<out>_launches.json (per-kernel share of one step from the launch list).
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import subprocess
from pathlib import Path

KEYS = {
    "duration_ms": "gpu__time_duration.sum",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "registers": "launch__registers_per_thread",
    "smem_dyn_bytes": "launch__shared_mem_per_block_dynamic",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "occ_limit_regs": "launch__occupancy_limit_registers",
    "occ_limit_smem": "launch__occupancy_limit_shared_mem",
    "warp_instructions": "smsp__inst_executed.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_pct_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
}


def _num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return s


def kernels(rep: Path):
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv", "--print-units",
                          "base"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head = rows[0]
    out = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        k = {"kernel": d["Kernel Name"].split("(")[0].replace("<unnamed>::", "")
             .replace("void ", "")}
        for name, m in KEYS.items():
            if m in d:
                k[name] = _num(d[m])
        if "duration_ms" in k and isinstance(k["duration_ms"], float):
            k["duration_ms"] /= 1e6  # base unit ns
        # FP64 flops of the launch: (DADD + DMUL + 2 DFMA) thread instructions,
        # from --set full's per-cycle rates x the elapsed SM cycles
        try:
            rate = sum(f * _num(d[f"smsp__sass_thread_inst_executed_op_{op}_pred_on"
                                  ".sum.per_cycle_elapsed"])
                       for op, f in (("dadd", 1), ("dmul", 1), ("dfma", 2)))
            k["fp64_flops"] = rate * _num(d["sm__cycles_elapsed.avg"])
        except (KeyError, TypeError):
            pass
        stalls = {key.replace("smsp__average_warps_issue_stalled_", "")
                  .replace("_per_issue_active.ratio", ""): _num(v)
                  for key, v in d.items()
                  if key.startswith("smsp__average_warps_issue_stalled_")
                  and key.endswith("_per_issue_active.ratio")}
        top = sorted(((v, s) for s, v in stalls.items() if isinstance(v, float)), reverse=True)
        k["top_stalls"] = {s: round(v, 2) for v, s in top[:6]}
        out.append(k)
    return out


def launches(path: Path):
    rows = list(csv.reader(open(path)))
    head, seq = None, []
    for r in rows:
        if "Kernel Name" in r:
            head = r
            continue
        if head is None or len(r) != len(head):
            continue
        d = dict(zip(head, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
        seq.append((name, _num(d["Metric Value"]) / 1e6))
    starts = [i for i, (n, _) in enumerate(seq) if n.startswith("k_stage1")]
    # one step = from the last stage-1 launch to the end (the last timed step
    # of a `bench.py --no-e2e` run; nothing launches after the loop)
    step = seq[starts[-1]:] if starts else seq
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, t in step:
        agg[n][0] += 1
        agg[n][1] += t
    tot = sum(v[1] for v in agg.values())
    return {"step_kernel_ms": round(tot, 3),
            "kernels": [{"kernel": n, "launches": c, "ms": round(t, 4),
                         "share": round(t / tot, 4)}
                        for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="*")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    if a.reports:
        ks = []
        for r in a.reports:
            ks.extend(kernels(Path(r)))
        Path(a.out + "_kernels.json").write_text(json.dumps(ks, indent=1))
    if a.launches:
        Path(a.out + "_launches.json").write_text(json.dumps(launches(Path(a.launches)),
                                                             indent=1))


if __name__ == "__main__":
    main()
