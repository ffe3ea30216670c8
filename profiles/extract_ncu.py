"""Summarise ncu captures into profiles/ncu_summary.json (+ a launch-share table).

    python profiles/extract_ncu.py gpurun_out/prof_fused.ncu-rep gpurun_out/prof_decide.ncu-rep \
        --launches gpurun_out/launches.csv --out profiles/ncu_summary.json

Per kernel: duration, DRAM bytes read/written per launch (`traffic` in
bench.py's roofline), DRAM throughput, issue-slot use, occupancy, registers
and the top warp-stall reasons.  The launch list (gpu__time_duration.sum of
every launch, cold-cache and serialised) gives each kernel's share of a step.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import re
import subprocess
from collections import defaultdict

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "warp_instructions",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
              "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1, "second": 1}


def short(name: str) -> str:
    m = re.search(r"(k_[a-z_]+)(?:<([^>]*)>)?", name)
    return (m.group(1) + (f"<{m.group(2)}>" if m.group(2) else "")) if m else name[:60]


def read_rep(path: str):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = defaultdict(list)
    for r in rows[2:]:
        d = {}
        for k, v in METRICS.items():
            if k in hdr:
                i = hdr.index(k)
                try:
                    x = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[v] = x * UNIT_SCALE.get(units[i], 1) if units[i] in UNIT_SCALE else x
        stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(r[i] or 0)
                  for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
        tot = sum(stalls.values()) or 1
        d["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:5]}
        out[short(r[hdr.index("Kernel Name")])].append(d)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reps", nargs="*")
    ap.add_argument("--launches")
    ap.add_argument("--out", default="profiles/ncu_summary.json")
    a = ap.parse_args()
    summary = {}
    for p in a.reps:
        for k, lst in read_rep(p).items():
            d = lst[-1]
            d["dram_bytes_per_launch"] = d.get("dram_read", 0) + d.get("dram_write", 0)
            d["source"] = p.split("/")[-1]
            d["captures"] = len(lst)
            summary[k] = d
            base = k.split("<")[0]
            summary.setdefault(base, d)
    if a.launches:
        rows = list(csv.reader(open(a.launches)))
        start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
        hdr = rows[start]
        tot = defaultdict(float)
        cnt = defaultdict(int)
        for r in rows[start + 1:]:
            if len(r) != len(hdr) or r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
                continue
            k = short(r[hdr.index("Kernel Name")])
            unit = r[hdr.index("Metric Unit")]
            v = float(r[hdr.index("Metric Value")].replace(",", "")) * UNIT_SCALE.get(unit, 1e-9)
            tot[k] += v
            cnt[k] += 1
        all_t = sum(tot.values()) or 1
        summary["launch_list"] = {k: {"launches": cnt[k], "total_s": tot[k], "share": tot[k] / all_t}
                                  for k in sorted(tot, key=lambda x: -tot[x])}
    with open(a.out, "w") as f:
        json.dump(summary, f, indent=1, sort_keys=True)
    print(json.dumps({k: {kk: v for kk, v in d.items() if kk in ("duration", "dram_bytes_per_launch", "dram_pct_of_peak",
                                                                      "issue_active_pct")} for k, d in summary.items()
                      if k != "launch_list"}, indent=1))


if __name__ == "__main__":
    main()
