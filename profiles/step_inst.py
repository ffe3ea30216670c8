"""One replay step's warp instructions from an ncu capture of exactly that
step (bench.py with COLO_PROFILE_STEP=1 under `ncu --profile-from-start off
--metrics smsp__inst_executed.sum,gpu__time_duration.sum --csv`):

    python profiles/step_inst.py gpurun_out/c4_step.csv --queries 1000000000 \
        --what "C4 per-rank step ..." --out profiles/r02_ncu_c4_step.json

bench.py's issue_roofline reads inst_per_query from the newest such file.
"""
from __future__ import annotations

import argparse
import csv
import json
import re
from collections import defaultdict

UNIT = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--queries", type=int, required=True)
    ap.add_argument("--what", default="")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[i]
    k_i, m_i, v_i, u_i = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    inst = defaultdict(float)
    dur = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[i + 1:]:
        if len(r) != len(hdr):
            continue
        m = re.search(r"(k_[a-z_0-9]+)", r[k_i])
        name = m.group(1) if m else r[k_i].split("(")[0][-40:]
        v = float(r[v_i].replace(",", ""))
        if r[m_i] == "smsp__inst_executed.sum":
            inst[name] += v
            cnt[name] += 1
        elif r[m_i] == "gpu__time_duration.sum":
            dur[name] += v * UNIT.get(r[u_i], 1e-9)
    total = sum(inst.values())
    out = {"what": a.what, "queries": a.queries, "inst_per_step": total, "inst_per_query": total / a.queries,
           "kernel_time_s": sum(dur.values()),
           "kernels": {k: {"launches": cnt[k], "warp_inst": inst[k], "time_s": dur[k]}
                       for k in sorted(inst, key=lambda x: -inst[x])}}
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "kernels"}, indent=1))


if __name__ == "__main__":
    main()
