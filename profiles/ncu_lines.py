"""Per-source-line totals of an ncu capture (warp instructions executed and
warp-stall samples), from the interleaved CUDA+SASS source page.

    python profiles/ncu_lines.py gpurun_out/c4full.ncu-rep [--top 40] [--kernel k_replay_full]

Needs a capture taken with --import-source on from a -lineinfo build.
"""
from __future__ import annotations

import argparse
import csv
import io
import subprocess
from collections import defaultdict


def line_totals(rep: str, kernel: str | None = None):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kernel:  # the import honours the kernel filter: only that kernel's launches
        cmd += ["--kernel-name", f"regex:{kernel}"]
    raw = subprocess.run(cmd, capture_output=True, text=True).stdout
    inst = defaultdict(int)
    samp = defaultdict(int)
    text = {}
    path, func, cur, hdr = None, None, None, None
    for r in csv.reader(io.StringIO(raw)):
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            func = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or (kernel and func and kernel not in func):
            continue
        if r[0]:
            cur = (path, int(r[0]))
            text[cur] = r[1].strip()
            continue
        if cur is None or len(r) < len(hdr) or r[2] == "...":
            continue
        try:
            inst[cur] += int(r[hdr.index("Instructions Executed")] or 0)
            samp[cur] += int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
    return inst, samp, text


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--kernel")
    ap.add_argument("--by", choices=["inst", "samples"], default="inst")
    a = ap.parse_args()
    inst, samp, text = line_totals(a.rep, a.kernel)
    ti, ts = sum(inst.values()) or 1, sum(samp.values()) or 1
    print(f"total warp instructions {ti:,}  stall samples {ts:,}")
    key = inst if a.by == "inst" else samp
    for k in sorted(key, key=lambda x: -key[x])[: a.top]:
        print(f"{100 * inst[k] / ti:5.1f}% inst {100 * samp[k] / ts:5.1f}% smp  {k[0]}:{k[1]:<5} {text.get(k, '')[:90]}")


if __name__ == "__main__":
    main()
