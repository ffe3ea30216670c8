"""Golden outputs of the reference's OWN driver (tools/colosim.cpp, built
unchanged with the CLI11 subset shim into oracle/_ref/colosim by
oracle/Makefile) for tests/golden/cli/small.config:

    colosim run     --config small.config --out <tmp>/run      (report.csv, report.jsonl, tpt_cdf.csv)
    colosim run     ... --mode baseline / serving-only
    colosim compare --config small.config --out <tmp>/compare  (the figure datasets)

Small files are stored whole; large ones (TPT CDFs, reports with every
sample) as sha256 plus their first and last lines.  Run in the build
container:  make -C oracle && python tests/golden/make_cli_golden.py
"""
import hashlib
import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
CLI = os.path.join(HERE, "cli")
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
BIN = os.path.join(ROOT, "oracle", "_ref", "colosim")
WHOLE_LIMIT = 4096


def write_inputs():
    from oracle.oracle import sharegpt_histogram

    v, p = sharegpt_histogram()
    with open(os.path.join(CLI, "lengths.jsonl"), "w") as f:
        for a, b in zip(v, p):
            f.write(json.dumps({"tokens": int(a), "probability": float(b)}) + "\n")


def digest(path):
    data = open(path, "rb").read()
    lines = data.decode().splitlines()
    rec = {"sha256": hashlib.sha256(data).hexdigest(), "bytes": len(data), "lines": len(lines)}
    if len(data) <= WHOLE_LIMIT:
        rec["text"] = data.decode()
    else:
        rec["head"] = [ln[:200] for ln in lines[:20]]
        rec["tail"] = [ln[:200] for ln in lines[-20:]]
    return rec


def main():
    write_inputs()
    out = {}
    with tempfile.TemporaryDirectory() as tmp:
        jobs = {"run_colocated": ["run"], "run_baseline": ["run", "--mode", "baseline"],
                "run_serving": ["run", "--mode", "serving-only"], "compare": ["compare"],
                "profile": ["profile", "--model", "llama8b.model", "--gpu", "b80.gpu", "--cached-step", "250"]}
        for name, args in jobs.items():
            d = os.path.join(tmp, name)
            cfg = [] if name == "profile" else ["--config", "small.config"]
            subprocess.run([BIN, args[0]] + cfg + ["--out", d] + args[1:], cwd=CLI, check=True, capture_output=True)
            out[name] = {f: digest(os.path.join(d, f)) for f in sorted(os.listdir(d))}
    with open(os.path.join(CLI, "expected.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print({k: sorted(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
