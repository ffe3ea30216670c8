"""Shared by tests/test_experiment.py (CPU, restated engine) and
tests/test_gpu_experiment.py (GPU engine): run the harness's `run` and
`compare` on tests/golden/cli/small.config and hold every output file to the
reference CLI's own outputs (tests/golden/cli/expected.json, written by
tests/golden/make_cli_golden.py from oracle/_ref/colosim)."""
import hashlib
import json
import os

import numpy as np

from paper_2503_01066_b200 import experiment as ex

CLI = os.path.join(os.path.dirname(__file__), "golden", "cli")


def check_dir(d, expected):
    assert sorted(os.listdir(d)) == sorted(expected), (sorted(os.listdir(d)), sorted(expected))
    for name, rec in expected.items():
        data = open(os.path.join(d, name), "rb").read()
        if "text" in rec:
            assert data.decode() == rec["text"], (name, data.decode()[:400], rec["text"][:400])
        lines = data.decode().splitlines()
        if "head" in rec:
            got = [ln[:200] for ln in lines[:20]]
            for i, (a, b) in enumerate(zip(got, rec["head"])):
                assert a == b, (name, i, a, b)
            got = [ln[:200] for ln in lines[-20:]]
            for i, (a, b) in enumerate(zip(got, rec["tail"])):
                assert a == b, (name, "tail", i, a, b)
        assert len(lines) == rec["lines"], (name, len(lines), rec["lines"])
        assert hashlib.sha256(data).hexdigest() == rec["sha256"], name


def run_all(engine, tmp):
    exp = json.load(open(os.path.join(CLI, "expected.json")))
    cwd = os.getcwd()
    os.chdir(CLI)  # trace.length_dist = histogram:lengths.jsonl is relative, as in the reference
    try:
        for name, mode in (("run_colocated", ""), ("run_baseline", "baseline"), ("run_serving", "serving-only")):
            d = os.path.join(tmp, name)
            ex.cmd_run(engine, "small.config", d, mode_override=mode)
            check_dir(d, exp[name])
        d = os.path.join(tmp, "compare")
        ex.cmd_compare(engine, "small.config", d)
        check_dir(d, exp["compare"])
    finally:
        os.chdir(cwd)


def run_cli_profile(tmp):
    """`python -m paper_2503_01066_b200 profile` vs the reference CLI's map files."""
    from paper_2503_01066_b200.__main__ import main

    exp = json.load(open(os.path.join(CLI, "expected.json")))
    cwd = os.getcwd()
    os.chdir(CLI)
    try:
        d = os.path.join(tmp, "profile")
        assert main(["profile", "--model", "llama8b.model", "--gpu", "b80.gpu", "--cached-step", "250", "--out", d]) == 0
        check_dir(d, exp["profile"])
        # the exit-code contract (tools/colosim.cpp:23-24, 347-353)
        assert main(["run", "--config", "missing.config", "--out", os.path.join(tmp, "x")]) == 2
    finally:
        os.chdir(cwd)
