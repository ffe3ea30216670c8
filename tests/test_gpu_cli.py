"""The reference's own driver, tools/colosim.cpp UNCHANGED, running on the
GPU: `make cli` compiles it against the include overlay
(paper_2503_01066_b200/cpp/overlay -- Simulation, run_simulation and the map
builders on sm_100a) and links it to libcolo_b200.so.  Every output of
`run` (three modes), `compare` and `profile` on tests/golden/cli/small.config
must be byte-identical to the reference CLI's (tests/golden/cli/expected.json,
written from oracle/_ref/colosim by tests/golden/make_cli_golden.py)."""
import json
import os
import subprocess

import pytest

from experiment_check import CLI, check_dir

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2503_01066_b200", "bin", "colosim")
JOBS = {"run_colocated": ["run"], "run_baseline": ["run", "--mode", "baseline"],
        "run_serving": ["run", "--mode", "serving-only"], "compare": ["compare"],
        "profile": ["profile", "--model", "llama8b.model", "--gpu", "b80.gpu", "--cached-step", "250"]}


def test_unchanged_driver_is_gpu_backed():
    """CPU check: the binary links libcolo_b200.so and carries none of the
    reference's own Simulation / run_simulation / map builders (the overlay
    renames them; nothing may call them)."""
    if not os.path.exists(BIN):
        pytest.skip("paper_2503_01066_b200/bin/colosim not built (needs /root/reference at build time)")
    syms = subprocess.run(["nm", "-C", BIN], capture_output=True, text=True, check=True).stdout
    assert "cpu_reference" not in syms
    assert "libcolo_b200.so" in subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout


@pytest.mark.gpu
@pytest.mark.parametrize("job", sorted(JOBS))
def test_unchanged_driver_on_gpu_matches_reference_cli(tmp_path, job):
    assert os.path.exists(BIN), "paper_2503_01066_b200/bin/colosim missing (make cli)"
    exp = json.load(open(os.path.join(CLI, "expected.json")))
    d = str(tmp_path / job)
    args = JOBS[job]
    cfg = [] if job == "profile" else ["--config", "small.config"]
    cp = subprocess.run([BIN, args[0]] + cfg + ["--out", d] + args[1:], cwd=CLI, capture_output=True, text=True)
    assert cp.returncode == 0, cp.stderr
    check_dir(d, exp[job])


@pytest.mark.gpu
def test_unchanged_driver_exit_codes(tmp_path):
    """tools/colosim.cpp:23-24, 347-353: validation errors exit 2."""
    cp = subprocess.run([BIN, "run", "--config", "missing.config", "--out", str(tmp_path / "x")], cwd=CLI,
                        capture_output=True, text=True)
    assert cp.returncode == 2
    bad = tmp_path / "bad.config"
    bad.write_text(open(os.path.join(CLI, "small.config")).read().replace("histogram:lengths.jsonl",
                                                                          "histogram:" + os.path.join(CLI, "lengths.jsonl"))
                   .replace("map.cached_step = 500", "map.cached_step = 300"))  # 8000 % 300: validate_grid throws
    cp = subprocess.run([BIN, "run", "--config", str(bad), "--out", str(tmp_path / "y")], cwd=CLI,
                        capture_output=True, text=True)
    assert cp.returncode == 2, (cp.returncode, cp.stderr)
