"""The experiment harness on the GPU engine (every Simulation::run is a
device of a colo_replay_colocated fleet; TPT samples sorted on the device):
`run` in all three modes and `compare` produce files byte-identical to the
reference CLI's (tests/golden/cli/expected.json)."""
import pytest

from paper_2503_01066_b200 import colosim as cs
from paper_2503_01066_b200 import experiment as ex

from experiment_check import run_all, run_cli_profile

pytestmark = pytest.mark.gpu


def test_harness_outputs_match_reference_cli_gpu(tmp_path):
    run_all(ex.GpuEngine(cs.Context(0)), str(tmp_path))


def test_cli_profile_matches_reference_cli(tmp_path):
    run_cli_profile(str(tmp_path))


def test_cli_run_long_trace_segmented(tmp_path):
    """`run` on a trace long enough for the colocated replay to split the
    device into parallel segments (qps 0.3 for 20000 s, about 6000 queries):
    report.csv / report.jsonl / tpt_cdf.csv byte-identical to the reference
    CLI's (oracle/_ref/colosim, run live on the same config), in all three
    modes."""
    import os
    import subprocess

    from experiment_check import CLI

    ref_bin = os.path.join(os.path.dirname(CLI), "..", "..", "oracle", "_ref", "colosim")
    if not os.path.exists(ref_bin):
        pytest.skip("oracle/_ref/colosim not built")
    cfg = open(os.path.join(CLI, "small.config")).read()
    cfg = cfg.replace("trace.qps = 0.12", "trace.qps = 0.3").replace("trace.duration = 900", "trace.duration = 20000")
    cfg = cfg.replace("histogram:lengths.jsonl", "histogram:" + os.path.join(CLI, "lengths.jsonl"))
    cp = tmp_path / "long.config"
    cp.write_text(cfg)
    eng = ex.GpuEngine(cs.Context(0))
    for mode in ("", "baseline", "serving-only"):
        dr, dg = tmp_path / f"ref{mode}", tmp_path / f"gpu{mode}"
        args = [ref_bin, "run", "--config", str(cp), "--out", str(dr)] + (["--mode", mode] if mode else [])
        subprocess.run(args, check=True, capture_output=True)
        ex.cmd_run(eng, str(cp), str(dg), mode_override=mode)
        names = sorted(os.listdir(dr))
        assert names == sorted(os.listdir(dg)), (mode, names)
        for nm in names:
            assert (dr / nm).read_bytes() == (dg / nm).read_bytes(), (mode, nm)


@pytest.mark.parametrize("variant", ["small", "timeout5", "cap48_d2h2", "cpa_label0", "cpt_label0"])
def test_cli_emit_events_matches_reference(tmp_path, variant):
    """`run --emit-events`: events.jsonl byte-identical to the reference CLI's
    (LoggedEvent::to_json in dispatch order) in all three modes, including
    cache timeouts, prefetch loads, training resumes, the SeparateCluster
    trainer's layers and zero label delays."""
    import os
    import subprocess

    from experiment_check import CLI

    ref_bin = os.path.join(os.path.dirname(CLI), "..", "..", "oracle", "_ref", "colosim")
    if not os.path.exists(ref_bin):
        pytest.skip("oracle/_ref/colosim not built")
    cfg = open(os.path.join(CLI, "small.config")).read()
    cfg = cfg.replace("histogram:lengths.jsonl", "histogram:" + os.path.join(CLI, "lengths.jsonl"))
    cfg = {"small": cfg,
           "timeout5": cfg.replace("sim.cache_timeout = 60", "sim.cache_timeout = 5"),
           "cap48_d2h2": cfg.replace("gpu.capacity_bytes = 85899345920", "gpu.capacity_bytes = 51539607552")
                            .replace("gpu.d2h_bandwidth = 24000000000", "gpu.d2h_bandwidth = 2000000000")
                            .replace("gpu.h2d_bandwidth = 24000000000", "gpu.h2d_bandwidth = 4000000000"),
           "cpa_label0": cfg.replace("trace.label_delay = uniform:0,30", "trace.label_delay = fixed:0"),
           "cpt_label0": cfg.replace("sim.training = cpa", "sim.training = cpt")
                            .replace("trace.label_delay = uniform:0,30", "trace.label_delay = fixed:0")}[variant]
    cp = tmp_path / "v.config"
    cp.write_text(cfg)
    eng = ex.GpuEngine(cs.Context(0))
    for mode in ("", "serving-only", "baseline"):
        dr, dg = tmp_path / f"ref{mode}", tmp_path / f"gpu{mode}"
        subprocess.run([ref_bin, "run", "--config", str(cp), "--out", str(dr), "--emit-events"] +
                       (["--mode", mode] if mode else []), check=True, capture_output=True)
        ex.cmd_run(eng, str(cp), str(dg), mode_override=mode, emit_events=True)
        for nm in ("events.jsonl", "report.csv", "report.jsonl", "tpt_cdf.csv"):
            assert (dr / nm).read_bytes() == (dg / nm).read_bytes(), (variant, mode, nm)


def test_cli_emit_events_random_configs(tmp_path):
    """Random configs (load, horizon, cache timeout, CPA/CPT, label delays,
    capacity and copy bandwidths) x the three modes: the run succeeds or
    breaches exactly when the reference's does, and events.jsonl is
    byte-identical."""
    import os
    import random
    import subprocess

    from experiment_check import CLI

    ref_bin = os.path.join(os.path.dirname(CLI), "..", "..", "oracle", "_ref", "colosim")
    if not os.path.exists(ref_bin):
        pytest.skip("oracle/_ref/colosim not built")
    base = open(os.path.join(CLI, "small.config")).read()
    base = base.replace("histogram:lengths.jsonl", "histogram:" + os.path.join(CLI, "lengths.jsonl"))
    rng = random.Random(31)
    eng = ex.GpuEngine(cs.Context(0))
    for it in range(8):
        cfg = (base.replace("trace.qps = 0.12", f"trace.qps = {rng.choice([0.03, 0.12, 0.3, 0.8])}")
               .replace("trace.duration = 900", f"trace.duration = {rng.choice([300, 900, 2000])}")
               .replace("sim.cache_timeout = 60", f"sim.cache_timeout = {rng.choice([2, 10, 60, 600])}")
               .replace("sim.training = cpa", f"sim.training = {rng.choice(['cpa', 'cpt'])}")
               .replace("sim.seed = 11", f"sim.seed = {rng.randint(1, 10**6)}")
               .replace("trace.label_delay = uniform:0,30",
                        "trace.label_delay = " + rng.choice(["uniform:0,30", "fixed:0", "fixed:0.5", "uniform:0,200"]))
               .replace("gpu.capacity_bytes = 85899345920", f"gpu.capacity_bytes = {rng.choice([48, 64, 80]) * 1024**3}")
               .replace("gpu.d2h_bandwidth = 24000000000", f"gpu.d2h_bandwidth = {rng.choice([2, 8, 24]) * 10**9}")
               .replace("gpu.h2d_bandwidth = 24000000000", f"gpu.h2d_bandwidth = {rng.choice([4, 24]) * 10**9}"))
        cp = tmp_path / f"c{it}.config"
        cp.write_text(cfg)
        for mode in ("", "serving-only", "baseline"):
            dr, dg = tmp_path / f"r{it}{mode}", tmp_path / f"g{it}{mode}"
            pr = subprocess.run([ref_bin, "run", "--config", str(cp), "--out", str(dr), "--emit-events"] +
                                (["--mode", mode] if mode else []), capture_output=True)
            try:
                ex.cmd_run(eng, str(cp), str(dg), mode_override=mode, emit_events=True)
                ok = True
            except cs.ColoBreachError:
                ok = False
            assert ok == (pr.returncode == 0), (it, mode, pr.returncode)
            if ok:
                assert (dr / "events.jsonl").read_bytes() == (dg / "events.jsonl").read_bytes(), (it, mode)
