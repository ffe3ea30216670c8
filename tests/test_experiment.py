"""The experiment harness (paper_2503_01066_b200/experiment.py: config files,
run / compare / plotdata, report exports) driven by the plain-C restatement
of Simulation::run instead of the GPU, so the host-side logic and the output
formats are pinned on CPU against the reference CLI's own output files."""
import os

import numpy as np
import pytest

from oracle.oracle import Gpu, Grid, Model, OracleLib
from paper_2503_01066_b200 import colosim as cs
from paper_2503_01066_b200 import experiment as ex

from experiment_check import CLI, run_all


class OracleEngine:
    """build_maps / run over oracle/colo_colocated.c (test infrastructure)."""

    def __init__(self):
        self.orc = OracleLib("oracle")
        self._cells = {}

    def build_maps(self, model, gpu, steps, bounds, mode):
        return (model, gpu, Grid(steps.cached_token_step, steps.incoming_token_step, steps.batch_step,
                                 bounds.max_cached_tokens, bounds.max_incoming_tokens, bounds.max_batch), int(mode))

    def sort(self, samples):
        return np.sort(np.asarray(samples, np.float64))

    def run(self, runs, keep_sorted=True):
        out = []
        for r in runs:
            model, gpu, grid, cpa = r.maps
            m = Model(*[getattr(r.model, f) for f, _ in Model._fields_])
            g = Gpu(*[getattr(r.gpu, f) for f, _ in Gpu._fields_])
            key = (bytes(m), bytes(g), bytes(grid), cpa)
            if key not in self._cells:
                self._cells[key] = (self.orc.build_offloading_map(m, g, grid, cpa),
                                    self.orc.build_hedging_map(m, g, grid.cached_step, grid.max_cached, cpa, 128))
            t = r.trace
            sim = {0: "serving-only", 1: "colocated", 2: "baseline"}[int(r.mode)]
            res = self.orc.replay_colocated(m, g, grid, int(r.training), t.arrival, t.prompt, t.output,
                                            t.label_delay, r.cache_timeout, want_batches=False, sim_mode=sim,
                                            cells=self._cells[key])
            if res["rc"] == 3:
                raise cs.ColoBreachError(3, "breach")
            rep = {f: res["report"][f] for f in cs.METRICS_FIELDS}
            rep["oom_flag"] = rep["oom_jobs"] > 0
            rep["tpt_samples"] = res["samples"].copy()
            rep["trace_hash"] = t.content_hash()
            rep["mode_tag"] = f"{ex._sm_str(r.mode)}/{ex._tm_str(r.training)}"
            if len(rep["tpt_samples"]):  # what the GPU engine gets from colo_finalize, here from the oracle
                rep["_finalized"] = list(self.orc.finalize(rep["tpt_samples"]))
                rep["_sorted_for_cdf"] = np.sort(rep["tpt_samples"])
            out.append(ex.finalize_report(rep))
        return out


def test_config_parsing(monkeypatch):
    monkeypatch.chdir(CLI)  # histogram:lengths.jsonl resolves against the working directory, as in the reference
    ec = ex.ExperimentConfig.from_file("small.config")
    assert ec.mode == cs.SimMode.COLOCATED and ec.training == cs.TrainingMode.CPA
    assert ec.sweep_qps == [0.02, 0.08, 0.14] and ec.sweep_token_lengths == [500, 2000, 4000]
    assert ec.sweep_modes == [cs.TrainingMode.CPT, cs.TrainingMode.CPA] and ec.sweep_min_tokens == 4000
    assert ec.trace_spec.label_delay == ("uniform", 0.0, 30.0)
    with pytest.raises(cs.ColoValidationError):
        ex.KvFile.parse_text("a = 1\na = 2\n")  # duplicate key (kvfile.hpp:41-43)
    kv = ex.KvFile.parse_text("x.y = 1\nz = 2\n")
    kv.section("x")
    with pytest.raises(cs.ColoValidationError):
        kv.reject_unknown()  # kvfile.hpp:96-101
    assert ex.parse_distribution("none") is None
    assert ex.KvFile.parse_text("k = 1e3").get_u64("k") == 1000  # kvfile.hpp:114-119


def test_trace_hash_matches_reference_fixture():
    # the trace_hash the reference CLI printed for small.config's trace (report.jsonl "run" group)
    import json
    exp = json.load(open(os.path.join(CLI, "expected.json")))
    head = exp["run_colocated"]["report.jsonl"]["head"][0]
    want = json.loads(head)["trace_hash"]
    cwd = os.getcwd()
    os.chdir(CLI)
    try:
        ec = ex.ExperimentConfig.from_file("small.config")
        assert ec.trace_spec.realize().content_hash() == want
    finally:
        os.chdir(cwd)


def test_harness_outputs_match_reference_cli(tmp_path):
    run_all(OracleEngine(), str(tmp_path))


def test_plotdata_roundtrip(tmp_path):
    cwd = os.getcwd()
    os.chdir(CLI)
    try:
        ex.cmd_run(OracleEngine(), "small.config", str(tmp_path / "r"))
    finally:
        os.chdir(cwd)
    ex.cmd_plotdata(str(tmp_path / "r" / "report.jsonl"), str(tmp_path / "p"), engine=OracleEngine())
    assert open(tmp_path / "p" / "tpt_cdf.csv").read() == open(tmp_path / "r" / "tpt_cdf.csv").read()
    r = ex.import_jsonl(str(tmp_path / "r" / "report.jsonl"))
    assert r["mode_tag"] == "colocated/cpa" and len(r["tpt_samples"]) == r["generated_tokens"]
