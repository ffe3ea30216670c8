"""The plain-C restatement of the colocated replay (oracle/colo_colocated.c)
against the golden fixtures written by the reference's own Simulation::run
(SimMode::Colocated, tests/golden/make_golden.py), and -- when oracle/_ref is
present -- directly against the reference on fresh random traces, profiles
and timeouts, including runs that end in InvariantBreach.  No GPU."""
import os

import numpy as np
import pytest

from oracle.oracle import (KGB, KGIB, METRICS_FIELDS, PATHS, ColoReport, Gpu, Grid, Model, OracleLib, default_gpu,
                           default_grid, default_model, phi14b_model, sharegpt_histogram)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def orc():
    return OracleLib("oracle")


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "colocated.npz"))


def case(z, name):
    m = Model.from_buffer_copy(z[f"{name}_model"].tobytes())
    g = Gpu.from_buffer_copy(z[f"{name}_gpu"].tobytes())
    grid = Grid.from_buffer_copy(z[f"{name}_grid"].tobytes())
    cpa, to, sim = z[f"{name}_cfg"]
    rep = ColoReport.from_buffer_copy(z[f"{name}_report"].tobytes())
    return (m, g, grid, int(cpa), float(to), z[f"{name}_a"], z[f"{name}_p"], z[f"{name}_o"], z[f"{name}_ld"], rep,
            ["serving-only", "colocated", "baseline"][int(sim)])


def same_report(a, b):
    bad = []
    for f in METRICS_FIELDS:
        x, y = a[f], (getattr(b, f) if not isinstance(b, dict) else b[f])
        if isinstance(x, float):
            if np.float64(x).view(np.uint64) != np.float64(y).view(np.uint64):
                bad.append((f, x, y))
        elif x != y:
            bad.append((f, x, y))
    return bad


def test_fixture_inventory(gold):
    names = list(gold["names"])
    assert len(names) >= 20
    modes = {float(gold[f"{n}_cfg"][2]) for n in names}
    assert modes == {0.0, 1.0, 2.0}
    assert sum(int(gold[f"{n}_rc"][0]) == 3 for n in names) >= 2  # InvariantBreach cases
    assert any(int(ColoReport.from_buffer_copy(gold[f"{n}_report"].tobytes()).loads) > 0 for n in names)
    assert any(int(ColoReport.from_buffer_copy(gold[f"{n}_report"].tobytes()).recomputes) > 0 for n in names)
    assert any(int(ColoReport.from_buffer_copy(gold[f"{n}_report"].tobytes()).labels_dropped) > 0 for n in names)


def test_oracle_matches_golden(orc, gold):
    """Every MetricsReport field bit-for-bit, samples bit-for-bit, batch
    timeline (start, end, first, n) and the breach verdicts."""
    for name in gold["names"]:
        m, g, grid, cpa, to, a, p, o, ld, rep, sim = case(gold, name)
        r = orc.replay_colocated(m, g, grid, cpa, a, p, o, ld, to, sim_mode=sim)
        assert r["rc"] == int(gold[f"{name}_rc"][0]), name
        if r["rc"] != 0:
            continue
        assert not same_report(r["report"], rep), (name, same_report(r["report"], rep))
        s = gold[f"{name}_samples"]
        assert np.array_equal(r["samples"].view(np.uint64), s.view(np.uint64)), name
        b = r["batches"]
        gb = gold[f"{name}_batches"]
        got = np.stack([b["start"], b["end"], b["first"].astype(np.float64), b["n"].astype(np.float64)], 1)
        assert got.shape == gb.shape and np.array_equal(got.view(np.uint64), gb.view(np.uint64)), name
        if len(s):  # finalize (metrics.hpp:56-69): nearest-rank percentiles and the sorted sequential mean
            assert np.array_equal(np.array(orc.finalize(s)).view(np.uint64), gold[f"{name}_pctl"].view(np.uint64))


def test_engine_kats(orc, gold):
    """The reference's own engine assertions (tests/test_engine.cpp:186-265) on
    the restatement."""
    m, g, grid = default_model(), default_gpu(), default_grid()
    # :189-195 late label: q0 holds the slot until the timeout; 2 labels dropped, no jobs
    r = orc.replay_colocated(m, g, grid, 1, np.array([0.0, 10.0]), np.array([1000, 1000], np.uint32),
                             np.full(2, 128, np.uint32), np.array([3600.0, 0.01]))["report"]
    assert r["completed_jobs"] == 0 and r["labels_dropped"] == 2
    # :197-204 slot clears at the timeout and admits the next eligible query
    r = orc.replay_colocated(m, g, grid, 1, np.array([0.0, 100.0]), np.array([1000, 900], np.uint32),
                             np.full(2, 128, np.uint32), np.array([-1.0, 0.01]))["report"]
    assert r["completed_jobs"] == 1 and r["trained_tokens"] == 900 + 256 and r["labels_dropped"] == 1
    # :241-248 streaming regime trains and loads back
    r = orc.replay_colocated(m, g, grid, 1, np.array([0.0]), np.array([6000], np.uint32), np.array([128], np.uint32),
                             np.array([0.01]))["report"]
    assert r["completed_jobs"] == 1 and r["trained_tokens"] == 6000 + 256 and r["loads"] > 0
    assert r["peak_device_bytes"] <= g.capacity_bytes
    # :250-265 slow copies surface a copy stall
    g2 = default_gpu()
    g2.d2h_bandwidth, g2.h2d_bandwidth = 2 * KGB, 1000 * KGB
    r = orc.replay_colocated(m, g2, grid, 1, np.array([0.0] + [5.0] * 10), np.full(11, 4000, np.uint32),
                             np.full(11, 128, np.uint32), None)["report"]
    assert r["layers_freed"] > 0 and r["copy_stall_seconds"] > 1.0
    # :54-59 empty trace: peak is the fixed footprint
    r = orc.replay_colocated(m, g, grid, 1, np.zeros(0), np.zeros(0, np.uint32), np.zeros(0, np.uint32), None)
    assert r["report"]["peak_device_bytes"] == m.weights_bytes + g.runtime_reserve_bytes
    assert r["report"]["trained_tokens"] == 0 and r["report"]["generated_tokens"] == 0
    # :304-309 freed layers cover loads
    a, p, o, ld = orc.generate_trace(0.25, 400, ("uniform", 3000, 6000), 31, ("fixed", 0.01), with_labels=True)
    r = orc.replay_colocated(m, g, grid, 1, a, p, o, ld)["report"]
    assert r["layers_freed"] >= r["loads"]


def test_serving_conservation(orc):
    """tests/test_engine.cpp:176-184: with no runnable training (labels never
    arrive in CPA) the colocated TPT samples equal the serving-only ones."""
    hv, hp = sharegpt_histogram()
    m, g, grid = default_model(), default_gpu(), default_grid()
    a, p, o = orc.generate_trace(0.05, 3000, ("histogram", hv, hp), 3)
    r = orc.replay_colocated(m, g, grid, 1, a, p, o, None)
    s = orc.replay_serving(m, g, a, p, o)
    assert np.array_equal(r["samples"].view(np.uint64), s["samples"].view(np.uint64))


def test_generate_trace_label_delays(orc):
    if not os.path.exists(PATHS["ref"]):
        pytest.skip("oracle/_ref not built")
    ref = OracleLib("ref")
    for spec in (("fixed", 0.01), ("uniform", 0.0, 30.0), None):
        x = orc.generate_trace(0.3, 500.0, ("uniform", 100, 3000), 11, spec, with_labels=True)
        y = ref.generate_trace(0.3, 500.0, ("uniform", 100, 3000), 11, spec, with_labels=True)
        for u, v in zip(x, y):
            assert np.array_equal(np.asarray(u).view(np.uint8), np.asarray(v).view(np.uint8))


def test_oracle_matches_reference_fuzz_modes(orc):
    """ServingOnly and SeparateCluster runs of the restated engine equal the
    reference's, including OOM jobs and varying / absent label delays."""
    if not os.path.exists(PATHS["ref"]):
        pytest.skip("oracle/_ref not built")
    ref = OracleLib("ref")
    rng = np.random.default_rng(99)
    n_oom = 0
    for it in range(40):
        m = default_model() if it % 2 else phi14b_model()
        g = default_gpu()
        grid = default_grid()
        cpa = int(rng.integers(0, 2))
        mode = "baseline" if it % 4 else "serving-only"
        qps = float(rng.choice([0.05, 0.3, 1.0, 3.0]))
        lo_, hi_ = sorted(rng.integers(1, 8000, 2))
        a, p, o, ld = orc.generate_trace(qps, 30 / qps + 60, ("uniform", float(lo_), float(hi_ + 1)),
                                         int(rng.integers(1 << 30)), ("uniform", 0.0, float(rng.choice([0.01, 300]))),
                                         with_labels=True)
        if it % 3 == 0:
            ld[::3] = -1.0
        try:
            r1 = ref.replay_colocated(m, g, grid, cpa, a, p, o, ld, 60.0, sim_mode=mode)
        except ValueError:
            continue
        r2 = orc.replay_colocated(m, g, grid, cpa, a, p, o, ld, 60.0, sim_mode=mode)
        assert r1["rc"] == r2["rc"] == 0
        assert not same_report(r2["report"], r1["report"]), (it, same_report(r2["report"], r1["report"]))
        assert np.array_equal(r1["samples"].view(np.uint64), r2["samples"].view(np.uint64))
        n_oom += r1["report"]["oom_jobs"] > 0
    assert n_oom >= 3


def test_oracle_matches_reference_fuzz(orc):
    """Fresh random profiles, grids, modes, loads, outputs and timeouts: the
    restatement equals the reference's Simulation::run (breach or report)."""
    if not os.path.exists(PATHS["ref"]):
        pytest.skip("oracle/_ref not built")
    ref = OracleLib("ref")
    rng = np.random.default_rng(2024)
    runs = breaches = 0
    for _ in range(60):
        m = default_model() if rng.random() < 0.5 else phi14b_model()
        g = default_gpu()
        g.capacity_bytes = int(rng.choice([40, 60, 80])) * KGIB
        g.d2h_bandwidth = int(rng.choice([1, 2, 24])) * KGB
        g.h2d_bandwidth = int(rng.choice([1, 24, 200])) * KGB
        if orc.validate_profile_pair(m, g):
            continue
        grid = Grid(int(rng.choice([250, 500])), 500, 5, 8000, 8000, 50)
        cpa = int(rng.integers(0, 2))
        qps = float(rng.choice([0.02, 0.1, 0.3, 1.0]))
        lo_, hi_ = sorted(rng.integers(1, 9000, 2))
        a, p, o, ld = orc.generate_trace(qps, 30 / qps + 100, ("uniform", float(lo_), float(hi_ + 1)),
                                         int(rng.integers(1 << 30)), ("uniform", 0.0, float(rng.choice([0.01, 50]))),
                                         with_labels=True)
        if rng.random() < 0.5:
            o = rng.integers(1, 200, len(a)).astype(np.uint32)
        to = float(rng.choice([1.0, 60.0]))
        try:
            r1 = ref.replay_colocated(m, g, grid, cpa, a, p, o, ld, to)
        except ValueError:  # a query that cannot fit the device alone (engine.hpp:70-74)
            with pytest.raises(ValueError):
                orc.replay_colocated(m, g, grid, cpa, a, p, o, ld, to)
            continue
        r2 = orc.replay_colocated(m, g, grid, cpa, a, p, o, ld, to)
        assert r1["rc"] == r2["rc"]
        runs += 1
        if r1["rc"]:
            breaches += 1
            continue
        assert not same_report(r2["report"], r1["report"])
        assert np.array_equal(r1["samples"].view(np.uint64), r2["samples"].view(np.uint64))
    assert runs >= 30 and breaches >= 1
