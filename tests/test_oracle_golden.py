"""The CPU oracle restatement against the golden fixtures written from the
compiled reference (tests/golden/make_golden.py), and -- when oracle/_ref is
present -- directly against the reference on fresh random inputs.  No GPU."""
import os

import numpy as np
import pytest

from oracle.oracle import (PATHS, Grid, OracleLib, TUPLE_DTYPE, default_grid, default_gpu, default_model,
                           phi14b_model, sharegpt_histogram)

GOLD = os.path.join(os.path.dirname(__file__), "golden")
MODELS = {"llama8b": default_model(), "phi14b": phi14b_model()}
GRIDS = {"s500": default_grid(), "s250": Grid(250, 250, 5, 8000, 8000, 50), "s100": Grid(100, 100, 5, 8000, 8000, 50)}
G = default_gpu()


@pytest.fixture(scope="module")
def orc():
    return OracleLib("oracle")


def load(name):
    return np.load(os.path.join(GOLD, name))


def test_maps_and_hashes(orc):
    z = load("maps.npz")
    for mn, m in MODELS.items():
        assert orc.profile_hash(m, G) == int(z[f"hash_{mn}"])
        for gn, gr in GRIDS.items():
            for cpa in (0, 1):
                assert (orc.build_offloading_map(m, G, gr, cpa) == z[f"off_{mn}_{gn}_{cpa}"]).all()
                assert (orc.build_hedging_map(m, G, gr.cached_step, gr.max_cached, cpa) == z[f"hed_{mn}_{gn}_{cpa}"]).all()
        for cpa in (0, 1):
            assert (orc.build_hedging_map(m, G, 250, 8000, cpa) == z[f"hed_{mn}_h250_{cpa}"]).all()


def test_cost_model_bits(orc):
    z = load("cost_model.npz")
    toks = z["tokens"]
    for mn, m in MODELS.items():
        f = lambda fn, *a: np.array([fn(m, int(t), *a)[0] for t in toks])
        assert (f(orc.prefill_latency).view(np.uint64) == z[f"prefill_{mn}"].view(np.uint64)).all()
        assert (f(orc.prefill_latency, 1, True).view(np.uint64) == z[f"prefill_rec_{mn}"].view(np.uint64)).all()
        assert (f(orc.decode_step_latency).view(np.uint64) == z[f"decode_{mn}"].view(np.uint64)).all()
        assert (f(orc.decode_step_latency, 1, True).view(np.uint64) == z[f"decode_rec_{mn}"].view(np.uint64)).all()
        assert (f(orc.forward_layer_latency).view(np.uint64) == z[f"fwd_{mn}"].view(np.uint64)).all()
        assert (f(orc.backward_layer_latency).view(np.uint64) == z[f"bwd_{mn}"].view(np.uint64)).all()
        need = np.array([orc.serving_memory(m, int(t), b)[0] for t in toks for b in (1, 5, 50)], np.uint64)
        assert (need == z[f"need_{mn}"]).all()
        rc = np.array([orc.hedge_recompute_time(m, cpa, int(t))[0] for t in toks for cpa in (0, 1)])
        assert (rc.view(np.uint64) == z[f"recompute_{mn}"].view(np.uint64)).all()
        res = np.array([orc.hedge_residual_load_time(m, G, int(t), f_)[0] for t in toks
                        for f_ in range(0, int(m.num_layers) + 1, 4)])
        assert (res.view(np.uint64) == z[f"residual_{mn}"].view(np.uint64)).all()


def test_verdicts(orc):
    z = load("verdicts.npz")
    for mn, m in MODELS.items():
        t = z[f"tuples_{mn}"]
        for cpa in (0, 1):
            assert (orc.decide(m, G, default_grid(), cpa, t) == z[f"v_{mn}_{cpa}"]).all()
            assert (orc.decide_exact(m, G, cpa, t) == z[f"x_{mn}_{cpa}"]).all()
            assert (orc.decide(m, G, default_grid(), cpa, t, hedge_step=250, hedge_max=8000) == z[f"vh250_{mn}_{cpa}"]).all()


def test_fused(orc):
    z = load("fused.npz")
    sets = [(default_model(), G, 1), (default_model(), G, 0), (phi14b_model(), G, 1), (phi14b_model(), G, 0)]
    v = orc.features_decide(sets, default_grid(), z["prompt"], z["output"], z["dev_offsets"], z["dev_set"])
    assert (v == z["verdicts"]).all()


@pytest.mark.parametrize("name", ["q005", "q03", "q17", "ties", "varout"])
def test_replay(orc, name):
    z = load("replay.npz")
    tau = float(z["tau"][0])
    r = orc.replay_serving(default_model(), G, z[f"{name}_arrival"], z[f"{name}_prompt"], z[f"{name}_output"],
                           tau=tau, grid=default_grid(), cpa=1)
    assert (r["samples"].view(np.uint64) == z[f"{name}_samples"].view(np.uint64)).all()
    assert (r["labels"] == z[f"{name}_labels"]).all()
    assert (r["batches"] == z[f"{name}_batches"]).all()
    s = r["summary"]
    assert [s["generated_tokens"], s["slow_tokens"], s["slow_queries"], s["batches"], s["peak_device_bytes"],
            s["max_batch_size"]] == list(z[f"{name}_summary"])
    assert s["end_time"] == z[f"{name}_end_time"][0]
    p = np.array(r["pctl"])
    ref = z[f"{name}_pctl"]
    assert (p[:3] == ref[:3]).all()  # nearest-rank percentiles: exact
    assert p[3] == ref[3]            # same sorted sequential mean


def test_generate_trace(orc):
    z = load("workload.npz")
    hv, hp = sharegpt_histogram()
    for seed in (7, 41):
        a, p, _ = orc.generate_trace(1.7, 300.0, ("histogram", hv, hp), seed, ("fixed", 0.01))
        assert (a == z[f"hist_{seed}_a"]).all() and (p == z[f"hist_{seed}_p"]).all()
    a, p, _ = orc.generate_trace(0.14, 2000.0, ("uniform", 4000, 7000, 4000), 5, ("uniform", 0.0, 1.0))
    assert (a == z["unif_a"]).all() and (p == z["unif_p"]).all()


@pytest.mark.skipif(not os.path.exists(PATHS["ref"]), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", [1, 2])
def test_random_against_reference(orc, seed):
    ref = OracleLib("ref")
    rng = np.random.default_rng(seed)
    n = 100000
    for m in MODELS.values():
        t = np.zeros(n, TUPLE_DTYPE)
        t["cached"] = rng.integers(0, 9000, n)
        t["incoming"] = rng.integers(0, 9000, n)
        t["charged"] = rng.integers(0, 9000, n)
        t["batch"] = rng.integers(0, 70, n)
        t["pending"] = rng.integers(0, 60, n)
        t["dev_layers"] = rng.integers(0, 60, n)
        for cpa in (0, 1):
            gr = GRIDS["s250"]
            assert (orc.decide(m, G, gr, cpa, t) == ref.decide(m, G, gr, cpa, t)).all()
            assert (orc.decide_exact(m, G, cpa, t) == ref.decide_exact(m, G, cpa, t)).all()
    hv, hp = sharegpt_histogram()
    a, p, o = ref.generate_trace(0.8, 1500.0, ("histogram", hv, hp), seed)
    o = rng.integers(1, 200, len(o)).astype(np.uint32)
    x = orc.replay_serving(phi14b_model(), G, a, p, o, tau=0.05, grid=default_grid(), cpa=0)
    y = ref.replay_serving(phi14b_model(), G, a, p, o, tau=0.05, grid=default_grid(), cpa=0)
    assert (x["samples"].view(np.uint64) == y["samples"].view(np.uint64)).all()
    assert (x["labels"] == y["labels"]).all() and (x["batches"] == y["batches"]).all()
