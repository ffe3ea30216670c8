"""Writes the golden fixtures under tests/golden/ from the REFERENCE itself.

Every array here comes out of oracle/_ref/libcolo_ref.so, i.e. the unchanged
colosim headers (/root/reference/proj/include) compiled by oracle/Makefile.
Run in the build container (needs /root/reference to rebuild _ref):

    make -C oracle && python tests/golden/make_golden.py

The fixtures pin both the plain-C oracle restatement (CPU tests) and the
sm_100a kernels (GPU tests) to the reference's own outputs.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import (KGB, KGIB, Grid, OracleLib, TUPLE_DTYPE, default_gpu, default_grid, default_model, phi14b_model,  # noqa: E402
                           sharegpt_histogram)


def models():
    return {"llama8b": default_model(), "phi14b": phi14b_model()}


def grids():
    return {"s500": default_grid(), "s250": Grid(250, 250, 5, 8000, 8000, 50), "s100": Grid(100, 100, 5, 8000, 8000, 50)}


def random_tuples(rng, n, L):
    t = np.zeros(n, TUPLE_DTYPE)
    t["cached"] = rng.integers(0, 8600, n)
    t["incoming"] = rng.integers(0, 8600, n)
    t["charged"] = rng.integers(0, 9200, n)
    t["batch"] = rng.integers(0, 60, n)
    t["pending"] = rng.integers(0, L + 3, n)
    t["dev_layers"] = rng.integers(0, L + 3, n)
    # edge cases from the reference tests and the lookup domain (maps.hpp:100-110, 276-280)
    edge = []
    for c in (0, 1, 499, 500, 501, 4000, 4200, 7999, 8000, 8001, 0xFFFFFFFF):
        for i in (0, 1, 420, 500, 2000, 8000, 8001):
            for b in (0, 1, 5, 6, 10, 50, 51, 0xFFFF):
                edge.append((c, i, c, b, 0, L))
    e = np.array(edge, dtype=[(k, "<u8") for k in ("cached", "incoming", "charged", "batch", "pending", "dev_layers")])
    k = min(len(e), n)
    for f in TUPLE_DTYPE.names:
        t[f][:k] = e[f][:k].astype(t[f].dtype)
    return t


def replay_traces(ref):
    hv, hp = sharegpt_histogram()
    out = {}
    for name, qps, dur, seed in (("q005", 0.05, 6000.0, 41), ("q03", 0.3, 2000.0, 41), ("q17", 1.7, 480.0, 41)):
        out[name] = ref.generate_trace(qps, dur, ("histogram", hv, hp), seed, ("fixed", 0.01))
    # forced same-time arrivals and an arrival exactly at a batch end
    a, p, o = ref.generate_trace(0.3, 600.0, ("uniform", 200, 3000), 5)
    a = np.repeat(a, 2)[: 2 * len(a)]
    p = np.repeat(p, 2)
    o = np.repeat(o, 2)
    a = np.concatenate([[0.0, 0.0, 0.0, 1.0], a + 2.0])
    p = np.concatenate([[1000, 500, 2000, 800], p]).astype(np.uint32)
    o = np.concatenate([[128, 128, 128, 128], o]).astype(np.uint32)
    out["ties"] = (a, p, o)
    # variable output lengths
    rng = np.random.default_rng(3)
    a, p, o = ref.generate_trace(0.6, 500.0, ("histogram", hv, hp), 77)
    o = rng.integers(1, 300, len(o)).astype(np.uint32)
    out["varout"] = (a, p, o)
    return out


def main():
    ref = OracleLib("ref")
    g = default_gpu()
    rng = np.random.default_rng(20251017)
    # ---- maps
    maps = {}
    for mn, m in models().items():
        for gn, gr in grids().items():
            for cpa in (0, 1):
                maps[f"off_{mn}_{gn}_{cpa}"] = ref.build_offloading_map(m, g, gr, cpa)
                maps[f"hed_{mn}_{gn}_{cpa}"] = ref.build_hedging_map(m, g, gr.cached_step, gr.max_cached, cpa)
        for cpa in (0, 1):  # hedge grid different from the offload grid
            maps[f"hed_{mn}_h250_{cpa}"] = ref.build_hedging_map(m, g, 250, 8000, cpa)
    hashes = {mn: np.uint64(ref.profile_hash(m, g)) for mn, m in models().items()}
    np.savez_compressed(os.path.join(HERE, "maps.npz"), **maps,
                        **{f"hash_{k}": v for k, v in hashes.items()})

    # ---- cost model values over a token sweep
    toks = np.array([1, 17, 64, 128, 420, 500, 1000, 1234, 3000, 4000, 4096, 7999, 8000, 70000], np.uint64)
    cm = {}
    for mn, m in models().items():
        cm[f"prefill_{mn}"] = np.array([ref.prefill_latency(m, int(t))[0] for t in toks])
        cm[f"prefill_rec_{mn}"] = np.array([ref.prefill_latency(m, int(t), 1, True)[0] for t in toks])
        cm[f"decode_{mn}"] = np.array([ref.decode_step_latency(m, int(t))[0] for t in toks])
        cm[f"decode_rec_{mn}"] = np.array([ref.decode_step_latency(m, int(t), 1, True)[0] for t in toks])
        cm[f"fwd_{mn}"] = np.array([ref.forward_layer_latency(m, int(t))[0] for t in toks])
        cm[f"bwd_{mn}"] = np.array([ref.backward_layer_latency(m, int(t))[0] for t in toks])
        cm[f"need_{mn}"] = np.array([ref.serving_memory(m, int(t), b)[0] for t in toks for b in (1, 5, 50)], np.uint64)
        cm[f"recompute_{mn}"] = np.array([ref.hedge_recompute_time(m, cpa, int(t))[0] for t in toks for cpa in (0, 1)])
        cm[f"residual_{mn}"] = np.array([ref.hedge_residual_load_time(m, g, int(t), f)[0] for t in toks
                                         for f in range(0, int(m.num_layers) + 1, 4)])
    np.savez_compressed(os.path.join(HERE, "cost_model.npz"), tokens=toks, **cm)

    # ---- composed verdicts on tuples (quantised + exact)
    tv = {}
    for mn, m in models().items():
        t = random_tuples(rng, 40000, int(m.num_layers))
        tv[f"tuples_{mn}"] = t
        for cpa in (0, 1):
            tv[f"v_{mn}_{cpa}"] = ref.decide(m, g, default_grid(), cpa, t)
            tv[f"x_{mn}_{cpa}"] = ref.decide_exact(m, g, cpa, t)
            tv[f"vh250_{mn}_{cpa}"] = ref.decide(m, g, default_grid(), cpa, t, hedge_step=250, hedge_max=8000)
    np.savez_compressed(os.path.join(HERE, "verdicts.npz"), **tv)

    # ---- trace-fused verdicts: 7 ragged devices (one empty), 4 map sets
    hv, hp = sharegpt_histogram()
    parts = []
    for d, (qps, seed) in enumerate([(0.05, 1000), (0.1, 1001), (0.2, 1002), (0.3, 1003), (0.1, 1004), (0.3, 1005)]):
        parts.append(ref.generate_trace(qps, 2000.0 + 700 * d, ("histogram", hv, hp), seed))
    sizes = [len(x[1]) for x in parts]
    sizes.insert(3, 0)
    parts.insert(3, (np.zeros(0), np.zeros(0, np.uint32), np.zeros(0, np.uint32)))
    prompt = np.concatenate([x[1] for x in parts]).astype(np.uint32)
    output = np.concatenate([x[2] for x in parts]).astype(np.uint32)
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint64)
    dev_set = np.array([d % 4 for d in range(len(sizes))], np.uint16)
    sets = [(default_model(), g, 1), (default_model(), g, 0), (phi14b_model(), g, 1), (phi14b_model(), g, 0)]
    fused = ref.features_decide(sets, default_grid(), prompt, output, offs, dev_set)
    np.savez_compressed(os.path.join(HERE, "fused.npz"), prompt=prompt, output=output, dev_offsets=offs,
                        dev_set=dev_set, verdicts=fused)

    # ---- serving replays (Simulation::run, ServingOnly)
    rp = {}
    for name, (a, p, o) in replay_traces(ref).items():
        for mn in ("llama8b",):
            m = models()[mn]
            tau = 0.03
            r = ref.replay_serving(m, g, a, p, o, tau=tau, grid=default_grid(), cpa=1)
            rp[f"{name}_arrival"], rp[f"{name}_prompt"], rp[f"{name}_output"] = a, p, o
            rp[f"{name}_samples"] = r["samples"]
            rp[f"{name}_labels"] = r["labels"]
            rp[f"{name}_batches"] = r["batches"]
            rp[f"{name}_pctl"] = r["pctl"]
            s = r["summary"]
            rp[f"{name}_summary"] = np.array([s["generated_tokens"], s["slow_tokens"], s["slow_queries"], s["batches"],
                                              s["peak_device_bytes"], s["max_batch_size"]], np.uint64)
            rp[f"{name}_end_time"] = np.array([s["end_time"]])
    np.savez_compressed(os.path.join(HERE, "replay.npz"), tau=np.array([0.03]), **rp)

    # ---- generate_trace (workload.hpp:193-220)
    gt = {}
    for seed in (7, 41):
        a, p, o = ref.generate_trace(1.7, 300.0, ("histogram", hv, hp), seed, ("fixed", 0.01))
        gt[f"hist_{seed}_a"], gt[f"hist_{seed}_p"] = a, p
    a, p, o = ref.generate_trace(0.14, 2000.0, ("uniform", 4000, 7000, 4000), 5, ("uniform", 0.0, 1.0))
    gt["unif_a"], gt["unif_p"] = a, p
    np.savez_compressed(os.path.join(HERE, "workload.npz"), **gt)
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


def colocated_cases(ref):
    """Colocated-replay cases (Simulation::run, SimMode::Colocated): name ->
    (model, gpu, grid, cpa, cache_timeout, arrival, prompt, output, label_delay)."""
    hv, hp = sharegpt_histogram()
    m, g, grid = default_model(), default_gpu(), default_grid()
    cases = {}
    a, p, o, ld = ref.generate_trace(0.3, 600.0, ("histogram", hv, hp), 41, ("fixed", 0.01), with_labels=True)
    cases["sharegpt_q03_cpa"] = (m, g, grid, 1, 60.0, a, p, o, ld)
    cases["sharegpt_q03_cpt"] = (m, g, grid, 0, 60.0, a, p, o, ld)
    a, p, o, ld = ref.generate_trace(1.7, 150.0, ("histogram", hv, hp), 42, ("fixed", 0.01), with_labels=True)
    cases["sharegpt_q17_cpa"] = (m, g, grid, 1, 60.0, a, p, o, ld)
    a, p, o, ld = ref.generate_trace(0.14, 1200.0, ("uniform", 4000, 7000), 5, ("uniform", 0.0, 30.0), with_labels=True)
    cases["long_q014_cpa_t5"] = (m, g, grid, 1, 5.0, a, p, o, ld)
    cases["long_q014_cpt"] = (m, g, grid, 0, 60.0, a, p, o, ld)
    a, p, o, ld = ref.generate_trace(0.2, 900.0, ("uniform", 2000, 7000), 9, ("fixed", 0.01), with_labels=True)
    cases["phi_q02_cpa"] = (phi14b_model(), g, Grid(250, 250, 5, 8000, 8000, 50), 1, 60.0, a, p, o, ld)
    cases["phi_q02_cpt"] = (phi14b_model(), g, grid, 0, 60.0, a, p, o, ld)
    a, p, o, ld = ref.generate_trace(0.1, 1500.0, ("uniform", 100, 9000), 7, ("uniform", 0.0, 100.0), with_labels=True)
    o = (np.arange(len(a)) * 37 % 199 + 1).astype(np.uint32)  # variable outputs
    cases["wide_varout_cpa"] = (m, g, grid, 1, 60.0, a, p, o, ld)
    # engine test cases (tests/test_engine.cpp:186-265)
    g2 = default_gpu()
    g2.d2h_bandwidth, g2.h2d_bandwidth = 2 * KGB, 1000 * KGB
    cases["copy_stall"] = (m, g2, grid, 1, 60.0, np.array([0.0] + [5.0] * 10), np.full(11, 4000, np.uint32),
                           np.full(11, 128, np.uint32), np.full(11, -1.0))
    cases["offload_path"] = (m, g, grid, 1, 60.0, np.array([0.0] + [4.6 + 0.001 * i for i in range(1, 11)]),
                             np.array([4000] + [2000] * 10, np.uint32), np.full(11, 128, np.uint32),
                             np.array([0.01] + [-1.0] * 10))
    cases["stream_6000"] = (m, g, grid, 1, 60.0, np.array([0.0, 2000.0]), np.array([6000, 6000], np.uint32),
                            np.full(2, 128, np.uint32), np.array([0.01, 0.01]))
    cases["late_label"] = (m, g, grid, 1, 60.0, np.array([0.0, 10.0]), np.array([1000, 1000], np.uint32),
                           np.full(2, 128, np.uint32), np.array([3600.0, 0.01]))
    cases["empty"] = (m, g, grid, 1, 60.0, np.zeros(0), np.zeros(0, np.uint32), np.zeros(0, np.uint32), np.zeros(0))
    # an InvariantBreach: small device, slow copies (found by fuzzing the reference)
    g3 = default_gpu()
    g3.capacity_bytes, g3.d2h_bandwidth, g3.h2d_bandwidth = 80 * KGIB, 2 * KGB, 200 * KGB
    a, p, o, ld = ref.generate_trace(0.3, 40 / 0.3 + 200, ("uniform", 6735.0, 8213.0), 206955, ("uniform", 0.0, 0.01),
                                     with_labels=True)
    cases["breach_slow_d2h"] = (m, g3, grid, 1, 60.0, a, p, o, ld)
    g4 = default_gpu()
    g4.capacity_bytes, g4.d2h_bandwidth, g4.h2d_bandwidth = 40 * KGIB, 1 * KGB, 200 * KGB
    a, p, o, ld = ref.generate_trace(0.1, 40 / 0.1 + 200, ("uniform", 6519.0, 8610.0), 867572, ("uniform", 0.0, 5.0),
                                     with_labels=True)
    cases["breach_small_cpt"] = (m, g4, Grid(250, 500, 5, 8000, 8000, 50), 0, 60.0, a, p, o, ld)
    # SeparateCluster ("baseline") and ServingOnly runs of the same engine
    a, p, o, ld = ref.generate_trace(0.3, 600.0, ("histogram", hv, hp), 41, ("fixed", 0.01), with_labels=True)
    cases["baseline_q03_cpa"] = (m, g, grid, 1, 60.0, a, p, o, ld, 2)
    cases["baseline_q03_cpt"] = (m, g, grid, 0, 60.0, a, p, o, ld, 2)
    cases["serving_q03"] = (m, g, grid, 1, 60.0, a, p, o, ld, 0)
    a, p, o, ld = ref.generate_trace(0.5, 400.0, ("uniform", 500, 7000), 13, ("uniform", 0.0, 200.0), with_labels=True)
    ld[::4] = -1.0
    cases["baseline_varlabels_cpa"] = (m, g, grid, 1, 60.0, a, p, o, ld, 2)  # label delays vary: sorted job stream
    cases["baseline_oom_phi_cpa"] = (phi14b_model(), g, grid, 1, 60.0, a, p, o, ld, 2)
    return cases


def colocated(ref):
    out = {}
    names = []
    for name, c in colocated_cases(ref).items():
        m, g, grid, cpa, to, a, p, o, ld = c[:9]
        sim = c[9] if len(c) > 9 else 1
        r = ref.replay_colocated(m, g, grid, cpa, a, p, o, ld, to, sim_mode=["serving-only", "colocated", "baseline"][sim])
        names.append(name)
        out[f"{name}_model"] = np.frombuffer(bytes(m), np.uint8)
        out[f"{name}_gpu"] = np.frombuffer(bytes(g), np.uint8)
        out[f"{name}_grid"] = np.frombuffer(bytes(grid), np.uint8)
        out[f"{name}_cfg"] = np.array([cpa, to, sim], np.float64)
        out[f"{name}_a"], out[f"{name}_p"], out[f"{name}_o"], out[f"{name}_ld"] = a, p, o, ld
        out[f"{name}_rc"] = np.array([r["rc"]])
        out[f"{name}_report"] = np.frombuffer(bytes(_report_struct(r["report"])), np.uint8)
        if r["rc"] == 0:
            out[f"{name}_samples"] = r["samples"]
            out[f"{name}_pctl"] = r["pctl"]
            b = r["batches"]
            out[f"{name}_batches"] = np.stack([b["start"], b["end"], b["first"].astype(np.float64),
                                               b["n"].astype(np.float64)], 1)
        print(name, len(a), r["rc"], {k: r["report"][k] for k in ("completed_jobs", "recomputes", "loads", "labels_dropped",
                                                                   "oom_jobs")})
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "colocated.npz"), **out)


def _report_struct(rep):
    from oracle.oracle import ColoReport
    c = ColoReport()
    for f, _ in ColoReport._fields_:
        setattr(c, f, rep[f])
    return c


if __name__ == "__main__":
    if sys.argv[1:] == ["colocated"]:
        colocated(OracleLib("ref"))
    else:
        main()
        colocated(OracleLib("ref"))
