"""Pins the CPU oracle restatement (oracle/colo_oracle.c) to the known-answer
values of the reference's own unit tests.  Each test cites the reference test
it restates (paths relative to /root/reference/proj/).  Runs without a GPU."""
import math
import os

import numpy as np
import pytest

from oracle.oracle import (PATHS, Grid, OracleLib, default_grid, default_gpu, default_model, grid_shape,
                           phi14b_model)

BACKENDS = ["oracle"] + (["ref"] if os.path.exists(PATHS["ref"]) else [])
KIB, MIB, GIB, KGB = 1024, 1024**2, 1024**3, 1000**3


@pytest.fixture(scope="module", params=BACKENDS)
def lib(request):
    return OracleLib(request.param)


M, G = default_model(), default_gpu()


def approx(a, b, eps):
    # doctest::Approx(b).epsilon(eps): |a-b| <= eps * (scale + max(|a|,|b|)), scale 1
    return abs(a - b) <= eps * (1.0 + max(abs(a), abs(b)))


def test_prefill_latency_kat(lib):  # tests/test_cost_model.cpp:15-23
    assert approx(lib.prefill_latency(M, 1000)[0], 0.120, 1e-12)
    assert approx(lib.prefill_latency(M, 1000, 1, True)[0], 0.120 * 1.21, 1e-12)
    assert approx(lib.prefill_latency(M, 1)[0], 1e-4, 1e-3)
    assert lib.prefill_latency(M, 0)[1] != 0  # std::invalid_argument
    assert lib.prefill_latency(M, 10, 0)[1] != 0


def test_prefill_monotone(lib):  # tests/test_cost_model.cpp:25-33
    prev = 0
    for t in range(100, 5001, 100):
        v = lib.prefill_latency(M, t)[0]
        assert v > prev
        prev = v
    assert lib.prefill_latency(M, 777, 3)[0] > lib.prefill_latency(M, 777, 2)[0]


def test_decode_step_kat(lib):  # tests/test_cost_model.cpp:35-42
    assert approx(lib.decode_step_latency(M, 1000)[0], 0.022, 1e-12)
    assert approx(lib.decode_step_latency(M, 1000, 1, True)[0], 0.0297, 1e-12)
    assert approx(lib.decode_step_latency(M, 1000, 2)[0], 2 * lib.decode_step_latency(M, 1000)[0], 1e-15)
    assert lib.decode_step_latency(M, 0)[1] != 0


def test_recording_ratio(lib):  # tests/test_cost_model.cpp:44-51
    for t in (1, 17, 420, 1000, 4096, 7999):
        assert approx(lib.prefill_latency(M, t, 1, True)[0] / lib.prefill_latency(M, t)[0], 1.21, 1e-12)
        assert approx(lib.decode_step_latency(M, t, 1, True)[0] / lib.decode_step_latency(M, t)[0], 1.35, 1e-12)


def test_layer_partition_exact(lib):  # tests/test_cost_model.cpp:53-62
    for t in (1000, 4000):
        assert lib.forward_layer_latency(M, t)[0] * 32.0 == lib.prefill_latency(M, t)[0]
    assert approx(lib.forward_layer_latency(M, 1000)[0], 0.00375, 1e-12)
    assert approx(lib.forward_layer_latency(M, 4000)[0], 0.0225, 1e-12)


def test_backward_layer(lib):  # tests/test_cost_model.cpp:64-73
    assert approx(lib.backward_layer_latency(M, 1000)[0], 0.0049725, 1e-9)
    unit = default_model()
    unit.backward_to_forward_ratio = 1.0
    assert lib.backward_layer_latency(unit, 123)[0] == lib.forward_layer_latency(unit, 123)[0]


def test_activation_bytes(lib):  # tests/test_cost_model.cpp:75-82
    b = lib.activation_bytes(M, 3000, 32)[0]
    assert 39600000000 <= b <= 40400000000
    assert lib.activation_bytes(M, 3000, 1)[0] == 1251000000
    assert lib.activation_bytes(M, 0, 5)[0] == 0
    assert lib.activation_bytes(M, 10, 33)[1] != 0


def test_kv_and_serving_memory(lib):  # tests/test_cost_model.cpp:84-97
    assert lib.kv_bytes(M, 3000, 1) == 1500 * MIB
    assert lib.kv_bytes(M, 500, 5) == 1250 * MIB
    assert lib.kv_bytes(M, 0, 9) == 0
    assert lib.serving_memory(M, 500, 5)[0] == 2500 * MIB
    assert lib.serving_memory(M, 500, 10)[0] == 2 * lib.serving_memory(M, 500, 5)[0]
    half = default_model()
    half.workspace_factor = 0.5
    assert lib.serving_memory(half, 1000, 1)[0] == lib.kv_bytes(half, 1000, 1) * 3 // 2


def test_transfer_time(lib):  # tests/test_cost_model.cpp:99-108
    assert approx(lib.transfer_time(G, 53376000000), 2.224, 1e-9)
    assert lib.transfer_time(G, 0, False) == 0.0


def test_profile_pair_and_hash(lib):  # tests/test_cost_model.cpp:137-158
    g = default_gpu()
    g.capacity_bytes = M.weights_bytes
    assert lib.validate_profile_pair(M, g) != 0
    assert lib.validate_profile_pair(phi14b_model(), default_gpu()) == 0
    base = lib.profile_hash(M, G)
    m2 = default_model()
    m2.prefill_coef_quad *= 2
    assert lib.profile_hash(m2, G) != base
    g2 = default_gpu()
    g2.h2d_bandwidth += 1
    assert lib.profile_hash(M, g2) != base
    assert lib.profile_hash(M, G) == base


def test_round_up_bucket(lib):  # tests/test_maps.cpp:23-29
    assert lib.round_up_bucket(420, 500) == 500
    assert lib.round_up_bucket(6, 5) == 10
    assert lib.round_up_bucket(1000, 500) == 1000
    assert lib.round_up_bucket(1, 500) == 500
    assert lib.round_up_bucket(0, 500) == 0


def test_frozen_offload_cells(lib):  # tests/test_maps.cpp:31-53
    assert lib.offload_cell_decision(M, G, 1, 4000, 500, 5) == (0, 0)      # NoAction
    assert lib.offload_cell_decision(M, G, 1, 4000, 2000, 10) == (1, 6)    # FreeLayers(6)
    assert lib.offload_cell_decision(M, G, 1, 0, 4000, 10)[0] == 0         # nothing cached
    assert lib.offload_cell_decision(M, G, 1, 5000, 500, 5)[0] == 2        # AllToHost


def _expected_decision(m, g, cpa, cached, incoming, batch):
    """tests/support/oracles.hpp:22-56, exact rational arithmetic (the reference uses long double)."""
    from fractions import Fraction as F
    budget = F(g.capacity_bytes) - g.runtime_reserve_bytes - m.weights_bytes
    acts = F(cached) * m.num_layers * m.act_bytes_per_token_per_layer
    kv = F(cached) * m.kv_bytes_per_token if cpa else F(0)
    kv_in = F(incoming) * batch * m.kv_bytes_per_token
    need = kv_in + kv_in * F(m.workspace_factor)
    per_layer = F(cached) * m.act_bytes_per_token_per_layer
    if acts + kv > budget:
        return (2, 0)
    headroom = budget - acts - kv
    if need <= headroom:
        return (0, 0)
    if per_layer <= 0:
        return (2, 0)
    n, rec = 0, F(0)
    while rec < need - headroom and n <= m.num_layers:
        n += 1
        rec += per_layer
    if n > m.num_layers:
        return (2, 0)
    return (1, n)


@pytest.mark.parametrize("cpa", [1, 0])
def test_every_cell_matches_independent_oracle(lib, cpa):  # tests/test_maps.cpp:55-67
    grid = default_grid()
    cells = lib.build_offloading_map(M, G, grid, cpa)
    C_, I_, B_ = grid_shape(grid)
    for ci in range(C_):
        for ii in range(I_):
            for bi in range(B_):
                a, n = _expected_decision(M, G, cpa, ci * 500, (ii + 1) * 500, (bi + 1) * 5)
                code = 0 if a == 0 else 1 if a == 2 else 2 + n
                assert cells[(ci * I_ + ii) * B_ + bi] == code


def test_map_monotone(lib):  # tests/test_maps.cpp:106-120
    grid = default_grid()
    C_, I_, B_ = grid_shape(grid)
    cells = lib.build_offloading_map(M, G, grid, 1).reshape(C_, I_, B_).astype(int)
    rank = np.where(cells == 0, 0, np.where(cells == 1, 33, cells - 2))
    assert (np.diff(rank, axis=0) >= 0).all()
    assert (np.diff(rank, axis=1) >= 0).all()
    assert (np.diff(rank, axis=2) >= 0).all()


def test_grid_validation(lib):  # tests/test_maps.cpp:141-150
    with pytest.raises(ValueError):
        lib.build_offloading_map(M, G, Grid(500, 500, 5, 8000, 8100, 50), 1)
    with pytest.raises(ValueError):
        lib.build_offloading_map(M, G, Grid(500, 500, 0, 8000, 8000, 50), 1)


def _hedge(lib, cpa):
    cells = lib.build_hedging_map(M, G, 500, 8000, cpa)
    return lambda c, f: (None if (math.ceil(c / 500) * 500 == 0 or math.ceil(c / 500) * 500 > 8000 or f > 32)
                         else int(cells[(math.ceil(c / 500) - 1) * 33 + f]))


def test_hedge_frozen_cells(lib):  # tests/test_maps.cpp:152-162
    h = _hedge(lib, 1)
    assert h(4000, 32) == 1  # Recompute
    assert h(4000, 1) == 0   # LoadBack
    assert h(4000, 0) == 0


def test_hedge_monotone_in_freed(lib):  # tests/test_maps.cpp:164-175
    for cpa in (1, 0):
        cells = lib.build_hedging_map(M, G, 500, 8000, cpa).reshape(16, 33)
        for row in cells:
            first = np.argmax(row) if row.any() else 33
            assert row[first:].all()


def test_hedge_lookup_roundup(lib):  # tests/test_maps.cpp:177-182
    h = _hedge(lib, 1)
    cells = lib.build_hedging_map(M, G, 500, 8000, 1)
    assert h(4200, 3) == cells[(4500 // 500 - 1) * 33 + 3]
    assert h(8200, 3) is None
    assert h(4000, 33) is None


def test_cpt_hedge_weighs_full_prompt(lib):  # tests/test_maps.cpp:184-194
    cpa, cpt = _hedge(lib, 1), _hedge(lib, 0)
    assert cpa(4000, 16) == 1
    assert cpt(4000, 16) == 0
    assert cpt(4000, 32) == 1


def test_map_rejects_tiny_gpu(lib):  # tests/test_maps.cpp:231-236
    tiny = default_gpu()
    tiny.capacity_bytes = 1 * GIB
    with pytest.raises(ValueError):
        lib.build_offloading_map(M, tiny, default_grid(), 1)


def test_finalize_nearest_rank(lib):  # tests/test_metrics.cpp:37-50
    s = np.array([i / 1000.0 for i in range(1, 101)])
    p50, p90, p99, mean = lib.finalize(s)
    assert approx(p50, 0.050, 1e-5 * 100) and approx(p90, 0.090, 1e-3) and approx(p99, 0.099, 1e-3)
    assert p50 == s[49] and p90 == s[89] and p99 == s[98]
    assert approx(mean, 0.0505, 1e-6)
    with pytest.raises(ValueError):
        lib.finalize(np.zeros(0))


def test_uncontended_serving_timeline(lib):  # tests/test_engine.cpp:61-68 (serving side: 128 samples)
    a = np.array([0.0])
    r = lib.replay_serving(M, G, a, np.array([1000], np.uint32), np.array([128], np.uint32))
    assert r["summary"]["generated_tokens"] == 128 and len(r["samples"]) == 128
    assert r["summary"]["peak_device_bytes"] == M.weights_bytes + G.runtime_reserve_bytes + lib.serving_memory(M, 1128, 1)[0]


def test_empty_trace(lib):  # tests/test_engine.cpp:54-59 (ServingOnly)
    r = lib.replay_serving(M, G, np.zeros(0), np.zeros(0, np.uint32), np.zeros(0, np.uint32))
    assert r["summary"]["generated_tokens"] == 0
    assert r["summary"]["peak_device_bytes"] == M.weights_bytes + G.runtime_reserve_bytes


def test_oversized_query_refused(lib):  # tests/test_engine.cpp:298-301
    with pytest.raises(ValueError):
        lib.replay_serving(M, G, np.array([0.0]), np.array([70000], np.uint32), np.array([128], np.uint32))


def test_generate_trace_statistics(lib):  # tests/test_workload.cpp:28-63 (count and mean gap)
    a, p, o = lib.generate_trace(2.0, 5000.0, ("fixed", 1000), 123)
    assert abs(len(a) - 10000) < 4 * math.sqrt(10000)
    gaps = np.diff(np.concatenate([[0.0], a]))
    assert abs(gaps.mean() - 0.5) < 0.02
    assert (o == 128).all() and (p == 1000).all()
    a2, _, _ = lib.generate_trace(2.0, 5000.0, ("fixed", 1000), 123)
    assert (a == a2).all()  # determinism, tests/test_workload.cpp:18-26
