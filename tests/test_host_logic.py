"""Host-side logic of the Python mirror (no GPU): map views and lookups over
cell arrays, verdict decoding, the exact-stats radix-select protocol."""
import math
import os

import numpy as np
import pytest
import torch

from oracle.oracle import OracleLib, TUPLE_DTYPE, default_grid, default_gpu, default_model
from paper_2503_01066_b200 import colosim as cs


class FakeSet:
    """Stands in for a device MapSet: same attributes, cells from the oracle."""

    def __init__(self, orc, cpa=1):
        self.model, self.gpu = cs.ModelProfile(), cs.GpuProfile()
        self.steps, self.bounds = cs.GridSteps(), cs.GridBounds()
        self.mode = cs.TrainingMode(cpa)
        self.hedge_step, self.hedge_max, self.assumed_output_tokens = 500, 8000, 128
        self.profile_hash_value = cs.profile_hash(self.model, self.gpu)
        self._c = (orc.build_offloading_map(default_model(), default_gpu(), default_grid(), cpa),
                   orc.build_hedging_map(default_model(), default_gpu(), 500, 8000, cpa))

    def cells(self):
        return self._c


@pytest.fixture(scope="module")
def orc():
    return OracleLib("oracle")


def test_offload_lookup_mirror(orc):  # tests/test_maps.cpp:122-139 through the mirror
    om = cs.OffloadingMap(FakeSet(orc))
    assert om.lookup(4000, 420, 5) == om.cell(8, 0, 0)
    assert om.lookup(4000, 500, 6) == om.cell(8, 0, 1)
    assert om.lookup(4000, 1000, 5) == om.cell(8, 1, 0)
    assert om.lookup(8001, 500, 5) is None
    assert om.lookup(4000, 8001, 5) is None
    assert om.lookup(4000, 500, 51) is None
    assert om.lookup(4000, 0, 5) is None and om.lookup(0, 500, 5) is not None
    assert om.cell(8, 3, 1) == cs.OffloadDecision(cs.OffloadAction.FreeLayers, 6)  # (4000,2000,10)
    assert (om.cached_count(), om.incoming_count(), om.batch_count()) == (17, 16, 10)


def test_hedge_lookup_mirror(orc):  # tests/test_maps.cpp:152-194 through the mirror
    hm = cs.HedgingMap(FakeSet(orc))
    assert hm.lookup(4000, 32) == cs.HedgeDecision.Recompute
    assert hm.lookup(4000, 1) == cs.HedgeDecision.LoadBack
    assert hm.lookup(4200, 3) == hm.cell(8, 3)
    assert hm.lookup(8200, 3) is None and hm.lookup(4000, 33) is None and hm.lookup(0, 3) is None
    assert cs.HedgingMap(FakeSet(orc, 0)).lookup(4000, 16) == cs.HedgeDecision.LoadBack


def test_map_save_format(orc, tmp_path):  # maps.hpp:118-140
    om = cs.OffloadingMap(FakeSet(orc))
    p = tmp_path / "offload_cpa.map"
    om.save(str(p))
    lines = p.read_text().splitlines()
    assert lines[:3] == ["version 1", "kind offload", "mode cpa"]
    assert lines[3] == f"profile_hash {cs.profile_hash(cs.ModelProfile(), cs.GpuProfile())}"
    assert len(lines) == 11 + 2720
    assert "4000,2000,10,free:6" in lines


def test_verdict_decoding(orc):
    t = np.zeros(3, TUPLE_DTYPE)
    t[0] = (4000, 2000, 0, 10, 0, 32)     # FreeLayers(6) -> hedge
    t[1] = (4000, 500, 0, 5, 0, 32)       # NoAction
    t[2] = (9000, 500, 9000, 5, 0, 32)    # offload out of range -> AllToHost + forced Recompute
    v = orc.decide(default_model(), default_gpu(), default_grid(), 1, t)
    f = cs.verdict_fields(v)
    assert list(f["action"]) == [1, 0, 2] and f["layers"][0] == 6 and f["free_now"][0] == 6
    assert list(f["verdict"]) == [f["verdict"][0], 0, 2] and f["offload_oor"][2] == 1 and f["recompute"][2] == 1
    assert f["stream"][2] == 1 and f["stream_oor"][2] == 1


def test_pack_tuples_layout():
    t = cs.pack_tuples(torch.tensor([1, 2]), torch.tensor([3, 4]), torch.tensor([5, 6]), torch.tensor([7, 65535]),
                       torch.tensor([8, 255]), torch.tensor([9, 255]))
    a = t.numpy().view(np.uint32).reshape(-1).view(TUPLE_DTYPE)
    assert list(a["batch"]) == [7, 65535] and list(a["pending"]) == [8, 255] and list(a["dev_layers"]) == [9, 255]
    assert list(a["cached"]) == [1, 2] and list(a["charged"]) == [5, 6]


def numpy_pass(samples_list, flags=0):
    """A stats pass computed from explicit samples (what the replay kernel accumulates);
    ``flags`` is the pass's summary flag word (bit 0: a sample the exact sum could not hold)."""
    bits = np.concatenate(samples_list).view(np.uint64) if samples_list else np.zeros(0, np.uint64)
    samples = bits.view(np.float64)

    def run_pass(hs, fs, prefixes):
        h = torch.zeros(len(prefixes) * cs.HIST_BINS, dtype=torch.int64)
        for f, p in enumerate(prefixes):
            sel = bits[(bits >> np.uint64(fs)) == np.uint64(p)]
            keys = ((sel >> np.uint64(hs)) & np.uint64(cs.HIST_BINS - 1)).astype(np.int64)
            h[f * cs.HIST_BINS:(f + 1) * cs.HIST_BINS] += torch.from_numpy(np.bincount(keys, minlength=cs.HIST_BINS))
        tot = None
        if fs == 63:
            tot = {"generated_tokens": len(samples), "slow_tokens": 0, "slow_queries": 0, "batches": 0, "flags": flags,
                   "exact_sum": sum(int(x) for x in (samples * 2.0**96))}
        return h, tot

    return run_pass


def test_stats_protocol_matches_finalize(orc):
    hv, hp = cs.sharegpt_histogram()
    a, p, o = orc.generate_trace(1.2, 400.0, ("histogram", hv, hp), 9)
    r = orc.replay_serving(default_model(), default_gpu(), a, p, o)
    s = r["samples"]
    out = cs.stats_protocol(numpy_pass([s]))
    p50, p90, p99, mean = orc.finalize(s)
    assert (out["p50"], out["p90"], out["p99"]) == (p50, p90, p99)
    assert abs(out["mean"] - mean) <= 1e-12 * mean
    assert out["generated_tokens"] == len(s)


def test_stats_protocol_edge_cases():
    assert cs.stats_protocol(numpy_pass([]))["p50"] is None
    one = np.array([0.25])
    out = cs.stats_protocol(numpy_pass([one]))
    assert out["p50"] == out["p99"] == 0.25 and out["mean"] == 0.25
    ties = np.array([0.5] * 7 + [0.0] * 3 + [1e-300, 3.0])
    out = cs.stats_protocol(numpy_pass([ties]))
    st = np.sort(ties)
    for q in (0.5, 0.9, 0.99):
        assert out[f"p{int(q * 100)}"] == st[max(1, math.ceil(q * len(st))) - 1]
