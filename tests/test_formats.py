"""File formats around the path, against the reference's
own writers and readers (oracle/_ref): map text files byte-identical to
OffloadingMap::save / HedgingMap::save, loads with profile-hash refusal,
JSON-lines traces read and validated like load_trace, histogram files."""
import ctypes as C
import json
import os

import numpy as np
import pytest

from oracle.oracle import PATHS, Grid, OracleLib, default_gpu, default_grid, default_model, phi14b_model
from paper_2503_01066_b200 import colosim as cs

HAVE_REF = os.path.exists(PATHS["ref"])
G = default_gpu()


@pytest.fixture(scope="module")
def orc():
    return OracleLib("oracle")


def ref_save_maps(m, grid, cpa, off_path, hed_path):
    ref = OracleLib("ref").lib
    rc = ref.ref_save_maps(C.byref(m), C.byref(G), C.byref(grid), C.c_int(cpa), C.c_uint64(128), off_path.encode(),
                           hed_path.encode())
    assert rc == 0


def cs_model(m):
    return cs.ModelProfile(**{f: getattr(m, f) for f, _ in m._fields_})


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
@pytest.mark.parametrize("mname", ["llama8b", "phi14b"])
@pytest.mark.parametrize("cpa", [0, 1])
@pytest.mark.parametrize("step", [500, 250])
def test_map_files_byte_identical(orc, tmp_path, mname, cpa, step):
    m = default_model() if mname == "llama8b" else phi14b_model()
    grid = Grid(step, step, 5, 8000, 8000, 50)
    ro, rh = str(tmp_path / "ref_off.map"), str(tmp_path / "ref_hed.map")
    ref_save_maps(m, grid, cpa, ro, rh)
    off = orc.build_offloading_map(m, G, grid, cpa)
    hed = orc.build_hedging_map(m, G, step, 8000, cpa)
    h = orc.profile_hash(m, G)
    steps, bounds = cs.GridSteps(step, step, 5), cs.GridBounds()
    co, ch = str(tmp_path / "off.map"), str(tmp_path / "hed.map")
    cs.save_map_cells(co, "offload", cs.TrainingMode(cpa), h, m.num_layers, steps, bounds, off)
    cs.save_map_cells(ch, "hedge", cs.TrainingMode(cpa), h, m.num_layers, cs.GridSteps(step, 1, 1),
                      cs.GridBounds(8000, 1, 1), hed)
    assert open(co, "rb").read() == open(ro, "rb").read()
    assert open(ch, "rb").read() == open(rh, "rb").read()
    # and the reference's files load back into the same cells
    hdr, cells = cs.load_map_cells(ro, h)
    assert (cells == off).all() and hdr["kind"] == "offload" and hdr["mode"] == cs.TrainingMode(cpa)
    assert hdr["steps"] == steps and hdr["bounds"] == bounds and hdr["num_layers"] == m.num_layers
    hdr, cells = cs.load_map_cells(rh, h)
    assert (cells == hed).all() and hdr["kind"] == "hedge" and hdr["assumed_output_tokens"] == 128


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
def test_map_load_refusals(orc, tmp_path):  # tests/test_maps.cpp:223-229 and maps.hpp:146-186
    m = default_model()
    ro, rh = str(tmp_path / "o.map"), str(tmp_path / "h.map")
    ref_save_maps(m, default_grid(), 1, ro, rh)
    h = orc.profile_hash(m, G)
    with pytest.raises(cs.ColoValidationError, match="hash"):
        cs.load_map_cells(ro, h + 1)
    text = open(ro).read()
    bad = tmp_path / "bad.map"
    bad.write_text(text.replace("noaction", "nope", 1))
    with pytest.raises(cs.ColoValidationError, match="bad decision token"):
        cs.load_map_cells(str(bad), h)
    bad.write_text(text.replace("version 1", "version 2", 1))
    with pytest.raises(cs.ColoValidationError, match="version"):
        cs.load_map_cells(str(bad), h)
    bad.write_text(text.replace("kind offload", "kind other", 1))
    with pytest.raises(cs.ColoValidationError):
        cs.load_map_cells(str(bad), h)
    with pytest.raises(cs.ColoValidationError, match="cannot open"):
        cs.load_map_cells(str(tmp_path / "missing.map"), h)


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
def test_trace_jsonl_matches_reference(orc, tmp_path):
    ref = OracleLib("ref").lib
    hv, hp = cs.sharegpt_histogram()
    a, p, o = orc.generate_trace(0.7, 800.0, ("histogram", hv, hp), 3)
    ld = np.where(np.arange(len(a)) % 3 == 0, np.nan, np.arange(len(a)) * 0.001)
    path = str(tmp_path / "t.jsonl")
    rc = ref.ref_save_trace(a.ctypes.data_as(C.c_void_p), p.ctypes.data_as(C.c_void_p), o.ctypes.data_as(C.c_void_p),
                            ld.ctypes.data_as(C.c_void_p), C.c_size_t(len(a)), path.encode())
    assert rc == 0
    # shuffle the lines: loading must restore validate_trace's (arrival, id) order
    lines = open(path).read().splitlines()
    rng = np.random.default_rng(0)
    rng.shuffle(lines)
    open(path, "w").write("\n".join(lines) + "\n\n")
    n = len(a)
    ra, rp, ro_, rq, rl = np.empty(n), np.empty(n, np.uint32), np.empty(n, np.uint32), np.empty(n, np.uint64), np.empty(n)
    ref.ref_load_trace.restype = C.c_int64
    rn = ref.ref_load_trace(path.encode(), ra.ctypes.data_as(C.c_void_p), rp.ctypes.data_as(C.c_void_p),
                            ro_.ctypes.data_as(C.c_void_p), rq.ctypes.data_as(C.c_void_p), rl.ctypes.data_as(C.c_void_p),
                            C.c_size_t(n))
    assert rn == n
    ca, cp, co, cq, cl = cs.load_trace(path)
    assert (ca.view(np.uint64) == ra.view(np.uint64)).all() and (cp == rp).all() and (co == ro_).all()
    assert (cq == rq).all() and (np.isnan(cl) == np.isnan(rl)).all() and (cl[~np.isnan(cl)] == rl[~np.isnan(rl)]).all()
    assert (ca.view(np.uint64) == a.view(np.uint64)).all()  # 17-digit JSON doubles round-trip exactly


def test_trace_jsonl_validation(tmp_path):  # workload.hpp:164-188, tests/test_workload.cpp:91-143
    def write(recs):
        path = tmp_path / "x.jsonl"
        path.write_text("\n".join(json.dumps(r) for r in recs) + "\n")
        return str(path)

    ok = write([{"query_id": 1, "arrival_time": 2.0, "prompt_tokens": 10},
                {"query_id": 0, "arrival_time": 2.0, "prompt_tokens": 20, "output_tokens": 7, "label_delay": None}])
    a, p, o, q, ld = cs.load_trace(ok)
    assert list(q) == [0, 1] and list(p) == [20, 10] and list(o) == [7, 128] and np.isnan(ld).all()
    for recs, msg in (([{"query_id": 0, "arrival_time": 1.0, "prompt_tokens": 5},
                        {"query_id": 0, "arrival_time": 2.0, "prompt_tokens": 5}], "duplicate"),
                      ([{"query_id": 0, "arrival_time": -1.0, "prompt_tokens": 5}], "negative"),
                      ([{"query_id": 0, "arrival_time": 1.0, "prompt_tokens": 0}], "prompt_tokens"),
                      ([{"query_id": 0, "arrival_time": 1.0, "prompt_tokens": 5, "output_tokens": 0}], "output_tokens"),
                      ([{"arrival_time": 1.0, "prompt_tokens": 5}], "query_id")):
        with pytest.raises(cs.ColoValidationError, match=msg):
            cs.load_trace(write(recs))
    bad = tmp_path / "bad.jsonl"
    bad.write_text('{"query_id": 0, "arrival_time": 1.0, "prompt_tokens": 5}\n{not json\n')
    with pytest.raises(cs.ColoValidationError, match=":2:"):
        cs.load_trace(str(bad))


def test_histogram_jsonl(tmp_path):  # proj/profiles/sharegpt_like_lengths.jsonl, workload.hpp:274-293
    hv, hp = cs.sharegpt_histogram()
    path = tmp_path / "h.jsonl"
    path.write_text("".join(json.dumps({"tokens": int(v), "probability": float(p)}) + "\n" for v, p in zip(hv, hp)))
    v, p = cs.load_histogram(str(path))
    assert (v == hv).all() and (p == hp).all()
    path.write_text('{"tokens": 64, "probability": 0.5}\n{"tokens": 128, "probability": 0.6}\n')
    with pytest.raises(cs.ColoValidationError, match="sum"):
        cs.load_histogram(str(path))


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
def test_save_trace_matches_reference(orc, tmp_path):
    """save_trace (workload.hpp:256-270): byte-identical file, label_delay null when absent."""
    from paper_2503_01066_b200 import experiment as ex

    ref = OracleLib("ref").lib
    hv, hp = cs.sharegpt_histogram()
    a, p, o = orc.generate_trace(0.7, 800.0, ("histogram", hv, hp), 5)
    ld = np.where(np.arange(len(a)) % 3 == 0, np.nan, np.arange(len(a)) * 0.001)
    rpath, gpath = str(tmp_path / "r.jsonl"), str(tmp_path / "g.jsonl")
    assert ref.ref_save_trace(a.ctypes.data_as(C.c_void_p), p.ctypes.data_as(C.c_void_p),
                              o.ctypes.data_as(C.c_void_p), ld.ctypes.data_as(C.c_void_p), C.c_size_t(len(a)),
                              rpath.encode()) == 0
    ex.save_trace(ex.Trace(a, p, o, ld, np.arange(len(a), dtype=np.uint64)), gpath)
    assert open(gpath, "rb").read() == open(rpath, "rb").read()
