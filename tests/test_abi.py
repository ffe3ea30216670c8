"""The C-ABI library loads, exports every symbol include/colo_abi.h declares,
and its host-only entry points (no GPU needed) agree with the oracle."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from oracle.oracle import OracleLib, default_gpu, default_model, phi14b_model, sharegpt_histogram
from paper_2503_01066_b200 import _lib, colosim as cs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "colo_abi.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = set(re.findall(r"^[A-Za-z_][\w\s\*]*?\b(colo_\w+)\s*\(", text, flags=re.M))
    return sorted(n for n in names if not n.startswith("colo_V_"))


def test_header_declarations_are_exported():
    L = _lib.lib()
    decl = declared_functions()
    assert len(decl) >= 30
    missing = [n for n in decl if not hasattr(L, n)]
    assert not missing, missing
    assert sorted(_lib.EXPORTS) == decl


def test_dynamic_symbol_table():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    syms = set(re.findall(r"\bT (colo_\w+)", out))
    assert set(declared_functions()) <= syms


def test_abi_version_and_struct_sizes():
    assert _lib.lib().colo_abi_version() == 1
    assert C.sizeof(_lib.Model) == 96 and C.sizeof(_lib.Gpu) == 32 and C.sizeof(_lib.Grid) == 48
    assert cs.TUPLE_DTYPE.itemsize == 16 and cs.BATCH_DTYPE.itemsize == 40


def test_profile_hash_matches_oracle():
    orc = OracleLib("oracle")
    for m, om in ((cs.ModelProfile(), default_model()), (cs.ModelProfile.phi14b_like(), phi14b_model())):
        assert cs.profile_hash(m, cs.GpuProfile()) == orc.profile_hash(om, default_gpu())
    m2 = cs.ModelProfile(prefill_coef_quad=4e-8)
    assert cs.profile_hash(m2, cs.GpuProfile()) != cs.profile_hash(cs.ModelProfile(), cs.GpuProfile())


def test_validation_errors():
    cs.validate_profile_pair(cs.ModelProfile(), cs.GpuProfile())
    with pytest.raises(cs.ColoValidationError):
        cs.validate_profile_pair(cs.ModelProfile(), cs.GpuProfile(capacity_bytes=16 * cs.GIB))
    with pytest.raises(cs.ColoValidationError):
        cs.validate_profile_pair(cs.ModelProfile(num_layers=0), cs.GpuProfile())
    with pytest.raises(cs.ColoValidationError):
        cs.validate_grid(cs.GridSteps(), cs.GridBounds(max_incoming_tokens=8100))
    cs.validate_grid(cs.GridSteps(), cs.GridBounds())


def test_generate_trace_bit_exact():
    z = np.load(os.path.join(ROOT, "tests", "golden", "workload.npz"))
    hv, hp = cs.sharegpt_histogram()
    for seed in (7, 41):
        a, p, o = cs.generate_trace(1.7, 300.0, ("histogram", hv, hp), seed, ("fixed", 0.01))
        assert (a == z[f"hist_{seed}_a"]).all() and (p == z[f"hist_{seed}_p"]).all() and (o == 128).all()
    a, p, _ = cs.generate_trace(0.14, 2000.0, ("uniform", 4000, 7000), 5, ("uniform", 0.0, 1.0), min_tokens=4000)
    assert (a == z["unif_a"]).all() and (p == z["unif_p"]).all()
    with pytest.raises(cs.ColoValidationError):
        cs.generate_trace(0.0, 10.0, ("fixed", 10), 1)
    with pytest.raises(cs.ColoValidationError):
        cs.generate_trace(1.0, 10.0, ("histogram", [1.0, 2.0], [0.5, 0.6]), 1)


def test_hist_select_and_rank():
    L = _lib.lib()
    h = np.array([0, 3, 0, 5, 2], np.uint64)
    b, r = C.c_uint32(), C.c_uint64()
    assert L.colo_hist_select(h.ctypes.data, 5, 4, C.byref(b), C.byref(r)) == 0 and (b.value, r.value) == (3, 1)
    assert L.colo_hist_select(h.ctypes.data, 5, 10, C.byref(b), C.byref(r)) == 0 and (b.value, r.value) == (4, 2)
    assert L.colo_hist_select(h.ctypes.data, 5, 11, C.byref(b), C.byref(r)) == _lib.COLO_EINVAL
    for n in (1, 2, 99, 100, 101, 641536, 10**12 + 7):
        for q in (0.5, 0.9, 0.99):
            import math
            assert cs.nearest_rank_index(q, n) == max(1, math.ceil(q * float(n)))


def test_context_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(cs.ColoError):
        cs.Context(0)
    h = C.c_void_p()
    assert _lib.lib().colo_ctx_create(0, C.byref(h)) == _lib.COLO_ECUDA


def test_generate_trace_label_delays_match_reference_fixture():
    """The label-delay output of colo_generate_trace (workload.hpp:118-120, 214-216)
    against the golden colocated fixtures written by the reference."""
    z = np.load(os.path.join(ROOT, "tests", "golden", "colocated.npz"))
    a, p, o, ld = cs.generate_trace(0.14, 1200.0, ("uniform", 4000, 7000), 5, ("uniform", 0.0, 30.0), with_labels=True)
    assert np.array_equal(a, z["long_q014_cpa_t5_a"]) and np.array_equal(ld.view(np.uint64),
                                                                           z["long_q014_cpa_t5_ld"].view(np.uint64))
    _, _, _, none = cs.generate_trace(0.3, 100.0, ("fixed", 100), 3, None, with_labels=True)
    assert (none == -1.0).all()


def test_trace_hash_matches_reference_report():
    """colo_trace_hash == Trace::content_hash (workload.hpp:140-161): the hash the
    reference CLI printed for tests/golden/cli/small.config's trace."""
    import json

    from paper_2503_01066_b200 import experiment as ex

    cli = os.path.join(ROOT, "tests", "golden", "cli")
    want = json.loads(json.load(open(os.path.join(cli, "expected.json")))["run_colocated"]["report.jsonl"]["head"][0])
    cwd = os.getcwd()
    os.chdir(cli)
    try:
        tr = ex.ExperimentConfig.from_file("small.config").trace_spec.realize()
    finally:
        os.chdir(cwd)
    assert tr.content_hash() == want["trace_hash"]
    # NaN and negative label delays are both nullopt (-1.0 in the hash)
    t2 = ex.Trace(tr.arrival, tr.prompt, tr.output, np.where(tr.label_delay < 0, np.nan, tr.label_delay), tr.query_id)
    assert t2.content_hash() == tr.content_hash()


def test_json_doubles_match_nlohmann_dump():
    """colo_json_doubles uses the reference's JSON library; a value where its
    Grisu2 output is not the shortest round trip stays 17 digits."""
    from paper_2503_01066_b200 import experiment as ex

    assert ex.json_doubles([0.020685999999997762, 0.5, 1e-05, 2.0]) == "0.020685999999997762,0.5,1e-05,2.0"
    assert repr(0.020685999999997762) == "0.02068599999999776"  # Python's shortest form differs
