"""CPU: the C-ABI library loads and exports every symbol include/oea_cuda.h
declares; its host-side logic (config resolution, validation) matches the
reference's messages; and without a GPU the product fails loudly (there is
no CPU fallback). No kernels are launched here."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
import paper_2511_02237_b200 as oea
from paper_2511_02237_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "oea_cuda.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|int64_t|const char\*)\s+(oea_\w+)\s*\(",
                                 text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_capi.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(_capi.EXPORTED), set(syms) ^ set(_capi.EXPORTED)
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}\b", out), s


def test_abi_version_and_sm100_code():
    lib = _capi.lib()
    assert lib.oea_abi_version() == 1
    sass = subprocess.run(["cuobjdump", "-lelf", _capi.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "sm_100a" in sass


def test_config_resolution_matches_reference_messages():
    R = oea.RoutingConfig
    cases = [R.vanilla(0), R.vanilla(5), R.pruned(0, 1.0, 1), R.pruned(2, 0.0, 2),
             R.pruned(2, 1.2, 2), R.oea(3, 1.0, 2, 4, 3), R.oea(2, 1.0, 2, 5, 2)]
    for c in cases:
        with pytest.raises(oea.InvalidArgument) as ours:
            c.resolved(4)
        with pytest.raises(oracle.OracleInvalidArgument) as theirs:
            oracle.resolve(c, 4)
        assert str(ours.value) == str(theirs.value)
    assert R.oea(2, 1.0, 2, 0, 2).resolved(4).max_p == 4
    s = R.simplified(2, 3).resolved(4)
    assert (s.p, s.k_max, s.max_p) == (1.0, 3, 4)
    with pytest.raises(oea.InvalidArgument, match="expert count must be >= 1"):
        R.vanilla(1).resolved(0)


def test_plan_set_stride():
    R = oea.RoutingConfig
    assert oea.plan_set_stride(R.vanilla(8).resolved(128)) == 8
    assert oea.plan_set_stride(R.pruned(3, 1.0, 8).resolved(128)) == 3
    assert oea.plan_set_stride(R.simplified(4, 8).resolved(128)) == 8
    assert oea.plan_set_stride(R.simplified(4, 8, oea.CapSemantics.PseudocodeStrict).resolved(128)) == 9


def test_mode_strings_round_trip():
    for m in oea.RoutingMode:
        assert oea.routing_mode_from_string(oea.to_string(m)) == m
    for c in oea.CapSemantics:
        assert oea.cap_semantics_from_string(oea.to_string(c)) == c
    with pytest.raises(oea.InvalidArgument):
        oea.routing_mode_from_string("bogus")


def test_score_matrix_validate_messages():
    # test_routing.cpp:304-323
    m = oea.ScoreMatrix(np.array([[0.5, 0.5, 0.0], [0.2, -0.1, 0.9]]))
    with pytest.raises(oea.InvalidArgument, match="row 1"):
        m.validate()
    with pytest.raises(oea.InvalidArgument, match="off the simplex"):
        oea.ScoreMatrix(np.array([[0.5, 0.3, 0.1]])).validate()
    with pytest.raises(oea.InvalidArgument, match="mask length"):
        oea.ScoreMatrix(np.array([[0.5, 0.5]]), np.array([True, False])).validate()
    ok = oea.ScoreMatrix(np.array([[0.5, 0.3, 0.15, 0.05], [0.25] * 4]), np.array([True, False]))
    ok.validate()
    assert ok.real_count() == 1


def test_batch_stats_host_recount():
    plan = oea.RoutingPlan(sets=[[0, 2], [2, 0], []], weights=[[0.5, 0.5], [0.5, 0.5], []],
                           n_experts=4)
    st = oea.batch_stats(plan)
    assert st.active_count == 2 and st.total_load == 4 and list(st.loads) == [2, 0, 2, 0]


def test_no_gpu_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    with pytest.raises(oea.OeaError, match="no CUDA device|sm_100"):
        oea.Context(0)
    with pytest.raises(oea.OeaError):
        oea.route(np.full((1, 4), 0.25), oea.RoutingConfig.vanilla(2))


def test_ep_owner_blocks():
    lib = _capi.lib()
    for N, P in [(128, 2), (128, 8), (10, 4)]:
        owners = [lib.oea_ep_owner(N, P, e) for e in range(N)]
        assert owners == sorted(owners) and owners[0] == 0 and owners[-1] == P - 1
        for r in range(P):
            lo, hi = N * r // P, N * (r + 1) // P
            assert owners[lo:hi] == [r] * (hi - lo)


def test_device_layer_header_compiles(tmp_path):
    """include/oea/device_layer.hpp is self-contained C++17 over oea_cuda.h
    (no Eigen, no CUDA headers needed by a caller)."""
    import subprocess
    src = tmp_path / "t.cpp"
    src.write_text('#include "oea/device_layer.hpp"\n'
                   "int main() { auto r = oea::device::Routing::simplified(4, 8); return r.c.k0 - 4; }\n")
    inc = os.path.join(ROOT, "include")
    r = subprocess.run(["g++", "-std=c++17", "-Wall", "-Wextra", "-Werror", "-fsyntax-only",
                        "-I", inc, str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
