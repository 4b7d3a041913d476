"""Latency-model mirror (paper_2511_02237_b200/latency.py) pinned against the
reference's own fit_linear / expected_active_experts (latency.cpp, compiled
into oracle/_ref) and the latency CSV schema of io.cpp:174-237."""
import math
import os

import numpy as np
import pytest

import oracle
from paper_2511_02237_b200 import latency as lat

needs_ref = pytest.mark.skipif(not oracle.reference_available(),
                               reason="oracle/_ref not built (no /root/reference here)")


@needs_ref
@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_fit_linear_matches_reference(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 200))
    T = rng.integers(1, 129, size=n)
    us = 20.0 + 1.44 * T + rng.normal(0, 2.0, size=n)
    obs = [lat.LatencyObservation(int(t), float(u)) for t, u in zip(T, us)]
    fit = lat.fit_linear(obs)
    ref = oracle.Reference().fit_linear(T, us)
    got = (fit.b_us, fit.intercept_us, fit.r_squared, fit.residual_std, fit.slope_stderr,
           fit.intercept_stderr)
    for g, r in zip(got, ref):
        assert math.isclose(g, r, rel_tol=1e-12, abs_tol=1e-12), (got, ref)


@needs_ref
@pytest.mark.parametrize("N,k,B", [(128, 8, 1), (128, 8, 16), (128, 4, 256), (16, 2, 3)])
def test_expected_active_experts_matches_reference(N, k, B):
    assert lat.expected_active_experts(N, k, B) == oracle.Reference().expected_active_experts(N, k, B)


def test_fit_linear_errors():
    with pytest.raises(ValueError, match="need at least 2 observations"):
        lat.fit_linear([lat.LatencyObservation(3, 1.0)])
    with pytest.raises(ArithmeticError, match="degenerate design"):
        lat.fit_linear([lat.LatencyObservation(3, 1.0), lat.LatencyObservation(3, 2.0)])
    with pytest.raises(ValueError):
        lat.expected_active_experts(8, 9, 1)


def test_latency_csv_round_trip(tmp_path):
    obs = [lat.LatencyObservation(51, 87.25), lat.LatencyObservation(82, 125.0625)]
    p = os.path.join(tmp_path, "lat.csv")
    lat.write_latency_csv(p, obs)
    assert open(p).read().splitlines()[0] == "T,latency_us"
    back = lat.read_latency_csv(p)
    assert [(o.active_experts, o.latency_us) for o in back] == [(51, 87.25), (82, 125.0625)]
    bad = os.path.join(tmp_path, "bad.csv")
    open(bad, "w").write("X,Y\n1,2\n")
    with pytest.raises(ValueError, match="must contain columns"):
        lat.read_latency_csv(bad)


def test_svg_renders():
    obs = [lat.LatencyObservation(t, 10 + 1.5 * t) for t in (8, 30, 51, 82, 128)]
    svg = lat.latency_svg(obs, lat.fit_linear(obs), "test")
    assert svg.startswith("<svg") and "R²" in svg
