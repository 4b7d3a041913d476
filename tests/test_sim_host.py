"""Host logic of the simulator / sweep (no GPU): latency model, aggregates,
the default sweep grid, Pareto selection vs the compiled reference, and the
sweep CSV round trip (sweep.cpp:48-228, simulate.cpp:56-121, latency.cpp)."""
import math

import numpy as np
import pytest

import oracle
from paper_2511_02237_b200 import routing as R
from paper_2511_02237_b200 import sim as S


def test_latency_model():
    p = S.LatencyParams(0.05, 2.0)
    assert S.expert_latency(0, p) == 0.0
    assert S.expert_latency(3, p) == 0.05 * 3 + 2.0
    with pytest.raises(R.InvalidArgument):
        S.expert_latency(-1, p)
    loads = np.array([0, 2, 0, 5], np.int32)
    assert S.moe_latency(loads, p) == (0.05 * 2 + 2.0) + (0.05 * 5 + 2.0)


def test_aggregates_ratios():
    recs = [S.StepRecord(0, s, 10 + s, 100, 5.0 + s) for s in range(4)]
    van = [S.StepRecord(0, s, 20, 128, 10.0) for s in range(4)]
    a = S._aggregates(recs, van)
    assert a.mean_active_experts == 11.5 and a.vanilla_mean_active_experts == 20.0
    assert a.normalized_active_experts == 11.5 / 20.0
    assert a.mean_divergence is None
    z = S._aggregates([S.StepRecord()], [S.StepRecord()])
    assert math.isnan(z.normalized_latency)


def test_default_sweep_grid_shape():
    g = S.default_sweep_grid(128, 8)
    assert len(g) == 673 and g[0].mode == R.RoutingMode.Vanilla and g[0].k == 8
    oea_pts = g[1:]
    assert {c.k0 for c in oea_pts} == set(range(4, 9))
    assert {c.p for c in oea_pts} == {i / 10.0 for i in range(4, 11)}
    assert {c.max_p for c in oea_pts} == {8, 16, 32, 128}
    assert all(c.k_max >= c.k0 for c in oea_pts)
    with pytest.raises(R.InvalidArgument):
        S.default_sweep_grid(4, 8)


@pytest.mark.skipif(not oracle.reference_available(), reason="oracle/_ref not built")
def test_pareto_matches_reference():
    rng = np.random.default_rng(4)
    for trial in range(20):
        n = int(rng.integers(1, 40))
        t = np.round(rng.uniform(10, 60, n), 1)
        q = np.where(rng.random(n) < 0.2, np.nan, np.round(rng.uniform(0, 0.3, n), 3))
        pts = [S.SweepPoint(R.RoutingConfig.vanilla(8), float(a), None if math.isnan(b) else float(b))
               for a, b in zip(t, q)]
        assert sorted(S.pareto_indices(pts)) == sorted(oracle.Reference().pareto_indices(t, q))
        front = S.pareto_frontier(pts)
        assert [p.mean_active_experts for p in front] == sorted(p.mean_active_experts for p in front)


def test_sweep_csv_round_trip(tmp_path):
    pts = [S.SweepPoint(c, 10.0 + i / 3, None if i % 2 else i / 7, bool(i % 3 == 0))
           for i, c in enumerate(S.default_sweep_grid(16, 4)[:12])]
    path = str(tmp_path / "sweep.csv")
    S.write_sweep_csv(path, pts)
    back = S.read_sweep_csv(path)
    assert [(b.config, b.mean_active_experts, b.quality_delta, b.rounded) for b in back] == \
           [(p.config, p.mean_active_experts, p.quality_delta, p.rounded) for p in pts]
    assert open(path).readline().strip() == \
        "mode,k,k0,p,k_max,max_p,cap,mean_active_experts,quality_delta,rounded"


def test_round_half_away_from_zero():
    assert S._round_half_away(2.5) == 3.0 and S._round_half_away(-2.5) == -3.0
    assert S._round_half_away(0.49999999999999994) == 0.0
