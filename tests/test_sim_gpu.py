"""GPU-backed simulator vs the reference's own
simulate_decode / padding_experiment compiled from its sources
(oracle/_ref): identical records (T, total load, modeled latency) and
aggregates; the writers' formats follow simulate.cpp:263-343."""
import json

import numpy as np
import pytest

import oracle
from paper_2511_02237_b200 import scoregen as G
from paper_2511_02237_b200 import sim as S
from paper_2511_02237_b200 import traces as T

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not oracle.reference_available(), reason="oracle/_ref not built")

LAT = S.LatencyParams(0.05, 2.0)


@needs_ref
@pytest.mark.parametrize("kind,kw", [("dirichlet", dict(alpha=0.3)), ("dirichlet", dict(alpha=1.0)),
                                     ("clustered", dict(groups=4, conc=4.0, spread=2.0))])
@pytest.mark.parametrize("cfg_name", ["simplified", "oea", "pruned"])
def test_simulate_decode_matches_reference(oea, kind, kw, cfg_name):
    cfg = {"simplified": oea.RoutingConfig.simplified(4, 8),
           "oea": oea.RoutingConfig.oea(2, 0.7, 8, 64, 8),
           "pruned": oea.RoutingConfig.pruned(3, 0.8, 8)}[cfg_name]
    gen = G.ScoreGenConfig(G.GenKind.Dirichlet if kind == "dirichlet" else G.GenKind.Clustered,
                           n_experts=128, batch=16, steps=6, layers=4, seed=31,
                           alpha=kw.get("alpha", 1.0), groups=kw.get("groups", 2),
                           within_group_concentration=kw.get("conc", 4.0),
                           between_group_spread=kw.get("spread", 2.0))
    tr = S.simulate_decode(gen, cfg, LAT)
    rT, rl, rlat, vT, vl, vlat, agg = oracle.Reference().simulate_decode(
        kind, 128, 16, 6, 4, 31, cfg, LAT.a_us, LAT.b_us, **kw)
    assert [r.active_experts for r in tr.records] == rT.tolist()
    assert [r.total_load for r in tr.records] == rl.tolist()
    assert [r.modeled_latency_us for r in tr.records] == rlat.tolist()
    assert [r.active_experts for r in tr.vanilla_records] == vT.tolist()
    assert [r.modeled_latency_us for r in tr.vanilla_records] == vlat.tolist()
    a = tr.aggregates
    got = [a.mean_active_experts, a.mean_total_load, a.mean_latency_us,
           a.vanilla_mean_active_experts, a.vanilla_mean_total_load, a.vanilla_mean_latency_us,
           a.normalized_active_experts, a.normalized_latency]
    assert got == agg.tolist()
    assert [(r.step, r.layer) for r in tr.records][:5] == [(0, 0), (0, 1), (0, 2), (0, 3), (1, 0)]


@needs_ref
def test_padding_experiment_matches_reference(oea):
    cfg = oea.RoutingConfig.simplified(4, 8)
    gen = G.ScoreGenConfig(G.GenKind.Dirichlet, n_experts=128, batch=12, steps=4, layers=3,
                           seed=8, alpha=0.5)
    rep = S.padding_experiment(gen, cfg, 16, LAT)
    Tr, lr, latr, match = oracle.Reference().padding_experiment(
        "dirichlet", 128, 12, 4, 3, 8, cfg, 16, LAT.a_us, LAT.b_us, alpha=0.5)
    for i, v in enumerate((rep.no_padding, rep.naive_padding, rep.masked_padding)):
        assert [r.active_experts for r in v.records] == Tr[i].tolist(), v.name
        assert [r.total_load for r in v.records] == lr[i].tolist(), v.name
        assert [r.modeled_latency_us for r in v.records] == latr[i].tolist(), v.name
    assert rep.masked_matches_no_padding is match is True
    assert rep.naive_padding.mean_active_experts >= rep.no_padding.mean_active_experts


def test_uniform_vanilla_closed_form(oea):
    # test_sim.cpp:198-215: mean T of vanilla top-8 on Dirichlet(1) scores
    gen = G.ScoreGenConfig(G.GenKind.Dirichlet, n_experts=128, batch=16, steps=200, layers=1,
                           seed=31, alpha=1.0)
    tr = S.simulate_decode(gen, oea.RoutingConfig.vanilla(8), S.LatencyParams(0.05, 2.0))
    Ts = np.array([r.active_experts for r in tr.records], float)
    se = np.sqrt(Ts.var(ddof=1) / len(Ts))
    assert abs(Ts.mean() - oracle.expected_active_experts(128, 8, 16)) <= 3.0 * se
    assert all(a == b for a, b in zip(tr.records, tr.vanilla_records))
    assert tr.aggregates.normalized_active_experts == 1.0


def test_replay_and_writers(oea, tmp_path):
    gen = G.ScoreGenConfig(G.GenKind.Dirichlet, n_experts=64, batch=8, steps=3, layers=2,
                           seed=4, alpha=0.4)
    cfg, cells = S.cell_scores(gen)
    recs = [T.ScoreRecord(i // 2, i % 2, m) for i, m in enumerate(cells)]
    path = str(tmp_path / "trace.ndjson")
    T.write_score_trace(path, recs[::-1])  # order in the file does not matter
    replay = G.ScoreGenConfig(G.GenKind.Replay, steps=3, layers=2, trace_path=path)
    a = S.simulate_decode(gen, oea.RoutingConfig.simplified(2, 4), LAT)
    b = S.simulate_decode(replay, oea.RoutingConfig.simplified(2, 4), LAT)
    assert a.records == b.records and a.aggregates == b.aggregates
    csv = tmp_path / "trace.csv"
    S.write_trace_csv(str(csv), a)
    lines = csv.read_text().splitlines()
    assert lines[0] == "layer,step,T,total_load,modeled_latency_us" and len(lines) == 7
    r0 = a.records[0]
    assert lines[1] == f"0,0,{r0.active_experts},{r0.total_load},{'%.17g' % r0.modeled_latency_us}"
    sj = tmp_path / "summary.json"
    S.write_trace_summary_json(str(sj), a, gen, LAT)
    j = json.loads(sj.read_text())
    assert j["type"] == "trace_summary" and j["steps_recorded"] == 6
    assert j["score_gen"] == {"kind": "dirichlet", "n_experts": 64, "batch": 8, "steps": 3,
                              "layers": 2, "seed": 4, "alpha": 0.4}
    missing = G.ScoreGenConfig(G.GenKind.Replay, steps=4, layers=2, trace_path=path)
    with pytest.raises(oea.InvalidArgument, match="no record for step 3 layer 0"):
        S.simulate_decode(missing, oea.RoutingConfig.vanilla(4), LAT)


@needs_ref
@pytest.mark.parametrize("rounding", [False, True])
def test_sweep_matches_reference(oea, rounding):
    gen = G.ScoreGenConfig(G.GenKind.Dirichlet, n_experts=64, batch=16, steps=4, layers=2,
                           seed=17, alpha=0.3)
    grid = S.default_sweep_grid(64, 8)
    pts = S.sweep(gen, grid, LAT, S.RoundingRule(enabled=rounding))
    want = oracle.Reference().sweep_default("dirichlet", 64, 16, 4, 2, 17, 8, LAT.a_us,
                                            LAT.b_us, rounding, alpha=0.3)
    assert len(pts) == len(want) == len(grid)
    assert [p.mean_active_experts for p in pts] == want.tolist()
    front = S.pareto_frontier(pts)
    ref_idx = oracle.Reference().pareto_indices([p.mean_active_experts for p in pts],
                                                [float("nan")] * len(pts))
    assert sorted(S.pareto_indices(pts)) == sorted(ref_idx)
    assert front[0].mean_active_experts == min(p.mean_active_experts for p in pts)


def test_sweep_csv_round_trip(oea, tmp_path):
    gen = G.ScoreGenConfig(G.GenKind.Dirichlet, n_experts=32, batch=8, steps=2, layers=1,
                           seed=2, alpha=0.5)
    pts = S.sweep(gen, S.default_sweep_grid(32, 4)[:20], LAT)
    path = str(tmp_path / "sweep.csv")
    S.write_sweep_csv(path, pts)
    back = S.read_sweep_csv(path)
    assert [(b.config, b.mean_active_experts, b.quality_delta) for b in back] == \
           [(p.config, p.mean_active_experts, p.quality_delta) for p in pts]
    bad = tmp_path / "bad.csv"
    bad.write_text("mode,k\n")
    with pytest.raises(oea.InvalidArgument, match="unexpected header"):
        S.read_sweep_csv(str(bad))


@needs_ref
@pytest.mark.parametrize("cfg_name", ["simplified", "oea"])
def test_toy_layer_simulation_matches_reference(oea, cfg_name):
    # simulate.cpp:153-183 on make_random_layer({64, 96, 16}, 7): routed T /
    # load / latency identical, divergence vs vanilla within fp64 rounding
    cfg = {"simplified": oea.RoutingConfig.simplified(2, 4),
           "oea": oea.RoutingConfig.oea(1, 0.6, 4, 16, 4)}[cfg_name]
    layer = oea.DeviceMoeLayer(64, 96, 16, dtype="f64")
    layer.init_random(7)
    gen = G.ScoreGenConfig(G.GenKind.Dirichlet, n_experts=16, batch=6, steps=3, layers=2, seed=5)
    tr = S.simulate_decode_layer(layer, gen, cfg, LAT)
    T_, ld, lat, dv, vT, md = oracle.Reference().simulate_decode_layer(
        64, 96, 16, 7, 6, 3, 2, 5, cfg, LAT.a_us, LAT.b_us)
    assert [r.active_experts for r in tr.records] == T_.tolist()
    assert [r.total_load for r in tr.records] == ld.tolist()
    assert [r.modeled_latency_us for r in tr.records] == lat.tolist()
    assert [r.active_experts for r in tr.vanilla_records] == vT.tolist()
    got = np.array([r.divergence for r in tr.records])
    assert np.allclose(got, dv, rtol=1e-9, atol=1e-12)
    assert abs(tr.aggregates.mean_divergence - md) <= 1e-9 * max(md, 1e-12)


def test_sweep_with_layer_reports_quality(oea):
    layer = oea.DeviceMoeLayer(64, 96, 16, dtype="f64")
    layer.init_random(3)
    gen = G.ScoreGenConfig(G.GenKind.Dirichlet, n_experts=16, batch=4, steps=2, layers=1, seed=1)
    grid = S.default_sweep_grid(16, 4)[:6]
    pts = S.sweep(gen, grid, LAT, layer=layer)
    assert pts[0].config.mode == oea.RoutingMode.Vanilla and pts[0].quality_delta == 0.0
    assert all(p.quality_delta is not None and p.quality_delta >= 0.0 for p in pts)
