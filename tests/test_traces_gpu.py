"""Batched routing of score traces on the GPU:
oea_route_f64_batched_host routes every record with its own union and
aggregates in one launch sequence; each record's plan must equal the
single-record route() bit for bit and the CPU oracle's route()."""
import numpy as np
import pytest

import oracle
from paper_2511_02237_b200 import traces as T

pytestmark = pytest.mark.gpu


def _records(oea, rng, N, n_rec, bmax, masks=True, alpha=0.3):
    recs = []
    for r in range(n_rec):
        B = int(rng.integers(1, bmax + 1))
        sc = rng.dirichlet(np.full(N, alpha), size=B)
        mask = None
        if masks and rng.integers(0, 3) == 0:
            mask = rng.integers(0, 2, size=B).astype(bool)
        recs.append(T.ScoreRecord(r // 4, r % 4, oea.ScoreMatrix(sc, mask)))
    return recs


def _same(a, b):
    return (a.sets == b.sets and a.weights == b.weights and a.active_union == b.active_union
            and a.active_count == b.active_count and a.total_load == b.total_load
            and np.array_equal(a.loads, b.loads))


CFGS = [("vanilla", lambda o, N: o.RoutingConfig.vanilla(min(8, N))),
        ("simplified", lambda o, N: o.RoutingConfig.simplified(min(4, N), min(8, N))),
        ("strict", lambda o, N: o.RoutingConfig.simplified(min(2, N), min(6, N), o.CapSemantics.PseudocodeStrict)),
        ("pruned", lambda o, N: o.RoutingConfig.pruned(min(3, N), 1.0, min(8, N))),
        ("oea_p", lambda o, N: o.RoutingConfig.oea(min(2, N), 0.6, min(6, N), N, min(6, N))),
        ("oea_maxp", lambda o, N: o.RoutingConfig.oea(min(2, N), 1.0, min(6, N), max(1, N // 2), min(6, N)))]


@pytest.mark.parametrize("N", [16, 64, 128, 200])
@pytest.mark.parametrize("name,mk", CFGS)
def test_batched_equals_per_record(oea, N, name, mk):
    rng = np.random.default_rng(N * 7 + len(name))
    recs = _records(oea, rng, N, 37, 40)
    cfg = mk(oea, N)
    got = T.route_trace(recs, cfg)
    assert len(got) == len(recs)
    for q, (r, g) in enumerate(zip(recs, got)):
        single = oea.route(r.scores, cfg)
        assert _same(g, single), f"record {q}"
        w = oracle.route(r.scores.scores, cfg, r.scores._mask_u8())
        B = r.scores.batch()
        assert g.sets == [w.set_list(i) for i in range(B)], f"record {q} vs oracle"
        assert g.weights == [[float(v) for v in w.weights[i, : w.set_len[i]]] for i in range(B)]
        assert g.active_count == w.active_count and g.total_load == w.total_load


def test_cli_uniform16_example(oea):
    # test_cli.cpp:80-102: equal scores tie-break to the lowest indices
    recs = [T.ScoreRecord(0, 0, oea.ScoreMatrix(np.full((1, 16), 1.0 / 16.0)))]
    doc = T.routing_plans_json(recs, oea.RoutingConfig.vanilla(8))
    assert doc["routing"]["mode"] == "vanilla" and doc["routing"]["k"] == 8
    plan = doc["records"][0]["plan"]
    assert plan["active_experts"] == 8 and plan["total_load"] == 8
    assert plan["active_union"] == list(range(8))
    assert len(plan["tokens"][0]["experts"]) == 8


def test_trace_file_to_plans(oea, tmp_path):
    rng = np.random.default_rng(3)
    recs = _records(oea, rng, 128, 64, 16)
    p = str(tmp_path / "trace.ndjson")
    T.write_score_trace(p, recs)
    back = T.read_score_trace(p)
    cfg = oea.RoutingConfig.simplified(4, 8)
    doc = T.routing_plans_json(back, cfg)
    assert len(doc["records"]) == 64
    for rec, r in zip(doc["records"], back):
        single = oea.route(r.scores, cfg)
        assert rec["plan"]["active_union"] == single.active_union
        assert [t["experts"] for t in rec["plan"]["tokens"]] == single.sets


def test_degenerate_mass_names_record(oea):
    good = oea.ScoreMatrix(np.full((2, 4), 0.25))
    # token 1 of record 1: all-zero scores, so its top-2 set has zero mass
    bad = oea.ScoreMatrix(np.array([[0.25] * 4, [0.0] * 4]))
    with pytest.raises(oea.DomainError) as e:
        oea.route_batched([good, bad], oea.RoutingConfig.vanilla(2))
    assert "record 1" in str(e.value) and "token 1" in str(e.value)


def test_large_trace_one_call(oea):
    # C5-sized: 256 records x 16 tokens x 128 experts
    rng = np.random.default_rng(11)
    recs = [oea.ScoreMatrix(rng.dirichlet(np.full(128, 0.3), size=16)) for _ in range(256)]
    cfg = oea.RoutingConfig.simplified(4, 8)
    got = oea.route_batched(recs, cfg)
    for q in (0, 17, 255):
        assert _same(got[q], oea.route(recs[q], cfg))
    Ts = np.array([p.active_count for p in got])
    assert 40 <= Ts.mean() <= 60
