"""Score-trace I/O and the routing_plans document (host logic; no GPU).

Mirrors the reference's trace tests (proj/tests/test_sim.cpp:138-196,
test_cli.cpp:104-118) for read_score_trace / write_score_trace (io.cpp:40-172)
and checks the routing_plans JSON layout (oea_cli.cpp:153-175, json_io.cpp)
on plans produced by the CPU oracle (test infrastructure only)."""
import json

import numpy as np
import pytest

import oracle
from paper_2511_02237_b200 import routing as R
from paper_2511_02237_b200 import traces as T


def dirichlet(rng, B, N, alpha=0.3):
    return rng.dirichlet(np.full(N, alpha), size=B)


def test_round_trip_with_mask(tmp_path):
    # test_sim.cpp:138-157
    rng = np.random.default_rng(21)
    recs = [T.ScoreRecord(s, 0, R.ScoreMatrix(dirichlet(rng, 3, 8))) for s in range(2)]
    recs[1].scores.mask = np.array([True, False, True])
    p = str(tmp_path / "trace.ndjson")
    T.write_score_trace(p, recs)
    back = T.read_score_trace(p)
    assert len(back) == 2
    for a, b in zip(back, recs):
        assert (a.step, a.layer) == (b.step, b.layer)
        assert np.array_equal(a.scores.scores, b.scores.scores)  # %.17g-exact doubles
    assert back[0].scores.mask is None
    assert back[1].scores.mask.tolist() == [True, False, True]
    first = open(p).readline().strip()
    assert first == '{"n_experts":8,"schema_version":1,"type":"score_trace"}'


def test_parse_errors_name_the_record(tmp_path):
    # test_sim.cpp:159-196
    p = tmp_path / "bad_trace.ndjson"
    p.write_text('{"schema_version":1,"type":"score_trace","n_experts":3}\n'
                 '{"step":0,"layer":0,"scores":[[0.5,0.25,0.25]]}\n'
                 '{"step":1,"layer":0,"scores":[[0.9,0.2,0.1]]}\n')
    with pytest.raises(R.InvalidArgument) as e:
        T.read_score_trace(str(p))
    assert "record 1" in str(e.value) and "row 0" in str(e.value)
    h = tmp_path / "headerless.ndjson"
    h.write_text('{"step":0,"layer":0,"scores":[[1.0]]}\n')
    with pytest.raises(R.InvalidArgument, match="score_trace header"):
        T.read_score_trace(str(h))


def test_malformed_rows_name_row_and_record(tmp_path):
    # test_cli.cpp:104-118 (the reader's half)
    p = tmp_path / "bad.ndjson"
    p.write_text('{"schema_version":1,"type":"score_trace","n_experts":2}\n'
                 '{"step":0,"layer":0,"scores":[[0.5,0.5],[-0.1,1.1]]}\n')
    with pytest.raises(R.InvalidArgument) as e:
        T.read_score_trace(str(p))
    assert "row 1" in str(e.value) and "record 0" in str(e.value)


@pytest.mark.parametrize("body,frag", [
    ("", "is empty"),
    ('{"schema_version":1,"type":"score_trace","n_experts":2}\n', "has a header but no records"),
    ('{"schema_version":2,"type":"score_trace","n_experts":2}\n', "schema version 1"),
    ('{"schema_version":1,"type":"score_trace","n_experts":0}\n', "n_experts must be >= 1"),
    ('{"schema_version":1,"type":"score_trace","n_experts":2}\n{"step":0,"layer":0,"scores":[]}\n',
     "scores must be a non-empty array"),
    ('{"schema_version":1,"type":"score_trace","n_experts":2}\n{"step":0,"layer":0,"scores":[[1.0]]}\n',
     "row 0 does not have n_experts entries"),
    ('{"schema_version":1,"type":"score_trace","n_experts":2}\n'
     '{"step":0,"layer":0,"scores":[[0.5,0.5]],"mask":[true,false]}\n', "mask length does not match"),
    ('{"schema_version":1,"type":"score_trace","n_experts":2}\nnot json\n', "line 2"),
])
def test_reader_errors(tmp_path, body, frag):
    p = tmp_path / "t.ndjson"
    p.write_text(body)
    with pytest.raises(R.InvalidArgument, match=frag):
        T.read_score_trace(str(p))


def test_masked_rows_may_be_off_simplex(tmp_path):
    p = tmp_path / "t.ndjson"
    p.write_text('{"schema_version":1,"type":"score_trace","n_experts":2}\n'
                 '{"step":3,"layer":7,"scores":[[0.5,0.5],[0.0,0.0]],"mask":[true,false]}\n')
    (r,) = T.read_score_trace(str(p))
    assert (r.step, r.layer) == (3, 7) and r.scores.mask.tolist() == [True, False]


def _oracle_plan(scores, cfg, N):
    w = oracle.route(scores.scores, cfg, scores._mask_u8())
    plan = R.RoutingPlan(n_experts=N)
    B = scores.batch()
    plan.sets = [w.set_list(i) for i in range(B)]
    plan.weights = [[float(v) for v in w.weights[i, : w.set_len[i]]] for i in range(B)]
    plan.active_count = int(w.active_count)
    plan.active_union = [int(v) for v in w.active_union]
    plan.loads = np.asarray(w.loads[:N])
    plan.total_load = int(w.total_load)
    return plan


def test_routing_plans_document(tmp_path):
    rng = np.random.default_rng(5)
    N = 16
    recs = [T.ScoreRecord(s, l, R.ScoreMatrix(dirichlet(rng, 4, N))) for s in range(2) for l in range(2)]
    cfg = R.RoutingConfig.simplified(2, 4)
    plans = [_oracle_plan(r.scores, cfg, N) for r in recs]
    doc = T.routing_plans_json(recs, cfg, plans)
    assert doc["type"] == "routing_plans" and doc["schema_version"] == 1
    assert doc["routing"] == {"mode": "simplified", "k": 4, "k0": 2, "p": 1.0, "k_max": 4,
                              "max_p": N, "cap": "exact"}
    assert [(r["step"], r["layer"]) for r in doc["records"]] == [(0, 0), (0, 1), (1, 0), (1, 1)]
    pl = doc["records"][0]["plan"]
    assert set(pl) == {"n_experts", "active_experts", "total_load", "active_union", "loads", "tokens"}
    assert pl["active_experts"] == len(pl["active_union"]) and pl["total_load"] == 16
    assert all(set(t) == {"experts", "weights"} for t in pl["tokens"])
    out = tmp_path / "plans.json"
    T.write_routing_plans(str(out), doc)
    text = out.read_text()
    assert text.endswith("}\n") and json.loads(text) == json.loads(json.dumps(doc))
    vdoc = T.routing_plans_json(recs[:1], R.RoutingConfig.vanilla(8), [plans[0]])
    assert vdoc["routing"] == {"mode": "vanilla", "k": 8}
