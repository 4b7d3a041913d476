"""Device score generators (score_gen.cpp:100-160) vs the oracle restatement
(itself pinned bit-exactly to the compiled reference in
tests/test_oracle_score_gen.py). Device libm differs from glibc in the last
ulps, so rows are compared at 1e-12 relative; rejection decisions in the
gamma sampler then agree (a flip would change the rest of a row by O(1))."""
import numpy as np
import pytest

import oracle
from paper_2511_02237_b200 import scoregen as G

pytestmark = pytest.mark.gpu
REL = 1e-12


def _close(a, b):
    return np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)) <= REL


@pytest.mark.parametrize("alpha", [0.05, 0.3, 1.0, 2.5, 30.0])
def test_dirichlet_matches_reference(oea, alpha):
    cfg = G.ScoreGenConfig(G.GenKind.Dirichlet, n_experts=128, batch=16, steps=3, layers=4,
                           seed=123, alpha=alpha)
    run = G.gen_run(cfg)
    assert run.shape == (3, 4, 16, 128)
    for s in range(3):
        for l in range(4):
            want = oracle.gen_dirichlet(128, 16, 123, alpha, s, l)
            assert _close(run[s, l], want), (s, l)
    assert np.allclose(run.sum(axis=-1), 1.0, atol=1e-12)


@pytest.mark.parametrize("groups,conc,spread", [(1, 4.0, 2.0), (3, 4.0, 2.0), (8, 0.5, 5.0),
                                                (2, 4.0, 0.0)])
def test_clustered_matches_reference(oea, groups, conc, spread):
    cfg = G.ScoreGenConfig(G.GenKind.Clustered, n_experts=64, batch=10, steps=2, layers=3,
                           seed=9, groups=groups, within_group_concentration=conc,
                           between_group_spread=spread)
    run = G.gen_run(cfg)
    for s in range(2):
        for l in range(3):
            want = oracle.gen_clustered(64, 10, 9, groups, conc, spread, s, l)
            assert _close(run[s, l], want), (s, l)
    if spread == 0.0:
        assert np.all(run == 1.0 / 64)  # collapses to uniform (score_gen.hpp:42-43)


def test_single_cell_and_step_window(oea):
    cfg = G.ScoreGenConfig(G.GenKind.Dirichlet, n_experts=32, batch=4, steps=5, layers=2,
                           seed=1, alpha=0.7)
    full = G.gen_run(cfg)
    assert np.array_equal(G.gen_run(cfg, 2, 2), full[2:4])
    assert np.array_equal(G.gen_scores(cfg, 4, 1).scores, full[4, 1])


def test_validation_messages(oea):
    bad = [(dict(steps=0), "steps and layers must be >= 1"),
           (dict(n_experts=0), "n_experts and batch must be >= 1"),
           (dict(alpha=0.0), "alpha must be > 0"),
           (dict(kind=G.GenKind.Clustered, groups=0), "groups must be in"),
           (dict(kind=G.GenKind.Clustered, within_group_concentration=0.0), "concentration must be > 0"),
           (dict(kind=G.GenKind.Clustered, between_group_spread=-1.0), "spread must be >= 0")]
    for kw, msg in bad:
        with pytest.raises(oea.InvalidArgument, match=msg):
            G.gen_run(G.ScoreGenConfig(**kw))
    with pytest.raises(oea.InvalidArgument, match="out of range"):
        G.gen_run(G.ScoreGenConfig(steps=2), 1, 2)


def test_generated_batches_route(oea):
    # C5-style stress input made on the device, routed through the batched path
    cfg = G.ScoreGenConfig(G.GenKind.Dirichlet, n_experts=128, batch=64, steps=4, layers=8,
                           seed=5, alpha=0.2)
    run = G.gen_run(cfg)
    recs = [oea.ScoreMatrix(run[s, l]) for s in range(4) for l in range(8)]
    plans = oea.route_batched(recs, oea.RoutingConfig.simplified(4, 8))
    for q in (0, 13, 31):
        w = oracle.route(recs[q].scores, oea.RoutingConfig.simplified(4, 8))
        assert plans[q].sets == [w.set_list(i) for i in range(64)]
