"""K1 route_f64 on the GPU vs the CPU oracle: bit-exact sets AND weights.

Mirrors the reference's routing tests (proj/tests/test_routing.cpp) through the
Python mirror of the operator API, plus randomized parity (acceptance.cpp
criterion 4 generator) and the B=4096 router stress config (BASELINE C5)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def plan_matches(plan, want, B):
    for i in range(B):
        if plan.sets[i] != want.set_list(i):
            return f"token {i}: sets {plan.sets[i]} != {want.set_list(i)}"
        w = [float(v) for v in want.weights[i, : want.set_len[i]]]
        if plan.weights[i] != w:
            return f"token {i}: weights differ"
    if plan.active_union != [int(v) for v in want.active_union]:
        return "active_union differs"
    if plan.active_count != want.active_count or plan.total_load != want.total_load:
        return "aggregates differ"
    if not np.array_equal(plan.loads, want.loads):
        return "loads differ"
    return ""


def test_sort_kat(oea):
    # test_routing.cpp:112-121
    m = oea.ScoreMatrix(np.array([[0.5, 0.3, 0.15, 0.05], [0.25] * 4, [0.1, 0.25, 0.6, 0.05]]))
    s = oea.sort_experts(m)
    assert s.order.tolist() == [[0, 1, 2, 3], [0, 1, 2, 3], [2, 1, 0, 3]]
    with pytest.raises(oea.InvalidArgument):
        oea.sort_experts(oea.ScoreMatrix(np.zeros((0, 4))))


def test_topk_kat(oea):
    # test_routing.cpp:123-151
    m = np.array([[0.5, 0.3, 0.15, 0.05]])
    plan = oea.route_topk(m, 2)
    assert plan.sets[0] == [0, 1]
    assert plan.weights[0][0] == pytest.approx(0.625, rel=1e-12)
    assert plan.weights[0][1] == pytest.approx(0.375, rel=1e-12)
    assert plan.active_count == 2 and plan.total_load == 2
    plan = oea.route_topk(m, 4)
    for j in range(4):
        assert plan.weights[0][j] == pytest.approx(m[0, plan.sets[0][j]], rel=1e-12)
    plan = oea.route_topk(np.array([[0.35, 0.35, 0.15, 0.15], [0.15, 0.15, 0.35, 0.35]]), 2)
    assert plan.active_count == 4 and plan.total_load == 4
    assert plan.active_union == [0, 1, 2, 3] and list(plan.loads) == [1, 1, 1, 1]


def test_phase1_kat(oea):
    # test_routing.cpp:153-183
    m = oea.ScoreMatrix(np.array([[0.4, 0.3, 0.2, 0.1]]))
    srt = oea.sort_experts(m)
    ph = oea.phase1_baseline(m, srt, oea.RoutingConfig.pruned(3, 0.6, 3).resolved(4))
    assert ph.t[0] == 2 and ph.n[0] == 2 and ph.base_sets[0] == [0, 1] and ph.base_union == [0, 1]
    ph = oea.phase1_baseline(m, srt, oea.RoutingConfig.pruned(3, 1.0, 3).resolved(4))
    assert ph.t[0] == 4 and ph.n[0] == 3
    ph = oea.phase1_baseline(m, srt, oea.RoutingConfig.pruned(1, 0.6, 1).resolved(4))
    assert ph.base_sets[0] == [0]
    plan = oea.route(np.array([[0.7, 0.3, 0.0, 0.0]]), oea.RoutingConfig.pruned(4, 1.0, 4))
    assert len(plan.sets[0]) == 4
    assert plan.weights[0][0] == pytest.approx(0.7, rel=1e-12)
    assert plan.weights[0][2] == 0.0 and plan.weights[0][3] == 0.0


def test_piggyback_walkthrough(oea):
    # test_routing.cpp:185-203
    m = np.array([[0.5, 0.3, 0.15, 0.05], [0.15, 0.25, 0.55, 0.05]])
    plan = oea.route(m, oea.RoutingConfig.oea(1, 1.0, 2, 4, 2))
    assert plan.sets == [[0, 2], [2, 0]]
    assert plan.active_union == [0, 2] and plan.active_count == 2 and plan.total_load == 4
    assert plan.loads[0] == 2 and plan.loads[2] == 2
    assert plan.weights[0][0] == pytest.approx(0.5 / 0.65, rel=1e-12)
    assert plan.weights[0][1] == pytest.approx(0.15 / 0.65, rel=1e-12)
    assert oea.route_topk(m, 2).active_count == 3


def test_strict_cap_and_masks(oea):
    # test_routing.cpp:244-278
    m = np.array([[0.4, 0.3, 0.2, 0.1], [0.1, 0.2, 0.3, 0.4]])
    ex = oea.route(m, oea.RoutingConfig.oea(3, 1.0, 3, 4, 3, oea.CapSemantics.ExactCap))
    st = oea.route(m, oea.RoutingConfig.oea(3, 1.0, 3, 4, 3, oea.CapSemantics.PseudocodeStrict))
    assert ex.sets == [[0, 1, 2], [3, 2, 1]]
    assert st.sets == [[0, 1, 2, 3], [3, 2, 1, 0]]
    sm = oea.ScoreMatrix(np.array([[0.5, 0.3, 0.15, 0.05], [0.05, 0.15, 0.3, 0.5],
                                   [0.25, 0.25, 0.25, 0.25]]), np.array([True, False, True]))
    sm.validate()
    plan = oea.route(sm, oea.RoutingConfig.vanilla(2))
    assert plan.sets[1] == [] and plan.weights[1] == []
    assert plan.active_union == [0, 1] and plan.total_load == 4
    sm.mask[:] = False
    plan = oea.route(sm, oea.RoutingConfig.vanilla(2))
    assert plan.active_count == 0 and plan.total_load == 0
    st = oea.batch_stats(plan)
    assert st.active_count == 0 and st.total_load == 0


def test_errors(oea):
    # test_routing.cpp:237-242, 280-302
    with pytest.raises(oea.DomainError, match="degenerate selected-set mass for token 0"):
        oea.route(np.zeros((1, 4)), oea.RoutingConfig.pruned(2, 1.0, 2))
    bad = [oea.RoutingConfig.vanilla(0), oea.RoutingConfig.vanilla(5),
           oea.RoutingConfig.pruned(0, 1.0, 1), oea.RoutingConfig.pruned(2, 0.0, 2),
           oea.RoutingConfig.pruned(2, 1.2, 2), oea.RoutingConfig.oea(3, 1.0, 2, 4, 3),
           oea.RoutingConfig.oea(2, 1.0, 2, 5, 2)]
    for c in bad:
        with pytest.raises(oea.InvalidArgument):
            c.resolved(4)
        with pytest.raises(oea.InvalidArgument):
            oea.route(np.full((1, 4), 0.25), c)
    assert oea.RoutingConfig.oea(2, 1.0, 2, 0, 2).resolved(4).max_p == 4
    simp = oea.RoutingConfig.simplified(2, 3).resolved(4)
    assert simp.p == 1.0 and simp.k_max == 3 and simp.max_p == 4


def _random_cfg(rng, n, oea):
    cap = oea.CapSemantics(int(rng.integers(0, 2)))
    p = 1.0 if rng.integers(0, 2) == 0 else int(rng.integers(1, 9)) / 8.0
    kind = int(rng.integers(0, 4))
    if kind == 0:
        return oea.RoutingConfig.vanilla(int(rng.integers(1, n + 1)))
    if kind == 1:
        k0 = int(rng.integers(1, n + 1))
        return oea.RoutingConfig.pruned(k0, p, k0)
    if kind == 2:
        k0 = int(rng.integers(1, n + 1))
        km = k0 + int(rng.integers(0, n - k0 + 1))
        return oea.RoutingConfig.oea(k0, p, km, int(rng.integers(1, n + 1)), km, cap)
    k = int(rng.integers(1, n + 1))
    return oea.RoutingConfig.simplified(int(rng.integers(1, k + 1)), k, cap)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_parity_bit_exact(oea, seed):
    """acceptance.cpp:220-253 generator (+ lattice rows with ties, masks,
    N up to 300): sets, weights and aggregates bit-identical to the oracle."""
    rng = np.random.default_rng(seed)
    for rep in range(400):
        n = int(rng.integers(1, 65)) if rep % 10 else int(rng.integers(65, 300))
        b = int(rng.integers(1, 33))
        s = rng.exponential(size=(b, n))
        s /= s.sum(axis=1, keepdims=True)
        if rep % 3 == 0:  # 1/8-lattice rows: exact ties
            s = np.zeros((b, n))
            for i in range(b):
                for _ in range(8):
                    s[i, rng.integers(0, n)] += 1.0 / 8
        mask = (rng.random(b) < 0.75) if rep % 5 == 0 else None
        cfg = _random_cfg(rng, n, oea)
        sm = oea.ScoreMatrix(s, mask)
        try:
            want = oracle.route(s, cfg, None if mask is None else mask.astype(np.uint8))
        except oracle.OracleDomainError as e:
            with pytest.raises(oea.DomainError, match=str(e).split("(")[0].strip()):
                oea.route(sm, cfg)
            continue
        got = oea.route(sm, cfg)
        msg = plan_matches(got, want, b)
        assert not msg, f"rep {rep} n={n} b={b} cfg={cfg}: {msg}"


def test_sort_matches_oracle_with_ties_and_negative_zero(oea):
    rng = np.random.default_rng(9)
    s = np.round(rng.random((64, 200)) * 4) / 4
    s[:, ::7] = -0.0
    s[:, 3::11] = 0.0
    got = oea.sort_experts(s).order
    assert np.array_equal(got, oracle.sort_experts(s))


def test_phase_functions_match_route(oea):
    rng = np.random.default_rng(5)
    for rep in range(50):
        n = int(rng.integers(2, 40))
        b = int(rng.integers(1, 12))
        s = rng.exponential(size=(b, n))
        s /= s.sum(1, keepdims=True)
        k0 = int(rng.integers(1, n + 1))
        km = k0 + int(rng.integers(0, n - k0 + 1))
        cfg = oea.RoutingConfig.oea(k0, 1.0, km, 0, km).resolved(n)
        srt = oea.sort_experts(s)
        ph = oea.phase1_baseline(s, srt, cfg)
        p2 = oea.phase2_piggyback(s, srt, ph, cfg)
        full = oea.route(s, cfg)
        assert p2.sets == full.sets
        assert full.active_union == ph.base_union  # conservation (acceptance c2)


def test_router_stress_b4096(oea):
    """BASELINE C5: B=4096, N=128, k=8, k0 sweep; sets bit-exact."""
    rng = np.random.default_rng(4096)
    logits = rng.standard_normal((4096, 128))
    s = oracle.softmax_rows(logits)
    for k0 in (1, 4, 8):
        cfg = oea.RoutingConfig.simplified(k0, 8)
        got = oea.route(s, cfg)
        want = oracle.route(s, cfg)
        assert not plan_matches(got, want, 4096)


@pytest.mark.parametrize("N,B", [(128, 4096), (64, 300), (20, 77), (128, 5)])
def test_fast_path_equals_sort_path(oea, N, B, monkeypatch):
    """The p == 1 / max_p = N fast path (top-m picks, no full sort) and the
    general sort path give bit-identical plans, masks and ties included."""
    rng = np.random.default_rng(N * 1000 + B)
    s = rng.exponential(size=(B, N))
    s[:, ::5] = s[:, 1::5]  # exact ties
    s /= s.sum(axis=1, keepdims=True)
    mask = rng.random(B) < 0.9
    sm = oea.ScoreMatrix(s, mask)
    cfgs = [oea.RoutingConfig.simplified(4, 8), oea.RoutingConfig.simplified(1, 8),
            oea.RoutingConfig.vanilla(8), oea.RoutingConfig.pruned(3, 1.0, 3),
            oea.RoutingConfig.oea(2, 1.0, 6, 0, 6, oea.CapSemantics.PseudocodeStrict)]
    for cfg in cfgs:
        monkeypatch.delenv("OEA_ROUTE_SORT", raising=False)
        fast = oea.route(sm, cfg)
        monkeypatch.setenv("OEA_ROUTE_SORT", "1")
        slow = oea.route(sm, cfg)
        assert fast.sets == slow.sets and fast.weights == slow.weights, cfg
        assert fast.active_union == slow.active_union and fast.total_load == slow.total_load
        assert np.array_equal(fast.loads, slow.loads)


def test_single_launch_speculative_phase2_fallback(oea):
    """The single-launch route picks phase 2 speculatively (the next experts of
    the whole list) before the batch union is known and re-picks among the
    union members when a speculative pick is not one. Token 0 prefers experts
    0, 1, 2, 3 and token 1 prefers 7, 6, 5, 4: with k0 = 1 the union is {0, 7},
    so both tokens' speculative picks (1, 2 / 6, 5) miss and the sets must be
    the reference's {0, 7} / {7, 0} (phase2_piggyback, routing.cpp:270-303).
    Also a batch with a full union (speculation kept) and a masked row."""
    s = np.array([[0.30, 0.20, 0.15, 0.10, 0.09, 0.07, 0.05, 0.04],
                  [0.04, 0.05, 0.07, 0.09, 0.10, 0.15, 0.20, 0.30]])
    cfg = oea.RoutingConfig.simplified(1, 3)
    got = oea.route(s, cfg)
    assert got.sets[0] == [0, 7] and got.sets[1] == [7, 0]
    assert plan_matches(got, oracle.route(s, cfg), 2) == ""
    rng = np.random.default_rng(11)
    for B, k0, k in ((300, 2, 6), (64, 4, 8), (7, 1, 8)):
        x = rng.random((B, 128)) ** 4
        x /= x.sum(axis=1, keepdims=True)
        mask = np.ones(B, bool)
        mask[B // 2] = False
        cfg = oea.RoutingConfig.simplified(k0, k)
        want = oracle.route(x, cfg, mask.astype(np.uint8))
        got = oea.route(oea.ScoreMatrix(x, mask), cfg)
        assert plan_matches(got, want, B) == "", (B, k0, k)
