"""Boundary behaviour that must equal the reference's on the same inputs.

* A caller plan that names an expert twice in one token's set: the
  reference's moe_forward adds w_j * expert_forward(E[e], x) once per
  occurrence, in set order (proj/include/oea/moe_layer.hpp:146-155), with no
  error. The drop-in (C ABI oea_moe_forward_plan_host, the Python mirror's
  moe_forward, and the C++ adapter behind include/oea/moe_layer.hpp) must
  return the compiled reference's output (oracle/_ref).
* Expert-parallel entry points at world == 1 (partial + combine) must not
  wait for peer arrivals that never come.
* A shard whose routing tables do not fit the fused prologue's shared
  memory is rejected up front (it cannot take the two-kernel path).
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _dup_plan():
    sets = np.array([[3, 3, 5, -1], [1, 2, 1, 1], [7, -1, -1, -1], [0, 9, 0, 4]], np.int32)
    set_len = np.array([3, 4, 1, 4], np.int32)
    w = np.array([[0.5, 0.25, 0.25, 0], [0.1, 0.2, 0.3, 0.4], [1.0, 0, 0, 0],
                  [0.4, 0.3, 0.2, 0.1]])
    return sets, set_len, w


@pytest.mark.parametrize("scalar", ["f64", "f32"])
def test_duplicate_experts_match_compiled_reference(oea, scalar):
    if not oracle.reference_available():
        pytest.skip("oracle/_ref not built")
    D, H, N = 64, 96, 16
    router, wg, wu, wd = oracle.make_random_layer(D, H, N, 3)
    x = oracle.make_random_batch(4, D, 9)
    sets, set_len, w = _dup_plan()
    ref = oracle.Reference().layer(router, wg, wu, wd, scalar).moe_forward(x, sets, set_len, w)
    dt = np.float64 if scalar == "f64" else np.float32
    layer = oea.DeviceMoeLayer(D, H, N, dtype=scalar)
    for e in range(N):
        layer.upload_expert(e, wg[e].astype(dt), wu[e].astype(dt), wd[e].astype(dt))
    got = layer.forward_plan(x, sets, set_len, w)
    _, max_rel = oracle.output_divergence(ref, got)
    assert max_rel <= (1e-12 if scalar == "f64" else 1e-5), max_rel
    # through the reference-shaped Python API as well
    params = oea.MoeLayerParams(router.astype(dt), [oea.ExpertParams(wg[e].astype(dt),
                                                                     wu[e].astype(dt),
                                                                     wd[e].astype(dt))
                                                    for e in range(N)])
    plan = oea.RoutingPlan(sets=[list(map(int, sets[i, : set_len[i]])) for i in range(4)],
                           weights=[list(map(float, w[i, : set_len[i]])) for i in range(4)],
                           n_experts=N)
    got2 = oea.moe_forward(params, oea.TokenBatch(x), plan)
    _, max_rel2 = oracle.output_divergence(ref, np.asarray(got2))
    assert max_rel2 <= (1e-12 if scalar == "f64" else 1e-5), max_rel2


def test_duplicate_experts_bf16_layer(oea):
    """bf16 layer (tensor-core FFN): the duplicated slot reuses the first
    occurrence's y; the result equals the oracle's moe_forward<double> on the
    stored bf16 weights within the bf16 bar."""
    D, H, N = 256, 128, 16
    layer = oea.DeviceMoeLayer(D, H, N, dtype="bf16")
    layer.init_random(4)
    x = oracle.bf16_round(oracle.make_random_batch(4, D, 19))
    sets, set_len, w = _dup_plan()
    got = layer.forward_plan(x, sets, set_len, w)
    ws = [layer.download_expert(e, "f64") for e in range(N)]
    ref = oracle.moe_forward(np.stack([a[0] for a in ws]), np.stack([a[1] for a in ws]),
                             np.stack([a[2] for a in ws]), x, sets, set_len, w)
    _, max_rel = oracle.output_divergence(ref, got)
    assert max_rel <= 2e-2, max_rel
    # the same plan without the duplicates but with their weights merged gives
    # the same mixture (to fp rounding): the duplicate is not dropped
    nodup = np.full_like(sets, -1)
    nlen = np.zeros_like(set_len)
    nw = np.zeros_like(w)
    for i in range(4):
        acc = {}
        for j in range(set_len[i]):
            acc[int(sets[i, j])] = acc.get(int(sets[i, j]), 0.0) + w[i, j]
        for j, (e, v) in enumerate(acc.items()):
            nodup[i, j], nw[i, j] = e, v
        nlen[i] = len(acc)
    got2 = layer.forward_plan(x, nodup, nlen, nw)
    assert np.abs(got - got2).max() <= 1e-5 * np.abs(got2).max()


def test_ep_world1_partial_then_combine_returns(oea):
    """world == 1: the partial decodes straight into the receive buffer and
    the combine is a copy (it must not wait for peer arrivals)."""
    import torch
    from paper_2511_02237_b200 import ep
    D, H, N, B = 512, 256, 32, 8
    layer = oea.DeviceMoeLayer(D, H, N, "bf16")
    layer.init_random(12)
    cfg = oea.RoutingConfig.simplified(4, 8)
    x = torch.randn(B, D, device="cuda").to(torch.bfloat16)
    want = torch.empty(B, D, device="cuda", dtype=torch.float32)
    layer.decode(x, cfg, want)
    layer.ctx.synchronize()
    m = ep.PeerExpertParallelMoE(layer, cfg, 1, 0, B)
    ep.PeerExpertParallelMoE.emulate_group([m])
    out = torch.empty(B, D, device="cuda", dtype=torch.float32)
    for _ in range(3):
        m.forward(x, out)
        layer.ctx.synchronize()
        assert torch.equal(out, want)
    m.close()


def test_shard_too_large_for_fused_prologue_rejected(oea):
    """B = 64 with a long set stride (pseudocode cap, k_max = 40) does not fit
    the fused prologue's tables: a shard must be rejected up front rather than
    take the two-kernel path (whose plan names experts it does not hold)."""
    import torch
    sh = oea.DeviceMoeLayer(256, 128, 128, "bf16", experts=(0, 64))
    sh.init_random(1)
    x = torch.zeros(64, 256, device="cuda", dtype=torch.bfloat16)
    out = torch.empty(64, 256, device="cuda", dtype=torch.float32)
    cfg = oea.RoutingConfig.simplified(4, 100, oea.CapSemantics.PseudocodeStrict)
    with pytest.raises(oea.InvalidArgument, match="expert-parallel shards need the fused path"):
        sh.decode(x, cfg, out)
