"""GPU vs oracle parity at the BASELINE.json shapes the fused-path tests
(test_decode_gpu.py) only reach at reduced D/H:

  * C3, the Qwen3-235B-shaped layer (N=128, k=8, D=4096, H=1536, B=16), OEA
    simplified(4, 8) and vanilla top-8 (BASELINE configs[2]);
  * the full C1 D/H (2048 x 768) at every C2 batch size, so the dense
    single-launch path (B <= 16), the token-list single launch (16 < B <= 64)
    and the route-only prologue + compaction + grouped FFN (B > 64) are all
    compared with the oracle at the real shape (BASELINE configs[0-1]);
  * expert-parallel shards at the C3 shape for P in {2, 4, 8}: the summed
    partial mixtures against the ORACLE (not only the unsharded GPU layer);
  * the fp32 SIMT FFN (drop-in moe_forward<float>) against the oracle's
    moe_forward<float> at 1e-5 (north_star: "1e-5 (fp32)").

Bars (north_star): expert sets bit-exact vs the reference routing on the same
router logits; gate weights within 1e-5; bf16 layer outputs within 2e-2
relative (output_divergence, moe_layer.cpp:57-74) of moe_forward<double>
(proj/include/oea/moe_layer.hpp:114-158) on the stored bf16 weights."""
import numpy as np
import pytest

import oracle
from _parity import oracle_output_streamed, to_bf16_bits

pytestmark = pytest.mark.gpu

W_TOL = 1e-5
OUT_TOL = 2e-2
F32_TOL = 1e-5


def _check_plan(plan, want, B):
    for i in range(B):
        got = [int(v) for v in plan["sets"][i, : plan["set_len"][i]]]
        assert got == want.set_list(i), f"token {i}: {got} != {want.set_list(i)}"
    assert plan["active_count"] == want.active_count
    assert list(plan["active_union"]) == list(want.active_union)
    assert plan["total_load"] == want.total_load
    assert np.array_equal(plan["loads"], want.loads)
    assert np.abs(plan["weights"] - want.weights).max() <= W_TOL


def _decode_and_check(oea, layer, B, cfg, seed):
    """Decode from host buffers, check routing vs the oracle on the exported
    logits, and return (x, plan, oracle routing, out)."""
    x, xbits = to_bf16_bits(oracle.make_random_batch(B, layer.D, 1000 + seed))
    out = layer.decode_host(xbits, cfg)
    plan = layer.last_plan(B, cfg)
    want = oracle.route(oracle.softmax_rows(plan["logits"].astype(np.float64)), cfg)
    _check_plan(plan, want, B)
    return x, plan, want, out


def _expert_getter(layers):
    def get(e):
        for L in layers:
            if L.experts[0] <= e < L.experts[1]:
                return L.download_expert(e, "f64")
        raise KeyError(e)
    return get


@pytest.fixture(scope="module")
def c3_layer(oea):
    layer = oea.DeviceMoeLayer(4096, 1536, 128, "bf16")
    layer.init_random(23)
    yield layer
    layer.close()


@pytest.mark.parametrize("policy", ["oea", "vanilla"])
def test_c3_qwen235b_layer_vs_oracle(oea, c3_layer, policy):
    cfg = oea.RoutingConfig.simplified(4, 8) if policy == "oea" else oea.RoutingConfig.vanilla(8)
    B = 16
    x, plan, want, out = _decode_and_check(oea, c3_layer, B, cfg, seed=31)
    assert plan["total_load"] == B * 8
    ref = oracle_output_streamed(_expert_getter([c3_layer]), x, want.sets, want.set_len,
                                 want.weights)
    _, max_rel = oracle.output_divergence(ref, out.astype(np.float64))
    assert max_rel <= OUT_TOL, f"C3 {policy}: output max relative error {max_rel}"


@pytest.fixture(scope="module")
def c1_layer(oea):
    layer = oea.DeviceMoeLayer(2048, 768, 128, "bf16")
    layer.init_random(5)
    yield layer
    layer.close()


@pytest.mark.parametrize("B,k0", [(1, 4), (4, 4), (8, 2), (16, 1), (16, 8), (32, 4), (48, 3),
                                  (64, 4), (65, 4), (128, 4), (256, 4), (256, 8)])
def test_c1_shape_every_batch_path_vs_oracle(oea, c1_layer, B, k0):
    """C2 grid points at the real C1 D/H: k0 = 8 is vanilla top-8."""
    cfg = oea.RoutingConfig.vanilla(8) if k0 == 8 else oea.RoutingConfig.simplified(k0, 8)
    x, plan, want, out = _decode_and_check(oea, c1_layer, B, cfg, seed=100 + B + k0)
    ref = oracle_output_streamed(_expert_getter([c1_layer]), x, want.sets, want.set_len,
                                 want.weights)
    _, max_rel = oracle.output_divergence(ref, out.astype(np.float64))
    assert max_rel <= OUT_TOL, f"B={B} k0={k0}: output max relative error {max_rel}"


@pytest.mark.parametrize("P", [2, 4, 8])
def test_c3_expert_parallel_shards_vs_oracle(oea, P):
    """Each shard holds experts [r N/P, (r+1) N/P) of the same random layer;
    every shard routes the whole batch (bit-identical plans, equal to the
    oracle's on the logits), and the partial mixtures summed over ranks
    equal the oracle's moe_forward."""
    from paper_2511_02237_b200 import ep
    D, H, N, B = 4096, 1536, 128, 16
    cfg = oea.RoutingConfig.simplified(4, 8)
    x, xbits = to_bf16_bits(oracle.make_random_batch(B, D, 4242))
    shards, total, plan0 = [], np.zeros((B, D)), None
    try:
        for r in range(P):
            e0, e1 = ep.ep_expert_range(N, P, r)
            sh = oea.DeviceMoeLayer(D, H, N, "bf16", experts=(e0, e1))
            sh.init_random(29)
            shards.append(sh)
            total += sh.decode_host(xbits, cfg).astype(np.float64)
            plan = sh.last_plan(B, cfg)
            if plan0 is None:
                plan0 = plan
                want = oracle.route(oracle.softmax_rows(plan["logits"].astype(np.float64)), cfg)
                _check_plan(plan, want, B)
            for key in ("sets", "set_len", "active_union", "loads", "weights"):
                assert np.array_equal(plan[key], plan0[key]), (r, key)
        ref = oracle_output_streamed(_expert_getter(shards), x, want.sets, want.set_len,
                                     want.weights)
    finally:
        for sh in shards:
            sh.close()
    _, max_rel = oracle.output_divergence(ref, total)
    assert max_rel <= OUT_TOL, f"EP P={P}: summed shard output max relative error {max_rel}"


@pytest.mark.parametrize("D,H,N,B,k0", [(256, 384, 16, 8, 4), (1024, 512, 32, 16, 4),
                                        (100, 72, 10, 7, 2)])
def test_fp32_layer_vs_oracle_float(oea, D, H, N, B, k0):
    """moe_forward<float> (moe_layer.hpp:92-107 with Scalar = float) on the
    GPU's SIMT fp32 FFN vs the oracle's float restatement at 1e-5, both on
    the same plan (the reference's route on the GPU's fp64 router scores)."""
    layer = oea.DeviceMoeLayer(D, H, N, dtype="f32")
    layer.init_random(17)
    x = oracle.make_random_batch(B, D, 77)
    scores = layer.router_scores(x)
    cfg = oea.RoutingConfig.simplified(k0, 8 if N >= 8 else N)
    want = oracle.route(scores, cfg)
    got = layer.forward_plan(x, want.sets, want.set_len, want.weights)
    ws = [layer.download_expert(e, "f32") for e in range(N)]
    wg = np.stack([w[0] for w in ws])
    wu = np.stack([w[1] for w in ws])
    wd = np.stack([w[2] for w in ws])
    ref = oracle.moe_forward(wg, wu, wd, x, want.sets, want.set_len, want.weights, scalar="f32")
    mean_rel, max_rel = oracle.output_divergence(ref, got)
    assert max_rel <= F32_TOL, f"fp32 output max relative error {max_rel} (mean {mean_rel})"
    # and the fp32 decode (router_scores -> route -> moe_forward<float>) end to end
    out = layer.decode_host(x, cfg)
    plan = layer.last_plan(B, cfg)
    want2 = oracle.route(plan["scores"], cfg)
    _check_plan(plan, want2, B)
    ref2 = oracle.moe_forward(wg, wu, wd, x, want2.sets, want2.set_len, want2.weights,
                              scalar="f32")
    _, max_rel2 = oracle.output_divergence(ref2, out)
    assert max_rel2 <= F32_TOL, f"fp32 decode max relative error {max_rel2}"
