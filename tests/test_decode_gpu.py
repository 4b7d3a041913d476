"""The fused bf16 decode layer (K2 router + K3 compaction + K4/K5 FFN) vs the
CPU oracle.

Parity bar (BASELINE.json north_star):
  * expert sets bit-exact vs the reference routing fed the same router logits
    (the exported fp32 logits, softmax in fp64 by the oracle);
  * gate weights within 1e-5;
  * layer output within 2e-2 relative (output_divergence, moe_layer.cpp:57-74)
    of moe_forward<double> on the same bf16-rounded weights and inputs.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

W_TOL = 1e-5
OUT_TOL = 2e-2


def to_bf16_bits(x):
    xb = oracle.bf16_round(x)
    return xb, (xb.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)


def oracle_output(layer, x, want):
    """moe_forward<double> on the layer's stored bf16 weights, restricted to
    the active experts (remapped), so large layers stay cheap to check."""
    act = [int(e) for e in want.active_union]
    if not act:
        return np.zeros((x.shape[0], layer.D))
    remap = {e: i for i, e in enumerate(act)}
    ws = [layer.download_expert(e, "f64") for e in act]
    wg = np.stack([w[0] for w in ws])
    wu = np.stack([w[1] for w in ws])
    wd = np.stack([w[2] for w in ws])
    sets = np.where(want.sets >= 0, np.vectorize(lambda e: remap.get(int(e), -1))(want.sets), -1)
    return oracle.moe_forward(wg, wu, wd, x, sets.astype(np.int32), want.set_len, want.weights)


def run_case(oea, D, H, N, B, cfg, seed=1, mask=None, check_logits=True, x_scale=1.0):
    layer = oea.DeviceMoeLayer(D, H, N, dtype="bf16")
    layer.init_random(seed)
    x, xbits = to_bf16_bits(oracle.make_random_batch(B, D, 1000 + seed) * x_scale)
    out = layer.decode_host(xbits, cfg, mask=mask)
    plan = layer.last_plan(B, cfg)
    m8 = None if mask is None else np.asarray(mask, np.uint8)
    if check_logits:
        R = layer.download_router("f64")
        ref_logits = x @ R
        err = np.abs(plan["logits"] - ref_logits).max() / max(np.abs(ref_logits).max(), 1e-30)
        assert err < 1e-4, f"router logits rel err {err}"
    want = oracle.route(oracle.softmax_rows(plan["logits"].astype(np.float64)), cfg, m8)
    for i in range(B):
        got = [int(v) for v in plan["sets"][i, : plan["set_len"][i]]]
        assert got == want.set_list(i), f"token {i}: {got} != {want.set_list(i)}"
    assert plan["active_count"] == want.active_count
    assert list(plan["active_union"]) == list(want.active_union)
    assert plan["total_load"] == want.total_load
    assert np.array_equal(plan["loads"], want.loads)
    assert np.abs(plan["weights"] - want.weights).max() <= W_TOL
    ref = oracle_output(layer, x, want)
    if want.active_count == 0:
        assert np.all(out == 0)
        return plan, 0.0
    real = np.ones(B, bool) if mask is None else np.asarray(mask, bool)
    _, max_rel = oracle.output_divergence(ref[real], out[real].astype(np.float64))
    assert max_rel <= OUT_TOL, f"output max relative error {max_rel}"
    if mask is not None:
        assert np.all(out[~real] == 0)
    return plan, max_rel


def test_decode_qwen30b_shape_oea(oea):
    """BASELINE C1 shape: N=128, k=8, D=2048, H=768, B=16, simplified(4, 8)."""
    plan, err = run_case(oea, 2048, 768, 128, 16, oea.RoutingConfig.simplified(4, 8))
    assert 20 <= plan["active_count"] <= 90
    assert plan["total_load"] == 16 * 8


def test_decode_qwen30b_shape_vanilla(oea):
    run_case(oea, 2048, 768, 128, 16, oea.RoutingConfig.vanilla(8), seed=2)


@pytest.mark.parametrize("mode", ["vanilla", "pruned", "oea", "simplified", "strict"])
def test_decode_modes_small(oea, mode):
    R = oea.RoutingConfig
    cfg = {"vanilla": R.vanilla(4), "pruned": R.pruned(2, 1.0, 4),
           "oea": R.oea(2, 1.0, 4, 10, 4), "simplified": R.simplified(2, 4),
           "strict": R.simplified(2, 4, oea.CapSemantics.PseudocodeStrict)}[mode]
    run_case(oea, 256, 128, 16, 8, cfg, seed=3)


@pytest.mark.parametrize("cfg_name,B", [("mass", 16), ("max_p", 16), ("mass", 48), ("both", 16)])
def test_decode_two_kernel_configs_c1_shape(oea, cfg_name, B):
    """p < 1 (the cumulative-mass baseline of routing.cpp:226-268) and
    max_p < N (phase 2 limited to the first max_p ranks, :270-303) at the C1
    layer shape, through the fused rank routing (B = 16: the single launch;
    B = 48: the route-only launch + tcgen05 FFN). Sets bit-exact vs the
    oracle on the exported logits (p < 1: the fp64 softmax of the fp32
    logits on both sides), phase-1 baseline sizes equal."""
    R = oea.RoutingConfig
    cfg = {"mass": R.oea(4, 0.5, 8, 128, 8), "max_p": R.oea(4, 1.0, 8, 24, 8),
           "both": R.oea(3, 0.4, 6, 40, 8)}[cfg_name]
    # x scaled so the softmax is peaked enough for the mass rule to bite
    plan, _ = run_case(oea, 2048, 768, 128, B, cfg, seed=21 + B, x_scale=2.0 if cfg.p < 1.0 else 1.0)
    want = oracle.route(oracle.softmax_rows(plan["logits"].astype(np.float64)), cfg, None)
    assert np.array_equal(plan["phase1_n"], want.n)
    if cfg.p < 1.0:  # the mass rule really cut some baselines below k0
        assert int(want.n.min()) < cfg.k0


@pytest.mark.parametrize("cfg_name", ["mass", "max_p"])
def test_decode_router_cluster_configs(oea, cfg_name):
    """N > 128 experts: the router cluster + FFN pair (k_router_fused's
    distributed warp-sort routing) with p < 1 and max_p < N."""
    R = oea.RoutingConfig
    cfg = {"mass": R.oea(3, 0.5, 8, 160, 8), "max_p": R.oea(3, 1.0, 8, 20, 8)}[cfg_name]
    plan, _ = run_case(oea, 512, 256, 160, 16, cfg, seed=31, x_scale=2.0 if cfg.p < 1.0 else 1.0)
    want = oracle.route(oracle.softmax_rows(plan["logits"].astype(np.float64)), cfg, None)
    assert np.array_equal(plan["phase1_n"], want.n)


def test_decode_odd_dims_and_mask(oea):
    mask = np.array([1, 0, 1, 1, 0, 1, 1], bool)
    run_case(oea, 100, 72, 10, 7, oea.RoutingConfig.simplified(2, 3), seed=4, mask=mask)


def test_decode_all_masked_is_zero(oea):
    mask = np.zeros(5, bool)
    run_case(oea, 128, 128, 8, 5, oea.RoutingConfig.simplified(2, 4), seed=5, mask=mask)


def test_decode_large_token_groups(oea):
    """More than 64 tokens on one expert -> several token groups per expert."""
    run_case(oea, 256, 256, 4, 150, oea.RoutingConfig.vanilla(4), seed=6)


@pytest.mark.parametrize("B", [1, 4, 32, 64, 128, 256])
def test_decode_batch_sweep(oea, B):
    """BASELINE C2 batch sizes (smaller D/H keeps the CPU check fast)."""
    run_case(oea, 512, 256, 128, B, oea.RoutingConfig.simplified(3, 8), seed=7 + B)


def test_decode_deterministic_and_graph(oea):
    import torch
    D, H, N, B = 1024, 512, 64, 16
    layer = oea.DeviceMoeLayer(D, H, N, dtype="bf16")
    layer.init_random(8)
    x = torch.randn(B, D, device="cuda").to(torch.bfloat16)
    out1 = torch.empty(B, D, device="cuda", dtype=torch.float32)
    out2 = torch.empty_like(out1)
    cfg = oea.RoutingConfig.simplified(4, 8)
    torch.cuda.synchronize()
    layer.decode(x, cfg, out1)
    layer.ctx.synchronize()
    g = layer.graph(x, cfg, out2)
    for _ in range(3):
        g.launch()
    layer.ctx.synchronize()
    assert torch.equal(out1, out2)


def test_mixed_shapes_share_workspace(oea):
    """Layers of different shapes and batch sizes decoded back to back on one
    context (one workspace, one set of self-resetting grid counters) give the
    same outputs as when each runs alone."""
    import torch
    cfg = oea.RoutingConfig.simplified(4, 8)
    shapes = [(2048, 768, 128, 16), (512, 256, 64, 60), (512, 256, 128, 200), (1024, 512, 64, 8)]
    layers, xs, solo = [], [], []
    for i, (D, H, N, B) in enumerate(shapes):
        L = oea.DeviceMoeLayer(D, H, N, "bf16")
        L.init_random(40 + i)
        x = torch.randn(B, D, device="cuda").to(torch.bfloat16)
        out = torch.empty(B, D, device="cuda", dtype=torch.float32)
        L.decode(x, cfg, out)
        L.ctx.synchronize()
        layers.append(L)
        xs.append(x)
        solo.append(out.clone())
    outs = [torch.empty_like(o) for o in solo]
    for rep in range(3):
        for i in (0, 2, 1, 3, 0, 1, 2, 0):
            layers[i].decode(xs[i], cfg, outs[i])
        layers[0].ctx.synchronize()
        for i in range(len(shapes)):
            assert torch.equal(outs[i], solo[i]), (rep, shapes[i])


def test_chained_decodes_on_torch_stream(oea):
    """x_{l+1} = out_l through torch ops on torch's default stream with no
    host sync in between (the C ABI gets cudaStreamLegacy for it) equals the
    per-layer synchronised chain."""
    import torch
    from paper_2511_02237_b200.moe_layer import torch_stream
    cfg = oea.RoutingConfig.simplified(4, 8)
    layers = []
    for s in range(4):
        L = oea.DeviceMoeLayer(2048, 768, 128, "bf16")
        L.init_random(60 + s)
        layers.append(L)
    x = torch.randn(16, 2048, device="cuda").to(torch.bfloat16)

    def run(sync):
        h, outs = x, []
        for L in layers:
            o = torch.empty(16, 2048, device="cuda", dtype=torch.float32)
            L.decode(h, cfg, o, stream=torch_stream())
            if sync:
                torch.cuda.synchronize()
            outs.append(o)
            h = o.to(torch.bfloat16)
        torch.cuda.synchronize()
        return outs
    ref = run(True)
    for _ in range(3):
        for o, r in zip(run(False), ref):
            assert torch.equal(o, r)


@pytest.mark.parametrize("D,H,B,cfg_name", [(2048, 768, 16, "oea"), (1000, 384, 40, "oea"),
                                             (2048, 768, 5, "vanilla"), (512, 256, 100, "oea")])
def test_decode_host_zero_copy_matches_device(oea, D, H, B, cfg_name):
    """oea_moe_decode_host with pinned host buffers (x staged in-kernel, out
    written over the host link; B > 64 falls back to the copies): the same
    plan and bit-identical outputs as the device-resident decode."""
    import torch
    cfg = oea.RoutingConfig.simplified(4, 8) if cfg_name == "oea" else oea.RoutingConfig.vanilla(8)
    layer = oea.DeviceMoeLayer(D, H, 64, dtype="bf16")
    layer.init_random(7)
    g = torch.Generator().manual_seed(3)
    # several calls with fresh host buffers: the first captures the launch,
    # the next replay it with the x / out pointers patched
    for it in range(3):
        xh = torch.randn(B, D, generator=g).to(torch.bfloat16).pin_memory()
        oh = torch.full((B, D), float("nan"), dtype=torch.float32).pin_memory()
        layer.decode_host_ptr(xh.data_ptr(), oh.data_ptr(), B, cfg)
        plan_h = layer.last_plan(B, cfg)
        xd = xh.cuda()
        od = torch.empty(B, D, dtype=torch.float32, device="cuda")
        layer.decode(xd, cfg, od)
        layer.ctx.synchronize()
        plan_d = layer.last_plan(B, cfg)
        assert np.array_equal(plan_h["sets"], plan_d["sets"])
        assert np.array_equal(plan_h["weights"], plan_d["weights"])
        assert torch.equal(oh, od.cpu()), f"call {it}"
