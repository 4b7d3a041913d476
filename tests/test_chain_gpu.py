"""Launch structure of the hot path on the GPU: the PDL-chained graph of
consecutive decode calls (oea_decode_chain_graph_create) and the persistent
cooperative launch next to other work.

* chain graph: K calls over rotating layers / batches in one graph equal the
  same calls made one by one (bit-identical outputs: the programmatic edges
  do not change what each call computes), replayed twice, and the last
  call's plan is the oracle's routing of its logits;
* a decode issued while a long GEMM stream occupies the SMs on another
  stream completes and equals the decode on an idle GPU (the grid-wide spin
  barriers need every CTA resident: the cooperative launch waits for the
  SMs instead of starting a partial grid).
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _layers(oea, n, D=1024, H=512, N=64):
    out = []
    for i in range(n):
        L = oea.DeviceMoeLayer(D, H, N, "bf16")
        L.init_random(40 + i)
        out.append(L)
    return out


@pytest.mark.parametrize("B,policy", [(16, "oea"), (16, "vanilla"), (5, "oea"), (32, "oea")])
def test_chain_graph_equals_calls_one_by_one(oea, B, policy):
    import torch
    layers = _layers(oea, 3)
    D = layers[0].D
    K = 7
    cfg = oea.RoutingConfig.simplified(4, 8) if policy == "oea" else oea.RoutingConfig.vanilla(8)
    gen = torch.Generator(device="cuda").manual_seed(B)
    xs = torch.randn(K, B, D, device="cuda", generator=gen).to(torch.bfloat16)
    want = []
    for i in range(K):
        o = torch.empty(B, D, device="cuda", dtype=torch.float32)
        layers[i % 3].decode(xs[i], cfg, o)
        layers[0].ctx.synchronize()
        want.append(o.clone())
    outs = [torch.full((B, D), float("nan"), device="cuda") for _ in range(K)]
    g = oea.DeviceMoeLayer.chain_graph([layers[i % 3] for i in range(K)], list(xs), cfg, outs)
    for _ in range(2):
        g.launch()
    layers[0].ctx.synchronize()
    for i in range(K):
        assert torch.equal(outs[i], want[i]), i
    plan = layers[(K - 1) % 3].last_plan(B, cfg)
    ref = oracle.route(oracle.softmax_rows(plan["logits"].astype(np.float64)), cfg)
    for t in range(B):
        assert list(plan["sets"][t, : plan["set_len"][t]]) == ref.set_list(t)
    g.close()


def test_decode_next_to_a_long_kernel_on_another_stream(oea):
    import torch
    (L,) = _layers(oea, 1, D=2048, H=768, N=128)
    B = 16
    cfg = oea.RoutingConfig.simplified(4, 8)
    x = torch.randn(B, L.D, device="cuda").to(torch.bfloat16)
    idle = torch.empty(B, L.D, device="cuda", dtype=torch.float32)
    L.decode(x, cfg, idle)
    L.ctx.synchronize()
    side = torch.cuda.Stream()
    a = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    busy = torch.empty_like(idle)
    for _ in range(3):
        with torch.cuda.stream(side):
            for _ in range(20):  # tens of ms of GEMMs on every SM
                a = torch.tanh(a @ a * 1e-3)
        L.decode(x, cfg, busy)  # the context's own stream, concurrently
        L.ctx.synchronize()
        torch.cuda.synchronize()
        assert torch.equal(busy, idle)
