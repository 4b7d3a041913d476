"""The tcgen05 (UMMA + TMEM) grouped FFN of large batches (64 < B <= 256,
umma_ffn.cu) vs the CPU oracle, on the cases its own machinery adds:

  * the per-layer UMMA-layout weight copy is made on first use and refreshed
    after the weights change (init_random / upload_expert mark it stale);
  * a CUDA graph captured BEFORE the first large-batch call cannot allocate
    that copy, so it captures the mma.sync FFN: both must match the oracle;
  * H not a multiple of 128 (padded h columns) and groups of > 64 tokens
    (several token groups per expert, N = round-up-16 of each);
  * masked tokens at a large batch.

Bars as the other decode tests: sets bit-exact vs the oracle on the exported
logits, weights within 1e-5, outputs within 2e-2 relative of
moe_forward<double> (proj/include/oea/moe_layer.hpp:114-158)."""
import numpy as np
import pytest
import torch

import oracle
from test_decode_gpu import OUT_TOL, oracle_output, run_case, to_bf16_bits

pytestmark = pytest.mark.gpu


def _check(oea, layer, x, out, cfg, B, mask=None):
    plan = layer.last_plan(B, cfg)
    m8 = None if mask is None else np.asarray(mask, np.uint8)
    want = oracle.route(oracle.softmax_rows(plan["logits"].astype(np.float64)), cfg, m8)
    for i in range(B):
        assert [int(v) for v in plan["sets"][i, : plan["set_len"][i]]] == want.set_list(i)
    ref = oracle_output(layer, x, want)
    real = np.ones(B, bool) if mask is None else np.asarray(mask, bool)
    _, max_rel = oracle.output_divergence(ref[real], np.asarray(out, np.float64)[real])
    assert max_rel <= OUT_TOL, f"output max relative error {max_rel}"


def test_weight_copy_refreshed_after_reinit_and_upload(oea):
    D, H, N, B = 512, 256, 32, 128
    cfg = oea.RoutingConfig.simplified(3, 8)
    layer = oea.DeviceMoeLayer(D, H, N, dtype="bf16")
    layer.init_random(3)
    x, xbits = to_bf16_bits(oracle.make_random_batch(B, D, 77))
    _check(oea, layer, x, layer.decode_host(xbits, cfg), cfg, B)  # makes the copy
    # the call runs the tcgen05 path: the route-only launch (routing, plan,
    # compaction, token-row gather), k_ffn_umma, the combine
    n0 = layer.ctx.kernel_launches
    layer.decode_host(xbits, cfg)
    assert layer.ctx.kernel_launches - n0 == 3
    layer.init_random(4)                                           # new weights: stale
    _check(oea, layer, x, layer.decode_host(xbits, cfg), cfg, B)
    # one expert re-uploaded with other weights: the copy follows again
    rng = np.random.default_rng(5)
    wg = rng.standard_normal((D, H)) / np.sqrt(D)
    wu = rng.standard_normal((D, H)) / np.sqrt(D)
    wd = rng.standard_normal((H, D)) / np.sqrt(H)
    layer.upload_expert(7, wg, wu, wd)
    _check(oea, layer, x, layer.decode_host(xbits, cfg), cfg, B)
    layer.close()


def test_graph_captured_before_first_use_then_eager(oea):
    D, H, N, B = 512, 256, 64, 96
    cfg = oea.RoutingConfig.simplified(4, 8)
    layer = oea.DeviceMoeLayer(D, H, N, dtype="bf16")
    layer.init_random(11)
    x, xbits = to_bf16_bits(oracle.make_random_batch(B, D, 99))
    xd = torch.from_numpy(xbits.view(np.int16)).view(torch.bfloat16).cuda()
    out_g = torch.empty(B, D, device="cuda", dtype=torch.float32)
    g = layer.graph(xd, cfg, out_g)  # no UMMA copy yet: the mma.sync FFN is captured
    g.launch()
    layer.ctx.synchronize()
    _check(oea, layer, x, out_g.cpu().numpy(), cfg, B)
    out_e = layer.decode_host(xbits, cfg)  # eager: tcgen05 FFN (makes the copy)
    _check(oea, layer, x, out_e, cfg, B)
    g.launch()  # the graph keeps its captured path
    layer.ctx.synchronize()
    _check(oea, layer, x, out_g.cpu().numpy(), cfg, B)
    g.close()
    layer.close()


@pytest.mark.parametrize("D,H,N,B,k0", [(256, 200, 16, 100, 2), (384, 328, 8, 200, 4),
                                        (1024, 512, 128, 256, 1)])
def test_padded_h_and_large_token_groups(oea, D, H, N, B, k0):
    # N = 8 / 16 with B = 100..200: experts with > 64 tokens (several groups)
    run_case(oea, D, H, N, B, oea.RoutingConfig.simplified(k0, min(8, N)), seed=B + k0,
             check_logits=False)


def test_masked_tokens_large_batch(oea):
    rng = np.random.default_rng(8)
    mask = rng.integers(0, 2, size=160).astype(bool)
    run_case(oea, 512, 256, 64, 160, oea.RoutingConfig.vanilla(8), seed=9, mask=mask)


_DENSE_OPT_IN = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
import oracle
import paper_2511_02237_b200 as oea
from test_decode_gpu import OUT_TOL, oracle_output, to_bf16_bits
for D, H, N, B, k0 in ((2048, 768, 128, 16, 4), (512, 256, 32, 1, 2), (1024, 328, 64, 9, 8)):
    cfg = oea.RoutingConfig.simplified(k0, 8) if k0 < 8 else oea.RoutingConfig.vanilla(8)
    layer = oea.DeviceMoeLayer(D, H, N, dtype="bf16")
    layer.init_random(B + k0)
    x, xbits = to_bf16_bits(oracle.make_random_batch(B, D, 50 + B))
    xd = torch.from_numpy(xbits.view(np.int16)).view(torch.bfloat16).cuda()
    out = torch.empty(B, D, device="cuda", dtype=torch.float32)
    layer.decode(xd, cfg, out)
    layer.ctx.synchronize()
    plan = layer.last_plan(B, cfg)
    want = oracle.route(oracle.softmax_rows(plan["logits"].astype(np.float64)), cfg, None)
    for i in range(B):
        assert [int(v) for v in plan["sets"][i, : plan["set_len"][i]]] == want.set_list(i)
    _, rel = oracle.output_divergence(oracle_output(layer, x, want), out.cpu().numpy().astype(np.float64))
    assert rel <= OUT_TOL, (D, H, N, B, rel)
    layer.close()
print("ok")
"""


def test_dense_tcgen05_opt_in():
    # OEA_UMMA_DENSE=1 (read once per process, hence the subprocess): the
    # experimental tcgen05 consumer of the dense decode (MODE 6) vs the oracle
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, OEA_UMMA_DENSE="1")
    r = subprocess.run([sys.executable, "-c", _DENSE_OPT_IN, here], env=env, cwd=os.path.dirname(here),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
