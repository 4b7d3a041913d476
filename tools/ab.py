"""A/B probe: chained-graph µs per decode call (bench.py's method) for a few
configs, in ONE line, so kernel variants (env switches, read once per
process) can be compared back to back:

  OEA_X=1 python tools/ab.py label
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_02237_b200 as oea  # noqa: E402

D, H, N = 2048, 768, 128
W, K = 5, int(os.environ.get("AB_STEPS", "40"))
layers = []
for r in range(4):
    L = oea.DeviceMoeLayer(D, H, N, "bf16")
    L.init_random(1 + r)
    layers.append(L)
ctx = layers[0].ctx
stream = torch.cuda.ExternalStream(ctx.stream)
res = []
SETS = {"small": ((16, 1), (16, 2), (16, 4), (16, 8), (4, 4), (1, 4)),
        "big": ((128, 4), (128, 8), (256, 4), (256, 8)),
        "mid": ((24, 4), (32, 4), (32, 8), (48, 4), (64, 4), (64, 8))}
for B, k0 in SETS[os.environ.get("AB_SET", "small")]:
    gen = torch.Generator(device="cuda").manual_seed(1234)
    xs = torch.randn(W + K, B, D, device="cuda", generator=gen).to(torch.bfloat16)
    out = torch.empty(B, D, device="cuda", dtype=torch.float32)
    cfg = oea.RoutingConfig.simplified(k0, 8) if k0 < 8 else oea.RoutingConfig.vanilla(8)
    if os.environ.get("AB_CFG") == "mass":  # p < 1 (x scaled so the mass rule cuts)
        cfg, xs = oea.RoutingConfig.oea(k0, 0.5, 8, 128, 8), (xs.float() * 2).to(torch.bfloat16)
    elif os.environ.get("AB_CFG") == "maxp":
        cfg = oea.RoutingConfig.oea(k0, 1.0, 8, 24, 8)
    us, _ = bench.time_chain(torch, stream, layers, xs, cfg, out, W, K, ctx)
    Ts, _ = bench.plan_stats(layers, xs, cfg, out, B, range(W, W + K), ctx)
    res.append(f"B{B}k{k0}: {us:6.2f}us T={np.mean(Ts):5.1f}")
print((sys.argv[1] if len(sys.argv) > 1 else "") + " | " + " | ".join(res), flush=True)
