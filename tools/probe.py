"""Quick device timing probe of the fused decode (not the bench contract)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_02237_b200 as oea

D, H, N, B = [int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (2048, 768, 128, 16))]
R = 4
layers = []
for r in range(R):
    L = oea.DeviceMoeLayer(D, H, N, "bf16"); L.init_random(r + 1); layers.append(L)
ctx = layers[0].ctx
xs = [torch.randn(B, D, device="cuda").to(torch.bfloat16) for _ in range(R)]
out = torch.empty(B, D, device="cuda", dtype=torch.float32)
torch.cuda.synchronize()
for name, cfg in [("vanilla", oea.RoutingConfig.vanilla(8)), ("oea_k0=4", oea.RoutingConfig.simplified(4, 8))]:
    gs = [layers[r].graph(xs[r], cfg, out) for r in range(R)]
    s = torch.cuda.ExternalStream(ctx.stream)
    for i in range(10): gs[i % R].launch()
    ctx.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    iters = 200
    with torch.cuda.stream(s):
        e0.record(s)
        for i in range(iters): gs[i % R].launch()
        e1.record(s)
    ctx.synchronize()
    us = e0.elapsed_time(e1) * 1000 / iters
    Ts = []
    for r in range(R):
        layers[r].decode(xs[r], cfg, out); ctx.synchronize()
        Ts.append(layers[r].last_plan(B, cfg)["active_count"])
    T = sum(Ts) / len(Ts)
    bytes_ = T * 3 * D * H * 2 + D * N * 2
    print(f"{name}: {us:.1f} us/call  T~{T:.1f}  {bytes_/us/1e3:.0f} GB/s")
