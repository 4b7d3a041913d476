"""Graph-timed C1-shape layer latency for a few batch sizes (A/B helper)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_02237_b200 as oea
D, H, N = 2048, 768, 128
Ls = []
for r in range(4):
    L = oea.DeviceMoeLayer(D, H, N, "bf16"); L.init_random(1 + r); Ls.append(L)
st = torch.cuda.ExternalStream(Ls[0].ctx.stream)
for B in [int(b) for b in os.environ.get("BS", "1,16,32,64,128,256").split(",")]:
    xs = torch.randn(24, B, D, device="cuda").to(torch.bfloat16)
    out = torch.empty(B, D, device="cuda", dtype=torch.float32)
    cfg = oea.RoutingConfig.simplified(4, 8)
    gs = [Ls[i % 4].graph(xs[i], cfg, out) for i in range(24)]
    for g in gs[:4]: g.launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        for g in gs[4:]: g.launch()
        e1.record(st)
    e1.synchronize()
    print(f"B={B:4d}  {e0.elapsed_time(e1) * 1000 / 20:7.1f} us")
    for g in gs: g.close()
