"""A few eager decode calls (for ncu): C1 shape, OEA and vanilla, rotating 2 layers."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_02237_b200 as oea
D, H, N, B = [int(v) for v in os.environ.get("SHAPE", "2048,768,128,16").split(",")]
Ls = []
for r in range(2):
    L = oea.DeviceMoeLayer(D, H, N, "bf16"); L.init_random(r + 1); Ls.append(L)
x = torch.randn(B, D, device="cuda").to(torch.bfloat16)
out = torch.empty(B, D, device="cuda", dtype=torch.float32)
torch.cuda.synchronize()
n = int(os.environ.get("ITERS", "4"))
for cfg in (oea.RoutingConfig.simplified(4, 8), oea.RoutingConfig.vanilla(8)):
    for i in range(n):
        Ls[i % 2].decode(x, cfg, out)
    Ls[0].ctx.synchronize()
print("done")
