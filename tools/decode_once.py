"""A few eager decodes of one shape (for ncu launch lists): SHAPE=D,H,N,B K0=k0."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_02237_b200 as oea
D, H, N, B = [int(v) for v in os.environ.get("SHAPE", "2048,768,128,16").split(",")]
k0 = int(os.environ.get("K0", "4"))
L = oea.DeviceMoeLayer(D, H, N, "bf16"); L.init_random(1)
x = torch.randn(B, D, device="cuda").to(torch.bfloat16)
out = torch.empty(B, D, device="cuda", dtype=torch.float32)
torch.cuda.synchronize()
for _ in range(int(os.environ.get("ITERS", "3"))):
    L.decode(x, oea.RoutingConfig.simplified(k0, 8), out)
L.ctx.synchronize()
T = L.last_plan(B, oea.RoutingConfig.simplified(k0, 8))["active_count"]
print(f"T={T} algorithmic_bytes={T * 3 * D * H * 2 + D * N * 2 + B * D * 2 + B * D * 4}")
