"""A few eager decodes at a large batch (for ncu launch lists / captures of
the tcgen05 path): B=$B (256), simplified(k0=$K0 (4), 8) on a C1 layer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_02237_b200 as oea  # noqa: E402

B, K0 = int(os.environ.get("B", "256")), int(os.environ.get("K0", "4"))
L = oea.DeviceMoeLayer(2048, 768, 128, "bf16")
L.init_random(1)
x = torch.randn(B, 2048, device="cuda").to(torch.bfloat16)
out = torch.empty(B, 2048, device="cuda", dtype=torch.float32)
cfg = oea.RoutingConfig.simplified(K0, 8) if K0 < 8 else oea.RoutingConfig.vanilla(8)
for _ in range(int(os.environ.get("REPS", "3"))):
    L.decode(x, cfg, out)
torch.cuda.synchronize()
print("ok", float(out.abs().sum()))
