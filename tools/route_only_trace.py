"""Stamp timeline of the route-only prologue launch (B > 64), OEA_FFN_TRACE=1."""
import os
import sys
import ctypes as C

os.environ["OEA_FFN_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_02237_b200 as oea  # noqa: E402
from paper_2511_02237_b200._capi import lib  # noqa: E402

B, K0 = int(os.environ.get("B", "256")), int(os.environ.get("K0", "4"))
L = oea.DeviceMoeLayer(2048, 768, 128, "bf16")
L.init_random(1)
x = torch.randn(B, 2048, device="cuda").to(torch.bfloat16)
out = torch.empty(B, 2048, device="cuda", dtype=torch.float32)
cfg = oea.RoutingConfig.simplified(K0, 8)
for _ in range(6):
    L.decode(x, cfg, out)
torch.cuda.synchronize()
LEG, NL, PER = 8192, 16, 16384
buf = np.zeros(LEG + NL * PER, np.uint64)
L.ctx.check(lib().oea_debug_ffn_trace(L.ctx.h, buf.ctypes.data_as(C.c_void_p), buf.size))
regs = buf[LEG:].reshape(NL, PER).astype(np.int64)
names = {0: "start", 8: "gemv start", 9: "gemv k-loop done (w0)", 10: "gemv partials in smem", 5: "gemv done", 11: "R1 done", 12: "union polled", 13: "union scan",
         6: "union known", 1: "R2 + plan rows out", 7: "compaction + row gather done", 15: "grid exit"}
for r in regs:
    t = r[:148 * 16].reshape(148, 16)
    if t[:, 0].min() <= 0 or t[:, 7].max() <= 0:
        continue
    t0 = t[:, 0].min()
    print("launch:")
    for sl, nm in names.items():
        a = t[:, sl]
        a = a[a > 0]
        if a.size:
            v = (a - t0) / 1e3
            print(f"  {nm:34s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f}  CTA0 {(t[0, sl] - t0) / 1e3:7.2f}")
    break
