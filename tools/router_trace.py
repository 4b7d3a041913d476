"""Per-CTA stamps of the two-kernel path's router cluster (k_router_fused,
OEA_FFN_TRACE=1) at the C1 shape for a config outside the fused prologue
(p < 1 by default; CFG=maxp for max_p < N), plus the event-timed router
stage (stage graph) in µs.

  python tools/router_trace.py
"""
import ctypes as C
import os
import sys

os.environ["OEA_FFN_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_02237_b200 as oea  # noqa: E402
from paper_2511_02237_b200._capi import lib  # noqa: E402

D, H, N, B = 2048, 768, 128, int(os.environ.get("B", "16"))
cfg = {"mass": oea.RoutingConfig.oea(4, 0.5, 8, 128, 8),
       "maxp": oea.RoutingConfig.oea(4, 1.0, 8, 24, 8)}[os.environ.get("CFG", "mass")]
L = oea.DeviceMoeLayer(D, H, N, "bf16")
L.init_random(1)
ctx = L.ctx
x = (torch.randn(B, D, device="cuda") * 2).to(torch.bfloat16)
out = torch.empty(B, D, device="cuda", dtype=torch.float32)
for _ in range(3):
    L.decode(x, cfg, out)
ctx.synchronize()
buf = np.zeros(8192, np.uint64)
ctx.check(lib().oea_debug_ffn_trace(ctx.h, buf.ctypes.data_as(C.c_void_p), buf.size))
r = buf[1000 * 8:1009 * 8].reshape(9, 8).astype(np.int64)
t0 = r[:8, 0][r[:8, 0] > 0].min()
names = ["start", "GEMV first pass", "GEMV done", "cluster sync", "logits reduced", "routed", "compacted"]
for sl, nm in enumerate(names):
    a = r[:8, sl]
    a = a[a > 0]
    if a.size:
        v = (a - t0) / 1e3
        print(f"  {nm:18s} min {v.min():6.2f} med {np.median(v):6.2f} max {v.max():6.2f}")
for sl, nm in ((1, "CTA0 phase1 done"), (2, "union sync"), (3, "phase2 done")):
    if r[8, sl] > 0:
        print(f"  {nm:18s} {(r[8, sl] - t0) / 1e3:6.2f}")
# the event-timed stage graphs (router | FFN)
gr, gf = L.stage_graphs(x, cfg, out)
stream = torch.cuda.ExternalStream(ctx.stream)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
rs, fs = [], []
for i in range(20):
    with torch.cuda.stream(stream):
        ev[0].record(stream)
        gr.launch()
        ev[1].record(stream)
        gf.launch()
        ev[2].record(stream)
    ev[2].synchronize()
    rs.append(ev[0].elapsed_time(ev[1]) * 1e3)
    fs.append(ev[1].elapsed_time(ev[2]) * 1e3)
print(f"router stage {np.median(rs[5:]):.2f} us, FFN stage {np.median(fs[5:]):.2f} us")
