"""Graph-timed per-call latency vs the kernel's own span (globaltimer trace)
for one fixed layer/batch: the difference is launch gap + CTA start."""
import os, sys, ctypes as C
os.environ["OEA_FFN_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2511_02237_b200 as oea
from paper_2511_02237_b200._capi import lib
D, H, N, B = 2048, 768, 128, 16
Ls = [oea.DeviceMoeLayer(D, H, N, "bf16") for _ in range(4)]
for i, L in enumerate(Ls): L.init_random(i + 1)
torch.manual_seed(0)
x = torch.randn(B, D, device="cuda").to(torch.bfloat16)
out = torch.empty(B, D, device="cuda", dtype=torch.float32)
cfg = oea.RoutingConfig.simplified(4, 8)
gs = [Ls[i % 4].graph(x, cfg, out) for i in range(60)]
for g in gs[:10]: g.launch()
torch.cuda.synchronize()
s = torch.cuda.ExternalStream(Ls[0].ctx.stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for g in gs[10:]: g.launch()
e1.record(s); e1.synchronize()
print("graph per call us", e0.elapsed_time(e1) * 1000 / 50)
spans = []
for rep in range(8):
    for L in Ls: L.decode(x, cfg, out)
    Ls[0].ctx.synchronize()
    buf = np.zeros(8 * 1024, np.uint64)
    Ls[0].ctx.check(lib().oea_debug_ffn_trace(Ls[0].ctx.h, buf.ctypes.data_as(C.c_void_p), buf.size))
    t = buf[:148 * 16].reshape(148, 16).astype(np.int64)
    spans.append([(t[:, c].max() - t[:, 0].min()) / 1000 for c in (4, 3, 9, 10, 2, 15)])
print("kernel span us (last call): producers done / warp0 done / all warps done / barrier passed / bar.sync / combine done",
      np.median(np.array(spans), axis=0), "T", Ls[3].last_plan(B, cfg)["active_count"])
