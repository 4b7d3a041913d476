"""Kernel timeline of the zero-copy host decode vs the device decode (C1)."""
import os, sys, ctypes as C
os.environ["OEA_FFN_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2511_02237_b200 as oea
from paper_2511_02237_b200._capi import lib
D, H, N, B = 2048, 768, 128, 16
L = oea.DeviceMoeLayer(D, H, N, "bf16"); L.init_random(1)
cfg = oea.RoutingConfig.simplified(4, 8)
xh = torch.randn(B, D).to(torch.bfloat16).pin_memory()
oh = torch.empty(B, D, dtype=torch.float32).pin_memory()
xd = xh.cuda(); od = torch.empty(B, D, device="cuda")
names = {0: "start", 8: "gemv start", 5: "gemv done", 6: "union", 4: "prod done", 3: "warp0 done",
         9: "arrive", 10: "passed", 15: "combine done"}
for mode in ("device", "host"):
    res = []
    for rep in range(10):
        if mode == "host":
            L.decode_host_ptr(xh.data_ptr(), oh.data_ptr(), B, cfg)
        else:
            L.decode(xd, cfg, od)
        L.ctx.synchronize()
        buf = np.zeros(8 * 1024, np.uint64)
        L.ctx.check(lib().oea_debug_ffn_trace(L.ctx.h, buf.ctypes.data_as(C.c_void_p), buf.size))
        t = buf[:148 * 16].reshape(148, 16).astype(np.int64)
        res.append([(t[:, c].max() - t[:, 0].min()) / 1000 for c in names])
    print(mode, {n: round(v, 2) for n, v in zip(names.values(), np.median(np.array(res), axis=0))})
