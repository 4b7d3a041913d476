"""Host-buffer decode: fresh pinned buffers per call vs one reused pair, vs
the device-resident graph (the e2e overhead breakdown)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_02237_b200 as oea
D, H, N, B = 2048, 768, 128, 16
L = oea.DeviceMoeLayer(D, H, N, "bf16"); L.init_random(1)
cfg = oea.RoutingConfig.simplified(4, 8)
xh = torch.randn(64, B, D).to(torch.bfloat16).pin_memory()
oh = torch.empty(B, D, dtype=torch.float32).pin_memory()
xd = xh[0].cuda(); od = torch.empty(B, D, device="cuda")
g = L.graph(xd, cfg, od)
def timeit(f, n=300):
    for i in range(30): f(i)
    t0 = time.perf_counter()
    for i in range(n): f(i)
    return (time.perf_counter() - t0) * 1e6 / n
print("host, rotating x buffers", timeit(lambda i: L.decode_host_ptr(xh[i % 64].data_ptr(), oh.data_ptr(), B, cfg)))
print("host, one x buffer      ", timeit(lambda i: L.decode_host_ptr(xh[0].data_ptr(), oh.data_ptr(), B, cfg)))
print("device graph + sync     ", timeit(lambda i: (g.launch(), L.ctx.synchronize())))
import ctypes as C
from paper_2511_02237_b200._capi import lib
cc = cfg.to_c()
fn = lib().oea_moe_decode_host
args = (L.ctx.h, L.h, C.c_void_p(xh[0].data_ptr()), None, B, C.byref(cc), C.c_void_p(oh.data_ptr()))
print("raw ctypes, prebuilt args", timeit(lambda i: fn(*args)))
print("cfg.to_c() alone         ", timeit(lambda i: cfg.to_c()))
