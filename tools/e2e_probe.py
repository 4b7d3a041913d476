"""Breakdown of the end-to-end (host buffers) decode latency, C1 shape."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_02237_b200 as oea
from paper_2511_02237_b200._capi import lib
D, H, N, B = 2048, 768, 128, 16
Ls = [oea.DeviceMoeLayer(D, H, N, "bf16") for _ in range(4)]
for i, L in enumerate(Ls): L.init_random(i + 1)
cfg = oea.RoutingConfig.simplified(4, 8)
xh = torch.randn(64, B, D).to(torch.bfloat16).pin_memory()
oh = torch.empty(B, D, dtype=torch.float32).pin_memory()
xd = xh.cuda(); od = torch.empty(B, D, device="cuda")
ctx = Ls[0].ctx
def timeit(f, n=200):
    for i in range(20): f(i)
    t0 = time.perf_counter()
    for i in range(n): f(i)
    return (time.perf_counter() - t0) * 1e6 / n
print("ctypes no-op (oea_last_error)", timeit(lambda i: lib().oea_last_error(ctx.h)))
print("sync only", timeit(lambda i: ctx.synchronize()))
def dev(i):
    Ls[i % 4].decode(xd[i % 64], cfg, od); ctx.synchronize()
print("device decode + sync", timeit(dev))
def host(i):
    Ls[i % 4].decode_host_ptr(xh[i % 64].data_ptr(), oh.data_ptr(), B, cfg)
print("host decode (C ABI)", timeit(host))
s = torch.cuda.ExternalStream(ctx.stream)
def h2d(i):
    with torch.cuda.stream(s):
        xd[0].copy_(xh[i % 64], non_blocking=True)
    ctx.synchronize()
print("H2D 64 KB + sync", timeit(h2d))
def d2h(i):
    with torch.cuda.stream(s):
        oh.copy_(od, non_blocking=True)
    ctx.synchronize()
print("D2H 128 KB + sync", timeit(d2h))
gs = [Ls[i % 4].graph(xd[i % 64], cfg, od) for i in range(64)]
def gl(i):
    gs[i % 64].launch(); ctx.synchronize()
print("graph decode + sync", timeit(gl))
def cpu_cost(f, n=200):
    tot = 0.0
    for i in range(n):
        ctx.synchronize()
        t0 = time.perf_counter(); f(i); tot += time.perf_counter() - t0
    ctx.synchronize()
    return tot * 1e6 / n
print("CPU submit: eager decode", cpu_cost(lambda i: Ls[i % 4].decode(xd[i % 64], cfg, od)))
print("CPU submit: graph launch", cpu_cost(lambda i: gs[i % 64].launch()))
cc = cfg.to_c()
import ctypes as C
def raw(i):
    lib().oea_moe_decode(ctx.h, Ls[i % 4].h, C.c_void_p(xd[i % 64].data_ptr()), None, B, C.byref(cc), C.c_void_p(od.data_ptr()), None)
print("CPU submit: raw ctypes decode", cpu_cost(raw))
