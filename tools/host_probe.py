import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2511_02237_b200 as oea
D, H, N, B = 2048, 768, 128, 16
Ls = [oea.DeviceMoeLayer(D, H, N, "bf16") for _ in range(4)]
for i, L in enumerate(Ls): L.init_random(i + 1)
cfg = oea.RoutingConfig.simplified(4, 8)
xh = torch.randn(64, B, D).to(torch.bfloat16).pin_memory()
oh = torch.empty(B, D, dtype=torch.float32).pin_memory()
def timeit(f, n=300):
    for i in range(20): f(i)
    t0 = time.perf_counter()
    for i in range(n): f(i)
    return (time.perf_counter() - t0) * 1e6 / n
print(os.environ.get("OEA_HOST_COPIES"), "host decode", timeit(lambda i: Ls[i % 4].decode_host_ptr(xh[i % 64].data_ptr(), oh.data_ptr(), B, cfg)))
