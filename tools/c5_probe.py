import sys; sys.path.insert(0, "/root/repo")
import torch, ctypes as C
import paper_2511_02237_b200 as oea
from paper_2511_02237_b200._capi import PlanViewC, lib, default_context
ctx = default_context()
Bc, Nc = 4096, 128
scores = torch.softmax(torch.randn(Bc, Nc, device="cuda", dtype=torch.float64), dim=1)
cfg = oea.RoutingConfig.simplified(4, 8)
stride = oea.plan_set_stride(cfg.resolved(Nc))
sets = torch.empty(Bc, stride, dtype=torch.int32, device="cuda"); set_len = torch.empty(Bc, dtype=torch.int32, device="cuda")
w = torch.empty(Bc, stride, dtype=torch.float64, device="cuda"); loads = torch.empty(Nc, dtype=torch.int32, device="cuda")
au = torch.empty(Nc, dtype=torch.int32, device="cuda"); cnt = torch.empty(1, dtype=torch.int32, device="cuda"); tot = torch.empty(1, dtype=torch.int64, device="cuda")
pv = PlanViewC(stride, sets.data_ptr(), set_len.data_ptr(), w.data_ptr(), None, loads.data_ptr(), au.data_ptr(), cnt.data_ptr(), tot.data_ptr(), None, None, None, None, None)
c = cfg.to_c()
for _ in range(5):
    ctx.check(lib().oea_route_f64(ctx.h, C.c_void_p(scores.data_ptr()), None, Bc, Nc, C.byref(c), C.byref(pv), None))
ctx.synchronize()
