"""Timeline of one FFN launch per CTA (OEA_FFN_TRACE=1) + stream-only mode."""
import os, sys, ctypes as C
os.environ["OEA_FFN_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2511_02237_b200 as oea
from paper_2511_02237_b200._capi import lib
D, H, N, B = [int(v) for v in os.environ.get("SHAPE", "2048,768,128,16").split(",")]
L = oea.DeviceMoeLayer(D, H, N, "bf16"); L.init_random(1)
L2 = oea.DeviceMoeLayer(D, H, N, "bf16"); L2.init_random(2)
x = torch.randn(B, D, device="cuda").to(torch.bfloat16)
out = torch.empty(B, D, device="cuda", dtype=torch.float32)
torch.cuda.synchronize()
K0 = int(os.environ.get("K0", "4"))
for name, cfg in (("oea", oea.RoutingConfig.simplified(K0, 8)), ("vanilla", oea.RoutingConfig.vanilla(8))):
    # back-to-back calls (no host sync in between, clocks stay up); the trace
    # buffer holds the last call
    for rep in range(int(os.environ.get("REPS", "20"))):
        (L if rep % 2 == 0 else L2).decode(x, cfg, out)
    L.ctx.synchronize()
    buf = np.zeros(8 * 1024, np.uint64)
    L.ctx.check(lib().oea_debug_ffn_trace(L.ctx.h, buf.ctypes.data_as(C.c_void_p), buf.size))
    t = buf[:148 * 16].reshape(148, 16).astype(np.int64)
    base = t[:, 0].min()
    rel = (t - base) / 1000.0
    def st(a): return f"min {a.min():7.1f} med {np.median(a):7.1f} max {a.max():7.1f}"
    print(f"== {name}  (us, relative to first CTA start)")
    print(" start      ", st(rel[:, 0]))
    print(" W1 end     ", st(rel[:, 1]))
    print(" W2 1st rdy ", st(rel[:, 2]))
    print(" end        ", st(rel[:, 3]))
    print(" prod done  ", st(rel[:, 4]))
    if t[:, 5].any():
        print(" fused: gemv start (xpad)  ", st(rel[:, 8]))
        print(" fused: gemv done          ", st(rel[:, 9]))
        print(" fused: barrier arrived    ", st(rel[:, 10]))
        print(" fused: logits barrier passed", st(rel[:, 5]))
        print(" fused: logits in smem     ", st(rel[:, 11]))
        print(" fused: union known (phase 1)", st(rel[:, 6]))
        print(" fused: plan ready (phase 2) ", st(rel[:, 7]))
        if t[:, 12].any():
            print(" fused: union words polled   ", st(rel[:, 12]))
            print(" fused: union ballots done   ", st(rel[:, 13]))
            print(" fused: union syncthreads    ", st(rel[:, 14]))
    r = buf.reshape(1024, 8)[1000:1008].astype(np.int64)
    r0 = r[0, 0]
    print(" router CTA stamps (us from CTA0 start): start, x-staged, gemv, sync1, end-gemv, routed, compacted")
    for k in range(8):
        print("  ", k, [round((v - r0) / 1000.0, 2) if v else None for v in r[k][:7]])
    f = buf.reshape(1024, 8)[1008].astype(np.int64)
    print(" routing detail (us from CTA0 start): sorted, phase1, synced, phase2, route_all done:",
          [round((v - r0) / 1000.0, 2) if v else None for v in f[:5]])
    print(" FFN first start - router CTA0 start:", (t[:, 0].min() - r0) / 1000.0)
