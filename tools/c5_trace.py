"""Per-CTA stamps of the single-launch route (OEA_FFN_TRACE=1), C5 shape."""
import os
import sys
import ctypes as C

os.environ["OEA_FFN_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "c5_probe.py")).read())
from paper_2511_02237_b200._capi import lib as _lib  # noqa: E402
buf = np.zeros(8192, np.uint64)
ctx.check(_lib().oea_debug_ffn_trace(ctx.h, buf.ctypes.data_as(C.c_void_p), buf.size))
t = buf[:256 * 8].reshape(256, 8).astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
names = ["start", "phase1 picks", "arrived", "barrier passed", "spec picks+sets", "loads flushed", "keys loaded", "sorted"]
for sl, nm in enumerate(names):
    a = t[:, sl]
    a = a[a > 0]
    if a.size:
        r = (a - t0) / 1e3
        print(f"{nm:22s} n={a.size:3d} min {r.min():7.2f} med {np.median(r):7.2f} max {r.max():7.2f}")
