"""C5 route timing (bench.py's c5 extra: B=4096 x N=128 fp64, graph of K calls) in one line."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

r = bench.c5_extra(torch, 5, 50)
print((sys.argv[1] if len(sys.argv) > 1 else "") + " | " +
      " ".join(f"k0={p['k0']}:{p['us']:.2f}us" for p in r["sweep"]), flush=True)
