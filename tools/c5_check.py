"""Fused single-launch route vs the plan's own sets: loads / union / total."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2511_02237_b200 as oea  # noqa: E402

rng = np.random.default_rng(3)
for B, N in ((16, 64), (64, 64), (4096, 128), (300, 128)):
    s = rng.random((B, N))
    s /= s.sum(1, keepdims=True)
    plan = oea.route(s, oea.RoutingConfig.simplified(3, 8))
    want = np.zeros(N, np.int64)
    for i in range(B):
        for e in plan.sets[i]:
            want[e] += 1
    bad = np.nonzero(want != np.asarray(plan.loads))[0]
    print(B, N, "loads ok" if bad.size == 0 else f"loads BAD at {bad[:10]} want {want[bad[:10]]} got {np.asarray(plan.loads)[bad[:10]]}",
          "total", plan.total_load, int(want.sum()))
