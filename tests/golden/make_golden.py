"""Generates tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref: the
reference sources under /root/reference/proj compiled against the Eigen-subset
shim, unmodified). Run here (the reference tree does not exist on the GPU box):

    make -C oracle && python tests/golden/make_golden.py

The fixtures pin the C restatement (oracle/) and, through it, the GPU kernels.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def cfg_random(rng, n):
    """test_routing.cpp:68-93 random_config (same distribution)."""
    cap = int(rng.integers(0, 2))
    p = 1.0 if rng.integers(0, 2) == 0 else int(rng.integers(1, 9)) / 8.0
    kind = int(rng.integers(0, 4))
    if kind == 0:
        k = int(rng.integers(1, n + 1))
        return (0, k, k, 1.0, k, 0, 0)
    if kind == 1:
        k0 = int(rng.integers(1, n + 1))
        return (1, k0, k0, p, max(k0, k0), 0, 0)
    if kind == 2:
        k0 = int(rng.integers(1, n + 1))
        km = k0 + int(rng.integers(0, n - k0 + 1))
        return (2, km, k0, p, km, int(rng.integers(1, n + 1)), cap)
    k = int(rng.integers(1, n + 1))
    return (3, k, int(rng.integers(1, k + 1)), 1.0, k, 0, cap)


def routing_cases(ref, seed=2511, count=300):
    rng = np.random.default_rng(seed)
    cases = []
    for rep in range(count):
        n = int(rng.integers(1, 40)) if rep % 8 else int(rng.integers(40, 130))
        b = int(rng.integers(1, 24))
        if rep % 3 == 0:  # 1/8-lattice rows: exact ties
            s = np.zeros((b, n))
            for i in range(b):
                for _ in range(8):
                    s[i, rng.integers(0, n)] += 1.0 / 8
        else:
            s = rng.exponential(size=(b, n))
            s /= s.sum(axis=1, keepdims=True)
        if rep % 7 == 0:
            s[:, rng.integers(0, n)] = 0.0
        mask = (rng.random(b) < 0.7).astype(np.uint8) if rep % 5 == 0 else None
        cfg = cfg_random(rng, n)
        try:
            plan = ref.route(s, cfg, mask)
            err = ""
        except (oracle.OracleDomainError, oracle.OracleInvalidArgument) as e:
            plan, err = None, f"{type(e).__name__}:{e}"
        cases.append((s, mask, cfg, plan, err))
    return cases


def main():
    ref = oracle.Reference()
    cases = routing_cases(ref)
    d = {}
    for i, (s, mask, cfg, plan, err) in enumerate(cases):
        d[f"r{i}_scores"] = s
        d[f"r{i}_mask"] = mask if mask is not None else np.zeros(0, np.uint8)
        d[f"r{i}_cfg"] = np.array(cfg, dtype=np.float64)
        d[f"r{i}_err"] = np.array(err)
        if plan is not None:
            d[f"r{i}_sets"] = plan.sets
            d[f"r{i}_set_len"] = plan.set_len
            d[f"r{i}_weights"] = plan.weights
            d[f"r{i}_loads"] = plan.loads
            d[f"r{i}_active"] = plan.active_union
            d[f"r{i}_total"] = np.array(plan.total_load)
    d["n_routing"] = np.array(len(cases))
    # sort_experts on rows with ties and signed zeros
    rng = np.random.default_rng(7)
    s = np.round(rng.random((12, 50)) * 4) / 4
    s[:, ::7] = -0.0
    d["sort_scores"] = s
    d["sort_order"] = ref.sort_experts(s)
    np.savez_compressed(os.path.join(OUT, "routing_golden.npz"), **d)

    # layer cases (moe_layer.hpp): make_random_layer / make_random_batch /
    # router_scores / route / moe_forward<double> and <float>
    L = {}
    for ci, (D, H, N, B, seed, cfg) in enumerate([
            (16, 24, 8, 6, 13, (3, 3, 2, 1.0, 3, 0, 0)),
            (48, 64, 16, 16, 3, (2, 4, 2, 1.0, 4, 0, 0)),
            (32, 48, 12, 5, 9, (0, 4, 4, 1.0, 4, 0, 0))]):
        router, wg, wu, wd = ref.make_random_layer(D, H, N, seed)
        x = ref.make_random_batch(B, D, seed, 2, 1)
        lay = ref.layer(router, wg, wu, wd, "f64")
        sc = lay.router_scores(x)
        plan = ref.route(sc, cfg)
        out64 = lay.moe_forward(x, plan.sets, plan.set_len, plan.weights)
        out32 = ref.layer(router, wg, wu, wd, "f32").moe_forward(x, plan.sets, plan.set_len,
                                                                  plan.weights)
        for k, v in dict(router=router, wg=wg, wu=wu, wd=wd, x=x, scores=sc, sets=plan.sets,
                         set_len=plan.set_len, weights=plan.weights, out64=out64, out32=out32,
                         cfg=np.array(cfg, np.float64), dims=np.array([D, H, N, B, seed])).items():
            L[f"l{ci}_{k}"] = v
    L["n_layer"] = np.array(3)
    np.savez_compressed(os.path.join(OUT, "layer_golden.npz"), **L)
    print("wrote", os.listdir(OUT))


if __name__ == "__main__":
    main()
