"""Expert parallelism host logic (paper_2511_02237_b200/ep.py) on CPU: block
ownership against the C ABI's oea_ep_owner, and the all-gather -> shard
partial mixture -> reduce-scatter orchestration over a world-size-2 gloo
group, with the CPU oracle standing in for the shard's CUDA decode (test
infrastructure only): the reduced outputs equal the unsharded oracle layer."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2511_02237_b200 import ep
from paper_2511_02237_b200._capi import lib


@pytest.mark.parametrize("N,P", [(128, 1), (128, 2), (128, 4), (128, 8), (30, 4), (7, 3)])
def test_expert_ranges_match_ep_owner(N, P):
    covered = []
    for r in range(P):
        e0, e1 = ep.ep_expert_range(N, P, r)
        covered += list(range(e0, e1))
        for e in range(e0, e1):
            assert lib().oea_ep_owner(N, P, e) == r
    assert covered == list(range(N))


def test_token_ranges():
    assert [ep.ep_token_range(16, 4, r) for r in range(4)] == [(0, 4), (4, 8), (8, 12), (12, 16)]
    with pytest.raises(ValueError):
        ep.ep_token_range(10, 4, 0)


D, H, N, B = 64, 96, 16, 8
CFG = (3, 4, 2, 1.0, 4, 0, 0)  # simplified(k0=2, k=4)


def _oracle_partial(x_all, owned, layer):
    router, wg, wu, wd = layer
    plan = oracle.route(oracle.router_scores(x_all, router), CFG)
    w = plan.weights.copy()
    for t in range(x_all.shape[0]):
        for j in range(plan.set_len[t]):
            if not owned[0] <= plan.sets[t, j] < owned[1]:
                w[t, j] = 0.0
    return oracle.moe_forward(wg, wu, wd, x_all, plan.sets, plan.set_len, w)


def _worker(rank, world, port, layer, x, want, results, kind="ag_rs"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        owned = ep.ep_expert_range(N, world, rank)

        def fn(x_all, out_partial):
            out_partial.copy_(torch.from_numpy(_oracle_partial(x_all.numpy(), owned, layer)))
        cls = {"ag_rs": ep.ExpertParallelMoE, "a2a": ep.AllToAllExpertParallelMoE}[kind]
        moe = cls(fn, world, rank, dist)
        t0, t1 = ep.ep_token_range(B, world, rank)
        x_local = torch.from_numpy(x[t0:t1].copy())
        out_local = torch.empty((t1 - t0, D), dtype=torch.float64)
        moe.forward(x_local, out_local,
                    x_all=torch.empty((B, D), dtype=torch.float64),
                    partial=torch.empty((B, D), dtype=torch.float64))
        err = float(np.max(np.abs(out_local.numpy() - want[t0:t1])))
        results[rank] = err
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,kind", [(2, "ag_rs"), (2, "a2a"), (4, "a2a")])
def test_ep_orchestration_gloo(world, kind):
    layer = oracle.make_random_layer(D, H, N, 3)
    x = oracle.make_random_batch(B, D, 17)
    router, wg, wu, wd = layer
    plan = oracle.route(oracle.router_scores(x, router), CFG)
    want = oracle.moe_forward(wg, wu, wd, x, plan.sets, plan.set_len, plan.weights)
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), layer, x, want, results, kind), nprocs=world,
             join=True)
    assert sorted(results.keys()) == list(range(world))
    for r, err in results.items():
        assert err < 1e-12, (r, err)
