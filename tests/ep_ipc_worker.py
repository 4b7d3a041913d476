"""Worker for tests/test_ep_gpu.py::test_peer_memory_ep_ipc_two_processes:
two processes on the same GPU form a world-2 EP group, exchange CUDA IPC
handles over gloo and run the peer-memory combine (the multi-GPU code path;
on one GPU the two contexts time-slice)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist
    import paper_2511_02237_b200 as oea
    from paper_2511_02237_b200 import ep
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    D, H, N, B = 1024, 512, 64, 16
    cfg = oea.RoutingConfig.simplified(4, 8)
    shard = oea.DeviceMoeLayer(D, H, N, "bf16", experts=ep.ep_expert_range(N, world, rank))
    shard.init_random(11)
    m = ep.PeerExpertParallelMoE(shard, cfg, world, rank, B)
    m.connect(dist)
    g = torch.Generator().manual_seed(5)
    worst = 0.0
    for it in range(2):
        x = torch.randn(B, D, generator=g).to(torch.bfloat16).cuda()  # same batch on every rank
        out = torch.empty(B // world, D, device="cuda")
        m.forward(x, out)
        torch.cuda.synchronize()
        full = oea.DeviceMoeLayer(D, H, N, "bf16")
        full.init_random(11)
        ref = torch.empty(B, D, device="cuda")
        full.decode(x, cfg, ref, stream=oea.moe_layer.torch_stream())
        torch.cuda.synchronize()
        mine = ref[rank * (B // world):(rank + 1) * (B // world)]
        err = ((out - mine).norm(dim=1) / mine.norm(dim=1).clamp_min(1e-12)).max().item()
        worst = max(worst, err)
        full.close()
        dist.barrier()
    m.close()
    dist.barrier()
    print(f"rank {rank} max_rel_err {worst:.3e}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if worst < 1e-5 else 1)


if __name__ == "__main__":
    main()
