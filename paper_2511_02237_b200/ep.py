"""Expert parallelism for the Qwen3-235B-shaped MoE stack (BASELINE C4,
SURVEY §8(e)): one process per GPU, experts sharded in contiguous blocks
(rank r holds experts [N r / P, N (r+1) / P), `oea_ep_owner`), tokens in a
data-parallel layout (B / P per rank).

Per MoE layer (one decode step of the stack):
  1. all-gather the ranks' token rows (bf16, B x D; 128 KiB at C4) over NCCL;
  2. every rank runs the fused single-launch decode on its shard
     (`DeviceMoeLayer(..., experts=(e0, e1))`): the full router routes the
     whole batch identically on every rank — the batch union, the per-token
     sets and gate weights are bit-identical to the single-GPU plan — and the
     grouped SwiGLU streams only the held active experts' weights, writing
     this rank's partial mixture out_r[t] = sum_{j in S_t held by r} w_j y_j;
  3. reduce-scatter (sum) of the B x D fp32 partials returns each rank the
     outputs of its own tokens.
Per-rank latency is driven by max_r T_r, the most active experts any rank
holds (PAPER §7).

The collectives are torch.distributed (backend "nccl" on the GPUs, "gloo" for
the CPU tests of this orchestration); the expert compute is a callable so the
orchestration is testable without a GPU.
"""
from __future__ import annotations

from typing import Callable, List, Optional

__all__ = ["ep_expert_range", "ep_token_range", "ExpertParallelMoE", "AllToAllExpertParallelMoE",
           "PeerExpertParallelMoE", "make_ep_layer"]


def ep_expert_range(n_experts: int, world: int, rank: int):
    """Experts [floor(N r / P), floor(N (r+1) / P)) of rank r (the block
    ownership of `oea_ep_owner`)."""
    if n_experts < 1 or world < 1 or not 0 <= rank < world:
        raise ValueError("ep_expert_range: need N >= 1, P >= 1, 0 <= rank < P")
    return (n_experts * rank) // world, (n_experts * (rank + 1)) // world


def ep_token_range(batch: int, world: int, rank: int):
    """Tokens [B r / P, B (r+1) / P) of rank r (data-parallel layout; B % P == 0)."""
    if batch % world != 0:
        raise ValueError("ep_token_range: the batch must split evenly over the EP group")
    per = batch // world
    return per * rank, per * (rank + 1)


class ExpertParallelMoE:
    """One rank's view of an expert-parallel MoE layer.

    partial_fn(x_all, out_partial) computes this rank's partial mixture for the
    whole batch x_all [B, D] into out_partial [B, D] (fp32); on the GPU it is
    the shard layer's decode (`from_shard`)."""

    def __init__(self, partial_fn: Callable, world: int, rank: int, dist=None, group=None):
        self.partial_fn = partial_fn
        self.world, self.rank = int(world), int(rank)
        self.dist, self.group = dist, group

    @classmethod
    def from_shard(cls, layer, cfg, world, rank, dist=None, group=None):
        """The GPU path: `layer` is a DeviceMoeLayer shard holding
        ep_expert_range(N, world, rank)."""
        want = ep_expert_range(layer.N, world, rank)
        if tuple(layer.experts) != want:
            raise ValueError(f"shard holds experts {layer.experts}, rank {rank} of {world} owns {want}")

        def fn(x_all, out_partial):
            from .moe_layer import torch_stream
            # on the caller's current stream: ordered with the NCCL collectives
            layer.decode(x_all, cfg, out_partial, stream=torch_stream())
        return cls(fn, world, rank, dist, group)

    def forward(self, x_local, out_local, x_all=None, partial=None):
        """x_local [B/P, D] (this rank's tokens) -> out_local [B/P, D] fp32.
        x_all / partial: optional preallocated [B, D] buffers."""
        import torch
        B = x_local.shape[0] * self.world
        D = x_local.shape[1]
        if x_all is None:
            x_all = torch.empty((B, D), dtype=x_local.dtype, device=x_local.device)
        if partial is None:
            partial = torch.empty((B, D), dtype=torch.float32, device=x_local.device)
        if self.world == 1:
            self.partial_fn(x_local, out_local)  # the whole batch is local
            return out_local
        self.dist.all_gather_into_tensor(x_all, x_local.contiguous(), group=self.group)
        self.partial_fn(x_all, partial)
        self.dist.reduce_scatter_tensor(out_local, partial, op=self.dist.ReduceOp.SUM,
                                        group=self.group)
        return out_local


class AllToAllExpertParallelMoE(ExpertParallelMoE):
    """The same EP layer with NCCL all-to-all token dispatch and combine
    (BASELINE C4's "NCCL all-to-all dispatch/combine"):

      dispatch  all_to_all_single: rank r sends its B/P token rows to every
                rank. OEA's union is batch-global (routing.cpp:262-266: the
                piggyback pool is the union of ALL tokens' base sets), so every
                expert owner routes the whole batch and needs every token: the
                dispatch payload is the whole batch, split by source rank.
      compute   the shard decode of the whole batch (partial mixture over the
                held experts, plan bit-identical on every rank).
      combine   all_to_all_single of the fp32 partials: rank r sends rows
                [B o / P, B (o+1) / P) to their owner o; the owner sums the P
                received slabs in source-rank order (deterministic, no float
                atomics), the same sum the reduce-scatter path computes.
    """

    def forward(self, x_local, out_local, x_all=None, partial=None, recv=None):
        import torch
        P = self.world
        rows, D = x_local.shape
        B = rows * P
        if self.world == 1:
            self.partial_fn(x_local, out_local)
            return out_local
        if x_all is None:
            x_all = torch.empty((B, D), dtype=x_local.dtype, device=x_local.device)
        if partial is None:
            partial = torch.empty((B, D), dtype=torch.float32, device=x_local.device)
        if recv is None:
            recv = torch.empty((P, rows, D), dtype=partial.dtype, device=x_local.device)
        # dispatch: the same B/P rows to each of the P destinations
        send = x_local.contiguous().unsqueeze(0).expand(P, rows, D).reshape(B, D)
        self.dist.all_to_all_single(x_all, send, group=self.group)
        self.partial_fn(x_all, partial)
        # combine: slab o of the partials goes to owner o; slab r received = rank r's
        self.dist.all_to_all_single(recv.view(B, D), partial, group=self.group)
        torch.sum(recv, dim=0, out=out_local)
        return out_local


def make_ep_layer(kind: str, layer, cfg, world: int, rank: int, dist=None, group=None):
    """The GPU EP layer of one data path: "ag_rs" (NCCL all-gather +
    reduce-scatter), "a2a" (NCCL all-to-all dispatch / combine)."""
    cls = {"ag_rs": ExpertParallelMoE, "a2a": AllToAllExpertParallelMoE}[kind]
    return cls.from_shard(layer, cfg, world, rank, dist, group)


def residual_stack_forward(layers: List[ExpertParallelMoE], h_local, out_local,
                           bufs: Optional[dict] = None, eps: float = 1e-6):
    """A decode step through a pre-norm residual stack of EP MoE layers (the
    MoE half of a Qwen3 decoder layer, attention omitted): for each layer
    x = RMSNorm(h) (bf16), h += moe(x). h_local [B/P, D] fp32 is updated in
    place; keeps activations at unit scale through any depth. On the GPU the
    residual add and the next layer's RMSNorm are one fused launch
    (oea_residual_rmsnorm); elsewhere (CPU tests) plain torch ops."""
    import torch
    if h_local.is_cuda:
        import ctypes as C
        from ._capi import default_context, lib
        from .moe_layer import torch_stream
        ctx = default_context()
        rows, D = h_local.shape
        x = torch.empty((rows, D), dtype=torch.bfloat16, device=h_local.device)
        st = C.c_void_p(torch_stream())
        ctx.check(lib().oea_residual_rmsnorm(ctx.h, h_local.data_ptr(), None, x.data_ptr(), rows,
                                             D, eps, st))
        for i, L in enumerate(layers):
            L.forward(x, out_local, **(bufs or {}))
            if i + 1 < len(layers):
                ctx.check(lib().oea_residual_rmsnorm(ctx.h, h_local.data_ptr(), out_local.data_ptr(),
                                                     x.data_ptr(), rows, D, eps, st))
            else:
                h_local.add_(out_local)
        return h_local
    for L in layers:
        x = (h_local * torch.rsqrt(h_local.pow(2).mean(dim=1, keepdim=True) + eps)).to(torch.bfloat16)
        L.forward(x, out_local, **(bufs or {}))
        h_local.add_(out_local)
    return h_local


def stack_forward(layers: List[ExpertParallelMoE], x_local, out_local, cast=None,
                  bufs: Optional[dict] = None):
    """A decode step through a stack of EP MoE layers: x_{l+1} = out_l (cast
    back to the activation dtype). Returns the last layer's fp32 output."""
    import torch
    x = x_local
    for i, L in enumerate(layers):
        L.forward(x, out_local, **(bufs or {}))
        if i + 1 < len(layers):
            x = out_local.to(x_local.dtype) if cast is None else cast(out_local)
    return out_local


class PeerExpertParallelMoE:
    """One rank's EP MoE layer with the combine fused into the decode kernel
    over peer memory (NVLink / NVSwitch): no NCCL on the data path after the
    token all-gather. The shard kernel's combine stores each token's partial
    mixture straight into the token owner's receive buffer and bumps the
    owner's arrival counter; the owner then sums the `world` slots in rank
    order (oea_ep_combine). Buffers come from oea_device_alloc and are mapped
    into the other ranks with CUDA IPC (`connect`), or, for a single-process
    emulation of the group on one GPU, shared directly (`emulate_group`).

    Reuse contract: each owner has ONE receive buffer, so a rank must not
    start its next `partial` before every owner's `combine` of the current
    launch has read it. The per-layer token all-gather that produces the next
    x_all (a collective over the group) orders this in the decode stack; a
    caller that replays partial / combine back to back without such a
    collective must put a group barrier between launches."""

    def __init__(self, layer, cfg, world: int, rank: int, B: int):
        import ctypes as C
        from ._capi import default_context, lib
        if B % world != 0:
            raise ValueError("PeerExpertParallelMoE: B must split evenly over the EP group")
        self.layer, self.cfg, self.world, self.rank, self.B = layer, cfg, world, rank, B
        self.tpr, self.D = B // world, layer.D
        self.ctx = default_context()
        self._lib = lib()
        recv, cnt = C.c_void_p(), C.c_void_p()
        self.ctx.check(self._lib.oea_device_alloc(self.ctx.h, world * self.tpr * self.D * 4,
                                                  C.byref(recv)))
        self.ctx.check(self._lib.oea_device_alloc(self.ctx.h, 64, C.byref(cnt)))
        self.recv_local, self.cnt_local = recv.value, cnt.value
        self.recv_ptrs = [0] * world
        self.cnt_ptrs = [0] * world
        self.recv_ptrs[rank], self.cnt_ptrs[rank] = self.recv_local, self.cnt_local
        self._opened = []

    def handles(self):
        """64-byte IPC handles of (receive buffer, counter)."""
        import ctypes as C
        out = []
        for p in (self.recv_local, self.cnt_local):
            h = (C.c_char * 64)()
            self.ctx.check(self._lib.oea_ipc_get_handle(self.ctx.h, C.c_void_p(p), h))
            out.append(bytes(h))
        return out

    def connect(self, dist, group=None):
        """Exchange IPC handles over torch.distributed and map every peer's
        receive buffer and counter (one process per GPU)."""
        import ctypes as C
        allh = [None] * self.world
        dist.all_gather_object(allh, self.handles(), group=group)
        for r, (hr, hc) in enumerate(allh):
            if r == self.rank:
                continue
            pr, pc = C.c_void_p(), C.c_void_p()
            self.ctx.check(self._lib.oea_ipc_open_handle(self.ctx.h, C.c_char_p(hr), C.byref(pr)))
            self.ctx.check(self._lib.oea_ipc_open_handle(self.ctx.h, C.c_char_p(hc), C.byref(pc)))
            self.recv_ptrs[r], self.cnt_ptrs[r] = pr.value, pc.value
            self._opened += [pr.value, pc.value]

    @staticmethod
    def emulate_group(members):
        """Single-GPU emulation: every member sees the others' buffers."""
        for m in members:
            m.recv_ptrs = [o.recv_local for o in members]
            m.cnt_ptrs = [o.cnt_local for o in members]

    def partial(self, x_all, stream=None):
        """This rank's shard decode of the whole batch; its combine writes
        the owners' receive buffers."""
        import ctypes as C
        from .moe_layer import torch_stream
        recv = (C.c_void_p * self.world)(*self.recv_ptrs)
        cnt = (C.c_void_p * self.world)(*self.cnt_ptrs)
        st = stream if stream is not None else torch_stream()
        self.ctx.check(self._lib.oea_moe_decode_ep_partial(
            self.ctx.h, self.layer.h, C.c_void_p(x_all.data_ptr()), self.B, self.cfg.c_ref(),
            self.world, self.rank, recv, cnt, C.c_void_p(st)))

    def combine(self, out_local, stream=None):
        """Owner side: wait for every rank's partials of this launch, then
        out_local [B / world][D] = sum over ranks in rank order."""
        import ctypes as C
        from .moe_layer import torch_stream
        st = stream if stream is not None else torch_stream()
        self.ctx.check(self._lib.oea_ep_combine(
            self.ctx.h, C.c_void_p(self.recv_local), C.c_void_p(self.cnt_local), self.world,
            self.tpr, self.D, C.c_void_p(out_local.data_ptr()), C.c_void_p(st)))

    def forward(self, x_all, out_local, stream=None):
        """x_all [B, D] bf16 (the all-gathered batch) -> out_local [B/world, D]."""
        self.partial(x_all, stream)
        self.combine(out_local, stream)
        return out_local

    def close(self):
        import ctypes as C
        for p in self._opened:
            self._lib.oea_ipc_close_handle(self.ctx.h, C.c_void_p(p))
        for p in (self.recv_local, self.cnt_local):
            self._lib.oea_device_free(self.ctx.h, C.c_void_p(p))
        self._opened, self.recv_local, self.cnt_local = [], 0, 0
