"""Python mirror of the reference MoE-layer API (proj/include/oea/moe_layer.hpp)
plus the device-resident decode layer (the hot path).

* ``DeviceMoeLayer`` — weights resident in HBM. bf16 layers use the fused
  router (K2/K3) and the tensor-core grouped SwiGLU FFN (K4/K5); f32/f64
  layers use fp64 router_scores + route_f64 (K1) + the SIMT FFN (K6).
* ``router_scores`` / ``expert_forward`` / ``moe_forward`` — the reference's
  templates over host ``MoeLayerParams`` (float64 or float32 arrays = the
  Scalar template argument); they upload to a temporary device layer of that
  precision and run on the GPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._capi import (DTYPES, InvalidArgument, PlanViewC, check, default_context, lib)
from .routing import RoutingConfig, RoutingPlan, ScoreMatrix, plan_set_stride

__all__ = [
    "LayerDims", "ExpertParams", "MoeLayerParams", "TokenBatch", "Divergence", "silu",
    "DeviceMoeLayer", "DecodeGraph", "router_scores", "expert_forward", "moe_forward",
    "output_divergence", "make_random_layer", "make_random_batch", "kDefaultToyTopK",
]

kDefaultToyTopK = 4


@dataclass
class LayerDims:
    """moe_layer.hpp:36-40"""
    embed: int = 64
    hidden: int = 96
    experts: int = 16


@dataclass
class ExpertParams:
    """moe_layer.hpp:29-34: w_gate D x H, w_up D x H, w_down H x D."""
    w_gate: np.ndarray
    w_up: np.ndarray
    w_down: np.ndarray


@dataclass
class MoeLayerParams:
    """moe_layer.hpp:44-54"""
    router: np.ndarray
    experts: list = field(default_factory=list)

    def embed_dim(self) -> int:
        return int(self.router.shape[0])

    def expert_count(self) -> int:
        return int(self.router.shape[1])

    def hidden_dim(self) -> int:
        return int(self.experts[0].w_gate.shape[1]) if self.experts else 0

    def scalar(self) -> str:
        return "f32" if self.router.dtype == np.float32 else "f64"


@dataclass
class TokenBatch:
    embeddings: np.ndarray  # B x D float64


@dataclass
class Divergence:
    mean_relative_error: float = 0.0
    max_relative_error: float = 0.0


def silu(z):
    return z / (1.0 + np.exp(-z))


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _ptr(t):
    """Device pointer of a torch tensor / int / None."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy: the legacy default stream


def torch_stream(stream=None) -> int:
    """A CUDA stream handle for the C ABI from a torch stream (default: the
    current one). torch's default stream has handle 0, which the C ABI reads
    as "the context's own stream", so it is passed as cudaStreamLegacy."""
    import torch
    h = (stream or torch.cuda.current_stream()).cuda_stream
    return h if h else CUDA_STREAM_LEGACY


class DecodeGraph:
    """A CUDA graph of one decode call (router -> FFN) with fixed buffers."""

    def __init__(self, layer, h):
        self.layer = layer
        self.h = h

    def launch(self, stream=None):
        self.layer.ctx.check(lib().oea_graph_launch(self.h, stream))

    def close(self):
        if self.h:
            lib().oea_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceMoeLayer:
    """A device-resident MoE layer (oea_layer_t)."""

    def __init__(self, D: int, H: int, N: int, dtype: str = "bf16", ctx=None, experts=None):
        """experts=(e_begin, e_end): an expert-parallel shard holding experts
        [e_begin, e_end) of the N its full router routes over (bf16); its decode
        returns this shard's partial sum (experts it does not hold contribute 0)."""
        self.ctx = ctx or default_context()
        self.D, self.H, self.N, self.dtype = int(D), int(H), int(N), dtype
        self.experts = (0, self.N) if experts is None else (int(experts[0]), int(experts[1]))
        self.h = C.c_void_p()
        self.ctx.check(lib().oea_layer_create_shard(
            self.ctx.h, self.D, self.H, self.N, DTYPES[dtype], self.experts[0], self.experts[1],
            C.byref(self.h)))

    def close(self):
        if getattr(self, "h", None):
            lib().oea_layer_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- weights -------------------------------------------------------
    @classmethod
    def from_params(cls, params: MoeLayerParams, dtype: str | None = None, ctx=None):
        dtype = dtype or params.scalar()
        L = cls(params.embed_dim(), params.hidden_dim(), params.expert_count(), dtype, ctx)
        L.upload_router(params.router)
        for e, ex in enumerate(params.experts):
            L.upload_expert(e, ex.w_gate, ex.w_up, ex.w_down)
        return L

    @staticmethod
    def _host(a):
        a = np.ascontiguousarray(a)
        if a.dtype == np.float64:
            return a, DTYPES["f64"]
        if a.dtype == np.float32:
            return a, DTYPES["f32"]
        return np.ascontiguousarray(a, dtype=np.float64), DTYPES["f64"]

    def upload_router(self, router):
        r, dt = self._host(router)
        if r.shape != (self.D, self.N):
            raise InvalidArgument("router must be D x N")
        self.ctx.check(lib().oea_layer_upload_router(self.h, _p(r), dt, 0))

    def upload_expert(self, e, w_gate, w_up, w_down):
        g, dt = self._host(w_gate)
        u, _ = self._host(np.asarray(w_up, dtype=g.dtype))
        d, _ = self._host(np.asarray(w_down, dtype=g.dtype))
        if g.shape != (self.D, self.H) or u.shape != (self.D, self.H) or d.shape != (self.H, self.D):
            raise InvalidArgument("expert_forward: dimension mismatch")
        self.ctx.check(lib().oea_layer_upload_expert(self.h, int(e), _p(g), _p(u), _p(d), dt, 0))

    def init_random(self, seed: int):
        """make_random_layer distributions (moe_layer.cpp:76-98), on device."""
        self.ctx.check(lib().oea_layer_init_random(self.h, C.c_uint64(seed)))

    def download_router(self, dtype="f64"):
        out = np.empty((self.D, self.N), np.float64 if dtype == "f64" else np.float32)
        self.ctx.check(lib().oea_layer_download_router(self.h, _p(out), DTYPES[dtype]))
        return out

    def download_expert(self, e, dtype="f64"):
        dt = np.float64 if dtype == "f64" else np.float32
        g = np.empty((self.D, self.H), dt)
        u = np.empty((self.D, self.H), dt)
        d = np.empty((self.H, self.D), dt)
        self.ctx.check(lib().oea_layer_download_expert(self.h, int(e), _p(g), _p(u), _p(d),
                                                       DTYPES[dtype]))
        return g, u, d

    def download_params(self, dtype="f64") -> MoeLayerParams:
        return MoeLayerParams(self.download_router(dtype),
                              [ExpertParams(*self.download_expert(e, dtype))
                               for e in range(*self.experts)])

    def info(self) -> dict:
        D, H, N, dt = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        bpe, dev = C.c_int64(), C.c_int64()
        self.ctx.check(lib().oea_layer_info(self.h, C.byref(D), C.byref(H), C.byref(N),
                                            C.byref(dt), C.byref(bpe), C.byref(dev)))
        return {"D": D.value, "H": H.value, "N": N.value, "dtype": dt.value,
                "bytes_per_expert": bpe.value, "device_bytes": dev.value}

    # ---- decode (the hot path) ------------------------------------------
    def decode(self, x, cfg: RoutingConfig, out, mask=None, stream=None):
        """Device decode: x (torch bf16 [B, D] for bf16 layers, f64 otherwise),
        out (torch f32 [B, D] for bf16 layers, f64 otherwise)."""
        B = int(x.shape[0])
        self.ctx.check(lib().oea_moe_decode(self.ctx.h, self.h, C.c_void_p(_ptr(x)),
                                            C.c_void_p(_ptr(mask)) if mask is not None else None,
                                            B, C.byref(cfg.to_c()), C.c_void_p(_ptr(out)),
                                            C.c_void_p(stream) if stream else None))

    def decode_host(self, x: np.ndarray, cfg: RoutingConfig, mask=None, out=None):
        """End to end from host buffers: x bf16 bits as uint16 (bf16 layers)
        or float64; returns out (float32 / float64)."""
        B = int(x.shape[0])
        bf = self.dtype == "bf16"
        x = np.ascontiguousarray(x, dtype=np.uint16 if bf else np.float64)
        if out is None:
            out = np.empty((B, self.D), np.float32 if bf else np.float64)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        self.ctx.check(lib().oea_moe_decode_host(self.ctx.h, self.h, _p(x), _p(m), B,
                                                 C.byref(cfg.to_c()), _p(out)))
        return out

    def decode_host_ptr(self, x_ptr: int, out_ptr: int, B: int, cfg: RoutingConfig, mask_ptr=None):
        """End-to-end decode from raw host pointers (e.g. pinned torch tensors):
        H2D of x, the fused decode, D2H of out, synchronise (oea_moe_decode_host)."""
        rc = lib().oea_moe_decode_host(self.ctx.h, self.h, x_ptr, mask_ptr or None, B,
                                       cfg.c_ref(), out_ptr)
        if rc:
            self.ctx.check(rc)

    def graph(self, x, cfg: RoutingConfig, out, mask=None) -> DecodeGraph:
        g = C.c_void_p()
        self.ctx.check(lib().oea_decode_graph_create(
            self.ctx.h, self.h, C.c_void_p(_ptr(x)),
            C.c_void_p(_ptr(mask)) if mask is not None else None, int(x.shape[0]),
            C.byref(cfg.to_c()), C.c_void_p(_ptr(out)), C.byref(g)))
        return DecodeGraph(self, g)

    @staticmethod
    def chain_graph(layers, xs, cfg: RoutingConfig, outs, mask=None) -> DecodeGraph:
        """ONE CUDA graph of len(layers) decode calls back to back (layers[i]:
        xs[i] -> outs[i]), the way a decode step's MoE layers run: the fused
        launches are programmatic dependents of their predecessor (PDL)."""
        n = len(layers)
        if n < 1 or len(xs) != n or len(outs) != n:
            raise InvalidArgument("chain_graph: need matching non-empty layers / xs / outs")
        ctx = layers[0].ctx
        hs = (C.c_void_p * n)(*[L.h.value for L in layers])
        xp = (C.c_void_p * n)(*[_ptr(x) for x in xs])
        op = (C.c_void_p * n)(*[_ptr(o) for o in outs])
        g = C.c_void_p()
        ctx.check(lib().oea_decode_chain_graph_create(
            ctx.h, n, hs, xp, C.c_void_p(_ptr(mask)) if mask is not None else None,
            int(xs[0].shape[0]), C.byref(cfg.to_c()), op, C.byref(g)))
        return DecodeGraph(layers[-1], g)

    def stage_graphs(self, x, cfg: RoutingConfig, out, mask=None):
        """(router graph, FFN graph) of one decode, for per-stage timing."""
        g1, g2 = C.c_void_p(), C.c_void_p()
        self.ctx.check(lib().oea_decode_stage_graphs_create(
            self.ctx.h, self.h, C.c_void_p(_ptr(x)),
            C.c_void_p(_ptr(mask)) if mask is not None else None, int(x.shape[0]),
            C.byref(cfg.to_c()), C.c_void_p(_ptr(out)), C.byref(g1), C.byref(g2)))
        return DecodeGraph(self, g1), DecodeGraph(self, g2)

    def last_plan(self, B: int, cfg: RoutingConfig) -> dict:
        """Routing of the most recent decode: sets/weights/aggregates and the
        router output (fp32 logits for bf16 layers, fp64 scores otherwise)."""
        N = self.N
        rcfg = cfg.resolved(N)
        stride = max(plan_set_stride(rcfg), 1)
        sets = np.full((B, stride), -1, np.int32)
        set_len = np.zeros(B, np.int32)
        w64 = np.zeros((B, stride), np.float64)
        w32 = np.zeros((B, stride), np.float32)
        loads = np.zeros(N, np.int32)
        au = np.full(N, -1, np.int32)
        cnt = np.zeros(1, np.int32)
        tot = np.zeros(1, np.int64)
        n1 = np.zeros(B, np.int32)
        bu = np.full(N, -1, np.int32)
        bcnt = np.zeros(1, np.int32)
        logits = np.zeros((B, N), np.float32)
        scores = np.zeros((B, N), np.float64)
        pv = PlanViewC(stride, _p(sets), _p(set_len), _p(w64), _p(w32), _p(loads), _p(au),
                       _p(cnt), _p(tot), None, None, _p(n1), _p(bu), _p(bcnt))
        self.ctx.check(lib().oea_last_plan_host(self.ctx.h, C.byref(pv), _p(logits), _p(scores)))
        return {"sets": sets, "set_len": set_len, "weights": w64, "weights_f32": w32,
                "loads": loads, "active_union": au[: cnt[0]].copy(), "active_count": int(cnt[0]),
                "total_load": int(tot[0]), "phase1_n": n1, "base_union": bu[: bcnt[0]].copy(),
                "logits": logits, "scores": scores}

    def forward_plan(self, x: np.ndarray, sets, set_len, weights, mask=None) -> np.ndarray:
        """moe_forward on a flat plan (host buffers), output fp64."""
        x = np.ascontiguousarray(x, np.float64)
        sets = np.ascontiguousarray(sets, np.int32)
        set_len = np.ascontiguousarray(set_len, np.int32)
        weights = np.ascontiguousarray(weights, np.float64)
        B = x.shape[0]
        out = np.empty((B, self.D), np.float64)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        self.ctx.check(lib().oea_moe_forward_plan_host(
            self.ctx.h, self.h, _p(x), B, _p(sets), _p(set_len), _p(weights), sets.shape[1],
            _p(m), _p(out)))
        return out

    def router_scores(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty((x.shape[0], self.N), np.float64)
        self.ctx.check(lib().oea_router_scores_host(self.ctx.h, self.h, _p(x), x.shape[0], _p(out)))
        return out


# ---------------------------------------------------------------------------
# Reference free functions over host MoeLayerParams.
# ---------------------------------------------------------------------------
def router_scores(layer: MoeLayerParams, batch: TokenBatch) -> ScoreMatrix:
    """moe_layer.hpp:71-90 (fp64 GEMV + softmax on the GPU)."""
    x = np.asarray(batch.embeddings, np.float64)
    if x.shape[1] != layer.embed_dim():
        raise InvalidArgument(f"router_scores: embedding dim {x.shape[1]} does not match "
                              f"router rows {layer.embed_dim()}")
    dims = (layer.embed_dim(), max(layer.hidden_dim(), 1), layer.expert_count())
    dev = DeviceMoeLayer(*dims, dtype=layer.scalar())
    dev.upload_router(layer.router)
    return ScoreMatrix(dev.router_scores(x))


def _flat_plan(plan: RoutingPlan):
    B = len(plan.sets)
    stride = max([len(s) for s in plan.sets] + [1])
    sets = np.full((B, stride), -1, np.int32)
    set_len = np.zeros(B, np.int32)
    w = np.zeros((B, stride), np.float64)
    for i, (s, ww) in enumerate(zip(plan.sets, plan.weights)):
        set_len[i] = len(s)
        sets[i, : len(s)] = s
        w[i, : len(ww)] = ww
    return sets, set_len, w


def moe_forward(layer: MoeLayerParams, batch: TokenBatch, plan: RoutingPlan, mask=None):
    """moe_layer.hpp:114-158 on the GPU (SIMT FFN in the layer's precision,
    fp64 mixture in set order). Same validation and messages."""
    x = np.asarray(batch.embeddings, np.float64)
    B = x.shape[0]
    if plan.n_experts != layer.expert_count():
        raise InvalidArgument("moe_forward: plan expert count mismatch")
    if len(plan.sets) != B or len(plan.weights) != len(plan.sets):
        raise InvalidArgument("moe_forward: plan batch size mismatch")
    if mask is not None and len(mask) != B:
        raise InvalidArgument("moe_forward: mask size mismatch")
    for i, (s, w) in enumerate(zip(plan.sets, plan.weights)):
        real = mask is None or bool(mask[i])
        if len(s) == 0:
            if real and mask is not None:
                raise InvalidArgument(f"moe_forward: empty selected set for unmasked token {i}")
            continue
        if len(w) != len(s):
            raise InvalidArgument(f"moe_forward: weights/set size mismatch for token {i}")
        for e in s:
            if e < 0 or e >= layer.expert_count():
                raise InvalidArgument("moe_forward: expert index out of range")
    sets, set_len, w = _flat_plan(plan)
    dev = DeviceMoeLayer.from_params(layer)
    return dev.forward_plan(x, sets, set_len, w, mask)


def expert_forward(expert: ExpertParams, x) -> np.ndarray:
    """moe_layer.hpp:92-107 — one expert on one token, on the GPU (a
    one-expert layer with weight 1.0; the mixture adds exactly y)."""
    x = np.asarray(x, np.float64).reshape(1, -1)
    D, H = expert.w_gate.shape
    if (x.shape[1] != D or expert.w_up.shape[0] != D or expert.w_down.shape[0] != H or
            expert.w_down.shape[1] != D):
        raise InvalidArgument("expert_forward: dimension mismatch")
    scalar = "f32" if np.asarray(expert.w_gate).dtype == np.float32 else "f64"
    dev = DeviceMoeLayer(D, H, 1, dtype=scalar)
    dev.upload_expert(0, expert.w_gate, expert.w_up, expert.w_down)
    return dev.forward_plan(x, np.zeros((1, 1), np.int32), np.ones(1, np.int32),
                            np.ones((1, 1), np.float64))[0]


def output_divergence(ref, test) -> Divergence:
    """moe_layer.cpp:57-74 (metric on outputs)."""
    ref = np.asarray(ref, np.float64)
    test = np.asarray(test, np.float64)
    if ref.shape != test.shape:
        raise InvalidArgument("output_divergence: shape mismatch")
    if ref.shape[0] == 0:
        raise InvalidArgument("output_divergence: empty input")
    denom = np.maximum(np.sqrt((ref * ref).sum(axis=1)), 1e-12)
    rel = np.sqrt(((ref - test) ** 2).sum(axis=1)) / denom
    return Divergence(float(rel.mean()), float(rel.max()))


def make_random_layer(dims: LayerDims, seed: int) -> MoeLayerParams:
    """make_random_layer (moe_layer.cpp:76-98), generated on the device in
    fp64 (the same counter stream and Box-Muller map; CUDA's libm may differ
    from glibc in the last ulp)."""
    if dims.embed < 1 or dims.hidden < 1 or dims.experts < 1:
        raise InvalidArgument("make_random_layer: dims must be positive")
    dev = DeviceMoeLayer(dims.embed, dims.hidden, dims.experts, dtype="f64")
    dev.init_random(seed)
    return dev.download_params("f64")


_GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def _splitmix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z ^ (z >> np.uint64(30))
        z = z * np.uint64(0xBF58476D1CE4E5B9)
        z = z ^ (z >> np.uint64(27))
        z = z * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def _stream_key(parts):
    h = np.uint64(0x853C49E6748FEA9B)
    with np.errstate(over="ignore"):
        for p in parts:
            h = _splitmix64(h + _GOLDEN + np.uint64(p))
    return h


def make_random_batch(batch: int, embed_dim: int, seed: int, step: int = 0,
                      layer: int = 0) -> TokenBatch:
    """make_random_batch (moe_layer.cpp:100-116): per-token counter streams
    keyed (seed, step, layer, token, 102), Box-Muller normals (host input
    generator)."""
    if batch < 1 or embed_dim < 1:
        raise InvalidArgument("make_random_batch: dims must be positive")
    out = np.empty((batch, embed_dim), np.float64)
    f = np.arange(embed_dim, dtype=np.uint64)
    pair = f // np.uint64(2)
    for i in range(batch):
        key = _stream_key([seed, step, layer, i, 102])
        with np.errstate(over="ignore"):
            u1 = _splitmix64(key + (np.uint64(2) * pair + np.uint64(1)) * _GOLDEN)
            u2 = _splitmix64(key + (np.uint64(2) * pair + np.uint64(2)) * _GOLDEN)
        u1 = ((u1 >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
        u2 = ((u2 >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
        r = np.sqrt(-2.0 * np.log(u1))
        th = 2.0 * np.pi * u2
        out[i] = np.where(f % np.uint64(2) == 1, r * np.sin(th), r * np.cos(th))
    return TokenBatch(out)
