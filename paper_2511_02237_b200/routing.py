"""Python mirror of the reference routing API (proj/include/oea/routing.hpp).

Same names, argument meaning and error behaviour as the C++ functions:
``std::invalid_argument`` -> :class:`InvalidArgument` (a ``ValueError``),
``std::domain_error`` -> :class:`DomainError` (an ``ArithmeticError``), with
the reference's messages. Every routing computation runs on the GPU through
the C ABI (``oea_route_f64_host`` and friends, kernel family K1); the host
side only marshals arrays. ``ScoreMatrix.validate`` and ``batch_stats`` are
host input checks / recounts of a host-resident plan, as in the reference.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import List

import numpy as np

from ._capi import (DomainError, InvalidArgument, PlanViewC, RoutingCfgC, default_context, lib)

__all__ = [
    "RoutingMode", "CapSemantics", "RoutingConfig", "ScoreMatrix", "SortedExperts",
    "Phase1Result", "RoutingPlan", "BatchStats", "to_string", "routing_mode_from_string",
    "cap_semantics_from_string", "sort_experts", "route_topk", "phase1_baseline",
    "phase2_piggyback", "route", "route_batched", "BatchedScores", "batch_stats", "plan_set_stride",
]


class RoutingMode(IntEnum):
    """routing.hpp:45"""
    Vanilla = 0
    Pruned = 1
    Oea = 2
    SimplifiedOea = 3


class CapSemantics(IntEnum):
    """routing.hpp:49"""
    ExactCap = 0
    PseudocodeStrict = 1


_MODE_NAMES = {RoutingMode.Vanilla: "vanilla", RoutingMode.Pruned: "pruned",
               RoutingMode.Oea: "oea", RoutingMode.SimplifiedOea: "simplified"}
_CAP_NAMES = {CapSemantics.ExactCap: "exact", CapSemantics.PseudocodeStrict: "pseudocode"}


def to_string(v) -> str:
    """routing.cpp:81-93"""
    if isinstance(v, RoutingMode):
        return _MODE_NAMES[v]
    if isinstance(v, CapSemantics):
        return _CAP_NAMES[v]
    return "?"


def routing_mode_from_string(s: str) -> RoutingMode:
    for k, v in _MODE_NAMES.items():
        if v == s:
            return k
    raise InvalidArgument("unknown routing mode: " + s)


def cap_semantics_from_string(s: str) -> CapSemantics:
    for k, v in _CAP_NAMES.items():
        if v == s:
            return k
    raise InvalidArgument("unknown cap semantics: " + s)


_C_CFG_CACHE: dict = {}


@dataclass
class RoutingConfig:
    """routing.hpp:56-76 (field for field, same defaults)."""
    mode: RoutingMode = RoutingMode.Vanilla
    k: int = 8
    k0: int = 8
    p: float = 1.0
    k_max: int = 8
    max_p: int = 0
    cap: CapSemantics = CapSemantics.ExactCap

    @staticmethod
    def vanilla(k: int) -> "RoutingConfig":
        return RoutingConfig(RoutingMode.Vanilla, k, k, 1.0, k, 0, CapSemantics.ExactCap)

    @staticmethod
    def pruned(k0: int, p: float, k: int) -> "RoutingConfig":
        return RoutingConfig(RoutingMode.Pruned, k, k0, p, max(k0, k), 0, CapSemantics.ExactCap)

    @staticmethod
    def oea(k0: int, p: float, k_max: int, max_p: int, k: int,
            cap: CapSemantics = CapSemantics.ExactCap) -> "RoutingConfig":
        return RoutingConfig(RoutingMode.Oea, k, k0, p, k_max, max_p, cap)

    @staticmethod
    def simplified(k0: int, k: int, cap: CapSemantics = CapSemantics.ExactCap) -> "RoutingConfig":
        return RoutingConfig(RoutingMode.SimplifiedOea, k, k0, 1.0, k, 0, cap)

    def to_c(self) -> RoutingCfgC:
        return RoutingCfgC(int(self.mode), int(self.k), int(self.k0), float(self.p),
                           int(self.k_max), int(self.max_p), int(self.cap))

    def c_ref(self):
        """A byref() of this config's C struct, cached by value (hot host
        paths call the C ABI once per decode)."""
        key = (int(self.mode), int(self.k), int(self.k0), float(self.p), int(self.k_max),
               int(self.max_p), int(self.cap))
        hit = _C_CFG_CACHE.get(key)
        if hit is None:
            c = RoutingCfgC(*key)
            hit = _C_CFG_CACHE[key] = (c, C.byref(c))
        return hit[1]

    @staticmethod
    def from_c(c: RoutingCfgC) -> "RoutingConfig":
        return RoutingConfig(RoutingMode(c.mode), c.k, c.k0, c.p, c.k_max, c.max_p,
                             CapSemantics(c.cap))

    def resolved(self, n_experts: int) -> "RoutingConfig":
        """routing.cpp:153-182 (oea_config_resolve)."""
        out = RoutingCfgC()
        rc = lib().oea_config_resolve(C.byref(self.to_c()), int(n_experts), C.byref(out))
        if rc:
            raise InvalidArgument(lib().oea_last_error(None).decode())
        return RoutingConfig.from_c(out)


def plan_set_stride(resolved: RoutingConfig) -> int:
    return int(lib().oea_plan_set_stride(C.byref(resolved.to_c())))


@dataclass
class ScoreMatrix:
    """routing.hpp:28-43: B x N router probabilities + optional mask."""
    scores: np.ndarray
    mask: np.ndarray | None = None

    def __post_init__(self):
        self.scores = np.ascontiguousarray(np.asarray(self.scores, dtype=np.float64))
        if self.scores.ndim == 1:
            self.scores = self.scores.reshape(1, -1)
        if self.mask is not None:
            self.mask = np.ascontiguousarray(np.asarray(self.mask, dtype=bool))
            if self.mask.size == 0:
                self.mask = None

    def batch(self) -> int:
        return int(self.scores.shape[0])

    def experts(self) -> int:
        return int(self.scores.shape[1]) if self.scores.ndim == 2 else 0

    def is_real(self, i: int) -> bool:
        return self.mask is None or bool(self.mask[i])

    def real_count(self) -> int:
        return self.batch() if self.mask is None else int(self.mask.sum())

    def validate(self) -> None:
        """routing.cpp:53-79 (host input check, same messages)."""
        if self.scores.size == 0 or self.batch() < 1 or self.experts() < 1:
            raise InvalidArgument("ScoreMatrix: dimensions must be >= 1")
        if self.mask is not None and self.mask.size != self.batch():
            raise InvalidArgument(f"ScoreMatrix: mask length {self.mask.size} does not match "
                                  f"batch size {self.batch()}")
        for i in range(self.batch()):
            row = self.scores[i]
            if not np.all(np.isfinite(row)) or np.any(row < 0.0):
                raise InvalidArgument(f"ScoreMatrix: row {i} has a negative or non-finite score")
            s = 0.0
            for v in row:  # sequential sum, as the reference
                s += float(v)
            if self.is_real(i) and abs(s - 1.0) > 1e-6:
                raise InvalidArgument(f"ScoreMatrix: row {i} is off the simplex (sum = {s:.6f})")

    def _mask_u8(self):
        return None if self.mask is None else np.ascontiguousarray(self.mask, dtype=np.uint8)


@dataclass
class SortedExperts:
    order: np.ndarray  # B x N int32


@dataclass
class Phase1Result:
    t: np.ndarray
    n: np.ndarray
    base_sets: list
    base_union: list


@dataclass
class RoutingPlan:
    """routing.hpp:95-103"""
    sets: list = field(default_factory=list)
    weights: list = field(default_factory=list)
    active_union: list = field(default_factory=list)
    active_count: int = 0
    loads: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    total_load: int = 0
    n_experts: int = 0

    def __eq__(self, o):
        return (isinstance(o, RoutingPlan) and self.sets == o.sets and
                self.weights == o.weights and self.active_union == o.active_union and
                self.active_count == o.active_count and self.total_load == o.total_load and
                self.n_experts == o.n_experts and np.array_equal(self.loads, o.loads))


@dataclass
class BatchStats:
    active_count: int = 0
    loads: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    total_load: int = 0


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _as_scores(scores) -> ScoreMatrix:
    return scores if isinstance(scores, ScoreMatrix) else ScoreMatrix(np.asarray(scores))


def _plan_from_arrays(B, N, sets, set_len, weights, loads, au, cnt, tot) -> RoutingPlan:
    plan = RoutingPlan(n_experts=N)
    lens = set_len[:B].tolist()
    srows = sets[:B].tolist()  # (ndarray.tolist: Python ints / floats in one call)
    plan.sets = [r[:n] for r, n in zip(srows, lens)]
    if weights is not None:
        wrows = weights[:B].tolist()
        plan.weights = [r[:n] for r, n in zip(wrows, lens)]
    else:
        plan.weights = [[] for _ in range(B)]
    plan.active_count = int(cnt)
    plan.active_union = au[: int(cnt)].tolist()
    plan.loads = loads.copy()
    plan.total_load = int(tot)
    return plan


def sort_experts(scores) -> SortedExperts:
    """routing.cpp:184-203 on the GPU (warp bitonic rank sort)."""
    sm = _as_scores(scores)
    B, N = sm.scores.shape if sm.scores.ndim == 2 else (0, 0)
    ctx = default_context()
    order = np.empty((max(B, 1), max(N, 1)), np.int32)
    ctx.check(lib().oea_sort_experts_f64_host(ctx.h, _p(sm.scores), B, N, _p(order)))
    return SortedExperts(order)


def _route_call(sm: ScoreMatrix, cfg: RoutingConfig, want_order=False):
    B, N = sm.scores.shape if sm.scores.ndim == 2 else (0, 0)
    ctx = default_context()
    rcfg = cfg.resolved(N)  # raises the reference's invalid_argument first
    stride = max(plan_set_stride(rcfg), 1)
    Bc, Nc = max(B, 1), max(N, 1)
    sets = np.full((Bc, stride), -1, np.int32)
    set_len = np.zeros(Bc, np.int32)
    weights = np.zeros((Bc, stride), np.float64)
    loads = np.zeros(Nc, np.int32)
    au = np.full(Nc, -1, np.int32)
    cnt = np.zeros(1, np.int32)
    tot = np.zeros(1, np.int64)
    order = np.zeros((Bc, Nc), np.int32) if want_order else None
    pv = PlanViewC(stride, _p(sets), _p(set_len), _p(weights), None, _p(loads), _p(au), _p(cnt),
                   _p(tot), _p(order), None, None, None, None)
    ctx.check(lib().oea_route_f64_host(ctx.h, _p(sm.scores), _p(sm._mask_u8()), B, N,
                                       C.byref(cfg.to_c()), C.byref(pv)))
    return _plan_from_arrays(B, N, sets, set_len, weights, loads, au, cnt[0], tot[0])


def route_batched(records, cfg: RoutingConfig) -> List[RoutingPlan]:
    """route() of every record (score matrices with one expert count) in one
    GPU launch sequence (oea_route_f64_batched_host): the per-record loop of
    the reference's `route` command (oea_cli.cpp:153-175). Returns one plan
    per record, each equal to route(record, cfg)."""
    sms = [_as_scores(r) for r in records]
    if not sms:
        return []
    N = sms[0].experts()
    if N < 1:
        raise InvalidArgument("RoutingConfig: expert count must be >= 1")
    for sm in sms:
        if sm.experts() != N:
            raise InvalidArgument("route_batched: inconsistent expert count")
    rcfg = cfg.resolved(N)
    stride = max(plan_set_stride(rcfg), 1)
    rows = np.array([sm.batch() for sm in sms], np.int32)
    R, B = len(sms), int(rows.sum())
    scores = np.ascontiguousarray(np.concatenate([sm.scores for sm in sms], axis=0), np.float64)
    any_mask = any(sm.mask is not None and len(sm.mask) > 0 for sm in sms)
    mask = (np.concatenate([sm._mask_u8() if sm._mask_u8() is not None else np.ones(sm.batch(), np.uint8)
                            for sm in sms]) if any_mask else None)
    sets = np.full((max(B, 1), stride), -1, np.int32)
    set_len = np.zeros(max(B, 1), np.int32)
    weights = np.zeros((max(B, 1), stride), np.float64)
    loads = np.zeros((R, N), np.int32)
    au = np.full((R, N), -1, np.int32)
    cnt = np.zeros(R, np.int32)
    tot = np.zeros(R, np.int64)
    pv = PlanViewC(stride, _p(sets), _p(set_len), _p(weights), None, _p(loads), _p(au), _p(cnt),
                   _p(tot), None, None, None, None, None)
    ctx = default_context()
    ctx.check(lib().oea_route_f64_batched_host(ctx.h, _p(scores), _p(mask), _p(rows), R, N,
                                               C.byref(cfg.to_c()), C.byref(pv)))
    plans, r0 = [], 0
    for q in range(R):
        b = int(rows[q])
        plans.append(_plan_from_arrays(b, N, sets[r0:r0 + b], set_len[r0:r0 + b],
                                       weights[r0:r0 + b], loads[q], au[q], cnt[q], tot[q]))
        r0 += b
    return plans


class BatchedScores:
    """Records concatenated once for repeated batched routing (a config
    sweep): route_counts(cfg) returns only each record's T and total load."""

    def __init__(self, records):
        sms = [_as_scores(r) for r in records]
        if not sms:
            raise InvalidArgument("route_batched: need R >= 1 records")
        self.N = sms[0].experts()
        if any(sm.experts() != self.N for sm in sms):
            raise InvalidArgument("route_batched: inconsistent expert count")
        self.rows = np.array([sm.batch() for sm in sms], np.int32)
        self.scores = np.ascontiguousarray(np.concatenate([sm.scores for sm in sms], axis=0))
        masked = any(sm.mask is not None for sm in sms)
        self.mask = (np.concatenate([sm._mask_u8() if sm.mask is not None
                                     else np.ones(sm.batch(), np.uint8) for sm in sms])
                     if masked else None)

    def route_counts(self, cfg: RoutingConfig):
        R = len(self.rows)
        cnt = np.zeros(R, np.int32)
        tot = np.zeros(R, np.int64)
        cfg.resolved(self.N)
        pv = PlanViewC(0, None, None, None, None, None, None, _p(cnt), _p(tot), None, None, None,
                       None, None)
        ctx = default_context()
        ctx.check(lib().oea_route_f64_batched_host(ctx.h, _p(self.scores), _p(self.mask),
                                                   _p(self.rows), R, self.N,
                                                   C.byref(cfg.to_c()), C.byref(pv)))
        return cnt, tot


def route_topk(scores, k: int) -> RoutingPlan:
    """routing.cpp:205-224"""
    sm = _as_scores(scores)
    n = sm.experts()
    if k < 1 or k > n:
        raise InvalidArgument("route_topk: k must be in [1, N]")
    return _route_call(sm, RoutingConfig.vanilla(k))


def route(scores, cfg: RoutingConfig) -> RoutingPlan:
    """routing.cpp:305-326: resolve, rank, Phase 1, Phase 2, renormalise —
    all on the GPU (oea_route_f64_host)."""
    sm = _as_scores(scores)
    if sm.experts() < 1:
        raise InvalidArgument("RoutingConfig: expert count must be >= 1")
    return _route_call(sm, cfg)


def phase1_baseline(scores, sorted_experts: SortedExperts, cfg: RoutingConfig) -> Phase1Result:
    """routing.cpp:226-268 from a caller-supplied order."""
    sm = _as_scores(scores)
    B, N = sm.scores.shape
    rcfg = cfg.resolved(N)
    ctx = default_context()
    order = np.ascontiguousarray(sorted_experts.order, np.int32)
    k0 = max(rcfg.k0, 1)
    t = np.zeros(B, np.int32)
    n = np.zeros(B, np.int32)
    base_sets = np.full((B, k0), -1, np.int32)
    bu = np.full(N, -1, np.int32)
    bcnt = np.zeros(1, np.int32)
    ctx.check(lib().oea_phase1_f64_host(ctx.h, _p(sm.scores), _p(sm._mask_u8()), B, N, _p(order),
                                        C.byref(cfg.to_c()), _p(t), _p(n), _p(base_sets), k0,
                                        _p(bu), _p(bcnt)))
    return Phase1Result(t, n, [[int(v) for v in base_sets[i, : n[i]]] for i in range(B)],
                        [int(v) for v in bu[: bcnt[0]]])


def phase2_piggyback(scores, sorted_experts: SortedExperts, phase1: Phase1Result,
                     cfg: RoutingConfig) -> RoutingPlan:
    """routing.cpp:270-303 from caller-supplied order / baseline sizes / union.
    Weights are left empty, as in the reference."""
    sm = _as_scores(scores)
    B, N = sm.scores.shape
    rcfg = cfg.resolved(N)
    ctx = default_context()
    order = np.ascontiguousarray(sorted_experts.order, np.int32)
    n = np.ascontiguousarray(phase1.n, np.int32)
    bu = np.ascontiguousarray(np.asarray(phase1.base_union, dtype=np.int32))
    limit = rcfg.k_max + (1 if rcfg.cap == CapSemantics.PseudocodeStrict else 0)
    stride = max(limit, int(n.max()) if n.size else 0, 1)
    sets = np.full((B, stride), -1, np.int32)
    set_len = np.zeros(B, np.int32)
    loads = np.zeros(N, np.int32)
    au = np.full(N, -1, np.int32)
    cnt = np.zeros(1, np.int32)
    tot = np.zeros(1, np.int64)
    pv = PlanViewC(stride, _p(sets), _p(set_len), None, None, _p(loads), _p(au), _p(cnt), _p(tot),
                   None, None, None, None, None)
    ctx.check(lib().oea_phase2_f64_host(ctx.h, _p(sm._mask_u8()), B, N, _p(order), _p(n),
                                        _p(bu) if bu.size else None, int(bu.size),
                                        C.byref(cfg.to_c()), C.byref(pv)))
    return _plan_from_arrays(B, N, sets, set_len, None, loads, au, cnt[0], tot[0])


def batch_stats(plan: RoutingPlan) -> BatchStats:
    """routing.cpp:328-338: recount of a host-resident plan."""
    loads = np.zeros(plan.n_experts, np.int32)
    total = 0
    for s in plan.sets:
        for e in s:
            loads[e] += 1
        total += len(s)
    return BatchStats(int((loads > 0).sum()), loads, total)
