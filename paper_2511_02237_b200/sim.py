"""GPU-backed decode simulator.

Mirror of the reference's simulate_decode / padding_experiment and their
writers (simulate.cpp:56-345, latency.cpp:10-28): every (step, layer) cell is
scored and routed, and each record carries T, the total load and the modeled
latency sum_e expert_latency(load_e) = a * load + b over active experts.

B200 shape of the loop: the reference routes cell by cell on a thread pool
(parallel_cells, simulate.cpp:22-54); here the scores of ALL cells come from
one generator launch (scoregen.gen_run) and all cells are routed by one
batched route per policy (routing.route_batched): a simulation of S steps x L
layers is 3-4 GPU launch sequences instead of 2 S L CPU routes. Records are
identical to the reference's (integer T / load; the latency is the same fp64
formula over the same loads).
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

from ._capi import InvalidArgument
from .routing import RoutingConfig, RoutingPlan, ScoreMatrix, route_batched
from .scoregen import GenKind, ScoreGenConfig, gen_run, to_string as gen_to_string
from .traces import read_score_trace, routing_config_json

__all__ = ["LatencyParams", "StepRecord", "TraceAggregates", "DecodeTrace", "expert_latency",
           "moe_latency", "simulate_decode", "PaddingVariant", "PaddingReport",
           "padding_experiment", "write_trace_csv", "write_trace_summary_json",
           "write_padding_json", "gen_config_json", "cell_scores", "RoundingRule", "SweepPoint",
           "default_sweep_grid", "sweep", "pareto_indices", "pareto_frontier", "write_sweep_csv",
           "read_sweep_csv", "simulate_decode_layer"]


@dataclass
class LatencyParams:
    """latency.hpp:19-22"""
    a_us: float = 0.0
    b_us: float = 0.0


@dataclass
class StepRecord:
    """simulate.hpp:23-30"""
    layer: int = 0
    step: int = 0
    active_experts: int = 0
    total_load: int = 0
    modeled_latency_us: float = 0.0
    divergence: Optional[float] = None


@dataclass
class TraceAggregates:
    """simulate.hpp:32-43"""
    mean_active_experts: float = 0.0
    mean_total_load: float = 0.0
    mean_latency_us: float = 0.0
    vanilla_mean_active_experts: float = 0.0
    vanilla_mean_total_load: float = 0.0
    vanilla_mean_latency_us: float = 0.0
    normalized_active_experts: float = 0.0
    normalized_latency: float = 0.0
    mean_divergence: Optional[float] = None


@dataclass
class DecodeTrace:
    """simulate.hpp:45-50"""
    routing: RoutingConfig
    records: List[StepRecord] = field(default_factory=list)
    vanilla_records: List[StepRecord] = field(default_factory=list)
    aggregates: TraceAggregates = field(default_factory=TraceAggregates)


def expert_latency(tokens: int, p: LatencyParams) -> float:
    """latency.cpp:10-16"""
    if tokens < 0:
        raise InvalidArgument("expert_latency: token count must be >= 0")
    return 0.0 if tokens == 0 else p.a_us * float(tokens) + p.b_us


def moe_latency(loads, p: LatencyParams) -> float:
    """latency.cpp:18-24: sequential sum over experts."""
    total = 0.0
    for v in np.asarray(loads).tolist():
        total += expert_latency(int(v), p)
    return total


def _record(step: int, layer: int, plan: RoutingPlan, lat: LatencyParams) -> StepRecord:
    """make_record, simulate.cpp:56-65"""
    return StepRecord(layer=layer, step=step, active_experts=int(plan.active_count),
                      total_load=int(plan.total_load),
                      modeled_latency_us=moe_latency(plan.loads, lat))


def _ratio_or_nan(num: float, den: float) -> float:
    return num / den if den != 0.0 else float("nan")


def _aggregates(records: List[StepRecord], vanilla: List[StepRecord]) -> TraceAggregates:
    """compute_aggregates, simulate.cpp:72-103 (sequential sums)."""
    a = TraceAggregates()
    n = float(len(records))
    div_sum, div_count = 0.0, 0
    for r in records:
        a.mean_active_experts += r.active_experts
        a.mean_total_load += float(r.total_load)
        a.mean_latency_us += r.modeled_latency_us
        if r.divergence is not None:
            div_sum += r.divergence
            div_count += 1
    for r in vanilla:
        a.vanilla_mean_active_experts += r.active_experts
        a.vanilla_mean_total_load += float(r.total_load)
        a.vanilla_mean_latency_us += r.modeled_latency_us
    a.mean_active_experts /= n
    a.mean_total_load /= n
    a.mean_latency_us /= n
    a.vanilla_mean_active_experts /= n
    a.vanilla_mean_total_load /= n
    a.vanilla_mean_latency_us /= n
    a.normalized_active_experts = _ratio_or_nan(a.mean_active_experts, a.vanilla_mean_active_experts)
    a.normalized_latency = _ratio_or_nan(a.mean_latency_us, a.vanilla_mean_latency_us)
    if div_count > 0:
        a.mean_divergence = div_sum / div_count
    return a


def cell_scores(gen: ScoreGenConfig) -> Tuple[ScoreGenConfig, List[ScoreMatrix]]:
    """ScoreSource (score_gen.cpp:78-117) for every (step, layer) cell in
    (step, layer) order: one device launch for the generators; Replay reads
    the trace (n_experts and batch adopted from its first record, duplicate
    and missing cells rejected with the reference's messages)."""
    if gen.steps < 1 or gen.layers < 1:
        raise InvalidArgument("score gen: steps and layers must be >= 1")
    if gen.kind == GenKind.Replay:
        if not gen.trace_path:
            raise InvalidArgument("score gen: replay requires a trace path")
        recs = read_score_trace(gen.trace_path)
        cfg = ScoreGenConfig(**{**gen.__dict__})
        cfg.n_experts = recs[0].scores.experts()
        cfg.batch = recs[0].scores.batch()
        by: Dict[Tuple[int, int], ScoreMatrix] = {}
        for r in recs:
            if (r.step, r.layer) in by:
                raise InvalidArgument(f"score gen: duplicate record for step {r.step} layer "
                                      f"{r.layer} in {gen.trace_path}")
            by[(r.step, r.layer)] = r.scores
        out = []
        for s in range(cfg.steps):
            for l in range(cfg.layers):
                if (s, l) not in by:
                    raise InvalidArgument(f"score source: trace has no record for step {s} "
                                          f"layer {l}")
                out.append(by[(s, l)])
        return cfg, out
    run = gen_run(gen)
    return gen, [ScoreMatrix(run[s, l]) for s in range(gen.steps) for l in range(gen.layers)]


def simulate_decode(gen: ScoreGenConfig, routing: RoutingConfig,
                    latency: LatencyParams) -> DecodeTrace:
    """simulate.cpp:128-151: routed and vanilla-shadow records per cell."""
    cfg, cells = cell_scores(gen)
    rcfg = routing.resolved(cfg.n_experts)
    vcfg = RoutingConfig.vanilla(routing.k).resolved(cfg.n_experts)
    plans = route_batched(cells, rcfg)
    vplans = route_batched(cells, vcfg)
    tr = DecodeTrace(routing=rcfg)
    for idx, (p, vp) in enumerate(zip(plans, vplans)):
        step, layer = idx // cfg.layers, idx % cfg.layers
        tr.records.append(_record(step, layer, p, latency))
        tr.vanilla_records.append(_record(step, layer, vp, latency))
    tr.aggregates = _aggregates(tr.records, tr.vanilla_records)
    return tr


@dataclass
class PaddingVariant:
    """simulate.hpp:68-74"""
    name: str
    records: List[StepRecord] = field(default_factory=list)
    mean_active_experts: float = 0.0
    mean_total_load: float = 0.0
    mean_latency_us: float = 0.0


@dataclass
class PaddingReport:
    """simulate.hpp:76-83"""
    real_batch: int = 0
    padded_batch: int = 0
    no_padding: PaddingVariant = field(default_factory=lambda: PaddingVariant("no_padding"))
    naive_padding: PaddingVariant = field(default_factory=lambda: PaddingVariant("naive_padding"))
    masked_padding: PaddingVariant = field(default_factory=lambda: PaddingVariant("masked_padding"))
    masked_matches_no_padding: bool = False


def _fill_means(v: PaddingVariant) -> None:
    """fill_variant_means, simulate.cpp:114-121"""
    n = len(v.records)
    def mean(get):
        s = 0.0
        for r in v.records:
            s += get(r)
        return s / n if n else 0.0
    v.mean_active_experts = mean(lambda r: float(r.active_experts))
    v.mean_total_load = mean(lambda r: float(r.total_load))
    v.mean_latency_us = mean(lambda r: r.modeled_latency_us)


def padding_experiment(gen: ScoreGenConfig, routing: RoutingConfig, pad_to: int,
                       latency: LatencyParams) -> PaddingReport:
    """simulate.cpp:185-257: the same token stream unpadded, padded (pad rows
    routed) and padded with the pad rows masked; token scores are keyed by
    token index, so the padded run's first `batch` rows ARE the real rows
    and the real batch is a slice of one generator launch."""
    if gen.kind == GenKind.Replay:
        raise InvalidArgument("padding_experiment: replay sources are not supported")
    gen.to_c()
    if pad_to < gen.batch:
        raise InvalidArgument(f"padding_experiment: pad_to {pad_to} is smaller than the real "
                              f"batch {gen.batch}")
    padded = ScoreGenConfig(**{**gen.__dict__})
    padded.batch = pad_to
    run = gen_run(padded)
    rcfg = routing.resolved(gen.n_experts)
    cells = [(s, l) for s in range(gen.steps) for l in range(gen.layers)]
    mask = np.arange(pad_to) < gen.batch
    real = [ScoreMatrix(run[s, l, : gen.batch]) for s, l in cells]
    pad = [ScoreMatrix(run[s, l]) for s, l in cells]
    masked = [ScoreMatrix(run[s, l], mask) for s, l in cells]
    rep = PaddingReport(real_batch=gen.batch, padded_batch=pad_to)
    for variant, mats in ((rep.no_padding, real), (rep.naive_padding, pad),
                          (rep.masked_padding, masked)):
        for (s, l), p in zip(cells, route_batched(mats, rcfg)):
            variant.records.append(_record(s, l, p, latency))
        _fill_means(variant)
    rep.masked_matches_no_padding = all(
        a.active_experts == b.active_experts and a.total_load == b.total_load
        and a.modeled_latency_us == b.modeled_latency_us
        for a, b in zip(rep.no_padding.records, rep.masked_padding.records))
    return rep


def _fmt(v: float) -> str:
    return "%.17g" % v  # format_double, io.cpp:34-38


def write_trace_csv(path: str, trace: DecodeTrace) -> None:
    """simulate.cpp:263-285"""
    has_div = any(r.divergence is not None for r in trace.records)
    try:
        out = open(path, "w")
    except OSError:
        raise InvalidArgument("write_trace_csv: cannot open " + path)
    with out:
        out.write("layer,step,T,total_load,modeled_latency_us" + (",divergence" if has_div else "")
                  + "\n")
        for r in trace.records:
            line = f"{r.layer},{r.step},{r.active_experts},{r.total_load},{_fmt(r.modeled_latency_us)}"
            if has_div:
                line += "," + _fmt(r.divergence if r.divergence is not None else 0.0)
            out.write(line + "\n")


def gen_config_json(gen: ScoreGenConfig) -> dict:
    """json_io.cpp:24-47"""
    j = {"kind": gen_to_string(gen.kind), "n_experts": gen.n_experts, "batch": gen.batch,
         "steps": gen.steps, "layers": gen.layers, "seed": int(gen.seed)}
    if gen.kind == GenKind.Dirichlet:
        j["alpha"] = float(gen.alpha)
    elif gen.kind == GenKind.Clustered:
        j.update({"groups": gen.groups,
                  "within_group_concentration": float(gen.within_group_concentration),
                  "between_group_spread": float(gen.between_group_spread)})
    else:
        j["trace_path"] = gen.trace_path
    return j


def _write_json(path: str, j: dict) -> None:
    with open(path, "w") as f:  # write_json_file, json_io.cpp:93-99
        f.write(json.dumps(j, sort_keys=True, indent=2) + "\n")


def write_trace_summary_json(path: str, trace: DecodeTrace, gen: ScoreGenConfig,
                             latency: LatencyParams) -> None:
    """simulate.cpp:287-312"""
    a = trace.aggregates
    agg = {k: getattr(a, k) for k in (
        "mean_active_experts", "mean_total_load", "mean_latency_us", "vanilla_mean_active_experts",
        "vanilla_mean_total_load", "vanilla_mean_latency_us", "normalized_active_experts",
        "normalized_latency")}
    if a.mean_divergence is not None:
        agg["mean_divergence"] = a.mean_divergence
    _write_json(path, {"schema_version": 1, "type": "trace_summary",
                       "routing": routing_config_json(trace.routing),
                       "score_gen": gen_config_json(gen),
                       "latency_model": {"a_us": latency.a_us, "b_us": latency.b_us},
                       "steps_recorded": len(trace.records), "aggregates": agg})


def write_padding_json(path: str, rep: PaddingReport, gen: ScoreGenConfig,
                       routing: RoutingConfig, latency: LatencyParams) -> None:
    """simulate.cpp:314-343"""
    _write_json(path, {
        "schema_version": 1, "type": "padding_report", "real_batch": rep.real_batch,
        "padded_batch": rep.padded_batch,
        "routing": routing_config_json(routing.resolved(gen.n_experts)),
        "score_gen": gen_config_json(gen),
        "latency_model": {"a_us": latency.a_us, "b_us": latency.b_us},
        "masked_matches_no_padding": rep.masked_matches_no_padding,
        "variants": {v.name: {"mean_active_experts": v.mean_active_experts,
                              "mean_total_load": v.mean_total_load,
                              "mean_latency_us": v.mean_latency_us}
                     for v in (rep.no_padding, rep.naive_padding, rep.masked_padding)}})


# ---------------------------------------------------------------------------
# Config sweep and Pareto frontier (sweep.cpp:48-230)
# ---------------------------------------------------------------------------
@dataclass
class RoundingRule:
    """sweep.hpp:24-28"""
    enabled: bool = False
    quality_bin: float = 0.005
    experts_bin: float = 0.1


@dataclass
class SweepPoint:
    """sweep.hpp:30-35"""
    config: RoutingConfig
    mean_active_experts: float = 0.0
    quality_delta: Optional[float] = None
    rounded: bool = False


def default_sweep_grid(n_experts: int, k: int) -> List[RoutingConfig]:
    """sweep.cpp:48-75: vanilla(k) then oea(k0, p, k_max, max_p, k) over
    k0 in [ceil(k/2), k], k_max in [max(k-1, k0), k + max(1, 3k/8)], p in
    0.4..1.0, max_p in {k, 2k, 4k, N} (deduplicated, capped at N)."""
    if n_experts < 1 or k < 1 or k > n_experts:
        raise InvalidArgument("default_sweep_grid: need 1 <= k <= N")
    max_ps: List[int] = []
    for m in (k, 2 * k, 4 * k, n_experts):
        m = min(m, n_experts)
        if m not in max_ps:
            max_ps.append(m)
    k0_lo = max(1, (k + 1) // 2)
    kmax_lo = max(1, k - 1)
    kmax_hi = min(n_experts, k + max(1, (3 * k) // 8))
    grid = [RoutingConfig.vanilla(k)]
    for k0 in range(k0_lo, min(k, n_experts) + 1):
        for kmax in range(max(kmax_lo, k0), kmax_hi + 1):
            for pi in range(4, 11):
                for max_p in max_ps:
                    grid.append(RoutingConfig.oea(k0, pi / 10.0, kmax, max_p, k))
    return grid


def _round_half_away(x: float) -> float:  # std::round
    import math
    f = math.floor(abs(x))
    r = f + 1.0 if abs(x) - f >= 0.5 else f
    return math.copysign(r, x)


def _snap(v: float, b: float) -> float:
    return _round_half_away(v / b) * b


def sweep(gen: ScoreGenConfig, grid: List[RoutingConfig], latency: LatencyParams,
          rounding: RoundingRule = RoundingRule(), layer=None) -> List[SweepPoint]:
    """sweep.cpp:77-106 for a score source: mean T per routing config. The
    cells are generated once (one launch) and each config routes all of them
    in one batched call; the reference re-simulates (and shadow-routes
    vanilla) per config. latency is part of the reference signature; the
    points carry only T and the quality delta (none for score sources)."""
    if not grid:
        raise InvalidArgument("sweep: empty config grid")
    if layer is not None:  # quality = mean output divergence vs vanilla (sweep.cpp:88-99)
        pts = []
        for c in grid:
            tr = simulate_decode_layer(layer, gen, c, latency)
            pt = SweepPoint(config=tr.routing, mean_active_experts=tr.aggregates.mean_active_experts,
                            quality_delta=tr.aggregates.mean_divergence)
            if rounding.enabled:
                pt.mean_active_experts = _snap(pt.mean_active_experts, rounding.experts_bin)
                if pt.quality_delta is not None:
                    pt.quality_delta = _snap(pt.quality_delta, rounding.quality_bin)
                pt.rounded = True
            pts.append(pt)
        return pts
    from .routing import BatchedScores
    cfg, cells = cell_scores(gen)
    batched = BatchedScores(cells)  # concatenated once; each config exports only T
    n = float(len(cells))
    pts = []
    for c in grid:
        rc = c.resolved(cfg.n_experts)
        s = 0.0
        for t in batched.route_counts(rc)[0].tolist():
            s += t
        pt = SweepPoint(config=rc, mean_active_experts=s / n)
        if rounding.enabled:
            pt.mean_active_experts = _snap(pt.mean_active_experts, rounding.experts_bin)
            pt.rounded = True
        pts.append(pt)
    return pts


def _dominates(a: SweepPoint, b: SweepPoint) -> bool:
    aq, bq = a.quality_delta or 0.0, b.quality_delta or 0.0
    if a.mean_active_experts > b.mean_active_experts or aq > bq:
        return False
    return a.mean_active_experts < b.mean_active_experts or aq < bq


def pareto_indices(pts: List[SweepPoint]) -> List[int]:
    """sweep.cpp:108-122"""
    return [i for i in range(len(pts))
            if not any(j != i and _dominates(pts[j], pts[i]) for j in range(len(pts)))]


def pareto_frontier(pts: List[SweepPoint]) -> List[SweepPoint]:
    """sweep.cpp:124-142: non-dominated points by (T, quality, index)."""
    idx = sorted(pareto_indices(pts),
                 key=lambda i: (pts[i].mean_active_experts, pts[i].quality_delta or 0.0, i))
    return [pts[i] for i in idx]


_SWEEP_HEADER = ["mode", "k", "k0", "p", "k_max", "max_p", "cap", "mean_active_experts",
                 "quality_delta", "rounded"]


def write_sweep_csv(path: str, pts: List[SweepPoint]) -> None:
    """sweep.cpp:144-162"""
    from .routing import to_string as rs
    try:
        out = open(path, "w")
    except OSError:
        raise InvalidArgument("write_sweep_csv: cannot open " + path)
    with out:
        out.write(",".join(_SWEEP_HEADER) + "\n")
        for p in pts:
            c = p.config
            q = _fmt(p.quality_delta) if p.quality_delta is not None else ""
            out.write(f"{rs(c.mode)},{c.k},{c.k0},{_fmt(c.p)},{c.k_max},{c.max_p},{rs(c.cap)},"
                      f"{_fmt(p.mean_active_experts)},{q},{1 if p.rounded else 0}\n")


def read_sweep_csv(path: str) -> List[SweepPoint]:
    """sweep.cpp:164-228 (same checks and messages)."""
    from .routing import cap_semantics_from_string, routing_mode_from_string
    try:
        f = open(path)
    except OSError:
        raise InvalidArgument("read_sweep_csv: cannot open " + path)
    with f:
        lines = f.read().split("\n")
    if not lines or lines == [""]:
        raise InvalidArgument(f"read_sweep_csv: {path} is empty")
    if [h.rstrip("\r ") for h in lines[0].split(",")] != _SWEEP_HEADER:
        raise InvalidArgument(f"read_sweep_csv: {path} has an unexpected header")
    pts = []
    for line_no, line in enumerate(lines[1:], start=2):
        if line.strip(" \t\r") == "":
            continue
        fl = line.rstrip("\r").split(",")
        where = f"read_sweep_csv: {path} line {line_no}"
        if len(fl) != len(_SWEEP_HEADER):
            raise InvalidArgument(where + ": wrong column count")
        try:
            cfg = RoutingConfig(routing_mode_from_string(fl[0]), int(fl[1]), int(fl[2]),
                                float(fl[3]), int(fl[4]), int(fl[5]),
                                cap_semantics_from_string(fl[6]))
            pts.append(SweepPoint(cfg, float(fl[7]), float(fl[8]) if fl[8] else None,
                                  int(fl[9]) != 0))
        except (ValueError, InvalidArgument) as e:
            raise InvalidArgument(f"{where}: {e}")
    if not pts:
        raise InvalidArgument(f"read_sweep_csv: {path} has no rows")
    return pts


# ---------------------------------------------------------------------------
# Toy-layer simulation (simulate.cpp:153-183): the layer's own router scores
# per-(step, layer, token) embeddings, and every record also carries the mean
# relative divergence of the routed output from the vanilla top-k mixture.
# ---------------------------------------------------------------------------
def simulate_decode_layer(layer, gen: ScoreGenConfig, routing: RoutingConfig,
                          latency: LatencyParams) -> DecodeTrace:
    """simulate_decode(layer, gen, routing, latency): `layer` is a
    DeviceMoeLayer (f64 / f32) or host MoeLayerParams; gen supplies batch,
    steps, layers and seed (gen.kind is ignored). Router scores, both routes
    (one batched call each for all cells) and both moe_forward mixtures run on
    the GPU."""
    from .moe_layer import DeviceMoeLayer, MoeLayerParams, _flat_plan, make_random_batch, \
        output_divergence
    if gen.batch < 1 or gen.steps < 1 or gen.layers < 1:
        raise InvalidArgument("simulate_decode: batch, steps and layers must be >= 1")
    dev = DeviceMoeLayer.from_params(layer) if isinstance(layer, MoeLayerParams) else layer
    if gen.n_experts != dev.N:
        raise InvalidArgument(f"simulate_decode: gen.n_experts {gen.n_experts} does not match "
                              f"layer expert count {dev.N}")
    rcfg = routing.resolved(dev.N)
    vcfg = RoutingConfig.vanilla(routing.k).resolved(dev.N)
    cells = [(s, l) for s in range(gen.steps) for l in range(gen.layers)]
    xs = [make_random_batch(gen.batch, dev.D, gen.seed, s, l).embeddings for s, l in cells]
    scores = [ScoreMatrix(dev.router_scores(x)) for x in xs]
    plans = route_batched(scores, rcfg)
    vplans = route_batched(scores, vcfg)
    tr = DecodeTrace(routing=rcfg)
    for (s, l), x, p, vp in zip(cells, xs, plans, vplans):
        ref = dev.forward_plan(x, *_flat_plan(vp))
        got = dev.forward_plan(x, *_flat_plan(p))
        rec = _record(s, l, p, latency)
        rec.divergence = output_divergence(ref, got).mean_relative_error
        tr.records.append(rec)
        tr.vanilla_records.append(_record(s, l, vp, latency))
    tr.aggregates = _aggregates(tr.records, tr.vanilla_records)
    return tr
