"""Score traces and batched routing of them.

Mirrors the reference's trace I/O and its `route` command:
  * read_score_trace / write_score_trace — ndjson, a `score_trace` header of
    schema version 1 then one record per (step, layer) batch (io.cpp:40-172,
    same validation and error texts);
  * route_trace — every record routed in one GPU launch sequence
    (routing.route_batched -> oea_route_f64_batched_host) instead of the
    reference's record-by-record loop (oea_cli.cpp:153-175);
  * routing_plans_json / write_routing_plans — the `routing_plans` document
    (oea_cli.cpp:166-171, plan_json and routing_config_json of json_io.cpp).
JSON objects are written with sorted keys, as nlohmann::json's std::map does.
"""
from __future__ import annotations

import json
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from ._capi import InvalidArgument
from .routing import RoutingConfig, RoutingMode, RoutingPlan, ScoreMatrix, route_batched, to_string

__all__ = ["SCORE_TRACE_SCHEMA_VERSION", "ScoreRecord", "read_score_trace", "write_score_trace",
           "route_trace", "routing_config_json", "plan_json", "routing_plans_json",
           "write_routing_plans"]

SCORE_TRACE_SCHEMA_VERSION = 1  # io.hpp:18


@dataclass
class ScoreRecord:
    """io.hpp:20-24"""
    step: int
    layer: int
    scores: ScoreMatrix


def _dumps(j) -> str:
    return json.dumps(j, sort_keys=True, separators=(",", ":"), allow_nan=False)


def write_score_trace(path: str, records: List[ScoreRecord]) -> None:
    """io.cpp:40-83"""
    if not records:
        raise InvalidArgument("write_score_trace: no records")
    n = records[0].scores.experts()
    try:
        out = open(path, "w")
    except OSError:
        raise InvalidArgument("write_score_trace: cannot open " + path)
    with out:
        out.write(_dumps({"schema_version": SCORE_TRACE_SCHEMA_VERSION, "type": "score_trace",
                          "n_experts": n}) + "\n")
        for rec in records:
            if rec.scores.experts() != n:
                raise InvalidArgument("write_score_trace: inconsistent expert count at step "
                                      + str(rec.step))
            j = {"step": int(rec.step), "layer": int(rec.layer),
                 "scores": [[float(v) for v in row] for row in rec.scores.scores]}
            if rec.scores.mask is not None and len(rec.scores.mask) > 0:
                j["mask"] = [bool(v) for v in rec.scores.mask]
            out.write(_dumps(j) + "\n")


def _get_int(j, key):
    v = j[key]
    if isinstance(v, bool) or not isinstance(v, (int, float)) or int(v) != v:
        raise InvalidArgument(f"[json.exception.type_error] {key} is not a number")
    return int(v)


def read_score_trace(path: str) -> List[ScoreRecord]:
    """io.cpp:85-172: header check, per-record shape checks, mask length,
    ScoreMatrix::validate (routing.cpp:53-79); errors name the file, record
    and line."""
    try:
        f = open(path)
    except OSError:
        raise InvalidArgument("read_score_trace: cannot open " + path)
    records: List[ScoreRecord] = []
    saw_header = False
    n_experts = 0
    with f:
        for line_no, line in enumerate(f, start=1):
            if line.strip(" \t\r\n") == "":
                continue
            try:
                j = json.loads(line)
            except ValueError as e:
                raise InvalidArgument(f"read_score_trace: {path} line {line_no}: {e}")
            if not saw_header:
                if (not isinstance(j, dict) or j.get("type", "") != "score_trace"
                        or j.get("schema_version", 0) != SCORE_TRACE_SCHEMA_VERSION):
                    raise InvalidArgument(
                        f"read_score_trace: {path} does not start with a score_trace header of "
                        f"schema version {SCORE_TRACE_SCHEMA_VERSION}")
                n_experts = int(j["n_experts"])
                if n_experts < 1:
                    raise InvalidArgument(f"read_score_trace: {path}: n_experts must be >= 1")
                saw_header = True
                continue
            where = f"{path} record {len(records)} (line {line_no})"
            try:
                if not isinstance(j, dict):
                    raise InvalidArgument("record is not an object")
                step = _get_int(j, "step")
                layer = _get_int(j, "layer")
                rows = j["scores"]
                if not isinstance(rows, list) or not rows:
                    raise InvalidArgument("scores must be a non-empty array")
                b = len(rows)
                sc = np.empty((b, n_experts), np.float64)
                for i, row in enumerate(rows):
                    if not isinstance(row, list) or len(row) != n_experts:
                        raise InvalidArgument(f"row {i} does not have n_experts entries")
                    sc[i] = [float(v) for v in row]
                mask = None
                if "mask" in j:
                    m = j["mask"]
                    if not isinstance(m, list) or len(m) != b:
                        raise InvalidArgument("mask length does not match batch")
                    mask = np.array([bool(v) for v in m], bool)
                sm = ScoreMatrix(sc, mask)
                sm.validate()
            except (InvalidArgument, KeyError, TypeError, ValueError) as e:
                msg = str(e) if not isinstance(e, KeyError) else f"key {e} not found"
                raise InvalidArgument(f"read_score_trace: {where}: {msg}")
            records.append(ScoreRecord(step, layer, sm))
    if not saw_header:
        raise InvalidArgument(f"read_score_trace: {path} is empty")
    if not records:
        raise InvalidArgument(f"read_score_trace: {path} has a header but no records")
    return records


def route_trace(records: List[ScoreRecord], cfg: RoutingConfig) -> List[RoutingPlan]:
    """Every record's route(scores, cfg) from one batched GPU call."""
    if not records:
        raise InvalidArgument("route_trace: no records")
    return route_batched([r.scores for r in records], cfg)


def routing_config_json(cfg: RoutingConfig) -> dict:
    """json_io.cpp:10-22"""
    j = {"mode": to_string(cfg.mode), "k": int(cfg.k)}
    if cfg.mode != RoutingMode.Vanilla:
        j.update({"k0": int(cfg.k0), "p": float(cfg.p), "k_max": int(cfg.k_max),
                  "max_p": int(cfg.max_p), "cap": to_string(cfg.cap)})
    return j


def plan_json(plan: RoutingPlan) -> dict:
    """json_io.cpp:64-84"""
    return {"n_experts": int(plan.n_experts), "active_experts": int(plan.active_count),
            "total_load": int(plan.total_load),
            "active_union": [int(e) for e in plan.active_union],
            "loads": [int(v) for v in plan.loads],
            "tokens": [{"experts": [int(e) for e in s], "weights": [float(w) for w in ws]}
                       for s, ws in zip(plan.sets, plan.weights)]}


def routing_plans_json(records: List[ScoreRecord], cfg: RoutingConfig,
                       plans: Optional[List[RoutingPlan]] = None) -> dict:
    """The `route` command's document (oea_cli.cpp:153-175): the resolved
    routing config and one plan per record (routed here on the GPU unless
    given)."""
    if not records:
        raise InvalidArgument("route_trace: no records")
    rcfg = cfg.resolved(records[0].scores.experts())
    if plans is None:
        plans = route_trace(records, rcfg)
    return {"schema_version": 1, "type": "routing_plans", "routing": routing_config_json(rcfg),
            "records": [{"step": int(r.step), "layer": int(r.layer), "plan": plan_json(p)}
                        for r, p in zip(records, plans)]}


def write_routing_plans(path: str, doc: dict) -> None:
    """write_json_file (json_io.cpp:93-99): 2-space indent, trailing newline."""
    try:
        out = open(path, "w")
    except OSError:
        raise InvalidArgument("write_json_file: cannot open " + path)
    with out:
        out.write(json.dumps(doc, sort_keys=True, indent=2, allow_nan=False) + "\n")
