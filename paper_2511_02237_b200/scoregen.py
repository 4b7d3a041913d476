"""Router-score generators on the GPU.

Mirror of the reference's ScoreGenConfig / ScoreSource / gen_scores
(score_gen.hpp, score_gen.cpp:46-160): Dirichlet(alpha) batches (Marsaglia-
Tsang gammas over the counter RNG, rng.hpp:82-98) and clustered batches
(softmax of a group template plus token noise). Replay sources are score
traces (traces.read_score_trace). Generation runs on the device
(oea_gen_scores: one thread per row, every (step, layer) cell of a run in one
launch); rows equal the reference's within ~1e-15 relative (device libm).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from ._capi import InvalidArgument, ScoreGenCfgC, default_context, lib
from .routing import ScoreMatrix

__all__ = ["GenKind", "ScoreGenConfig", "gen_scores", "gen_run", "gen_run_device",
           "to_string", "gen_kind_from_string"]


class GenKind(IntEnum):
    Dirichlet = 0
    Clustered = 1
    Replay = 2


_NAMES = {GenKind.Dirichlet: "dirichlet", GenKind.Clustered: "clustered", GenKind.Replay: "replay"}


def to_string(kind: GenKind) -> str:
    """score_gen.cpp:27-37"""
    return _NAMES[GenKind(kind)]


def gen_kind_from_string(s: str) -> GenKind:
    """score_gen.cpp:39-44"""
    for k, v in _NAMES.items():
        if v == s:
            return k
    raise InvalidArgument(f"unknown score generator '{s}'")


@dataclass
class ScoreGenConfig:
    """score_gen.hpp:29-52 (defaults as the reference)."""
    kind: GenKind = GenKind.Dirichlet
    n_experts: int = 128
    batch: int = 16
    steps: int = 1
    layers: int = 1
    seed: int = 0
    alpha: float = 1.0
    groups: int = 2
    within_group_concentration: float = 4.0
    between_group_spread: float = 2.0
    trace_path: str = ""

    def to_c(self) -> ScoreGenCfgC:
        if self.kind == GenKind.Replay:
            raise InvalidArgument("score gen: replay is read on the host (read_score_trace)")
        return ScoreGenCfgC(int(self.kind), self.n_experts, self.batch, self.steps, self.layers,
                            int(self.seed) & 0xFFFFFFFFFFFFFFFF, float(self.alpha), self.groups,
                            float(self.within_group_concentration),
                            float(self.between_group_spread))


def gen_run(cfg: ScoreGenConfig, step0: int = 0, nsteps: int | None = None) -> np.ndarray:
    """Every (step, layer) cell of steps [step0, step0 + nsteps) from one
    launch: [nsteps][layers][batch][n_experts] f64 (host)."""
    nsteps = cfg.steps - step0 if nsteps is None else nsteps
    out = np.empty((max(nsteps, 1), max(cfg.layers, 1), max(cfg.batch, 1),
                    max(cfg.n_experts, 1)), np.float64)
    ctx = default_context()
    c = cfg.to_c()
    ctx.check(lib().oea_gen_scores_host(ctx.h, C.byref(c), step0, nsteps,
                                        out.ctypes.data_as(C.c_void_p)))
    return out


def gen_run_device(cfg: ScoreGenConfig, out_ptr: int, step0: int = 0,
                   nsteps: int | None = None, stream=None) -> None:
    """Device variant: writes [nsteps][layers][batch][n_experts] f64 at out_ptr."""
    nsteps = cfg.steps - step0 if nsteps is None else nsteps
    ctx = default_context()
    c = cfg.to_c()
    ctx.check(lib().oea_gen_scores(ctx.h, C.byref(c), step0, nsteps, C.c_void_p(out_ptr),
                                   C.c_void_p(stream) if stream else None))


def gen_scores(cfg: ScoreGenConfig, step: int, layer: int) -> ScoreMatrix:
    """gen_scores (score_gen.cpp:163-165) of one (step, layer) cell."""
    if layer < 0 or layer >= cfg.layers:
        raise InvalidArgument("score source: step/layer out of range")
    return ScoreMatrix(gen_run(cfg, step, 1)[0, layer])
