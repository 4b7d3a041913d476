"""Latency model on measured decode data — the host-side mirror of the
reference's `proj/include/oea/latency.hpp` / `proj/src/latency.cpp` and the
latency CSV I/O of `proj/src/io.cpp:174-237`.

The B200 bench (`bench.py --config c2`) measures (T, µs) per layer call over
the B x k0 sweep; `fit_linear` is the OLS of µs on T with the reference's
exact formulas and error texts, so the reference's own `fit-latency` reads
the CSV this module writes.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Sequence


@dataclass
class LatencyObservation:
    """`LatencyObservation` (latency.hpp): one layer call's active experts T
    and its latency in µs."""
    active_experts: int
    latency_us: float


@dataclass
class FitResult:
    """`FitResult` (latency.hpp): latency ≈ intercept_us + b_us · T."""
    b_us: float
    intercept_us: float
    r_squared: float
    residual_std: float = 0.0
    slope_stderr: float = 0.0
    intercept_stderr: float = 0.0


def expected_active_experts(n_experts: int, k: int, batch: int) -> float:
    """E[T] = N (1 - (1 - k/N)^B) for i.i.d. uniform top-k (latency.cpp:30-37)."""
    if n_experts < 1 or k < 1 or k > n_experts or batch < 1:
        raise ValueError("expected_active_experts: need 1 <= k <= N and B >= 1")
    miss = 1.0 - k / n_experts
    return n_experts * (1.0 - miss ** batch)


def fit_linear(observations: Sequence[LatencyObservation]) -> FitResult:
    """Ordinary least squares of latency_us on T (latency.cpp:39-85): slope
    sxy/sxx, intercept mean_y - b mean_x, R^2 = 1 - ssr/syy, and for n > 2 the
    residual std and standard errors."""
    n = len(observations)
    if n < 2:
        raise ValueError("fit_linear: need at least 2 observations")
    mean_x = sum(o.active_experts for o in observations) / n
    mean_y = sum(o.latency_us for o in observations) / n
    sxx = sxy = syy = 0.0
    for o in observations:
        dx = o.active_experts - mean_x
        dy = o.latency_us - mean_y
        sxx += dx * dx
        sxy += dx * dy
        syy += dy * dy
    if sxx <= 0.0:
        raise ArithmeticError(
            "fit_linear: all observations share one T value (degenerate design)")
    b = sxy / sxx
    a = mean_y - b * mean_x
    ssr = 0.0
    for o in observations:
        e = o.latency_us - (a + b * o.active_experts)
        ssr += e * e
    fit = FitResult(b_us=b, intercept_us=a, r_squared=1.0 - ssr / syy if syy > 0.0 else 1.0)
    if n > 2:
        sigma2 = ssr / (n - 2)
        fit.residual_std = math.sqrt(sigma2)
        fit.slope_stderr = math.sqrt(sigma2 / sxx)
        fit.intercept_stderr = math.sqrt(sigma2 * (1.0 / n + mean_x * mean_x / sxx))
    return fit


def _format_double(v: float) -> str:
    # io.cpp format_double: shortest round-trip representation
    return repr(float(v))


def write_latency_csv(path: str, obs: Sequence[LatencyObservation]) -> None:
    """`write_latency_csv` (io.cpp:174-184): header `T,latency_us`."""
    with open(path, "w") as f:
        f.write("T,latency_us\n")
        for o in obs:
            f.write(f"{int(o.active_experts)},{_format_double(o.latency_us)}\n")


def read_latency_csv(path: str) -> List[LatencyObservation]:
    """`read_latency_csv` (io.cpp:186-237): columns located by header name."""
    try:
        lines = open(path).read().splitlines()
    except OSError:
        raise ValueError(f"read_latency_csv: cannot open {path}")
    if not lines:
        raise ValueError(f"read_latency_csv: {path} is empty")
    header = [h.strip() for h in lines[0].split(",")]
    if "T" not in header or "latency_us" not in header:
        raise ValueError(f"read_latency_csv: {path} header must contain columns 'T' and 'latency_us'")
    tc, lc = header.index("T"), header.index("latency_us")
    obs = []
    for no, line in enumerate(lines[1:], start=2):
        if not line.strip():
            continue
        fields = line.split(",")
        where = f"read_latency_csv: {path} line {no}"
        if len(fields) <= max(tc, lc):
            raise ValueError(f"{where}: too few columns")
        try:
            t = int(fields[tc])
            us = float(fields[lc])
        except ValueError as e:
            raise ValueError(f"{where}: {e}")
        if t < 0 or not math.isfinite(us):
            raise ValueError(f"{where}: non-finite or negative value")
        obs.append(LatencyObservation(t, us))
    if not obs:
        raise ValueError(f"read_latency_csv: {path} has no observations")
    return obs


def latency_svg(obs: Sequence[LatencyObservation], fit: FitResult, title: str,
                width: int = 640, height: int = 420) -> str:
    """A dependency-free SVG scatter of (T, µs) with the fitted line."""
    xs = [o.active_experts for o in obs]
    ys = [o.latency_us for o in obs]
    x0, x1 = 0.0, max(xs) * 1.05
    y0, y1 = 0.0, max(ys) * 1.1
    ml, mr, mt, mb = 60, 20, 40, 50
    pw, ph = width - ml - mr, height - mt - mb

    def px(x):
        return ml + (x - x0) / (x1 - x0) * pw

    def py(y):
        return mt + ph - (y - y0) / (y1 - y0) * ph

    out = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{width}" height="{height}" '
           f'font-family="sans-serif" font-size="12">',
           f'<rect width="{width}" height="{height}" fill="white"/>',
           f'<text x="{width / 2}" y="20" text-anchor="middle" font-size="14">{title}</text>',
           f'<line x1="{ml}" y1="{mt + ph}" x2="{ml + pw}" y2="{mt + ph}" stroke="black"/>',
           f'<line x1="{ml}" y1="{mt}" x2="{ml}" y2="{mt + ph}" stroke="black"/>']
    for i in range(6):
        xv = x0 + (x1 - x0) * i / 5
        yv = y0 + (y1 - y0) * i / 5
        out.append(f'<text x="{px(xv):.1f}" y="{mt + ph + 16}" text-anchor="middle">{xv:.0f}</text>')
        out.append(f'<text x="{ml - 6}" y="{py(yv) + 4:.1f}" text-anchor="end">{yv:.0f}</text>')
    out.append(f'<text x="{ml + pw / 2}" y="{height - 10}" text-anchor="middle">'
               f'unique activated experts T</text>')
    out.append(f'<text x="14" y="{mt + ph / 2}" text-anchor="middle" '
               f'transform="rotate(-90 14 {mt + ph / 2})">layer latency (µs)</text>')
    for x, y in zip(xs, ys):
        out.append(f'<circle cx="{px(x):.1f}" cy="{py(y):.1f}" r="2.5" fill="#1f77b4" '
                   f'fill-opacity="0.6"/>')
    out.append(f'<line x1="{px(x0):.1f}" y1="{py(fit.intercept_us):.1f}" x2="{px(x1):.1f}" '
               f'y2="{py(fit.intercept_us + fit.b_us * x1):.1f}" stroke="#d62728" stroke-width="2"/>')
    out.append(f'<text x="{ml + 10}" y="{mt + 14}">fit: {fit.intercept_us:.2f} µs + '
               f'{fit.b_us:.3f} µs·T, R² = {fit.r_squared:.4f}, n = {len(obs)}</text>')
    out.append("</svg>")
    return "\n".join(out)
