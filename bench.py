#!/usr/bin/env python
"""Benchmark of the B200-native OEA MoE decode layer (BASELINE.json metric:
"MoE-layer decode µs at B=16 (OEA vs top-k), % HBM roofline, unique experts").

Workload (BASELINE.json configs[0], the 1-GPU headline): a Qwen3-30B-A3B-shaped
MoE decode layer (N=128 experts, k=8, d_model=2048, d_ff=768), B=16 tokens,
random bf16 weights with make_random_layer's distributions, OEA simplified
routing k0=4 (headline) and vanilla top-8 (comparison).

One "step" = one layer call: fused router (gate GEMV, ranking, batch union,
piggyback, renormalisation, compaction) + grouped SwiGLU FFN + combine, one
kernel launch. The K timed steps run back to back as ONE CUDA graph of K
layer calls (the way a decode step's layers run; each fused launch is a
programmatic dependent of its predecessor, PDL), between CUDA events on the
launching stream; `value` = device µs per step, inputs resident. L2 is
defeated by rotating 4 distinct layer copies (4.8 GB) and a distinct token
batch per step (each call streams ~480 MB of expert weights, >> 126 MB L2).
The same steps as one graph per call are reported as `isolated_graph_us`.
`e2e` = the same call through the C ABI from pinned host buffers (the input
copy in and the output copy out inside the timed region).

Extra keys of the default line (same run, same clocks record): C3 (the
Qwen3-235B-shaped layer, OEA and top-8), the C2 points at B=16 for k0=1..8
(latency vs unique experts), and C5 (router-only B=4096 route).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

--gpus N without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one per GPU). For N > 1 the line is
EXPERT PARALLEL (BASELINE configs[3]): the C1 layer's experts sharded in
contiguous blocks over the N GPUs, tokens data-parallel (B/N per rank), with
NCCL all-to-all dispatch / combine (`value`), plus the all-gather +
reduce-scatter and the peer-memory combine paths, the C3 layer sharded and
the 94-layer C3-shaped stack; timings are max over ranks.

--impl reference times the reference's own CPU path (router_scores + route +
moe_forward<double>, compiled from the reference sources into oracle/_ref) on
the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE-layer decode µs at B=16 (OEA vs top-k), % HBM roofline, unique experts"
D, H, N, K_TOP, B = 2048, 768, 128, 8, 16
K0 = 4
ROTATE = 4
FALLBACK_HBM_GBS = 6650.0


def load_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (of measured)"
    except Exception:
        return FALLBACK_HBM_GBS, "B200_PROFILING.md fallback (of fallback)"


def load_traffic():
    """(dram bytes per launch, dram / algorithmic bytes of that launch) of the
    fused kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f).get("k_ffn_bf16<2>", {})
        return d.get("dram_bytes_per_launch"), d.get("dram_over_algorithmic")
    except Exception:
        return None, None


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([v.strip() for v in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference itself (oracle/_ref) or the C port.
# ---------------------------------------------------------------------------
def cpu_reference_decode(calls: int, threads: int, cfg_tuple, steps: int = 1, warmup: int = 0):
    """Times the reference CPU decode cell (router_scores -> route ->
    moe_forward<double>, moe_layer.hpp:71-158 + routing.cpp:305-326) on a
    make_random_layer C1 layer (built once): `warmup` untimed steps, then
    `steps` timed steps of `calls` decode calls each on `threads` host
    threads. Returns (per-step us per call list, kind, cores, sample)."""
    import numpy as np

    import oracle
    kind = "reference" if oracle.reference_available() else "port"
    xs = [oracle.make_random_batch(B, D, 1000 + i, step=i) for i in range(calls)]
    if kind == "reference":
        ref = oracle.Reference()
        layer = ref.random_layer(D, H, N, 1, "f64", threads=os.cpu_count() or 1)
        run = lambda x: layer.decode(x, cfg_tuple)  # noqa: E731
    else:
        router, wg, wu, wd = oracle.make_random_layer(D, H, N, 1)

        def run(x):
            plan = oracle.route(oracle.router_scores(x, router), cfg_tuple)
            return oracle.moe_forward(wg, wu, wd, x, plan.sets, plan.set_len, plan.weights)
    run(xs[0])  # warm caches / page in

    def one_step():
        t0 = time.perf_counter()
        if threads <= 1:
            for x in xs:
                run(x)
        else:
            idx = list(range(calls))
            lock = threading.Lock()

            def worker():
                while True:
                    with lock:
                        if not idx:
                            return
                        i = idx.pop()
                    run(xs[i])
            ths = [threading.Thread(target=worker) for _ in range(threads)]
            for t in ths:
                t.start()
            for t in ths:
                t.join()
        return (time.perf_counter() - t0) * 1e6 / calls

    for _ in range(warmup):
        one_step()
    vals = [one_step() for _ in range(max(1, steps))]
    sample = (f"{calls} C1 decode call(s) per sample (B=16, D=2048, H=768, N=128, simplified "
              f"k0=4/k=8): router_scores + route + moe_forward<double> of the "
              f"{'reference sources compiled unmodified against the repo Eigen-subset shim (-O3; its naive loops stand in for Eigen GEMMs)' if kind == 'reference' else 'C restatement'}"
              f", {threads} thread(s), {max(1, steps)} sample(s)")
    return vals, kind, threads, sample


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    calls = max(threads, 4)
    cfg = (3, K_TOP, K0, 1.0, K_TOP, 0, 0)  # simplified(4, 8)
    # each sample: `calls` layer calls spread over the host threads (~0.5 s);
    # the layer is built once. A step = one layer call (as in our arm).
    vals, kind, cores, sample = cpu_reference_decode(calls, threads, cfg, steps=args.steps,
                                                     warmup=args.warmup)
    us = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": us, "unit": "us/layer-call",
            "n_gpus": args.gpus, "steps": len(vals) * calls, "warmup": args.warmup * calls,
            "ms_per_step": us / 1000.0,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: make_random_layer weights, make_random_batch tokens",
            "config": {"workload": "C1 Qwen3-30B-A3B-shaped MoE decode layer (BASELINE configs[0])",
                       "D": D, "H": H, "N": N, "k": K_TOP, "B": B,
                       "routing": f"simplified(k0={K0}, k={K_TOP})", "parallelism": "host threads",
                       "samples": len(vals), "calls_per_sample": calls,
                       "statistic": "median over samples of (sample wall time / calls)"},
            "cpu_baseline": {"value": us, "unit": "us/layer-call", "cores": cores, "kind": kind,
                             "sample": sample, "nproc": os.cpu_count(), "cpu_model": cpu_model()},
            "e2e": {"value": us, "unit": "us/layer-call", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# Our arm.
# ---------------------------------------------------------------------------
def layer_bytes(T, D, H, N, B):
    """Algorithmic HBM bytes of one decode layer call: the T
    active experts' bf16 gate/up/down weights, the bf16 router, bf16 tokens in,
    fp32 outputs out."""
    return T * 3 * D * H * 2 + D * N * 2 + B * D * 2 + B * D * 4


def time_graphs(torch, stream, graphs, W, per_step=False, ctx=None):
    """Replays graphs[0:W] untimed, then graphs[W:] back to back between two
    events on the launching stream; per_step adds an event pair per launch.
    Returns (mean µs per launch, per-step µs or None, kernels launched in the
    timed region by this library)."""
    for i in range(W):
        graphs[i].launch()
    torch.cuda.synchronize()
    l0 = ctx.kernel_launches if ctx is not None else 0
    n = len(graphs) - W
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1 if per_step else 2)]
    with torch.cuda.stream(stream):
        ev[0].record(stream)
        for i in range(W, len(graphs)):
            graphs[i].launch()
            if per_step:
                ev[i - W + 1].record(stream)
        if not per_step:
            ev[1].record(stream)
    ev[-1].synchronize()
    total = ev[0].elapsed_time(ev[-1]) * 1000.0 / n
    steps = [ev[j].elapsed_time(ev[j + 1]) * 1000.0 for j in range(n)] if per_step else None
    launched = (ctx.kernel_launches - l0) if ctx is not None else None
    return total, steps, launched


def plan_stats(layers, xs, cfg, out, B, idx, ctx):
    Ts, loads = [], []
    for i in idx:
        L = layers[i % len(layers)]
        L.decode(xs[i], cfg, out)
        ctx.synchronize()
        p = L.last_plan(B, cfg)
        Ts.append(int(p["active_count"]))
        loads.append(int(p["total_load"]))
    return Ts, loads


def _free_port() -> int:
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    return port


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c1", choices=["c1", "c2", "c3", "c4", "c5", "sweep"],
                    help="c1 = the headline line (default; N > 1: expert parallel); c2 = full "
                         "B x k0 sweep + latency fit; c3 = Qwen3-235B-shaped layer; c4 = 94-layer "
                         "EP stack; c5 = router-only B=4096; sweep = the 673-config routing "
                         "sweep on the GPU simulator vs the reference's sweep on the host")
    ap.add_argument("--out-dir", default=os.path.join(ROOT, "gpurun_out", "bench"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="headline only (skip the C3 / C2 / C5 keys of the default line)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("OEA_BENCH_ONE_GPU"):  # functional check of N > 1 on one GPU
        local = 0
    torch.cuda.set_device(local)
    os.environ["OEA_DEVICE"] = str(local)
    dist = None
    if world > 1 and os.environ.get("OEA_BENCH_ONE_GPU"):
        # functional check of the N > 1 code on ONE GPU (NCCL refuses two ranks
        # per device): gloo collectives staged through host memory; timings
        # from such a run mean nothing
        import torch.distributed as tdist
        tdist.init_process_group("gloo")
        dist = _HostStagedDist(tdist, torch)
    elif world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    env = {"torch": torch, "dist": dist, "rank": rank, "world": world, "local": local}
    fn = {"c1": bench_c1 if world == 1 else bench_ep, "c2": bench_c2, "c3": bench_c3,
          "c4": bench_c4, "c5": bench_c5, "sweep": bench_sweep}[args.config]
    rc = fn(args, env)
    if dist is not None:
        dist.destroy_process_group()
    return rc


class _HostStagedDist:
    """torch.distributed look-alike over a gloo group that stages CUDA tensors
    through host memory (OEA_BENCH_ONE_GPU functional runs only)."""

    def __init__(self, d, torch):
        self.d, self.torch = d, torch
        self.ReduceOp = d.ReduceOp

    def __getattr__(self, name):
        return getattr(self.d, name)

    def _rt(self, fn, out, *ins, **kw):
        outs = out.cpu()
        fn(outs, *[i.cpu() for i in ins], **kw)
        out.copy_(outs)

    def all_gather_into_tensor(self, out, inp, group=None):
        self._rt(self.d.all_gather_into_tensor, out, inp, group=group)

    def reduce_scatter_tensor(self, out, inp, op=None, group=None):
        # (gloo has no reduce_scatter: all-reduce the whole tensor, keep ours)
        full = inp.cpu()
        self.d.all_reduce(full, group=group)
        out.copy_(full.chunk(self.d.get_world_size())[self.d.get_rank()])

    def all_to_all_single(self, out, inp, group=None):
        self._rt(self.d.all_to_all_single, out, inp, group=group)

    def all_reduce(self, t, op=None, group=None):
        c = t.cpu()
        self.d.all_reduce(c, op=op or self.d.ReduceOp.SUM, group=group)
        t.copy_(c)

    def all_gather(self, outs, t, group=None):
        co = [o.cpu() for o in outs]
        self.d.all_gather(co, t.cpu(), group=group)
        for o, c in zip(outs, co):
            o.copy_(c)


def _barrier(env):
    if env["dist"] is not None:
        env["dist"].barrier()


def _max_over_ranks(env, v):
    if env["dist"] is None:
        return v
    torch = env["torch"]
    t = torch.tensor([v], device="cuda", dtype=torch.float64)
    env["dist"].all_reduce(t, op=env["dist"].ReduceOp.MAX)
    return float(t.item())


def time_chain(torch, stream, layers, xs, cfg, out, W, K, ctx):
    """W warm-up then K timed layer calls (layers[i % len]: xs[i] -> out), each
    block captured as ONE CUDA graph of back-to-back decode calls (PDL edges),
    timed with CUDA events on the launching stream. Returns (µs per call,
    kernels launched by this library in the timed region)."""
    import paper_2511_02237_b200 as oea
    R = len(layers)
    # one eager call per layer first: large batches (B > 64) run the tcgen05
    # FFN, whose per-layer UMMA-layout weight copy is made on first use (a
    # stream capture cannot allocate it)
    for i in range(R):
        layers[i].decode(xs[i], cfg, out)
    warm = oea.DeviceMoeLayer.chain_graph([layers[i % R] for i in range(W)], list(xs[:W]), cfg,
                                          [out] * W)
    timed = oea.DeviceMoeLayer.chain_graph([layers[i % R] for i in range(W, W + K)],
                                           list(xs[W:W + K]), cfg, [out] * K)
    warm.launch()
    torch.cuda.synchronize()
    l0 = ctx.kernel_launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        timed.launch()
        e1.record(stream)
    e1.synchronize()
    us = e0.elapsed_time(e1) * 1000.0 / K
    launched = ctx.kernel_launches - l0
    warm.close()
    timed.close()
    return us, launched


def fit_points(pts):
    """OLS of µs on T over (T, µs) points (latency.cpp fit_linear's model)."""
    from paper_2511_02237_b200 import latency as lat
    f = lat.fit_linear([lat.LatencyObservation(t, u) for t, u in pts])
    return {"slope_us_per_expert": f.b_us, "intercept_us": f.intercept_us,
            "r_squared": f.r_squared}


def c3_extra(torch, stream, W, K, peak):
    """C3 (BASELINE configs[2]): the Qwen3-235B-A22B-shaped layer (D=4096,
    H=1536, N=128, k=8), B=16, OEA simplified(4, 8) and top-8."""
    import numpy as np
    import paper_2511_02237_b200 as oea
    D3, H3 = 4096, 1536
    layers = []
    for r in range(2):  # 2 x 4.83 GB; each call streams ~2-3 GB (>> 126 MB L2)
        L = oea.DeviceMoeLayer(D3, H3, N, "bf16")
        L.init_random(11 + r)
        layers.append(L)
    ctx = layers[0].ctx
    gen = torch.Generator(device="cuda").manual_seed(99)
    xs = torch.randn(W + K, B, D3, device="cuda", generator=gen).to(torch.bfloat16)
    out = torch.empty(B, D3, device="cuda", dtype=torch.float32)
    res = {}
    for name, cfg in (("oea", oea.RoutingConfig.simplified(K0, K_TOP)),
                      ("vanilla", oea.RoutingConfig.vanilla(K_TOP))):
        us, _ = time_chain(torch, stream, layers, xs, cfg, out, W, K, ctx)
        Ts, _ = plan_stats(layers, xs, cfg, out, B, range(W, W + K), ctx)
        T = float(np.mean(Ts))
        lb = layer_bytes(T, D3, H3, N, B)
        res[name] = {"us": us, "T_mean": T, "GBps": lb / us / 1e3, "frac": lb / us / 1e3 / peak}
    res["latency_ratio_oea_vs_vanilla"] = res["oea"]["us"] / res["vanilla"]["us"]
    res["unique_expert_ratio_oea_vs_vanilla"] = res["oea"]["T_mean"] / res["vanilla"]["T_mean"]
    res["config"] = {"D": D3, "H": H3, "N": N, "k": K_TOP, "B": B, "steps": K}
    for L in layers:
        L.close()
    return res


def c2_b16_extra(torch, stream, layers, W, K, peak):
    """C2 (BASELINE configs[1]) at B=16: k0 = 1..8 (k0 = 8 is top-8) on the C1
    layers: unique experts T vs µs per call, and the OLS line through them."""
    import numpy as np
    import paper_2511_02237_b200 as oea
    ctx = layers[0].ctx
    gen = torch.Generator(device="cuda").manual_seed(4321)
    xs = torch.randn(W + K, B, D, device="cuda", generator=gen).to(torch.bfloat16)
    out = torch.empty(B, D, device="cuda", dtype=torch.float32)
    pts = []
    for k0 in range(1, K_TOP + 1):
        cfg = oea.RoutingConfig.simplified(k0, K_TOP)
        us, _ = time_chain(torch, stream, layers, xs, cfg, out, W, K, ctx)
        Ts, _ = plan_stats(layers, xs, cfg, out, B, range(W, W + K), ctx)
        T = float(np.mean(Ts))
        lb = layer_bytes(T, D, H, N, B)
        pts.append({"k0": k0, "T_mean": T, "us": us, "frac": lb / us / 1e3 / peak})
    return {"B": B, "steps_per_point": K, "points": pts,
            "fit": fit_points([(p["T_mean"], p["us"]) for p in pts]),
            "slope_at_measured_hbm_us": 3 * D * H * 2 / peak / 1e3}


def c2_large_extra(torch, stream, layers, W, K, peak):
    """C2 (BASELINE configs[1]) large batches on the C1 layers: B = 32..256
    (B >= 32: route-only prologue + compaction + the tcgen05 (UMMA/TMEM)
    grouped FFN), OEA simplified(4, 8) and top-8: µs, T, fraction of the
    measured HBM peak for the active experts' bytes."""
    import numpy as np
    import paper_2511_02237_b200 as oea
    ctx = layers[0].ctx
    gen = torch.Generator(device="cuda").manual_seed(8765)
    pts = []
    for Bs in (32, 64, 128, 256):
        xs = torch.randn(W + K, Bs, D, device="cuda", generator=gen).to(torch.bfloat16)
        out = torch.empty(Bs, D, device="cuda", dtype=torch.float32)
        for name, cfg in (("oea", oea.RoutingConfig.simplified(K0, K_TOP)),
                          ("vanilla", oea.RoutingConfig.vanilla(K_TOP))):
            us, launched = time_chain(torch, stream, layers, xs, cfg, out, W, K, ctx)
            Ts, _ = plan_stats(layers, xs, cfg, out, Bs, range(W, W + K), ctx)
            T = float(np.mean(Ts))
            lb = layer_bytes(T, D, H, N, Bs)
            pts.append({"B": Bs, "routing": name, "us": us, "T_mean": T,
                        "frac": lb / us / 1e3 / peak, "kernels_per_call": launched / K,
                        "ffn": "tcgen05 (UMMA + TMEM)" if Bs >= 32 else "fused mma.sync"})
    return {"steps_per_point": K, "points": pts}


def c5_extra(torch, W, K):
    """C5 (BASELINE configs[4]): router-only B=4096 x N=128 fp64 route (the
    bit-exact route_f64 path on device-resident scores), k0 = 1..8."""
    import ctypes as C
    import paper_2511_02237_b200 as oea
    from paper_2511_02237_b200._capi import PlanViewC, default_context, lib
    from paper_2511_02237_b200.moe_layer import torch_stream
    ctx = default_context()
    Bc, Nc = 4096, 128
    gen = torch.Generator(device="cuda").manual_seed(5)
    scores = torch.softmax(torch.randn(Bc, Nc, device="cuda", dtype=torch.float64,
                                       generator=gen), dim=1)
    res = []
    for k0 in range(1, K_TOP + 1):
        cfg = oea.RoutingConfig.simplified(k0, K_TOP)
        stride = oea.plan_set_stride(cfg.resolved(Nc))
        sets = torch.empty(Bc, stride, dtype=torch.int32, device="cuda")
        set_len = torch.empty(Bc, dtype=torch.int32, device="cuda")
        w = torch.empty(Bc, stride, dtype=torch.float64, device="cuda")
        loads = torch.empty(Nc, dtype=torch.int32, device="cuda")
        au = torch.empty(Nc, dtype=torch.int32, device="cuda")
        cnt = torch.empty(1, dtype=torch.int32, device="cuda")
        tot = torch.empty(1, dtype=torch.int64, device="cuda")
        pv = PlanViewC(stride, sets.data_ptr(), set_len.data_ptr(), w.data_ptr(), None,
                       loads.data_ptr(), au.data_ptr(), cnt.data_ptr(), tot.data_ptr(),
                       None, None, None, None, None)
        c = cfg.to_c()

        def call():
            ctx.check(lib().oea_route_f64(ctx.h, C.c_void_p(scores.data_ptr()), None, Bc, Nc,
                                          C.byref(c), C.byref(pv), C.c_void_p(torch_stream())))
        for _ in range(W):
            call()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for _ in range(K):  # K route calls back to back in one graph
                call()
        graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        graph.replay()
        e1.record()
        e1.synchronize()
        us = e0.elapsed_time(e1) * 1000.0 / K
        del graph
        # algorithmic bytes: fp64 scores in; sets (int32), weights (fp64), set_len out
        byts = Bc * Nc * 8 + Bc * stride * 12 + Bc * 4
        res.append({"k0": k0, "us": us, "tokens_per_s": Bc / us * 1e6, "T": int(cnt.item()),
                    "GBps": byts / us / 1e3})
    return {"B": Bc, "N": Nc, "k": K_TOP, "steps": K, "sweep": res,
            "us_k0_4": res[3]["us"]}


def bench_c1(args, env):
    """The headline: C1 Qwen3-30B-A3B-shaped layer, B=16, OEA simplified(4, 8)
    vs vanilla top-8 (BASELINE.json configs[0]); one GPU."""
    import numpy as np
    torch, rank, world, local = env["torch"], env["rank"], env["world"], env["local"]
    import paper_2511_02237_b200 as oea

    W, K = max(3, args.warmup), max(1, args.steps)
    layers = []
    for r in range(ROTATE):
        L = oea.DeviceMoeLayer(D, H, N, "bf16")
        L.init_random(1 + r + 100 * rank)
        layers.append(L)
    ctx = layers[0].ctx
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    xs = torch.randn(W + K, B, D, device="cuda", generator=gen).to(torch.bfloat16)
    out = torch.empty(B, D, device="cuda", dtype=torch.float32)
    torch.cuda.synchronize()
    stream = torch.cuda.ExternalStream(ctx.stream)
    cfgs = {"oea": oea.RoutingConfig.simplified(K0, K_TOP), "vanilla": oea.RoutingConfig.vanilla(K_TOP)}
    peak, peak_src = load_peak()

    results = {}
    clocks = None
    launches = 0
    for name, cfg in cfgs.items():
        sampler = ClockSampler(local) if name == "oea" else None
        if sampler:
            sampler.__enter__()
        us, launched = time_chain(torch, stream, layers, xs, cfg, out, W, K, ctx)
        if sampler:
            sampler.__exit__()
            clocks = sampler.summary()
        if name == "oea":
            launches = launched
        Ts, loads = plan_stats(layers, xs, cfg, out, B, range(W, W + K), ctx)
        T = float(np.mean(Ts))
        lb = layer_bytes(T, D, H, N, B)
        results[name] = {"us": us, "T_mean": T, "T_min": int(min(Ts)), "T_max": int(max(Ts)),
                         "total_load_mean": float(np.mean(loads)), "active_bytes": lb,
                         "GBps": lb / us / 1e3, "frac": lb / us / 1e3 / peak,
                         "kernels_per_call": launched / K}

    # The previous methodology: one graph (one launch) per call, so each call
    # pays the graph-to-graph launch gap.
    cfg = cfgs["oea"]
    graphs = [layers[i % ROTATE].graph(xs[i], cfg, out) for i in range(W + K)]
    iso_us, _, _ = time_graphs(torch, stream, graphs, W, ctx=ctx)
    for g in graphs:
        g.close()

    # The two-kernel path (router cluster | FFN), for reference: per-stage times.
    stage = [layers[r].stage_graphs(xs[r], cfg, out) for r in range(ROTATE)]
    for i in range(W):
        stage[i % ROTATE][0].launch()
        stage[i % ROTATE][1].launch()
    ctx.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    with torch.cuda.stream(stream):
        for i in range(K):
            g_r, g_f = stage[i % ROTATE]
            ev[i][0].record(stream)
            g_r.launch()
            ev[i][1].record(stream)
            g_f.launch()
            ev[i][2].record(stream)
    torch.cuda.synchronize()
    two_kernel = {"router_us": statistics.mean(ev[i][0].elapsed_time(ev[i][1]) * 1000 for i in range(K)),
                  "ffn_us": statistics.mean(ev[i][1].elapsed_time(ev[i][2]) * 1000 for i in range(K)),
                  "used_for": "fallback only: layers with N > 128 and expert-parallel shards whose fused "
                              "prologue does not fit in shared memory (every N <= 128 config, p < 1 and "
                              "max_p < N included, takes the fused single launch); timed here for reference"}
    for gr, gf in stage:
        gr.close()
        gf.close()

    # Roofline of the dominant (and only) kernel of the layer call: the fused
    # single-launch decode k_ffn_bf16<2> (gate GEMV + routing + grouped SwiGLU
    # + combine). One call = one launch, so the event-timed step IS the
    # kernel's average launch duration (plus the ~1 µs PDL launch gap).
    o, v = results["oea"], results["vanilla"]
    traffic, traffic_ratio = load_traffic()
    roofline = {"bound": "hbm", "achieved": o["GBps"], "peak": peak, "unit": "GB/s",
                "frac": o["GBps"] / peak, "traffic": traffic,
                "traffic_over_algorithmic_in_capture": traffic_ratio,
                "kernel": "k_ffn_bf16<2> (fused layer)",
                "algorithmic_bytes_per_launch": o["active_bytes"], "kernel_us": o["us"],
                "bytes_formula": "T*3*D*H*2 + D*N*2 + B*D*2 + B*D*4",
                "peak_source": peak_src, "frac_of_8TBps_nominal": o["GBps"] / 8000.0,
                "vanilla_frac": v["GBps"] / peak}

    # ---- e2e through the C ABI from pinned host buffers ----
    # End to end through the C ABI, timed from C (lib/e2e_host,
    # tools/e2e_host.c: oea_moe_decode_host, no Python in the loop): every
    # step's tokens sit in pinned host memory (a distinct slice per step), the
    # decode reads that step's slice over the host link (the H2D transfer, in
    # the timed step) and writes out to a pinned buffer, and the call returns
    # when out is on the host. Also measured: the same with a CPU copy of the
    # tokens from pageable memory into one pinned staging buffer per step
    # (mode 0), and through the Python API (ctypes).
    import ctypes

    def e2e_run(mode):
        exe = os.path.join(ROOT, "paper_2511_02237_b200", "lib", "e2e_host")
        try:
            r = subprocess.run([exe, str(D), str(H), str(N), str(B), str(K0), str(max(K, 100)), str(W),
                                str(ROTATE), str(mode)], capture_output=True, text=True, timeout=300,
                               env=dict(os.environ, CUDA_VISIBLE_DEVICES=str(local)))
            return json.loads(r.stdout.strip().splitlines()[-1])
        except Exception as e:  # reported, the Python loop below still measures e2e
            return {"error": f"{type(e).__name__}: {e}"}
    e2e_c = e2e_run(3)
    e2e_c_staged = e2e_run(0)
    x_src = xs.cpu().contiguous()          # the steps' inputs, host memory
    x_stage = torch.empty(B, D, dtype=torch.bfloat16).pin_memory()
    out_host = torch.empty(B, D, dtype=torch.float32).pin_memory()
    xb, sp, op = B * D * 2, x_stage.data_ptr(), out_host.data_ptr()
    for i in range(W):
        ctypes.memmove(sp, x_src[i].data_ptr(), xb)
        layers[i % ROTATE].decode_host_ptr(sp, op, B, cfg)
    t0 = time.perf_counter()
    for i in range(W, W + K):
        ctypes.memmove(sp, x_src[i].data_ptr(), xb)
        layers[i % ROTATE].decode_host_ptr(sp, op, B, cfg)
    e2e_py = (time.perf_counter() - t0) * 1e6 / K
    e2e_us = e2e_c["us_per_step_mean"] if "us_per_step_mean" in e2e_c else e2e_py

    extras = {}
    if not args.no_extras:
        for key, fn in (("c2_b16", lambda: c2_b16_extra(torch, stream, layers, W, min(K, 20), peak)),
                        ("c2_large_b", lambda: c2_large_extra(torch, stream, layers, W, min(K, 20), peak)),
                        ("c3", lambda: c3_extra(torch, stream, W, min(K, 20), peak)),
                        ("c5", lambda: c5_extra(torch, W, 50))):
            try:
                extras[key] = fn()
            except Exception as e:  # an extra key never costs the headline line
                extras[key] = {"error": f"{type(e).__name__}: {e}"}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            vals, kind, cores, sample = cpu_reference_decode(1, 1, (3, K_TOP, K0, 1.0, K_TOP, 0, 0),
                                                             steps=5)
            cpu = {"value": statistics.median(vals), "unit": "us/layer-call", "cores": cores,
                   "kind": kind, "sample": sample + "; median of the samples",
                   "nproc": os.cpu_count(), "cpu_model": cpu_model()}
        except Exception as e:  # the CPU baseline is reported, never required
            cpu = {"value": None, "unit": "us/layer-call", "cores": 1, "kind": "port",
                   "sample": f"failed: {e}"}

    line = {
        "metric": METRIC, "value": o["us"], "unit": "us/layer-call", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": o["us"] / 1000.0, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: random bf16 weights with make_random_layer distributions "
                "(N(0,1/D), N(0,1/H)), N(0,1) bf16 tokens",
        "config": {"workload": "C1 Qwen3-30B-A3B-shaped MoE decode layer (BASELINE configs[0])",
                   "D": D, "H": H, "N": N, "k": K_TOP, "B": B,
                   "routing": f"simplified(k0={K0}, k={K_TOP}) vs vanilla top-{K_TOP}",
                   "parallelism": "single GPU",
                   "timing": f"{K} layer calls back to back in one CUDA graph (PDL edges), "
                             "CUDA events on the launching stream",
                   "l2": f"rotating {ROTATE} distinct layer copies ({ROTATE * 1.21:.1f} GB) and a "
                         "distinct token batch per step; each call streams >400 MB of expert "
                         "weights (> 126 MB L2)"},
        "oea": o, "vanilla": v,
        "latency_ratio_oea_vs_vanilla": o["us"] / v["us"],
        "unique_expert_ratio_oea_vs_vanilla": o["T_mean"] / v["T_mean"],
        "isolated_graph_us": iso_us,
        "two_kernel_path_us": two_kernel,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_us, "unit": "us/layer-call", "h2d_bytes_per_step": B * D * 2,
                "d2h_bytes_per_step": B * D * 4,
                "how": "C caller (lib/e2e_host mode 3) of oea_moe_decode_host: each step's "
                       "tokens in pinned host memory (a distinct slice per step), the fused "
                       "decode reads them over the host link (x_stage) and writes out to pinned "
                       "host memory, the call returns when out is on the host; mean over the steps",
                "c_harness": e2e_c,
                "with_pageable_staging_copy": e2e_c_staged,
                "python_api_us": e2e_py},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    line.update(extras)
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def _ep_time(env, step, W, K, capture=True):
    """Two eager steps (workspace sizing, NCCL communicators), then K steps
    captured as ONE CUDA graph (collectives included), replayed once as the
    warm-up and once between CUDA events; max over ranks. Without capture: W
    eager warm-up steps and K timed eager steps. Returns (µs per step, mode)."""
    torch = env["torch"]
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    graph, mode = None, "eager"
    if capture:
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                for _ in range(K):
                    step()
            mode = "cuda-graph"
        except Exception as e:  # pragma: no cover - eager fallback
            graph, mode = None, f"eager ({type(e).__name__})"
            torch.cuda.synchronize()

    def timed():
        if graph is not None:
            graph.replay()
        else:
            for _ in range(K):
                step()
    if graph is not None:
        graph.replay()
    else:
        for _ in range(W):
            step()
    torch.cuda.synchronize()
    _barrier(env)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    timed()
    e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) * 1000.0 / K
    del graph
    return _max_over_ranks(env, us), mode


def bench_ep(args, env):
    """N > 1 (torchrun): expert parallelism (BASELINE configs[3], SURVEY
    §8(e)). The C1 layer's experts are sharded in contiguous blocks over the
    N ranks (ep.ep_expert_range), tokens data-parallel (B/N rows per rank).
    `value` = µs per layer call (max over ranks) with NCCL all-to-all token
    dispatch and fp32 combine (ep.AllToAllExpertParallelMoE); the
    all-gather + reduce-scatter path and the peer-memory combine fused into
    the shard decode are reported next to it, with the C3 layer sharded the
    same way and the 94-layer C3-shaped stack."""
    import numpy as np
    torch, dist, rank, world, local = (env["torch"], env["dist"], env["rank"], env["world"],
                                       env["local"])
    import paper_2511_02237_b200 as oea
    from paper_2511_02237_b200 import ep
    W, K = max(3, args.warmup), max(1, min(args.steps, 40))
    if B % world:
        raise SystemExit(f"EP: B={B} must split over {world} ranks")
    peak, peak_src = load_peak()
    e0, e1 = ep.ep_expert_range(N, world, rank)
    t0, t1 = ep.ep_token_range(B, world, rank)
    rows = t1 - t0
    # the same seeds on every rank: shard r holds experts [e0, e1) of the same
    # full layer (the router is whole on every rank)
    shards = []
    for r in range(ROTATE):
        L = oea.DeviceMoeLayer(D, H, N, "bf16", experts=(e0, e1))
        L.init_random(1 + r)
        shards.append(L)
    ctx = shards[0].ctx
    gen = torch.Generator(device="cuda").manual_seed(1234)
    xs_full = torch.randn(W + K, B, D, device="cuda", generator=gen).to(torch.bfloat16)
    xs = xs_full[:, t0:t1].contiguous()
    out_local = torch.empty(rows, D, device="cuda", dtype=torch.float32)
    bufs = {"x_all": torch.empty(B, D, device="cuda", dtype=torch.bfloat16),
            "partial": torch.empty(B, D, device="cuda", dtype=torch.float32)}
    cfgs = {"oea": oea.RoutingConfig.simplified(K0, K_TOP), "vanilla": oea.RoutingConfig.vanilla(K_TOP)}

    def per_rank_T(layer, cfg, x_all):
        layer.decode(x_all, cfg, bufs["partial"])
        torch.cuda.synchronize()
        plan = layer.last_plan(B, cfg)
        act = [int(e) for e in plan["active_union"]]
        t_r = torch.tensor([sum(1 for e in act if e0 <= e < e1)], device="cuda")
        allt = [torch.zeros_like(t_r) for _ in range(world)]
        dist.all_gather(allt, t_r)
        return int(plan["active_count"]), [int(v.item()) for v in allt]

    res = {}
    clocks = None
    launches = 0
    for name, cfg in cfgs.items():
        mods = [ep.make_ep_layer("a2a", shards[r], cfg, world, rank, dist) for r in range(ROTATE)]
        recv = torch.empty(world, rows, D, device="cuda", dtype=torch.float32)
        it = [0]

        def step():
            i = it[0] % (W + K)
            it[0] += 1
            mods[i % ROTATE].forward(xs[i], out_local, recv=recv, **bufs)
        sampler = ClockSampler(local) if name == "oea" else None
        if sampler:
            sampler.__enter__()
        l0 = ctx.kernel_launches
        us, mode = _ep_time(env, step, W, K)
        if sampler:
            sampler.__exit__()
            clocks = sampler.summary()
        if name == "oea":
            launches = (ctx.kernel_launches - l0)
        Ts, Trs = [], []
        for i in range(W, W + min(K, 8)):
            T, tr = per_rank_T(shards[i % ROTATE], cfg, xs_full[i])
            Ts.append(T)
            Trs.append(tr)
        T = float(np.mean(Ts))
        maxTr = float(np.mean([max(v) for v in Trs]))
        lb_rank = maxTr * 3 * D * H * 2 + D * N * 2 + B * D * 2 + B * D * 4
        res[name] = {"us": us, "mode": mode, "T_mean": T, "max_rank_T_mean": maxTr,
                     "per_rank_T_first": Trs[0],
                     "GBps_busiest_rank": lb_rank / us / 1e3,
                     "frac_busiest_rank": lb_rank / us / 1e3 / peak}
    o = res["oea"]

    # the other data paths (OEA): all-gather + reduce-scatter, peer memory
    paths = {"a2a": {"us": o["us"]}}
    cfg = cfgs["oea"]
    try:
        mods = [ep.make_ep_layer("ag_rs", shards[r], cfg, world, rank, dist) for r in range(ROTATE)]
        it = [0]

        def step_ag():
            i = it[0] % (W + K)
            it[0] += 1
            mods[i % ROTATE].forward(xs[i], out_local, **bufs)
        paths["ag_rs"] = {"us": _ep_time(env, step_ag, W, K)[0]}
    except Exception as e:
        paths["ag_rs"] = {"error": f"{type(e).__name__}: {e}"}
    try:
        peers = [ep.PeerExpertParallelMoE(shards[r], cfg, world, rank, B) for r in range(ROTATE)]
        for pm in peers:
            pm.connect(dist)
        it = [0]

        def step_peer():
            i = it[0] % (W + K)
            it[0] += 1
            dist.all_gather_into_tensor(bufs["x_all"], xs[i])
            peers[i % ROTATE].forward(bufs["x_all"], out_local)
        paths["peer"] = {"us": _ep_time(env, step_peer, W, K)[0],
                         "note": "NCCL all-gather of the tokens, shard decode whose combine "
                                 "stores partials into the owners' memory (CUDA IPC), owner sum"}
        _barrier(env)
        torch.cuda.synchronize()
        for pm in peers:
            pm.close()
    except Exception as e:
        paths["peer"] = {"error": f"{type(e).__name__}: {e}"}

    extras = {}
    if not args.no_extras:
        try:
            extras["c3_sharded"] = _ep_c3(env, W, min(K, 20), peak)
        except Exception as e:
            extras["c3_sharded"] = {"error": f"{type(e).__name__}: {e}"}
        try:
            extras["c4_stack"] = _ep_c4(env, W, min(K, 5))
        except Exception as e:
            extras["c4_stack"] = {"error": f"{type(e).__name__}: {e}"}

    line = {"metric": METRIC, "value": o["us"], "unit": "us/layer-call", "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": o["us"] / 1000.0, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic: random bf16 weights with make_random_layer distributions, "
                    "N(0,1) bf16 tokens",
            "config": {"workload": "C1 Qwen3-30B-A3B-shaped MoE decode layer, expert parallel "
                                   "(BASELINE configs[0] layer, configs[3] parallelism)",
                       "D": D, "H": H, "N": N, "k": K_TOP, "B": B,
                       "routing": f"simplified(k0={K0}, k={K_TOP}) vs vanilla top-{K_TOP}",
                       "parallelism": f"ep{world}: experts [{N}r/{world}, {N}(r+1)/{world}) on "
                                      f"rank r, tokens {B // world} per rank; NCCL all-to-all "
                                      "dispatch + combine",
                       "timing": f"{K} layer calls in one CUDA graph per rank, CUDA events, "
                                 "max over ranks",
                       "l2": f"rotating {ROTATE} distinct layers and a distinct batch per step"},
            "oea": o, "vanilla": res["vanilla"],
            "latency_ratio_oea_vs_vanilla": o["us"] / res["vanilla"]["us"],
            "unique_expert_ratio_oea_vs_vanilla": o["T_mean"] / res["vanilla"]["T_mean"],
            "paths_oea_us": paths,
            "roofline": {"bound": "hbm", "achieved": o["GBps_busiest_rank"], "peak": peak,
                         "unit": "GB/s", "frac": o["frac_busiest_rank"], "traffic": None,
                         "kernel": "k_ffn_bf16<2> shard decode + NCCL all-to-all",
                         "note": "bytes of the busiest rank (max_r T_r experts) over the whole "
                                 "layer call incl. the collectives", "peak_source": peak_src},
            "cpu_baseline": None,
            "e2e": None,
            "gpu_launches": launches,
            "clocks": clocks}
    line.update(extras)
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def _ep_c3(env, W, K, peak):
    """The C3 layer (D=4096, H=1536) sharded over the ranks, a2a path."""
    import numpy as np
    torch, dist, rank, world = env["torch"], env["dist"], env["rank"], env["world"]
    import paper_2511_02237_b200 as oea
    from paper_2511_02237_b200 import ep
    D3, H3 = 4096, 1536
    e0, e1 = ep.ep_expert_range(N, world, rank)
    t0, t1 = ep.ep_token_range(B, world, rank)
    shards = []
    for r in range(2):
        L = oea.DeviceMoeLayer(D3, H3, N, "bf16", experts=(e0, e1))
        L.init_random(11 + r)
        shards.append(L)
    gen = torch.Generator(device="cuda").manual_seed(99)
    xs = torch.randn(W + K, B, D3, device="cuda", generator=gen).to(torch.bfloat16)[:, t0:t1].contiguous()
    out_local = torch.empty(t1 - t0, D3, device="cuda", dtype=torch.float32)
    bufs = {"x_all": torch.empty(B, D3, device="cuda", dtype=torch.bfloat16),
            "partial": torch.empty(B, D3, device="cuda", dtype=torch.float32)}
    recv = torch.empty(world, t1 - t0, D3, device="cuda", dtype=torch.float32)
    res = {}
    for name, cfg in (("oea", oea.RoutingConfig.simplified(K0, K_TOP)),
                      ("vanilla", oea.RoutingConfig.vanilla(K_TOP))):
        mods = [ep.make_ep_layer("a2a", shards[r], cfg, world, rank, dist) for r in range(2)]
        it = [0]

        def step():
            i = it[0] % (W + K)
            it[0] += 1
            mods[i % 2].forward(xs[i], out_local, recv=recv, **bufs)
        res[name] = {"us": _ep_time(env, step, W, K)[0]}
    res["latency_ratio_oea_vs_vanilla"] = res["oea"]["us"] / res["vanilla"]["us"]
    for L in shards:
        L.close()
    return res


def _ep_c4(env, W, K):
    """The 94-layer C3-shaped stack (BASELINE configs[3]), a2a path: per
    layer the fused residual + RMSNorm, the EP layer; one graph per step."""
    torch, dist, rank, world = env["torch"], env["dist"], env["rank"], env["world"]
    import paper_2511_02237_b200 as oea
    from paper_2511_02237_b200 import ep
    D4, H4, NL = 4096, 1536, 94
    e0, e1 = ep.ep_expert_range(N, world, rank)
    t0, t1 = ep.ep_token_range(B, world, rank)
    shard_bytes = (e1 - e0) * 3 * D4 * H4 * 2 + D4 * N * 2 * 2
    free, _ = torch.cuda.mem_get_info()
    R = int(max(1, min(16, (free * 0.70 - (4 << 30)) // shard_bytes)))
    t = torch.tensor([R], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    R = int(t.item())
    pool = []
    for l in range(R):
        L = oea.DeviceMoeLayer(D4, H4, N, "bf16", experts=(e0, e1))
        L.init_random(1000 + l)
        pool.append(L)
    gen = torch.Generator(device="cuda").manual_seed(7)
    x_full = torch.randn(B, D4, device="cuda", generator=gen).to(torch.bfloat16)
    h0 = x_full[t0:t1].float().contiguous()
    h_local = torch.empty_like(h0)
    out_local = torch.empty(t1 - t0, D4, device="cuda", dtype=torch.float32)
    bufs = {"x_all": torch.empty(B, D4, device="cuda", dtype=torch.bfloat16),
            "partial": torch.empty(B, D4, device="cuda", dtype=torch.float32),
            "recv": torch.empty(world, t1 - t0, D4, device="cuda", dtype=torch.float32)}
    res = {"layers": NL, "distinct_layers_resident": R, "experts_per_rank": e1 - e0}
    for name, cfg in (("oea", oea.RoutingConfig.simplified(K0, K_TOP)),
                      ("vanilla", oea.RoutingConfig.vanilla(K_TOP))):
        stack = [ep.make_ep_layer("a2a", pool[l % R], cfg, world, rank, dist) for l in range(NL)]

        def step():
            h_local.copy_(h0)
            ep.residual_stack_forward(stack, h_local, out_local, bufs=bufs)
        us, mode = _ep_time(env, step, 1, K)
        res[name] = {"us_per_step": us, "us_per_layer": us / NL, "mode": mode}
    res["latency_ratio_oea_vs_vanilla"] = res["oea"]["us_per_step"] / res["vanilla"]["us_per_step"]
    for L in pool:
        L.close()
    return res


def bench_c2(args, env):
    """C2: the C1 layer over B in {1..256} x k0 in {1..8} (k0 = 8 is top-8):
    per-step (T, µs) observations -> latency CSV (io.cpp schema), the OLS fit
    of µs on T (latency.cpp fit_linear) and an SVG of the curve."""
    import numpy as np
    from paper_2511_02237_b200 import latency as lat
    torch, rank = env["torch"], env["rank"]
    import paper_2511_02237_b200 as oea

    W, K = max(3, args.warmup), max(2, min(args.steps, 20))
    layers = []
    for r in range(ROTATE):
        L = oea.DeviceMoeLayer(D, H, N, "bf16")
        L.init_random(1 + r)
        layers.append(L)
    ctx = layers[0].ctx
    stream = torch.cuda.ExternalStream(ctx.stream)
    gen = torch.Generator(device="cuda").manual_seed(4321)
    obs, points = [], []
    for Bs in (1, 4, 8, 16, 32, 64, 128, 256):
        xs = torch.randn(W + K, Bs, D, device="cuda", generator=gen).to(torch.bfloat16)
        out = torch.empty(Bs, D, device="cuda", dtype=torch.float32)
        if Bs >= 32:  # eager first call: the tcgen05 FFN's weight copy (see time_chain)
            for L in layers:
                L.decode(xs[0], oea.RoutingConfig.simplified(1, K_TOP), out)
        for k0 in range(1, K_TOP + 1):
            cfg = oea.RoutingConfig.simplified(k0, K_TOP)
            graphs = [layers[i % ROTATE].graph(xs[i], cfg, out) for i in range(W + K)]
            _, steps, _ = time_graphs(torch, stream, graphs, W, per_step=True)
            for g in graphs:
                g.close()
            Ts, _ = plan_stats(layers, xs, cfg, out, Bs, range(W, W + K), ctx)
            for t, us in zip(Ts, steps):
                obs.append(lat.LatencyObservation(t, us))
            points.append({"B": Bs, "k0": k0, "T_mean": float(np.mean(Ts)),
                           "us_median": float(np.median(steps)),
                           "E_T_topk0": lat.expected_active_experts(N, k0, Bs)})
    fit = lat.fit_linear(obs)
    os.makedirs(args.out_dir, exist_ok=True)
    csv_path = os.path.join(args.out_dir, "c2_latency.csv")
    lat.write_latency_csv(csv_path, obs)
    with open(os.path.join(args.out_dir, "c2_latency.svg"), "w") as f:
        f.write(lat.latency_svg(obs, fit, "C1 layer (D=2048, H=768, N=128, k=8) on 1 B200: "
                                          "latency vs unique experts"))
    with open(os.path.join(args.out_dir, "c2_points.json"), "w") as f:
        json.dump(points, f, indent=1)
    per_expert_bytes = 3 * D * H * 2
    peak, _ = load_peak()
    line = {"metric": "C2 sweep: layer µs vs unique experts T (B x k0)", "config": {
                "workload": "C2 Qwen3-30B-A3B-shaped layer, B in {1..256} x k0 in {1..8}, k=8",
                "steps_per_point": K, "points": len(points)},
            "fit": {"slope_us_per_expert": fit.b_us, "intercept_us": fit.intercept_us,
                    "r_squared": fit.r_squared, "slope_stderr": fit.slope_stderr,
                    "observations": len(obs),
                    "slope_at_measured_hbm_us": per_expert_bytes / peak / 1e3},
            "csv": os.path.relpath(csv_path, ROOT), "points": points}
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def bench_c3(args, env):
    """C3: Qwen3-235B-A22B-shaped layer (N=128, k=8, D=4096, H=1536), B=16,
    OEA simplified(4, 8) vs top-8 on one B200."""
    import numpy as np
    torch, rank = env["torch"], env["rank"]
    import paper_2511_02237_b200 as oea
    D3, H3 = 4096, 1536
    W, K = max(3, args.warmup), max(1, min(args.steps, 20))
    layers = []
    for r in range(2):  # 2 x 4.83 GB; each call streams ~2-3 GB (>> 126 MB L2)
        L = oea.DeviceMoeLayer(D3, H3, N, "bf16")
        L.init_random(1 + r)
        layers.append(L)
    ctx = layers[0].ctx
    stream = torch.cuda.ExternalStream(ctx.stream)
    gen = torch.Generator(device="cuda").manual_seed(99)
    xs = torch.randn(W + K, B, D3, device="cuda", generator=gen).to(torch.bfloat16)
    out = torch.empty(B, D3, device="cuda", dtype=torch.float32)
    res = {}
    peak, _ = load_peak()
    for name, cfg in (("oea", oea.RoutingConfig.simplified(K0, K_TOP)),
                      ("vanilla", oea.RoutingConfig.vanilla(K_TOP))):
        graphs = [layers[i % 2].graph(xs[i], cfg, out) for i in range(W + K)]
        us, _, _ = time_graphs(torch, stream, graphs, W)
        for g in graphs:
            g.close()
        Ts, _ = plan_stats(layers, xs, cfg, out, B, range(W, W + K), ctx)
        T = float(np.mean(Ts))
        lb = layer_bytes(T, D3, H3, N, B)
        res[name] = {"us": us, "T_mean": T, "GBps": lb / us / 1e3, "frac": lb / us / 1e3 / peak}
    line = {"metric": "C3 MoE-layer decode µs at B=16 (Qwen3-235B-A22B shape)", "value": res["oea"]["us"],
            "unit": "us/layer-call", "higher_is_better": False, "config": {
                "workload": "C3 Qwen3-235B-A22B-shaped single MoE layer", "D": D3, "H": H3, "N": N,
                "k": K_TOP, "B": B, "routing": "simplified(4, 8) vs vanilla top-8"},
            "oea": res["oea"], "vanilla": res["vanilla"],
            "latency_ratio_oea_vs_vanilla": res["oea"]["us"] / res["vanilla"]["us"]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def bench_sweep(args, env):
    """the default 673-config OEA sweep (sweep.cpp:48-106) of
    Dirichlet(0.3) score batches (N=128, B=16, 8 steps x 4 layers) on the GPU
    simulator (cells generated once on the device, one batched route per
    config) vs the reference's sweep compiled in oracle/_ref (1 host thread,
    cell by cell, + its vanilla shadow routes); the points are compared."""
    import time
    import numpy as np
    torch, rank = env["torch"], env["rank"]
    from paper_2511_02237_b200 import scoregen as G, sim as S
    gen = G.ScoreGenConfig(G.GenKind.Dirichlet, n_experts=128, batch=16, steps=8, layers=4,
                           seed=3, alpha=0.3)
    lat = S.LatencyParams(0.05, 2.0)
    grid = S.default_sweep_grid(128, K_TOP)
    S.sweep(gen, grid[:4], lat)  # warm-up (contexts, workspaces)
    t0 = time.perf_counter()
    pts = S.sweep(gen, grid, lat)
    gpu_s = time.perf_counter() - t0
    line = {"metric": "default 673-config routing sweep, wall s (GPU simulator)", "value": gpu_s,
            "unit": "s", "higher_is_better": False,
            "config": {"workload": "sweep (SURVEY 8f-3)", "grid_points": len(grid), "N": 128,
                       "B": 16, "steps": 8, "layers": 4, "scores": "dirichlet(0.3), device-generated"},
            "routes": len(grid) * 32, "pareto_points": len(S.pareto_frontier(pts))}
    try:
        import oracle
        if rank == 0 and oracle.reference_available():
            t0 = time.perf_counter()
            want = oracle.Reference().sweep_default("dirichlet", 128, 16, 8, 4, 3, K_TOP, 0.05,
                                                    2.0, alpha=0.3)
            line["cpu_baseline"] = {"value": time.perf_counter() - t0, "unit": "s", "cores": 1,
                                    "kind": "reference",
                                    "sample": "the same sweep: sweep.cpp over simulate_decode, 1 thread"}
            line["points_identical"] = bool(np.array_equal(
                np.array([p.mean_active_experts for p in pts]), want))
    except Exception as e:  # the CPU baseline is reported, never required
        line["cpu_baseline"] = {"value": None, "sample": f"failed: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)


def bench_c5(args, env):
    """C5: router-only stress, B=4096 tokens x N=128, k=8, k0 in 1..8: the
    fp64 route_f64 path (K1) on device-resident scores (softmax of N(0,1)
    logits), per call µs and tokens/s."""
    import ctypes as C
    torch, rank = env["torch"], env["rank"]
    import paper_2511_02237_b200 as oea
    from paper_2511_02237_b200._capi import PlanViewC, lib, default_context
    ctx = default_context()
    Bc, Nc = 4096, 128
    gen = torch.Generator(device="cuda").manual_seed(5)
    scores = torch.softmax(torch.randn(Bc, Nc, device="cuda", dtype=torch.float64, generator=gen), dim=1)
    W, K = max(3, args.warmup), max(5, min(args.steps, 50))
    res = []
    for k0 in range(1, K_TOP + 1):
        cfg = oea.RoutingConfig.simplified(k0, K_TOP)
        stride = oea.plan_set_stride(cfg.resolved(Nc))
        sets = torch.empty(Bc, stride, dtype=torch.int32, device="cuda")
        set_len = torch.empty(Bc, dtype=torch.int32, device="cuda")
        w = torch.empty(Bc, stride, dtype=torch.float64, device="cuda")
        loads = torch.empty(Nc, dtype=torch.int32, device="cuda")
        au = torch.empty(Nc, dtype=torch.int32, device="cuda")
        cnt = torch.empty(1, dtype=torch.int32, device="cuda")
        tot = torch.empty(1, dtype=torch.int64, device="cuda")
        pv = PlanViewC(stride, sets.data_ptr(), set_len.data_ptr(), w.data_ptr(), None,
                       loads.data_ptr(), au.data_ptr(), cnt.data_ptr(), tot.data_ptr(),
                       None, None, None, None, None)
        c = cfg.to_c()

        from paper_2511_02237_b200.moe_layer import torch_stream

        def call():
            ctx.check(lib().oea_route_f64(ctx.h, C.c_void_p(scores.data_ptr()), None, Bc, Nc,
                                          C.byref(c), C.byref(pv), C.c_void_p(torch_stream())))
        for _ in range(W):
            call()
        torch.cuda.synchronize()
        # one route call (memsets + kernels) captured in a CUDA graph: the GPU
        # time per call, not the host's launch overhead
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            call()
        for _ in range(W):
            graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(K):
            graph.replay()
        e1.record()
        e1.synchronize()
        us = e0.elapsed_time(e1) * 1000.0 / K
        del graph
        res.append({"k0": k0, "us": us, "tokens_per_s": Bc / us * 1e6, "T": int(cnt.item())})
    # Score-trace routing: 256 (step, layer) records of 16
    # tokens, host buffers, one batched call (oea_route_f64_batched_host) vs
    # the reference's record-by-record loop through the single-batch API.
    import numpy as np
    import time
    rng = np.random.default_rng(9)
    recs = [oea.ScoreMatrix(rng.dirichlet(np.full(Nc, 0.3), size=16)) for _ in range(256)]
    cfg = oea.RoutingConfig.simplified(4, K_TOP)
    oea.route_batched(recs, cfg)
    t0 = time.perf_counter()
    for _ in range(5):
        oea.route_batched(recs, cfg)
    batched_ms = (time.perf_counter() - t0) * 1e3 / 5
    t0 = time.perf_counter()
    for r in recs:
        oea.route(r, cfg)
    loop_ms = (time.perf_counter() - t0) * 1e3
    trace = {"records": len(recs), "tokens_per_record": 16, "routing": "simplified(4, 8)",
             "batched_ms": batched_ms, "per_record_loop_ms": loop_ms,
             "records_per_s_batched": len(recs) / batched_ms * 1e3,
             "note": "host buffers, wall clock incl. H2D/D2H and plan unpacking"}
    line = {"metric": "C5 router-only µs per B=4096 route (fp64 route_f64, bit-exact path, CUDA-graph replay)",
            "value": res[3]["us"], "unit": "us/route-call", "higher_is_better": False,
            "config": {"workload": "C5 router stress", "B": Bc, "N": Nc, "k": K_TOP,
                       "scores": "softmax of N(0,1) fp64 logits, device-resident"},
            "sweep": res, "trace_routing": trace}
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def bench_c4(args, env):
    """C4: Qwen3-235B-A22B-shaped MoE stack (94 layers of N=128, k=8, D=4096,
    H=1536), B=16 decode, expert parallel over the torchrun ranks (P = world
    size): per layer RMSNorm of the fp32 residual stream, all-gather of the
    tokens -> fused shard decode -> NCCL reduce-scatter of the partial
    mixtures -> residual add (ep.residual_stack_forward; attention omitted). A
    decode step (94 layers) is captured in one CUDA graph. When 94 distinct
    shard layers do not fit one GPU's HBM the stack cycles through a pool of
    R distinct layers (stated in the line)."""
    import numpy as np
    torch, dist, rank, world = env["torch"], env["dist"], env["rank"], env["world"]
    import paper_2511_02237_b200 as oea
    from paper_2511_02237_b200 import ep
    D4, H4, NL = 4096, 1536, 94
    if B % world:
        raise SystemExit(f"C4: B={B} must split over {world} ranks")
    e0, e1 = ep.ep_expert_range(N, world, rank)
    shard_bytes = (e1 - e0) * 3 * D4 * H4 * 2 + D4 * N * 2 * 2
    free, _ = torch.cuda.mem_get_info()
    R = int(max(1, min(NL, (free * 0.80 - (4 << 30)) // shard_bytes)))
    if dist is not None:  # the same pool size on every rank
        t = torch.tensor([R], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        R = int(t.item())
    pool = []
    for l in range(R):
        L = oea.DeviceMoeLayer(D4, H4, N, "bf16", experts=(e0, e1))
        L.init_random(1000 + l)
        pool.append(L)
    torch.cuda.synchronize()
    t0, t1 = ep.ep_token_range(B, world, rank)
    gen = torch.Generator(device="cuda").manual_seed(7)
    x_full = torch.randn(B, D4, device="cuda", generator=gen).to(torch.bfloat16)
    h0 = x_full[t0:t1].float().contiguous()   # residual stream (fp32)
    h_local = torch.empty_like(h0)
    out_local = torch.empty(t1 - t0, D4, device="cuda", dtype=torch.float32)
    bufs = {"x_all": torch.empty(B, D4, device="cuda", dtype=torch.bfloat16),
            "partial": torch.empty(B, D4, device="cuda", dtype=torch.float32)}
    W, K = max(3, args.warmup), max(1, min(args.steps, 10))
    res = {}
    for name, cfg in (("oea", oea.RoutingConfig.simplified(K0, K_TOP)),
                      ("vanilla", oea.RoutingConfig.vanilla(K_TOP))):
        stack = [ep.ExpertParallelMoE.from_shard(pool[l % R], cfg, world, rank, dist)
                 for l in range(NL)]

        def step():
            h_local.copy_(h0)
            return ep.residual_stack_forward(stack, h_local, out_local, bufs=bufs)
        for _ in range(2):  # eager warm-up (workspace sizing, NCCL comms)
            step()
        torch.cuda.synchronize()
        graph = None
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                step()
            run = graph.replay
            mode = "cuda-graph"
        except Exception as e:  # pragma: no cover - eager fallback
            graph = None
            run = step
            mode = f"eager ({type(e).__name__})"
        for _ in range(W):
            run()
        torch.cuda.synchronize()
        _barrier(env)
        e_0, e_1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_0.record()
        for _ in range(K):
            run()
        e_1.record()
        e_1.synchronize()
        us_step = e_0.elapsed_time(e_1) * 1000.0 / K
        us_step = _max_over_ranks(env, us_step)
        # per-rank held active experts T_r of the first layer's plan (eager)
        stack[0].forward(x_full[t0:t1].contiguous(), out_local, **bufs)
        torch.cuda.synchronize()
        plan = pool[0].last_plan(B, cfg)
        act = [int(e) for e in plan["active_union"]]
        T_r = sum(1 for e in act if e0 <= e < e1)
        tr = torch.tensor([T_r], device="cuda", dtype=torch.float64)
        if dist is not None:
            dist.all_reduce(tr, op=dist.ReduceOp.MAX)
        res[name] = {"us_per_step": us_step, "us_per_layer": us_step / NL, "mode": mode,
                     "T_layer0": int(plan["active_count"]), "max_rank_T_layer0": int(tr.item())}
        del graph
    line = {"metric": "C4 MoE-stack decode: µs per 94-layer step (expert parallel, B=16)",
            "value": res["oea"]["us_per_step"], "unit": "us/decode-step", "n_gpus": world,
            "higher_is_better": False, "scaling": "strong", "dtype": "bf16",
            "data": "synthetic: make_random_layer-distributed bf16 weights, N(0,1) tokens",
            "config": {"workload": "C4 Qwen3-235B-A22B-shaped 94-layer MoE stack", "D": D4,
                       "H": H4, "N": N, "k": K_TOP, "B": B, "layers": NL,
                       "distinct_layers_resident": R, "experts_per_rank": e1 - e0,
                       "parallelism": f"ep{world} (NCCL all-gather + reduce-scatter)",
                       "routing": "simplified(4, 8) vs vanilla top-8"},
            "oea": res["oea"], "vanilla": res["vanilla"],
            "latency_ratio_oea_vs_vanilla": res["oea"]["us_per_step"] / res["vanilla"]["us_per_step"]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
