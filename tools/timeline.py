"""Per-CTA stamp timeline of the fused decode launch (OEA_FFN_TRACE=1), for the
last of REPS back-to-back graph replays, plus the event-timed µs per call, so
the launch gap = per-call time - (last CTA done - first CTA start).

  SHAPE=2048,768,128,16 K0=4 python tools/timeline.py
"""
import os
import sys

os.environ["OEA_FFN_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_02237_b200 as oea  # noqa: E402
from paper_2511_02237_b200._capi import lib  # noqa: E402

D, H, N, B = [int(v) for v in os.environ.get("SHAPE", "2048,768,128,16").split(",")]
K0 = int(os.environ.get("K0", "4"))
REPS = int(os.environ.get("REPS", "20"))
layers = []
for r in range(4):
    L = oea.DeviceMoeLayer(D, H, N, "bf16")
    L.init_random(1 + r)
    layers.append(L)
ctx = layers[0].ctx
torch.manual_seed(int(os.environ.get("SEED", "5")))
xs = torch.randn(REPS, B, D, device="cuda").to(torch.bfloat16)
out = torch.empty(B, D, device="cuda", dtype=torch.float32)
torch.cuda.synchronize()
stream = torch.cuda.ExternalStream(ctx.stream)

SLOTS = [(0, "start"), (5, "logits published"), (8, "slot8 (dense: logits polled)"), (11, "R1 ranked"), (12, "logits polled (local) / union words polled"),
         (13, "union ballots"), (14, "union syncthreads"), (6, "union known"), (7, "plan ready"),
         (1, "first W2 round"), (4, "producer done"), (3, "consumers done"), (9, "combine arrive"),
         (10, "combine barrier"), (2, "combine start"), (15, "combine done")]

for name, cfg in (("oea", oea.RoutingConfig.simplified(K0, 8)), ("vanilla", oea.RoutingConfig.vanilla(8))):
    for L in layers:  # eager first call (a tcgen05 path's weight copy is made outside capture)
        L.decode(xs[0], cfg, out)
    chain = os.environ.get("CHAIN", "0") == "1"
    if chain:  # one graph of REPS - 4 calls (PDL edges) + a 4-call warm-up graph
        warm = oea.DeviceMoeLayer.chain_graph([layers[i % 4] for i in range(4)], list(xs[:4]),
                                              cfg, [out] * 4)
        graphs = [warm, oea.DeviceMoeLayer.chain_graph(
            [layers[i % 4] for i in range(4, REPS)], list(xs[4:]), cfg, [out] * (REPS - 4))]
        runs = graphs[1:]
    else:
        graphs = [layers[i % 4].graph(xs[i], cfg, out) for i in range(REPS)]
        runs = graphs[4:]
    for g in graphs[:len(graphs) - len(runs)]:
        g.launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for g in runs:
            g.launch()
        e1.record(stream)
    e1.synchronize()
    per_call = e0.elapsed_time(e1) * 1000.0 / (REPS - 4)
    LEG, NL, PER, INFO = 8192, 16, 16384, 2400
    RLOG, NR = 4096, 24
    buf = np.zeros(LEG + NL * PER, np.uint64)
    ctx.check(lib().oea_debug_ffn_trace(ctx.h, buf.ctypes.data_as(C.c_void_p), buf.size))
    regs = buf[LEG:].reshape(NL, PER).astype(np.int64)
    launches = []
    for r in regs:
        t = r[:148 * 16].reshape(148, 16)
        if t[:, 0].min() <= 0 or t[:, 15].max() <= 0:
            continue
        launches.append((t[:, 0].min(), t, int(r[INFO]), r))
        if r[INFO + 1]:
            print(f"    CTA0: poll {int(r[INFO + 1])} cyc in {int(r[INFO + 2])} passes, "
                  f"select {int(r[INFO + 3])} cyc (load+sort {int(r[INFO + 4])}, merge {int(r[INFO + 5])})")
    launches.sort(key=lambda v: v[0])
    print(f"== {name} B={B} D={D} H={H} N={N}: {per_call:.2f} us per call (events), "
          f"{len(launches)} launches traced")
    if os.environ.get("PERCTA"):  # per-CTA medians over the launches of a few prologue slots
        sl = [0, 8, 5, 11, 12, 6]
        per = np.median(np.stack([np.stack([(t[:, s] - t0) / 1000.0 for s in sl], 1)
                                  for t0, t, _, _ in launches]), 0)
        print("    per CTA (median us):", " ".join(f"s{s}" for s in sl))
        r1 = np.median(np.stack([(r[2368:2400].reshape(16, 2) - t0) / 1000.0
                                 for t0, _, _, r in launches]), 0)
        print("    R1 CTAs 0..15: own logit word polled / all polled (median us):",
              " ".join(f"{a:.2f}/{b:.2f}" for a, b in r1))
        worst = np.argsort(-per[:, 3])[:6]
        for c in list(range(0, 20)) + [int(w) for w in worst]:
            print(f"    CTA {c:3d}: " + " ".join(f"{v:6.2f}" for v in per[c]))
    # median over the traced launches of each slot's (min, med, max) over CTAs
    rows = {s: [] for s, _ in SLOTS}
    spans, gaps, Ts = [], [], []
    for i, (t0, t, T, _) in enumerate(launches):
        for s, _ in SLOTS:
            a = t[:, s]
            a = a[a > 0]
            if a.size:
                r = (a - t0) / 1000.0
                rows[s].append((r.min(), np.median(r), r.max()))
        spans.append((t[:, 15].max() - t0) / 1000.0)
        Ts.append(T)
        if i + 1 < len(launches):
            gaps.append((launches[i + 1][0] - t[:, 15].max()) / 1000.0)
    for s, lab in SLOTS:
        if rows[s]:
            m = np.median(np.array(rows[s]), axis=0)
            print(f"  {lab:20s} min {m[0]:7.2f} med {m[1]:7.2f} max {m[2]:7.2f}")
    print(f"  T per launch {Ts}")
    print(f"  span (first start -> last combine done) median {np.median(spans):.2f} us "
          f"[{min(spans):.2f}, {max(spans):.2f}]")
    if gaps:
        print(f"  gap (last combine done -> next first start) median {np.median(gaps):.2f} us "
              f"[{min(gaps):.2f}, {max(gaps):.2f}]")
    if os.environ.get("ROUNDS") == "1" and launches:
        # producer round log of the median-span launch: per-kind round times and
        # the aggregate weight stream rate per 2 us bin
        order = np.argsort(spans)
        li = int(order[len(order) // 2])
        t0, t, T = launches[li]
        reg = [r for r in regs if r[:148 * 16].reshape(148, 16)[:, 0].min() == t0][0]
        rl = reg[RLOG:RLOG + 148 * NR * 3].reshape(148, NR, 3)
        KT1, KT2 = (D + 15) // 16 // 8, (H + 15) // 16 // 8
        rows = []
        for c in range(148):
            ends = list(rl[c, 1:, 0]) + [0]
            for j in range(NR):
                st, desc, hr = rl[c, j]
                if st <= 0:
                    break
                kind, n = int(desc) >> 56, (int(desc) >> 48) & 0xff
                if n == 0:
                    break
                en = ends[j] if ends[j] > 0 else t[c, 4]
                nst = KT1 if kind == 1 else KT2
                rows.append((c, kind, (st - t0) / 1e3, (en - t0) / 1e3, n * 4096 * nst,
                             (hr - t0) / 1e3 if hr > 0 else None))
        for kind in (1, 2):
            d = [r[3] - r[2] for r in rows if r[1] == kind]
            if d:
                print(f"  kind {kind}: {len(d)} rounds, dur med {np.median(d):.2f} min {min(d):.2f} max {max(d):.2f} us")
        w2w = [r[5] - r[2] for r in rows if r[1] == 2 and r[5] is not None]
        if w2w:
            print(f"  W2 h-wait (ready - round start): med {np.median(w2w):.2f} max {max(w2w):.2f} us, >0.5us: {sum(1 for v in w2w if v > 0.5)}")
        end = max(r[3] for r in rows)
        bins = np.zeros(int(end // 2) + 2)
        act = np.zeros_like(bins)
        for r in rows:
            a, b, by = r[2], r[3], r[4]
            rate = by / max(b - a, 1e-3)  # bytes per us
            for k in range(int(a // 2), int(b // 2) + 1):
                lo, hi = max(a, 2 * k), min(b, 2 * k + 2)
                if hi > lo:
                    bins[k] += rate * (hi - lo) / 2.0
                    act[k] += (hi - lo) / 2.0
        print("  stream TB/s per 2us bin: " + " ".join(f"{v / 1e6:.1f}" for v in bins))
        print("  active SMs per 2us bin:  " + " ".join(f"{v:.0f}" for v in act))
    for (t0, t, T), sp in zip(launches, spans):
        pd = (t[:, 4] - t0) / 1000.0
        print(f"    T={T:3d} span {sp:6.2f}  union {(t[:, 6].max() - t0) / 1000.0:5.2f}  "
              f"producers done {pd.min():6.2f}..{pd.max():6.2f}  "
              f"us/expert {(sp) / max(T, 1):.3f}")
    for g in graphs:
        g.close()
