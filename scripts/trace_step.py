"""Trace a few SVT iterations with torch.profiler (CUPTI): kernel activity of
libsvt_b200 plus the CUDA runtime calls of the host thread, then report the
device-idle gaps and the host calls that overlap them.  Development tool."""
import argparse
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05528_b200 import api as G  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from explore import load  # noqa: E402


def union(iv):
    iv = sorted(iv)
    out = []
    for a, b in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def inter_len(A, B):
    i = j = 0
    t = 0.0
    while i < len(A) and j < len(B):
        lo, hi = max(A[i][0], B[j][0]), min(A[i][1], B[j][1])
        if hi > lo:
            t += hi - lo
        if A[i][1] < B[j][1]:
            i += 1
        else:
            j += 1
    return t

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--warm", type=int, default=5)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--out", default="gpurun_out/trace.json")
args = ap.parse_args()

ctx = G.default_context()
A, test, cfg, stop, _ = load(args.config, 1)
S = G.Solver(A, cfg, stop, test=test)
for _ in range(args.warm):
    S.step()
ctx.sync()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(args.iters):
        S.step()
    ctx.sync()
prof.export_chrome_trace(args.out)
ev = json.load(open(args.out))["traceEvents"]
kern = sorted([(e["ts"], e["ts"] + e.get("dur", 0), e["name"]) for e in ev
               if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda x: x[0])
rt = sorted([(e["ts"], e["ts"] + e.get("dur", 0), e["name"]) for e in ev if e.get("cat") == "cuda_runtime"],
            key=lambda x: x[0])
busy = sum(b - a for a, b, _ in kern)
by_stream = {}
for e in ev:
    if e.get("cat") == "kernel":
        by_stream.setdefault(e.get("args", {}).get("stream"), []).append((e["ts"], e["ts"] + e.get("dur", 0)))
streams = {k: union(v) for k, v in by_stream.items()}
for k, v in streams.items():
    print(f"stream {k}: {len(by_stream[k])} kernels, busy {sum(b - a for a, b in v)/1e3:.1f} ms")
ks = list(streams)
if len(ks) >= 2:
    print(f"overlap of streams {ks[0]} and {ks[1]}: {inter_len(streams[ks[0]], streams[ks[1]])/1e3:.1f} ms")
allu = union([iv for v in streams.values() for iv in v])
print(f"device busy (union): {sum(b - a for a, b in allu)/1e3:.1f} ms")
span = kern[-1][1] - kern[0][0]
print(f"kernels {len(kern)}  device busy {busy/1e3:.1f} ms of span {span/1e3:.1f} ms  runtime calls {len(rt)}")
gaps = []
for (a0, a1, an), (b0, b1, bn) in zip(kern, kern[1:]):
    if b0 - a1 > 200:
        gaps.append((b0 - a1, a1, b0, an, bn))
gaps.sort(reverse=True)
tot = sum(g[0] for g in gaps)
print(f"idle gaps > 200 us: {len(gaps)}, total {tot/1e3:.1f} ms")
from collections import Counter
for g, a1, b0, an, bn in gaps[:25]:
    calls = Counter()
    for r0, r1, rn in rt:
        ov = min(r1, b0) - max(r0, a1)
        if ov > 0:
            calls[rn] += ov
    top = ", ".join(f"{k} {v/1e3:.2f}ms" for k, v in calls.most_common(4))
    print(f"  gap {g/1e3:8.2f} ms after {an[:40]:40s} before {bn[:40]:40s} | host: {top}")
# host-side totals per runtime call
tot_rt = Counter()
for r0, r1, rn in rt:
    tot_rt[rn] += r1 - r0
print("runtime call totals:", ", ".join(f"{k} {v/1e3:.1f}ms" for k, v in tot_rt.most_common(10)))
# per-stream kernel time by name, and how the streams share the span
byname = {}
for e in ev:
    if e.get("cat") == "kernel":
        s = e.get("args", {}).get("stream")
        nm = e["name"].replace("void ", "").replace("svtb::(anonymous namespace)::", "").split("(")[0][:48]
        d = byname.setdefault(s, {})
        d[nm] = d.get(nm, 0.0) + e.get("dur", 0)
for s, d in byname.items():
    top = sorted(d.items(), key=lambda kv: -kv[1])[:12]
    print(f"stream {s} top kernels: " + ", ".join(f"{k} {v/1e3:.1f}" for k, v in top))
if len(ks) >= 2:
    # the library's streams in creation order: main, side, then the helper
    # streams of main and side (dense-corner products); group each helper
    # with its parent by the kernels it runs first
    order = sorted(ks, key=lambda k: int(k) if str(k).isdigit() else 0)
    main_ids = [order[0]] + ([order[2]] if len(order) > 2 else [])
    side_ids = [order[1]] + ([order[3]] if len(order) > 3 else [])
    a = union([iv for k in main_ids for iv in by_stream[k]])
    b = union([iv for k in side_ids for iv in by_stream[k]])
    ov = inter_len(a, b)
    ta, tb = sum(y - x for x, y in a), sum(y - x for x, y in b)
    print(f"span {span/1e3:.1f} ms: main-side busy {ta/1e3:.1f} / {tb/1e3:.1f}; only main {(ta-ov)/1e3:.1f}, "
          f"only side {(tb-ov)/1e3:.1f}, both {ov/1e3:.1f}, idle {(span - (ta + tb - ov))/1e3:.1f} "
          f"(streams main {main_ids}, side {side_ids})")
