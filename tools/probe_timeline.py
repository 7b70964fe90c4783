"""Per-CTA timeline of one DIPR layer call (diagnostic): prep / scan / attend /
combine CTA start and end stamps (%globaltimer, alaya_debug_trace) for B
sessions of a 128K-token Llama-3.1-8B-shaped layer, steady state (the second of
two back-to-back calls). Prints one JSON line per batch size, times in us from
the first prep CTA start.

  python tools/probe_timeline.py --batches 1,4 [--chunk 0] [--out file.jsonl]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_10326_b200 import _lib, engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batches", default="1,4")
ap.add_argument("--ctx", type=int, default=131072)
ap.add_argument("--hq", type=int, default=32)
ap.add_argument("--chunk", type=int, default=0)
ap.add_argument("--beta", type=float, default=110.0)
ap.add_argument("--label", default="base")
ap.add_argument("--out", default=None)
ap.add_argument("--isolated", action="store_true", help="trace one call on an idle GPU")
ap.add_argument("--scan-only", action="store_true", help="prep + scan only (alaya_scan, no attend)")
a = ap.parse_args()
dev = torch.device("cuda")
lib = _lib.load()
KINDS = ("prep", "scan", "attend", "combine")
NCTA, NSLOT = 1024, 16


def pct(xs, p):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(p * (len(xs) - 1) + 0.5))] if xs else None


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for B in [int(x) for x in a.batches.split(",")]:
    hkv, d = 8, 128
    g = torch.Generator(device=dev).manual_seed(B)
    c = torch.randn(16, d, generator=g, device=dev)
    centers = c / c.norm(dim=1, keepdim=True) * math.sqrt(d)
    K = torch.empty(B, hkv, a.ctx, d, dtype=torch.bfloat16, device=dev)
    V = torch.empty_like(K)
    for b in range(B):
        a_ = torch.randint(0, 16, (hkv, a.ctx), generator=g, device=dev)
        K[b] = (centers[a_] + 0.25 * torch.randn(hkv, a.ctx, d, generator=g, device=dev)).to(K.dtype)
        V[b] = torch.randn(hkv, a.ctx, d, generator=g, device=dev).to(K.dtype)
    params = engine.make_params(a.hq, hkv, d, K.dtype, a.beta, 16, 64, a.chunk, 0)
    call = engine.Call([engine.SeqView(k=K[b], v=V[b], n=a.ctx) for b in range(B)], params, K.dtype, dev)
    pick = torch.randint(0, 16, (B, a.hq), generator=g, device=dev)
    q = (centers[pick] + 0.25 * torch.randn(B, a.hq, d, generator=g, device=dev)).float()
    out = torch.empty_like(q)
    fn = (lambda: call.scan_only(q)) if a.scan_only else (lambda: call.dipr_attention(q, out=out))
    t_call = timed(fn)
    buf = torch.zeros(4 * NCTA * NSLOT, dtype=torch.int64, device=dev)
    _lib.check(lib.alaya_debug_trace(ctypes.c_void_p(buf.data_ptr()), buf.numel() * 8))
    try:
        fn()
        if a.isolated:
            torch.cuda.synchronize()
            buf.zero_()
        fn()
        torch.cuda.synchronize()
    finally:
        _lib.check(lib.alaya_debug_trace(None, 0))
    tr = buf.view(4, NCTA, NSLOT).cpu().tolist()
    stamps = [x for ki, k in enumerate(tr) for cta in k for si, x in enumerate(cta)
              if x > 0 and not (ki == 2 and si in (4, 5)) and not (ki == 1 and si >= 10)]  # sums
    t0 = min(stamps)
    us = lambda x: round((x - t0) / 1e3, 2)  # noqa: E731
    line = {"label": a.label + ("/isolated" if a.isolated else "") + ("/scan" if a.scan_only else ""), "B": B, "ctx": a.ctx, "chunk": a.chunk, "us_call_timed": round(t_call, 1)}
    for ki, name in enumerate(KINDS):
        ctas = [cta for cta in tr[ki] if cta[0] > 0]
        if not ctas:
            continue
        starts = [us(x[0]) for x in ctas]
        ends = [us(x[1]) for x in ctas if x[1] > 0]
        line[name] = {"ctas": len(ctas), "start_min": min(starts), "start_max": max(starts),
                      "end_p10": pct(ends, 0.1), "end_p50": pct(ends, 0.5), "end_p90": pct(ends, 0.9),
                      "end_max": max(ends) if ends else None}
        if name == "scan":  # chunk-completion times of each round (slot 2 + round)
            for si, key in ((13, "producer_wait_ring"), (14, "epi_publish"), (15, "publisher")):
                v = [x[si] / 1e3 for x in ctas]
                line[name][key + "_us_mean"] = round(sum(v) / len(v), 2)
            rounds = []
            line[name]["end_hist_us"] = [sum(1 for x in ends if lo <= x < lo + 5) for lo in range(0, 400, 5)]
            for r in range(8):
                e = [us(x[2 + r]) for x in ctas if x[2 + r] > 0]
                if not e:
                    break
                rounds.append({"n": len(e), "min": min(e), "p50": pct(e, 0.5), "max": max(e)})
            line[name]["chunk_rounds"] = rounds
        if name == "attend":
            line[name]["pair_ready_max"] = max(us(x[2]) for x in ctas if x[2] > 0) if any(x[2] > 0 for x in ctas) else None
            line[name]["task_end_p50"] = pct([us(x[3]) for x in ctas if x[3] > 0], 0.5)
            line[name]["task_us_max"] = round(max(x[4] for x in ctas) / 1e3, 2)
            line[name]["tasks"] = sum(x[5] for x in ctas)
        if name in ("prep", "combine"):
            w = [us(x[2]) for x in ctas if x[2] > 0]
            line[name]["after_wait_p50"] = pct(w, 0.5)
    print(json.dumps(line), flush=True)
    if a.out:
        with open(a.out, "a") as fh:
            fh.write(json.dumps(line) + "\n")
    del K, V, call
    torch.cuda.empty_cache()
