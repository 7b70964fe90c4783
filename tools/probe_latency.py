"""Per-layer-call latency of the decode step vs batch size (diagnostic).

For B sessions of a 128K-token Llama-3.1-8B-shaped layer (32 q / 8 kv heads,
bf16, reference-generator distribution): CUDA-event mean of the full
``alaya_dipr_attention`` call and of the scan stage alone. Knobs come from
the environment (ALAYA_TC_*), so a sweep runs one process per variant:

  python tools/probe_latency.py --label base --batches 1,2,4,8 --chunk 0
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_10326_b200 import engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--label", default="base")
ap.add_argument("--batches", default="1,2,4,8")
ap.add_argument("--ctx", type=int, default=131072)
ap.add_argument("--hq", type=int, default=32)
ap.add_argument("--chunk", type=int, default=0)
ap.add_argument("--beta", type=float, default=110.0)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--locality", action="store_true")
ap.add_argument("--fp32", action="store_true", help="fp32 K/V (CUDA-core scan)")
ap.add_argument("--block-filter", action="store_true", help="coarse block filter before the scan")
ap.add_argument("--out", default=None)
a = ap.parse_args()
dev = torch.device("cuda")


def make(B, hkv, n, d, seed):
    g = torch.Generator(device=dev).manual_seed(seed)
    c = torch.randn(16, d, generator=g, device=dev)
    centers = c / c.norm(dim=1, keepdim=True) * math.sqrt(d)
    dt = torch.float32 if a.fp32 else torch.bfloat16
    K = torch.empty(B, hkv, n, d, dtype=dt, device=dev)
    V = torch.empty_like(K)
    for b in range(B):
        a_ = torch.randint(0, 16, (hkv, n), generator=g, device=dev)
        if a.locality:
            a_ = torch.sort(a_, dim=1).values
        K[b] = (centers[a_] + 0.25 * torch.randn(hkv, n, d, generator=g, device=dev)).to(dt)
        V[b] = torch.randn(hkv, n, d, generator=g, device=dev).to(dt)
    return K, V, centers, g


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


lines = []
for B in [int(x) for x in a.batches.split(",")]:
    hkv, d = 8, 128
    K, V, centers, g = make(B, hkv, a.ctx, d, seed=B)
    params = engine.make_params(a.hq, hkv, d, K.dtype, a.beta, 16, 64, a.chunk, 0,
                                int(a.block_filter))
    bnd = [engine.block_bounds(K[b]) if a.block_filter else None for b in range(B)]
    call = engine.Call([engine.SeqView(k=K[b], v=V[b], n=a.ctx, bounds=bnd[b]) for b in range(B)],
                       params, K.dtype, dev)
    pick = torch.randint(0, 16, (B, a.hq), generator=g, device=dev)
    q = (centers[pick] + 0.25 * torch.randn(B, a.hq, d, generator=g, device=dev)).float()
    out = torch.empty_like(q)
    t_full = timed(lambda: call.dipr_attention(q, out=out), a.reps)
    t_scan = timed(lambda: call.scan_only(q), a.reps)
    kbytes = B * hkv * a.ctx * d * K.element_size()
    d_ = {"label": a.label, "B": B, "hq": a.hq, "ctx": a.ctx, "chunk": a.chunk,
          "locality": a.locality, "dtype": str(K.dtype), "block_filter": a.block_filter, "us_call": round(t_full, 1), "us_scan": round(t_scan, 1),
          "scan_GBps": round(kbytes / t_scan / 1e3, 1),
          "qh_per_s": round(B * a.hq / t_full * 1e6),
          "env": {k: v for k, v in os.environ.items() if k.startswith("ALAYA_")}}
    print(json.dumps(d_), flush=True)
    lines.append(d_)
    del K, V, call
    torch.cuda.empty_cache()
if a.out:
    with open(a.out, "a") as fh:
        for d_ in lines:
            fh.write(json.dumps(d_) + "\n")
