"""Decode step eager vs CUDA graph (DecodeStepGraph), per layer call (diagnostic).

B sessions, L layers of a Llama-3.1-8B-shaped layer (32 q / 8 kv heads, bf16), the
bench's per-layer calls: window append + DIPR attention. Eager = prebuilt calls
(the bench's fast path: cached descriptors, host window counts); graph = one
replay per step. CUDA-event time per layer, after warm-up.

  python tools/probe_graph.py --ctx 8192,32768,131072 --batch 1 --layers 8
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_10326_b200 import DecodeStepGraph, engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ctx", default="8192,32768,131072")
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--steps", type=int, default=20)
a = ap.parse_args()
dev = torch.device("cuda")
hq, hkv, d, L, B = 32, 8, 128, a.layers, a.batch
params = engine.make_params(hq, hkv, d, torch.bfloat16, 110.0, 16, 64)
for n in (int(x) for x in a.ctx.split(",")):
    g = torch.Generator(device=dev).manual_seed(0)
    c = torch.randn(16, d, generator=g, device=dev)
    centers = c / c.norm(dim=1, keepdim=True) * math.sqrt(d)
    K = torch.empty(L, B, hkv, n, d, dtype=torch.bfloat16, device=dev)
    V = torch.empty_like(K)
    for l in range(L):
        for b in range(B):
            asg = torch.randint(0, 16, (hkv, n), generator=g, device=dev)
            K[l, b] = (centers[asg] + 0.25 * torch.randn(hkv, n, d, generator=g, device=dev)).to(torch.bfloat16)
            V[l, b] = torch.randn(hkv, n, d, generator=g, device=dev).to(torch.bfloat16)
    cap = 16 + 2 * (a.steps + 10)
    WK = torch.zeros(L, B, hkv, cap, d, dtype=torch.bfloat16, device=dev)
    WV = torch.zeros_like(WK)
    Q = (centers[torch.randint(0, 16, (L, B, hq), generator=g, device=dev)]
         + 0.25 * torch.randn(L, B, hq, d, generator=g, device=dev)).float()
    KN = torch.randn(L, B, hkv, d, generator=g, device=dev)
    VN = torch.randn_like(KN)
    res = {"ctx": n, "B": B, "layers": L}
    # eager
    views = [[engine.SeqView(k=K[l, b], v=V[l, b], n=n, wk=WK[l, b], wv=WV[l, b], w=16) for b in range(B)]
             for l in range(L)]
    calls = [engine.Call(v, params, torch.bfloat16, dev) for v in views]
    apps = [engine.append_array(v, params, torch.bfloat16) for v in views]
    out = torch.empty(L, B, hq, d, device=dev)
    w = [16]

    def eager_step():
        for l in range(L):
            for i in range(B):
                apps[l][i].w = w[0]
            engine.window_append_raw(apps[l], B, params, KN[l], VN[l])
            calls[l].set_window_rows(w[0] + 1)
            calls[l].dipr_attention(Q[l], out=out[l])
        w[0] += 1

    for label, fn in (("eager", eager_step),):
        for _ in range(5):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[f"{label}_us_per_layer"] = round(e0.elapsed_time(e1) * 1e3 / (a.steps * L), 1)
    # graph
    counts = [torch.full((1,), 16, dtype=torch.int32, device=dev) for _ in range(L * B)]
    layers = [[engine.SeqView(k=K[l, b], v=V[l, b], n=n, wk=WK[l, b], wv=WV[l, b], w_dev=counts[l * B + b])
               for b in range(B)] for l in range(L)]
    gr = DecodeStepGraph(layers, params, torch.bfloat16, dev)
    gr.q.copy_(Q)
    gr.k.copy_(KN)
    gr.v.copy_(VN)
    for _ in range(5):
        gr.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.steps):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    res["graph_us_per_layer"] = round(e0.elapsed_time(e1) * 1e3 / (a.steps * L), 1)
    res["graph_qh_per_s"] = round(B * hq / (res["graph_us_per_layer"] * 1e-6))
    res["eager_qh_per_s"] = round(B * hq / (res["eager_us_per_layer"] * 1e-6))
    print(json.dumps(res), flush=True)
    del K, V, WK, WV, gr, calls
    torch.cuda.empty_cache()
