"""Host issue cost of one DIPR layer call vs its GPU period (diagnostic).

For B sessions of a 128K-token Llama-3.1-8B-shaped layer: wall time per call of
the enqueue loop (no synchronisation inside; the stream queue does not fill at
this count), of the bare C-ABI call with prebuilt arguments, and the GPU period
(CUDA events over the same loop). host >= GPU means the call is host-bound.

  python tools/probe_host.py --batches 1,4
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_10326_b200 import engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batches", default="1,4")
ap.add_argument("--ctx", type=int, default=131072)
ap.add_argument("--reps", type=int, default=100)
ap.add_argument("--label", default="base")
a = ap.parse_args()
dev = torch.device("cuda")

for B in [int(x) for x in a.batches.split(",")]:
    hq, hkv, d = 32, 8, 128
    g = torch.Generator(device=dev).manual_seed(B)
    c = torch.randn(16, d, generator=g, device=dev)
    centers = c / c.norm(dim=1, keepdim=True) * math.sqrt(d)
    K = torch.empty(B, hkv, a.ctx, d, dtype=torch.bfloat16, device=dev)
    V = torch.empty_like(K)
    for b in range(B):
        a_ = torch.randint(0, 16, (hkv, a.ctx), generator=g, device=dev)
        K[b] = (centers[a_] + 0.25 * torch.randn(hkv, a.ctx, d, generator=g, device=dev)).to(K.dtype)
        V[b] = torch.randn(hkv, a.ctx, d, generator=g, device=dev).to(K.dtype)
    params = engine.make_params(hq, hkv, d, K.dtype, 110.0, 16, 64)
    call = engine.Call([engine.SeqView(k=K[b], v=V[b], n=a.ctx) for b in range(B)], params, K.dtype, dev)
    pick = torch.randint(0, 16, (B, hq), generator=g, device=dev)
    q = (centers[pick] + 0.25 * torch.randn(B, hq, d, generator=g, device=dev)).float()
    out = torch.empty_like(q)
    lib, p, seqs = call.lib, ctypes.byref(call.params), call.seqs
    ws, wsb, st = call.ws.data_ptr(), call.ws_bytes, call.stream
    qp, op = q.data_ptr(), out.data_ptr()

    def raw():
        lib.alaya_dipr_attention(p, seqs, B, qp, op, ws, wsb, st)

    def api():
        call.dipr_attention(q, out=out)

    res = {"label": a.label, "B": B}
    for name, fn in (("api", api), ("raw", raw)):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.perf_counter()
        for _ in range(a.reps):
            fn()
        t_host = (time.perf_counter() - t0) / a.reps * 1e6
        e1.record()
        torch.cuda.synchronize()
        res[name] = {"host_us": round(t_host, 1), "gpu_us": round(e0.elapsed_time(e1) / a.reps * 1e3, 1)}
    print(json.dumps(res), flush=True)
    del K, V, call
    torch.cuda.empty_cache()
