"""Host issue cost of one decode step as bench.py issues it (diagnostic).

B sessions x L layers at 128K bf16: per layer a window append + a DIPR call.
Reports, per layer, the host wall time of the enqueue loop (no sync inside)
for the whole step, for the appends alone and for the DIPR calls alone, next
to the GPU time of the step (CUDA events). host >= GPU: the step is host-bound.

  python tools/probe_host_step.py --batch 1
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_10326_b200 import engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--ctx", type=int, default=131072)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
dev = torch.device("cuda")
B, L, hq, hkv, d, n = a.batch, a.layers, 32, 8, 128, a.ctx
g = torch.Generator(device=dev).manual_seed(0)
c = torch.randn(16, d, generator=g, device=dev)
centers = c / c.norm(dim=1, keepdim=True) * math.sqrt(d)
K = torch.empty(L, B, hkv, n, d, dtype=torch.bfloat16, device=dev)
V = torch.empty_like(K)
for l in range(L):
    for b in range(B):
        a_ = torch.randint(0, 16, (hkv, n), generator=g, device=dev)
        K[l, b] = (centers[a_] + 0.25 * torch.randn(hkv, n, d, generator=g, device=dev)).to(K.dtype)
        V[l, b] = torch.randn(hkv, n, d, generator=g, device=dev).to(K.dtype)
cap = 64
WK = torch.zeros(L, B, hkv, cap, d, dtype=torch.bfloat16, device=dev)
WV = torch.zeros_like(WK)
Q = (centers[torch.randint(0, 16, (L, B, hq), generator=g, device=dev)] +
     0.25 * torch.randn(L, B, hq, d, generator=g, device=dev)).float()
KN = torch.randn(L, B, hkv, d, generator=g, device=dev)
VN = torch.randn_like(KN)
ap_params = engine.make_params(hq, hkv, d, torch.bfloat16, 0.0, 0, 0)
params = engine.make_params(hq, hkv, d, torch.bfloat16, 110.0, 16, 64)
app = [[engine.SeqView(k=None, v=None, n=0, wk=WK[l, b], wv=WV[l, b], w=16) for b in range(B)] for l in range(L)]
calls = [engine.Call([engine.SeqView(k=K[l, b], v=V[l, b], n=n, wk=WK[l, b], wv=WV[l, b], w=17)
                      for b in range(B)], params, torch.bfloat16, dev) for l in range(L)]
out = torch.empty(L, B, hq, d, device=dev)


def step(do_append=True, do_attn=True):
    for l in range(L):
        if do_append:
            engine.window_append(app[l], ap_params, torch.bfloat16, KN[l], VN[l])
        if do_attn:
            calls[l].dipr_attention(Q[l], out=out[l])


res = {"B": B, "layers": L}
for name, kw in (("step", {}), ("append_only", {"do_attn": False}), ("dipr_only", {"do_append": False})):
    step(**kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    host = []
    e0.record()
    for _ in range(a.reps):
        t0 = time.perf_counter()
        step(**kw)
        host.append(time.perf_counter() - t0)
    e1.record()
    torch.cuda.synchronize()
    res[name] = {"host_us_per_layer": round(min(host) / L * 1e6, 1),
                 "gpu_us_per_layer": round(e0.elapsed_time(e1) / a.reps / L * 1e3, 1)}
print(json.dumps(res))
