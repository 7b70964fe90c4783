"""Can the V-gather attend stage overlap the K scan? (diagnostic)

B sessions of a 128K Llama-shaped layer (bf16). Variants, CUDA-event mean per
layer call:
  one      one alaya_dipr_attention over all B sessions
  halves   two half-batch calls, one stream
  streams  two half-batch calls on two streams (separate workspaces), so the
           second half's scan can run beside the first half's attend
"""

from __future__ import annotations

import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_10326_b200 import engine  # noqa: E402

B = int(os.environ.get("PB", "4"))
n, hkv, hq, d = 131072, 8, 32, 128
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
c = torch.randn(16, d, generator=g, device=dev)
centers = c / c.norm(dim=1, keepdim=True) * math.sqrt(d)
K = torch.empty(B, hkv, n, d, dtype=torch.bfloat16, device=dev)
V = torch.empty_like(K)
for b in range(B):
    a_ = torch.randint(0, 16, (hkv, n), generator=g, device=dev)
    K[b] = (centers[a_] + 0.25 * torch.randn(hkv, n, d, generator=g, device=dev)).to(torch.bfloat16)
    V[b] = torch.randn(hkv, n, d, generator=g, device=dev).to(torch.bfloat16)
pick = torch.randint(0, 16, (B, hq), generator=g, device=dev)
q = (centers[pick] + 0.25 * torch.randn(B, hq, d, generator=g, device=dev)).float()
params = engine.make_params(hq, hkv, d, torch.bfloat16, 110.0, 16, 64)
seqs = [engine.SeqView(k=K[b], v=V[b], n=n) for b in range(B)]
h = B // 2
one = engine.Call(seqs, params, torch.bfloat16, dev)
ws0 = torch.empty(one.ws_bytes, dtype=torch.uint8, device=dev)
ws1 = torch.empty(one.ws_bytes, dtype=torch.uint8, device=dev)
c0 = engine.Call(seqs[:h], params, torch.bfloat16, dev, ws=ws0)
c1 = engine.Call(seqs[h:], params, torch.bfloat16, dev, ws=ws1)
out = torch.empty_like(q)
s1 = torch.cuda.Stream()


def v_one():
    one.dipr_attention(q, out=out)


def v_halves():
    c0.dipr_attention(q[:h], out=out[:h])
    c1.dipr_attention(q[h:], out=out[h:])


def v_streams():
    main = torch.cuda.current_stream()
    s1.wait_stream(main)
    c0.dipr_attention(q[:h], out=out[:h])
    with torch.cuda.stream(s1):
        c1.dipr_attention(q[h:], out=out[h:])
    main.wait_stream(s1)


res = {}
for name, fn in (("one", v_one), ("halves", v_halves), ("streams", v_streams)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        fn()
    e1.record()
    torch.cuda.synchronize()
    res[name] = round(e0.elapsed_time(e1) / 20 * 1e3, 1)
print(json.dumps({"B": B, "us_per_layer_call": res}))
