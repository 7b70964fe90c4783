"""Cost of the per-layer Session.update append next to the attention call
(diagnostic): B sessions x 128K bf16, one layer, CUDA-event mean per
(append + dipr_attention) for: no append, two torch copies (bench step),
alaya_window_append."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_10326_b200 import engine  # noqa: E402

B, n, hkv, hq, d = 4, 131072, 8, 32, 128
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
cap = 4096
WK = torch.zeros(B, hkv, cap, d, dtype=torch.bfloat16, device=dev)
WV = torch.zeros_like(WK)
q = (centers[torch.randint(0, 16, (B, hq), generator=g, device=dev)] + 0.25 * torch.randn(B, hq, d, generator=g, device=dev)).float()
kn = torch.randn(B, hkv, d, device=dev)
vn = torch.randn(B, hkv, d, device=dev)
params = engine.make_params(hq, hkv, d, torch.bfloat16, 110.0, 16, 64)
seqs = [engine.SeqView(k=K[b], v=V[b], n=n, wk=WK[b], wv=WV[b], w=16) for b in range(B)]
call = engine.Call(seqs, params, torch.bfloat16, dev)
out = torch.empty_like(q)
state = {"w": 16}


def none_():
    call.dipr_attention(q, out=out)


def torch_copies():
    w = state["w"] = state["w"] % 4000 + 1
    WK[:, :, w - 1] = kn.to(torch.bfloat16)
    WV[:, :, w - 1] = vn.to(torch.bfloat16)
    call.set_window_rows(w)
    call.dipr_attention(q, out=out)


aseqs = [engine.SeqView(k=None, v=None, n=0, wk=WK[b], wv=WV[b], w=0) for b in range(B)]


def alaya_append():
    w = state["w"] = state["w"] % 4000 + 1
    for s in aseqs:
        s.w = w - 1
    engine.window_append(aseqs, params, torch.bfloat16, kn, vn)
    call.set_window_rows(w)
    call.dipr_attention(q, out=out)


res = {}
for name, fn in (("no_append", none_), ("torch_copies", torch_copies), ("alaya_window_append", alaya_append)):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        fn()
    e1.record()
    torch.cuda.synchronize()
    res[name] = round(e0.elapsed_time(e1) / 50 * 1e3, 1)
print(json.dumps({"B": B, "us_per_layer": res}))
