"""Scan-kernel probe: times the scan stage alone (CUDA events, 5 reps over L layers)
for the bench workload shape, plus a torch read-bandwidth reference.
Usage: python tools/probe_scan.py [--scan-kernel tcgen05] (env ALAYA_TC_STAGES/PROMO)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_10326_b200 import engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scan-kernel", default="tcgen05")
ap.add_argument("--batch", type=int, default=4)
ap.add_argument("--ctx", type=int, default=131072)
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--hq", type=int, default=32)
ap.add_argument("--torch-ref", action="store_true")
a = ap.parse_args()
dev = torch.device("cuda")
L, B, Hkv, n, d = a.layers, a.batch, 8, a.ctx, 128
K = torch.randn(L, B, Hkv, n, d, device=dev, dtype=torch.bfloat16)
q = torch.randn(B, a.hq, d, device=dev)
params = engine.make_params(a.hq, Hkv, d, torch.bfloat16, 110.0, 16, 64, 0,
                            {"auto": 0, "cuda_core": 1, "tcgen05": 2}[a.scan_kernel])
calls = [engine.Call([engine.SeqView(k=K[l, b], v=K[l, b], n=n) for b in range(B)], params,
                     torch.bfloat16, dev) for l in range(L)]
for c in calls:
    c.scan_only(q)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
e0.record()
for _ in range(reps):
    for c in calls:
        c.scan_only(q)
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / (reps * L) / 1e3
kb = B * Hkv * n * d * 2
out = {"scan": a.scan_kernel, "stages": os.environ.get("ALAYA_TC_STAGES"),
       "promo": os.environ.get("ALAYA_TC_PROMO"), "us": round(t * 1e6, 1),
       "GBps": round(kb / t / 1e9, 1)}
if a.torch_ref:
    x = K.view(-1)
    torch.sum(x[: 1 << 31])
    torch.cuda.synchronize()
    e0.record()
    for _ in range(3):
        torch.sum(x[: 1 << 31], dtype=torch.float32)
    e1.record()
    torch.cuda.synchronize()
    tt = e0.elapsed_time(e1) / 3 / 1e3
    out["torch_sum_read_GBps"] = round((1 << 32) / tt / 1e9, 1)
    y = torch.empty_like(K[:2])
    y.copy_(K[2:4])
    torch.cuda.synchronize()
    e0.record()
    for _ in range(3):
        y.copy_(K[2:4])
    e1.record()
    torch.cuda.synchronize()
    tt = e0.elapsed_time(e1) / 3 / 1e3
    out["torch_copy_GBps"] = round(2 * y.numel() * 2 / tt / 1e9, 1)
print(json.dumps(out), flush=True)
