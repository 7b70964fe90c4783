"""BASELINE configs 3 and 4 as sweeps (one JSON line per point):

  config 3: ctx 128K, batch B, Llama 32/8: beta sweep (retrieved-set size vs
            throughput), coarse block filter on/off, plus a LOCALITY variant
            (tokens sorted by cluster -- not the reference generator) where the
            block bound can prune;
  config 4: Qwen2.5-14B shape (40 q / 8 kv heads, G = 5) at 128K: tcgen05
            q.K^T scan vs the CUDA-core scan.

Times are CUDA-event means over `--reps` layer calls after warm-up on one
B200 (single layer; K/V of 256 MiB+ per session exceed L2). Usage:
  python tools/sweep.py --which 3 --out profiles/sweep_config3.jsonl
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
ap.add_argument("--which", default="3,4")
ap.add_argument("--ctx", type=int, default=131072)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--out", default=None)
a = ap.parse_args()
dev = torch.device("cuda")
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 6650.0
lines = []


def emit(d):
    print(json.dumps(d), flush=True)
    lines.append(d)


def make(B, hkv, n, d, locality, seed=0):
    g = torch.Generator(device=dev).manual_seed(seed)
    c = torch.randn(16, d, generator=g, device=dev)
    centers = c / c.norm(dim=1, keepdim=True) * math.sqrt(d)
    K = torch.empty(B, hkv, n, d, dtype=torch.bfloat16, device=dev)
    V = torch.empty_like(K)
    for b in range(B):
        a_ = torch.randint(0, 16, (hkv, n), generator=g, device=dev)
        if locality:
            a_ = torch.sort(a_, dim=1).values
        K[b] = (centers[a_] + 0.25 * torch.randn(hkv, n, d, generator=g, device=dev)).to(torch.bfloat16)
        V[b] = torch.randn(hkv, n, d, generator=g, device=dev).to(torch.bfloat16)
    return K, V, centers, g


def run_point(K, V, centers, g, hq, beta, scan, block_filter, bounds=None, label=""):
    B, hkv, n, d = K.shape
    params = engine.make_params(hq, hkv, d, torch.bfloat16, beta, 16, 64, 0,
                                {"auto": 0, "cuda_core": 1, "tcgen05": 2}[scan], int(block_filter))
    seqs = [engine.SeqView(k=K[b], v=V[b], n=n, bounds=bounds[b] if bounds is not None else None)
            for b in range(B)]
    call = engine.Call(seqs, params, torch.bfloat16, dev)
    pick = torch.randint(0, 16, (B, hq), generator=g, device=dev)
    q = (centers[pick] + 0.25 * torch.randn(B, hq, d, generator=g, device=dev)).float()
    out = torch.empty_like(q)
    for _ in range(3):
        call.dipr_attention(q, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        call.dipr_attention(q, out=out)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / a.reps / 1e3
    ids, nsel, _ = call.selected(n)
    g_ = hq // hkv
    union = 0
    for b in range(B):
        for h in range(hkv):
            rows = [ids[b * hq + h * g_ + j, : int(nsel[b * hq + h * g_ + j])] for j in range(g_)]
            union += int(torch.unique(torch.cat(rows)).numel())
    kept, total = call.block_stats() if block_filter else (None, None)
    kbytes = B * hkv * n * d * 2
    alg = kbytes if not block_filter else kbytes * kept / max(total, 1)
    alg += union * d * 2
    emit({"label": label, "B": B, "Hq": hq, "Hkv": hkv, "ctx": n, "beta": beta, "scan": scan,
          "block_filter": bool(block_filter), "us_per_layer_call": round(t * 1e6, 1),
          "query_heads_per_s": round(B * hq / t), "sel_frac_per_head": round(float(nsel.float().mean()) / n, 5),
          "union_frac": round(union / (B * hkv * n), 5),
          "blocks_kept": kept, "blocks_total": total,
          "key_scan_GBps": round(kbytes / t / 1e9, 1), "alg_GBps": round(alg / t / 1e9, 1),
          "alg_frac_of_measured_hbm": round(alg / t / 1e9 / peak, 4)})


which = a.which.split(",")
if "3" in which:
    for B in (1, 4, 16):
        K, V, centers, g = make(B, 8, a.ctx, 128, locality=False, seed=B)
        for beta in (1, 2, 5, 10, 20, 110, 115, 120, 125, 130, 140):
            run_point(K, V, centers, g, 32, beta, "auto", False,
                      label="config3 reference-generator data")
        bnd = torch.stack([engine.block_bounds(K[b]) for b in range(B)])
        for beta in (20, 50, 110):
            run_point(K, V, centers, g, 32, beta, "auto", True, bnd,
                      label="config3 reference-generator data + block filter")
        del K, V, bnd
        torch.cuda.empty_cache()
        if B != 16:
            K, V, centers, g = make(B, 8, a.ctx, 128, locality=True, seed=100 + B)
            bnd = torch.stack([engine.block_bounds(K[b]) for b in range(B)])
            for beta in (5, 20, 50, 110):
                for flt in (False, True):
                    run_point(K, V, centers, g, 32, beta, "auto", flt, bnd if flt else None,
                              label="config3 LOCALITY variant (tokens sorted by cluster)")
            del K, V, bnd
            torch.cuda.empty_cache()
if "4" in which:
    for B in (1, 8, 16):
        K, V, centers, g = make(B, 8, a.ctx, 128, locality=False, seed=200 + B)
        for scan in ("tcgen05", "cuda_core"):
            run_point(K, V, centers, g, 40, 110.0, scan, False,
                      label="config4 Qwen2.5-14B shape (40/8)")
        del K, V
        torch.cuda.empty_cache()
if "topk" in which:
    # TOP_K plans at 128K: exact flat top-k (scan with every token a candidate +
    # radix select) and the coarse block index (r=4 reps per 128-token block),
    # each followed by sparse attention over the retrieved ids + window
    from paper_2504_10326_b200 import engine as E
    for B in (1, 4):
        K, V, centers, g = make(B, 8, a.ctx, 128, locality=False, seed=300 + B)
        hq, hkv, n, d = 32, 8, a.ctx, 128
        params = E.make_params(hq, hkv, d, torch.bfloat16, 0.0, 16, 64)
        call = E.Call([E.SeqView(k=K[b], v=V[b], n=n) for b in range(B)], params, torch.bfloat16, dev)
        pick = torch.randint(0, 16, (B, hq), generator=g, device=dev)
        q = (centers[pick] + 0.25 * torch.randn(B, hq, d, generator=g, device=dev)).float()
        reps = [(E.block_reps(K[b], 128, 4), n) for b in range(B)]
        for mode, k in (("flat", 100), ("flat", 2048), ("coarse", 100), ("coarse", 2048)):
            def step():
                if mode == "flat":
                    ids, cnt = call.topk(q, k)
                else:
                    ids, cnt = call.block_topk(q, reps, 128, max(1, -(-k // 128)))
                call.sparse_attention(q, ids, cnt)
            for _ in range(3):
                step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                step()
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / a.reps / 1e3
            kbytes = B * hkv * n * d * 2 if mode == "flat" else B * hkv * (n // 128) * 4 * d * 2
            emit({"label": f"TOP_K {mode}", "B": B, "Hq": hq, "ctx": n, "k": k,
                  "us_per_layer_call": round(t * 1e6, 1), "query_heads_per_s": round(B * hq / t),
                  "scanned_bytes": kbytes, "scanned_GBps": round(kbytes / t / 1e9, 1),
                  "frac_of_measured_hbm": round(kbytes / t / 1e9 / peak, 4)})
        del K, V, call, reps
        torch.cuda.empty_cache()
if a.out:
    with open(a.out, "w") as fh:
        for d in lines:
            fh.write(json.dumps(d) + "\n")
