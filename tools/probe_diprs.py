"""Graph DIPRS vs the flat scan on the GPU (diagnostic).

Loads a graph built by the REAL reference (`build_shared_graph`, default
GraphParams) over one Llama-shaped head (d=128) -- generated in the build
container by tools/make_graph.py into gpurun_in/ (not committed: 16+ MB) --
and times, for 32 query heads (4 sessions x 8 heads sharing the head):
  diprs   alaya_diprs (the candidate-list walk) + alaya_sparse_attention
  flat    alaya_dipr_attention (exact flat scan + attend + combine)
and reports explored nodes per query and the recall of the walk vs the flat
(exact) set.
"""

from __future__ import annotations

import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_10326_b200 import engine  # noqa: E402

path = sys.argv[1]
z = np.load(path)
dev = torch.device("cuda")
keys = torch.from_numpy(z["keys"]).to(dev, torch.bfloat16)
vals = torch.from_numpy(z["values"]).to(dev, torch.bfloat16)
n, d = keys.shape
deg = z["degrees"].astype(np.int64)
off = np.zeros(n + 1, np.int64)
off[1:] = np.cumsum(deg)
graph = (torch.from_numpy(off).to(dev)[None], torch.from_numpy(z["nbrs"].astype(np.int32)).to(dev)[None],
         torch.tensor([int(z["entry"])], dtype=torch.int32, device=dev))
centers = torch.from_numpy(z["centers"]).to(dev, torch.float32)
B, hq = 4, 8
g = torch.Generator(device=dev).manual_seed(1)
pick = torch.randint(0, centers.shape[0], (B, hq), generator=g, device=dev)
q = (centers[pick] + 0.25 * torch.randn(B, hq, d, generator=g, device=dev)).float()
K, V = keys[None], vals[None]


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for beta in (6.0, 20.0, 110.0):
    params = engine.make_params(hq, 1, d, torch.bfloat16, beta, 16, 64)
    call = engine.Call([engine.SeqView(k=K, v=V, n=n) for _ in range(B)], params, torch.bfloat16, dev)
    res = {}

    def walk():
        ids, cnt, exp = call.diprs(q, [graph] * B, 128, floor_mode=1)
        call.sparse_attention(q, ids, cnt)
        res["w"] = (ids, cnt, exp)

    def flat():
        call.dipr_attention(q)

    t_walk, t_flat = timed(walk), timed(flat)
    ids, cnt, exp = res["w"]
    call.dipr_attention(q)
    fid, fsel, fret = call.selected(n)
    rec = []
    for r in range(B * hq):
        got = set(ids[r, : int(cnt[r])].tolist())
        want = set(fid[r, : int(fsel[r])].tolist())
        rec.append(len(got & want) / max(1, len(want)))
    print(json.dumps({"n": n, "beta": beta, "q_heads": B * hq, "us_diprs": round(t_walk, 1),
                      "us_flat": round(t_flat, 1), "explored_per_q": round(float(exp.float().mean()), 1),
                      "selected_per_q_flat": round(float(fsel.float().mean()), 1),
                      "recall_vs_exact": round(float(np.mean(rec)), 4)}), flush=True)
