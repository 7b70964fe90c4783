"""Host-side issue cost of the public API per layer (diagnostic): how long
Session.update_batch + Session.attention_batch take on the CPU to enqueue one
layer for B sessions, vs the device time of the same layer."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_10326_b200 as P  # noqa: E402

B, n, L, hq, hkv, d = 4, 131072, 4, 32, 8, 128
dev = torch.device("cuda")
shape = P.ModelShape(L, hq, hkv, d)
cfg = P.EngineConfig(beta=110.0, first_layers=tuple(range(L)), short_context_threshold=0,
                     kv_dtype="bfloat16", diagnostics=False)
db = P.ContextStore(shape, cfg, device=dev, log_queries=False)
K = torch.randn(L, B, hkv, n, d, device=dev).to(torch.bfloat16)
V = torch.randn(L, B, hkv, n, d, device=dev).to(torch.bfloat16)
sessions = []
for b in range(B):
    tok = np.arange(n, dtype=np.int64) + b * 7919
    rec = P.ContextRecord(P.store.context_id_for(tok, shape), tok, K[:, b], V[:, b], shape,
                          db._plans_for(n))
    db.contexts[rec.context_id] = rec
    s, _ = db.create_session(tok)
    sessions.append(s)
q = torch.randn(L, B, hq, d, device=dev)
k = torch.randn(L, B, hkv, d, device=dev)
v = torch.randn(L, B, hkv, d, device=dev)
out = torch.empty(L, B, hq, d, device=dev)


def layer(l):
    P.Session.update_batch(sessions, q[l], k[l], v[l], l)
    P.Session.attention_batch(sessions, q[l], l, out=out[l])


for _ in range(3):
    for l in range(L):
        layer(l)
torch.cuda.synchronize()
t_upd = t_att = 0.0
reps = 20
for _ in range(reps):
    for l in range(L):
        t0 = time.perf_counter()
        P.Session.update_batch(sessions, q[l], k[l], v[l], l)
        t1 = time.perf_counter()
        P.Session.attention_batch(sessions, q[l], l, out=out[l])
        t2 = time.perf_counter()
        t_upd += t1 - t0
        t_att += t2 - t1
    torch.cuda.synchronize()
print(f"host us per layer: update_batch {t_upd / reps / L * 1e6:.1f}, attention_batch {t_att / reps / L * 1e6:.1f}")
