"""Candidate-superset statistics of the scan on the bench workload shape (diagnostics)."""
import os, sys, json, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_10326_b200 import engine
dev = torch.device("cuda")
B, Hkv, n, d, Hq = int(os.environ.get("B", "4")), 8, 131072, 128, 32
CH = 2048 if B >= 4 else 1024  # the auto chunk at 128K
g = torch.Generator(device=dev).manual_seed(0)
c = torch.randn(16, d, generator=g, device=dev); c = c / c.norm(dim=1, keepdim=True) * math.sqrt(d)
K = torch.empty(B, Hkv, n, d, dtype=torch.bfloat16, device=dev)
for b in range(B):
    a = torch.randint(0, 16, (Hkv, n), generator=g, device=dev)
    K[b] = (c[a] + 0.25 * torch.randn(Hkv, n, d, generator=g, device=dev)).to(torch.bfloat16)
q = (c[torch.randint(0, 16, (B, Hq), generator=g, device=dev)] + 0.25 * torch.randn(B, Hq, d, generator=g, device=dev)).float()
for scan in (2, 1):
    p = engine.make_params(Hq, Hkv, d, torch.bfloat16, 110.0, 16, 64, 0, scan)
    call = engine.Call([engine.SeqView(k=K[b], v=K[b], n=n) for b in range(B)], p, torch.bfloat16, dev)
    call.dipr_attention(q)
    torch.cuda.synchronize()
    cnt = call.candidate_counts(CH).sum(-1).float()
    ids, nsel, _ = call.selected(n)
    print(json.dumps({"B": B, "chunk": CH, "scan": scan, "pairs": cnt.numel(), "mean": cnt.mean().item(), "max": cnt.max().item(),
                      "p99": cnt.quantile(0.99).item(), "gt512": int((cnt > 512).sum()),
                      "selected_mean_per_head": nsel.float().mean().item()}))
