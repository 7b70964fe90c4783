timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"topk|prep|scan_tc|sparse_attn|chunk_topk" --csv --log-file gpurun_out/topk3.csv python - <<'PY' > /dev/null 2>&1
import sys, math, torch
sys.path.insert(0, '.')
from paper_2504_10326_b200 import engine as E
dev = torch.device('cuda'); B, hq, hkv, n, d = 1, 32, 8, 131072, 128
g = torch.Generator(device=dev).manual_seed(0)
c = torch.randn(16, d, generator=g, device=dev); centers = c / c.norm(dim=1, keepdim=True) * math.sqrt(d)
a_ = torch.randint(0, 16, (B, hkv, n), generator=g, device=dev)
K = (centers[a_] + 0.25 * torch.randn(B, hkv, n, d, generator=g, device=dev)).to(torch.bfloat16)
V = torch.randn(B, hkv, n, d, generator=g, device=dev).to(torch.bfloat16)
params = E.make_params(hq, hkv, d, torch.bfloat16, 0.0, 16, 64)
call = E.Call([E.SeqView(k=K[b], v=V[b], n=n) for b in range(B)], params, torch.bfloat16, dev)
q = (centers[torch.randint(0, 16, (B, hq), generator=g, device=dev)] + 0.25 * torch.randn(B, hq, d, generator=g, device=dev)).float()
for _ in range(3):
    ids, cnt = call.topk(q, 100); call.sparse_attention(q, ids, cnt)
torch.cuda.synchronize()
PY
python tools/launches.py gpurun_out/topk3.csv 14
