"""``alaya_dipr_attention_update`` (Session.update + Session.attention in one
call, the append done by the call's first kernel) equals the two-call sequence
``alaya_window_append`` then ``alaya_dipr_attention``: same ring contents, same
outputs, step after step (bf16 tcgen05 and fp32 CUDA-core paths)."""

from __future__ import annotations

import pytest
import torch

from oracle import alaya_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype,B", [(torch.bfloat16, 3), (torch.float32, 2)])
def test_update_attention_fused_equals_two_calls(cuda_ok, dtype, B):
    from paper_2504_10326_b200 import engine
    dev = torch.device("cuda")
    hq, hkv, d, n, cap, w0, steps = 32, 8, 128, 9000, 12, 2, 4
    K, V = [], []
    for b in range(B):
        _, k, v, _, _ = O.make_context(n + 500 * b, 1, hkv, d, seed=40 + b)
        K.append(torch.from_numpy(k[0]).to(dev, dtype))
        V.append(torch.from_numpy(v[0]).to(dev, dtype))
    g = torch.Generator(device=dev).manual_seed(9)
    WK = torch.randn(2, B, hkv, cap, d, generator=g, device=dev).to(dtype)
    WV = torch.randn(2, B, hkv, cap, d, generator=g, device=dev).to(dtype)
    WK[1], WV[1] = WK[0], WV[0]  # ring 0: fused path, ring 1: two calls
    Q = torch.randn(steps, B, hq, d, generator=g, device=dev) * 4
    KN = torch.randn(steps, B, hkv, d, generator=g, device=dev)
    VN = torch.randn(steps, B, hkv, d, generator=g, device=dev)
    params = engine.make_params(hq, hkv, d, dtype, 60.0, 16, 64)
    app_params = engine.make_params(hq, hkv, d, dtype, 0.0, 0, 0)
    for s in range(steps):
        w = w0 + s + 1
        fused = engine.Call([engine.SeqView(k=K[b], v=V[b], n=K[b].shape[1], wk=WK[0, b], wv=WV[0, b], w=w)
                             for b in range(B)], params, dtype, dev)
        o_f = fused.dipr_attention(Q[s], append=(KN[s], VN[s])).clone()
        app = [engine.SeqView(k=None, v=None, n=0, wk=WK[1, b], wv=WV[1, b], w=w - 1) for b in range(B)]
        engine.window_append(app, app_params, dtype, KN[s], VN[s])
        two = engine.Call([engine.SeqView(k=K[b], v=V[b], n=K[b].shape[1], wk=WK[1, b], wv=WV[1, b], w=w)
                           for b in range(B)], params, dtype, dev)
        o_t = two.dipr_attention(Q[s])
        torch.cuda.synchronize()
        assert torch.equal(WK[0], WK[1]) and torch.equal(WV[0], WV[1]), s
        err = float(((o_f - o_t).norm() / o_t.norm()).item())
        assert err <= 1e-6, (s, err)


def test_update_attention_rejects_bad_windows(cuda_ok):
    from paper_2504_10326_b200 import _lib, engine
    dev = torch.device("cuda")
    k = torch.randn(2, 300, 64, device=dev)
    params = engine.make_params(4, 2, 64, torch.float32, 5.0, 0, 0)
    call = engine.Call([engine.SeqView(k=k, v=k, n=300)], params, torch.float32, dev)  # no ring
    kn = torch.zeros(1, 2, 64, device=dev)
    with pytest.raises((ValueError, _lib.AlayaError)):
        call.dipr_attention(torch.randn(1, 4, 64, device=dev), append=(kn, kn))
