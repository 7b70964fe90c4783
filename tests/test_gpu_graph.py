"""A decode step captured as a CUDA graph (``DecodeStepGraph``: device window row
counts, ``alaya_seq.d_w``) replays the same per-layer window append + DIPR
attention as the eager calls, step after step while the windows grow, and the
graph-mode append stops at the ring capacity."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import alaya_oracle as O

pytestmark = pytest.mark.gpu


def _setup(L, B, hq, hkv, d, n, cap, w0, seed):
    dev = torch.device("cuda")
    K, V = [], []
    for b in range(B):
        _, k, v, _, _ = O.make_context(n + 700 * b, L, hkv, d, seed=seed + b)
        K.append(torch.from_numpy(O.bf16_round(k)).to(dev, torch.bfloat16))
        V.append(torch.from_numpy(O.bf16_round(v)).to(dev, torch.bfloat16))
    g = torch.Generator(device=dev).manual_seed(seed)
    WK = torch.randn(L, B, hkv, cap, d, generator=g, device=dev).to(torch.bfloat16)
    WV = torch.randn(L, B, hkv, cap, d, generator=g, device=dev).to(torch.bfloat16)
    return dev, K, V, WK, WV


@pytest.mark.parametrize("B,beta", [(1, 110.0), (3, 5.0)])
def test_graph_replay_matches_eager(cuda_ok, B, beta):
    from paper_2504_10326_b200 import DecodeStepGraph, engine
    L, hq, hkv, d, n, cap, w0, steps = 2, 8, 2, 128, 5000, 16, 2, 4
    dev, K, V, WK, WV = _setup(L, B, hq, hkv, d, n, cap, w0, 11)
    params = engine.make_params(hq, hkv, d, torch.bfloat16, beta, 16, 64)
    g = torch.Generator(device=dev).manual_seed(5)
    Q = torch.randn(steps, L, B, hq, d, generator=g, device=dev) * 4
    KN = torch.randn(steps, L, B, hkv, d, generator=g, device=dev)
    VN = torch.randn(steps, L, B, hkv, d, generator=g, device=dev)
    # eager: host window counts
    WKe, WVe = WK.clone(), WV.clone()
    eager = []
    for s in range(steps):
        outs = []
        for l in range(L):
            views = [engine.SeqView(k=K[b][l], v=V[b][l], n=K[b].shape[2], wk=WKe[l, b], wv=WVe[l, b],
                                    w=w0 + s) for b in range(B)]
            engine.window_append(views, params, torch.bfloat16, KN[s, l], VN[s, l])
            for vw in views:
                vw.w += 1
            outs.append(engine.Call(views, params, torch.bfloat16, dev).dipr_attention(Q[s, l]).clone())
        eager.append(torch.stack(outs))
    # graph: device window counts, one capture
    counts = [torch.full((1,), w0, dtype=torch.int32, device=dev) for _ in range(L * B)]
    layers = [[engine.SeqView(k=K[b][l], v=V[b][l], n=K[b].shape[2], wk=WK[l, b], wv=WV[l, b],
                              w_dev=counts[l * B + b]) for b in range(B)] for l in range(L)]
    gr = DecodeStepGraph(layers, params, torch.bfloat16, dev)
    assert all(int(c.item()) == w0 for c in counts)  # the warm-up step was undone
    for s in range(steps):
        gr.q.copy_(Q[s])
        gr.k.copy_(KN[s])
        gr.v.copy_(VN[s])
        out = gr.replay()
        torch.cuda.synchronize()
        err = float(((out - eager[s]).norm() / eager[s].norm()).item())
        assert err <= 1e-6, (s, err)
    assert all(int(c.item()) == w0 + steps for c in counts)
    assert torch.equal(WK, WKe) and torch.equal(WV, WVe)  # same rows appended


def test_graph_mode_append_stops_at_capacity(cuda_ok):
    from paper_2504_10326_b200 import engine
    dev = torch.device("cuda")
    params = engine.make_params(4, 2, 64, torch.float32, 5.0, 0, 0)
    wk = torch.zeros(2, 3, 64, device=dev)
    wv = torch.zeros_like(wk)
    cnt = torch.tensor([2], dtype=torch.int32, device=dev)
    view = engine.SeqView(k=None, v=None, n=0, wk=wk, wv=wv, w_dev=cnt)
    for i in range(3):
        engine.window_append([view], params, torch.float32, torch.full((1, 2, 64), i + 1.0, device=dev),
                             torch.full((1, 2, 64), -(i + 1.0), device=dev))
    torch.cuda.synchronize()
    assert int(cnt.item()) == 3  # row 2 written, then the ring is full
    assert torch.all(wk[:, 2] == 1.0) and torch.all(wv[:, 2] == -1.0)
    assert torch.all(wk[:, :2] == 0)


def test_graph_replay_refuses_a_full_ring(cuda_ok):
    """the device append drops rows at capacity, so DecodeStepGraph.replay
    must refuse the replay that would need a row the ring does not have."""
    from paper_2504_10326_b200 import DecodeStepGraph, engine
    L, B, hq, hkv, d, n, cap, w0 = 1, 1, 8, 2, 128, 3000, 5, 2
    dev, K, V, WK, WV = _setup(L, B, hq, hkv, d, n, cap, w0, 3)
    params = engine.make_params(hq, hkv, d, torch.bfloat16, 20.0, 16, 64)
    counts = [torch.full((1,), w0, dtype=torch.int32, device=dev)]
    layers = [[engine.SeqView(k=K[0][0], v=V[0][0], n=n, wk=WK[0, 0], wv=WV[0, 0], w_dev=counts[0])]]
    gr = DecodeStepGraph(layers, params, torch.bfloat16, dev)
    assert gr.remaining == cap - w0
    for _ in range(cap - w0):
        gr.replay()
    torch.cuda.synchronize()
    assert int(counts[0].item()) == cap and gr.remaining == 0
    with pytest.raises(RuntimeError, match="window ring full"):
        gr.replay()
    counts[0].fill_(w0)  # the caller rewinds the ring: re-read the counts
    assert gr.sync_rows() == w0 and gr.remaining == cap - w0
