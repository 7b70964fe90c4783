"""Coarse block filter: the sound per-block box bound
must never change results -- identical selections and outputs with the
filter on and off -- while skipping blocks when the keys have locality."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import alaya_oracle as O
from tests.parity import EPS_SET, set_flips

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


def locality_context(n, hkv, d, seed):
    """Reference-generator keys with tokens sorted by cluster (labelled a
    locality variant: the reference's own generator draws clusters i.i.d.)."""
    _, keys, vals, centers, _ = O.make_context(n, 1, hkv, d, seed=seed)
    r = np.random.default_rng(seed)
    out_k = np.empty_like(keys)
    for h in range(hkv):
        a = r.integers(0, 16, n)
        order = np.argsort(a, kind="stable")
        out_k[0, h] = (centers[a[order]] + 0.25 * r.standard_normal((n, d))).astype(np.float32)
    return out_k, vals, centers


def test_block_index_is_sound(cuda_ok):
    """Box exact; representative = largest-norm key (ties by position); the ball
    q.mu + |q| r bounds every key of the block."""
    from paper_2504_10326_b200 import engine
    k = torch.randn(3, 1000, 128, device="cuda").to(torch.bfloat16)
    b = engine.block_bounds(k)
    assert b.shape == (3, 8, 5, 128)
    for blk in range(8):
        seg = k[:, blk * 128:(blk + 1) * 128].float()
        assert torch.equal(b[:, blk, 0].float(), seg.amin(1))
        assert torch.equal(b[:, blk, 1].float(), seg.amax(1))
        norms = seg.norm(dim=2)
        for h in range(3):
            rep = seg[h, int(torch.argmax(norms[h]))]
            assert torch.equal(b[h, blk, 3].float(), rep)
            dist = (seg[h] - b[h, blk, 2].float()).norm(dim=1).max()
            assert float(b[h, blk, 4, 0]) >= float(dist)


@pytest.mark.parametrize("kv,scan", [("bfloat16", "tcgen05"), ("bfloat16", "cuda_core"),
                                     ("float32", "cuda_core")])
@pytest.mark.parametrize("beta", [5.0, 50.0, 110.0])
def test_filter_is_exact_and_prunes_with_locality(cuda_ok, kv, scan, beta):
    import paper_2504_10326_b200 as P
    n, hkv, g, d = 40000, 2, 4, 128
    keys, vals, centers = locality_context(n, hkv, d, seed=int(beta))
    if kv == "bfloat16":
        keys, vals = O.bf16_round(keys), O.bf16_round(vals)
    r = np.random.default_rng(1)
    q = (centers[r.integers(0, 16, hkv * g)] + 0.25 * r.standard_normal((hkv * g, d))).astype(np.float32)
    tok = np.arange(n)
    outs, sels, stats = [], [], []
    for flt in (False, True):
        cfg = P.EngineConfig(beta=beta, first_layers=(0,), short_context_threshold=0, kv_dtype=kv,
                             scan_kernel=scan, block_filter=flt)
        db = P.ContextStore(P.ModelShape(1, hkv * g, hkv, d), cfg)
        db.import_context(tok, keys, vals)
        s, _ = db.create_session(tok)
        outs.append(s.attention(q, 0))
        sels.append([h["selected_base"] for h in s.last_diagnostics["heads"]])
        if flt:
            call = next(iter(db._calls.values()))[1]
            stats.append(call.block_stats())
    kept, total = stats[0]
    assert total == hkv * ((n + 127) // 128)
    if beta <= 50.0:  # sorted clusters prune at beta 20/50, not at 110
        assert kept < total, "sorted clusters must let the block bound prune"
    assert sels[0] == sels[1]  # exact: pruning never drops a selected token
    # same rows, but pruned tiles change candidate batching -> summation order
    assert rel(outs[1], outs[0].astype(np.float64)) <= 1e-6
    ref, rsel, _ = O.session_attention_flat(q, keys[0], vals[0], None, None, beta)
    window = O.window_base_ids(n)
    for qh in range(hkv * g):
        h = qh // g
        flips, _ = set_flips(sels[1][qh], O.inner_products(keys[0, h], q[qh]), beta,
                             EPS_SET[kv], window)
        o_sel = O.head_attention_on_selection(q[qh], keys[0, h], vals[0, h], None, None, sels[1][qh])
        assert rel(outs[1][qh], o_sel) <= 1e-5
        if not flips:
            assert rel(outs[1][qh], ref[qh]) <= 1e-5


def test_filter_keeps_everything_on_reference_generator(cuda_ok):
    """i.i.d. cluster draws defeat any box bound."""
    import paper_2504_10326_b200 as P
    n, hkv, g, d = 20000, 2, 4, 128
    tok, keys, vals, centers, _ = O.make_context(n, 1, hkv, d, seed=3)
    keys, vals = O.bf16_round(keys), O.bf16_round(vals)
    cfg = P.EngineConfig(beta=110.0, first_layers=(0,), short_context_threshold=0,
                         kv_dtype="bfloat16", block_filter=True)
    db = P.ContextStore(P.ModelShape(1, hkv * g, hkv, d), cfg)
    db.import_context(tok, keys, vals)
    s, _ = db.create_session(tok)
    q = (centers[:hkv * g] + 0.1).astype(np.float32)
    out = s.attention(q, 0)
    kept, total = next(iter(db._calls.values()))[1].block_stats()
    assert kept == total
    ref, _, _ = O.session_attention_flat(q, keys[0], vals[0], None, None, 110.0)
    assert rel(out, ref) <= 1e-5


@pytest.mark.parametrize("ordered,beta,want", [(True, 20.0, True), (True, 110.0, False),
                                               (False, 20.0, False)])
def test_auto_filter_decision(cuda_ok, ordered, beta, want):
    """block_filter="auto" (the default): on only for a context whose 128-key blocks
    are tight (locality) at a beta small enough for their bounds to prune; results
    equal the oracle either way."""
    import paper_2504_10326_b200 as P
    n, hkv, g, d = 20000, 2, 4, 128
    if ordered:
        keys, vals, centers = locality_context(n, hkv, d, seed=7)
        tok = np.arange(n)
    else:
        tok, keys, vals, centers, _ = O.make_context(n, 1, hkv, d, seed=7)
    keys, vals = O.bf16_round(keys), O.bf16_round(vals)
    cfg = P.EngineConfig(beta=beta, first_layers=(0,), short_context_threshold=0,
                         kv_dtype="bfloat16")
    assert cfg.block_filter == "auto"
    db = P.ContextStore(P.ModelShape(1, hkv * g, hkv, d), cfg)
    db.import_context(tok, keys, vals)
    s, _ = db.create_session(tok)
    assert db._filter_for([s], 0, beta) is want
    q = (centers[:hkv * g] + 0.1).astype(np.float32)
    out = s.attention(q, 0)
    call = next(iter(db._calls.values()))[1]
    assert bool(call.params.block_filter) is want
    if want:
        kept, total = call.block_stats()
        assert kept < total
    ref, _, _ = O.session_attention_flat(q, keys[0], vals[0], None, None, beta)
    assert rel(out, ref) <= 1e-5
