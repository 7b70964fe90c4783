"""Randomised GPU parity sweep (fixed seeds): shapes, GQA groups, head dims,
dtypes, betas (0 .. inf), window configurations, session-window rows, batch
sizes and prefix reuse, each through Session.attention_batch (the C-ABI path)
against the fp64 oracle evaluated on the GPU's own selection, plus the set
rule of SURVEY §8c."""

from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import alaya_oracle as O

pytestmark = pytest.mark.gpu

EPS = {"float32": 1e-4, "bfloat16": 1e-3}


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.parametrize("seed", range(24))
def test_random_configurations(cuda_ok, seed):
    import paper_2504_10326_b200 as P
    r = np.random.default_rng(1000 + seed)
    hkv = int(r.choice([1, 2, 4, 8]))
    g = int(r.integers(1, 9))
    d = int(r.choice([16, 32, 64, 128, 128, 128, 256]))
    kv = str(r.choice(["float32", "bfloat16"]))
    B = int(r.integers(1, 5))
    beta = float(r.choice([0.0, 0.5, 5.0, 30.0, 110.0, math.inf]))
    wi, wl = int(r.integers(0, 20)), int(r.integers(0, 70))
    scan = str(r.choice(["auto", "cuda_core"]))
    shape = P.ModelShape(1, hkv * g, hkv, d)
    cfg = P.EngineConfig(beta=min(beta, 1e30), window_initial=wi, window_last=wl,
                         first_layers=(0,), short_context_threshold=0, kv_dtype=kv,
                         scan_kernel=scan)
    db = P.ContextStore(shape, cfg)
    sessions, data = [], []
    for b in range(B):
        n = int(r.integers(1, 20000))
        tok, keys, vals, centers, _ = O.make_context(n, 1, hkv, d, clusters=int(r.integers(2, 17)),
                                                     seed=seed * 10 + b)
        if kv == "bfloat16":
            keys, vals = O.bf16_round(keys), O.bf16_round(vals)
        tok = tok + 100000 * (seed * 10 + b)  # distinct contexts
        db.import_context(tok, keys, vals)
        reuse = tok if r.random() < 0.7 else tok[: max(1, int(n * r.random()))]
        s, _ = db.create_session(reuse)
        p = s.reused_prefix_len
        s.plan_override = P.Plan(P.QueryKind.DIPR, P.IndexKind.FLAT, beta=min(beta, 1e30))
        for _ in range(int(r.integers(0, 4))):  # session-window rows
            kk = r.standard_normal((hkv, d)).astype(np.float32)
            vv = r.standard_normal((hkv, d)).astype(np.float32)
            if kv == "bfloat16":
                kk, vv = O.bf16_round(kk), O.bf16_round(vv)
            s.update(r.standard_normal((hkv * g, d)).astype(np.float32), kk, vv, 0)
        sessions.append(s)
        data.append((keys[0, :, :p], vals[0, :, :p], centers))
    q = np.stack([(c[r.integers(0, c.shape[0], hkv * g)] + 0.25 * r.standard_normal((hkv * g, d)))
                  for _, _, c in data]).astype(np.float32)
    out = P.Session.attention_batch(sessions, q, 0)
    for b, s in enumerate(sessions):
        keys, vals, _ = data[b]
        w = s._wlen[0]
        wk = s._wk[0, :, :w].float().cpu().numpy() if w else None
        wv = s._wv[0, :, :w].float().cpu().numpy() if w else None
        diag = s.last_diagnostics
        for qh in range(hkv * g):
            h = qh // g
            got = diag["heads"][qh]["selected_base"]
            _, want, _ = O.head_attention_flat(q[b, qh], keys[h], vals[h],
                                               None if wk is None else wk[h],
                                               None if wv is None else wv[h], min(beta, 1e300), wi, wl)
            diff = set(got) ^ set(want.tolist())
            if diff:
                sc = O.inner_products(keys[h], q[b, qh])
                thr = sc.max() - beta
                assert all(abs(sc[t] - thr) <= EPS[kv] for t in diff), (seed, b, qh)
            o_ref, _, _ = O.head_attention_flat(q[b, qh], keys[h], vals[h],
                                                None if wk is None else wk[h],
                                                None if wv is None else wv[h], min(beta, 1e300),
                                                wi, wl, selected_override=got)
            assert rel(out[b, qh], o_ref) <= 1e-5, (seed, b, qh, rel(out[b, qh], o_ref))


@pytest.mark.parametrize("seed", range(12))
def test_random_topk_plans(cuda_ok, seed):
    """TOP_K over the flat index and over the coarse block index, random k /
    block sizes / representatives / shapes, vs the restated reference."""
    import paper_2504_10326_b200 as P
    r = np.random.default_rng(5000 + seed)
    hkv, g = int(r.choice([1, 2, 8])), int(r.integers(1, 6))
    d = int(r.choice([32, 64, 128]))
    n = int(r.integers(50, 9000))
    k = int(r.choice([1, 7, 100, 333, 2500]))
    coarse = bool(r.random() < 0.5)
    bs, reps = int(r.choice([16, 64, 128])), int(r.integers(1, 5))
    wi, wl = int(r.integers(0, 10)), int(r.integers(0, 40))
    shape = P.ModelShape(1, hkv * g, hkv, d)
    common = dict(window_initial=wi, window_last=wl, short_context_threshold=0, first_layers=(0,),
                  top_k=k)
    cfg = (P.EngineConfig(memory_budget_bytes=10**12, block_size=bs, representatives=reps, **common)
           if coarse else P.EngineConfig(**common))
    db = P.ContextStore(shape, cfg)
    tok, keys, vals, centers, _ = O.make_context(n, 1, hkv, d, seed=seed)
    db.import_context(tok, keys, vals)
    s, _ = db.create_session(tok)
    if not coarse:
        s.plan_override = P.Plan(P.QueryKind.TOP_K, P.IndexKind.FLAT, k=k)
    kk = r.standard_normal((hkv, d)).astype(np.float32)
    vv = r.standard_normal((hkv, d)).astype(np.float32)
    s.update(r.standard_normal((hkv * g, d)).astype(np.float32), kk, vv, 0)
    q = (centers[r.integers(0, 16, hkv * g)] + 0.25 * r.standard_normal((hkv * g, d))).astype(np.float32)
    out = s.attention(q, 0)
    diag = s.last_diagnostics
    assert diag["plan"].query is P.QueryKind.TOP_K
    for qh in range(hkv * g):
        h = qh // g
        got = np.asarray(diag["heads"][qh]["selected_base"], np.int64)
        if coarse:
            bi = O.build_block_index(keys[0, h], bs, reps)
            want_ret = O.retrieve_top_k_coarse(q[qh], bi, k, n)
        else:
            want_ret = O.retrieve_top_k_flat(q[qh], keys[0, h], k)
        want = np.setdiff1d(np.fromiter(want_ret, np.int64), O.window_base_ids(n, wi, wl))
        if not np.array_equal(np.sort(got), want):
            sc = bi.block_scores(q[qh]) if coarse else O.inner_products(keys[0, h], q[qh])
            kth = np.sort(sc)[::-1][min(max(1, -(-k // bs)) if coarse else k, sc.size) - 1]
            flips = ({int(t) // bs for t in set(got.tolist()) ^ set(want.tolist())} if coarse
                     else set(got.tolist()) ^ set(want.tolist()))
            assert all(abs(sc[t] - kth) <= 1e-4 for t in flips), (seed, qh)
        o_ref, _, _ = O.head_attention_retrieved(q[qh], keys[0, h], vals[0, h], kk[h][None],
                                                 vv[h][None], got, wi, wl)
        assert rel(out[qh], o_ref) <= 1e-5, (seed, qh)
