"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle / golden
fixtures from the real reference.

Rules (BASELINE.json north_star):
  * sets: identical except tokens with |s_j - (s_max - beta)| <= EPS_SET
    (fp64 scores on the same, possibly bf16-rounded, inputs);
  * outputs: norm-relative error <= 1e-5 (fp32 KV) / 2e-2 (bf16 KV), with
    the oracle evaluated on the GPU-returned selection so that a legitimate
    epsilon-boundary flip is not counted as an arithmetic error.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import alaya_oracle as O
from tests.golden_cases import SESSION_CASES, load_session_case, window_rows

pytestmark = pytest.mark.gpu

EPS_SET = {"float32": 1e-4, "bfloat16": 1e-3}
TOL_OUT = {"float32": 1e-5, "bfloat16": 2e-2}


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


def boundary_ok(got, want, q, keys, beta, eps):
    """Set equality up to tokens within eps of the threshold."""
    got, want = set(int(x) for x in got), set(int(x) for x in want)
    diff = got ^ want
    if not diff:
        return True
    s = O.inner_products(keys, q)
    thr = s.max() - beta
    return all(abs(s[t] - thr) <= eps for t in diff)


def make_store(case, kv_dtype, **kw):
    import paper_2504_10326_b200 as P
    shape = P.ModelShape(case.n_layers, case.hq, case.hkv, case.d)
    cfg = P.EngineConfig(beta=case.beta, window_initial=case.win_init, window_last=case.win_last,
                         first_layers=tuple(range(case.n_layers)), short_context_threshold=0,
                         kv_dtype=kv_dtype, **kw)
    return P, P.ContextStore(shape, cfg)


@pytest.mark.parametrize("name", SESSION_CASES)
def test_session_attention_matches_reference(cuda_ok, name):
    c = load_session_case(name)
    kv_dtype = "bfloat16" if c.bf16 else "float32"
    P, db = make_store(c, kv_dtype)
    tokens = np.arange(c.n, dtype=np.int64) + 7
    db.import_context(tokens, c.keys, c.values)
    sess, _ = db.create_session(tokens)
    worst = 0.0
    for step in range(c.steps):
        for layer in range(c.n_layers):
            sess.update(c.q[step, layer], c.k[step, layer], c.v[step, layer], layer)
        for li, layer in enumerate(c.layers):
            out = sess.attention(c.q[step, layer], layer)
            diag = sess.last_diagnostics
            assert diag["layer"] == layer and diag["plan"].query is P.QueryKind.DIPR
            idx = c.call_index(step, li)
            wk, wv = window_rows(c, step, layer)
            for qh in range(c.hq):
                h = qh // (c.hq // c.hkv)
                info = diag["heads"][qh]
                want_sel = c.selected(step, li, qh)
                assert boundary_ok(info["selected_base"], want_sel, c.q[step, layer, qh],
                                   c.keys[layer, h], c.beta, EPS_SET[kv_dtype]), (step, layer, qh)
                assert abs(info["retrieved"] - c.retrieved[idx * c.hq + qh]) <= \
                    len(set(info["selected_base"]) ^ set(want_sel.tolist()))
                # oracle on the GPU's own selection (fp64 arithmetic of the reference)
                o_ref, _, _ = O.head_attention_flat(
                    c.q[step, layer, qh], c.keys[layer, h], c.values[layer, h], wk[h], wv[h],
                    c.beta, c.win_init, c.win_last, selected_override=info["selected_base"])
                e = rel(out[qh], o_ref)
                worst = max(worst, e)
                assert e <= TOL_OUT[kv_dtype], (step, layer, qh, e)
                if np.array_equal(info["selected_base"], want_sel):
                    assert rel(out[qh], c.out[idx, qh]) <= TOL_OUT[kv_dtype]
    print(f"{name}: worst norm-relative error {worst:.2e}")


def test_dipr_bruteforce_known_answers(cuda_ok):
    import paper_2504_10326_b200 as P
    from tests.golden_cases import GOLDEN
    z = np.load(GOLDEN / "known_answers.npz")
    # hand case (reference tests/test_dipr.py:69-72) needs d >= 16: pad with zeros
    q = np.zeros(16, np.float32); q[:2] = z["hand_q"]
    k = np.zeros((3, 16), np.float32); k[:, :2] = z["hand_k"]
    assert sorted(P.dipr_bruteforce(q, k, 1.0)) == z["hand_out"].tolist()
    off = z["rand_off"]
    for i, b in enumerate(z["rand_betas"]):
        want = z["rand_sel"][off[i]:off[i + 1]]
        got = sorted(P.dipr_bruteforce(z["rand_q"], z["rand_k"], float(b)))
        assert boundary_ok(got, want, z["rand_q"], z["rand_k"], float(b), 1e-4), b


def test_dipr_edge_cases(cuda_ok, rng):
    import paper_2504_10326_b200 as P
    keys = rng.standard_normal((20, 16)).astype(np.float32)
    q = rng.standard_normal(16).astype(np.float32)
    s = O.inner_products(keys, q)
    assert P.dipr_bruteforce(q, keys, 0.0) == {int(np.argmax(s))}
    assert P.dipr_bruteforce(q, keys, float(s.max() - s.min()) + 1) == set(range(20))
    with pytest.raises(ValueError):
        P.dipr_bruteforce(q, np.empty((0, 16), np.float32), 1.0)
    with pytest.raises(ValueError):
        P.dipr_bruteforce(q, keys, -0.1)
    perm = rng.permutation(20)
    assert P.dipr_bruteforce(q, keys[perm], 2.0, token_ids=perm) == P.dipr_bruteforce(q, keys, 2.0)
    # monotone in beta (reference tests/test_dipr.py:91-98)
    prev = set()
    for b in [0.0, 0.5, 1.0, 2.0, 5.0, 100.0]:
        cur = P.dipr_bruteforce(q, keys, b)
        assert prev <= cur
        prev = cur


@pytest.mark.parametrize("n", [1, 255, 256, 257, 2047, 5000, 70001])
def test_dipr_ragged_sizes(cuda_ok, n):
    import paper_2504_10326_b200 as P
    r = np.random.default_rng(n)
    keys = r.standard_normal((n, 128)).astype(np.float32) * 2
    q = r.standard_normal(128).astype(np.float32) * 2
    for beta in (3.0, 30.0):
        got = P.dipr_bruteforce(q, keys, beta)
        want = O.dipr_bruteforce(q, keys, beta)
        assert boundary_ok(got, want, q, keys, beta, 1e-4)


def test_full_and_partial_attention(cuda_ok, rng):
    import paper_2504_10326_b200 as P
    keys = rng.standard_normal((300, 64)).astype(np.float32)
    vals = rng.standard_normal((300, 64)).astype(np.float32)
    q = rng.standard_normal(64).astype(np.float32)
    ref = O.full_attention(q, keys, vals)
    assert rel(P.full_attention(q, keys, vals), ref) <= 1e-5
    # partition -> merge == single pass (reference tests/test_attention.py:162-174)
    parts = [P.PartialAttention.over(q, keys[a:b], vals[a:b]) for a, b in
             [(0, 10), (10, 11), (11, 200), (200, 300)]]
    acc = P.PartialAttention.empty()
    for p in parts:
        acc = acc.merge(p)
    assert rel(acc.finalize(), ref) <= 1e-5
    assert P.PartialAttention.over(q, keys[:0], vals[:0]).is_empty
    with pytest.raises(ValueError):
        P.PartialAttention.empty().finalize()
    # singleton returns its value (tests/test_attention.py:28-31)
    assert rel(P.full_attention(q, keys[:1], vals[:1]), vals[0]) <= 1e-6


def test_session_edge_cases(cuda_ok):
    import paper_2504_10326_b200 as P
    shape = P.ModelShape(2, 4, 2, 16)
    cfg = P.EngineConfig(window_initial=4, window_last=8, beta=8.0, short_context_threshold=64)
    db = P.ContextStore(shape, cfg)
    # single-token session returns v (reference tests/test_store.py:203-214)
    sess, _ = db.create_session([5])
    r = np.random.default_rng(0)
    q = r.standard_normal((4, 16)).astype(np.float32)
    k = r.standard_normal((2, 16)).astype(np.float32)
    v = r.standard_normal((2, 16)).astype(np.float32)
    sess.update(q, k, v, 0)
    sess.update(q, k, v, 1)
    out = sess.attention(q, 0)
    for qh in range(4):
        assert np.allclose(out[qh], v[shape.kv_head_of(qh)], atol=1e-6)
    # empty session (tests/test_store.py:216-221)
    sess2, _ = db.create_session([1, 2])
    with pytest.raises(ValueError):
        sess2.attention(np.zeros((4, 16), np.float32), 0)
    with pytest.raises(ValueError):
        sess.attention(np.zeros((3, 16), np.float32), 0)
    with pytest.raises(ValueError):
        sess.attention(q, 5)


def test_full_plan_and_huge_beta_equal_full_attention(cuda_ok):
    """tests/test_store.py:184-201 on the GPU engine."""
    import paper_2504_10326_b200 as P
    c = load_session_case("tiny_gqa")
    shape = P.ModelShape(c.n_layers, c.hq, c.hkv, c.d)
    db = P.ContextStore(shape, P.EngineConfig(window_initial=4, window_last=8, beta=8.0,
                                              short_context_threshold=64))
    tokens = np.arange(c.n)
    db.import_context(tokens, c.keys, c.values)
    sess, _ = db.create_session(tokens)
    for layer in range(c.n_layers):
        sess.update(c.q[0, layer], c.k[0, layer], c.v[0, layer], layer)
    q = c.q[0, 1]
    sess.plan_override = P.Plan(P.QueryKind.FULL_ATTENTION, P.IndexKind.NONE)
    full = sess.attention(q, 1)
    for qh in range(c.hq):
        h = qh // (c.hq // c.hkv)
        keys = np.concatenate([c.keys[1, h], c.k[:1, 1, h]])
        vals = np.concatenate([c.values[1, h], c.v[:1, 1, h]])
        assert rel(full[qh], O.full_attention(q[qh], keys, vals)) <= 1e-5
    sess.plan_override = P.Plan(P.QueryKind.DIPR, P.IndexKind.FINE, beta=1e9)
    sparse = sess.attention(q, 1)
    assert np.allclose(full, sparse, atol=1e-5)


def test_batched_sessions_ragged(cuda_ok):
    """attention_batch over sessions with different prefix/window lengths."""
    import paper_2504_10326_b200 as P
    r = np.random.default_rng(7)
    shape = P.ModelShape(1, 8, 2, 128)
    cfg = P.EngineConfig(beta=40.0, first_layers=(0,), short_context_threshold=0,
                         kv_dtype="bfloat16")
    db = P.ContextStore(shape, cfg)
    sessions, data = [], []
    for i, n in enumerate([100, 1000, 3333, 9000]):
        tok, keys, vals, centers, _ = O.make_context(n, 1, 2, 128, seed=10 + i)
        keys, vals = O.bf16_round(keys), O.bf16_round(vals)
        db.import_context(tok, keys, vals)
        s, _ = db.create_session(tok)
        for _ in range(i):  # different window lengths
            kk = O.bf16_round(r.standard_normal((2, 128)).astype(np.float32))
            vv = O.bf16_round(r.standard_normal((2, 128)).astype(np.float32))
            s.update(r.standard_normal((8, 128)).astype(np.float32), kk, vv, 0)
        sessions.append(s)
        data.append((keys, vals))
    q = (np.stack([O.make_context(10, 1, 1, 128, seed=99)[3][r.integers(0, 16, 8)]
                   for _ in sessions]) + 0.25 * r.standard_normal((4, 8, 128))).astype(np.float32)
    out = P.Session.attention_batch(sessions, q, 0)
    for b, s in enumerate(sessions):
        keys, vals = data[b]
        wk = s._wk[0, :, : s._wlen[0]].float().cpu().numpy() if s._wlen[0] else np.zeros((2, 0, 128), np.float32)
        wv = s._wv[0, :, : s._wlen[0]].float().cpu().numpy() if s._wlen[0] else np.zeros((2, 0, 128), np.float32)
        ref, sels, _ = O.session_attention_flat(q[b], keys[0], vals[0], wk, wv, 40.0)
        for qh in range(8):
            assert rel(out[b, qh], ref[qh]) <= 2e-2


def test_bf16_and_fp32_paths_agree_on_bf16_data(cuda_ok):
    """Same bf16-representable data through the fp32 and bf16 kernels."""
    import paper_2504_10326_b200 as P
    c = load_session_case("llama_4k_bf16")
    outs = []
    for kv in ("float32", "bfloat16"):
        _, db = make_store(c, kv)
        tokens = np.arange(c.n)
        db.import_context(tokens, c.keys, c.values)
        s, _ = db.create_session(tokens)
        s.update(c.q[0, 0], c.k[0, 0], c.v[0, 0], 0)
        outs.append(s.attention(c.q[0, 0], 0))
    assert rel(outs[0], outs[1].astype(np.float64)) <= 1e-5


@pytest.mark.parametrize("scan", ["tcgen05", "cuda_core"])
@pytest.mark.parametrize("g,n,beta", [(1, 1000, 20.0), (2, 4097, 110.0), (4, 70001, 110.0),
                                      (5, 33333, 50.0), (8, 5000, 110.0), (4, 300, 1e9)])
def test_bf16_scan_kernels_vs_oracle(cuda_ok, scan, g, n, beta):
    """Both scan kernels on bf16 K/V (Llama/Qwen-like groups, ragged lengths) vs
    the fp64 oracle on the same bf16-rounded inputs."""
    import paper_2504_10326_b200 as P
    hkv, d = 2, 128
    shape = P.ModelShape(1, hkv * g, hkv, d)
    cfg = P.EngineConfig(beta=beta, first_layers=(0,), short_context_threshold=0,
                         kv_dtype="bfloat16", scan_kernel=scan)
    db = P.ContextStore(shape, cfg)
    tok, keys, vals, centers, _ = O.make_context(n, 1, hkv, d, seed=n + g)
    keys, vals = O.bf16_round(keys), O.bf16_round(vals)
    db.import_context(tok, keys, vals)
    s, _ = db.create_session(tok)
    r = np.random.default_rng(g)
    q = (centers[r.integers(0, 16, hkv * g)] + 0.25 * r.standard_normal((hkv * g, d))).astype(np.float32)
    kk = O.bf16_round(r.standard_normal((hkv, d)).astype(np.float32))
    vv = O.bf16_round(r.standard_normal((hkv, d)).astype(np.float32))
    s.update(q, kk, vv, 0)
    out = s.attention(q, 0)
    diag = s.last_diagnostics
    ref, sels, cnts = O.session_attention_flat(q, keys[0], vals[0], kk[:, None], vv[:, None], beta)
    for qh in range(hkv * g):
        h = qh // g
        got = diag["heads"][qh]["selected_base"]
        assert boundary_ok(got, sels[qh], q[qh], keys[0, h], beta, EPS_SET["bfloat16"]), qh
        o_ref, _, _ = O.head_attention_flat(q[qh], keys[0, h], vals[0, h], kk[h][None], vv[h][None],
                                            beta, selected_override=got)
        assert rel(out[qh], o_ref) <= 1e-5, (qh, rel(out[qh], o_ref))


def test_tcgen05_multi_context_batch(cuda_ok):
    """Sessions on different contexts (one TMA map each) and prefix reuse (head
    stride > prefix) in one tcgen05 launch."""
    import paper_2504_10326_b200 as P
    shape = P.ModelShape(1, 8, 2, 128)
    cfg = P.EngineConfig(beta=110.0, first_layers=(0,), short_context_threshold=0,
                         kv_dtype="bfloat16", scan_kernel="tcgen05")
    db = P.ContextStore(shape, cfg)
    sessions, data = [], []
    for i, n in enumerate([2000, 9999, 4096]):
        tok, keys, vals, centers, _ = O.make_context(n, 1, 2, 128, seed=40 + i)
        keys, vals = O.bf16_round(keys), O.bf16_round(vals)
        db.import_context(tok, keys, vals)
        reuse = tok if i != 1 else tok[:7777]  # partial prefix reuse on context 1
        s, _ = db.create_session(reuse)
        p = s.reused_prefix_len
        s.plan_override = P.Plan(P.QueryKind.DIPR, P.IndexKind.FLAT, beta=110.0)
        sessions.append(s)
        data.append((keys[0, :, :p], vals[0, :, :p], centers))
    r = np.random.default_rng(3)
    q = np.stack([(c[r.integers(0, 16, 8)] + 0.25 * r.standard_normal((8, 128))) for _, _, c in data]
                 ).astype(np.float32)
    out = P.Session.attention_batch(sessions, q, 0)
    for b, (keys, vals, _) in enumerate(data):
        ref, sels, _ = O.session_attention_flat(q[b], keys, vals, None, None, 110.0)
        diag = sessions[b].last_diagnostics
        for qh in range(8):
            got = diag["heads"][qh]["selected_base"]
            assert boundary_ok(got, sels[qh], q[b, qh], keys[qh // 4], 110.0, 1e-3)
            o_ref, _, _ = O.head_attention_flat(q[b, qh], keys[qh // 4], vals[qh // 4], None, None,
                                                110.0, selected_override=got)
            assert rel(out[b, qh], o_ref) <= 1e-5


def test_overlapped_attend_path_batch(cuda_ok):
    """>= 32 (session, kv head) groups: the default path runs the attend beside
    the tcgen05 scan (per-group readiness counters). Ragged Llama-shaped
    sessions with windows vs the fp64 oracle on the GPU's own selection."""
    import paper_2504_10326_b200 as P
    hq, hkv, d, beta = 32, 8, 128, 110.0
    shape = P.ModelShape(1, hq, hkv, d)
    cfg = P.EngineConfig(beta=beta, first_layers=(0,), short_context_threshold=0,
                         kv_dtype="bfloat16")
    db = P.ContextStore(shape, cfg)
    r = np.random.default_rng(11)
    sessions, data = [], []
    for i, n in enumerate([3000, 40000, 70001, 5000]):
        tok, keys, vals, centers, _ = O.make_context(n, 1, hkv, d, seed=70 + i)
        keys, vals = O.bf16_round(keys), O.bf16_round(vals)
        db.import_context(tok, keys, vals)
        s, _ = db.create_session(tok)
        for _ in range(i + 1):
            kk = O.bf16_round(r.standard_normal((hkv, d)).astype(np.float32))
            vv = O.bf16_round(r.standard_normal((hkv, d)).astype(np.float32))
            s.update(r.standard_normal((hq, d)).astype(np.float32), kk, vv, 0)
        sessions.append(s)
        data.append((keys[0], vals[0], centers))
    q = np.stack([(c[r.integers(0, 16, hq)] + 0.25 * r.standard_normal((hq, d)))
                  for _, _, c in data]).astype(np.float32)
    for rep in range(2):  # twice: the workspace header must be fully re-seeded per call
        out = P.Session.attention_batch(sessions, q, 0)
        for b, s in enumerate(sessions):
            keys, vals, _ = data[b]
            w = s._wlen[0]
            wk = s._wk[0, :, :w].float().cpu().numpy()
            wv = s._wv[0, :, :w].float().cpu().numpy()
            ref, sels, _ = O.session_attention_flat(q[b], keys, vals, wk, wv, beta)
            diag = s.last_diagnostics
            for qh in range(hq):
                h = qh // (hq // hkv)
                got = diag["heads"][qh]["selected_base"]
                assert boundary_ok(got, sels[qh], q[b, qh], keys[h], beta, EPS_SET["bfloat16"])
                o_ref, _, _ = O.head_attention_flat(q[b, qh], keys[h], vals[h], wk[h], wv[h], beta,
                                                    selected_override=got)
                assert rel(out[b, qh], o_ref) <= 1e-5, (rep, b, qh)
