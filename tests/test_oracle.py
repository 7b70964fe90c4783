"""Pin the CPU oracle against the real reference's golden fixtures (CPU only)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import alaya_oracle as O
from tests.golden_cases import GOLDEN, SESSION_CASES, TOPK_CASES, load_session_case, window_rows


def test_known_answer_hand_case():
    z = np.load(GOLDEN / "known_answers.npz")
    got = sorted(O.dipr_bruteforce(z["hand_q"], z["hand_k"], 1.0))
    assert got == z["hand_out"].tolist() == [0, 1]


def test_known_answer_beta_ladder():
    z = np.load(GOLDEN / "known_answers.npz")
    off = z["rand_off"]
    for i, b in enumerate(z["rand_betas"]):
        want = z["rand_sel"][off[i]:off[i + 1]].tolist()
        assert sorted(O.dipr_bruteforce(z["rand_q"], z["rand_k"], float(b))) == want


def test_known_answer_windows():
    z = np.load(GOLDEN / "known_answers.npz")["windows"]
    i = 0
    while i < z.size:
        p, ini, last, m = (int(x) for x in z[i:i + 4])
        want = z[i + 4:i + 4 + m]
        assert np.array_equal(O.window_base_ids(p, ini, last), want)
        i += 4 + m


def test_dipr_errors():
    with pytest.raises(ValueError):
        O.dipr_bruteforce(np.ones(3, np.float32), np.empty((0, 3), np.float32), 1.0)
    with pytest.raises(ValueError):
        O.dipr_bruteforce(np.ones(3, np.float32), np.ones((4, 3), np.float32), -0.1)


def test_alpha_beta():
    assert O.alpha_to_beta(1.0, 128) == 0.0
    assert O.alpha_to_beta(np.exp(-2.0), 64) == pytest.approx(16.0, rel=1e-12)
    with pytest.raises(ValueError):
        O.alpha_to_beta(0.0, 8)


@pytest.mark.parametrize("name", SESSION_CASES)
def test_session_attention_bit_exact_vs_reference(name):
    """The restatement reproduces ``Session.attention`` on the flat plan bit for bit."""
    c = load_session_case(name)
    for step in range(c.steps):
        for li, layer in enumerate(c.layers):
            wk, wv = window_rows(c, step, layer)
            out, sels, counts = O.session_attention_flat(
                c.q[step, layer], c.keys[layer], c.values[layer], wk, wv, c.beta,
                c.win_init, c.win_last)
            idx = c.call_index(step, li)
            assert np.array_equal(out, c.out[idx])
            for qh in range(c.hq):
                assert np.array_equal(sels[qh], c.selected(step, li, qh))
                assert counts[qh] == c.retrieved[idx * c.hq + qh]


def test_bf16_round_is_rne():
    x = np.array([1.0, 1.00390625, 1.0078125 + 2 ** -9, -3.5, 1e-40], dtype=np.float32)
    r = O.bf16_round(x)
    assert r[0] == 1.0 and r[1] == 1.0  # tie to even
    assert r[3] == -3.5
    import torch
    t = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(r, t)


def test_box_bound_is_sound(rng):
    keys = rng.standard_normal((1000, 32)).astype(np.float32)
    q = rng.standard_normal(32).astype(np.float32)
    lo, hi = O.block_box_bounds(keys, 128)
    ub = O.block_upper_bounds(q, lo, hi)
    s = O.inner_products(keys, q)
    for b in range(ub.size):
        assert s[b * 128:(b + 1) * 128].max() <= ub[b] + 1e-9


# --------------------------------------------------------------------------
# TOP_K plans (flat FlatIndex.top_k and the coarse BlockIndex)
# --------------------------------------------------------------------------

def test_topk_reference_hand_cases():
    """Known answers of the reference's tests/test_index.py:33-41,205-224."""
    q = np.array([1.0, 0.0], np.float32)
    assert O.flat_top_k(q, np.array([[3, 0], [1, 0], [2, 0]], np.float32), 2) == [0, 2]
    assert O.flat_top_k(q, np.array([[2, 0], [2, 0], [3, 0]], np.float32), 3) == [2, 0, 1]
    with pytest.raises(ValueError):
        O.flat_top_k(q, np.ones((4, 2), np.float32), 5)
    idx = O.build_block_index(np.array([[4.0], [1.0], [3.0], [2.0]], np.float32), 1, 1)
    assert idx.top_blocks(np.array([1.0], np.float32), 4) == [(0, 1), (2, 3), (3, 4), (1, 2)]
    idx = O.build_block_index(np.array([[2.0], [2.0], [1.0]], np.float32), 1, 1)
    assert idx.top_blocks(np.array([1.0], np.float32), 2) == [(0, 1), (1, 2)]
    keys = np.array([[1, 0], [1, 0], [0, 1], [0, 1]], np.float32)
    assert O.build_block_index(keys, 2, 1).top_blocks(q, 1) == [(0, 2)]


def test_topk_known_answers_vs_reference():
    z = np.load(GOLDEN / "topk_known_answers.npz")
    off = z["topk_off"]
    for i, k in enumerate(z["ks"]):
        assert O.flat_top_k(z["q"], z["k"], int(k)) == z["topk"][off[i]:off[i + 1]].tolist()
    t1, t2 = (int(x) for x in z["tie_k"])
    assert O.flat_top_k(z["q"], z["k"], t1) == z["tie_topk1"].tolist()
    assert O.flat_top_k(z["q"], z["k"], t2) == z["tie_topk2"].tolist()
    bi = O.build_block_index(z["k"], 64, 4)
    assert np.array_equal(np.concatenate(bi.reps), z["blk_reps"])
    boff = z["blk_off"]
    for i, kb in enumerate((1, 3, bi.n_blocks)):
        got = [s for s, _ in bi.top_blocks(z["q"], kb)]
        assert got == z["blk_top"][boff[i]:boff[i + 1]].tolist()


@pytest.mark.parametrize("name", TOPK_CASES)
def test_topk_session_bit_exact_vs_reference(name):
    c = load_session_case(name)
    k, bs, reps, coarse = c.topk
    for step in range(c.steps):
        for li, layer in enumerate(c.layers):
            wk, wv = window_rows(c, step, layer)
            out, sels, counts = O.session_attention_topk(
                c.q[step, layer], c.keys[layer], c.values[layer], wk, wv, k, bool(coarse), bs,
                reps, c.win_init, c.win_last)
            idx = c.call_index(step, li)
            assert np.array_equal(out, c.out[idx])
            for qh in range(c.hq):
                assert np.array_equal(sels[qh], c.selected(step, li, qh))
                assert counts[qh] == c.retrieved[idx * c.hq + qh]


# --------------------------------------------------------------------------
# graph DIPRS (dipr.py:107-289) on reference-built graphs
# --------------------------------------------------------------------------

def csr(degrees, flat):
    off = np.zeros(degrees.size + 1, np.int64)
    off[1:] = np.cumsum(degrees)
    return off, flat.astype(np.int64)


def test_diprs_restatement_vs_reference():
    z = np.load(GOLDEN / "graph_diprs.npz")
    keys, q = z["keys"], z["q"]
    off, nb = csr(z["degrees"], z["nbrs"])
    smax = (keys.astype(np.float64) @ q.astype(np.float64).T).max(axis=0)
    so = z["sel_off"]
    i = 0
    for beta, l0, wo in z["runs"]:
        for j in range(q.shape[0]):
            wm = None if np.isnan(wo) else float(smax[j] + wo)
            got = sorted(O.diprs(keys, off, nb, q[j], int(z["entry"]), int(l0), float(beta), wm))
            assert got == z["sel"][so[i]:so[i + 1]].tolist(), (beta, l0, wo, j)
            i += 1


def test_diprs_complete_graph_is_exact(rng):
    """reference tests/test_dipr.py:184-190: a complete graph gives the brute-force set."""
    keys = rng.integers(-5, 6, size=(12, 4)).astype(np.float32)
    q = rng.integers(-5, 6, size=4).astype(np.float32)
    nb = np.concatenate([[v for v in range(12) if v != u] for u in range(12)])
    off = np.arange(0, 12 * 11 + 1, 11)
    for beta in (0.0, 2.0, 10.0):
        assert O.diprs(keys, off, nb, q, 0, 16, beta) == O.dipr_bruteforce(q, keys, beta)


def test_package_alpha_to_beta_matches_oracle():
    """The package's host formula (dipr.py:29-39) against the pinned oracle's copy."""
    from paper_2504_10326_b200 import dipr as D
    for alpha, d in ((1.0, 128), (np.exp(-2.0), 64), (0.05, 128), (1e-6, 16)):
        assert D.alpha_to_beta(alpha, d) == pytest.approx(O.alpha_to_beta(alpha, d), rel=1e-15)
    for bad in ((0.0, 8), (1.5, 8), (0.5, 0)):
        with pytest.raises(ValueError):
            D.alpha_to_beta(*bad)


def test_engine_config_block_filter_modes():
    from paper_2504_10326_b200.config import EngineConfig
    assert EngineConfig().block_filter == "auto"
    for v in (True, False, "auto"):
        assert EngineConfig(block_filter=v).block_filter == v
    with pytest.raises(ValueError):
        EngineConfig(block_filter="sometimes")
