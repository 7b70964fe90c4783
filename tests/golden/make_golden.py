"""Generate golden fixtures from the REAL reference (``sparsekv``).

Run in the build container, where ``/root/reference`` exists:

    python tests/golden/make_golden.py

It imports the unmodified reference from ``/root/reference/pkg/src`` and
drives its public API (``ContextStore`` / ``Session.update`` /
``Session.attention`` on the DIPR/FLAT plan, ``dipr_bruteforce``,
``WindowConfig``, ``workload``). Outputs go to ``tests/golden/*.npz``; the
GPU box never reads ``/root/reference`` -- only these committed fixtures.
Large inputs are NOT stored: the reference generator is pinned by a sha256
of its arrays, and the tests regenerate them with the restated generator in
``oracle/alaya_oracle.py`` and check the hash first.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(OUT.parents[1]))

from sparsekv import (  # noqa: E402
    ContextStore, EngineConfig, ModelShape, WindowConfig, dipr_bruteforce,
)
from sparsekv.workload import WorkloadSpec, decode_step_inputs, make_context  # noqa: E402

from oracle.alaya_oracle import bf16_round  # noqa: E402


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def flat_session_case(name, n_layers, hq, hkv, d, n, steps, seed, beta, win_init, win_last,
                      clusters=16, bf16=False, store_inputs=False, layers_checked=None):
    """Drive the reference session API on the DIPR/FLAT plan and record it."""
    shape = ModelShape(n_layers, hq, hkv, d)
    cfg = EngineConfig(beta=beta, window_initial=win_init, window_last=win_last,
                       first_layers=tuple(range(n_layers)), short_context_threshold=0)
    spec = WorkloadSpec(n_tokens=n, shape=shape, seed=seed, clusters=clusters)
    ctx = make_context(spec)
    keys, values = ctx.keys, ctx.values
    gen_hash = sha(ctx.token_ids, keys, values, ctx.centers)
    if bf16:
        keys, values = bf16_round(keys), bf16_round(values)
    tids, qs, ks, vs = decode_step_inputs(spec, steps, ctx.centers)
    step_hash = sha(tids, qs, ks, vs)
    if bf16:
        ks, vs = bf16_round(ks), bf16_round(vs)
    db = ContextStore(shape, cfg)
    db.import_context(ctx.token_ids, keys, values)
    session, _ = db.create_session(ctx.token_ids)
    layers_checked = list(range(n_layers)) if layers_checked is None else layers_checked
    rec = {"shape": np.array([n_layers, hq, hkv, d, n, steps, seed, clusters]),
           "beta": np.float64(beta), "window": np.array([win_init, win_last]),
           "bf16": np.int64(bf16), "layers": np.array(layers_checked)}
    outs, sel_flat, sel_off, retrieved = [], [], [0], []
    for step in range(steps):
        for layer in range(n_layers):
            session.update(qs[step, layer], ks[step, layer], vs[step, layer], layer)
        session.record_token(int(tids[step]))
        for layer in layers_checked:
            assert session.active_plan(layer).query.value == "dipr"
            assert session.active_plan(layer).index.value == "flat"
            o = session.attention(qs[step, layer], layer)
            outs.append(o)
            for info in session.last_diagnostics["heads"]:
                sel_flat.extend(info["selected_base"])
                sel_off.append(len(sel_flat))
                retrieved.append(info["retrieved"])
    rec.update(out=np.stack(outs), sel=np.array(sel_flat, dtype=np.int32),
               sel_off=np.array(sel_off, dtype=np.int64),
               retrieved=np.array(retrieved, dtype=np.int64))
    rec["gen_sha"] = np.array(gen_hash)
    rec["step_sha"] = np.array(step_hash)
    if store_inputs:
        rec.update(keys=keys, values=values, q=qs, k=ks, v=vs)
    np.savez_compressed(OUT / f"{name}.npz", **rec)
    print(name, "out", rec["out"].shape, "sel", rec["sel"].size)


def topk_session_case(name, mode, k, n_layers, hq, hkv, d, n, steps, seed, win_init, win_last,
                      clusters=16, block_size=128, reps=4, store_inputs=False):
    """Drive the reference session API on a TOP_K plan and record it: mode
    "flat" = Plan(TOP_K, FLAT, k) over the FlatIndex (store.py:314-318), mode
    "coarse" = the planner's TOP_K/COARSE plan from a large memory budget
    (planner.py:113-115) over BlockIndex(block_size, reps) (store.py:305-312)."""
    from sparsekv.planner import IndexKind, Plan, QueryKind
    shape = ModelShape(n_layers, hq, hkv, d)
    common = dict(window_initial=win_init, window_last=win_last, short_context_threshold=0,
                  first_layers=tuple(range(n_layers)), top_k=k)
    if mode == "coarse":
        cfg = EngineConfig(memory_budget_bytes=10**12, block_size=block_size,
                           representatives=reps, **common)
    else:
        cfg = EngineConfig(**common)
    spec = WorkloadSpec(n_tokens=n, shape=shape, seed=seed, clusters=clusters)
    ctx = make_context(spec)
    keys, values = ctx.keys, ctx.values
    gen_hash = sha(ctx.token_ids, keys, values, ctx.centers)
    tids, qs, ks, vs = decode_step_inputs(spec, steps, ctx.centers)
    step_hash = sha(tids, qs, ks, vs)
    db = ContextStore(shape, cfg)
    db.import_context(ctx.token_ids, keys, values)
    session, _ = db.create_session(ctx.token_ids)
    if mode == "flat":
        session.plan_override = Plan(QueryKind.TOP_K, IndexKind.FLAT, k=k)
    rec = {"shape": np.array([n_layers, hq, hkv, d, n, steps, seed, clusters]),
           "beta": np.float64(0.0), "window": np.array([win_init, win_last]),
           "bf16": np.int64(0), "layers": np.arange(n_layers),
           "topk": np.array([k, block_size, reps, 1 if mode == "coarse" else 0])}
    outs, sel_flat, sel_off, retrieved = [], [], [0], []
    for step in range(steps):
        for layer in range(n_layers):
            session.update(qs[step, layer], ks[step, layer], vs[step, layer], layer)
        session.record_token(int(tids[step]))
        for layer in range(n_layers):
            plan = session.active_plan(layer)
            assert plan.query is QueryKind.TOP_K
            assert plan.index is (IndexKind.COARSE if mode == "coarse" else IndexKind.FLAT)
            o = session.attention(qs[step, layer], layer)
            outs.append(o)
            for info in session.last_diagnostics["heads"]:
                sel_flat.extend(info["selected_base"])
                sel_off.append(len(sel_flat))
                retrieved.append(info["retrieved"])
    rec.update(out=np.stack(outs), sel=np.array(sel_flat, dtype=np.int32),
               sel_off=np.array(sel_off, dtype=np.int64),
               retrieved=np.array(retrieved, dtype=np.int64))
    rec["gen_sha"] = np.array(gen_hash)
    rec["step_sha"] = np.array(step_hash)
    if store_inputs:
        rec.update(keys=keys, values=values, q=qs, k=ks, v=vs)
    np.savez_compressed(OUT / f"{name}.npz", **rec)
    print(name, "out", rec["out"].shape, "sel", rec["sel"].size)


def topk_known_answers():
    """FlatIndex.top_k / BlockIndex.top_blocks vectors from the real reference."""
    from sparsekv.index import FlatIndex, build_block_index
    rng = np.random.default_rng(4242)
    cases = {}
    q = rng.standard_normal(64).astype(np.float32) * 3
    keys = rng.standard_normal((1200, 64)).astype(np.float32) * 3
    keys[700] = keys[300]  # an exact tie: smaller id first (index.py:64-65)
    keys[701] = keys[300]
    cases["q"], cases["k"] = q, keys
    ks = np.array([1, 2, 3, 10, 100, 1200])
    cases["ks"] = ks
    flat, off = [], [0]
    for k in ks:
        flat.extend(FlatIndex(keys).top_k(q, int(k)))
        off.append(len(flat))
    cases["topk"], cases["topk_off"] = np.array(flat, np.int64), np.array(off)
    # tie at the cut: k such that the tied triple straddles the boundary
    scores = keys.astype(np.float64) @ q.astype(np.float64)
    rank = int((scores > scores[300]).sum())
    cases["tie_k"] = np.array([rank + 1, rank + 2])
    cases["tie_topk1"] = np.array(FlatIndex(keys).top_k(q, rank + 1))
    cases["tie_topk2"] = np.array(FlatIndex(keys).top_k(q, rank + 2))
    # block index: 1200 keys, blocks of 64 (last block partial: 1200 = 18*64 + 48), r = 4
    bi = build_block_index(keys, 64, 4)
    cases["blk_reps"] = np.concatenate([r for r in bi.reps])
    blocks, boff = [], [0]
    for kb in (1, 3, bi.n_blocks):
        blocks.extend([s for s, _ in bi.top_blocks(q, kb)])
        boff.append(len(blocks))
    cases["blk_top"], cases["blk_off"] = np.array(blocks, np.int64), np.array(boff)
    np.savez_compressed(OUT / "topk_known_answers.npz", **cases)
    print("topk_known_answers")


AVDB_HASH_CASES = [  # (name, n, dim, element_width, seed): sha256 of the reference's bytes
    ("empty32", 0, 16, 32, 1), ("one32", 1, 16, 32, 2), ("small32", 37, 16, 32, 3),
    ("multi32", 300, 32, 32, 4), ("small16", 37, 16, 16, 5), ("multi16", 500, 128, 16, 6),
    ("dirchain32", 20000, 16, 32, 7), ("edge16", 64, 16, 16, 8),
]


def avdb_vectors(n, dim, seed, width):
    rng = np.random.default_rng(seed)
    v = (rng.standard_normal((n, dim)) * 3).astype(np.float32)
    if width == 16 and n:  # exercise rounding ties, overflow and subnormals
        v[0, :8] = np.array([65504, 65520, 1e-8, 6e-8, -2.98e-8, 1.0009765625, 2 ** -24, -0.0],
                            dtype=np.float32)
    return v


def avdb_fixtures():
    """AVDB files written by the real reference (sparsekv/vfs.py)."""
    import tempfile

    from sparsekv.vfs import append_vectors, delete_vectors, read_vector_file, write_vector_file
    out = OUT / "avdb"
    out.mkdir(exist_ok=True)
    hashes = {}
    with tempfile.TemporaryDirectory() as td:
        for name, n, dim, width, seed in AVDB_HASH_CASES:
            f = Path(td) / f"{name}.avdb"
            write_vector_file(f, avdb_vectors(n, dim, seed, width), element_width=width)
            b = f.read_bytes()
            hashes[name] = (hashlib.sha256(b).hexdigest(), len(b))
    import json
    (out / "hashes.json").write_text(json.dumps(
        {"cases": AVDB_HASH_CASES, "sha256": hashes}, indent=1) + "\n")
    # mutated files (append + tombstone) and a file with a graph index chain
    rng = np.random.default_rng(99)
    v1 = (rng.standard_normal((100, 32))).astype(np.float32)
    v2 = (rng.standard_normal((150, 32))).astype(np.float32)
    f = out / "appended_tomb16.avdb"
    write_vector_file(f, v1, element_width=16)
    append_vectors(f, v2)
    delete_vectors(f, [3, 7, 120])
    c = read_vector_file(f)
    np.savez_compressed(out / "appended_tomb16.npz", vectors=c.vectors,
                        tombstones=np.array(sorted(c.tombstones)))
    adj = [rng.choice(60, size=int(rng.integers(0, 9)), replace=False).astype(np.int32)
           for _ in range(60)]
    v3 = (rng.standard_normal((60, 16))).astype(np.float32)
    f = out / "graph32.avdb"
    write_vector_file(f, v3, adjacency=adj, entry_point=5, max_degree=8)
    c = read_vector_file(f)
    np.savez_compressed(out / "graph32.npz", vectors=c.vectors)
    print("avdb fixtures")


def graph_fixtures():
    """Graph DIPRS on reference-built graphs (sparsekv index.py build_graph,
    dipr.py diprs), plus a reference-persisted context whose FINE layer runs
    DIPRS inside Session.attention."""
    import shutil
    import tempfile

    from sparsekv.dipr import diprs
    from sparsekv.index import GraphParams, build_graph
    from sparsekv.workload import make_queries
    cases = {}
    # reference tests/test_dipr.py:192-205 setup (2000 tokens, d=32)
    shape = ModelShape(1, 1, 1, 32)
    spec = WorkloadSpec(n_tokens=2000, shape=shape, seed=21)
    ctx = make_context(spec)
    keys = ctx.keys[0, 0]
    g = build_graph(keys, make_queries(spec, 800, ctx.centers, stream=5), GraphParams(enhance_ef=48))
    deg, flat = g.to_arrays()
    test_q = make_queries(spec, 30, ctx.centers, stream=6)
    cases.update(keys=keys, degrees=deg, nbrs=flat, entry=np.int64(g.entry_point), q=test_q)
    smax = (keys.astype(np.float64) @ test_q.astype(np.float64).T).max(axis=0)
    runs = []  # (beta, l0, window offset or nan)
    for beta in (0.0, 1.0, 6.0, 20.0):
        for l0 in (8, 128):
            runs.append((beta, l0, np.nan))
    runs += [(6.0, 128, -0.5), (6.0, 128, 3.0), (20.0, 16, 1.0)]
    sel, off = [], [0]
    for beta, l0, wo in runs:
        for i, q in enumerate(test_q):
            wm = None if np.isnan(wo) else float(smax[i] + wo)
            sel.extend(sorted(diprs(g, q, g.entry_point, l0, beta, window_max=wm)))
            off.append(len(sel))
    cases["runs"] = np.array(runs)
    cases["sel"], cases["sel_off"] = np.array(sel, np.int64), np.array(off)
    np.savez_compressed(OUT / "graph_diprs.npz", **cases)
    # a persisted context with graph indexes (layer 1 = FINE, layer 0 = FLAT)
    shape = ModelShape(2, 4, 2, 16)
    cfg = EngineConfig(window_initial=4, window_last=8, l0=64, beta=8.0, max_degree=8, knn_k=8,
                       enhance_ef=16, short_context_threshold=64)
    spec = WorkloadSpec(n_tokens=300, shape=shape, seed=31, clusters=6)
    ctx = make_context(spec)
    queries = np.stack([np.stack([make_queries(spec, 40, ctx.centers, stream=10 + 4 * layer + qh)
                                  for qh in range(4)]) for layer in range(2)])
    root = OUT / "ctx_graph"
    if root.exists():
        shutil.rmtree(root)
    with tempfile.TemporaryDirectory() as td:
        db = ContextStore(shape, cfg, root=td)
        cid = db.import_context(ctx.token_ids, ctx.keys, ctx.values, queries)
        shutil.copytree(Path(td) / "contexts", root / "contexts")
    session, _ = db.create_session(ctx.token_ids)
    tids, qs, ks, vs = decode_step_inputs(spec, 3, ctx.centers)
    outs, sel, off, ret = [], [], [0], []
    for step in range(3):
        for layer in range(2):
            session.update(qs[step, layer], ks[step, layer], vs[step, layer], layer)
        for layer in range(2):
            o = session.attention(qs[step, layer], layer)
            outs.append(o)
            for info in session.last_diagnostics["heads"]:
                sel.extend(info["selected_base"])
                off.append(len(sel))
                ret.append(info["retrieved"])
        plans = [session.active_plan(layer).index.value for layer in range(2)]
    assert plans == ["flat", "fine"], plans
    np.savez_compressed(OUT / "ctx_graph_session.npz", out=np.stack(outs), sel=np.array(sel, np.int64),
                        sel_off=np.array(off), retrieved=np.array(ret), q=qs, k=ks, v=vs,
                        keys=ctx.keys, values=ctx.values, tokens=ctx.token_ids,
                        context_id=np.array(cid))
    print("graph fixtures")


def known_answers():
    """Known-answer DIPR / window cases lifted from the reference's own tests."""
    rng = np.random.default_rng(12345)  # reference tests/conftest.py:7-9
    cases = {}
    # tests/test_dipr.py:69-72 hand case
    q = np.array([1.0, 0.0], dtype=np.float32)
    keys = np.array([[3.0, 0.0], [2.5, 0.0], [0.0, 1.0]], dtype=np.float32)
    cases["hand_q"], cases["hand_k"] = q, keys
    cases["hand_out"] = np.array(sorted(dipr_bruteforce(q, keys, 1.0)))
    # random DIPR sets over a beta ladder (tests/test_dipr.py:63-98 style)
    q = rng.standard_normal(64).astype(np.float32) * 3
    keys = rng.standard_normal((1200, 64)).astype(np.float32) * 3
    cases["rand_q"], cases["rand_k"] = q, keys
    betas = np.array([0.0, 1.0, 5.0, 20.0, 50.0, 110.0, 1e9])
    cases["rand_betas"] = betas
    flat, off = [], [0]
    for b in betas:
        s = sorted(dipr_bruteforce(q, keys, float(b)))
        flat.extend(s)
        off.append(len(flat))
    cases["rand_sel"], cases["rand_off"] = np.array(flat, np.int32), np.array(off)
    # WindowConfig.base_ids (tests/test_core.py:139-150)
    wins = []
    for p, ini, last in [(0, 16, 64), (10, 16, 64), (80, 16, 64), (81, 16, 64),
                         (4096, 16, 64), (100, 0, 8), (100, 4, 0)]:
        ids = WindowConfig(ini, last).base_ids(p)
        wins.append(np.concatenate([[p, ini, last, ids.size], ids]))
    cases["windows"] = np.concatenate(wins)
    np.savez_compressed(OUT / "known_answers.npz", **cases)
    print("known_answers")


def main():
    known_answers()
    avdb_fixtures()
    graph_fixtures()
    topk_known_answers()
    topk_session_case("tiny_topk_flat", "flat", 20, 2, 4, 2, 16, 200, 2, seed=11, win_init=4,
                      win_last=8, clusters=6, store_inputs=True)
    topk_session_case("tiny_topk_coarse", "coarse", 40, 2, 4, 2, 16, 203, 2, seed=12, win_init=4,
                      win_last=8, clusters=6, block_size=16, reps=3, store_inputs=True)
    topk_session_case("llama_4k_topk_flat", "flat", 100, 1, 32, 8, 128, 4096, 1, seed=0,
                      win_init=16, win_last=64)
    topk_session_case("llama_4k_topk_coarse", "coarse", 300, 1, 32, 8, 128, 4096, 1, seed=0,
                      win_init=16, win_last=64)
    # tiny shapes with stored inputs: edge cases of the window/selection logic
    flat_session_case("tiny_gqa", 2, 4, 2, 16, 200, 3, seed=1, beta=8.0,
                      win_init=4, win_last=8, clusters=6, store_inputs=True)
    flat_session_case("tiny_short", 1, 4, 1, 16, 10, 2, seed=2, beta=8.0,
                      win_init=4, win_last=8, clusters=3, store_inputs=True)
    flat_session_case("tiny_nowin", 1, 6, 2, 32, 333, 2, seed=3, beta=30.0,
                      win_init=0, win_last=0, clusters=4, store_inputs=True)
    # BASELINE config 1: Llama-3.1-8B layer (32 q / 8 kv, d=128), ctx 4K, fp32
    flat_session_case("llama_4k_fp32", 1, 32, 8, 128, 4096, 2, seed=0, beta=110.0,
                      win_init=16, win_last=64)
    # bf16-rounded K/V variant of the same layer
    flat_session_case("llama_4k_bf16", 1, 32, 8, 128, 4096, 1, seed=0, beta=110.0,
                      win_init=16, win_last=64, bf16=True)
    # Qwen2.5-14B-shaped layer (40 q / 8 kv), smaller ctx, beta 20
    flat_session_case("qwen_2k_fp32", 1, 40, 8, 128, 2048, 1, seed=5, beta=20.0,
                      win_init=16, win_last=64)


if __name__ == "__main__":
    main()
