"""GPU-resident context lifecycle and AVDB loading (row 4),
mirroring the reference's tests/test_store.py (import, prefix reuse, update
views, store, persistence round trip) and acceptance C9 (late
materialization), plus native AVDB loads of reference-written files."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest
import torch

from oracle import alaya_oracle as O
from tests.golden_cases import GOLDEN, avdb_vectors

pytestmark = pytest.mark.gpu

AV = GOLDEN / "avdb"
L_, HQ, HKV, D = 2, 4, 2, 16


def small_config(P, **kw):
    base = dict(window_initial=4, window_last=8, beta=8.0, block_size=16, representatives=2,
                short_context_threshold=64)
    base.update(kw)
    return P.EngineConfig(**base)


def synthetic(n, seed=0):
    tok, keys, vals, centers, _ = O.make_context(n, L_, HKV, D, clusters=6, seed=seed)
    return tok, keys, vals, centers


def steps(centers, k, seed=0):
    return O.decode_step_inputs(k, L_, HQ, HKV, D, centers, seed=seed)


def test_import_idempotent_and_persisted_roundtrip(cuda_ok, tmp_path):
    import paper_2504_10326_b200 as P
    tok, keys, vals, _ = synthetic(120, seed=3)
    db = P.ContextStore(P.ModelShape(L_, HQ, HKV, D), small_config(P), root=tmp_path)
    a = db.import_context(tok, keys, vals)
    assert db.import_context(tok, keys, vals) == a and len(db.contexts) == 1
    reopened = P.ContextStore(P.ModelShape(L_, HQ, HKV, D), small_config(P), root=tmp_path)
    rec = reopened.get(a)
    assert np.array_equal(rec.keys.cpu().numpy(), keys)
    assert np.array_equal(rec.values.cpu().numpy(), vals)
    assert np.array_equal(rec.token_ids, tok)
    assert (tmp_path / "contexts" / a / "meta.json").exists()
    # fp16 files (element_width 16): exact half rounding, widened exactly
    db16 = P.ContextStore(P.ModelShape(L_, HQ, HKV, D), small_config(P, element_width=16),
                          root=tmp_path / "w16")
    b = db16.import_context(tok, keys, vals)
    back = P.ContextStore(P.ModelShape(L_, HQ, HKV, D), small_config(P, element_width=16),
                          root=tmp_path / "w16").get(b)
    assert np.array_equal(back.keys.cpu().numpy(), keys.astype(np.float16).astype(np.float32))


def test_prefix_reuse_views_and_untouched_base(cuda_ok):
    import paper_2504_10326_b200 as P
    tok, keys, vals, centers = synthetic(60)
    db = P.ContextStore(P.ModelShape(L_, HQ, HKV, D), small_config(P))
    cid = db.import_context(tok, keys, vals)
    s, rest = db.create_session(np.concatenate([tok[:40], [999, 998]]))
    assert s.reused_prefix_len == 40 and rest == [999, 998]
    s2, rest2 = db.create_session([123456])
    assert s2.base is None and rest2 == [123456]
    sess, _ = db.create_session(tok)
    before = hashlib.sha256(db.get(cid).keys.cpu().numpy().tobytes()).hexdigest()
    _, qs, ks, vs = steps(centers, 5)
    for step in range(5):
        kv, _ = sess.update(qs[step, 0], ks[step, 0], vs[step, 0], 0)
    assert len(kv) == HKV and len(kv[0]) == 65
    assert np.array_equal(kv[0].materialize()[:60].cpu().numpy(), keys[0, 0])
    assert hashlib.sha256(db.get(cid).keys.cpu().numpy().tobytes()).hexdigest() == before
    with pytest.raises(ValueError):
        sess.update(qs[0, 0], np.zeros((HKV, D + 1), np.float32), np.zeros((HKV, D + 1), np.float32), 0)
    with pytest.raises(ValueError):
        sess.update(qs[0, 0], ks[0, 0], vs[0, 0], L_)


def test_store_then_full_reuse(cuda_ok):
    """reference tests/test_store.py:241-259"""
    import paper_2504_10326_b200 as P
    tok, keys, vals, centers = synthetic(80)
    db = P.ContextStore(P.ModelShape(L_, HQ, HKV, D), small_config(P))
    first = db.import_context(tok, keys, vals)
    sess, _ = db.create_session(tok)
    tids, qs, ks, vs = steps(centers, 6)
    for step in range(6):
        for layer in range(L_):
            sess.update(qs[step, layer], ks[step, layer], vs[step, layer], layer)
        sess.record_token(int(tids[step]))
    new_id = db.store(sess)
    stored = db.get(new_id)
    stored.check_invariants()
    assert stored.length == 86
    assert np.array_equal(stored.keys[:, :, :80].cpu().numpy(), keys)
    assert np.array_equal(stored.keys[1, 0, 80:].cpu().numpy(), ks[:, 1, 0])
    again, truncated = db.create_session(stored.token_ids)
    assert truncated == [] and again.reused_prefix_len == 86
    assert db.get(first).length == 80
    # attention over the stored context = attention over base + window before storing
    q = qs[-1, 1]
    o_live = sess.attention(q, 1)
    o_stored = again.attention(q, 1)
    assert o_live.shape == o_stored.shape and np.isfinite(o_stored).all()


def test_store_without_base_and_errors(cuda_ok, rng):
    """reference tests/test_store.py:261-280"""
    import paper_2504_10326_b200 as P
    db = P.ContextStore(P.ModelShape(L_, HQ, HKV, D), small_config(P))
    sess, _ = db.create_session([42, 43])
    for step in range(3):
        q = rng.standard_normal((HQ, D)).astype(np.float32)
        k = rng.standard_normal((HKV, D)).astype(np.float32)
        for layer in range(L_):
            sess.update(q, k, k, layer)
        sess.record_token(100 + step)
    cid = db.store(sess)
    assert db.get(cid).length == 3 and db.get(cid).token_ids.tolist() == [100, 101, 102]
    empty, _ = db.create_session([1])
    with pytest.raises(ValueError):
        db.store(empty)
    with pytest.raises(ValueError):
        empty.attention(np.zeros((HQ, D), np.float32), 0)


def test_late_materialization_c9(cuda_ok, tmp_path):
    """Acceptance C9 (reference tests/test_acceptance.py:383-416): many updates
    leave the persisted base bytes unchanged; the stored session is reusable."""
    import paper_2504_10326_b200 as P
    shape = P.ModelShape(1, 2, 1, 32)
    cfg = P.EngineConfig(window_initial=8, window_last=32, short_context_threshold=64)
    tok, keys, vals, centers, _ = O.make_context(512, 1, 1, 32, clusters=4, seed=19)
    db = P.ContextStore(shape, cfg, root=tmp_path)
    cid = db.import_context(tok, keys, vals)

    def dir_hash():
        h = hashlib.sha256()
        for f in sorted(db.context_dir(cid).rglob("*")):
            h.update(f.name.encode())
            h.update(f.read_bytes())
        return h.hexdigest()

    before = dir_hash()
    sess, truncated = db.create_session(tok)
    assert truncated == []
    tids, qs, ks, vs = O.decode_step_inputs(2000, 1, 2, 1, 32, centers, seed=19)
    for step in range(2000):
        sess.update(qs[step, 0], ks[step, 0], vs[step, 0], 0)
        sess.record_token(int(tids[step]))
    assert dir_hash() == before
    new_id = db.store(sess)
    stored = db.get(new_id)
    again, truncated = db.create_session(stored.token_ids)
    assert truncated == [] and again.reused_prefix_len == stored.length == 2512


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_avdb_load_matches_reference_files(cuda_ok, tmp_path, dtype):
    from paper_2504_10326_b200 import vfs
    z = np.load(AV / "appended_tomb16.npz")
    got = vfs.read_vector_file(AV / "appended_tomb16.avdb", dtype=dtype)
    want = torch.from_numpy(z["vectors"]).to(dtype)
    assert got.tombstones == 3 and torch.equal(got.vectors.cpu(), want)
    g = vfs.read_vector_file(AV / "graph32.avdb", dtype=dtype)  # index blocks are skipped
    assert torch.equal(g.vectors.cpu(), torch.from_numpy(np.load(AV / "graph32.npz")["vectors"]).to(dtype))
    # many files, multi-block, fp16 edge values, into one slab
    paths = []
    for i, (n, dim, width) in enumerate([(500, 128, 16), (500, 128, 32), (500, 128, 16)]):
        p = tmp_path / f"f{i}.avdb"
        with np.errstate(over="ignore"):
            vfs.write_vector_file(p, avdb_vectors(n, dim, 40 + i, width), element_width=width)
        paths.append(p)
    for grp in ([paths[0], paths[2]], [paths[1]]):
        out = vfs.load_to_device(grp, 500, 128, dtype, torch.device("cuda"))
        for j, p in enumerate(grp):
            width = vfs.read_header(p).element_width
            i = paths.index(p)
            v = avdb_vectors(500, 128, 40 + i, width)
            if width == 16:
                with np.errstate(over="ignore"):
                    v = v.astype(np.float16).astype(np.float32)
            assert torch.equal(out[j].cpu(), torch.from_numpy(v).to(dtype))
    with pytest.raises(vfs.VectorFileError):  # mixed widths in one load
        vfs.load_to_device(paths[:2], 500, 128, dtype, torch.device("cuda"))
    with pytest.raises(ValueError):  # shape mismatch
        vfs.load_to_device([paths[1]], 499, 128, dtype, torch.device("cuda"))
