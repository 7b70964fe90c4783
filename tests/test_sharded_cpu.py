"""Sequence-sharded orchestration on CPU: world_size 2 and 3 over ``gloo``.

The collectives, token offsets, window ownership and the partial merge of
``paper_2504_10326_b200.sharded`` are exercised with a host double of the
local stages built from the oracle (test-only); the CUDA stages are covered
by the single-GPU shard emulation in ``test_gpu_sharded.py``.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import alaya_oracle as O


class OracleShardStages:
    """Host double with the kernels' shard semantics (global window ids,
    session rows on the last rank, reference point = global max)."""

    def __init__(self, keys, values, wk, wv, lo, hi, P, beta, wi, wl, last):
        self.k, self.v = keys[:, :, lo:hi], values[:, :, lo:hi]  # [B, Hkv, n_loc, d]
        self.wk, self.wv = (wk, wv) if last else (None, None)
        self.lo, self.P, self.beta, self.wi, self.wl = lo, P, beta, wi, wl

    def scan(self, q):
        qn = q.numpy()
        B, Hq, _ = qn.shape
        g = Hq // self.k.shape[1]
        out = np.full((B, Hq), -np.inf, np.float32)
        for b in range(B):
            for qh in range(Hq):
                if self.k.shape[2]:
                    out[b, qh] = O.inner_products(self.k[b, qh // g], qn[b, qh]).max()
        return torch.from_numpy(out)

    def attend(self, q, smax):
        qn, sm = q.numpy(), smax.numpy()
        B, Hq, d = qn.shape
        g = Hq // self.k.shape[1]
        win = set(O.window_base_ids(self.P, self.wi, self.wl).tolist())
        parts = np.zeros((B * Hq, d + 2), np.float32)
        for b in range(B):
            for qh in range(Hq):
                h = qh // g
                kk, vv = self.k[b, h], self.v[b, h]
                ids = self.lo + np.arange(kk.shape[0])
                s = O.inner_products(kk, qn[b, qh]) if kk.shape[0] else np.zeros(0)
                mask = (s >= np.float32(sm[b, qh]) - self.beta) & ~np.isin(ids, list(win))
                part = O.partial_over(qn[b, qh], kk[mask], vv[mask])
                wmask = np.isin(ids, list(win))
                wkeys, wvals = [kk[wmask]], [vv[wmask]]
                if self.wk is not None:
                    wkeys.append(self.wk[b, h])
                    wvals.append(self.wv[b, h])
                part = O.partial_merge(part, O.partial_over(qn[b, qh], np.concatenate(wkeys),
                                                            np.concatenate(wvals)))
                row = b * Hq + qh
                if part.is_empty:
                    parts[row, 0] = -np.inf
                else:
                    parts[row, 0], parts[row, 1], parts[row, 2:] = part.m, part.l, part.acc
        return torch.from_numpy(parts)

    def merge(self, parts):
        p = parts.numpy()
        out = np.zeros((p.shape[1], p.shape[2] - 2), np.float32)
        for row in range(p.shape[1]):
            acc = O.Partial()
            for r in range(p.shape[0]):
                if p[r, row, 0] != -np.inf:
                    acc = O.partial_merge(acc, O.Partial(float(p[r, row, 0]), float(p[r, row, 1]),
                                                         p[r, row, 2:].astype(np.float64)))
            out[row] = O.partial_finalize(acc)
        return torch.from_numpy(out)


def _case(seed=0, B=2, n=700, hkv=2, g=3, d=32, w=3):
    tok, keys, vals, centers, _ = O.make_context(n, B, hkv, d, clusters=6, seed=seed)
    # reuse the layer axis as the batch axis: keys [B, Hkv, n, d]
    r = np.random.default_rng(seed)
    q = (centers[r.integers(0, 6, (B, hkv * g))] + 0.25 * r.standard_normal((B, hkv * g, d))).astype(np.float32)
    wk = r.standard_normal((B, hkv, w, d)).astype(np.float32)
    wv = r.standard_normal((B, hkv, w, d)).astype(np.float32)
    return keys, vals, wk, wv, q


def _worker(rank, world, port, beta, wi, wl, ret):
    from paper_2504_10326_b200.sharded import shard_bounds, sharded_attention
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    keys, vals, wk, wv, q = _case()
    lo, hi = shard_bounds(keys.shape[2], world, rank)
    st = OracleShardStages(keys, vals, wk, wv, lo, hi, keys.shape[2], beta, wi, wl, rank == world - 1)
    out = sharded_attention(st, torch.from_numpy(q))
    ret[rank] = out.numpy()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("beta,wi,wl", [(20.0, 4, 8), (5.0, 16, 64), (1e9, 0, 0)])
def test_sharded_matches_unsharded_oracle(world, beta, wi, wl):
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), beta, wi, wl, ret), nprocs=world,
                       join=True, start_method="spawn")
    keys, vals, wk, wv, q = _case()
    B, Hq, d = q.shape
    for b in range(B):
        ref, _, _ = O.session_attention_flat(q[b], keys[b], vals[b], wk[b], wv[b], beta, wi, wl)
        for r in range(world):
            got = ret[r].reshape(B, Hq, d)[b]
            assert np.abs(got - ref).max() <= 1e-5 * max(1.0, np.abs(ref).max())
    # every rank returns the same result
    for r in range(1, world):
        assert np.array_equal(ret[0], ret[r])


def test_shard_bounds_cover_exactly():
    from paper_2504_10326_b200.sharded import shard_bounds
    for n in (1, 7, 1000, 1 << 20):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)
