"""Sequence-sharded mode on ONE GPU: R shards run sequentially through the CUDA
stages (alaya_scan / alaya_attend with token offsets), host-side max over the
shards stands in for the NCCL max-allreduce, the stacked partials for the
allgather; the merge runs in alaya_merge_partials. Must equal the unsharded
kernel path and the CPU oracle (SURVEY.md §4 "single-GPU shard emulation")."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import alaya_oracle as O
from tests.parity import EPS_SET, set_flips

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.parametrize("kv", ["bfloat16", "float32"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_shard_emulation_matches_unsharded(cuda_ok, kv, world):
    from paper_2504_10326_b200 import engine
    from paper_2504_10326_b200.sharded import EngineStages, local_view, shard_bounds
    dev = torch.device("cuda")
    dtype = torch.bfloat16 if kv == "bfloat16" else torch.float32
    B, hkv, g, d, n, w, beta = 2, 2, 4, 128, 20000, 3, 110.0
    r = np.random.default_rng(world)
    keys, vals, qs, wks, wvs = [], [], [], [], []
    for b in range(B):
        _, k, v, centers, _ = O.make_context(n, 1, hkv, d, seed=100 + b)
        if kv == "bfloat16":
            k, v = O.bf16_round(k), O.bf16_round(v)
        keys.append(k[0]); vals.append(v[0])
        qs.append(centers[r.integers(0, 16, hkv * g)] + 0.25 * r.standard_normal((hkv * g, d)))
        wks.append(O.bf16_round(r.standard_normal((hkv, w, d)).astype(np.float32)))
        wvs.append(O.bf16_round(r.standard_normal((hkv, w, d)).astype(np.float32)))
    q = torch.tensor(np.stack(qs), dtype=torch.float32, device=dev)
    K = [torch.from_numpy(k).to(dev, dtype) for k in keys]
    V = [torch.from_numpy(v).to(dev, dtype) for v in vals]
    WK = [torch.from_numpy(x).to(dev, dtype) for x in wks]
    WV = [torch.from_numpy(x).to(dev, dtype) for x in wvs]
    params = engine.make_params(hkv * g, hkv, d, dtype, beta, 16, 64)

    # unsharded reference run through the same kernels
    full = engine.Call([engine.SeqView(k=K[b], v=V[b], n=n, wk=WK[b], wv=WV[b], w=w)
                        for b in range(B)], params, dtype, dev)
    o_full = full.dipr_attention(q).cpu().numpy()

    stages = [EngineStages([local_view(K[b], V[b], world, rk, WK[b], WV[b], w) for b in range(B)],
                           params, dtype, dev) for rk in range(world)]
    # each shard needs its own workspace: the stages run interleaved
    for st in stages:
        st.call.ws = torch.empty(st.call.ws_bytes, dtype=torch.uint8, device=dev)
    smax = torch.stack([st.scan(q) for st in stages]).amax(0)           # all_reduce(MAX)
    parts = torch.stack([st.attend(q, smax) for st in stages])          # all_gather
    o_sh = stages[0].merge(parts).view(B, hkv * g, d).cpu().numpy()

    sel_sh = [[[] for _ in range(hkv * g)] for _ in range(B)]
    for rk, st in enumerate(stages):
        lo, hi = shard_bounds(n, world, rk)
        ids, nsel, _ = st.call.selected(hi - lo)
        ids, nsel = ids.cpu().numpy(), nsel.cpu().numpy()
        for b in range(B):
            for qh in range(hkv * g):
                row = b * hkv * g + qh
                sel_sh[b][qh].extend(ids[row, : nsel[row]].tolist())
    for b in range(B):
        ref, sels, _ = O.session_attention_flat(qs[b].astype(np.float32), keys[b], vals[b],
                                                wks[b], wvs[b], beta)
        for qh in range(hkv * g):
            assert sorted(sel_sh[b][qh]) == sel_sh[b][qh]  # ascending across shards
            h = qh // g
            flips, _ = set_flips(sel_sh[b][qh], O.inner_products(keys[b][h], qs[b][qh].astype(np.float32)),
                                 beta, EPS_SET[kv], O.window_base_ids(n))
            o_sel = O.head_attention_on_selection(qs[b][qh].astype(np.float32), keys[b][h], vals[b][h],
                                                  wks[b][h], wvs[b][h], sel_sh[b][qh])
            assert rel(o_sh[b, qh], o_sel) <= 1e-5
            if not flips:
                assert rel(o_sh[b, qh], ref[qh]) <= 1e-5
            assert rel(o_sh[b, qh], o_full[b, qh]) <= 2e-6


def _exchange_group(world, cap, dev):
    """`world` emulated ranks in ONE process: each owns an exchange buffer and
    sees all of them as its peers (the IPC mapping step is the only part a
    multi-process run adds). Each rank's kernels go on its own stream."""
    import ctypes

    from paper_2504_10326_b200 import _lib
    from paper_2504_10326_b200.sharded import PeerExchange
    lib = _lib.load()
    bufs = []
    for _ in range(world):
        own, h = ctypes.c_void_p(), (ctypes.c_char * 64)()
        assert lib.alaya_exch_alloc(lib.alaya_exch_bytes(world, cap), ctypes.byref(own), h) == 0
        bufs.append(own.value)
    return [PeerExchange(bufs, bufs[r], r, world, cap, dev, []) for r in range(world)], bufs


@pytest.mark.parametrize("world", [2, 4, 8])
def test_peer_exchange_collectives(cuda_ok, world):
    dev = torch.device("cuda")
    rows, d = 64, 128
    cap = rows * (d + 2)
    exs, bufs = _exchange_group(world, cap, dev)
    streams = [torch.cuda.Stream() for _ in range(world)]
    g = torch.Generator(device=dev).manual_seed(world)
    for step in range(5):  # epochs 1..5 on both kinds (slot parity alternates)
        loc = [torch.randn(rows, generator=g, device=dev) for _ in range(world)]
        parts = [torch.randn(rows, d + 2, generator=g, device=dev) for _ in range(world)]
        torch.cuda.synchronize()
        mx, gathered = [None] * world, [None] * world
        # launches return at once, so the ranks' kernels run concurrently. Emulated ranks
        # share one GPU's launch queues, so each exchange is issued for every rank before
        # the next one (issuing rank by rank can leave a rank's exchange queued behind
        # another rank's spinning kernel; one process per GPU has no such coupling)
        for r in range(world):
            with torch.cuda.stream(streams[r]):
                mx[r] = exs[r].allreduce_max(loc[r])
        for r in range(world):
            with torch.cuda.stream(streams[r]):
                gathered[r] = exs[r].allgather(parts[r]).clone()
        torch.cuda.synchronize()
        want = torch.stack(loc).amax(0)
        for r in range(world):
            exs[r].check()
            assert torch.equal(mx[r], want)
            assert torch.equal(gathered[r], torch.stack(parts))
    from paper_2504_10326_b200 import _lib
    for b in bufs:
        _lib.load().alaya_exch_free(b)


def test_sharded_attention_over_peer_exchange(cuda_ok):
    """The full sharded step with the peer-memory collectives (ranks emulated on
    streams of one GPU) equals the unsharded kernels."""
    from paper_2504_10326_b200 import engine
    from paper_2504_10326_b200.sharded import EngineStages, local_view
    dev = torch.device("cuda")
    world, B, hkv, g, d, n, w, beta = 3, 2, 2, 4, 128, 30000, 2, 110.0
    dtype = torch.bfloat16
    r = np.random.default_rng(5)
    K, V, WK, WV, qs = [], [], [], [], []
    for b in range(B):
        _, k, v, centers, _ = O.make_context(n, 1, hkv, d, seed=300 + b)
        K.append(torch.from_numpy(O.bf16_round(k)[0]).to(dev, dtype))
        V.append(torch.from_numpy(O.bf16_round(v)[0]).to(dev, dtype))
        WK.append(torch.randn(hkv, w, d, device=dev).to(dtype))
        WV.append(torch.randn(hkv, w, d, device=dev).to(dtype))
        qs.append(centers[r.integers(0, 16, hkv * g)] + 0.25 * r.standard_normal((hkv * g, d)))
    q = torch.tensor(np.stack(qs), dtype=torch.float32, device=dev)
    params = engine.make_params(hkv * g, hkv, d, dtype, beta, 16, 64)
    full = engine.Call([engine.SeqView(k=K[b], v=V[b], n=n, wk=WK[b], wv=WV[b], w=w)
                        for b in range(B)], params, dtype, dev,
                       ws=torch.empty(1, dtype=torch.uint8, device=dev))
    o_full = full.dipr_attention(q).clone()
    stages = [EngineStages([local_view(K[b], V[b], world, rk, WK[b], WV[b], w) for b in range(B)],
                           params, dtype, dev) for rk in range(world)]
    for st in stages:
        st.call.ws = torch.empty(st.call.ws_bytes, dtype=torch.uint8, device=dev)
    exs, bufs = _exchange_group(world, B * hkv * g * (d + 2), dev)
    streams = [torch.cuda.Stream() for _ in range(world)]
    torch.cuda.synchronize()
    for _ in range(3):
        # sharded_attention's exchange branch, phase by phase across the emulated ranks
        # (see test_peer_exchange_collectives for why); bench.py --check with
        # ALAYA_BENCH_SHARE_GPU=1 runs the branch itself in separate processes
        smax, parts, outs = [None] * world, [None] * world, [None] * world
        for rk in range(world):
            with torch.cuda.stream(streams[rk]):
                smax[rk] = exs[rk].allreduce_max(stages[rk].scan(q))
        for rk in range(world):
            with torch.cuda.stream(streams[rk]):
                parts[rk] = exs[rk].allgather(stages[rk].attend(q, smax[rk]).contiguous())
        for rk in range(world):
            with torch.cuda.stream(streams[rk]):
                outs[rk] = stages[rk].merge(parts[rk]).view(q.shape[0], q.shape[1], -1)
        torch.cuda.synchronize()
        for rk in range(world):
            exs[rk].check()
            assert float(((outs[rk] - o_full).norm() / o_full.norm()).item()) <= 2e-6
    from paper_2504_10326_b200 import _lib
    for b in bufs:
        _lib.load().alaya_exch_free(b)


@pytest.mark.parametrize("world,lens,beta", [(2, (6000, 7000), 5.0), (3, (2, 9000), 5.0), (4, (5000, 1), 5.0),
                                             (3, (7000, 9000), 140.0)])
def test_fused_sharded_step_emulated(cuda_ok, world, lens, beta):
    """alaya_sharded_step (scan -> per-group max over peer memory -> attend) for
    2-4 ranks emulated on streams of one GPU at a size whose grids co-reside
    (each rank's attend waits on the others' scans: the bounded poll turns a
    missed arrival into the error flag, not a hang), vs the unsharded kernels.
    Sequences shorter than the world leave shards with no tokens of them: those
    ranks export -inf maxima from prep_kernel. beta = 140 runs the group candidate
    format (attend_grp_kernel reading the ranks' pushed maxima)."""
    from paper_2504_10326_b200 import _lib, engine
    from paper_2504_10326_b200.sharded import EngineStages, local_view
    dev = torch.device("cuda")
    B, hkv, g, d, w = len(lens), 2, 4, 128, 3
    dtype = torch.bfloat16
    r = np.random.default_rng(9 + world)
    K, V, WK, WV, qs = [], [], [], [], []
    for b in range(B):
        _, k, v, centers, _ = O.make_context(lens[b], 1, hkv, d, seed=700 + b)
        K.append(torch.from_numpy(O.bf16_round(k)[0]).to(dev, dtype))
        V.append(torch.from_numpy(O.bf16_round(v)[0]).to(dev, dtype))
        WK.append(torch.randn(hkv, w, d, device=dev).to(dtype))
        WV.append(torch.randn(hkv, w, d, device=dev).to(dtype))
        qs.append(centers[r.integers(0, 16, hkv * g)] + 0.25 * r.standard_normal((hkv * g, d)))
    q = torch.tensor(np.stack(qs), dtype=torch.float32, device=dev)
    params = engine.make_params(hkv * g, hkv, d, dtype, beta, 16, 64)
    full = engine.Call([engine.SeqView(k=K[b], v=V[b], n=K[b].shape[1], wk=WK[b], wv=WV[b], w=w)
                        for b in range(B)], params, dtype, dev,
                       ws=torch.empty(1, dtype=torch.uint8, device=dev))
    o_full = full.dipr_attention(q).clone()
    stages = [EngineStages([local_view(K[b], V[b], world, rk, WK[b], WV[b], w) for b in range(B)],
                           params, dtype, dev) for rk in range(world)]
    for st in stages:
        st.call.ws = torch.empty(st.call.ws_bytes, dtype=torch.uint8, device=dev)
    exs, bufs = _exchange_group(world, B * hkv * g * (d + 2), dev)
    streams = [torch.cuda.Stream() for _ in range(world)]
    torch.cuda.synchronize()
    rows = q.shape[0] * q.shape[1]
    for it in range(4):
        parts, outs = [None] * world, [None] * world
        if it % 2 == 0:  # fused scan/max/attend, then the alaya_exch allgather + merge
            for rk in range(world):
                with torch.cuda.stream(streams[rk]):
                    parts[rk] = stages[rk].fused(q, exs[rk])
                    assert parts[rk] is not None and stages[rk].fused_used
            for rk in range(world):
                with torch.cuda.stream(streams[rk]):
                    parts[rk] = exs[rk].allgather(parts[rk])
            for rk in range(world):
                with torch.cuda.stream(streams[rk]):
                    outs[rk] = stages[rk].merge(parts[rk])
        else:  # fully fused: the combine pushes the partials, the merge waits for the flags
            ge = exs[0].epoch[1] + 1
            for rk in range(world):
                with torch.cuda.stream(streams[rk]):
                    e = exs[rk].epoch[0] + 1
                    assert stages[rk].call.sharded_step(q, exs[rk]._arr, world, rk, exs[rk].cap, e,
                                                        exs[rk].err, ge) is True
                    exs[rk].epoch[0], exs[rk].epoch[1] = e, ge
            for rk in range(world):
                with torch.cuda.stream(streams[rk]):
                    outs[rk] = exs[rk].merge_exchanged(rows, d, ge)
        torch.cuda.synchronize()
        for rk in range(world):
            exs[rk].check()
            o = outs[rk].view(q.shape[0], q.shape[1], -1)
            assert float(((o - o_full).norm() / o_full.norm()).item()) <= 2e-6, (it, rk)
    for b in bufs:
        _lib.load().alaya_exch_free(b)


def test_fused_sharded_step_falls_back_when_ineligible(cuda_ok):
    """fp32 K/V (CUDA-core scan): alaya_sharded_step answers UNSUPPORTED, the
    stage reports it (None) and sharded_attention takes the staged peer path."""
    from paper_2504_10326_b200 import _lib, engine
    from paper_2504_10326_b200.sharded import EngineStages, local_view
    dev = torch.device("cuda")
    world, hkv, g, d, n = 2, 2, 4, 128, 3000
    _, k, v, centers, _ = O.make_context(n, 1, hkv, d, seed=41)
    K = torch.from_numpy(k[0]).to(dev)
    V = torch.from_numpy(v[0]).to(dev)
    params = engine.make_params(hkv * g, hkv, d, torch.float32, 5.0, 16, 64)
    q = torch.tensor(centers[:hkv * g][None], dtype=torch.float32, device=dev)
    st = EngineStages([local_view(K, V, world, 0)], params, torch.float32, dev)
    exs, bufs = _exchange_group(world, hkv * g * (d + 2), dev)
    assert st.fused(q, exs[0]) is None and not st.fused_used
    assert st.fused(q, exs[0], gather=True) is None
    assert exs[0].epoch == [0, 0]  # nothing was consumed
    for b in bufs:
        _lib.load().alaya_exch_free(b)
