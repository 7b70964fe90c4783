"""Device-side engine: torch tensors in, C-ABI calls out.

PyTorch is plumbing here (device memory, streams, collectives); every
arithmetic step of the hot path runs in ``libalaya_b200.so``. The stages map
onto the reference's flat decode step (``store.py:252-293``):

=====================  =================================================
``scan``               scores + per-head max + candidate superset
``attend``             exact ``>= max - beta`` filter, window exclusion,
                       V gather, online softmax -> (m, l, acc) per head
``merge_partials``     ``PartialAttention.merge`` + ``finalize``
``dipr_attention``     all three in one stream-ordered call
``selected``           the critical id sets (``dipr_bruteforce`` output)
=====================  =================================================
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import AlayaBlockIndex, AlayaGraph, AlayaParams, AlayaSeq, check

_DTYPES = {torch.float32: _lib.ALAYA_F32, torch.bfloat16: _lib.ALAYA_BF16}


def require_cuda() -> None:
    """Fail loudly: the product path has no CPU fallback."""
    _lib.load()
    if not torch.cuda.is_available():
        raise _lib.AlayaError("no CUDA device: the alaya B200 path has no CPU fallback")


@dataclass
class SeqView:
    """One sequence (session) at one layer, as device tensors.

    ``k``/``v``: ``[Hkv, rows >= n, d]`` base prefix (row stride must be d);
    ``wk``/``wv``: ``[Hkv, rows >= w, d]`` session-window rows or None.
    ``token_offset``/``prefix_len`` describe a sequence shard.
    """

    k: torch.Tensor | None
    v: torch.Tensor | None
    n: int
    wk: torch.Tensor | None = None
    wv: torch.Tensor | None = None
    w: int = 0
    token_offset: int = 0
    prefix_len: int | None = None
    bounds: torch.Tensor | None = None  # [Hkv, blocks, 5, d] (block_bounds), block filter only
    # CUDA-graph mode: int32 [1] device row count of the window ring (``w`` is ignored;
    # the capacity is wk.shape[1]); window_append advances it on the device
    w_dev: torch.Tensor | None = None


def _w_dev_ptr(s: SeqView):
    if s.w_dev is None:
        return None
    if s.w_dev.dtype != torch.int32 or not s.w_dev.is_cuda or s.w_dev.numel() < 1:
        raise ValueError("w_dev must be an int32 CUDA tensor")
    if s.wk is None or s.wv is None:
        raise ValueError("w_dev needs the window ring tensors")
    return s.w_dev.data_ptr()


def _window_rows(s: SeqView) -> int:
    """Host row count, or the ring capacity in device-count (graph) mode."""
    return int(s.wk.shape[1]) if s.w_dev is not None and s.wk is not None else int(s.w)


def _check_kv(t: torch.Tensor, name: str, dtype, d: int) -> None:
    if t.dtype != dtype:
        raise ValueError(f"{name} dtype {t.dtype} != {dtype}")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dim() != 3 or t.shape[2] != d or t.stride(2) != 1 or t.stride(1) != d:
        raise ValueError(f"{name} must be [heads, rows, {d}] with unit row stride, got "
                         f"{tuple(t.shape)} strides {t.stride()}")


def make_params(n_query_heads: int, n_kv_heads: int, dim: int, dtype: torch.dtype, beta: float,
                win_initial: int, win_last: int, chunk: int = 0, scan_kind: int = 0,
                block_filter: int = 0) -> AlayaParams:
    if dtype not in _DTYPES:
        raise ValueError(f"unsupported KV dtype {dtype}")
    if beta < 0:
        raise ValueError(f"beta must be non-negative, got {beta}")
    return AlayaParams(n_query_heads, n_kv_heads, dim, _DTYPES[dtype], float(beta),
                       int(win_initial), int(win_last), int(chunk), int(scan_kind),
                       int(block_filter))


def seq_array(seqs: list[SeqView], params: AlayaParams, dtype: torch.dtype):
    d = params.dim
    arr = (AlayaSeq * len(seqs))()
    for i, s in enumerate(seqs):
        e = arr[i]
        if s.n:
            _check_kv(s.k, "k", dtype, d)
            _check_kv(s.v, "v", dtype, d)
            if s.k.shape[0] != params.n_kv_heads or s.k.shape[1] < s.n:
                raise ValueError(f"base K shape {tuple(s.k.shape)} vs n={s.n}")
            if s.v.stride(0) != s.k.stride(0):
                raise ValueError("k and v must share a head stride")
            e.k, e.v, e.head_stride = s.k.data_ptr(), s.v.data_ptr(), s.k.stride(0)
        w = _window_rows(s)
        if w:
            _check_kv(s.wk, "wk", dtype, d)
            _check_kv(s.wv, "wv", dtype, d)
            if s.wk.shape[1] < w or s.wv.stride(0) != s.wk.stride(0):
                raise ValueError("window K/V shape mismatch")
            e.wk, e.wv, e.w_head_stride = s.wk.data_ptr(), s.wv.data_ptr(), s.wk.stride(0)
        if s.bounds is not None:
            if s.bounds.dtype != dtype or not s.bounds.is_contiguous() or s.bounds.shape[0] != params.n_kv_heads:
                raise ValueError("bounds must be a contiguous [Hkv, blocks, 5, d] tensor in the KV dtype")
            e.bounds, e.bounds_head_stride = s.bounds.data_ptr(), s.bounds.stride(0)
        e.n, e.w = int(s.n), w
        e.d_w = _w_dev_ptr(s)
        e.token_offset = int(s.token_offset)
        e.prefix_len = int(s.n + s.token_offset if s.prefix_len is None else s.prefix_len)
    return arr


class _Workspace(threading.local):
    """Shared call workspaces, one per (device, stream): the kernels of one call
    hand off through the workspace header (prep zeroes it while the previous
    call's combine may still read it), which is only safe in stream order."""

    def __init__(self):
        self.buf: dict[tuple[int, int], torch.Tensor] = {}

    def get(self, nbytes: int, device: torch.device, stream: int | None = None) -> torch.Tensor:
        idx = device.index if device.index is not None else torch.cuda.current_device()
        if stream is None:
            stream = torch.cuda.current_stream(device).cuda_stream
        t = self.buf.get((idx, stream))
        if t is None or t.numel() < nbytes:
            t = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
            self.buf[(idx, stream)] = t
        return t


_WS = _Workspace()
_DWS = _Workspace()  # graph-walk scratch (separate from the scan workspace)


class Call:
    """One validated batch: params + descriptors + workspace (reused by stages)."""

    def __init__(self, seqs: list[SeqView], params: AlayaParams, dtype: torch.dtype,
                 device: torch.device, ws: torch.Tensor | None = None):
        require_cuda()
        self.lib = _lib.load()
        if not 1 <= len(seqs) <= _lib.MAX_BATCH:
            raise ValueError(f"batch must be in [1, {_lib.MAX_BATCH}]")
        self.params = params
        self.seqs = seq_array(seqs, params, dtype)
        self.B = len(seqs)
        self.device = device
        nbytes = self.lib.alaya_workspace_bytes(ctypes.byref(params), self.seqs, self.B)
        if nbytes == 0:
            check(_lib.ALAYA_ERR_ARG)
        self._nbytes = nbytes
        self._ws_stream = torch.cuda.current_stream(device).cuda_stream
        self._ws_shared = not (ws is not None and ws.numel() >= nbytes)
        self._ws = _WS.get(nbytes, device, self._ws_stream) if self._ws_shared else ws
        self.ws_bytes = self._ws.numel()
        self._dtype = dtype

    @property
    def ws(self) -> torch.Tensor:
        """The call's workspace. A shared (cached) workspace belongs to one stream: a
        call issued on another stream switches to that stream's workspace, so two
        streams never race on one header."""
        if self._ws_shared:
            self._bind(torch.cuda.current_stream(self.device).cuda_stream)
        return self._ws

    def _bind(self, st: int) -> None:
        if self._ws_shared and st != self._ws_stream:
            self._ws = _WS.get(self._nbytes, self.device, st)
            self._ws_stream, self.ws_bytes = st, self._ws.numel()

    @ws.setter
    def ws(self, t: torch.Tensor) -> None:  # a caller-owned workspace (e.g. a captured graph's)
        self._ws, self._ws_shared, self.ws_bytes = t, False, t.numel()

    @property
    def stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def _q(self, q: torch.Tensor) -> torch.Tensor:
        p = self.params
        if q.shape != (self.B, p.n_query_heads, p.dim):
            raise ValueError(f"q must be {(self.B, p.n_query_heads, p.dim)}, got {tuple(q.shape)}")
        if q.dtype == torch.float32 and q.is_cuda and q.is_contiguous() and q.device == self.device:
            return q
        return q.to(device=self.device, dtype=torch.float32).contiguous()

    def dipr_attention(self, q: torch.Tensor, out: torch.Tensor | None = None,
                       append: tuple[torch.Tensor, torch.Tensor] | None = None) -> torch.Tensor:
        """DIPR retrieval + sparse attention for the batch. ``append=(k, v)``
        (``[B, Hkv, d]`` fp32): first write them as window row ``w - 1`` of every
        sequence (``Session.update``; the sequences' ``w`` already count the row),
        inside the same call (``alaya_dipr_attention_update``)."""
        q = self._q(q)
        if out is None:
            out = torch.empty_like(q)
        st = torch.cuda.current_stream(self.device).cuda_stream  # (once per call: the hot path)
        self._bind(st)
        if append is None:
            check(self.lib.alaya_dipr_attention(ctypes.byref(self.params), self.seqs, self.B,
                                                q.data_ptr(), out.data_ptr(), self._ws.data_ptr(),
                                                self.ws_bytes, st))
        else:
            p = self.params
            kn, vn = (t.to(device=self.device, dtype=torch.float32).contiguous() for t in append)
            if kn.shape != (self.B, p.n_kv_heads, p.dim) or vn.shape != kn.shape:
                raise ValueError(f"k/v must be {(self.B, p.n_kv_heads, p.dim)}")
            check(self.lib.alaya_dipr_attention_update(ctypes.byref(self.params), self.seqs, self.B,
                                                       kn.data_ptr(), vn.data_ptr(), q.data_ptr(),
                                                       out.data_ptr(), self._ws.data_ptr(),
                                                       self.ws_bytes, st))
            self._kv_keep = (kn, vn)
        self._q_keep = q
        return out

    def set_window_rows(self, w: int) -> None:
        """Update every sequence's session-window row count (fast per-step rebind;
        the caller guarantees the window tensors hold >= w rows)."""
        for i in range(self.B):
            self.seqs[i].w = int(w)

    def scan_only(self, q: torch.Tensor) -> None:
        """Stage 1 alone (no max export): used to time the scan kernel."""
        check(self.lib.alaya_scan(ctypes.byref(self.params), self.seqs, self.B, q.data_ptr(),
                                  None, self.ws.data_ptr(), self.ws_bytes, self.stream))

    def block_stats(self) -> tuple[int, int]:
        """(128-key blocks kept, blocks considered) by the block filter in the last scan."""
        p = self.lib.alaya_ws_block_stats(ctypes.byref(self.params), self.seqs, self.B,
                                          self.ws.data_ptr())
        off = p - self.ws.data_ptr()
        v = self.ws[off:off + 8].view(torch.int32).tolist()
        return int(v[0]), int(v[1])

    def candidate_counts(self, chunk: int) -> torch.Tensor:
        """Candidate-superset sizes of the last scan: int32 ``[chunks, G, 4]`` (diagnostics;
        ``chunk`` = the tokens per work chunk the call used)."""
        p = self.lib.alaya_ws_candidate_counts(ctypes.byref(self.params), self.seqs, self.B,
                                               self.ws.data_ptr())
        off = p - self.ws.data_ptr()
        g = self.params.n_query_heads // self.params.n_kv_heads
        nch = sum((self.seqs[i].n + chunk - 1) // chunk for i in range(self.B))
        return self.ws[off:off + 16 * g * nch * self.params.n_kv_heads].view(torch.int32).view(-1, g, 4)

    def status(self) -> int:
        """Device status word of the last dipr_attention (synchronises)."""
        return int(self.ws[:4].view(torch.int32).item())

    def scan(self, q: torch.Tensor) -> torch.Tensor:
        q = self._q(q)
        smax = torch.empty(self.B, self.params.n_query_heads, dtype=torch.float32,
                           device=self.device)
        check(self.lib.alaya_scan(ctypes.byref(self.params), self.seqs, self.B, q.data_ptr(),
                                  smax.data_ptr(), self.ws.data_ptr(), self.ws_bytes,
                                  self.stream))
        self._q_keep = q
        return smax

    def attend(self, q: torch.Tensor, smax: torch.Tensor, want_values: bool = True):
        q = self._q(q)
        smax = smax.to(device=self.device, dtype=torch.float32).contiguous()
        part = None
        if want_values:
            part = torch.empty(self.B * self.params.n_query_heads, self.params.dim + 2,
                               dtype=torch.float32, device=self.device)
        check(self.lib.alaya_attend(ctypes.byref(self.params), self.seqs, self.B, q.data_ptr(),
                                    smax.data_ptr(), part.data_ptr() if part is not None else None,
                                    int(want_values), self.ws.data_ptr(), self.ws_bytes,
                                    self.stream))
        self._q_keep = q
        return part

    def sharded_step(self, q: torch.Tensor, bufs, n_ranks: int, rank: int, cap: int, epoch: int,
                     err: torch.Tensor, gather_epoch: int = 0) -> torch.Tensor | bool | None:
        """Scan + global max over peer memory + attend in one launch sequence
        (``alaya_sharded_step``): ``[B*Hq, dim+2]`` partials filtered at the global
        max, or (``gather_epoch``) ``True`` once the partials were pushed to every
        rank's exchange slots; ``None`` when the call is not eligible."""
        q = self._q(q)
        part = None
        if not gather_epoch:
            part = torch.empty(self.B * self.params.n_query_heads, self.params.dim + 2,
                               dtype=torch.float32, device=self.device)
        rc = self.lib.alaya_sharded_step(ctypes.byref(self.params), self.seqs, self.B, q.data_ptr(),
                                         bufs, n_ranks, rank, cap, epoch, gather_epoch,
                                         part.data_ptr() if part is not None else None,
                                         err.data_ptr(), self.ws.data_ptr(), self.ws_bytes,
                                         self.stream)
        if rc == 6:  # ALAYA_ERR_UNSUPPORTED
            return None
        check(rc)
        self._q_keep = q
        return part if part is not None else True

    def topk(self, q: torch.Tensor, k: int, with_scores: bool = False):
        """Exact flat top-k per (seq, q head) (``FlatIndex.top_k``, ``index.py:60-66``):
        ``(ids [rows, k] int64, counts [rows] int32[, scores [rows, k] fp32])``,
        ids unordered within a row (global token ids)."""
        q = self._q(q)
        rows = self.B * self.params.n_query_heads
        ids = torch.empty(rows, k, dtype=torch.int64, device=self.device)
        cnt = torch.empty(rows, dtype=torch.int32, device=self.device)
        sc = torch.empty(rows, k, dtype=torch.float32, device=self.device) if with_scores else None
        check(self.lib.alaya_topk(ctypes.byref(self.params), self.seqs, self.B, q.data_ptr(), int(k),
                                  ids.data_ptr(), sc.data_ptr() if sc is not None else None, k,
                                  cnt.data_ptr(), self.ws.data_ptr(), self.ws_bytes, self.stream))
        self._q_keep = q
        return (ids, cnt, sc) if with_scores else (ids, cnt)

    def block_topk(self, q: torch.Tensor, indexes: list, block_size: int, k_blocks: int,
                   with_blocks: bool = False):
        """TOP_K on the coarse block index (``store.py:305-312``): token ids of the
        best ``k_blocks`` blocks per (seq, q head), clipped to the prefix.
        ``indexes[b]`` = ``(reps [Hkv, nb, r, d], n_tokens)`` of sequence b."""
        q = self._q(q)
        rows = self.B * self.params.n_query_heads
        arr = (AlayaBlockIndex * self.B)()
        for i, (reps, n_tok) in enumerate(indexes):
            if reps.dtype != self._dtype or not reps.is_contiguous() or reps.dim() != 4:
                raise ValueError("block reps must be a contiguous [Hkv, blocks, r, d] tensor")
            arr[i].reps, arr[i].head_stride = reps.data_ptr(), reps.stride(0)
            arr[i].n_tokens, arr[i].n_blocks, arr[i].r = int(n_tok), reps.shape[1], reps.shape[2]
        nb_max = max(int(r.shape[1]) for r, _ in indexes)
        cap = max(1, min(k_blocks, nb_max) * block_size)
        ids = torch.empty(rows, cap, dtype=torch.int64, device=self.device)
        cnt = torch.empty(rows, dtype=torch.int32, device=self.device)
        blk = sc = None
        if with_blocks:
            blk = torch.full((rows, k_blocks), -1, dtype=torch.int32, device=self.device)
            sc = torch.empty(rows, k_blocks, dtype=torch.float32, device=self.device)
        check(self.lib.alaya_block_topk(ctypes.byref(self.params), self.seqs, arr, self.B,
                                        int(block_size), int(k_blocks), q.data_ptr(), ids.data_ptr(),
                                        cap, cnt.data_ptr(),
                                        blk.data_ptr() if blk is not None else None,
                                        sc.data_ptr() if sc is not None else None, self.stream))
        self._q_keep = q
        return (ids, cnt, blk, sc) if with_blocks else (ids, cnt)

    def diprs(self, q: torch.Tensor, graphs: list, l0: int, floor_mode: int = 0,
              floors: torch.Tensor | None = None):
        """Graph DIPRS per (seq, q head) (``dipr.py:265-289``): ``graphs[b]`` =
        ``(offsets [Hkv, n+1] int64, nbrs [Hkv, E] int32, entry [Hkv] int32)`` over
        sequence b's prefix. floor_mode 0 none, 1 window-cache max, 2 ``floors``.
        Returns ``(ids [rows, n] int64 (unordered), counts, explored)``."""
        q = self._q(q)
        rows = self.B * self.params.n_query_heads
        arr = (AlayaGraph * self.B)()
        keep = []
        for i, (off, nb, ent) in enumerate(graphs):
            if off.dtype != torch.int64 or nb.dtype != torch.int32 or ent.dtype != torch.int32:
                raise ValueError("graph arrays must be int64 offsets, int32 nbrs and entry")
            off, nb, ent = off.contiguous(), nb.contiguous(), ent.contiguous()
            keep += [off, nb, ent]
            arr[i].offsets, arr[i].nbrs, arr[i].entry = off.data_ptr(), nb.data_ptr(), ent.data_ptr()
            arr[i].offsets_head_stride, arr[i].nbrs_head_stride = off.stride(0), max(1, nb.stride(0))
            arr[i].n_nodes = off.shape[1] - 1
        cap = max(1, max(int(self.seqs[i].n) for i in range(self.B)))
        nbytes = self.lib.alaya_diprs_workspace_bytes(ctypes.byref(self.params), self.seqs, arr, self.B)
        if nbytes == 0:
            check(_lib.ALAYA_ERR_ARG)
        ws = self.ws if self.ws.numel() >= nbytes else _DWS.get(nbytes, self.device)
        ids = torch.empty(rows, cap, dtype=torch.int64, device=self.device)
        cnt = torch.empty(rows, dtype=torch.int32, device=self.device)
        exp = torch.empty(rows, dtype=torch.int32, device=self.device)
        fl = None
        if floor_mode == 2:
            fl = floors.to(device=self.device, dtype=torch.float32).contiguous()
        check(self.lib.alaya_diprs(ctypes.byref(self.params), self.seqs, arr, self.B, q.data_ptr(),
                                   int(l0), int(floor_mode), fl.data_ptr() if fl is not None else None,
                                   ids.data_ptr(), cap, cnt.data_ptr(), exp.data_ptr(), ws.data_ptr(),
                                   ws.numel(), self.stream))
        self._q_keep = (q, keep, fl)
        return ids, cnt, exp

    def sparse_attention(self, q: torch.Tensor, ids: torch.Tensor, counts: torch.Tensor,
                         out: torch.Tensor | None = None):
        """Attention over explicit base ids minus the window ids, merged with the
        window partial (``store.py:268-293``) -> ``(out [B, Hq, d], selected counts)``."""
        q = self._q(q)
        if out is None:
            out = torch.empty_like(q)
        rows = self.B * self.params.n_query_heads
        if ids.dtype != torch.int64 or ids.dim() != 2 or ids.shape[0] != rows or not ids.is_contiguous():
            raise ValueError(f"ids must be a contiguous int64 [{rows}, cap] tensor")
        nsel = torch.empty(rows, dtype=torch.int32, device=self.device)
        status = self.ws[:4].view(torch.int32)
        status.zero_()
        check(self.lib.alaya_sparse_attention(ctypes.byref(self.params), self.seqs, self.B,
                                              q.data_ptr(), ids.data_ptr(), ids.shape[1],
                                              counts.data_ptr(), out.data_ptr(), nsel.data_ptr(),
                                              status.data_ptr(), self.stream))
        self._q_keep = q
        return out, nsel

    def selected(self, cap: int):
        """Per (seq, q head) selected ids (ascending, global) + counts; after attend/attention."""
        rows = self.B * self.params.n_query_heads
        ids = torch.empty(rows, max(cap, 1), dtype=torch.int64, device=self.device)
        nsel = torch.empty(rows, dtype=torch.int32, device=self.device)
        nret = torch.empty(rows, dtype=torch.int32, device=self.device)
        check(self.lib.alaya_selected(ctypes.byref(self.params), self.seqs, self.B, ids.data_ptr(),
                                      ids.shape[1], nsel.data_ptr(), nret.data_ptr(),
                                      self.ws.data_ptr(), self.ws_bytes, self.stream))
        # rows come back ascending from the kernel (the reference's diagnostics are
        # sorted, store.py:289); only the first nsel[row] entries of a row are written
        return ids, nsel, nret


def merge_partials(parts: torch.Tensor, dim: int, status: torch.Tensor | None = None
                   ) -> torch.Tensor:
    """Merge ``parts [R, rows, dim+2]`` in order and finalize -> ``[rows, dim]``."""
    require_cuda()
    lib = _lib.load()
    parts = parts.to(torch.float32).contiguous()
    R, rows = parts.shape[0], parts.shape[1]
    out = torch.empty(rows, dim, dtype=torch.float32, device=parts.device)
    check(lib.alaya_merge_partials(parts.data_ptr(), R, rows, dim, out.data_ptr(),
                                   status.data_ptr() if status is not None else None,
                                   torch.cuda.current_stream(parts.device).cuda_stream))
    return out


def merge_states(parts: torch.Tensor, dim: int) -> torch.Tensor:
    """Merge ``parts [R, rows, dim+2]`` in order -> state ``[rows, dim+2]`` (no finalize)."""
    require_cuda()
    lib = _lib.load()
    parts = parts.to(torch.float32).contiguous()
    R, rows = parts.shape[0], parts.shape[1]
    out = torch.empty(rows, dim + 2, dtype=torch.float32, device=parts.device)
    check(lib.alaya_merge_states(parts.data_ptr(), R, rows, dim, out.data_ptr(),
                                 torch.cuda.current_stream(parts.device).cuda_stream))
    return out


def append_array(seqs: list[SeqView], params: AlayaParams, dtype: torch.dtype):
    """Validated ``alaya_seq`` descriptors of window rings for ``window_append_raw``."""
    arr = (AlayaSeq * len(seqs))()
    for i, s in enumerate(seqs):
        _check_kv(s.wk, "wk", dtype, params.dim)
        _check_kv(s.wv, "wv", dtype, params.dim)
        e = arr[i]
        e.wk, e.wv, e.w_head_stride = s.wk.data_ptr(), s.wv.data_ptr(), s.wk.stride(0)
        e.w = _window_rows(s)
        e.d_w = _w_dev_ptr(s)
    return arr


def window_append_raw(arr, n: int, params: AlayaParams, k: torch.Tensor, v: torch.Tensor) -> None:
    lib = _lib.load()
    k = k.to(torch.float32).contiguous()
    v = v.to(torch.float32).contiguous()
    check(lib.alaya_window_append(ctypes.byref(params), arr, n, k.data_ptr(), v.data_ptr(),
                                  torch.cuda.current_stream(k.device).cuda_stream))


def window_append(seqs: list[SeqView], params: AlayaParams, dtype: torch.dtype,
                  k: torch.Tensor, v: torch.Tensor) -> None:
    """Append ``k``/``v`` ``[B, Hkv, d]`` (fp32) as row ``seqs[b].w`` of each
    sequence's window ring (``Session.update``, reference ``store.py:179-181``)."""
    require_cuda()
    window_append_raw(append_array(seqs, params, dtype), len(seqs), params, k, v)


def block_bounds(k: torch.Tensor) -> torch.Tensor:
    """Coarse block index of a ``[Hkv, n, d]`` key slab -> ``[Hkv, ceil(n/128), 5, d]``
    in the key dtype: per 128-token block the per-dim min and max, the mean, the
    largest-norm key (reference representative, ``index.py:217-228``) and the
    radius ``max ||k - mean||`` (row 4, element 0, rounded up)."""
    require_cuda()
    lib = _lib.load()
    if k.dtype not in _DTYPES:
        raise ValueError(f"unsupported KV dtype {k.dtype}")
    if k.dim() != 3 or k.stride(2) != 1 or k.stride(1) != k.shape[2]:
        raise ValueError("keys must be [heads, rows, d] with unit row stride")
    hkv, n, d = k.shape
    out = torch.empty(hkv, (n + 127) // 128, 5, d, dtype=k.dtype, device=k.device)
    check(lib.alaya_block_bounds(k.data_ptr(), _DTYPES[k.dtype], hkv, k.stride(0), n, d,
                                 out.data_ptr(), out.stride(0),
                                 torch.cuda.current_stream(k.device).cuda_stream))
    return out


def block_reps(k: torch.Tensor, block_size: int, r: int) -> torch.Tensor:
    """BlockIndex representatives of a ``[Hkv, n, d]`` key slab (``index.py:217-243``):
    ``[Hkv, ceil(n/block_size), r, d]`` in the key dtype, per block the r keys of
    largest L2 norm (ties by position; a short block repeats its first)."""
    require_cuda()
    lib = _lib.load()
    if k.dtype not in _DTYPES:
        raise ValueError(f"unsupported KV dtype {k.dtype}")
    if k.dim() != 3 or k.stride(2) != 1 or k.stride(1) != k.shape[2]:
        raise ValueError("keys must be [heads, rows, d] with unit row stride")
    if block_size < 1 or r < 1:
        raise ValueError("block_size and r must be positive")
    hkv, n, d = k.shape
    nb = (n + block_size - 1) // block_size
    out = torch.empty(hkv, nb, r, d, dtype=k.dtype, device=k.device)
    check(lib.alaya_block_reps(k.data_ptr(), _DTYPES[k.dtype], hkv, k.stride(0), n, d, block_size,
                               r, out.data_ptr(), out.stride(0),
                               torch.cuda.current_stream(k.device).cuda_stream))
    return out
