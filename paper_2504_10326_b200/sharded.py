"""Sequence-sharded decode over several GPUs of one box (north star item 4).

Rank ``r`` of ``R`` holds tokens ``[lo_r, hi_r)`` of every sequence's base
prefix (``shard_bounds``); global ids are ``token_offset + local row``, the
same idea as ``dipr_bruteforce(token_ids=...)`` in the reference
(``dipr.py:51,67-70``). Per layer:

1. local scan -> per (sequence, q head) local max (``alaya_scan``);
2. ``all_reduce(MAX)`` of ``[B, Hq]`` fp32 -> exactly the reference's global
   ``scores.max()`` over the whole prefix (``dipr.py:64``);
3. local exact filter at the global ``max - beta``, V gather and the window
   rows this shard owns (base ids ``[0, initial)`` live on the shard holding
   them, ``[p - last, p)`` likewise, session rows on the last rank) ->
   one (m, l, acc) partial per q head (``alaya_attend``);
4. ``all_gather`` of the partials and an in-order ``PartialAttention.merge``
   + ``finalize`` (``attention.py:128-152``; merge is associative and
   commutative, reference ``tests/test_attention.py:162-182``).

Both collectives are latency-bound (128 B and ~16.6 KB per rank at B=1,
Llama shape). The orchestration is generic over the local stages so that
CPU (gloo) tests can drive it with a host double; the product path passes
:class:`EngineStages`, i.e. the CUDA kernels.
"""

from __future__ import annotations

import ctypes
import os
from typing import Protocol

import torch
import torch.distributed as dist

from . import engine


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous split of ``n`` tokens; the first ``n % world`` shards get one more."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class LocalStages(Protocol):
    def scan(self, q: torch.Tensor) -> torch.Tensor: ...            # [B, Hq] local max
    def attend(self, q: torch.Tensor, smax: torch.Tensor) -> torch.Tensor: ...  # [B*Hq, d+2]
    def merge(self, parts: torch.Tensor) -> torch.Tensor: ...       # [R, B*Hq, d+2] -> [B*Hq, d]


class EngineStages:
    """The CUDA kernels behind :class:`LocalStages` for one layer's local shards."""

    def __init__(self, seqs: list[engine.SeqView], params, dtype: torch.dtype,
                 device: torch.device):
        self.call = engine.Call(seqs, params, dtype, device)
        self.dim = params.dim

    @classmethod
    def from_call(cls, call: engine.Call) -> "EngineStages":
        self = cls.__new__(cls)
        self.call, self.dim = call, call.params.dim
        return self

    def scan(self, q):
        return self.call.scan(q)

    def attend(self, q, smax):
        return self.call.attend(q, smax, want_values=True)

    def merge(self, parts):
        return engine.merge_partials(parts, self.dim)

    def fused(self, q, exchange: "PeerExchange", gather: bool = False):
        """Scan -> max over peers -> attend as one launch sequence (the max
        travels over NVLink per (seq, kv head) group as the scan completes it).
        Returns the local partials, or with ``gather`` the merged output
        ``[B*Hq, d]`` (the combine pushes the partials to every rank, the merge
        waits for the ranks' flags: no collective kernel at all). ``None`` when
        not eligible."""
        rows = q.shape[0] * q.shape[1]
        if rows > exchange.cap or (gather and rows * (self.dim + 2) > exchange.cap):
            return None
        e, ge = exchange.epoch[0] + 1, (exchange.epoch[1] + 1 if gather else 0)
        part = self.call.sharded_step(q, exchange._arr, exchange.world, exchange.rank, exchange.cap,
                                      e, exchange.err, ge)
        self.fused_used = part is not None
        if part is None:
            return None
        exchange.epoch[0] = e
        if not gather:
            return part
        exchange.epoch[1] = ge
        return exchange.merge_exchanged(rows, self.dim, ge)


def _staged(t: torch.Tensor, group) -> tuple[torch.Tensor, bool]:
    """gloo cannot run these collectives on CUDA tensors: stage through host."""
    if t.is_cuda and dist.get_backend(group) == "gloo":
        return t.cpu(), True
    return t, False


class PeerExchange:
    """The two collectives over peer memory instead of NCCL (``alaya_exch``):
    every rank owns one symmetric device buffer, exports its CUDA IPC handle,
    maps every peer's buffer (NVLink P2P) and exchanges by direct stores plus
    release/acquire epoch flags. Messages up to ``cap`` floats. Build it
    collectively on every rank of ``group``; ``None`` from :meth:`create` means
    peer mapping is unavailable (the caller keeps NCCL)."""

    def __init__(self, bufs: list[int], own: int, rank: int, world: int, cap: int,
                 device: torch.device, opened: list[int]):
        self.bufs, self.own, self.rank, self.world, self.cap = bufs, own, rank, world, cap
        self.device = device
        self._opened = opened
        self.epoch = [0, 0]
        self.fused = os.environ.get("ALAYA_FUSED_SHARD", "1") != "0"  # scan+max+attend fused
        self.err = torch.zeros(1, dtype=torch.int32, device=device)
        self._arr = (ctypes.c_void_p * world)(*bufs)

    @classmethod
    def create(cls, group, cap: int, device: torch.device) -> "PeerExchange | None":
        from . import _lib
        lib = _lib.load()
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        nbytes = lib.alaya_exch_bytes(world, cap)
        ok, own, handle = False, ctypes.c_void_p(), (ctypes.c_char * 64)()
        if nbytes:
            with torch.cuda.device(device):
                ok = lib.alaya_exch_alloc(nbytes, ctypes.byref(own), handle) == 0
        handles = [None] * world
        dist.all_gather_object(handles, bytes(handle) if ok else None, group=group)
        if not all(h is not None for h in handles):
            return None
        bufs, opened, good = [], [], True
        with torch.cuda.device(device):
            for r, h in enumerate(handles):
                if r == rank:
                    bufs.append(own.value)
                    continue
                ptr = ctypes.c_void_p()
                hb = (ctypes.c_char * 64).from_buffer_copy(h)
                if lib.alaya_exch_open(hb, ctypes.byref(ptr)) != 0:
                    good = False
                    break
                bufs.append(ptr.value)
                opened.append(ptr.value)
        flags = [None] * world
        dist.all_gather_object(flags, good, group=group)
        if not all(flags):
            return None
        dist.barrier(group=group)
        return cls(bufs, own.value, rank, world, cap, device, opened)

    def _run(self, kind: int, local: torch.Tensor, out: torch.Tensor | None) -> int:
        from . import _lib
        local = local.to(torch.float32).contiguous()
        if local.numel() > self.cap:
            raise ValueError(f"exchange of {local.numel()} floats > cap {self.cap}")
        self.epoch[kind] += 1
        e = self.epoch[kind]
        _lib.check(_lib.load().alaya_exch(self._arr, self.world, self.rank, self.cap, kind,
                                          local.data_ptr(), local.numel(), e,
                                          out.data_ptr() if out is not None else None,
                                          self.err.data_ptr(),
                                          torch.cuda.current_stream(self.device).cuda_stream))
        self._keep = local
        return e

    def allreduce_max(self, local: torch.Tensor) -> torch.Tensor:
        out = torch.empty_like(local, dtype=torch.float32)
        self._run(0, local, out)
        return out.view(local.shape)

    def allgather(self, local: torch.Tensor) -> torch.Tensor:
        """``[world, *local.shape]`` view of this rank's slots (valid until the
        exchange after next of this kind)."""
        from . import _lib
        e = self._run(1, local, None)
        ptr = _lib.load().alaya_exch_slots(self.own, self.world, self.cap, 1, e)
        n = local.numel()
        flat = _tensor_at(ptr, self.world * self.cap, self.device)
        return flat.view(self.world, self.cap)[:, :n].reshape((self.world,) + tuple(local.shape))

    def merge_exchanged(self, rows: int, dim: int, epoch: int) -> torch.Tensor:
        """Wait for every rank's kind-1 flag at ``epoch`` and merge the pushed
        partials (``alaya_merge_exchanged``) -> ``[rows, dim]``."""
        from . import _lib
        out = torch.empty(rows, dim, dtype=torch.float32, device=self.device)
        _lib.check(_lib.load().alaya_merge_exchanged(
            self.own, self.world, self.cap, epoch, rows, dim, out.data_ptr(), None,
            self.err.data_ptr(), torch.cuda.current_stream(self.device).cuda_stream))
        return out

    def check(self) -> None:
        if int(self.err.item()):
            raise RuntimeError("peer exchange timed out: a rank never arrived")

    def close(self) -> None:
        """Unmap the peers' buffers and free this rank's (after a barrier, so no
        peer still writes into it)."""
        from . import _lib
        lib = _lib.load()
        torch.cuda.synchronize(self.device)
        for p in self._opened:
            lib.alaya_exch_close(ctypes.c_void_p(p))
        self._opened = []
        if self.own:
            lib.alaya_exch_free(ctypes.c_void_p(self.own))
            self.own = 0


def _tensor_at(ptr: int, numel: int, device: torch.device) -> torch.Tensor:
    """A float32 tensor over existing device memory (no copy, not owned)."""
    class _Arr:
        __cuda_array_interface__ = {"shape": (numel,), "typestr": "<f4", "data": (ptr, False),
                                    "version": 3, "strides": None}
    return torch.as_tensor(_Arr(), device=device)


def sharded_attention(stages: LocalStages, q: torch.Tensor, group=None,
                      exchange: PeerExchange | None = None) -> torch.Tensor:
    """One decode step of one layer over sequence-sharded KV -> ``[B, Hq, d]``
    (identical on every rank). With ``exchange`` the two collectives run over
    peer memory: fused into the kernels (``alaya_sharded_step`` +
    ``alaya_merge_exchanged``) when the call is tcgen05-eligible, else as
    ``alaya_exch`` kernels; without, through ``torch.distributed``."""
    if exchange is not None:
        fused = getattr(stages, "fused", None) if exchange.fused else None
        out = fused(q, exchange, gather=True) if fused is not None else None
        if out is not None:
            return out.view(q.shape[0], q.shape[1], -1)
        smax = exchange.allreduce_max(stages.scan(q))
        part = stages.attend(q, smax).contiguous()
        parts = exchange.allgather(part)
        out = stages.merge(parts)
        return out.view(q.shape[0], q.shape[1], -1)
    world = dist.get_world_size(group)
    smax = stages.scan(q)
    sm, moved = _staged(smax, group)
    dist.all_reduce(sm, op=dist.ReduceOp.MAX, group=group)
    if moved:
        smax.copy_(sm)
    part = stages.attend(q, smax).contiguous()
    pt, moved = _staged(part, group)
    parts = torch.empty((world * pt.shape[0],) + tuple(pt.shape[1:]), dtype=pt.dtype,
                        device=pt.device)
    dist.all_gather_into_tensor(parts, pt, group=group)
    if moved:
        parts = parts.to(part.device)
    out = stages.merge(parts.view((world,) + tuple(part.shape)))
    return out.view(q.shape[0], q.shape[1], -1)


def local_view(k_full: torch.Tensor, v_full: torch.Tensor, world: int, rank: int,
               wk: torch.Tensor | None = None, wv: torch.Tensor | None = None,
               w: int = 0) -> engine.SeqView:
    """This rank's shard of one sequence at one layer. ``k_full`` is
    ``[Hkv, n, d]``; the session window (``wk``/``wv``, ``w`` rows) is owned by
    the last rank."""
    n = k_full.shape[1]
    lo, hi = shard_bounds(n, world, rank)
    last = rank == world - 1
    return engine.SeqView(k=k_full[:, lo:hi], v=v_full[:, lo:hi], n=hi - lo,
                          wk=wk if last else None, wv=wv if last else None,
                          w=w if last else 0, token_offset=lo, prefix_len=n)
