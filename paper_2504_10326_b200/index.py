"""Flat and coarse indexes (reference ``sparsekv/index.py``) over device-resident keys.

The reference's ``FlatIndex`` keeps an fp64 copy of K (``index.py:48-50``);
here the keys stay in HBM in their storage dtype and the scan kernel
accumulates in fp32. ``BlockIndex`` (``index.py:195-243``) holds the
representatives as one device tensor ``[blocks, r, d]`` built by
``alaya_block_reps``; ``top_blocks`` runs ``alaya_block_topk``.
``GraphIndex`` holds a proximity graph as device CSR for ``dipr.diprs``
(``alaya_diprs``); graph construction is out of scope.
"""

from __future__ import annotations

import numpy as np
import torch

from . import dipr as _dipr
from . import engine


def _device_keys(keys, device) -> torch.Tensor:
    if isinstance(keys, torch.Tensor):
        t = keys.to(device)
        if t.dtype not in (torch.float32, torch.bfloat16):
            t = t.float()
        return t.contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.atleast_2d(keys), dtype=np.float32)).to(device)


def _q_tensor(q, d, device) -> torch.Tensor:
    qt = q if isinstance(q, torch.Tensor) else torch.from_numpy(np.asarray(q, dtype=np.float32))
    return qt.to(device=device, dtype=torch.float32).reshape(1, 1, d)


class FlatIndex:
    """Dense key array scanned exhaustively; token ids are 0..n-1."""

    def __init__(self, keys, device=None):
        engine.require_cuda()
        self.keys = _device_keys(keys, torch.device(device or "cuda"))

    @property
    def n(self) -> int:
        return self.keys.shape[0]

    def top_k(self, q, k: int) -> list[int]:
        """Exact top-k ids by inner product, descending, ties by smaller id
        (``index.py:60-66``). Selection on the GPU (``alaya_topk``); the k
        results are ordered on the host by (-score, id)."""
        if not 1 <= k <= self.n:
            raise ValueError(f"k must be in [1, {self.n}], got {k}")
        d = self.keys.shape[1]
        dev = self.keys.device
        params = engine.make_params(1, 1, d, self.keys.dtype, 0.0, 0, 0)
        seq = engine.SeqView(k=self.keys.unsqueeze(0), v=self.keys.unsqueeze(0), n=self.n)
        call = engine.Call([seq], params, self.keys.dtype, dev)
        ids, cnt, sc = call.topk(_q_tensor(q, d, dev), k, with_scores=True)
        c = int(cnt[0].item())
        ids, sc = ids[0, :c].cpu().numpy(), sc[0, :c].cpu().numpy()
        order = np.lexsort((ids, -sc.astype(np.float64)))
        return ids[order].tolist()

    def dipr(self, q, beta: float) -> set[int]:
        """Exact DIPR result (``index.py:68-70``)."""
        return _dipr.dipr_bruteforce(q, self.keys, beta)


class BlockIndex:
    """Coarse index: contiguous token blocks scored by representative vectors
    (``index.py:195-214``). ``reps`` is a device tensor ``[blocks, r, d]``."""

    def __init__(self, block_size: int, n: int, reps: torch.Tensor):
        self.block_size = int(block_size)
        self.n_tokens = int(n)
        self.reps_tensor = reps
        self.starts = np.arange(0, n, block_size, dtype=np.int64)
        self.ends = np.minimum(self.starts + block_size, n)

    @property
    def n_blocks(self) -> int:
        return int(self.starts.shape[0])

    @property
    def reps(self) -> list[np.ndarray]:
        """Per-block representatives as the reference lists them (min(r, len) rows)."""
        r = self.reps_tensor.float().cpu().numpy()
        return [r[i, : min(r.shape[1], int(e - s))] for i, (s, e) in
                enumerate(zip(self.starts, self.ends))]

    def top_blocks(self, q, k_blocks: int) -> list[tuple[int, int]]:
        """Best ``k_blocks`` token ranges by max representative inner product,
        ties by smaller start (``index.py:206-214``)."""
        if not 1 <= k_blocks <= self.n_blocks:
            raise ValueError(f"k_blocks must be in [1, {self.n_blocks}], got {k_blocks}")
        reps = self.reps_tensor
        d = reps.shape[-1]
        dev = reps.device
        params = engine.make_params(1, 1, d, reps.dtype, 0.0, 0, 0)
        # the sequence view only carries the prefix length (no K rows are read)
        seq = engine.SeqView(k=None, v=None, n=0, prefix_len=self.n_tokens)
        call = engine.Call([seq], params, reps.dtype, dev)
        _, _, blk, sc = call.block_topk(_q_tensor(q, d, dev), [(reps.unsqueeze(0), self.n_tokens)],
                                        self.block_size, k_blocks, with_blocks=True)
        blk, sc = blk[0].cpu().numpy(), sc[0].cpu().numpy()
        keep = blk >= 0
        blk, sc = blk[keep], sc[keep]
        order = np.lexsort((blk, -sc.astype(np.float64)))
        return [(int(self.starts[i]), int(self.ends[i])) for i in blk[order]]


class GraphIndex:
    """Fixed-max-degree proximity graph over one head's keys (``index.py:73-192``),
    held on the device as CSR: ``offsets [n+1]`` int64, ``nbrs`` int32. Built
    by the reference (``build_graph``) and persisted in AVDB index blocks, or
    given as arrays (``from_arrays``); graph construction itself is out of
    scope on the B200 engine."""

    def __init__(self, keys, adjacency, entry_point: int, max_degree: int, device=None):
        dev = torch.device(device or "cuda")
        self.keys = _device_keys(keys, dev)
        adjacency = [np.asarray(a, dtype=np.int32) for a in adjacency]
        degrees = np.array([a.size for a in adjacency], dtype=np.int64)
        flat = np.concatenate(adjacency) if degrees.sum() else np.empty(0, np.int32)
        self._set(degrees, flat, entry_point, max_degree)

    def _set(self, degrees, flat, entry_point, max_degree):
        dev = self.keys.device
        n = self.keys.shape[0]
        if degrees.shape[0] != n:
            raise ValueError("adjacency length != node count")
        if flat.size and (flat.min() < 0 or flat.max() >= n):
            raise ValueError("neighbour id out of range")
        if not 0 <= entry_point < n:
            raise ValueError("entry point out of range")
        off = np.zeros(n + 1, dtype=np.int64)
        off[1:] = np.cumsum(degrees)
        self.offsets = torch.from_numpy(off).to(dev)
        pad = flat if flat.size else np.zeros(1, np.int32)  # a C-ABI pointer even without edges
        self.nbrs = torch.from_numpy(np.ascontiguousarray(pad, dtype=np.int32)).to(dev)
        self.entry_point = int(entry_point)
        self.max_degree = int(max_degree)
        self._degrees = degrees.astype(np.int32)
        self._flat = np.ascontiguousarray(flat, dtype=np.int32)

    @classmethod
    def from_arrays(cls, keys, degrees, flat_neighbors, entry_point, max_degree, device=None):
        """``index.py:172-188``."""
        self = cls.__new__(cls)
        self.keys = _device_keys(keys, torch.device(device or "cuda"))
        self._set(np.asarray(degrees, dtype=np.int64), np.asarray(flat_neighbors, dtype=np.int32),
                  entry_point, max_degree)
        return self

    def to_arrays(self):
        return self._degrees.copy(), self._flat.copy()

    @property
    def n(self) -> int:
        return self.keys.shape[0]

    @property
    def adjacency(self) -> list[np.ndarray]:
        off = self.offsets.cpu().numpy()
        return [self._flat[off[i]:off[i + 1]] for i in range(self.n)]

    def neighbors(self, node: int) -> np.ndarray:
        off = self.offsets[node:node + 2].cpu().numpy()
        return self._flat[off[0]:off[1]]

    def device_arrays(self, start: int | None = None):
        """``(offsets [1, n+1], nbrs [1, E], entry [1])`` for ``Call.diprs``."""
        ent = torch.tensor([self.entry_point if start is None else int(start)], dtype=torch.int32,
                           device=self.keys.device)
        return self.offsets.unsqueeze(0), self.nbrs.unsqueeze(0), ent


def select_representatives(block_keys, r: int) -> np.ndarray:
    """The r keys with the largest L2 norms, ties by position (``index.py:217-228``)."""
    bk = _device_keys(block_keys, torch.device("cuda"))
    if not 1 <= r <= bk.shape[0]:
        raise ValueError(f"r must be in [1, {bk.shape[0]}], got {r}")
    reps = engine.block_reps(bk.unsqueeze(0), bk.shape[0], r)
    return reps[0, 0].cpu().numpy()


def build_block_index(keys, block_size: int, r: int) -> BlockIndex:
    """Partition 0..n-1 into contiguous blocks and pick representatives
    (``index.py:231-243``) on the GPU."""
    if block_size < 1:
        raise ValueError("block_size must be positive")
    k = _device_keys(keys, torch.device("cuda"))
    n = k.shape[0]
    reps = engine.block_reps(k.unsqueeze(0), block_size, r)[0]
    return BlockIndex(block_size, n, reps)
