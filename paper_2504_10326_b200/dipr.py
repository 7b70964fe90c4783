"""DIPR retrieval (reference ``sparsekv/dipr.py``) on the B200 kernels.

``dipr_bruteforce`` runs the scan + exact-filter stages of the C-ABI over a
single (q, keys) pair; the batched decode path lives in :mod:`.store`.
The graph search (``diprs``, ``dipr.py:107-289``) runs on the device as
``alaya_diprs`` (decision-identical walk over a ``GraphIndex``); only graph
CONSTRUCTION (``index.py:245-639``) is out of scope.
"""

from __future__ import annotations

import math
from typing import Iterable

import numpy as np
import torch

from . import engine


def alpha_to_beta(alpha: float, d: int) -> float:
    """``beta = -sqrt(d) ln(alpha)`` (reference ``dipr.py:29-39``)."""
    if not 0.0 < alpha <= 1.0:
        raise ValueError(f"alpha must be in (0, 1], got {alpha}")
    if d < 1:
        raise ValueError(f"dimension must be positive, got {d}")
    return -math.sqrt(d) * math.log(alpha)


def is_critical_by_attention(a_j: float, a_max: float, alpha: float) -> bool:
    """``a_j >= alpha * a_max`` (reference ``dipr.py:42-44``)."""
    return a_j >= alpha * a_max


def _device_keys(keys, device) -> torch.Tensor:
    if isinstance(keys, torch.Tensor):
        t = keys.to(device)
        if t.dtype not in (torch.float32, torch.bfloat16):
            t = t.float()
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.atleast_2d(keys), dtype=np.float32)).to(device)
    return t.contiguous()


def dipr_ids(q, keys, beta: float, device=None) -> torch.Tensor:
    """Ascending critical ids (device int64) of ``s_j >= max s - beta``."""
    engine.require_cuda()
    device = torch.device(device or "cuda")
    k = _device_keys(keys, device)
    if k.dim() == 1:
        k = k.reshape(1, -1)
    n, d = k.shape
    if n == 0:
        raise ValueError("DIPR over an empty key set is undefined")
    if beta < 0:
        raise ValueError(f"beta must be non-negative, got {beta}")
    qt = torch.as_tensor(np.asarray(q, dtype=np.float32) if not isinstance(q, torch.Tensor) else q)
    qt = qt.to(device=device, dtype=torch.float32).reshape(1, 1, d)
    params = engine.make_params(1, 1, d, k.dtype, beta, 0, 0)
    seq = engine.SeqView(k=k.unsqueeze(0), v=k.unsqueeze(0), n=n)
    call = engine.Call([seq], params, k.dtype, device)
    smax = call.scan(qt)
    call.attend(qt, smax, want_values=False)
    ids, nsel, _ = call.selected(cap=n)
    return ids[0, : int(nsel[0].item())]


def dipr_bruteforce(q, keys, beta: float, token_ids: Iterable[int] | None = None) -> set[int]:
    """Exact DIPR id set (reference ``dipr.py:47-70``), computed on the GPU."""
    ids = dipr_ids(q, keys, beta).cpu().numpy()
    if token_ids is None:
        return set(ids.tolist())
    tid = np.asarray(list(token_ids), dtype=np.int64)
    n = keys.shape[0] if keys.ndim == 2 else 1
    if tid.shape[0] != n:
        raise ValueError("token_ids length must match key count")
    return set(tid[ids].tolist())


def diprs(index, q, start: int, l0: int, beta: float, window_max: float | None = None) -> set[int]:
    """Approximate DIPR over a proximity graph (``dipr.py:265-289``): the
    candidate-list walk of ``traverse`` on the GPU (``alaya_diprs``), with the
    reference's acceptance rule and final cut ``s >= max(best, floor) - beta``."""
    engine.require_cuda()
    if l0 < 1:
        raise ValueError(f"capacity threshold must be >= 1, got {l0}")
    if beta < 0:
        raise ValueError(f"beta must be non-negative, got {beta}")
    n = index.n
    if n == 0:
        raise ValueError("search over an empty index")
    if not 0 <= start < n:
        raise ValueError(f"start node {start} out of range")
    k = index.keys
    d = k.shape[1]
    dev = k.device
    params = engine.make_params(1, 1, d, k.dtype, beta, 0, 0)
    call = engine.Call([engine.SeqView(k=k.unsqueeze(0), v=k.unsqueeze(0), n=n)], params, k.dtype, dev)
    qt = torch.as_tensor(np.asarray(q, dtype=np.float32) if not isinstance(q, torch.Tensor) else q)
    qt = qt.to(device=dev, dtype=torch.float32).reshape(1, 1, d)
    floors = None if window_max is None else torch.tensor([float(window_max)], device=dev)
    ids, cnt, _ = call.diprs(qt, [index.device_arrays(start)], l0, 0 if floors is None else 2, floors)
    c = int(cnt[0].item())
    if c < 0:
        raise _lib_error("graph walk scratch overflow")
    return set(ids[0, :c].cpu().numpy().tolist())


def _lib_error(msg):
    from ._lib import AlayaError
    return AlayaError(msg)
