"""DIPR retrieval (reference ``sparsekv/dipr.py``) on the B200 kernels.

``dipr_bruteforce`` runs the scan + exact-filter stages of the C-ABI over a
single (q, keys) pair; the batched decode path lives in :mod:`.store`.
The graph search (``diprs``/``traverse``/``CandidateList``) is out of scope.
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
