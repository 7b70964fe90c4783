"""Attention API of the reference (``sparsekv/attention.py``) on the B200 kernels.

``PartialAttention`` keeps its (m, l, acc) state as a device tensor
``[d + 2]``; ``over`` runs the window-row path of the combine stage,
``merge``/``finalize`` the merge stage. ``full_attention`` is the decode
kernel with every token selected (beta = +inf, no window).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import engine


def _dev(x, device, dtype=None) -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
    t = t.to(device)
    if dtype is not None:
        t = t.to(dtype)
    elif t.dtype not in (torch.float32, torch.bfloat16):
        t = t.float()
    return t.contiguous()


def _rows(keys, values, device):
    k = _dev(keys, device)
    v = _dev(values, device, k.dtype)
    if k.dim() == 1:
        k = k.reshape(1, -1)
    if v.dim() == 1:
        v = v.reshape(1, -1)
    if k.shape[0] != v.shape[0]:
        raise ValueError(f"keys/values length mismatch: {k.shape[0]} vs {v.shape[0]}")
    return k, v


def full_attention(q, keys, values, device=None) -> np.ndarray:
    """Exact softmax attention (reference ``attention.py:25-42``)."""
    engine.require_cuda()
    device = torch.device(device or "cuda")
    k, v = _rows(keys, values, device)
    n, d = k.shape
    if n == 0:
        raise ValueError("attention over an empty key set is undefined")
    params = engine.make_params(1, 1, d, k.dtype, math.inf, 0, 0)
    call = engine.Call([engine.SeqView(k=k.unsqueeze(0), v=v.unsqueeze(0), n=n)], params,
                       k.dtype, device)
    out = call.dipr_attention(_dev(q, device, torch.float32).reshape(1, 1, d))
    o = out.reshape(d).cpu().numpy()
    if call.status() != 0 or not np.isfinite(o).all():
        raise FloatingPointError("attention output is non-finite")
    return o


def sparse_attention(q, selected) -> np.ndarray:
    """Attention over an explicit ``(token_id, key, value)`` list (``attention.py:45-60``)."""
    if not selected:
        raise ValueError("sparse attention requires a nonempty selection")
    ids = [t for t, _, _ in selected]
    if len(set(ids)) != len(ids):
        raise ValueError("duplicate token id in selection")
    keys = np.stack([np.asarray(k, dtype=np.float32) for _, k, _ in selected])
    values = np.stack([np.asarray(v, dtype=np.float32) for _, _, v in selected])
    return full_attention(q, keys, values)


class PartialAttention:
    """Online-softmax state (m, l, acc) over a token subset (``attention.py:80-152``).

    The empty state (no token absorbed) merges as the identity.
    """

    def __init__(self, state: torch.Tensor | None = None):
        self.state = state  # device [d + 2] = (m, l, acc...) or None when empty

    @classmethod
    def empty(cls) -> "PartialAttention":
        return cls()

    @property
    def is_empty(self) -> bool:
        return self.state is None

    @property
    def m(self) -> float:
        return -math.inf if self.state is None else float(self.state[0].item())

    @property
    def l(self) -> float:
        return 0.0 if self.state is None else float(self.state[1].item())

    @property
    def acc(self):
        return None if self.state is None else self.state[2:].double().cpu().numpy()

    @classmethod
    def over(cls, q, keys, values, device=None) -> "PartialAttention":
        """Absorb a token group (``attention.py:98-110``)."""
        engine.require_cuda()
        device = torch.device(device or "cuda")
        k, v = _rows(keys, values, device)
        n, d = k.shape
        if n == 0:
            return cls.empty()
        params = engine.make_params(1, 1, d, k.dtype, 0.0, 0, 0)
        seq = engine.SeqView(k=None, v=None, n=0, wk=k.unsqueeze(0), wv=v.unsqueeze(0), w=n,
                             prefix_len=0)
        call = engine.Call([seq], params, k.dtype, device)
        qd = _dev(q, device, torch.float32).reshape(1, 1, d)
        smax = torch.full((1, 1), -math.inf, device=device)
        part = call.attend(qd, smax, want_values=True)
        return cls(part[0])

    def merge(self, other: "PartialAttention") -> "PartialAttention":
        """Combine two partials over disjoint token sets (``attention.py:128-143``)."""
        if self.is_empty:
            return other
        if other.is_empty:
            return self
        if self.state.shape != other.state.shape:
            raise ValueError("cannot merge partials of different dimension")
        d = self.state.numel() - 2
        return PartialAttention(engine.merge_states(torch.stack([self.state, other.state])
                                                    .reshape(2, 1, d + 2), d)[0])

    def finalize(self) -> np.ndarray:
        """``acc / l`` as float32 (``attention.py:145-152``)."""
        if self.is_empty:
            raise ValueError("cannot finalize an empty partial")
        d = self.state.numel() - 2
        status = torch.zeros(1, dtype=torch.int32, device=self.state.device)
        o = engine.merge_partials(self.state.reshape(1, 1, d + 2), d, status)
        out = o.reshape(d).cpu().numpy()
        if int(status.item()) != 0:
            raise FloatingPointError("partial attention finalized to non-finite output")
        return out
