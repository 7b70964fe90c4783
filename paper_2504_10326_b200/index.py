"""Flat index (reference ``sparsekv/index.py:42-70``) over device-resident keys.

The reference's ``FlatIndex`` keeps an fp64 copy of K (``index.py:48-50``);
here the keys stay in HBM in their storage dtype and the scan kernel
accumulates in fp32. Graph construction and the coarse ``BlockIndex``
heuristic are out of scope.
"""

from __future__ import annotations

import numpy as np
import torch

from . import dipr as _dipr


class FlatIndex:
    """Dense key array scanned exhaustively; token ids are 0..n-1."""

    def __init__(self, keys, device=None):
        k = keys if isinstance(keys, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(np.atleast_2d(keys), dtype=np.float32))
        self.keys = k.to(device or "cuda").contiguous()

    @property
    def n(self) -> int:
        return self.keys.shape[0]

    def dipr(self, q, beta: float) -> set[int]:
        """Exact DIPR result (``index.py:68-70``)."""
        return _dipr.dipr_bruteforce(q, self.keys, beta)
