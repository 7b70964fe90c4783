"""Parity rules shared by the GPU tests (BASELINE.json north_star).

* Sets: the GPU's selected base ids equal the reference's
  ``{s >= max(s) - beta} \\ window`` (``dipr.py:63-66``, ``store.py:271-273``)
  except tokens whose fp64 score lies within ``eps`` of the threshold
  (1e-4 fp32 CUDA-core scan, 1e-3 bf16 split-q tcgen05 scan).
* Outputs: norm-relative error <= 1e-5 (fp32 mode) / 2e-2 (bf16 mode), with the
  oracle evaluated on the GPU-returned selection so that an epsilon-boundary
  flip is not counted as an arithmetic error.
"""

from __future__ import annotations

import numpy as np

from oracle import alaya_oracle as O

EPS_SET = {"float32": 1e-4, "bfloat16": 1e-3}
TOL_OUT = {"float32": 1e-5, "bfloat16": 2e-2}


def rel(a, b) -> float:
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


def set_flips(got, scores: np.ndarray, beta: float, eps: float, window_ids=None, offset: int = 0):
    """Check one head's selection against the epsilon rule.

    ``scores`` are the fp64 scores of the head over ITS base prefix (global
    ids ``offset + i``); ``got`` the GPU's selected global ids (window ids
    excluded, as ``selected_base``). Returns ``(flips, worst_margin)``: the
    number of differing ids and the largest ``|s - thr|`` among them. Raises
    AssertionError naming the first id outside the epsilon band.
    """
    thr = float(scores.max()) - beta
    want = np.flatnonzero(scores >= thr) + offset
    if window_ids is not None and len(window_ids):
        want = np.setdiff1d(want, np.asarray(window_ids, np.int64))
    got = np.unique(np.asarray(got, np.int64))
    diff = np.setxor1d(got, want)
    if diff.size == 0:
        return 0, 0.0
    margins = np.abs(scores[diff - offset] - thr)
    worst = float(margins.max())
    bad = diff[margins > eps]
    assert bad.size == 0, (f"{bad.size} ids outside the eps={eps} band, e.g. id {int(bad[0])} "
                           f"margin {float(np.abs(scores[bad[0] - offset] - thr)):.3e}")
    return int(diff.size), worst


def retrieved_ok(got_retrieved: int, scores: np.ndarray, beta: float, eps: float) -> bool:
    """``retrieved`` count (window ids included) differs from the reference's
    ``|{s >= max - beta}|`` by at most the tokens inside the epsilon band."""
    thr = float(scores.max()) - beta
    want = int(np.count_nonzero(scores >= thr))
    band = int(np.count_nonzero(np.abs(scores - thr) <= eps))
    return abs(int(got_retrieved) - want) <= band
