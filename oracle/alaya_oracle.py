"""CPU oracle for the DIPR retrieval + sparse-attention hot path.

TEST INFRASTRUCTURE ONLY. This module is the checker, never the product:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it. The product
path (``paper_2504_10326_b200``) never imports anything under ``oracle/``
and fails loudly when its CUDA library is missing.

It is a numpy restatement of the reference package ``sparsekv``
(``/root/reference/pkg/src/sparsekv``), written from the reference's
behaviour, with every function citing the reference file:line it follows.
All score arithmetic widens to float64 exactly like the reference
(``core.py:64-67``), so the restatement is bit-identical to the reference
on the same inputs; ``tests/golden/make_golden.py`` generated fixtures from
the real reference in the build container and ``tests/test_oracle.py`` pins
this restatement against them (parity PINNED, not unpinned).

The synthetic workload generator (``workload.py:31-195``) is restated too,
call for call on the same ``numpy.random.Generator`` streams, so the GPU box
(which has no reference checkout) regenerates the reference's exact inputs.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

F32 = np.float32


# --------------------------------------------------------------------------
# core.py
# --------------------------------------------------------------------------

def inner_products(keys: np.ndarray, q: np.ndarray) -> np.ndarray:
    """fp64 GEMV ``keys @ q`` -- reference ``core.py:64-67``."""
    if keys.shape[-1] != q.shape[-1]:
        raise ValueError(f"dimension mismatch: {keys.shape[-1]} vs {q.shape[-1]}")
    return keys.astype(np.float64, copy=False) @ q.astype(np.float64, copy=False)


def group_scores(keys: np.ndarray, qs: np.ndarray) -> np.ndarray:
    """fp64 scores of a GQA group's query heads over one kv head's keys,
    ``(n, G)`` = ``inner_products(keys, qs[j])`` for every j in one GEMM
    (``core.py:64-67`` per head; the group shares ``kv_head_of``, ``core.py:108-112``)."""
    qs = np.atleast_2d(qs)
    if keys.shape[-1] != qs.shape[-1]:
        raise ValueError(f"dimension mismatch: {keys.shape[-1]} vs {qs.shape[-1]}")
    return keys.astype(np.float64, copy=False) @ qs.astype(np.float64, copy=False).T


def scaled_scores(keys: np.ndarray, q: np.ndarray) -> np.ndarray:
    """Raw scores divided by sqrt(d) -- reference ``core.py:75-77``."""
    return inner_products(keys, q) / np.sqrt(q.shape[-1])


def window_base_ids(prefix_len: int, initial: int = 16, last: int = 64) -> np.ndarray:
    """Sorted base-window ids ``[0,initial) U [p-last,p)`` -- ``core.py:159-165``."""
    if initial < 0 or last < 0:
        raise ValueError("window sizes must be non-negative")
    if prefix_len <= initial + last:
        return np.arange(prefix_len, dtype=np.int64)
    head = np.arange(initial, dtype=np.int64)
    tail = np.arange(prefix_len - last, prefix_len, dtype=np.int64)
    return np.concatenate([head, tail])


# --------------------------------------------------------------------------
# dipr.py
# --------------------------------------------------------------------------

def alpha_to_beta(alpha: float, d: int) -> float:
    """``beta = -sqrt(d) ln(alpha)`` -- reference ``dipr.py:29-39``."""
    if not 0.0 < alpha <= 1.0:
        raise ValueError(f"alpha must be in (0, 1], got {alpha}")
    if d < 1:
        raise ValueError(f"dimension must be positive, got {d}")
    return -math.sqrt(d) * math.log(alpha)


def dipr_scores_and_mask(q: np.ndarray, keys: np.ndarray, beta: float):
    """fp64 scores and the inclusive ``s >= max - beta`` mask -- ``dipr.py:58-64``."""
    keys = np.atleast_2d(keys)
    if keys.shape[0] == 0:
        raise ValueError("DIPR over an empty key set is undefined")
    if beta < 0:
        raise ValueError(f"beta must be non-negative, got {beta}")
    scores = inner_products(keys, q)
    return scores, scores >= scores.max() - beta


def dipr_bruteforce(q, keys, beta, token_ids=None) -> set[int]:
    """Exact DIPR id set -- reference ``dipr.py:47-70``."""
    keys = np.atleast_2d(keys)
    _, mask = dipr_scores_and_mask(q, keys, beta)
    if token_ids is None:
        return set(np.flatnonzero(mask).tolist())
    ids = np.asarray(list(token_ids), dtype=np.int64)
    if ids.shape[0] != keys.shape[0]:
        raise ValueError("token_ids length must match key count")
    return set(ids[mask].tolist())


# --------------------------------------------------------------------------
# attention.py
# --------------------------------------------------------------------------

@dataclass
class Partial:
    """(m, l, acc) online-softmax state -- reference ``attention.py:80-96``."""

    m: float = -np.inf
    l: float = 0.0
    acc: np.ndarray | None = None

    @property
    def is_empty(self) -> bool:
        return self.acc is None


def partial_over(q, keys, values) -> Partial:
    """Vectorised absorb of a token group -- ``attention.py:98-110``."""
    keys = np.atleast_2d(keys)
    values = np.atleast_2d(values)
    if keys.shape[0] == 0:
        return Partial()
    if keys.shape[0] != values.shape[0]:
        raise ValueError("keys/values length mismatch")
    z = scaled_scores(keys, q)
    m = float(z.max())
    w = np.exp(z - m)
    return Partial(m=m, l=float(w.sum()), acc=w @ values.astype(np.float64, copy=False))


def partial_merge(a: Partial, b: Partial) -> Partial:
    """Combine two disjoint partials -- ``attention.py:128-143``."""
    if a.is_empty:
        return b
    if b.is_empty:
        return a
    m = max(a.m, b.m)
    f1 = np.exp(a.m - m)
    f2 = np.exp(b.m - m)
    return Partial(m=m, l=a.l * f1 + b.l * f2, acc=a.acc * f1 + b.acc * f2)


def partial_finalize(p: Partial) -> np.ndarray:
    """``acc / l`` cast to fp32 -- ``attention.py:145-152``."""
    if p.is_empty:
        raise ValueError("cannot finalize an empty partial")
    o = p.acc / p.l
    if not np.isfinite(o).all():
        raise FloatingPointError("partial attention finalized to non-finite output")
    return o.astype(F32)


def full_attention(q, keys, values) -> np.ndarray:
    """Exact softmax attention -- ``attention.py:25-42``."""
    keys = np.atleast_2d(keys)
    values = np.atleast_2d(values)
    if keys.shape[0] == 0:
        raise ValueError("attention over an empty key set is undefined")
    z = scaled_scores(keys, q)
    w = np.exp(z - z.max())
    o = (w @ values.astype(np.float64, copy=False)) / w.sum()
    if not np.isfinite(o).all():
        raise FloatingPointError("attention output is non-finite")
    return o.astype(F32)


# --------------------------------------------------------------------------
# store.py: the flat-DIPR decode step
# --------------------------------------------------------------------------

def head_attention_flat(q, base_k, base_v, win_k, win_v, beta, initial=16, last=64,
                        selected_override=None):
    """One query head on the DIPR/FLAT plan -- ``store.py:252-293`` via ``:337``.

    ``base_k/base_v`` are the base prefix (p, d); ``win_k/win_v`` the session
    window rows (w, d). Returns ``(o, selected_sorted, retrieved_count)``.
    ``selected_override`` evaluates the same arithmetic on a given selection
    (used to separate an epsilon-boundary set flip from an arithmetic error).
    """
    p = base_k.shape[0]
    window_ids = window_base_ids(p, initial, last)
    if p == 0:
        retrieved = np.empty(0, dtype=np.int64)
    else:
        _, mask = dipr_scores_and_mask(q, base_k, beta)  # store.py:337
        retrieved = np.flatnonzero(mask)
    if selected_override is not None:
        selected = np.asarray(selected_override, dtype=np.int64)
    else:
        selected = np.setdiff1d(retrieved, window_ids)  # store.py:271-273
    o = head_attention_on_selection(q, base_k, base_v, win_k, win_v, selected, initial, last)
    return o, np.sort(selected), int(retrieved.size)


def head_attention_on_selection(q, base_k, base_v, win_k, win_v, selected, initial=16, last=64):
    """The tail of ``_head_attention`` for a given selection (``store.py:274-293``):
    partial over the selected base rows, merged with the partial over the base
    window rows + session window rows, finalized. Used on its own when the
    caller already holds the fp64 scores (large parity cases)."""
    p = base_k.shape[0]
    window_ids = window_base_ids(p, initial, last)
    selected = np.asarray(selected, dtype=np.int64)
    part = Partial()
    if selected.size:  # store.py:274-278
        part = partial_merge(part, partial_over(q, base_k[selected], base_v[selected]))
    win_keys = [base_k[window_ids]] if window_ids.size else []
    win_vals = [base_v[window_ids]] if window_ids.size else []
    if win_k is not None and win_k.shape[0]:  # store.py:279-287
        win_keys.append(win_k)
        win_vals.append(win_v)
    if win_keys:
        part = partial_merge(
            part, partial_over(q, np.concatenate(win_keys), np.concatenate(win_vals)))
    return partial_finalize(part)


def session_attention_flat(q, base_k, base_v, win_k=None, win_v=None, beta=110.0,
                           initial=16, last=64):
    """``Session.attention`` on the flat plan for one layer -- ``store.py:191-216``.

    ``q`` (Hq, d); ``base_k/base_v`` (Hkv, p, d); ``win_k/win_v`` (Hkv, w, d)
    or None. GQA map ``kv = qh // g`` (``core.py:108-112``). Returns
    ``(out (Hq, d) fp32, [selected ids per q head], [retrieved count per q head])``.
    """
    q = np.atleast_2d(np.asarray(q, dtype=F32))
    hq, d = q.shape
    hkv = base_k.shape[0]
    if hq % hkv:
        raise ValueError("n_query_heads must be a multiple of n_kv_heads")
    g = hq // hkv
    p = base_k.shape[1]
    w = 0 if win_k is None else win_k.shape[1]
    if p + w == 0:
        raise ValueError("attention on an empty session")
    out = np.empty((hq, d), dtype=F32)
    sels, counts = [], []
    for qh in range(hq):
        h = qh // g
        o, sel, cnt = head_attention_flat(
            q[qh], base_k[h], base_v[h],
            None if win_k is None else win_k[h], None if win_v is None else win_v[h],
            beta, initial, last)
        out[qh] = o
        sels.append(sel)
        counts.append(cnt)
    return out, sels, counts


# --------------------------------------------------------------------------
# index.py: coarse block index (the sound-bound filter input)
# --------------------------------------------------------------------------

def select_representatives(block_keys: np.ndarray, r: int) -> np.ndarray:
    """The r largest-L2-norm keys, ties by position -- ``index.py:217-228``."""
    block_keys = np.atleast_2d(block_keys)
    if not 1 <= r <= block_keys.shape[0]:
        raise ValueError(f"r must be in [1, {block_keys.shape[0]}], got {r}")
    norms = np.linalg.norm(block_keys.astype(np.float64), axis=1)
    order = np.lexsort((np.arange(block_keys.shape[0]), -norms))
    return block_keys[order[:r]]


def flat_top_k(q: np.ndarray, keys: np.ndarray, k: int) -> list[int]:
    """Exact top-k ids, scores descending, ties by smaller id -- ``index.py:60-66``."""
    keys = np.atleast_2d(keys)
    n = keys.shape[0]
    if not 1 <= k <= n:
        raise ValueError(f"k must be in [1, {n}], got {k}")
    scores = inner_products(keys, q)
    order = np.lexsort((np.arange(n), -scores))
    return order[:k].tolist()


@dataclass
class BlockIndex:
    """Contiguous token blocks scored by representatives -- ``index.py:195-214``."""

    block_size: int
    starts: np.ndarray
    ends: np.ndarray
    reps: list

    @property
    def n_blocks(self) -> int:
        return len(self.reps)

    def block_scores(self, q: np.ndarray) -> np.ndarray:
        return np.array([inner_products(r, q).max() for r in self.reps])

    def top_blocks(self, q: np.ndarray, k_blocks: int) -> list:
        """Best ``k_blocks`` ranges by max representative score, ties by start."""
        if not 1 <= k_blocks <= self.n_blocks:
            raise ValueError(f"k_blocks must be in [1, {self.n_blocks}], got {k_blocks}")
        scores = self.block_scores(q)
        order = np.lexsort((self.starts, -scores))
        return [(int(self.starts[i]), int(self.ends[i])) for i in order[:k_blocks]]


def build_block_index(keys: np.ndarray, block_size: int, r: int) -> BlockIndex:
    """Contiguous blocks + representatives -- ``index.py:231-243``."""
    keys = np.atleast_2d(keys)
    if block_size < 1:
        raise ValueError("block_size must be positive")
    n = keys.shape[0]
    starts = np.arange(0, n, block_size, dtype=np.int64)
    ends = np.minimum(starts + block_size, n)
    reps = [select_representatives(keys[s:e], min(r, e - s)) for s, e in zip(starts, ends)]
    return BlockIndex(block_size=block_size, starts=starts, ends=ends, reps=reps)


def retrieve_top_k_flat(q, base_k, k):
    """TOP_K branch on a flat index -- ``store.py:314-318`` (k clamped to p)."""
    p = base_k.shape[0]
    if p == 0:
        return set()
    return set(flat_top_k(q, base_k, min(k, p)))


def retrieve_top_k_coarse(q, index: BlockIndex, k, p):
    """TOP_K on the coarse block index -- ``store.py:305-312``."""
    if p == 0:
        return set()
    want = max(1, -(-k // index.block_size))
    out = set()
    for lo, hi in index.top_blocks(q, min(want, index.n_blocks)):
        out.update(range(lo, min(hi, p)))
    return out


def head_attention_retrieved(q, base_k, base_v, win_k, win_v, retrieved, initial=16, last=64):
    """``_head_attention`` after retrieval -- ``store.py:268-293``: selected =
    retrieved minus the base window ids, partial(selected) merged with
    partial(base window + session rows), finalized."""
    p = base_k.shape[0]
    window_ids = window_base_ids(p, initial, last)
    ret = np.fromiter(retrieved, dtype=np.int64, count=len(retrieved))
    selected = np.setdiff1d(ret, window_ids)
    part = Partial()
    if selected.size:
        part = partial_merge(part, partial_over(q, base_k[selected], base_v[selected]))
    win_keys = [base_k[window_ids]] if window_ids.size else []
    win_vals = [base_v[window_ids]] if window_ids.size else []
    if win_k is not None and win_k.shape[0]:
        win_keys.append(win_k)
        win_vals.append(win_v)
    if win_keys:
        part = partial_merge(
            part, partial_over(q, np.concatenate(win_keys), np.concatenate(win_vals)))
    return partial_finalize(part), np.sort(selected), int(ret.size)


def session_attention_topk(q, base_k, base_v, win_k, win_v, k, coarse=False, block_size=128,
                           reps=4, initial=16, last=64, indexes=None):
    """``Session.attention`` on a TOP_K plan for one layer (``store.py:191-216``
    with ``_retrieve`` ``:305-318``). ``indexes[h]`` may hold prebuilt
    BlockIndexes (built over the full context, as at import, ``store.py:506-509``).
    Returns ``(out, [selected per q head], [retrieved per q head])``."""
    q = np.atleast_2d(np.asarray(q, dtype=F32))
    hq, d = q.shape
    hkv = base_k.shape[0]
    g = hq // hkv
    p = base_k.shape[1]
    out = np.empty((hq, d), dtype=F32)
    sels, counts = [], []
    for qh in range(hq):
        h = qh // g
        if coarse:
            idx = indexes[h] if indexes is not None else build_block_index(base_k[h], block_size, reps)
            ret = retrieve_top_k_coarse(q[qh], idx, k, p)
        else:
            ret = retrieve_top_k_flat(q[qh], base_k[h], k)
        o, sel, cnt = head_attention_retrieved(
            q[qh], base_k[h], base_v[h], None if win_k is None else win_k[h],
            None if win_v is None else win_v[h], ret, initial, last)
        out[qh] = o
        sels.append(sel)
        counts.append(cnt)
    return out, sels, counts


# --------------------------------------------------------------------------
# dipr.py: graph DIPRS over a proximity graph (plain walk, no prefix filter)
# --------------------------------------------------------------------------

class CandidateList:
    """Append-only candidate list with a capacity threshold -- ``dipr.py:107-158``."""

    def __init__(self, l0: int, beta: float, floor: float = -np.inf):
        if l0 < 1:
            raise ValueError(f"capacity threshold must be >= 1, got {l0}")
        if beta < 0:
            raise ValueError(f"beta must be non-negative, got {beta}")
        self.l0, self.beta, self.floor = l0, beta, floor
        self.ids: list[int] = []
        self.scores: list[float] = []
        self.best_score, self.best_id = -np.inf, -1

    def __len__(self) -> int:
        return len(self.ids)

    def _push(self, token_id, score):
        self.ids.append(token_id)
        self.scores.append(score)
        if score > self.best_score or (score == self.best_score and token_id < self.best_id):
            self.best_score, self.best_id = score, token_id

    @property
    def bound(self) -> float:
        return max(self.best_score, self.floor)

    def try_append(self, token_id, score) -> bool:
        if len(self.ids) <= self.l0 or score >= self.bound - self.beta:
            self._push(token_id, score)
            return True
        return False

    def result(self) -> set:
        cut = self.bound - self.beta
        return {t for t, sc in zip(self.ids, self.scores) if sc >= cut}


def diprs(keys, offsets, nbrs, q, start, l0, beta, window_max=None) -> set:
    """Graph DIPRS -- ``dipr.py:265-289`` via ``traverse`` ``:166-262`` (no
    ``admitted_limit``): walk the list in insertion order in batches; each
    batch offers its entries' neighbours (adjacency order, deduplicated keeping
    the first occurrence), unvisited ones are scored and offered in order.
    The graph is CSR: neighbours of u = ``nbrs[offsets[u]:offsets[u+1]]``."""
    n = keys.shape[0]
    if n == 0:
        raise ValueError("search over an empty index")
    if not 0 <= start < n:
        raise ValueError(f"start node {start} out of range")
    keys64 = keys.astype(np.float64)
    q64 = np.asarray(q).astype(np.float64)
    floor = -np.inf if window_max is None else float(window_max)
    cands = CandidateList(l0, beta, floor=floor)
    cands._push(start, float(keys64[start] @ q64))  # CandidateList.seed
    visited = np.zeros(n, dtype=bool)
    visited[start] = True
    cursor = 0
    while cursor < len(cands):
        batch = cands.ids[cursor:]
        cursor = len(cands)
        pieces = [nbrs[offsets[u]:offsets[u + 1]] for u in batch]
        offered = np.concatenate(pieces) if pieces else np.empty(0, np.int64)
        if offered.size == 0:
            continue
        _, first = np.unique(offered, return_index=True)
        first.sort()
        offered = offered[first]
        fresh = offered[~visited[offered]]
        if fresh.size == 0:
            continue
        visited[fresh] = True
        scores = keys64[fresh] @ q64
        for token_id, score in zip(fresh.tolist(), scores.tolist()):
            cands.try_append(token_id, score)
    return cands.result()


def block_box_bounds(keys: np.ndarray, block_size: int):
    """Per-block per-dim (min, max) boxes over contiguous blocks.

    The reference's ``BlockIndex`` (``index.py:195-243``) ranks blocks by
    representative scores, which is a heuristic, not a bound; a filter that
    must preserve the exact DIPR set needs a sound upper bound. The box bound
    ``UB_b(q) = sum_k max(q_k lo_k, q_k hi_k)`` is >= every score in block b.
    """
    n, d = keys.shape
    nb = -(-n // block_size)
    lo = np.empty((nb, d), dtype=F32)
    hi = np.empty((nb, d), dtype=F32)
    for b in range(nb):
        blk = keys[b * block_size:(b + 1) * block_size]
        lo[b] = blk.min(axis=0)
        hi[b] = blk.max(axis=0)
    return lo, hi


def block_upper_bounds(q: np.ndarray, lo: np.ndarray, hi: np.ndarray) -> np.ndarray:
    q64 = q.astype(np.float64)
    return np.maximum(lo.astype(np.float64) * q64, hi.astype(np.float64) * q64).sum(axis=1)


# --------------------------------------------------------------------------
# workload.py: the reference's seeded synthetic inputs, restated
# --------------------------------------------------------------------------

VOCAB = 50_000


def _rng(seed: int, stream: int) -> np.random.Generator:
    """``WorkloadSpec.rng`` -- ``workload.py:60-61``."""
    return np.random.default_rng(np.random.SeedSequence([seed, stream]))


def _cluster_centers(rng, clusters: int, dim: int) -> np.ndarray:
    """``workload.py:73-75``."""
    centers = rng.standard_normal((clusters, dim))
    return centers / np.linalg.norm(centers, axis=1, keepdims=True) * np.sqrt(dim)


def make_context(n_tokens, n_layers, n_kv_heads, dim, clusters=16, spread=0.25, seed=0):
    """gaussian-clusters / uniform sizes context -- ``workload.py:90-134``.

    Returns ``(token_ids, keys (L,Hkv,n,d) fp32, values, centers, assignments)``.
    """
    rng = _rng(seed, 1)
    token_ids = rng.integers(0, VOCAB, size=n_tokens, dtype=np.int64)
    centers = _cluster_centers(rng, clusters, dim)
    keys = np.empty((n_layers, n_kv_heads, n_tokens, dim), dtype=F32)
    values = np.empty_like(keys)
    assignments = None
    for layer in range(n_layers):
        for head in range(n_kv_heads):
            a = rng.integers(0, centers.shape[0], size=n_tokens)
            keys[layer, head] = (centers[a] + spread * rng.standard_normal((n_tokens, dim))
                                 ).astype(F32)
            values[layer, head] = rng.standard_normal((n_tokens, dim)).astype(F32)
            if layer == 0 and head == 0:
                assignments = a
    return token_ids, keys, values, centers, assignments


def decode_step_inputs(steps, n_layers, n_query_heads, n_kv_heads, dim, centers,
                       spread=0.25, seed=0, stream=4):
    """Per-step (token_ids, q, k, v) -- ``workload.py:169-195``."""
    rng = _rng(seed, stream)
    token_ids = rng.integers(0, VOCAB, size=steps, dtype=np.int64)
    picks = rng.integers(0, centers.shape[0], size=(steps, n_layers, n_query_heads))
    q = centers[picks] + spread * rng.standard_normal((steps, n_layers, n_query_heads, dim))
    kpicks = rng.integers(0, centers.shape[0], size=(steps, n_layers, n_kv_heads))
    k = centers[kpicks] + spread * rng.standard_normal((steps, n_layers, n_kv_heads, dim))
    v = rng.standard_normal((steps, n_layers, n_kv_heads, dim))
    return token_ids, q.astype(F32), k.astype(F32), v.astype(F32)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 -> fp32 (the bf16-mode oracle input)."""
    u = np.ascontiguousarray(x, dtype=F32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return (r & 0xFFFFFFFF).astype(np.uint32).view(F32).reshape(x.shape)
