"""Loader for the committed golden fixtures (see ``tests/golden/make_golden.py``).

Regenerates large inputs with the restated reference generator and checks
its sha256 against the hash the real reference produced before any use.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from oracle import alaya_oracle as O

GOLDEN = Path(__file__).resolve().parent / "golden"
SESSION_CASES = ["tiny_gqa", "tiny_short", "tiny_nowin", "llama_4k_fp32", "llama_4k_bf16",
                 "qwen_2k_fp32"]
# TOP_K plans (flat FlatIndex.top_k and coarse BlockIndex.top_blocks)
TOPK_CASES = ["tiny_topk_flat", "tiny_topk_coarse", "llama_4k_topk_flat", "llama_4k_topk_coarse"]


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@dataclass
class SessionCase:
    name: str
    n_layers: int
    hq: int
    hkv: int
    d: int
    n: int
    steps: int
    seed: int
    beta: float
    win_init: int
    win_last: int
    bf16: bool
    layers: list
    keys: np.ndarray      # (L, Hkv, n, d) fp32 (bf16-rounded in bf16 cases)
    values: np.ndarray
    q: np.ndarray         # (steps, L, Hq, d)
    k: np.ndarray         # (steps, L, Hkv, d)
    v: np.ndarray
    out: np.ndarray       # reference outputs, (steps*len(layers), Hq, d)
    sel: list             # reference selected ids per (step, layer, q head)
    retrieved: np.ndarray
    topk: tuple | None = None  # (k, block_size, reps, coarse) for TOP_K cases

    def call_index(self, step: int, li: int) -> int:
        return step * len(self.layers) + li

    def selected(self, step: int, li: int, qh: int) -> np.ndarray:
        return self.sel[self.call_index(step, li) * self.hq + qh]


def load_session_case(name: str) -> SessionCase:
    z = np.load(GOLDEN / f"{name}.npz")
    L, hq, hkv, d, n, steps, seed, clusters = (int(x) for x in z["shape"])
    bf16 = bool(z["bf16"])
    if "keys" in z:
        keys, values = z["keys"], z["values"]
        q, k, v = z["q"], z["k"], z["v"]
    else:
        tids, keys, values, centers, _ = O.make_context(n, L, hkv, d, clusters=clusters, seed=seed)
        if sha(tids, keys, values, centers) != str(z["gen_sha"]):
            raise AssertionError(f"{name}: restated generator diverged from the reference")
        st, q, k, v = O.decode_step_inputs(steps, L, hq, hkv, d, centers, seed=seed)
        if sha(st, q, k, v) != str(z["step_sha"]):
            raise AssertionError(f"{name}: restated decode inputs diverged from the reference")
        if bf16:
            keys, values = O.bf16_round(keys), O.bf16_round(values)
            k, v = O.bf16_round(k), O.bf16_round(v)
    off = z["sel_off"]
    sel = [z["sel"][off[i]:off[i + 1]].astype(np.int64) for i in range(off.size - 1)]
    w = z["window"]
    return SessionCase(name, L, hq, hkv, d, n, steps, seed, float(z["beta"]), int(w[0]),
                       int(w[1]), bf16, [int(x) for x in z["layers"]], keys, values, q, k, v,
                       z["out"], sel, z["retrieved"],
                       tuple(int(x) for x in z["topk"]) if "topk" in z else None)


def window_rows(case: SessionCase, step: int, layer: int):
    """Session-window K/V after ``step+1`` updates: (Hkv, step+1, d)."""
    wk = np.transpose(case.k[: step + 1, layer], (1, 0, 2))
    wv = np.transpose(case.v[: step + 1, layer], (1, 0, 2))
    return np.ascontiguousarray(wk), np.ascontiguousarray(wv)


def avdb_vectors(n, dim, seed, width):
    """Inputs of the AVDB hash fixtures (same as tests/golden/make_golden.py)."""
    rng = np.random.default_rng(seed)
    v = (rng.standard_normal((n, dim)) * 3).astype(np.float32)
    if width == 16 and n:  # exercise rounding ties, overflow and subnormals
        v[0, :8] = np.array([65504, 65520, 1e-8, 6e-8, -2.98e-8, 1.0009765625, 2 ** -24, -0.0],
                            dtype=np.float32)
    return v
