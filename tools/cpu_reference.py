"""CPU reference timings for bench.py (the reference arm and ``cpu_baseline``).

When ``baseline/_ref`` holds the installed reference (``pip install --target
baseline/_ref``) this times the UNMODIFIED ``sparsekv``:
``Session.attention(q, layer)`` on the flat DIPR plan (``store.py:191-216``)
over a context from the reference's own generator (``workload.py:107-134,
169-195``). Otherwise it times the oracle port (``oracle/alaya_oracle.py``,
pinned bit-exact to the reference), and says so (``kind``).

Three variants, one session-layer (Hq query heads) per step:
  * ``threads_1``   -- ``threadpool_limits(1)``, the reference's deterministic
                       mode (``cli.py:127-134``);
  * ``threads_all`` -- OpenBLAS on every core;
  * ``process_pool``-- the Hq heads of the call spread over a fork pool of
                       ``os.cpu_count()`` workers, each running the reference's
                       own per-head code (``Session._head_attention``,
                       ``store.py:252-293``) -- the strongest CPU baseline.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"

_G: dict = {}  # fork-shared state of the process-pool variant


def load_reference():
    """The installed reference package, or None."""
    if not (REF / "sparsekv" / "__init__.py").exists():
        return None
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    try:
        import sparsekv
    except Exception:  # noqa: BLE001 - an unusable install falls back to the port
        return None
    return sparsekv


def _bf16(x):
    from oracle import alaya_oracle as O
    return O.bf16_round(x)


class CpuWorkload:
    """One Llama/Qwen-shaped layer of one session at ``ctx`` tokens."""

    def __init__(self, ctx: int, hq: int, hkv: int, d: int, beta: float, bf16: bool,
                 window_rows: int, steps: int, seed: int = 0, force_port: bool = False):
        self.sk = None if force_port else load_reference()
        self.kind = "reference" if self.sk is not None else "port"
        self.hq, self.hkv, self.d, self.beta, self.ctx = hq, hkv, d, beta, ctx
        if self.sk is not None:
            sk = self.sk
            from sparsekv import workload as W
            shape = sk.ModelShape(1, hq, hkv, d)
            spec = W.WorkloadSpec(n_tokens=ctx, shape=shape, seed=seed)
            sc = W.make_context(spec)
            tok, keys, vals, centers = sc.token_ids, sc.keys, sc.values, sc.centers
            _, q, k, v = W.decode_step_inputs(spec, steps + window_rows, centers)
        else:
            from oracle import alaya_oracle as O
            tok, keys, vals, centers, _ = O.make_context(ctx, 1, hkv, d, seed=seed)
            _, q, k, v = O.decode_step_inputs(steps + window_rows, 1, hq, hkv, d, centers, seed=seed)
        if bf16:  # bf16 mode: the CPU gets the bf16-rounded K/V widened to fp32
            keys, vals, k, v = _bf16(keys), _bf16(vals), _bf16(k), _bf16(v)
        self.tok, self.keys, self.vals = tok, keys, vals
        self.q = q[window_rows:, 0]
        self.win_k = np.ascontiguousarray(np.transpose(k[:window_rows, 0], (1, 0, 2)))
        self.win_v = np.ascontiguousarray(np.transpose(v[:window_rows, 0], (1, 0, 2)))
        if self.sk is not None:
            sk = self.sk
            cfg = sk.EngineConfig(beta=beta, first_layers=(0,), short_context_threshold=0)
            self.store = sk.ContextStore(sk.ModelShape(1, hq, hkv, d), cfg)
            self.store.import_context(tok, keys, vals)
            self.sess, _ = self.store.create_session(tok)
            for r in range(window_rows):  # Session.update, store.py:160-189
                self.sess.update(q[r, 0], k[r, 0], v[r, 0], 0)
            self.plan = self.sess.active_plan(0)

    # -- one session-layer ----------------------------------------------
    def call(self, s: int):
        if self.sk is not None:
            return self.sess.attention(self.q[s % len(self.q)], 0)
        from oracle import alaya_oracle as O
        return O.session_attention_flat(self.q[s % len(self.q)], self.keys[0], self.vals[0],
                                        self.win_k, self.win_v, self.beta)[0]

    def time_calls(self, steps: int, warmup: int, threads: int | None) -> list[float]:
        from threadpoolctl import threadpool_limits
        ts = []
        with threadpool_limits(limits=threads):
            for s in range(warmup + steps):
                t0 = time.perf_counter()
                self.call(s)
                if s >= warmup:
                    ts.append(time.perf_counter() - t0)
        return ts

    def time_pool(self, steps: int, warmup: int, workers: int | None = None) -> list[float]:
        workers = workers or os.cpu_count() or 1
        _G["w"] = self
        ctx = mp.get_context("fork")
        ts = []
        with ctx.Pool(workers, initializer=_pool_init) as pool:
            for s in range(warmup + steps):
                t0 = time.perf_counter()
                pool.map(_pool_head, [(s, qh) for qh in range(self.hq)], chunksize=1)
                if s >= warmup:
                    ts.append(time.perf_counter() - t0)
        return ts


def _pool_init():
    from threadpoolctl import threadpool_limits
    _G["lim"] = threadpool_limits(limits=1)  # one core per worker process


def _pool_head(arg):
    s, qh = arg
    w = _G["w"]
    q = w.q[s % len(w.q)][qh]
    g = w.hq // w.hkv
    if w.sk is not None:  # the reference's own per-head step (store.py:252-293)
        o, _ = w.sess._head_attention(np.asarray(q, np.float32), 0, qh // g, w.plan)
        return o
    from oracle import alaya_oracle as O
    h = qh // g
    return O.head_attention_flat(q, w.keys[0, h], w.vals[0, h], w.win_k[h], w.win_v[h], w.beta)[0]


def cpu_info() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def variants(wl: CpuWorkload, steps: int, warmup: int, which=("threads_1", "threads_all", "process_pool")):
    """query*heads/s per variant on this workload (mean step time)."""
    cores = os.cpu_count() or 1
    out = {}
    for name in which:
        if name == "threads_1":
            ts, c = wl.time_calls(steps, warmup, 1), 1
        elif name == "threads_all":
            ts, c = wl.time_calls(steps, warmup, cores), cores
        else:
            ts, c = wl.time_pool(steps, warmup), cores
        t = statistics.mean(ts)
        out[name] = {"value": wl.hq / t, "seconds_per_call": t, "cores": c}
    return out
