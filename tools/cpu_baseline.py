"""CPU baselines for BASELINE configs 1, 3 (B=1) and 4 (B=1), one layer:
Session.attention on the flat plan, timed with 1 BLAS thread and with all cores.

  python tools/cpu_baseline.py --impl port       # oracle restatement (runs anywhere)
  python tools/cpu_baseline.py --impl reference  # the REAL reference (build container only:
                                                 # imports /root/reference/pkg/src)

The oracle port is bit-exact to the reference (tests/test_oracle.py); timing both
in the build container shows the port is a faithful stand-in for the GPU box,
where the reference is absent.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--impl", default="port", choices=["port", "reference"])
ap.add_argument("--configs", default="1,3,4")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()

CONFIGS = {  # name: (n, Hq, Hkv)
    "1": ("config1 Llama 32/8 ctx 4K fp32", 4096, 32, 8),
    "3": ("config3 Llama 32/8 ctx 128K", 131072, 32, 8),
    "4": ("config4 Qwen 40/8 ctx 128K", 131072, 40, 8),
}


def run(limit):
    from threadpoolctl import threadpool_limits
    from oracle import alaya_oracle as O
    out = []
    for c in a.configs.split(","):
        label, n, hq, hkv = CONFIGS[c]
        tok, keys, vals, centers, _ = O.make_context(n, 1, hkv, 128, seed=0)
        _, q, k, v = O.decode_step_inputs(1, 1, hq, hkv, 128, centers, seed=0)
        if a.impl == "reference":
            sys.path.insert(0, "/root/reference/pkg/src")
            from sparsekv import ContextStore, EngineConfig, ModelShape
            shape = ModelShape(1, hq, hkv, 128)
            db = ContextStore(shape, EngineConfig(first_layers=(0,), short_context_threshold=0))
            db.import_context(tok, keys, vals)
            sess, _ = db.create_session(tok)
            sess.update(q[0, 0], k[0, 0], v[0, 0], 0)
            fn = lambda: sess.attention(q[0, 0], 0)  # noqa: E731
        else:
            wk, wv = k[0, 0][:, None], v[0, 0][:, None]
            fn = lambda: O.session_attention_flat(q[0, 0], keys[0], vals[0], wk, wv, 110.0)  # noqa: E731
        with threadpool_limits(limits=limit):
            fn()
            ts = []
            for _ in range(a.reps):
                t0 = time.perf_counter()
                fn()
                ts.append(time.perf_counter() - t0)
        t = min(ts)
        out.append({"impl": a.impl, "config": label, "threads": limit or os.cpu_count(),
                    "s_per_layer_call": round(t, 4), "query_heads_per_s": round(hq / t, 2)})
        print(json.dumps(out[-1]), flush=True)
    return out


run(1)
run(None)
