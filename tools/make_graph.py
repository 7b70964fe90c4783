"""Build a graph with the REAL reference (build container only: needs
/root/reference) for tools/probe_diprs.py: one Llama-shaped head (d=128) of
the reference generator, queries of 4 GQA heads sampled for the shared graph
(`build_shared_graph`, default GraphParams). Output: gpurun_in/graph_<n>.npz.

  python tools/make_graph.py 16384
"""
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from sparsekv import ModelShape  # noqa: E402
from sparsekv.index import GraphParams, build_shared_graph  # noqa: E402
from sparsekv.workload import WorkloadSpec, make_context, make_queries  # noqa: E402

n = int(sys.argv[1])
spec = WorkloadSpec(n_tokens=n, shape=ModelShape(1, 4, 1, 128), seed=0)
ctx = make_context(spec)
t = time.time()
qs = [make_queries(spec, max(64, n // 10), ctx.centers, stream=20 + i) for i in range(4)]
g = build_shared_graph(ctx.keys[0, 0], qs, 0.4, GraphParams())
deg, flat = g.to_arrays()
print("built", n, round(time.time() - t, 1), "s", flush=True)
np.savez_compressed(f"gpurun_in/graph_{n}.npz", keys=ctx.keys[0, 0], values=ctx.values[0, 0],
                    degrees=deg, nbrs=flat, entry=g.entry_point, centers=ctx.centers)
