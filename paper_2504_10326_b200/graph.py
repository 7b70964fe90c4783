"""A whole decode step captured once as a CUDA graph (small-batch / short-context
decode, where the per-call host path -- descriptor marshalling, ctypes, tensor-map
encoding, a dozen launches per layer -- costs more than the GPU work).

For every layer the step is ``Session.update`` (window append, reference
``store.py:160-189``) followed by ``Session.attention`` on the DIPR/FLAT plan
(``store.py:191-216``) over all sessions of the batch, i.e. exactly the calls
``bench.py`` issues eagerly. The window row count lives on the device
(``SeqView.w_dev`` -> ``alaya_seq.d_w``): the append kernel writes row ``*d_w`` and a
commit kernel advances it, so one capture stays valid while the windows grow (up
to the ring capacity). Inputs go through static buffers: write the step's
``q``/``k``/``v`` into :attr:`q`, :attr:`k`, :attr:`v`, call :meth:`replay`, read
:attr:`out`.

Not for the fused sharded step (its exchange epochs are per call).

Graph-mode handshake: the step's first node advances a device sequence number
(``alaya_params.d_call_seq``); each captured call combines it with its capture
slot, so prep's published header is told apart from the previous replay's and the
scan can start before prep finishes, as in the eager path.
"""

from __future__ import annotations

import torch

from . import engine


class DecodeStepGraph:
    """``layers``: per layer the ``SeqView`` list of the batch (all with ``w_dev``
    set, one counter per (session, layer)) -- the append targets and the attention
    inputs are the same views."""

    def __init__(self, layers: list[list[engine.SeqView]], params, dtype: torch.dtype,
                 device: torch.device):
        if not layers or any(len(l) != len(layers[0]) for l in layers):
            raise ValueError("every layer needs the same batch of sequences")
        if any(s.w_dev is None for l in layers for s in l):
            raise ValueError("graph mode needs SeqView.w_dev (device window counts)")
        self.L, self.B = len(layers), len(layers[0])
        hq, hkv, d = params.n_query_heads, params.n_kv_heads, params.dim
        # replay sequence number (first node of the step): gives every captured call a
        # per-replay identity, so the scan starts on prep's published header as eagerly
        self.seq = torch.zeros(1, dtype=torch.int64, device=device)
        params = type(params).from_buffer_copy(params)
        params.d_call_seq = self.seq.data_ptr()
        self.params, self.dtype, self.device = params, dtype, device
        self.q = torch.zeros(self.L, self.B, hq, d, dtype=torch.float32, device=device)
        self.k = torch.zeros(self.L, self.B, hkv, d, dtype=torch.float32, device=device)
        self.v = torch.zeros_like(self.k)
        self.out = torch.zeros_like(self.q)
        # the graph owns its workspace (the layers run back to back, as eagerly): a shared
        # buffer could be reallocated under the captured pointers
        self.calls = [engine.Call(l, params, dtype, device) for l in layers]
        self.ws = torch.empty(max(c.ws_bytes for c in self.calls), dtype=torch.uint8, device=device)
        for c in self.calls:
            c.ws, c.ws_bytes = self.ws, self.ws.numel()
        self.appends = [engine.append_array(l, params, dtype) for l in layers]
        self.counters = [s.w_dev for l in layers for s in l]
        # every replay appends one row to every ring: the device append kernel drops a
        # row once the ring is full, so the host refuses that replay instead
        self.capacity = min(int(sv.wk.shape[1]) for l in layers for sv in l)
        self.graph = torch.cuda.CUDAGraph()
        self._capture()
        self.sync_rows()

    def _step(self) -> None:
        self.seq.add_(1)
        for l in range(self.L):
            engine.window_append_raw(self.appends[l], self.B, self.params, self.k[l], self.v[l])
            self.calls[l].dipr_attention(self.q[l], out=self.out[l])

    def _capture(self) -> None:
        saved = [c.clone() for c in self.counters]
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):  # one eager step first (lazy per-kernel setup), then undo it
            self._step()
        torch.cuda.current_stream(self.device).wait_stream(s)
        for c, v in zip(self.counters, saved):
            c.copy_(v)
        torch.cuda.synchronize(self.device)
        with torch.cuda.graph(self.graph):
            self._step()
        torch.cuda.synchronize(self.device)

    def sync_rows(self) -> int:
        """Re-read the device window row counts (after the caller changed them) and
        return the fullest ring's row count."""
        self.rows = int(torch.stack([c[:1] for c in self.counters]).max().item())
        return self.rows

    @property
    def remaining(self) -> int:
        """Replays left before the fullest window ring is at capacity."""
        return self.capacity - self.rows

    def replay(self) -> torch.Tensor:
        """One decode step of every layer (stream-ordered); returns :attr:`out`.

        Raises ``RuntimeError`` when a ring has no free row left (the reference's
        ``Session.update`` always appends, ``store.py:160-189``; the captured ring
        cannot grow): re-create the step with larger rings."""
        if self.rows >= self.capacity:
            raise RuntimeError(f"decode-step graph: window ring full ({self.rows}/{self.capacity} rows); "
                               "re-capture with a larger ring")
        self.graph.replay()
        self.rows += 1
        return self.out
