"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol ``include/alaya.h`` declares, the ctypes structs match the C layout,
and host-side validation maps to the reference's exception types."""

from __future__ import annotations

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

from paper_2504_10326_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "alaya.h"


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = set(re.findall(r"^\s*(?:int|size_t|const char\*|int\*|float\*)\s+(alaya_\w+)\(",
                              HEADER.read_text(), re.M))
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name


def test_struct_layout_matches_header(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(f'''#include <stdio.h>
#include <stddef.h>
#include "{HEADER}"
int main(void) {{
  printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(alaya_seq), offsetof(alaya_seq, n),
         offsetof(alaya_seq, prefix_len), offsetof(alaya_seq, bounds), sizeof(alaya_params),
         offsetof(alaya_params, beta), offsetof(alaya_params, block_filter));
  return 0;
}}''')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    S, P = _lib.AlayaSeq, _lib.AlayaParams
    assert got == [ctypes.sizeof(S), S.n.offset, S.prefix_len.offset, S.bounds.offset,
                   ctypes.sizeof(P), P.beta.offset, P.block_filter.offset]


def _params(**kw):
    base = dict(n_query_heads=32, n_kv_heads=8, dim=128, dtype=_lib.ALAYA_BF16, beta=110.0,
                win_initial=16, win_last=64, chunk=0, scan_kind=0, block_filter=0)
    base.update(kw)
    return _lib.AlayaParams(**base)


def _seqs(n=131072, B=1):
    arr = (_lib.AlayaSeq * B)()
    for s in arr:
        s.k = s.v = 0x1000
        s.head_stride = n * 128
        s.n = n
        s.prefix_len = n
    return arr


def test_workspace_sizing_is_host_only():
    lib = _lib.load()
    nb = lib.alaya_workspace_bytes(ctypes.byref(_params()), _seqs(), 1)
    # candidates (idx+score) for every (token, q head) plus the chunk partials:
    # between 1x and 2x of 8 B * n * Hq, far below the K slab (256 B * n * Hkv)
    assert 8 * 131072 * 32 <= nb < 2 * 8 * 131072 * 32
    assert lib.alaya_workspace_bytes(ctypes.byref(_params(n_query_heads=30)), _seqs(), 1) == 0


@pytest.mark.parametrize("kw,exc", [
    (dict(n_query_heads=30), ValueError),      # not a multiple of n_kv_heads
    (dict(beta=-0.5), ValueError),             # dipr.py:61-62
    (dict(win_initial=-1), ValueError),        # core.py:155-157
    (dict(dim=100), NotImplementedError),
    (dict(chunk=300), ValueError),
])
def test_validation_maps_to_reference_exceptions(kw, exc):
    lib = _lib.load()
    ws = ctypes.create_string_buffer(16)
    rc = lib.alaya_dipr_attention(ctypes.byref(_params(**kw)), _seqs(), 1, 1, 1, ws, 16, None)
    with pytest.raises(exc):
        _lib.check(rc)


def test_workspace_too_small_is_reported():
    lib = _lib.load()
    rc = lib.alaya_dipr_attention(ctypes.byref(_params()), _seqs(), 1, 1, 1, 1, 16, None)
    assert rc == _lib.ALAYA_ERR_WORKSPACE
    assert b"workspace" in lib.alaya_last_error()


def test_shard_outside_prefix_rejected():
    lib = _lib.load()
    s = _seqs(1000)
    s[0].token_offset = 500
    s[0].prefix_len = 1200
    rc = lib.alaya_dipr_attention(ctypes.byref(_params()), s, 1, 1, 1, 1, 1 << 40, None)
    assert rc == _lib.ALAYA_ERR_SHAPE
