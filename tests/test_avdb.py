"""AVDB vector files (reference vfs.py): the native writer is byte-identical to
the reference's (sha256 of files the real reference wrote for the same
inputs), and the native parser reads reference-written files -- appended,
tombstoned and graph-indexed ones included. Host-only C++: no GPU needed.
GPU loads (pinned host -> device slab) are in the gpu-marked tests."""

from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

from tests.golden_cases import GOLDEN, avdb_vectors

AV = GOLDEN / "avdb"


def _vfs():
    from paper_2504_10326_b200 import vfs
    return vfs


@pytest.mark.parametrize("case", json.loads((AV / "hashes.json").read_text())["cases"])
def test_writer_byte_identical_to_reference(tmp_path, case):
    vfs = _vfs()
    name, n, dim, width, seed = case
    want_sha, want_len = json.loads((AV / "hashes.json").read_text())["sha256"][name]
    f = tmp_path / f"{name}.avdb"
    with np.errstate(over="ignore"):
        vfs.write_vector_file(f, avdb_vectors(n, dim, seed, width), element_width=width)
    b = f.read_bytes()
    assert len(b) == want_len
    assert hashlib.sha256(b).hexdigest() == want_sha
    h = vfs.read_header(f)
    assert (h.n_vectors, h.dim, h.element_width) == (n, dim, width)
    assert h.n_data_blocks == (0 if n == 0 else -(-n // h.slots_per_block))


def test_parse_reference_mutated_files():
    vfs = _vfs()
    h = vfs.read_header(AV / "appended_tomb16.avdb")
    z = np.load(AV / "appended_tomb16.npz")
    assert (h.n_vectors, h.dim, h.element_width, h.n_tombstones) == (250, 32, 16, 3)
    assert h.n_vectors == z["vectors"].shape[0]
    g = vfs.read_header(AV / "graph32.avdb")
    assert (g.n_vectors, g.dim, g.n_index_blocks) == (60, 16, 1) and g.index_head_offset == 4096


def test_format_errors(tmp_path):
    vfs = _vfs()
    bad = tmp_path / "bad.avdb"
    bad.write_bytes(b"XXXX" + b"\0" * 4092)
    with pytest.raises(vfs.VectorFileError, match="bad magic"):
        vfs.read_header(bad)
    short = tmp_path / "short.avdb"
    short.write_bytes(b"AVDB")
    with pytest.raises(vfs.VectorFileError):
        vfs.read_header(short)
    good = tmp_path / "g.avdb"
    vfs.write_vector_file(good, np.ones((10, 16), np.float32))
    raw = bytearray(good.read_bytes())
    raw[4:8] = (2).to_bytes(4, "little")  # version
    (tmp_path / "v.avdb").write_bytes(bytes(raw))
    with pytest.raises(vfs.VectorFileError, match="version"):
        vfs.read_header(tmp_path / "v.avdb")
    raw = bytearray(good.read_bytes())
    raw[12:20] = (11).to_bytes(8, "little")  # n_vectors disagrees with the directory
    (tmp_path / "n.avdb").write_bytes(bytes(raw))
    with pytest.raises(vfs.VectorFileError, match="expected 11 vectors"):
        vfs.read_header(tmp_path / "n.avdb")
    with pytest.raises(NotImplementedError):
        vfs.write_vector_file(good, np.ones((2, 16), np.float32), adjacency=[[1], [0]])
