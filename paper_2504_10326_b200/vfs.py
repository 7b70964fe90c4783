"""AVDB vector files (reference ``sparsekv/vfs.py``, ``docs/file-format.md``).

Native (``libalaya_b200.so``): header/directory parsing and the writer run on
the host in C++ (byte-identical to the reference's ``write_vector_file`` for
vector-only files); ``load_to_device`` reads file images into pinned host
memory and one kernel per call unpacks the data blocks straight into a
device KV slab (``alaya_avdb_load``) -- the path ``ContextStore(root=...)``
uses to bring stored contexts into HBM (reference ``store.py:569-609``).
Graph index blocks (adjacency) are parsed for counts only: graph search is
out of scope.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import AlayaAvdbInfo

BLOCK_SIZE = 4096
MAGIC = b"AVDB"
VERSION = 1


class VectorFileError(Exception):
    """I/O or format failure, annotated with file path and offset (``vfs.py:62-67``)."""


def _check(rc: int) -> None:
    if rc != _lib.ALAYA_OK:
        msg = _lib.load().alaya_last_error().decode(errors="replace")
        if rc == _lib.ALAYA_ERR_ARG:
            raise VectorFileError(msg)
        _lib.check(rc)


@dataclass(frozen=True)
class FileHeader:
    """``vfs.py:70-84``."""

    dim: int
    n_vectors: int
    element_width: int
    directory_offset: int
    index_head_offset: int
    n_data_blocks: int = 0
    n_index_blocks: int = 0
    n_tombstones: int = 0
    file_bytes: int = 0

    @property
    def slot_size(self) -> int:
        return self.dim * self.element_width // 8

    @property
    def slots_per_block(self) -> int:
        return (BLOCK_SIZE - 16) // self.slot_size


def read_header(path) -> FileHeader:
    """Header + directory summary of one file (``vfs.py:247-286``)."""
    info = AlayaAvdbInfo()
    _check(_lib.load().alaya_avdb_stat(os.fsencode(path), ctypes.byref(info)))
    return FileHeader(int(info.dim), int(info.n_vectors), int(info.element_width),
                      int(info.directory_offset), int(info.index_head), int(info.n_data_blocks),
                      int(info.n_index_blocks), int(info.n_tombstones), int(info.file_bytes))


def write_vector_file(path, vectors, adjacency=None, entry_point: int = 0, max_degree: int = 0,
                      element_width: int = 32) -> None:
    """Create a vector file (``vfs.py:188-244``); vectors ``(n, d)`` float32
    (numpy or torch, any device). Graph adjacency is not supported here."""
    if adjacency is not None:
        raise NotImplementedError("graph index blocks are out of scope on the B200 engine")
    if isinstance(vectors, torch.Tensor):
        vectors = vectors.detach().to("cpu", torch.float32).numpy()
    v = np.ascontiguousarray(np.atleast_2d(np.asarray(vectors, dtype=np.float32)))
    if v.shape[1] < 1:
        raise ValueError("vectors must have at least one column")
    if element_width not in (16, 32):
        raise ValueError(f"unsupported element width {element_width}")
    _check(_lib.load().alaya_avdb_write(os.fsencode(path), v.ctypes.data if v.size else None,
                                        v.shape[0], v.shape[1], element_width))


class PinnedStaging:
    """Reusable pinned host buffer for file images (grown on demand)."""

    def __init__(self):
        self.buf: torch.Tensor | None = None

    def get(self, nbytes: int) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8).pin_memory()
        return self.buf


_STAGING = PinnedStaging()


def load_to_device(paths, n: int, dim: int, dtype: torch.dtype, device,
                   out: torch.Tensor | None = None, staging: PinnedStaging | None = None
                   ) -> torch.Tensor:
    """Load ``len(paths)`` files of ``n`` vectors into a device tensor
    ``[files, n, dim]`` (``read_vector_file``, ``vfs.py:289-338``), fp32
    (exact widening of 16-bit payloads) or bf16. Synchronises the stream
    before returning (the pinned staging buffer is reused)."""
    if not torch.cuda.is_available():
        raise _lib.AlayaError("no CUDA device: the alaya B200 path has no CPU fallback")
    lib = _lib.load()
    enc = [os.fsencode(p) for p in paths]
    arr = (ctypes.c_char_p * len(enc))(*enc)
    need = lib.alaya_avdb_staging_bytes(arr, len(enc))
    if need == 0:
        for p in paths:  # surface the format error
            read_header(p)
        raise VectorFileError("cannot size the staging buffer")
    st = (staging or _STAGING).get(need)
    if out is None:
        out = torch.empty(len(paths), n, dim, dtype=dtype, device=device)
    if dtype not in (torch.float32, torch.bfloat16) or out.dtype != dtype or not out.is_contiguous():
        raise ValueError("out must be a contiguous fp32/bf16 [files, n, dim] tensor")
    stream = torch.cuda.current_stream(out.device)
    _check(lib.alaya_avdb_load(arr, len(enc), n, dim,
                               _lib.ALAYA_F32 if dtype == torch.float32 else _lib.ALAYA_BF16,
                               out.data_ptr(), out.stride(0) if out.dim() == 3 else n * dim,
                               st.data_ptr(), st.numel(), stream.cuda_stream))
    stream.synchronize()
    return out


@dataclass
class VectorFileContents:
    """``vfs.py:95-104`` (vectors as a device tensor)."""

    dim: int
    element_width: int
    vectors: torch.Tensor
    tombstones: int = 0


def read_vector_file(path, device="cuda", dtype=torch.float32) -> VectorFileContents:
    h = read_header(path)
    v = load_to_device([path], h.n_vectors, h.dim, dtype, torch.device(device))[0]
    return VectorFileContents(h.dim, h.element_width, v, h.n_tombstones)


def read_graph(path):
    """Adjacency of a file's index chain (``vfs.py:126-145``) as
    ``(degrees int32 [n], flat int32 [E], entry_point, max_degree)``, or None."""
    lib = _lib.load()
    nn, ne = ctypes.c_int64(), ctypes.c_int64()
    ep, md = ctypes.c_int32(), ctypes.c_int32()
    p = os.fsencode(path)
    _check(lib.alaya_avdb_graph(p, ctypes.byref(nn), ctypes.byref(ne), ctypes.byref(ep),
                                ctypes.byref(md), None, None))
    if nn.value == 0:
        return None
    deg = np.empty(nn.value, dtype=np.int32)
    flat = np.empty(max(ne.value, 1), dtype=np.int32)
    _check(lib.alaya_avdb_graph(p, ctypes.byref(nn), ctypes.byref(ne), ctypes.byref(ep),
                                ctypes.byref(md), deg.ctypes.data, flat.ctypes.data))
    return deg, flat[: ne.value], int(ep.value), int(md.value)
