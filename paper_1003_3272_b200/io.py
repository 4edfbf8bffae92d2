"""MMX1 matrices straight to the device.

The reference's binary matrix format (``pkg/src/mmkit/io.py:22-23, 90-106``):
the 4-byte magic ``b"MMX1"``, two little-endian u64 dimensions, then the
row-major float64 payload.  ``load_matrix_device`` validates the header with
the reference's checks and messages (``MatrixFormatError``), then streams the
payload from the file through two pinned staging buffers into HBM: reading
chunk k+1 from the file overlaps the host->device copy of chunk k, and in a
single-precision run the library narrows each landed fp64 chunk to fp32 on
the device (``mmk_f64_to_f32``, round-to-nearest-even = numpy's
``astype(float32)``).  No host copy of the matrix is ever materialised, so an
NNMF input larger than host memory (C4's X is 17 GB as fp64) can be loaded.
"""

import os
import struct
import sys

from .backend import SERIAL, Backend
from .errors import MatrixFormatError, ShapeError
from . import _lib

__all__ = ["MAGIC", "read_mmx_header", "load_matrix_device"]

MAGIC = b"MMX1"
_HEADER = struct.Struct("<QQ")
_PAYLOAD_OFFSET = len(MAGIC) + _HEADER.size


def read_mmx_header(path):
    """(rows, cols) of an MMX1 file, with the reference's validation
    (io.py:90-103): magic, complete header, exact payload length."""
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        head = fh.read(_PAYLOAD_OFFSET)
    if head[:4] != MAGIC:
        raise MatrixFormatError(f"{path}: bad magic {head[:4]!r}, expected {MAGIC!r}")
    if size < _PAYLOAD_OFFSET:
        raise MatrixFormatError(f"{path}: truncated header ({size} bytes)")
    rows, cols = _HEADER.unpack_from(head, 4)
    expected = _PAYLOAD_OFFSET + rows * cols * 8
    if size != expected:
        raise MatrixFormatError(f"{path}: payload for {rows}x{cols} needs {expected} bytes, "
                                f"file has {size}")
    return rows, cols


def load_matrix_device(path, backend=SERIAL, chunk_bytes=64 << 20):
    """Load an MMX1 matrix into a device tensor of ``backend``'s dtype.

    Same result as ``torch.from_numpy(mmkit.load_matrix(path))`` cast to the
    backend dtype on its device (bitwise for fp64; fp32 rounded to nearest),
    without the host-side decode.  ``chunk_bytes`` is the pinned staging size.
    """
    if not isinstance(backend, Backend):
        raise TypeError("backend must be a Backend")
    if sys.byteorder != "little":
        raise MatrixFormatError("MMX1 streaming needs a little-endian host")
    rows, cols = read_mmx_header(path)
    torch = _lib.torch_mod()
    dev = backend.torch_device()
    dtype = backend.torch_dtype()
    out = torch.empty((rows, cols), dtype=dtype, device=dev)
    n = rows * cols
    if n == 0:
        return out
    if int(chunk_bytes) < 32:
        raise ShapeError(f"chunk_bytes must be at least 32, got {chunk_bytes}")
    total = n * 8
    # multiples of 32 bytes keep every fp32 destination slice 16-byte aligned
    chunk = min((int(chunk_bytes) // 32) * 32, (total + 31) // 32 * 32)
    pinned = [torch.empty(chunk, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    views = [memoryview(p.numpy()) for p in pinned]
    done = [None, None]
    narrow = dtype == torch.float32
    stage = ([torch.empty(chunk // 8, dtype=torch.float64, device=dev) for _ in range(2)]
             if narrow else None)
    flat = out.view(-1)
    stream = torch.cuda.Stream(device=dev)
    with open(path, "rb", buffering=0) as fh, torch.cuda.stream(stream):
        fh.seek(_PAYLOAD_OFFSET)
        off, k = 0, 0
        while off < total:
            b = k & 1
            if done[b] is not None:
                done[b].synchronize()          # the copy out of this buffer finished
            want = min(chunk, total - off)
            got = fh.readinto(views[b][:want])
            if got != want:
                raise MatrixFormatError(f"{path}: short read at payload byte {off}")
            e0, e1 = off // 8, (off + want) // 8
            if narrow:
                dst = stage[b][:e1 - e0]
                dst.view(torch.uint8).copy_(pinned[b][:want], non_blocking=True)
                _lib.call("mmk_f64_to_f32", _lib.ptr(dst), _lib.ptr(flat[e0:e1]), e1 - e0,
                          stream.cuda_stream)
            else:
                flat[e0:e1].view(torch.uint8).copy_(pinned[b][:want], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            done[b] = ev
            off += want
            k += 1
    torch.cuda.current_stream(dev).wait_stream(stream)
    return out
