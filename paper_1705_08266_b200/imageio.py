"""Image files: binary PGM and the reference's raw float format.

Same formats, normalisation and errors as ``liftfuse/imageio.py``:

* PGM ``P5`` with 8-bit (maxval <= 255) or 16-bit big-endian samples; comments
  may sit between header tokens (imageio.py:27-52).  Samples are scaled to
  [0, 1] float64 on read; on write they are clipped to [0, 1], scaled by
  maxval and rounded half-to-even (imageio.py:55-63).
* raw ``LFRW``: 16-byte header -- magic, little-endian uint32 width, height and
  bytes per sample (4 = float32, 8 = float64) -- then row-major little-endian
  samples (imageio.py:65-98).
* :func:`read_image` sniffs the magic; :func:`write_image` picks PGM for a
  ``.pgm`` suffix and raw otherwise (imageio.py:100-109).

New here: :func:`read_raw_pinned` reads a raw image's payload straight into a
page-locked host tensor in chunks (no intermediate bytes object), the buffer
:meth:`Transform.dwt_host` streams to the GPU; :func:`read_raw_device` does the
same while uploading each chunk as soon as it is read, so disk and PCIe
overlap for 16-64 GiB images.
"""

from __future__ import annotations

import re
import struct

import numpy as np

from .engine import Image2D

__all__ = [
    "RAW_MAGIC",
    "read_image",
    "write_image",
    "read_pgm",
    "write_pgm",
    "read_raw",
    "write_raw",
    "raw_header",
    "read_raw_pinned",
    "read_raw_device",
]

RAW_MAGIC = b"LFRW"
_RAW_DTYPES = {4: np.dtype("<f4"), 8: np.dtype("<f8")}
_PGM_TOKEN = re.compile(rb"(?:\s+|\s*#[^\n]*\n)*(\d+)")


def read_pgm(path) -> Image2D:
    """Binary PGM -> float64 image in [0, 1]."""
    with open(path, "rb") as fh:
        data = fh.read()
    if not data.startswith(b"P5"):
        raise ValueError(f"{path}: not a binary PGM file")
    pos, vals = 2, []
    for _ in range(3):  # width, height, maxval
        m = _PGM_TOKEN.match(data, pos)
        if m is None:
            raise ValueError(f"{path}: malformed PGM header")
        vals.append(int(m.group(1)))
        pos = m.end()
    width, height, maxval = vals
    pos += 1  # the single whitespace byte that ends the header
    if not 0 < maxval < 65536:
        raise ValueError(f"{path}: unsupported PGM maxval {maxval}")
    dt = np.dtype(">u2") if maxval > 255 else np.dtype("u1")
    n = width * height
    if len(data) - pos < n * dt.itemsize:
        raise ValueError(f"{path}: truncated PGM data")
    px = np.frombuffer(data, dtype=dt, count=n, offset=pos).reshape(height, width)
    return Image2D(px.astype(np.float64) / float(maxval))


def write_pgm(path, image: Image2D, maxval: int = 255) -> None:
    if not 0 < maxval < 65536:
        raise ValueError(f"unsupported PGM maxval {maxval}")
    q = np.rint(np.clip(image.data.astype(np.float64), 0.0, 1.0) * maxval)
    dt = np.dtype(">u2") if maxval > 255 else np.dtype("u1")
    with open(path, "wb") as fh:
        fh.write(b"P5\n%d %d\n%d\n" % (image.width, image.height, maxval))
        fh.write(q.astype(dt).tobytes())


def raw_header(path):
    """(width, height, numpy little-endian dtype) of a raw file; validates the magic."""
    with open(path, "rb") as fh:
        head = fh.read(16)
    if len(head) != 16 or head[:4] != RAW_MAGIC:
        raise ValueError(f"{path}: not a raw image file (bad magic)")
    width, height, sb = struct.unpack("<III", head[4:])
    if sb not in _RAW_DTYPES:
        raise ValueError(f"{path}: unsupported sample width {sb}")
    return width, height, _RAW_DTYPES[sb]


def read_raw(path) -> Image2D:
    width, height, dt = raw_header(path)
    n = width * height
    with open(path, "rb") as fh:
        fh.seek(16)
        payload = fh.read(n * dt.itemsize)
    if len(payload) < n * dt.itemsize:
        raise ValueError(f"{path}: truncated raw data")
    arr = np.frombuffer(payload, dtype=dt, count=n).reshape(height, width)
    return Image2D(arr.astype(dt.newbyteorder("=")))


def write_raw(path, image: Image2D) -> None:
    arr = image.data
    with open(path, "wb") as fh:
        fh.write(RAW_MAGIC + struct.pack("<III", image.width, image.height, arr.dtype.itemsize))
        fh.write(np.ascontiguousarray(arr, dtype=arr.dtype.newbyteorder("<")).tobytes())


def read_image(path) -> Image2D:
    with open(path, "rb") as fh:
        magic = fh.read(4)
    if magic[:2] == b"P5":
        return read_pgm(path)
    if magic == RAW_MAGIC:
        return read_raw(path)
    raise ValueError(f"{path}: unrecognized image format (expected PGM or raw)")


def write_image(path, image: Image2D) -> None:
    if str(path).lower().endswith(".pgm"):
        write_pgm(path, image)
    else:
        write_raw(path, image)


# -- large-image ingest ------------------------------------------------------------------

_CHUNK = 64 << 20  # bytes per read


def _readinto_rows(fh, view: memoryview, path) -> None:
    done = 0
    while done < len(view):
        got = fh.readinto(view[done:done + _CHUNK])
        if not got:
            raise ValueError(f"{path}: truncated raw data")
        done += got


def read_raw_pinned(path, out=None):
    """Raw image -> page-locked CPU tensor ``[H, W]`` (float32/float64), read in
    64 MiB chunks straight into the pinned pages.  ``out`` may be a preallocated
    pinned tensor of the right shape and dtype (reused across files)."""
    import torch

    width, height, dt = raw_header(path)
    tdt = torch.float32 if dt.itemsize == 4 else torch.float64
    if out is None:
        out = torch.empty((height, width), dtype=tdt, pin_memory=torch.cuda.is_available())
    elif tuple(out.shape) != (height, width) or out.dtype != tdt or not out.is_contiguous():
        raise ValueError(f"{path}: output buffer must be a contiguous {height}x{width} {tdt} tensor")
    view = memoryview(out.numpy()).cast("B")  # little-endian hosts: the payload is the tensor's bytes
    with open(path, "rb") as fh:
        fh.seek(16)
        _readinto_rows(fh, view, path)
    return out


def read_raw_device(path, device="cuda", rows_per_chunk: int | None = None):
    """Raw image -> CUDA tensor, reading the next chunk from disk while the
    previous one uploads (two pinned staging buffers, one copy stream)."""
    import torch

    width, height, dt = raw_header(path)
    tdt = torch.float32 if dt.itemsize == 4 else torch.float64
    dev = torch.empty((height, width), dtype=tdt, device=device)
    row_bytes = width * dt.itemsize
    rows = rows_per_chunk or max(1, _CHUNK // max(1, row_bytes))
    stage = [torch.empty((min(rows, height), width), dtype=tdt, pin_memory=True) for _ in range(2)]
    done = [None, None]
    copy = torch.cuda.Stream(device=dev.device)
    with open(path, "rb") as fh:
        fh.seek(16)
        for i, r0 in enumerate(range(0, height, rows)):
            n = min(rows, height - r0)
            buf = stage[i % 2]
            if done[i % 2] is not None:
                done[i % 2].synchronize()  # the upload that last used this buffer
            _readinto_rows(fh, memoryview(buf[:n].numpy()).cast("B"), path)
            with torch.cuda.stream(copy):
                dev[r0:r0 + n].copy_(buf[:n], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy)
            done[i % 2] = ev
    torch.cuda.current_stream(dev.device).wait_stream(copy)
    return dev
