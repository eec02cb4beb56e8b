"""TBSF tensor files for coefficient checkpoints.

Same on-disk format and error behaviour as the reference
(``/root/reference/pkg/src/bspde/io.py:20-82``): a little-endian header
``b"TBSF", u32 version = 1, u32 ndim`` (``ndim`` in 1..3), ``ndim`` u64
extents, ``u8`` dtype tag (0 = f4, 1 = f8), ``i8`` spline degree, then the
row-major payload; written to a temporary file and renamed into place.

The B200 side: fields live in HBM in the ghosted-slab layout
(:mod:`.device`), so :func:`write_field` / :func:`read_field` move the owned
region through one pinned staging buffer in slices of z planes (one
device<->host copy per slice, overlapping nothing but the file system) instead
of materialising a pageable host copy of a 6.4 GB field first.
"""

from __future__ import annotations

import os
import struct
import tempfile

import numpy as np

from .errors import FormatError

TBSF_MAGIC = b"TBSF"
TBSF_VERSION = 1
_TAG_OF = {np.dtype("<f4"): 0, np.dtype("<f8"): 1}
_DTYPE_OF = {0: np.dtype("<f4"), 1: np.dtype("<f8")}
_SLICE_BYTES = 256 << 20


def _header(shape, dtype, degree) -> bytes:
    return (struct.pack("<4sII", TBSF_MAGIC, TBSF_VERSION, len(shape))
            + struct.pack(f"<{len(shape)}Q", *shape)
            + struct.pack("<Bb", _TAG_OF[dtype], int(degree)))


def _atomic(path, write_body):
    """Write through a temporary file in the target directory, then rename
    (``io.py:26-37``)."""
    directory = os.path.dirname(os.path.abspath(path)) or "."
    fd, tmp = tempfile.mkstemp(dir=directory, prefix=".tbsf-tmp")
    try:
        with os.fdopen(fd, "wb") as f:
            write_body(f)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def _parse_header(f, size):
    """Validate the header (``io.py:52-79``); returns (extents, dtype, degree,
    payload offset).  Error messages and byte offsets follow the reference."""
    if size < 12:
        raise FormatError("file shorter than the fixed header", offset=size)
    head = f.read(12)
    magic, version, ndim = struct.unpack_from("<4sII", head, 0)
    if magic != TBSF_MAGIC:
        raise FormatError(f"bad magic {magic!r}, expected {TBSF_MAGIC!r}", offset=0)
    if version != TBSF_VERSION:
        raise FormatError(f"unsupported version {version}", offset=4)
    if not 1 <= ndim <= 3:
        raise FormatError(f"dimension {ndim} not in 1..3", offset=8)
    off = 12
    if size < off + 8 * ndim + 2:
        raise FormatError("truncated extents header", offset=size)
    rest = f.read(8 * ndim + 2)
    extents = struct.unpack_from(f"<{ndim}Q", rest, 0)
    dtag, degree = struct.unpack_from("<Bb", rest, 8 * ndim)
    off += 8 * ndim + 2
    if dtag not in _DTYPE_OF:
        raise FormatError(f"unknown dtype tag {dtag}", offset=off - 2)
    dt = _DTYPE_OF[dtag]
    want = int(np.prod(extents)) * dt.itemsize
    have = size - off
    if have != want:
        raise FormatError(
            f"payload holds {have} bytes, extents {tuple(extents)} require {want}", offset=off)
    return tuple(int(e) for e in extents), dt, int(degree), off


def write_tensor(path, array, degree=-1):
    """Write a TBSF file from a numpy array or a (CUDA) torch tensor; float32
    stays f4, everything else is stored as f8 (``io.py:40-49``)."""
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(array, torch.Tensor):
        if array.dtype == torch.float32:
            array = array.detach().cpu().numpy()
        else:
            array = array.detach().to(torch.float64).cpu().numpy()
    arr = np.ascontiguousarray(array)
    dt = np.dtype("<f4") if arr.dtype == np.float32 else np.dtype("<f8")
    arr = arr.astype(dt, copy=False)
    head = _header(arr.shape, dt, degree)
    _atomic(path, lambda f: (f.write(head), f.write(memoryview(arr).cast("B"))))


def read_tensor(path):
    """Read a TBSF file; returns ``(array, degree)`` (``io.py:52-82``)."""
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        extents, dt, degree, _ = _parse_header(f, size)
        arr = np.empty(extents, dtype=dt)
        f.readinto(memoryview(arr).cast("B"))
    return arr, degree


def _staging(layout, torch):
    plane = layout.ny * layout.nx * 8
    zs = max(1, min(layout.nz, _SLICE_BYTES // plane))
    return zs, torch.empty((zs, layout.ny, layout.nx), dtype=torch.float64, pin_memory=True)


def write_field(path, layout, buf, degree=-1, extents=None):
    """Checkpoint the owned region of a device field (slab layout) as an f8
    TBSF file, staged through pinned memory in z slices.  ``extents``: the
    header extents (default the 3-D owned shape); a 1-D / 2-D problem passes
    its real coefficient extents (``data.cext``), whose product is the same."""
    import torch

    own = layout.owned(buf)
    zs, stage = _staging(layout, torch)
    extents = tuple(layout.owned_shape) if extents is None else tuple(int(e) for e in extents)
    if int(np.prod(extents)) != int(np.prod(layout.owned_shape)):
        raise FormatError(f"extents {extents} do not match the field {layout.owned_shape}")
    head = _header(extents, np.dtype("<f8"), degree)

    def body(f):
        f.write(head)
        for z0 in range(0, layout.nz, zs):
            n = min(zs, layout.nz - z0)
            stage[:n].copy_(own[z0:z0 + n])  # synchronous D2H into pinned memory
            f.write(memoryview(stage[:n].numpy()).cast("B"))

    _atomic(path, body)


def read_field(path, layout, device, buf=None, degree=None, extents=None):
    """Load a TBSF file into a (new or given) device field; checks the
    extents (``extents``: the expected ones, default the 3-D owned shape --
    a 1-D / 2-D problem passes ``data.cext``) and, if given, the degree."""
    import torch

    want = tuple(layout.owned_shape) if extents is None else tuple(int(e) for e in extents)
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        extents, dt, deg, _ = _parse_header(f, size)
        if extents != want:
            raise FormatError(f"file extents {extents} != field extents {want}")
        if degree is not None and deg != int(degree):
            raise FormatError(f"file holds degree {deg}, expected {int(degree)}")
        if buf is None:
            buf = layout.alloc(device)
        own = layout.owned(buf)
        zs, stage = _staging(layout, torch)
        item = dt.itemsize
        for z0 in range(0, layout.nz, zs):
            n = min(zs, layout.nz - z0)
            if dt == np.dtype("<f8"):
                f.readinto(memoryview(stage[:n].numpy()).cast("B"))
                own[z0:z0 + n].copy_(stage[:n])
            else:
                raw = np.frombuffer(f.read(n * layout.ny * layout.nx * item), dtype=dt)
                own[z0:z0 + n].copy_(torch.from_numpy(raw.astype(np.float64))
                                     .reshape(n, layout.ny, layout.nx))
    return buf, deg


# ---------------------------------------------------------------------------
# mask volumes and VTK export (io.py:85-144): the input and output formats of
# the masked (CT-leg) runs

MASK_MAGIC = "TBSM"


def write_mask(path, volume, threshold=128):
    """Mask file: ``TBSM v1`` / ``extents ...`` / ``threshold t`` text lines,
    then the raw uint8 volume (C order)."""
    vol = np.ascontiguousarray(volume, dtype=np.uint8)
    head = (f"{MASK_MAGIC} v1\nextents {' '.join(str(e) for e in vol.shape)}\n"
            f"threshold {int(threshold)}\n").encode()
    _atomic(path, lambda f: (f.write(head), f.write(memoryview(vol).cast("B"))))


def read_mask(path):
    """``(occupancy, threshold)``: the volume thresholded at ``>= threshold``."""
    with open(path, "rb") as f:
        blob = f.read()
    k = blob.find(b"threshold")
    end = blob.find(b"\n", k) + 1 if k >= 0 else 0
    if k < 0 or end == 0:
        raise FormatError("missing mask header lines", offset=0)
    lines = blob[:end].decode(errors="replace").splitlines()
    if not lines[0].startswith(MASK_MAGIC):
        raise FormatError(f"bad mask magic {lines[0][:8]!r}", offset=0)
    extents = tuple(int(t) for t in lines[1].split()[1:])
    threshold = int(lines[2].split()[1])
    want = int(np.prod(extents))
    if len(blob) - end != want:
        raise FormatError(f"mask payload holds {len(blob) - end} bytes, extents {extents} "
                          f"require {want}", offset=end)
    vol = np.frombuffer(blob, dtype=np.uint8, count=want, offset=end).reshape(extents)
    return vol >= threshold, threshold


def export_vtk(path, samples, grid, name="field"):
    """Legacy ASCII VTK STRUCTURED_POINTS of a 2-D / 3-D node field (array
    axis 0 is VTK's x, so values go out in Fortran order)."""
    from .errors import ValidationError

    arr = np.asarray(samples, dtype=float)
    if arr.ndim not in (2, 3):
        raise ValidationError(f"VTK export needs a 2-D or 3-D field, got {arr.ndim}-D")
    pad = 3 - arr.ndim
    dims = arr.shape + (1,) * pad
    spacing = tuple(grid.step) + (1.0,) * pad
    origin = tuple(grid.origin) + (0.0,) * pad
    head = ["# vtk DataFile Version 3.0", name, "ASCII", "DATASET STRUCTURED_POINTS",
            "DIMENSIONS {} {} {}".format(*dims),
            "ORIGIN {:.10g} {:.10g} {:.10g}".format(*origin),
            "SPACING {:.10g} {:.10g} {:.10g}".format(*spacing),
            f"POINT_DATA {arr.size}", f"SCALARS {name} double 1", "LOOKUP_TABLE default"]
    body = "\n".join(f"{v:.10e}" for v in arr.ravel(order="F"))
    text = "\n".join(head) + "\n" + body + ("\n" if arr.size else "")
    _atomic(path, lambda f: f.write(text.encode()))


__all__ = ["TBSF_MAGIC", "TBSF_VERSION", "write_tensor", "read_tensor", "write_field", "read_field",
           "MASK_MAGIC", "write_mask", "read_mask", "export_vtk"]
