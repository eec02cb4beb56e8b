"""B-spline field transforms on the GPU (setup and I/O).

* ``direct_transform`` / ``prefilter_device``: node samples -> B-spline
  coefficients by the separable causal/anticausal recursive prefilter of the
  reference (``/root/reference/pkg/src/bspde/bspline.py:140-242``): gain,
  truncated-series causal init at relative tolerance 1e-12, closed-form
  anticausal init, ``mirror`` / ``replicate`` / ``zero`` extensions.  Runs in
  ``prefilter_kernel`` (one thread per line, every axis in place) through
  ``bspde_prefilter_lines``.
* ``transform_field`` / ``transform_field_device``: constants stay exact,
  arrays / callables are sampled, prefiltered and reflect-padded by ``ext``
  (``problem.py:178-194``) straight into the ghosted-slab layout.
* ``sample_solution`` / ``sample_solution_device``: coefficients -> node
  values, the separable b^n correlation (``problem.py:330-348``), three
  ``fir_axis_kernel`` passes.

Pole and sampled-spline values are computed on the host exactly as the
reference does (``np.roots``), so results agree to rounding.  There is no CPU
implementation here: without the native library and a B200 these raise
``NativeLibraryError`` (the oracle keeps its own numpy restatement for tests).
"""

from __future__ import annotations

import ctypes as C
from functools import lru_cache

import numpy as np

from . import _native as N
from .errors import OutOfDomainError, ValidationError
from .gram import basis_extension, bspline_pieces

EXTENSIONS = ("mirror", "replicate", "zero")


@lru_cache(maxsize=None)
def sampled_bspline(n: int) -> np.ndarray:
    """``beta^n`` at the integers -n//2..n//2 (exact, then rounded)."""
    m = n // 2
    vals = []
    for x in range(-m, m + 1):
        v = 0.0
        for lo, hi, poly in bspline_pieces(n):
            if lo <= x < hi or (x == hi and hi == bspline_pieces(n)[-1][1]):
                v = float(sum(c * x ** k for k, c in enumerate(poly)))
                break
        vals.append(v)
    return np.array(vals)


@lru_cache(maxsize=None)
def compute_poles(n: int):
    """Poles in (-1, 0) and gain of the inverse sampled-B-spline filter
    (bspline.py:140-155)."""
    b = sampled_bspline(n)
    if len(b) == 1:
        return (), 1.0
    roots = np.roots(b)
    inside = sorted(z.real for z in roots if abs(z) < 1.0)
    gain = 1.0
    for z in inside:
        gain *= (1.0 - z) * (1.0 - 1.0 / z)
    return tuple(inside), gain


def _degree_of(basis_or_degree) -> int:
    return int(getattr(basis_or_degree, "degree", basis_or_degree))


def _torch():
    import torch

    return torch


def _as3(t):
    while t.dim() < 3:
        t = t.unsqueeze(0)
    return t


def _i32(vals):
    return (C.c_int32 * 3)(*[int(v) for v in vals])


def _i64(vals):
    return (C.c_int64 * 3)(*[int(v) for v in vals])


# ---------------------------------------------------------------------------
# device-resident API (torch float64 CUDA tensors, any strides, d <= 3)


def prefilter_device(t, degree, extension="mirror", ndim=None, stream=None):
    """In place: direct B-spline transform along the last ``ndim`` (default
    all) axes of ``t``, in the reference's order (first real axis first)."""
    if extension not in EXTENSIONS:
        raise ValidationError(f"unknown extension {extension!r}; pick from {EXTENSIONS}")
    poles, gain = compute_poles(int(degree))
    if not poles:
        return t
    lib = N.load()
    t3 = _as3(t)
    ndim = t.dim() if ndim is None else int(ndim)
    parr = (C.c_double * 2)(*(list(poles) + [0.0] * (2 - len(poles))))
    code = EXTENSIONS.index(extension)
    for ax in range(3 - ndim, 3):
        n = t3.shape[ax]
        if n < 2:
            raise ValidationError(f"extent {n} too small for degree {degree} (need >= 2)")
        a, b = sorted((q for q in range(3) if q != ax), key=lambda q: t3.stride(q))
        N.check(lib.bspde_prefilter_lines(
            N.ptr(t3), n, t3.stride(ax), t3.shape[a], t3.shape[b], t3.stride(a), t3.stride(b),
            parr, len(poles), float(gain), code, N.stream_handle(stream)))
    return t


def reflect_pad_device(t, ext, ndim=None, stream=None):
    """In place: ``np.pad(inner, ext, mode='reflect')`` on the real axes of
    ``t`` whose inner region ``[ext, n - ext)`` holds the values."""
    if ext == 0:
        return t
    lib = N.load()
    t3 = _as3(t)
    ndim = t.dim() if ndim is None else ndim
    for ax in range(3 - ndim, 3):
        N.check(lib.bspde_reflect_pad(N.ptr(t3), _i32(t3.shape), _i64(t3.stride()), ax, int(ext),
                                      N.stream_handle(stream)))
    return t


def fir_axis_device(src, out, axis, offset, taps, stream=None):
    lib = N.load()
    s3, o3 = _as3(src), _as3(out)
    tp = (C.c_double * len(taps))(*[float(v) for v in taps])
    N.check(lib.bspde_fir_axis(N.ptr(s3), _i64(s3.stride()), N.ptr(o3), _i32(o3.shape),
                               _i64(o3.stride()), int(axis), int(offset), tp, len(taps),
                               N.stream_handle(stream)))
    return out


def transform_field_device(value, grid, degree: int, layout, device, out=None, stream=None,
                           prefilter="interpolation"):
    """Scalar, node samples or callable -> extended-grid coefficients in the
    ghosted-slab buffer ``out`` (allocated if None).  Constants stay exact.
    ``prefilter``: "interpolation" (direct transform) or "l2" (projection,
    degree >= 2; problem.py:178-194)."""
    torch = _torch()
    ext = basis_extension(degree)
    buf = layout.alloc(device) if out is None else out
    own = layout.owned(buf)
    samples = sample_field(value, grid)
    if samples is None:
        own.fill_(float(value))
        return buf
    if not np.all(np.isfinite(samples)):
        raise ValidationError("samples contain non-finite values")
    d = grid.dim
    own3 = own.reshape(own.shape)  # (cz, cy, cx) view
    inner = own3[tuple(slice(ext, own3.shape[a] - ext) if a >= 3 - d else slice(None)
                       for a in range(3))]
    inner.copy_(torch.from_numpy(np.ascontiguousarray(samples).reshape(inner.shape)))
    if prefilter == "l2" and degree >= 2:
        dense = inner.contiguous()
        l2_project_device(dense, degree, ndim=d)
        inner.copy_(dense)
    elif prefilter in ("interpolation", "l2"):
        prefilter_device(inner, degree, ndim=d, stream=stream)
    else:
        raise ValidationError(f"prefilter must be interpolation/l2, got {prefilter!r}")
    reflect_pad_device(own3, ext, ndim=d, stream=stream)
    return buf


def sample_solution_device(buf, grid, degree: int, layout, stream=None):
    """Ghosted-slab coefficients -> node values (torch, grid extents)."""
    torch = _torch()
    b = sampled_bspline(int(degree))
    m = len(b) // 2
    ext = basis_extension(degree)
    cur = layout.owned(buf)  # (cz, cy, cx)
    d = grid.dim
    for ax in range(3 - d, 3):
        shp = list(cur.shape)
        shp[ax] = grid.extents[ax - (3 - d)]
        nxt = torch.empty(shp, dtype=torch.float64, device=cur.device)
        fir_axis_device(cur, nxt, ax, ext - m, b, stream)
        cur = nxt
    return cur.reshape(tuple(grid.extents))


# ---------------------------------------------------------------------------
# host-array API (reference signatures; the work runs on the GPU)


def sample_field(value, grid):
    if callable(value):
        coords = np.meshgrid(*[grid.node_coordinates(a) for a in range(grid.dim)],
                             indexing="ij")
        return np.asarray(value(*coords), dtype=np.float64) * np.ones(grid.extents)
    arr = np.asarray(value, dtype=np.float64)
    if arr.ndim == 0:
        return None
    if arr.shape != tuple(grid.extents):
        raise ValidationError(f"field samples {arr.shape} != grid extents {grid.extents}")
    return arr


def direct_transform(samples, basis, extension="mirror", device=None):
    """Node samples -> spline coefficients (reference ``direct_transform``,
    bspline.py:214-242; ``basis`` may be a degree or an object with ``degree``)."""
    from .device import require_cuda

    torch = _torch()
    n = _degree_of(basis)
    if extension not in EXTENSIONS:
        raise ValidationError(f"unknown extension {extension!r}; pick from {EXTENSIONS}")
    arr = np.asarray(samples, dtype=np.float64)
    if hasattr(basis, "dim") and arr.ndim != basis.dim:
        raise ValidationError(f"samples are {arr.ndim}-d but basis is {basis.dim}-d")
    if arr.ndim > 3:
        raise ValidationError("at most 3-d samples")
    if not np.all(np.isfinite(arr)):
        raise ValidationError("samples contain non-finite values")
    if n >= 2 and any(e < 2 for e in arr.shape):
        raise ValidationError(f"extents {arr.shape} too small for degree {n} (need >= 2)")
    if n <= 1:
        return arr.copy()
    dev = require_cuda(device)
    t = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
    prefilter_device(t, n, extension)
    return t.cpu().numpy()


def transform_field(value, grid, degree: int, device=None, prefilter="interpolation") -> np.ndarray:
    """Scalar, node samples or callable -> extended-grid coefficients (host)."""
    from .device import SlabLayout, require_cuda

    ext = basis_extension(degree)
    cext = tuple(n + 2 * ext for n in grid.extents)
    if sample_field(value, grid) is None:
        return np.full(cext, float(value))
    dev = require_cuda(device)
    c3 = (1,) * (3 - len(cext)) + cext
    lay = SlabLayout(c3[0], c3[1], c3[2], ghost=0)
    buf = transform_field_device(value, grid, degree, lay, dev, prefilter=prefilter)
    return lay.download(buf).reshape(cext)


def sample_solution(coeffs_ext, grid, degree: int, device=None) -> np.ndarray:
    """Coefficients on the extended grid -> node values (host)."""
    from .device import SlabLayout, require_cuda

    dev = require_cuda(device)
    ext = basis_extension(degree)
    cext = tuple(n + 2 * ext for n in grid.extents)
    c = np.asarray(coeffs_ext, dtype=np.float64)
    if c.shape != cext:
        raise ValidationError(f"coefficients {c.shape} != extended extents {cext}")
    c3 = (1,) * (3 - len(cext)) + cext
    lay = SlabLayout(c3[0], c3[1], c3[2], ghost=0)
    buf = lay.upload(c.reshape(c3), dev)
    return sample_solution_device(buf, grid, degree, lay).cpu().numpy()


# ---------------------------------------------------------------------------
# spline evaluation on point lattices (indirect_transform, bspline.py:245-310)

_PAD_FOLD = {"mirror", "replicate", "zero"}


@lru_cache(maxsize=None)
def _float_pieces(n: int):
    return tuple((float(lo), tuple(float(c) for c in poly)) for lo, _, poly in bspline_pieces(n))


def bspline_eval(n: int, x) -> np.ndarray:
    """``beta^n(x)`` in float64 (piecewise polynomial, Horner), vectorized."""
    x = np.asarray(x, dtype=np.float64)
    pieces = _float_pieces(n)
    a0 = pieces[0][0]
    m = np.floor(x - a0).astype(np.int64)
    out = np.zeros_like(x)
    for k, (_, poly) in enumerate(pieces):
        sel = m == k
        if not sel.any():
            continue
        xs = x[sel]
        v = np.zeros_like(xs)
        for c in reversed(poly):
            v = v * xs + c
        out[sel] = v
    return out


def lattice_taps(n: int, step: float, points, size: int, first: int = 0, extension="mirror"):
    """Gather indices (extension folded in) and weights of the ``n+1`` taps of
    each point: ``k0 = floor(u - (n-1)/2)``, ``w_t = beta(u - k0 - t)`` with
    ``u = x / h`` (``_tap_matrix``, bspline.py:245-250); coefficient ``k`` is
    array index ``k - first``."""
    if extension not in _PAD_FOLD:
        raise ValidationError(f"unknown extension {extension!r}")
    u = np.asarray(points, dtype=np.float64) / float(step)
    lo, hi = first, first + size - 1
    bad = (u < lo - 1e-12) | (u > hi + 1e-12)
    if np.any(bad):
        raise OutOfDomainError(f"grid coordinate {u[bad][0]} outside node span [{lo}, {hi}]")
    k0 = np.floor(u - (n - 1) / 2.0).astype(np.int64)
    taps = np.arange(n + 1)
    w = bspline_eval(n, u[:, None] - (k0[:, None] + taps[None, :]))
    idx = k0[:, None] + taps[None, :] - first
    if size == 1:
        idx = np.zeros_like(idx)
    elif extension == "mirror":  # np.pad "reflect"
        period = 2 * (size - 1)
        idx = np.abs(idx) % period
        idx = np.where(idx >= size, period - idx, idx)
    elif extension == "replicate":
        idx = np.clip(idx, 0, size - 1)
    else:
        w = np.where((idx < 0) | (idx >= size), 0.0, w)
        idx = np.clip(idx, 0, size - 1)
    return idx.astype(np.int32), w


def evaluate_lattice_device(coeffs, degree: int, steps, axis_points, first_index=None,
                            extension="mirror", stream=None):
    """Evaluate the expansion with coefficients ``coeffs`` (dense torch CUDA
    tensor, 1-3 d) at the tensor lattice ``axis_points`` (one 1-d array of
    physical coordinates relative to the origin per axis): one
    ``bspde_resample_axis`` launch per axis.  Returns a dense tensor."""
    torch = _torch()
    lib = N.load()
    d = coeffs.dim()
    first = tuple(first_index) if first_index is not None else (0,) * d
    cur = coeffs.reshape((1,) * (3 - d) + tuple(coeffs.shape))
    for ax in range(d):
        a3 = ax + 3 - d
        idx, w = lattice_taps(int(degree), steps[ax], axis_points[ax], cur.shape[a3], first[ax],
                              extension)
        shape = list(cur.shape)
        shape[a3] = len(axis_points[ax])
        out = torch.empty(shape, dtype=torch.float64, device=cur.device)
        it = torch.from_numpy(np.ascontiguousarray(idx)).to(cur.device)
        wt = torch.from_numpy(np.ascontiguousarray(w)).to(cur.device)
        N.check(lib.bspde_resample_axis(N.ptr(cur), _i64(cur.stride()), N.ptr(out),
                                        _i32(out.shape), _i64(out.stride()), a3, N.ptr(it),
                                        N.ptr(wt), int(idx.shape[1]), N.stream_handle(stream)))
        cur = out
    return cur.reshape(tuple(len(p) for p in axis_points))


def indirect_transform_lattice(coeffs, degree: int, steps, axis_points, first_index=None,
                               extension="mirror", device=None) -> np.ndarray:
    """Host wrapper of :func:`evaluate_lattice_device` (reference
    ``indirect_transform`` at the points of a tensor lattice)."""
    from .device import require_cuda

    torch = _torch()
    dev = require_cuda(device)
    c = torch.from_numpy(np.ascontiguousarray(coeffs, dtype=np.float64)).to(dev)
    return evaluate_lattice_device(c, degree, steps, axis_points, first_index,
                                   extension).cpu().numpy()


def indirect_transform(coeffs, basis, points, extension="mirror", first_index=None, step=None,
                       device=None) -> np.ndarray:
    """The expansion at arbitrary points (reference ``indirect_transform``,
    bspline.py:253-310): ``points`` (npts, dim) physical coordinates with node
    ``k`` at ``k*h``; ``basis`` a degree (then ``step`` gives h per axis) or an
    object with ``degree`` and ``step``.  One thread per point on the GPU."""
    from .device import require_cuda

    torch = _torch()
    n = _degree_of(basis)
    arr = np.asarray(coeffs, dtype=np.float64)
    d = arr.ndim
    steps = tuple(getattr(basis, "step", None) or step or (1.0,) * d)
    if hasattr(basis, "dim") and basis.dim != d:
        raise ValidationError(f"coefficients are {d}-d but basis is {basis.dim}-d")
    if extension not in EXTENSIONS:
        raise ValidationError(f"unknown extension {extension!r}; pick from {EXTENSIONS}")
    pts = np.asarray(points, dtype=np.float64)
    if d == 1 and pts.ndim == 1:
        pts = pts[:, None]
    if pts.ndim == 1:
        pts = pts[None, :]
    if pts.shape[-1] != d:
        raise ValidationError(f"points have {pts.shape[-1]} components, basis is {d}-d")
    first = tuple(first_index) if first_index is not None else (0,) * d
    npts, nt = pts.shape[0], n + 1
    idx = np.zeros((3, npts, nt), dtype=np.int32)
    w = np.zeros((3, npts, nt))
    w[: 3 - d, :, 0] = 1.0  # leading singleton axes
    for ax in range(d):
        i, wt = lattice_taps(n, steps[ax], pts[:, ax], arr.shape[ax], first[ax], extension)
        idx[3 - d + ax], w[3 - d + ax] = i, wt
    dev = require_cuda(device)
    c3 = torch.from_numpy(np.ascontiguousarray(arr.reshape((1,) * (3 - d) + arr.shape))).to(dev)
    it = torch.from_numpy(idx).to(dev)
    wt_ = torch.from_numpy(w).to(dev)
    out = torch.empty(npts, dtype=torch.float64, device=dev)
    N.check(N.load().bspde_eval_points(N.ptr(c3), _i64(c3.stride()), npts, nt, N.ptr(it),
                                       N.ptr(wt_), N.ptr(out), N.stream_handle()))
    return out.cpu().numpy()


# ---------------------------------------------------------------------------
# "l2" prefilter (ProblemSpec(prefilter="l2"); _l2_project_axis,
# problem.py:142-175): per axis, the projection of the piecewise-linear
# interpolant onto the degree-n spline space -- rhs through the (1, n) cross
# table (terms falling off the line are dropped), then the Gram system of the
# sampled beta^(2n+1) with mirror folding.  On the GPU: the FIR is one
# bspde_resample_axis launch, the solve one bspde_banded_solve_lines launch
# with banded LU factors (no pivoting; shared by every line) from the host.


@lru_cache(maxsize=None)
def l2_cross(degree: int) -> np.ndarray:
    """``r[o] = int beta^1(x - o) beta^n(x) dx`` for o = -R..R (exact)."""
    from .gram import multi_product_integral

    R = (degree + 3) // 2
    taps = [float(multi_product_integral([(1, o, 0), (int(degree), 0, 0)]))
            for o in range(-R, R + 1)]
    while taps and taps[0] == 0.0 and taps[-1] == 0.0:
        taps = taps[1:-1]
    return np.array(taps)


@lru_cache(maxsize=None)
def l2_factors(n: int, degree: int):
    """(lb, ub, m): banded LU of the mirror-folded Gram matrix of the sampled
    beta^(2 degree + 1) on a line of n samples."""
    gd = 2 * int(degree) + 1
    m = gd // 2
    if n < m + 1:
        raise ValidationError(f"line of {n} samples too short for the l2 prefilter of degree "
                              f"{degree} (need >= {m + 1})")
    g = bspline_eval(gd, np.arange(-m, m + 1).astype(float))
    A = np.zeros((n, n))
    for t in range(-m, m + 1):
        j = np.arange(n) + t
        j = np.where(j < 0, -j, np.where(j >= n, 2 * n - 2 - j, j))
        np.add.at(A, (np.arange(n), j), g[t + m])
    U, lb = A.copy(), np.zeros((n, m))
    for k in range(n):
        hi = min(n, k + m + 1)
        for i in range(k + 1, hi):
            f = U[i, k] / U[k, k]
            lb[i, i - k - 1] = f
            U[i, k:hi] -= f * U[k, k:hi]
    ub = np.zeros((n, m + 1))
    for k in range(m + 1):
        ub[: n - k, k] = np.diagonal(U, k)
    return lb, ub, m


def l2_project_device(t, degree, ndim=None, stream=None):
    """In place: the "l2" prefilter along the last ``ndim`` axes of the dense
    CUDA tensor ``t`` (first real axis first, like the reference).  Runs on
    the current stream (``stream`` must be None or the current stream: the
    per-axis tables are uploaded there)."""
    torch = _torch()
    lib = N.load()
    ndim = t.dim() if ndim is None else int(ndim)
    cross = l2_cross(int(degree))
    rw = (len(cross) - 1) // 2
    cur = _as3(t)
    for ax in range(3 - ndim, 3):
        n = cur.shape[ax]
        lb, ub, m = l2_factors(n, int(degree))
        i = np.arange(n)[:, None] + (np.arange(len(cross)) - rw)[None, :]
        w = np.where((i >= 0) & (i < n), cross[None, :], 0.0)
        idx = np.clip(i, 0, n - 1).astype(np.int32)
        it = torch.from_numpy(np.ascontiguousarray(idx)).to(cur.device)
        wt = torch.from_numpy(np.ascontiguousarray(w)).to(cur.device)
        out = torch.empty_like(cur)
        N.check(lib.bspde_resample_axis(N.ptr(cur), _i64(cur.stride()), N.ptr(out),
                                        _i32(out.shape), _i64(out.stride()), ax, N.ptr(it),
                                        N.ptr(wt), len(cross), N.stream_handle(stream)))
        lbt = torch.from_numpy(np.ascontiguousarray(lb)).to(cur.device)
        ubt = torch.from_numpy(np.ascontiguousarray(ub)).to(cur.device)
        a, b = sorted((q for q in range(3) if q != ax), key=lambda q: out.stride(q))
        N.check(lib.bspde_banded_solve_lines(N.ptr(out), n, out.stride(ax), out.shape[a],
                                             out.shape[b], out.stride(a), out.stride(b),
                                             N.ptr(lbt), N.ptr(ubt), m,
                                             N.stream_handle(stream)))
        cur = out
    _as3(t).copy_(cur)
    return t
