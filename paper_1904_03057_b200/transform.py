"""Host-side field transforms (setup only; not on the solve hot path).

* ``direct_transform``: node samples -> B-spline coefficients by the
  separable causal/anticausal recursive prefilter with whole-sample mirror
  boundary, as in the reference (``/root/reference/pkg/src/bspde/bspline.py:
  140-242``; truncated-series causal init at 1e-12, closed-form anticausal
  init).
* ``transform_field``: constants stay exact, arrays/callables are sampled,
  prefiltered and reflect-padded by ``ext`` (``problem.py:178-194``).
* ``sample_solution``: coefficients -> node values, the b^n correlation
  (``problem.py:330-348``).
"""

from __future__ import annotations

import math
from functools import lru_cache

import numpy as np

from .errors import ValidationError
from .gram import basis_extension, bspline_pieces


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
    """Poles in (-1, 0) and gain of the inverse sampled-B-spline filter."""
    b = sampled_bspline(n)
    if len(b) == 1:
        return (), 1.0
    roots = np.roots(b)
    inside = sorted(z.real for z in roots if abs(z) < 1.0)
    gain = 1.0
    for z in inside:
        gain *= (1.0 - z) * (1.0 - 1.0 / z)
    return tuple(inside), gain


def _mirror_index(i, n):
    if n == 1:
        return 0
    period = 2 * n - 2
    i = i % period
    return period - i if i >= n else i


def _prefilter_last_axis(c, poles, gain, tol=1e-12):
    n = c.shape[-1]
    c = c * gain
    for z in poles:
        horizon = int(math.ceil(math.log(tol) / math.log(abs(z)))) + 1
        init = c[..., 0].copy()
        zk = 1.0
        for k in range(1, horizon):
            zk *= z
            init += zk * c[..., _mirror_index(k, n)]
        c[..., 0] = init
        for k in range(1, n):
            c[..., k] += z * c[..., k - 1]
        c[..., n - 1] = (z / (z * z - 1.0)) * (c[..., n - 1] + z * c[..., n - 2])
        for k in range(n - 2, -1, -1):
            c[..., k] = z * (c[..., k + 1] - c[..., k])
    return c


def direct_transform(samples, degree: int) -> np.ndarray:
    arr = np.asarray(samples, dtype=np.float64)
    if not np.all(np.isfinite(arr)):
        raise ValidationError("samples contain non-finite values")
    if degree <= 1:
        return arr.copy()
    if any(e < 2 for e in arr.shape):
        raise ValidationError(f"extents {arr.shape} too small for degree {degree}")
    poles, gain = compute_poles(degree)
    out = arr.copy()
    for axis in range(arr.ndim):
        moved = np.ascontiguousarray(np.moveaxis(out, axis, -1))
        moved = _prefilter_last_axis(moved, poles, gain)
        out = np.moveaxis(moved, -1, axis)
    return np.ascontiguousarray(out)


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


def transform_field(value, grid, degree: int) -> np.ndarray:
    """Scalar, node samples or callable -> extended-grid coefficients."""
    ext = basis_extension(degree)
    samples = sample_field(value, grid)
    if samples is None:
        return np.full(tuple(n + 2 * ext for n in grid.extents), float(value))
    coeffs = direct_transform(samples, degree)
    if ext > 0:
        coeffs = np.pad(coeffs, ext, mode="reflect")
    return coeffs


def sample_solution(coeffs_ext, grid, degree: int) -> np.ndarray:
    b = sampled_bspline(degree)
    m = len(b) // 2
    ext = basis_extension(degree)
    out = np.asarray(coeffs_ext, dtype=np.float64)
    for ax in range(grid.dim):
        acc = None
        for t, w in enumerate(b):
            sl = [slice(None)] * grid.dim
            sl[ax] = slice(ext - m + t, ext - m + t + grid.extents[ax])
            term = w * out[tuple(sl)]
            acc = term if acc is None else acc + term
        out = acc
    return out
