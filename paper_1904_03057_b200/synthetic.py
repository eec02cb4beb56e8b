"""Synthetic heat inputs for large configs, generated on the GPU (setup only).

The SURVEY.md §8(d) initial condition and source are separable Gaussians,
``amp * exp(-w |x - c|^2) = amp * gz(z) gy(y) gx(x)``, and the prefilter
(``transform.direct_transform``) and the reflect padding act axis by axis,
so the extended-grid coefficients are the outer product of three 1-D
coefficient vectors.  Those are computed on the host (O(N)) and expanded on
the device straight into the ghosted-slab layout -- no 6 GB host arrays at
the 930^3 paper scale.  Outside every timed region.
"""

from __future__ import annotations

import numpy as np

from .gram import basis_extension
from .transform import direct_transform


def gaussian_1d_coeffs(N, h, p, center, width):
    x = np.arange(N) * h
    c = direct_transform(np.exp(-width * (x - center) ** 2), p)
    ext = basis_extension(p)
    return np.pad(c, ext, mode="reflect") if ext else c


def gaussian_coeffs(N, h, p, center, width, amp, device, out=None, layout=None, z_range=None):
    """Coefficients of ``amp*exp(-width*|x-center|^2)`` on the (N+2ext)^3
    extended grid (center given as (z, y, x)).  Writes the owned planes
    ``z_range`` (default all) into ``out`` when a layout is given."""
    import torch

    cz, cy, cx = (gaussian_1d_coeffs(N, h, p, center[a], width) for a in range(3))
    if z_range is not None:
        cz = cz[z_range[0]:z_range[1]]
    tz, ty, tx = (torch.from_numpy(np.ascontiguousarray(v)).to(device) for v in (cz, cy, cx))
    if out is None:
        return amp * tz[:, None, None] * ty[None, :, None] * tx[None, None, :]
    dst = layout.owned(out)
    for k in range(dst.shape[0]):  # plane by plane: no full-size temporaries
        dst[k].copy_((amp * tz[k]) * ty[:, None] * tx[None, :])
    return out


def heat_c_inputs(ncoef, p=3, lam=4.0):
    """(N, h, dt) of the synthetic heat problem with ncoef^3 coefficients."""
    ext = basis_extension(p)
    N = ncoef - 2 * ext
    h = 1.0 / (N - 1)
    return N, h, lam * h * h


IC = dict(center=(0.5, 0.4, 0.6), width=40.0, amp=1.0)
SOURCE = dict(center=(0.3, 0.6, 0.5), width=60.0, amp=10.0)


def leg_mask(extents=(60, 60, 240)):
    """The reference's synthetic leg (``make_leg_mask``, domain.py:275-293):
    cells of a tube along axis 2 whose centre wanders (sin / cos in the
    axial coordinate) and whose radius tapers from 0.30 to 0.20 of the
    axis-0 cell count, with an 'arteria' of 0.22 x that radius inside.
    Returns ``(mask, arteria)`` bool cell arrays."""
    n0, n1, n2 = (e - 1 for e in extents)
    t = (np.arange(n2) + 0.5) / n2
    c0 = n0 / 2.0 + 0.08 * n0 * np.sin(2 * np.pi * t)
    c1 = n1 / 2.0 + 0.06 * n1 * np.cos(np.pi * t)
    rad = n0 * (0.30 - 0.10 * t)
    a0 = (np.arange(n0) + 0.5)[:, None, None]
    a1 = (np.arange(n1) + 0.5)[None, :, None]
    d2 = (a0 - c0[None, None, :]) ** 2 + (a1 - c1[None, None, :]) ** 2
    return d2 <= rad[None, None, :] ** 2, d2 <= (0.22 * rad[None, None, :]) ** 2
