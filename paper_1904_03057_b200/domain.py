"""Uniform node grids and box domains.

Same semantics as the reference's ``Grid`` / ``BoxDomain``
(``/root/reference/pkg/src/bspde/domain.py:27-88``): extents are node
counts per axis, node ``k`` of axis ``a`` sits at ``origin[a] + k*step[a]``,
and the unknowns live on the *extended* grid of ``N + 2*ext(p)``
coefficients per axis.  :class:`MaskDomain` (voxel occupancy, reference
``domain.py:92-113``) with the node classification of ``domain.py:185-219``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import EmptyDomainError, ValidationError
from .gram import basis_extension  # noqa: F401  (re-exported API name)


@dataclass(frozen=True)
class Grid:
    extents: tuple
    step: tuple
    origin: tuple = None

    def __post_init__(self):
        extents = tuple(int(e) for e in np.atleast_1d(self.extents))
        step = tuple(float(h) for h in np.atleast_1d(self.step))
        origin = (0.0,) * len(extents) if self.origin is None else tuple(
            float(o) for o in np.atleast_1d(self.origin))
        object.__setattr__(self, "extents", extents)
        object.__setattr__(self, "step", step)
        object.__setattr__(self, "origin", origin)
        if not 1 <= len(extents) <= 3:
            raise ValidationError(f"dimension {len(extents)} not in 1..3")
        if len(step) != len(extents) or len(origin) != len(extents):
            raise ValidationError("extents, step and origin must have matching length")
        if any(e < 2 for e in extents):
            raise ValidationError(f"need at least 2 nodes per axis, got {extents}")
        if any(h <= 0 for h in step):
            raise ValidationError(f"grid steps must be positive, got {step}")

    @property
    def dim(self) -> int:
        return len(self.extents)

    @property
    def cell_extents(self) -> tuple:
        return tuple(e - 1 for e in self.extents)

    @property
    def num_nodes(self) -> int:
        return int(np.prod(self.extents))

    @property
    def lengths(self) -> tuple:
        return tuple((e - 1) * h for e, h in zip(self.extents, self.step))

    def node_coordinates(self, axis) -> np.ndarray:
        return self.origin[axis] + self.step[axis] * np.arange(self.extents[axis])


@dataclass(frozen=True)
class BoxDomain:
    """The full rectangular domain spanned by the grid."""

    grid: Grid

    @property
    def dim(self) -> int:
        return self.grid.dim

    def occupancy(self) -> np.ndarray:
        return np.ones(self.grid.cell_extents, dtype=bool)


@dataclass(frozen=True)
class MaskDomain:
    """Domain given by a boolean occupancy mask over the grid's cells
    (``domain.py:92-113``)."""

    grid: Grid
    mask: np.ndarray

    def __post_init__(self):
        mask = np.asarray(self.mask, dtype=bool)
        object.__setattr__(self, "mask", mask)
        if mask.shape != self.grid.cell_extents:
            raise ValidationError(
                f"mask extents {mask.shape} != cell extents {self.grid.cell_extents}")
        if not mask.any():
            raise EmptyDomainError("mask has no occupied cells")

    @property
    def dim(self) -> int:
        return self.grid.dim

    def occupancy(self) -> np.ndarray:
        return self.mask


def support_cell_radius(degree) -> int:
    """Cells on each side of a node that its spline support touches."""
    return (int(degree) + 2) // 2


def _node_windows(occ, degree, reduce):
    """Reduce (any / all) the occupancy over the 2r cells each extended node's
    support touches, separably per axis; cells beyond the grid are empty.
    Node i (spline index i - ext) touches cells i - ext - r .. i - ext + r - 1."""
    ext = basis_extension(degree)
    r = support_cell_radius(degree)
    out = np.pad(occ, ext + r, mode="constant", constant_values=False)
    for ax in range(occ.ndim):
        n = out.shape[ax] - 2 * r + 1
        acc = None
        for k in range(2 * r):
            sl = np.take(out, np.arange(k, k + n), axis=ax)
            acc = sl.copy() if acc is None else reduce(acc, sl)
        out = acc
    return out


def active_nodes(domain, degree) -> np.ndarray:
    """Extended-grid mask: the node's support touches an occupied cell
    (``domain.py:206-219``)."""
    return _node_windows(domain.occupancy(), degree, np.logical_or)


def interior_nodes(domain, degree) -> np.ndarray:
    """Extended-grid mask: every cell the node's support touches is occupied
    (``domain.py:185-203``)."""
    return _node_windows(domain.occupancy(), degree, np.logical_and)


NODE_INACTIVE, NODE_INTERIOR, NODE_BOUNDARY = 0, 1, 2


def node_classes(domain, degree) -> np.ndarray:
    """uint8 per extended node: 0 inactive, 1 interior (free-space stencil),
    2 boundary (stencil from the occupied cells of its support)."""
    act = active_nodes(domain, degree)
    inter = interior_nodes(domain, degree)
    cls = np.zeros(act.shape, dtype=np.uint8)
    cls[act] = NODE_BOUNDARY
    cls[inter] = NODE_INTERIOR
    return cls
