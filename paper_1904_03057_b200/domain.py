"""Uniform node grids and box domains.

Same semantics as the reference's ``Grid`` / ``BoxDomain``
(``/root/reference/pkg/src/bspde/domain.py:27-88``): extents are node
counts per axis, node ``k`` of axis ``a`` sits at ``origin[a] + k*step[a]``,
and the unknowns live on the *extended* grid of ``N + 2*ext(p)``
coefficients per axis.  Mask (voxel) domains are out of scope for this
build.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ValidationError
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
