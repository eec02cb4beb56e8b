"""Box-face boundary conditions -> surface-term specs (host setup).

Mirrors the reference's condition types and their realization
(``/root/reference/pkg/src/bspde/problem.py:23-45`` and ``realize_bc``,
``problem.py:237-300``) for box domains: ``Neumann`` (no term), ``Robin``
(weight ``1/(2 gamma)``) and ``DirichletPenalty`` (weight ``1/epsilon``,
right-hand-side value ``g``; ``epsilon`` defaults to ``1e-4 * min(h)``).
The resulting ``(axis, side, weight, rhs_value)`` specs feed
:func:`.system.build_system` / :func:`.system.heat_system`, where each face
folds into the edge rows of one axis' stiffness factor.
Mask domains are out of scope for the b200 strategy.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigurationError

FACE_NAMES = ("x0", "x1", "y0", "y1", "z0", "z1")  # reference axis order (axis 0 = "x")


@dataclass(frozen=True)
class Robin:
    """``2 gamma D (grad phi . n) + phi = 0``: surface weight ``1/(2 gamma)``."""

    gamma: float = 1.0

    def surface(self, grid):
        if self.gamma <= 0:
            raise ConfigurationError(f"Robin gamma must be positive, got {self.gamma}")
        return 1.0 / (2.0 * self.gamma), None


@dataclass(frozen=True)
class Neumann:
    """Homogeneous natural condition: no surface term."""

    def surface(self, grid):
        return None


@dataclass(frozen=True)
class DirichletPenalty:
    """Dirichlet value ``value`` enforced by a penalty term of weight
    ``1/epsilon`` (``epsilon=None``: ``1e-4 * min(h)``)."""

    value: float = 0.0
    epsilon: float = None

    def surface(self, grid):
        eps = 1e-4 * min(grid.step) if self.epsilon is None else self.epsilon
        if eps <= 0:
            raise ConfigurationError(f"penalty epsilon must be positive, got {eps}")
        return 1.0 / eps, self.value


def _surface_of(cond, grid):
    """(weight, rhs value) of a face condition, or None (no surface term)."""
    fn = getattr(cond, "surface", None)
    if fn is None:
        raise ConfigurationError(
            f"{type(cond).__name__} boundary conditions are not realized by this solver")
    return fn(grid)


def _face_table(bc, d):
    """Condition of every face, indexed 2*axis + side, from a single
    condition or a ``{face: condition}`` dict ("all" fills the faces the
    dict leaves unnamed)."""
    nf = 2 * d
    if not isinstance(bc, dict):
        return [bc] * nf
    table = [None] * nf
    fallback = bc.get("all")
    for key, cond in bc.items():
        if key == "all":
            continue
        if key not in FACE_NAMES[:nf]:
            raise ConfigurationError(f"unknown face {key!r} for a {d}-d box")
        table[FACE_NAMES.index(key)] = cond
    if fallback is not None:
        table = [fallback if c is None else c for c in table]
    missing = [FACE_NAMES[i] for i, c in enumerate(table) if c is None]
    if missing:
        raise ConfigurationError(f"boundary conditions missing on faces {missing}")
    return table


def realize_bc(spec_or_bc, grid=None, mask=None):
    """BC -> ``[(axis, side, weight, rhs_value)]`` (the reference's
    ``realize_bc``, ``problem.py:237-300``: same rules and errors).

    Accepts the reference's ``ProblemSpec``-like object (attributes ``bc`` and
    ``grid``) or a condition / ``{face: condition}`` dict plus ``grid``.  A
    dict may use ``"all"`` and must cover every face of the box; unknown face
    names and non-positive gamma / epsilon raise ``ConfigurationError``.
    Mask domains (``mask=True``, or a spec whose ``domain`` is a
    :class:`.domain.MaskDomain`) take one global Neumann or DirichletPenalty
    condition and return at most one spec, whose weight applies to every
    exposed mask face.
    """
    from .domain import MaskDomain

    if grid is None:
        grid, bc = spec_or_bc.grid, spec_or_bc.bc
        if mask is None:
            mask = isinstance(getattr(spec_or_bc, "domain", None), MaskDomain)
    else:
        bc = spec_or_bc
    if mask:
        if isinstance(bc, dict):
            raise ConfigurationError("mask domains take a single global BC")
        if isinstance(bc, Robin):  # exposed faces take Neumann / DirichletPenalty only
            raise ConfigurationError("mask domains support Neumann or DirichletPenalty conditions only")
        term = _surface_of(bc, grid)
        return [] if term is None else [(0, 0, term[0], term[1])]
    specs = []
    for face, cond in enumerate(_face_table(bc, grid.dim)):
        term = _surface_of(cond, grid)
        if term is not None:
            specs.append((face // 2, face % 2, term[0], term[1]))
    return specs


__all__ = ["FACE_NAMES", "Robin", "Neumann", "DirichletPenalty", "realize_bc"]
