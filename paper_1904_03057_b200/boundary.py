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


@dataclass(frozen=True)
class Neumann:
    """Homogeneous natural condition: no surface term."""


@dataclass(frozen=True)
class DirichletPenalty:
    """Dirichlet value ``value`` enforced by a penalty term of weight
    ``1/epsilon`` (``epsilon=None``: ``1e-4 * min(h)``)."""

    value: float = 0.0
    epsilon: float = None


def _face_key(axis, side):
    return FACE_NAMES[2 * axis + side]


def realize_bc(spec_or_bc, grid=None, mask=None):
    """BC -> ``[(axis, side, weight, rhs_value)]`` (``problem.py:237-300``).

    Accepts the reference's ``ProblemSpec``-like object (attributes ``bc`` and
    ``grid``) or a condition / ``{face: condition}`` dict plus ``grid``.
    Same rules as the reference: a dict may use ``"all"`` and must cover every
    face of the box; unknown face names and non-positive gamma / epsilon raise
    ``ConfigurationError``.  Mask domains (``mask=True``, or a spec whose
    ``domain`` is a :class:`.domain.MaskDomain`) take one global Neumann or
    DirichletPenalty condition and return at most one spec, whose weight
    applies to every exposed mask face.
    """
    from .domain import MaskDomain

    if grid is None:
        grid = spec_or_bc.grid
        bc = spec_or_bc.bc
        if mask is None:
            mask = isinstance(getattr(spec_or_bc, "domain", None), MaskDomain)
    else:
        bc = spec_or_bc
    d = grid.dim
    if isinstance(bc, dict) and mask:
        raise ConfigurationError("mask domains take a single global BC")
    if isinstance(bc, dict):
        per_face = {}
        for key, val in bc.items():
            if key == "all":
                for ax in range(d):
                    for s in (0, 1):
                        per_face.setdefault(_face_key(ax, s), val)
            elif key in FACE_NAMES[: 2 * d]:
                per_face[key] = val
            else:
                raise ConfigurationError(f"unknown face {key!r} for a {d}-d box")
        missing = [f for f in FACE_NAMES[: 2 * d] if f not in per_face]
        if missing:
            raise ConfigurationError(f"boundary conditions missing on faces {missing}")
    else:
        per_face = {f: bc for f in FACE_NAMES[: 2 * d]}

    def weight_of(cond):
        if isinstance(cond, Neumann):
            return None
        if isinstance(cond, Robin):
            if cond.gamma <= 0:
                raise ConfigurationError(f"Robin gamma must be positive, got {cond.gamma}")
            return (1.0 / (2.0 * cond.gamma), None)
        if isinstance(cond, DirichletPenalty):
            eps = cond.epsilon if cond.epsilon is not None else 1e-4 * min(grid.step)
            if eps <= 0:
                raise ConfigurationError(f"penalty epsilon must be positive, got {eps}")
            return (1.0 / eps, cond.value)
        raise ConfigurationError(
            f"{type(cond).__name__} boundary conditions are not realized by this solver")

    if mask:
        if isinstance(bc, Robin):
            raise ConfigurationError("mask domains support Neumann or DirichletPenalty conditions only")
        w = weight_of(bc)
        return [] if w is None else [(0, 0, w[0], w[1])]

    specs = []
    for ax in range(d):
        for s in (0, 1):
            w = weight_of(per_face[_face_key(ax, s)])
            if w is not None:
                specs.append((ax, s, w[0], w[1]))
    return specs


__all__ = ["FACE_NAMES", "Robin", "Neumann", "DirichletPenalty", "realize_bc"]
