"""Steady problem pipeline with coarse-grid initialisation (SURVEY.md §8(f)
item 4: the CT-leg experiment).

Mirrors the reference's ``ProblemSpec`` / ``transform_inputs`` /
``assemble_system`` / ``coarse_initialize`` / ``solve_problem``
(``/root/reference/pkg/src/bspde/problem.py:66-127, 197-217, 316-327,
374-482``) on the B200 path: field transforms, operator assembly (box:
Kronecker kernels; mask / variable fields: assembled stencil), RHS, the
coarse solve and the fine solve all run on the GPU; the host only
classifies mask nodes and builds small index/weight tables.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass

import numpy as np

from .boundary import Neumann, realize_bc
from .domain import BoxDomain, Grid, MaskDomain
from .errors import ConfigurationError, ValidationError
from .gram import basis_extension, min_axis_length
from .solver import SolveConfig, SolveReport, pcg
from .transform import (direct_transform, indirect_transform_lattice, sample_field,
                        sample_solution, transform_field)


@dataclass
class ProblemSpec:
    """Domain, fields (scalar, node samples or callable), degrees, BCs
    (``problem.py:66-116``).  The B200 path computes in float64 with
    ``source_degree == basis_degree``; both prefilters are realized."""

    domain: object
    basis_degree: int
    diffusion: object = 1.0
    absorption: object = 0.0
    source: object = 0.0
    bc: object = None
    param_degree: int = None
    source_degree: int = None
    precision: str = "f64"
    prefilter: str = "interpolation"

    def __post_init__(self):
        if self.param_degree is None:
            self.param_degree = self.basis_degree
        if self.source_degree is None:
            self.source_degree = self.basis_degree
        if self.bc is None:
            self.bc = Neumann()
        if self.precision not in ("f64", "f32"):
            raise ValidationError(f"precision must be f64/f32, got {self.precision!r}")
        if self.prefilter not in ("interpolation", "l2"):
            raise ValidationError(f"prefilter must be interpolation/l2, got {self.prefilter!r}")
        for name, n in (("basis", self.basis_degree), ("param", self.param_degree),
                        ("source", self.source_degree)):
            if not 0 <= n <= 5:
                raise ValidationError(f"{name} degree {n} not in 0..5")
        need = min_axis_length(self.basis_degree) + 1
        if any(n < need for n in self.grid.extents):
            raise ValidationError(
                f"extents {self.grid.extents} too small for degree {self.basis_degree} "
                f"(need >= {need})")
        if self.precision != "f64":
            raise ConfigurationError("the b200 path computes in float64 (precision='f64')")

    @property
    def dtype(self):
        return np.float64

    @property
    def grid(self) -> Grid:
        return self.domain.grid

    def default_epsilon(self):
        return 1e-4 * min(self.grid.step)


@dataclass
class FieldSet:
    d_coeffs: np.ndarray
    m_coeffs: np.ndarray
    q_coeffs: np.ndarray
    clamped_d: int = 0
    clamped_m: int = 0


@dataclass
class AssembledSystem:
    data: object
    operator: object
    rhs: np.ndarray
    fields: FieldSet
    face_specs: list


@dataclass
class Solution:
    samples: np.ndarray
    coeffs: np.ndarray
    report: SolveReport
    spec: ProblemSpec
    system: AssembledSystem
    coarse_info: dict = None


def transform_inputs(spec: ProblemSpec) -> FieldSet:
    """D, mu (degree n_p) and q (degree n_s) to coefficients on the GPU;
    negative D / mu overshoots are clamped with a warning (``problem.py:197-217``)."""
    grid = spec.grid
    pf = spec.prefilter
    d = transform_field(spec.diffusion, grid, spec.param_degree, prefilter=pf)
    m = transform_field(spec.absorption, grid, spec.param_degree, prefilter=pf)
    q = transform_field(spec.source, grid, spec.source_degree, prefilter=pf)
    cd, cm = int(np.sum(d < 0)), int(np.sum(m < 0))
    if cd:
        warnings.warn(f"clamped {cd} negative diffusion coefficients after prefiltering")
        d = np.maximum(d, 0.0)
    if cm:
        warnings.warn(f"clamped {cm} negative absorption coefficients after prefiltering")
        m = np.maximum(m, 0.0)
    return FieldSet(d, m, q, cd, cm)


def assemble_system(spec: ProblemSpec, strategy="b200", workers=1) -> AssembledSystem:
    """Transform -> build_system -> make_operator -> assembled_rhs
    (``problem.py:316-327``)."""
    from .operator import assembled_rhs, make_operator
    from .system import build_system

    fields = transform_inputs(spec)
    specs = realize_bc(spec)
    data = build_system(spec.domain, spec.basis_degree, spec.param_degree, fields.d_coeffs,
                        fields.m_coeffs, specs)
    op = make_operator(data, strategy, workers)
    rhs = assembled_rhs(data, spec.source_degree, fields.q_coeffs, workers)
    return AssembledSystem(data, op, rhs, fields, specs)


def _coarsen_mask(mask, cgrid: Grid) -> np.ndarray:
    """Majority vote of the fine cells under each coarse cell; the cell
    ranges are ``floor(i F / C) .. max(ceil((i+1) F / C), 1)`` per axis
    (``problem.py:446-462``), summed through a summed-area table."""
    fine, coarse = mask.shape, cgrid.cell_extents
    sat = np.pad(np.asarray(mask, dtype=np.int64), [(1, 0)] * mask.ndim)
    for ax in range(mask.ndim):
        sat = np.cumsum(sat, axis=ax)
    bounds = []
    for ax in range(mask.ndim):
        i = np.arange(coarse[ax])
        lo = np.floor(i * fine[ax] / coarse[ax]).astype(np.int64)
        hi = np.maximum(np.ceil((i + 1) * fine[ax] / coarse[ax]).astype(np.int64), 1)
        bounds.append((lo, hi))
    total = np.zeros(coarse, dtype=np.int64)
    count = np.ones(coarse, dtype=np.int64)
    for corner in np.ndindex(*(2,) * mask.ndim):
        idx = np.ix_(*[bounds[ax][1] if corner[ax] else bounds[ax][0] for ax in range(mask.ndim)])
        sign = (-1) ** (mask.ndim - sum(corner))
        total += sign * sat[idx]
    for ax in range(mask.ndim):
        shape = [1] * mask.ndim
        shape[ax] = coarse[ax]
        count = count * (bounds[ax][1] - bounds[ax][0]).reshape(shape)
    out = 2 * total >= count
    if not out.any():
        out.flat[0] = True  # the reference's fallback (argmax of a scalar mean)
    return out


def coarse_initialize(spec: ProblemSpec, factor, config: SolveConfig = None, strategy="b200",
                      workers=1):
    """Initial fine-grid coefficients from a factor-reduced solve
    (``problem.py:374-443``): fields restricted by spline resampling, mask by
    majority vote, coarse solve, prolongation by spline evaluation at the
    fine nodes + direct transform + reflect padding.  Returns (x0, info)."""
    if factor < 2:
        raise ValidationError(f"coarse factor must be >= 2, got {factor}")
    grid = spec.grid
    n_b = spec.basis_degree
    min_nodes = min_axis_length(n_b) + 1
    cN = tuple(max(int(math.ceil(n / factor)), min_nodes) for n in grid.extents)
    ch = tuple((n - 1) * h / (cn - 1) for n, h, cn in zip(grid.extents, grid.step, cN))
    cgrid = Grid(cN, ch, grid.origin)
    info = {"coarse_extents": cN, "coarse_step": ch,
            "divisible": all(n % factor == 0 for n in grid.extents)}
    fine_pts = [grid.node_coordinates(ax) - grid.origin[ax] for ax in range(grid.dim)]
    coarse_pts = [cgrid.node_coordinates(ax) - grid.origin[ax] for ax in range(grid.dim)]

    def restrict(value, degree):
        samples = sample_field(value, grid)
        if samples is None:
            return float(value)
        if callable(value):
            return sample_field(value, cgrid)
        coeffs = direct_transform(samples, degree)
        return indirect_transform_lattice(coeffs, degree, grid.step, coarse_pts)

    if isinstance(spec.domain, MaskDomain):
        cdom = MaskDomain(cgrid, _coarsen_mask(spec.domain.mask, cgrid))
    else:
        cdom = BoxDomain(cgrid)
    cspec = ProblemSpec(domain=cdom, basis_degree=n_b,
                        diffusion=restrict(spec.diffusion, spec.param_degree),
                        absorption=restrict(spec.absorption, spec.param_degree),
                        source=restrict(spec.source, spec.source_degree), bc=spec.bc,
                        param_degree=spec.param_degree, source_degree=spec.source_degree,
                        precision=spec.precision)
    csol = solve_problem(cspec, config or SolveConfig(tol=1e-8, max_iter=2000), strategy,
                         workers)
    info["coarse_iterations"] = csol.report.iterations
    ext = basis_extension(n_b)
    fine_samples = indirect_transform_lattice(csol.coeffs, n_b, ch, fine_pts,
                                              first_index=(-ext,) * grid.dim)
    x0 = direct_transform(fine_samples, n_b)
    if ext > 0:
        x0 = np.pad(x0, ext, mode="reflect")
    return x0, info


def solve_problem(spec: ProblemSpec, config: SolveConfig = None, strategy="b200",
                  workers=1) -> Solution:
    """Transform -> assemble -> (coarse init) -> pcg -> node samples
    (``problem.py:465-482``)."""
    config = config or SolveConfig()
    system = assemble_system(spec, strategy, workers)
    active = system.data.mask.active if getattr(system.data, "mask", None) is not None else None
    x0, coarse_info = None, None
    if config.coarse_init_factor and config.coarse_init_factor >= 2:
        x0, coarse_info = coarse_initialize(spec, config.coarse_init_factor, strategy=strategy,
                                            workers=workers)
        if active is not None:
            x0[~active] = 0.0
    coeffs, report = pcg(system.operator, system.rhs, config, x0=x0)
    if active is not None:
        coeffs[~active] = 0.0
    samples = sample_solution(coeffs, spec.grid, spec.basis_degree)
    return Solution(samples=samples, coeffs=coeffs, report=report, spec=spec, system=system,
                    coarse_info=coarse_info)


__all__ = ["ProblemSpec", "FieldSet", "AssembledSystem", "Solution", "transform_inputs",
           "assemble_system", "coarse_initialize", "solve_problem"]
