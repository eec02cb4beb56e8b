"""System assembly for the B200 strategy (host setup, runs once).

Mirrors the reference's ``build_system`` signature
(``/root/reference/pkg/src/bspde/assembly.py:396-457``) for the operator the
hot path realizes: constant diffusion ``D`` and absorption ``mu`` on a box
domain with natural (Neumann) faces.  With constant fields the reference's
per-node stencil collapses (partition of unity over the parameter splines)
into the Kronecker sum documented in :mod:`.gram`; this module computes the
1-D factors, the axis scales and the Jacobi diagonal by class, i.e. all the
data the sm_100a kernels need.  Everything is O(p) host work.

Reference dims ``d < 3`` are right-aligned onto the kernel's (z, y, x) axes;
padded axes are degenerate (length 1, mass factor 1, no stiffness term).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .domain import BoxDomain, Grid
from .errors import ConfigurationError, ValidationError
from .gram import (GramFactor, basis_extension, degenerate_factor, edge_width, face_table,
                   face_vector, gram_factor, min_axis_length, surface_single_vector)


def _constant_value(f, what):
    """The field's constant value, or None for a variable field."""
    arr = np.asarray(f, dtype=np.float64)
    if arr.size == 0:
        raise ValidationError(f"{what} field is empty")
    if not np.all(np.isfinite(arr)):
        raise ValidationError(f"{what} field contains non-finite values")
    v = float(arr.flat[0])
    if arr.size > 1 and not np.all(arr == v):
        return None
    return v


@dataclass(frozen=True)
class FaceTerm:
    """One box-face surface term (reference ``FaceTerm``, assembly.py:183-198).

    ``axis``/``side`` use reference axis order; the operator term is
    ``weight * (v v^T)_axis (x) (h M)_other axes`` with ``v`` the face point
    values, the right-hand side ``rhs_weight * v (x) (h s)_other axes``.
    """

    axis: int
    side: int
    weight: float
    rhs_weight: float


@dataclass
class SystemData:
    """What the B200 operator, RHS and solver share (cf. reference SystemData)."""

    domain: object
    n_b: int
    n_p: int
    step: tuple
    cext: tuple
    ext: int
    dtype: np.dtype
    diffusion: float
    absorption: float
    faces: list = field(default_factory=list)
    # kernel-space (z, y, x) data
    dims3: tuple = None
    mass: tuple = None
    stiff: tuple = None
    c_mass: float = 0.0
    c_stiff: tuple = (0.0, 0.0, 0.0)
    vol: float = 1.0

    @property
    def dim(self):
        return len(self.cext)

    @property
    def a_flat_size(self):
        return (2 * self.n_b + 1) ** self.dim

    def num_unknowns(self):
        return int(np.prod(self.cext))

    @property
    def ew3(self):
        return tuple(f.ew for f in self.mass)

    def face_rhs(self) -> np.ndarray:
        return face_rhs(self)

    # -- Jacobi diagonal by class (operator.py:190-209 for constant fields) --
    def diag_table(self) -> np.ndarray:
        mz, my, mx = (f.diagonal_by_class() for f in self.mass)
        kz, ky, kx = (f.diagonal_by_class() for f in self.stiff)
        Z, Y, X = np.ix_(np.arange(len(mz)), np.arange(len(my)), np.arange(len(mx)))
        cz, cy, cx = self.c_stiff
        d = cz * kz[Z] * my[Y] * mx[X]
        d = d + cy * mz[Z] * ky[Y] * mx[X]
        d = d + cx * mz[Z] * my[Y] * kx[X]
        d = d + self.c_mass * mz[Z] * my[Y] * mx[X]
        return np.ascontiguousarray(d, dtype=np.float64)

    def inv_diag_table(self, precond="jacobi") -> np.ndarray:
        d = self.diag_table()
        if precond == "none":
            return np.ones_like(d)
        with np.errstate(divide="ignore"):
            return np.where(d != 0.0, 1.0 / d, 1.0)

    def class_index(self, axis3, n=None) -> np.ndarray:
        f = self.mass[axis3]
        return f.row_class(np.arange(f.n if n is None else n))

    def expand_table(self, table) -> np.ndarray:
        """Class table (z,y,x) -> full array on the reference extents."""
        cz, cy, cx = (self.class_index(a) for a in range(3))
        full = table[np.ix_(cz, cy, cx)]
        return full.reshape(self.cext)


def face_rhs(data) -> np.ndarray:
    """Penalty right-hand-side surface additions (reference ``face_rhs``,
    assembly.py:488-501): a rank-1 tensor per face with a value."""
    grid = data.domain.grid
    out = np.zeros(data.cext)
    for ft in data.faces:
        if ft.rhs_weight == 0.0:
            continue
        vecs = []
        for ax in range(grid.dim):
            n = grid.extents[ax]
            if ax == ft.axis:
                vecs.append(face_vector(data.n_b, n, ft.side))
            else:
                vecs.append(surface_single_vector(data.n_b, n) * grid.step[ax])
        t = vecs[0]
        for v in vecs[1:]:
            t = np.multiply.outer(t, v)
        out += ft.rhs_weight * t
    return out


def _as3(seq, pad):
    seq = tuple(seq)
    return (pad,) * (3 - len(seq)) + seq


def build_system(domain, n_b, n_p, dcoef_ext, mcoef_ext, face_specs=(), dtype=np.float64,
                 block_bytes=4 << 20) -> SystemData:
    """Reference-compatible constructor (assembly.py:396-457) for the b200 path.

    ``dcoef_ext``/``mcoef_ext`` are the (constant) diffusion and absorption
    coefficient fields on the extended parameter grid, or scalars.
    ``face_specs``: ``(axis, side, weight, rhs_value_or_None)`` box-face
    surface terms (Robin / DirichletPenalty, see :func:`.boundary.realize_bc`).
    """
    from .domain import MaskDomain

    if not isinstance(domain, (BoxDomain, MaskDomain)):
        raise ConfigurationError(f"unsupported domain type {type(domain).__name__}")
    if not 1 <= int(n_b) <= 5:
        raise ValidationError(f"basis degree {n_b} not in 1..5")
    D = _constant_value(dcoef_ext, "diffusion")
    mu = _constant_value(mcoef_ext, "absorption")
    if D is None or mu is None or isinstance(domain, MaskDomain):
        # spline-valued fields or a mask domain: the assembled-stencil
        # operator (varcoef.py; mask rows from the occupied cells)
        from .varcoef import build_var_system

        return build_var_system(domain, int(n_b), int(n_p), dcoef_ext, mcoef_ext, face_specs,
                                dtype)
    return _make(domain, int(n_b), int(n_p), D, mu, np.dtype(dtype), face_specs)


def _face_terms(face_specs, dim):
    out = []
    for spec in face_specs or ():
        try:
            axis, side, weight, rhs_value = spec
        except (TypeError, ValueError):
            raise ValidationError(f"face spec {spec!r} is not (axis, side, weight, rhs_value)")
        if not (isinstance(axis, (int, np.integer)) and 0 <= axis < dim):
            raise ValidationError(f"face axis {axis!r} not in 0..{dim - 1}")
        if side not in (0, 1):
            raise ValidationError(f"face side {side!r} not 0 or 1")
        weight = float(weight)
        if not np.isfinite(weight):
            raise ValidationError(f"face weight {weight} is not finite")
        rhs_w = 0.0 if rhs_value is None else float(rhs_value) * weight
        out.append(FaceTerm(int(axis), int(side), weight, rhs_w))
    return out


def _make(domain, p, n_p, D, mu, dtype, face_specs=()) -> SystemData:
    grid = domain.grid
    ext = basis_extension(p)
    for n in grid.extents:
        if n - 1 < min_axis_length(p):
            raise ValidationError(
                f"axis with {n} nodes too short for degree {p} edge tables")
    cext = tuple(n + 2 * ext for n in grid.extents)
    vol = float(np.prod(grid.step))
    mass = [gram_factor(p, n, "mass") for n in grid.extents]
    stiff = [gram_factor(p, n, "stiff") for n in grid.extents]
    cst = [vol * D / h ** 2 for h in grid.step]
    faces = _face_terms(face_specs, grid.dim)
    # A face on axis a adds weight * (v v^T)_a (x) (h M)_others =
    # c_a * [(weight * h_a / D) * (v v^T)]_a (x) M_others to the c_a K_a term
    # (c_a = vol * D / h_a^2): the normal factor folds into the edge-row
    # classes of K_a; interior taps are unchanged.
    for ft in faces:
        if not D > 0.0:
            raise ConfigurationError(
                "the b200 strategy realizes face terms inside the diffusion factors; "
                "they need a positive diffusion coefficient")
        h = grid.step[ft.axis]
        stiff[ft.axis] = stiff[ft.axis].plus((ft.weight * h / D) * face_table(p, ft.side))
    pad = 3 - grid.dim
    mass3 = tuple([degenerate_factor(p, "mass")] * pad + mass)
    stiff3 = tuple([degenerate_factor(p, "stiff")] * pad + stiff)
    c_stiff3 = tuple([0.0] * pad + cst)
    return SystemData(
        domain=domain, n_b=p, n_p=n_p, step=grid.step, cext=cext, ext=ext, dtype=dtype,
        diffusion=D, absorption=mu, faces=faces, dims3=_as3(cext, 1), mass=mass3,
        stiff=stiff3, c_mass=vol * mu, c_stiff=c_stiff3, vol=vol)


def heat_system(grid: Grid, degree: int, dt: float, conductivity: float = 1.0,
                face_specs=()) -> SystemData:
    """``A = M + dt*(kappa*K + W)`` of one implicit-Euler step (D = dt*kappa,
    mu = 1).  ``face_specs`` are the steady surface terms ``W`` (e.g. from
    :func:`.boundary.realize_bc`); their weights are scaled by ``dt`` here,
    so ``face_rhs()`` is ``dt`` times the steady penalty right-hand side."""
    if not dt > 0:
        raise ValidationError(f"dt must be positive, got {dt}")
    scaled = [(a, s, float(w) * float(dt), v) for a, s, w, v in (face_specs or ())]
    return _make(BoxDomain(grid), int(degree), int(degree), float(dt) * float(conductivity),
                 1.0, np.dtype(np.float64), scaled)


def mass_system(grid: Grid, degree: int) -> SystemData:
    """The mass operator ``M`` (D = 0, mu = 1)."""
    return _make(BoxDomain(grid), int(degree), int(degree), 0.0, 1.0, np.dtype(np.float64))


__all__ = ["SystemData", "FaceTerm", "build_system", "heat_system", "mass_system",
           "edge_width", "GramFactor"]
