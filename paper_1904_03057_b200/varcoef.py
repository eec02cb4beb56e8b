"""Variable-coefficient operator on the B200.

For spline-valued diffusion D(x) and absorption mu(x) fields the reference
operator (``OnTheFlyOperator`` over ``build_system``,
``/root/reference/pkg/src/bspde/assembly.py:396-472``) is no longer a
Kronecker product: the stencil of node l is

    P[a, l] = sum_b D[l+b] (vol/hz^2 Tz'Ty Tx + vol/hy^2 Tz Ty' Tx + vol/hx^2 Tz Ty Tx')[a, b]
            + sum_b mu[l+b] vol (Tz Ty Tx)[a, b]

with per-axis trilinear tables T[a, b] = int D^d beta(x-a) D^d beta(x)
beta_np(x-b) (``kernels.py:158-173``; positional edge rows
``assembly.py:83-108``), computed exactly here (:func:`.gram.trilinear_tables`).
The sm_100a kernels (``csrc/stencil.cuh``) assemble all stencils once into HBM
and apply them as a streaming gather; Jacobi-PCG reuses the device-side
scalar state of the constant-coefficient solver.  3-D box domains with
natural faces; the stencil array costs (2p+1)^3 doubles per DoF (2.7 KB at
p = 3), so one B200 holds problems up to ~300^3.
"""

from __future__ import annotations

import ctypes as C
import time
import warnings
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import ConditioningWarning, ConfigurationError, ResourceError, ValidationError
from .gram import (basis_extension, edge_width, face_values, gram_factor, min_axis_length,
                   param_reach, trilinear_tables)


@dataclass
class VarSystemData:
    """Variable-coefficient system (cf. the reference SystemData)."""

    domain: object
    n_b: int
    n_p: int
    step: tuple
    cext: tuple
    ext: int
    ext_p: int
    dtype: np.dtype
    dfield: np.ndarray  # on the extended parameter grid
    mfield: np.ndarray
    tables: tuple  # (value, derivative) trilinear class tables
    scale_stiff: tuple
    scale_mass: float
    faces: tuple = ()
    mask: "MaskInfo" = None  # mask domains: node classes + exposed-face terms

    def face_rhs(self) -> np.ndarray:
        if self.mask is not None:
            raise ConfigurationError("mask surface RHS terms are assembled on the device "
                                     "(B200StencilOperator.surface_rhs_device)")
        from .system import face_rhs

        return face_rhs(self)

    @property
    def dim(self):
        return len(self.cext)

    @property
    def a_flat_size(self):
        return (2 * self.n_b + 1) ** self.dim

    def num_unknowns(self):
        return int(np.prod(self.cext))

    @property
    def vol(self):
        return self.scale_mass


@dataclass
class MaskInfo:
    """Mask-domain data (cf. the reference SystemData fields ``active``,
    ``bnode_rows``, assembly.py:538-560): node classes on the extended grid,
    the boundary rows and the global exposed-face surface term."""

    occupancy: np.ndarray   # bool cells
    node_class: np.ndarray  # uint8 extended nodes (domain.NODE_*)
    brows: np.ndarray       # int64 flat extended indices of boundary nodes
    surface_weight: float = 0.0
    surface_value: float = None  # None: no surface RHS term

    @property
    def active(self):
        return self.node_class != 0

    @property
    def dropped_unknowns(self):
        return int((self.node_class == 0).sum())


def _mask_info(domain, n_b, face_specs) -> MaskInfo:
    from .domain import NODE_BOUNDARY, node_classes

    cls = node_classes(domain, n_b)
    brows = np.flatnonzero(cls.ravel() == NODE_BOUNDARY).astype(np.int64)
    weight, value = 0.0, None
    specs = list(face_specs or ())
    if specs:
        # one global surface weight on every exposed mask face (assembly.py:657-665)
        for spec in specs:
            if len(spec) != 4:
                raise ValidationError(f"face spec {spec!r} is not (axis, side, weight, rhs_value)")
        weight = float(specs[0][2])
        value = None if specs[0][3] is None else float(specs[0][3])
        if not np.isfinite(weight):
            raise ValidationError(f"face weight {weight} is not finite")
    return MaskInfo(occupancy=np.ascontiguousarray(domain.occupancy(), dtype=bool),
                    node_class=cls, brows=brows, surface_weight=weight, surface_value=value)


def build_var_system(domain, n_b, n_p, dfield, mfield, face_specs, dtype) -> VarSystemData:
    from .domain import MaskDomain

    grid = domain.grid
    from .system import _face_terms

    is_mask = isinstance(domain, MaskDomain)
    faces = () if is_mask else tuple(_face_terms(face_specs, grid.dim))
    if not 1 <= int(n_b) <= 5:
        raise ValidationError(f"basis degree {n_b} not in 1..5")
    if not 0 <= int(n_p) <= 5:
        raise ValidationError(f"parameter degree {n_p} not in 0..5")
    if not is_mask:
        for n in grid.extents:
            if n - 1 < min_axis_length(n_b):
                raise ValidationError(f"axis with {n} nodes too short for degree {n_b} edge tables")
    ext, ext_p = basis_extension(n_b), basis_extension(n_p)
    pext = tuple(n + 2 * ext_p for n in grid.extents)
    fields = []
    for f, what in ((dfield, "diffusion"), (mfield, "absorption")):
        a = np.asarray(f, dtype=np.float64)
        if a.ndim == 0:
            a = np.full(pext, float(a))
        if a.shape != pext:
            raise ValidationError(f"{what} field {a.shape} != extended parameter grid {pext}")
        if not np.all(np.isfinite(a)):
            raise ValidationError(f"{what} field contains non-finite values")
        fields.append(np.ascontiguousarray(a))
    vol = float(np.prod(grid.step))
    tabs = (trilinear_tables(int(n_b), int(n_p), 0), trilinear_tables(int(n_b), int(n_p), 1))
    if is_mask:  # free-space (untruncated) rows; boundary rows come from the cells
        ew = edge_width(int(n_b))
        tabs = tuple(t[ew:ew + 1] for t in tabs)
    return VarSystemData(
        domain=domain, n_b=int(n_b), n_p=int(n_p), step=grid.step,
        cext=tuple(n + 2 * ext for n in grid.extents), ext=ext, ext_p=ext_p,
        dtype=np.dtype(dtype), dfield=fields[0], mfield=fields[1], tables=tabs,
        scale_stiff=tuple(vol / h ** 2 for h in grid.step), scale_mass=vol, faces=faces,
        mask=_mask_info(domain, int(n_b), face_specs) if is_mask else None)


def _var_strategy(data, lib, handle):
    """"otf" (matrix-free, csrc/otf.cuh) when the plan supports it and the
    system is not a mask (3-D box, no face terms, n_b = n_p <= 3), else
    "stencil" (assembled).  ``BSPDE_VAR_STRATEGY`` = stencil / otf forces one."""
    import os

    want = os.environ.get("BSPDE_VAR_STRATEGY", "auto")
    if want not in ("auto", "otf", "stencil"):
        raise ConfigurationError(f"BSPDE_VAR_STRATEGY must be auto, otf or stencil, got {want!r}")
    ok = data.mask is None and bool(lib.bspde_otf_supported(handle))
    if want == "otf" and not ok:
        raise ConfigurationError("the matrix-free operator needs a 3-D box without face terms "
                                 "and n_b = n_p <= 3")
    return "otf" if (ok and want != "stencil") else "stencil"


class B200StencilOperator:
    """Variable-coefficient operator on one B200 (strategy ``"b200"`` for
    variable coefficients); same protocol as the reference operators.

    Matrix-free (``kind == "otf"``: the reference's on-the-fly algorithm,
    sum-factorised, nothing stored) for 3-D boxes without face terms and
    n_b = n_p <= 3; otherwise the assembled stencil (``kind == "stencil"``,
    (2p+1)^3 doubles per DoF)."""

    strategy = "b200"

    def __init__(self, data: VarSystemData, workers=1, device=None):
        import torch

        from .device import require_cuda

        self.data = data
        self.workers = int(workers)
        self.device = require_cuda(device)
        self.lib = N.load()
        # 1-D / 2-D systems run as 3-D with unit leading axes (identity factor)
        self.lead = lead = 3 - data.dim
        d = N.StencilDesc()
        d.device = int(self.device.index)
        d.degree, d.param_degree = data.n_b, data.n_p
        d.nz, d.ny, d.nx = (1,) * lead + tuple(data.cext)
        d.pz, d.py, d.px = (1,) * lead + tuple(data.dfield.shape)
        d.ext, d.ext_p = data.ext, data.ext_p
        self._keep = [np.ascontiguousarray(t, dtype=np.float64) for t in data.tables]
        A, B = 2 * data.n_b + 1, 2 * param_reach(data.n_b, data.n_p) + 1
        unit_v = np.zeros((1, A, B))
        unit_v[0, data.n_b, B // 2] = 1.0
        unit = [unit_v, np.zeros((1, A, B))]
        self._keep += unit
        for a in range(3):
            real = a >= lead
            d.degenerate[a] = 0 if real else 1
            d.ew[a] = edge_width(data.n_b) if (real and data.mask is None) else 0
            for k in range(2):
                d.tables[a][k] = (self._keep[k] if real else unit[k]).ctypes.data_as(N._dptr)
            d.scale_stiff[a] = data.scale_stiff[a - lead] if real else 0.0
        d.scale_mass = data.scale_mass
        d.nfaces = len(data.faces)
        for f, ft in enumerate(data.faces):
            d.face_axis[f], d.face_side[f], d.face_weight[f] = ft.axis + lead, ft.side, ft.weight
        if data.faces:
            fv = np.array([float(v) for v in face_values(data.n_b)])
            gram = np.ascontiguousarray(gram_factor(data.n_b, data.domain.grid.extents[0],
                                                    "mass").table)
            self._keep += [fv, gram]
            d.face_values = fv.ctypes.data_as(N._dptr)
            d.mass_gram = gram.ctypes.data_as(N._dptr)
        for a in range(3):
            d.step[a] = data.step[a - lead] if a >= lead else 1.0
        h = C.c_void_p()
        N.check(self.lib.bspde_stencil_create(C.byref(d), C.byref(h)))
        self.handle = h
        self._scratch = None
        self._mask = None
        self._rows = None
        self.kind = _var_strategy(data, self.lib, h)
        if self.kind == "otf":
            # device parameter fields stay resident (read by every apply)
            self._df = torch.from_numpy(np.ascontiguousarray(data.dfield)).to(self.device)
            self._mf = torch.from_numpy(np.ascontiguousarray(data.mfield)).to(self.device)
            self._diag = torch.empty(tuple(data.cext), dtype=torch.float64, device=self.device)
            self.P = None
            N.check(self.lib.bspde_otf_prepare(h, N.ptr(self._df), N.ptr(self._mf),
                                               N.ptr(self._diag), N.stream_handle()))
            return
        if data.mask is not None:
            # compact: only the active rows are stored (inactive rows are zero;
            # the leg of the paper has ~21% active nodes)
            rows = np.flatnonzero(data.mask.node_class.ravel() != 0).astype(np.int64)
            self._rows = torch.from_numpy(rows).to(self.device)
            self._rows_host = rows
            N.check(self.lib.bspde_stencil_set_rows(h, N.ptr(self._rows), int(len(rows))))
        n_entries = int(self.lib.bspde_stencil_entries(h))
        free, _ = torch.cuda.mem_get_info(self.device)
        if n_entries * 8 > 0.9 * free:
            raise ResourceError(f"stencil array needs {n_entries * 8 / 1e9:.1f} GB "
                                f"(free {free / 1e9:.1f} GB)")
        self.P = torch.empty(n_entries, dtype=torch.float64, device=self.device)
        df = torch.from_numpy(np.ascontiguousarray(data.dfield)).to(self.device)
        mf = torch.from_numpy(np.ascontiguousarray(data.mfield)).to(self.device)
        N.check(self.lib.bspde_stencil_assemble(h, N.ptr(df), N.ptr(mf), N.ptr(self.P),
                                                N.stream_handle()))
        if data.mask is not None:
            self._mask = self._mask_desc(data.mask)
            N.check(self.lib.bspde_stencil_mask_patch(h, C.byref(self._mask[0]), N.ptr(df),
                                                      N.ptr(mf), N.ptr(self.P),
                                                      N.stream_handle()))
        self._scratch = None

    def _mask_desc(self, m):
        """Upload the mask tables; returns (MaskDesc, keep-alive tensors)."""
        import torch

        from .gram import (cell_bilinear, cell_offsets, cell_single, cell_trilinear,
                           face_normal_values, first_clean_position)

        nb, npar, dev = self.data.n_b, self.data.n_p, self.device

        def up(a, dt=torch.float64):
            return torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)

        brows_k = (np.searchsorted(self._rows_host, m.brows).astype(np.int64)
                   if self._rows is not None and len(m.brows) else np.zeros(1, np.int64))
        keep = dict(
            occ=up(m.occupancy.astype(np.uint8), torch.uint8),
            cls=up(m.node_class, torch.uint8),
            brows=up(m.brows if len(m.brows) else np.zeros(1, np.int64), torch.int64),
            brows_k=up(brows_k, torch.int64),
            tri=up(np.stack([cell_trilinear(nb, npar, 0), cell_trilinear(nb, npar, 1)])),
            bil=up(cell_bilinear(nb, nb)), single=up(cell_single(nb)),
            fv=up(face_normal_values(nb)))
        d = N.MaskDesc()
        d.occupancy, d.node_class, d.brows = (N.ptr(keep["occ"]), N.ptr(keep["cls"]),
                                              N.ptr(keep["brows"]))
        cells = (1,) * self.lead + tuple(m.occupancy.shape)
        for a in range(3):
            d.cells[a] = cells[a]
            d.degenerate[a] = 1 if a < self.lead else 0
        d.nbrows = len(m.brows)
        d.brows_k = N.ptr(keep["brows_k"]) if self._rows is not None else None
        (jlo, jhi), (blo, bhi) = cell_offsets(nb), cell_offsets(npar)
        d.jlo, d.nj, d.blo, d.nbp = jlo, jhi - jlo + 1, blo, bhi - blo + 1
        d.cell_tri, d.cell_bil, d.cell_single, d.face_vals = (
            N.ptr(keep["tri"]), N.ptr(keep["bil"]), N.ptr(keep["single"]), N.ptr(keep["fv"]))
        d.fc = first_clean_position(nb)
        d.has_surface = int(m.surface_weight != 0.0)
        d.surface_weight = float(m.surface_weight)
        return d, keep

    def surface_rhs_device(self, out, weight=None, value=None, stream=None):
        """out += the exposed-face surface RHS of a mask system
        (``surface_rhs_entries``, assembly.py:728-737); ``weight``/``value``
        default to the system's own."""
        m = self.data.mask
        if m is None:
            raise ConfigurationError("surface_rhs_device is for mask systems")
        d = N.MaskDesc.from_buffer_copy(self._mask[0])
        w = m.surface_weight if weight is None else float(weight)
        v = m.surface_value if value is None else float(value)
        if v is None or w == 0.0:
            return out
        d.has_surface, d.surface_weight = 1, w
        N.check(self.lib.bspde_stencil_mask_surface_rhs(self.handle, C.byref(d), float(v),
                                                        N.ptr(out), N.stream_handle(stream)))
        return out

    def __del__(self):
        try:
            if getattr(self, "handle", None) and self.handle.value:
                self.lib.bspde_stencil_destroy(self.handle)
                self.handle = C.c_void_p()
        except Exception:  # pragma: no cover - interpreter shutdown
            pass

    @property
    def shape(self):
        return self.data.cext

    @property
    def dtype(self):
        return self.data.dtype

    def launches(self) -> int:
        return int(self.lib.bspde_stencil_launch_count(self.handle))

    def _dev(self, arr, what):
        import torch

        a = np.asarray(arr, dtype=np.float64)
        if a.shape != self.data.cext:
            raise ValidationError(f"{what} {a.shape} != extended extents {self.data.cext}")
        if not np.all(np.isfinite(a)):
            raise ValidationError(f"{what} contains non-finite values")
        return torch.from_numpy(np.ascontiguousarray(a)).to(self.device)

    def apply_device(self, c, out, stream=None):
        if self.kind == "otf":
            N.check(self.lib.bspde_otf_apply(self.handle, N.ptr(c), N.ptr(out),
                                             N.stream_handle(stream)))
            return out
        if self._rows is not None:
            out.zero_()  # compact plans write the active rows only (inactive rows are zero)
        N.check(self.lib.bspde_stencil_apply(self.handle, N.ptr(self.P), N.ptr(c), N.ptr(out),
                                             N.stream_handle(stream)))
        return out

    def apply(self, c, out=None):
        import torch

        cd = self._dev(c, "input coefficients")
        od = torch.empty_like(cd)
        self.apply_device(cd, od)
        t = od.cpu().numpy().astype(self.data.dtype, copy=False)
        if out is not None:
            out[...] = t
            return out
        return t

    def jacobi_diagonal(self):
        import torch

        if self.kind == "otf":
            diag = self._diag.cpu().numpy().copy()
        else:
            od = torch.empty(self.data.cext, dtype=torch.float64, device=self.device)
            N.check(self.lib.bspde_stencil_diagonal(self.handle, N.ptr(self.P), N.ptr(od),
                                                    N.stream_handle()))
            diag = od.cpu().numpy()
        if self.data.mask is not None:  # inactive unknowns get 1 (operator.py:156-170)
            diag[self.data.mask.node_class == 0] = 1.0
        bad = diag <= 0
        if np.any(bad):
            idx = np.argwhere(bad)[0]
            warnings.warn(
                f"non-positive operator diagonal at node {tuple(int(i) for i in idx)}",
                ConditioningWarning)
        return diag.astype(self.data.dtype, copy=False)

    def flop_byte_report(self, seconds=0.0):
        from .operator import OpStats

        n = self.data.num_unknowns()
        A = 2 * self.data.n_b + 1
        if self.kind == "otf":
            B = 2 * param_reach(self.data.n_b, self.data.n_p) + 1
            # per output: y-stage (3 B FMAs per (ay, ax)) + scatter (2 B per
            # (ay, ax)); x-stage 3 A B, C0 2 A B per staged position
            fmas = A * A * 5 * B + 5 * A * B
            return OpStats(flops=int(2 * fmas * n), bytes_read=int(n * 8 * 3),
                           bytes_written=int(n * 8), seconds=seconds)
        a3 = A ** 3
        return OpStats(flops=int(2 * a3 * n), bytes_read=int(n * 8 * (a3 + 1)),
                       bytes_written=int(n * 8), seconds=seconds)

    def pcg(self, rhs, config, x0=None):
        """Jacobi-PCG (reference recurrence) on the device: (x, SolveReport)."""
        import torch

        b = self._dev(rhs, "rhs")
        x = self._dev(x0, "x0") if x0 is not None else torch.zeros_like(b)
        report = self.pcg_device(b, x, config, has_x0=x0 is not None)
        return x.cpu().numpy(), report

    def pcg_device(self, b, x, config, has_x0=True, stream=None):
        """Solve on dense device tensors (cext shape); x holds x0 on entry
        (if ``has_x0``) and the solution on return.  Returns SolveReport."""
        import torch

        from .solver import report_from

        t0 = time.perf_counter()
        r, p, ap = torch.empty_like(b), torch.empty_like(b), torch.empty_like(b)
        if self._scratch is None:
            n = int(self.lib.bspde_scratch_bytes(None))
            self._scratch = torch.zeros(n, dtype=torch.uint8, device=self.device)
        hist = torch.zeros(config.max_iter + 1, dtype=torch.float64, device=self.device)
        cfg = N.CgConfig(float(config.tol), int(config.max_iter), int(bool(config.record_history)),
                         int(bool(has_x0)), int(config.poll_every))
        rep = N.CgReport()
        precond = 1 if config.precond == "jacobi" else 0
        if self.kind == "otf":
            N.check(self.lib.bspde_otf_pcg(self.handle, N.ptr(b), N.ptr(x), N.ptr(r), N.ptr(p),
                                           N.ptr(ap), N.ptr(self._scratch), N.ptr(hist),
                                           C.byref(cfg), C.byref(rep), precond,
                                           N.stream_handle(stream)))
            return report_from(rep, config, time.perf_counter() - t0, hist)
        N.check(self.lib.bspde_stencil_pcg(self.handle, N.ptr(self.P), N.ptr(b), N.ptr(x), N.ptr(r),
                                           N.ptr(p), N.ptr(ap), N.ptr(self._scratch), N.ptr(hist),
                                           C.byref(cfg), C.byref(rep), precond,
                                           N.stream_handle(stream)))
        return report_from(rep, config, time.perf_counter() - t0, hist)


__all__ = ["VarSystemData", "build_var_system", "B200StencilOperator", "param_reach"]
