"""The ``b200`` operator strategy: drop-in for the reference operator protocol.

``make_operator(data, "b200")`` returns an object with the same protocol as
the reference's ``OnTheFlyOperator`` (``/root/reference/pkg/src/bspde/
operator.py:112-251``): ``apply(c, out=None)``, ``jacobi_diagonal()``,
``flop_byte_report(seconds)``, ``shape``, ``dtype``, ``data``, ``workers``
and the class attribute ``strategy``.  ``apply`` runs the sm_100a streaming
kernel (``sep_kernel<P, M_APPLY>``) through the C ABI; host arrays are
copied to/from the device layout around it.  Device-resident callers use
``apply_device`` with ghosted-slab torch tensors and no copies.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np

from .device import NativePlan, SlabLayout, check_host_field, require_cuda
from .errors import ConditioningWarning, ConfigurationError, ValidationError
from .system import SystemData


@dataclass
class OpStats:
    """Operation/traffic model of one apply (cf. operator.py:32-43)."""

    flops: int
    bytes_read: int
    bytes_written: int
    seconds: float = 0.0

    @property
    def gflops(self):
        return self.flops / self.seconds / 1e9 if self.seconds > 0 else 0.0

    @property
    def gbytes_per_s(self):
        b = self.bytes_read + self.bytes_written
        return b / self.seconds / 1e9 if self.seconds > 0 else 0.0


def apply_flops_per_dof(p: int) -> int:
    """7 banded filters of width 2p+1 (x: Mx,Kx; y: My twice, Ky; z: Mz,Kz)
    as FMAs, plus the per-point axis combination."""
    return 2 * 7 * (2 * p + 1) + 4


class B200Operator:
    """Matrix-free separable operator on one B200 (strategy ``"b200"``)."""

    strategy = "b200"

    def __init__(self, data: SystemData, workers=1, device=None):
        if not isinstance(data, SystemData):
            raise ConfigurationError(
                "make_operator(..., 'b200') takes SystemData from "
                "paper_1904_03057_b200.build_system / heat_system")
        self.data = data
        self.workers = int(workers)  # kept for API compatibility; the GPU ignores it
        self.device = require_cuda(device)
        nz, ny, nx = data.dims3
        self.layout = SlabLayout(nz, ny, nx, ghost=data.n_b)
        self._plans = {}
        self._bufs = None

    # -- plumbing -----------------------------------------------------------
    def plan(self, precond="jacobi") -> NativePlan:
        if precond not in self._plans:
            self._plans[precond] = NativePlan(self.data, self.layout, self.device, precond)
        return self._plans[precond]

    def _io_buffers(self):
        if self._bufs is None:
            self._bufs = (self.layout.alloc(self.device), self.layout.alloc(self.device))
        return self._bufs

    @property
    def shape(self):
        return self.data.cext

    @property
    def dtype(self):
        return self.data.dtype

    # -- reference protocol -------------------------------------------------
    def apply(self, c, out=None):
        c = check_host_field(c, self.data.cext)
        if out is not None and (out.shape != self.data.cext or out.dtype != self.data.dtype):
            raise ValidationError("output buffer has wrong extents or dtype")
        cb, ob = self._io_buffers()
        self.layout.upload(c.reshape(self.layout.owned_shape), self.device, cb)
        self.plan().apply(cb, ob)
        t = self.layout.download(ob).reshape(self.data.cext).astype(self.data.dtype, copy=False)
        if out is not None:
            out[...] = t
            return out
        return t

    def jacobi_diagonal(self):
        cb, ob = self._io_buffers()
        self.plan().jacobi_diagonal(ob)
        diag = self.layout.download(ob).reshape(self.data.cext)
        bad = diag <= 0
        if np.any(bad):
            idx = np.argwhere(bad)[0]
            warnings.warn(
                f"non-positive operator diagonal at node {tuple(int(i) for i in idx)}",
                ConditioningWarning)
        return diag.astype(self.data.dtype, copy=False)

    def flop_byte_report(self, seconds=0.0) -> OpStats:
        n = self.data.num_unknowns()
        return OpStats(flops=int(n * apply_flops_per_dof(self.data.n_b)),
                       bytes_read=int(n * 8), bytes_written=int(n * 8), seconds=seconds)

    # -- device-resident API ------------------------------------------------
    def apply_device(self, c_buf, out_buf, stream=None):
        """``out = A c`` on ghosted-slab device tensors (no host copies)."""
        self.plan().apply(c_buf, out_buf, stream)
        return out_buf

    def mass_apply_device(self, c_buf, out_buf, f_buf=None, a=0.0, cm=None, stream=None):
        """``out = cm*(Mz(x)My(x)Mx) c + a*f`` (cm defaults to vol)."""
        cm = self.data.vol if cm is None else cm
        self.plan().mass_apply(c_buf, f_buf, cm, a, out_buf, stream)
        return out_buf


def make_operator(data, strategy="b200", workers=1, memory_budget=None, device=None):
    """Strategy dispatch (cf. operator.py:407-414).  Only ``"b200"`` lives here;
    the reference's host strategies stay in the reference package."""
    if strategy == "b200":
        from .varcoef import B200StencilOperator, VarSystemData

        if isinstance(data, VarSystemData):
            return B200StencilOperator(data, workers, device)
        return B200Operator(data, workers, device)
    raise ValidationError(f"unknown strategy {strategy!r} (this package provides 'b200')")


def assembled_rhs(data: SystemData, n_s, qcoef_ext, workers=1, device=None):
    """``t = vol * (R(x)R(x)R) q + face_rhs`` (cf. operator.py:417-441).

    For a box and ``n_s == n_b`` the source band R equals the mass Gram
    factor (edge rows included), so the volume part is the mass apply (GPU);
    penalty faces add their rank-1 surface terms (``SystemData.face_rhs``).
    """
    if int(n_s) != int(data.n_b):
        raise ConfigurationError("the b200 RHS realizes n_s == n_b (source degree = basis degree)")
    from .varcoef import VarSystemData

    if isinstance(data, VarSystemData) and data.mask is not None:
        # mask: the mass-only mask operator reproduces the free-space rows, the
        # cell-wise boundary rows and the zeroed inactive rows of
        # _mask_rhs_fixup (operator.py:444-488); exposed faces add the surface
        # entries on the device
        import torch

        from .varcoef import B200StencilOperator, build_var_system

        q = check_host_field(qcoef_ext, data.cext, "source coefficients")
        mop = B200StencilOperator(build_var_system(data.domain, data.n_b, 1, 0.0, 1.0, (),
                                                   np.float64), workers, device)
        qd = torch.from_numpy(q).to(mop.device)
        t = torch.empty_like(qd)
        mop.apply_device(qd, t)
        m = data.mask
        if m.surface_value is not None and m.surface_weight != 0.0:
            mop.surface_rhs_device(t, m.surface_weight, m.surface_value)
        return t.cpu().numpy().astype(data.dtype, copy=False)
    if isinstance(data, VarSystemData):
        # the source term does not involve D or mu: the box mass operator
        from .system import mass_system

        t = assembled_rhs(mass_system(data.domain.grid, data.n_b), n_s, qcoef_ext, workers, device)
        if any(ft.rhs_weight != 0.0 for ft in data.faces):
            t = t + data.face_rhs()
        return t.astype(data.dtype, copy=False)
    q = check_host_field(qcoef_ext, data.cext, "source coefficients")
    op = B200Operator(data, workers, device)
    cb, ob = op._io_buffers()
    op.layout.upload(q.reshape(op.layout.owned_shape), op.device, cb)
    op.mass_apply_device(cb, ob)
    t = op.layout.download(ob).reshape(data.cext)
    if any(ft.rhs_weight != 0.0 for ft in data.faces):
        t = t + data.face_rhs()
    return t.astype(data.dtype, copy=False)
