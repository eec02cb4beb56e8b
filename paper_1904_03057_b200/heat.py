"""Implicit-Euler heat stepping on the B200 (the loop the reference lacks).

The reference solves steady problems only.  One implicit
Euler step of ``u_t = kappa * Laplace(u) + f`` in the Galerkin B-spline space
is exactly a reference system solve:

    b = M u_prev + dt (F + G)            M: mass system (D=0, mu=1)
    (M + dt*(kappa*K + W)) u = b, x0 = u_prev  Jacobi-PCG

with ``F = assembled_rhs(mass system, p, q)`` the Galerkin source and
``W``/``G`` the box-face surface terms of the boundary conditions (Robin /
DirichletPenalty; ``G`` the penalty right-hand side, cf. ``face_rhs``).  Here both
the RHS (``sep_kernel<P, M_MASS>``: fused mass apply + axpy) and the CG run
on the GPU with every field resident in HBM between steps.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .domain import BoxDomain, Grid
from .errors import ValidationError
from .operator import B200Operator
from .solver import SolveConfig, SolveReport, _work, pcg_device
from .boundary import realize_bc
from .system import heat_system
from .transform import sample_solution_device, transform_field_device


@dataclass
class HeatProblem:
    """Heat problem on a box, or on a voxel mask (``mask``: bool cells,
    SURVEY.md §8(f) item 4; one global Neumann / DirichletPenalty ``bc``).

    ``conductivity``: a constant, or a field on the extended parameter grid
    (degree = ``degree``), which selects the
    assembled-stencil operator.

    ``bc``: a condition or ``{face: condition}`` dict (:mod:`.boundary`;
    default: natural Neumann faces everywhere).

    ``initial`` and ``source`` accept a scalar, node samples or a callable of
    the node coordinates (like the reference's ProblemSpec fields); pass
    ``initial_coeffs`` / ``source_coeffs`` to give extended-grid coefficients
    directly.
    """

    grid: Grid
    degree: int
    dt: float
    conductivity: object = 1.0
    initial: object = 0.0
    source: object = 0.0
    initial_coeffs: np.ndarray = None
    source_coeffs: np.ndarray = None
    bc: object = None
    mask: np.ndarray = None

    def __post_init__(self):
        if not self.dt > 0:
            raise ValidationError(f"dt must be positive, got {self.dt}")


@dataclass
class HeatState:
    """Device-resident state of a running heat solve."""

    op: B200Operator
    u: object          # ghosted-slab tensor (current coefficients)
    F: object          # Galerkin source (or None)
    b: object          # RHS work buffer (the CG's Ap field on a box)
    reports: list = field(default_factory=list)


class HeatSolver:
    """Holds the heat operator and resident fields; ``step()`` advances dt."""

    def __init__(self, problem: HeatProblem, config: SolveConfig = None, device=None):
        self.problem = problem
        self.config = config or SolveConfig(tol=1e-10, max_iter=5000)
        is_mask = problem.mask is not None
        specs = (realize_bc(problem.bc, problem.grid, mask=is_mask)
                 if problem.bc is not None else ())
        kappa = np.asarray(problem.conductivity, dtype=np.float64)
        self.sop = self.mop = None
        if is_mask:
            # mask: A = M + dt (K(kappa) + W) and the mass M as mask stencils
            # (boundary rows from the occupied cells, inactive rows zero);
            # the box mass plan only provides the state layout and transforms
            from .domain import MaskDomain
            from .system import build_system, mass_system
            from .varcoef import B200StencilOperator, build_var_system

            grid, p, dt = problem.grid, int(problem.degree), float(problem.dt)
            dom = MaskDomain(grid, problem.mask)
            data = build_system(dom, p, p, dt * kappa if kappa.ndim else dt * float(kappa), 1.0,
                                [(a, s_, w * dt, v) for a, s_, w, v in specs])
            self.sop = B200StencilOperator(data, device=device)
            self.mop = B200StencilOperator(build_var_system(dom, p, 1, 0.0, 1.0, (), np.float64),
                                           device=device)
            self.op = B200Operator(mass_system(grid, p), device=device)
        elif kappa.ndim > 0 and not np.all(kappa == kappa.flat[0]):
            # variable conductivity: A = M + dt (K(kappa) + W) as an assembled
            # stencil; the RHS mass operator keeps the slab layout of the state
            from .system import build_system, mass_system
            from .varcoef import B200StencilOperator

            grid, p, dt = problem.grid, int(problem.degree), float(problem.dt)
            data = build_system(BoxDomain(grid), p, p, dt * kappa, 1.0,
                                [(a, s, w * dt, v) for a, s, w, v in specs])
            self.sop = B200StencilOperator(data, device=device)
            self.op = B200Operator(mass_system(grid, p), device=device)
        else:
            data = heat_system(problem.grid, problem.degree, problem.dt,
                               float(kappa.flat[0]) if kappa.ndim else float(kappa),
                               face_specs=specs)
            self.op = B200Operator(data, device=device)
        self.data = data
        self.dt = float(problem.dt)
        lay = self.op.layout
        dev = self.op.device
        u0 = problem.initial_coeffs
        if u0 is None:  # GPU direct transform straight into the slab layout
            self.u = transform_field_device(problem.initial, problem.grid, problem.degree, lay, dev)
        else:
            self.u = lay.upload(np.asarray(u0).reshape(lay.owned_shape), dev)
        self.b = lay.alloc(dev) if self.sop is not None or self.mop is not None else None
        q = problem.source_coeffs
        has_source = q is not None or not (np.ndim(problem.source) == 0
                                           and not callable(problem.source)
                                           and float(problem.source) == 0.0)
        self.F = None
        if is_mask:
            # dense F = M_mask q + (surface source per unit time)
            import torch

            self.F = torch.zeros(data.cext, dtype=torch.float64, device=dev)
            if has_source:
                if q is None:
                    qb = transform_field_device(problem.source, problem.grid, problem.degree, lay,
                                                dev)
                else:
                    qb = lay.upload(np.asarray(q).reshape(lay.owned_shape), dev)
                self.mop.apply_device(lay.owned(qb).contiguous(), self.F)
                del qb
            if specs and specs[0][3] is not None:
                self.mop.surface_rhs_device(self.F, specs[0][2], specs[0][3])
            self.reports = []
            return
        if has_source:
            if q is None:
                qb = transform_field_device(problem.source, problem.grid, problem.degree, lay, dev)
            else:
                qb = lay.upload(np.asarray(q).reshape(lay.owned_shape), dev)
            self.F = lay.alloc(dev)
            self.op.mass_apply_device(qb, self.F)  # F = vol * (M(x)M(x)M) q
            del qb
        if any(ft.rhs_weight != 0.0 for ft in data.faces):
            # penalty values: heat_system scaled the face terms by dt, so the
            # per-unit-time surface source is face_rhs / dt (added once)
            g = lay.upload((data.face_rhs() / self.dt).reshape(lay.owned_shape), dev)
            if self.F is None:
                self.F = g
            else:
                self.F.add_(g)
        if self.b is None:
            # box: b lives in the CG's Ap field (dead once r0 = b - A x0 is
            # formed); the work set is allocated after u and F so the ring
            # length sees the free HBM (device.choose_ring)
            self.b = _work(self.op, self.config.max_iter).ap
        self.reports = []

    @classmethod
    def from_device(cls, op: B200Operator, dt, u_buf, F_buf=None, config=None):
        """Wrap already-resident fields (bench / multi-step pipelines)."""
        self = cls.__new__(cls)
        self.problem = None
        self.sop = self.mop = None
        self.dt = float(dt)
        self.config = config or SolveConfig(tol=1e-10, max_iter=5000)
        self.data = op.data
        self.op = op
        self.u = u_buf
        self.F = F_buf
        self.b = _work(op, self.config.max_iter).ap  # b shares the CG's Ap field
        self.reports = []
        return self

    def rhs(self, stream=None):
        """b = M u + dt F (one fused kernel; mask: dense mask-mass apply + axpy)."""
        if self.mop is not None:
            x = self.op.layout.owned(self.u).contiguous()
            b = self.mop.apply_device(x, torch_empty_like(x), stream=stream)
            return b.add_(self.F, alpha=self.dt)
        self.op.mass_apply_device(self.u, self.b, self.F,
                                  a=self.dt if self.F is not None else 0.0, stream=stream)
        return self.b

    def step(self, stream=None) -> SolveReport:
        """Advance one dt.  Box: one fused native call (bspde_heat_step: the
        RHS rides in the first residual kernel, b is never formed); mask /
        variable conductivity: b = M u + dt F, then the stencil solve."""
        if self.mop is not None:  # mask: b = M_mask u + dt F on dense buffers
            lay = self.op.layout
            x = lay.owned(self.u).contiguous()
            b = self.mop.apply_device(x, torch_empty_like(x), stream=stream)
            b.add_(self.F, alpha=self.dt)
            rep = self.sop.pcg_device(b, x, self.config, has_x0=True, stream=stream)
            lay.owned(self.u).copy_(x)
            self.reports.append(rep)
            return rep
        if self.sop is not None:  # variable conductivity: dense buffers for the stencil solve
            self.rhs(stream)
            lay = self.op.layout
            b, x = lay.owned(self.b).contiguous(), lay.owned(self.u).contiguous()
            rep = self.sop.pcg_device(b, x, self.config, has_x0=True, stream=stream)
            lay.owned(self.u).copy_(x)
            self.reports.append(rep)
            return rep
        rep = heat_step_device(self.op, self.u, self.F, self.dt, self.config, stream=stream)
        self.reports.append(rep)
        return rep

    def run(self, steps: int):
        for _ in range(int(steps)):
            self.step()
        return self.reports

    def run_host(self, host_u, steps: int, chunks: int = 16):
        """Steps with the state in (pinned) host memory: every step uploads
        ``host_u`` and downloads the result into it (run_steps_host)."""
        own = self.op.layout.owned(self.u)
        return run_steps_host(self.step, own, host_u, steps, chunks)

    def save(self, path):
        """Checkpoint the current coefficients as a TBSF file (extended-grid
        extents, spline degree in the header; :func:`.io.write_field`)."""
        from .io import write_field

        write_field(path, self.op.layout, self.u, degree=self.data.n_b,
                    extents=self.data.cext)

    def restore(self, path):
        """Load coefficients written by :meth:`save` (or the reference's
        ``write_tensor`` of the same extents and degree) into the state."""
        from .io import read_field

        read_field(path, self.op.layout, self.op.device, buf=self.u, degree=self.data.n_b,
                   extents=self.data.cext)

    def coefficients(self) -> np.ndarray:
        return self.op.layout.download(self.u).reshape(self.data.cext)

    def node_values(self) -> np.ndarray:
        """The solution at the grid nodes (GPU sample_solution)."""
        grid = self.data.domain.grid
        return sample_solution_device(self.u, grid, self.data.n_b, self.op.layout).cpu().numpy()


def heat_step_device(op, u_buf, F_buf, dt, config: SolveConfig, stream=None) -> SolveReport:
    """(M + dt K) u <- vol M u + dt F in place on a box operator (x0 = u)."""
    import time

    from .solver import report_from

    t0 = time.perf_counter()
    w = _work(op, config.max_iter)
    w.ensure_history(op, config.max_iter)
    plan = op.plan(config.precond)
    rep = plan.heat_step(u_buf, F_buf, op.data.vol, dt if F_buf is not None else 0.0, w.r,
                         w.pring, w.ap, w.scratch,
                         w.history if config.record_history else None, config.tol,
                         config.max_iter, config.record_history, config.poll_every, stream)
    return report_from(rep, config, time.perf_counter() - t0, w.history)


def torch_empty_like(t):
    import torch

    return torch.empty_like(t)


def run_steps_host(step, dev, host, steps: int, chunks: int = 16, stream=None):
    """Step a device-resident state whose input and result live in host memory.

    ``dev``: the device view of the state (owned region, leading axis = z);
    ``host``: a pinned CPU tensor of the same shape holding the input.  Every
    step copies ``host -> dev``, runs ``step()`` on ``stream`` (default: the
    current stream) and copies ``dev -> host``.  The result copy of step k and
    the input copy of step k+1 move the same bytes through host memory, so
    they are split into ``chunks`` z-ranges and chunk i goes back up as soon as
    it is down (PCIe is full duplex; copies run on two side streams).  Returns
    the step reports.
    """
    import torch

    comp = stream if stream is not None else torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    nz = dev.shape[0]
    cuts = np.linspace(0, nz, max(1, min(int(chunks), nz)) + 1).astype(int)
    bounds = [(int(a), int(b)) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]
    start = torch.cuda.Event()
    start.record(comp)
    s_in.wait_event(start)
    with torch.cuda.stream(s_in):
        for a, b in bounds:
            dev[a:b].copy_(host[a:b], non_blocking=True)
    ready = torch.cuda.Event()
    ready.record(s_in)
    reports = []
    for k in range(int(steps)):
        comp.wait_event(ready)
        with torch.cuda.stream(comp):
            reports.append(step())
        done = torch.cuda.Event()
        done.record(comp)
        s_out.wait_event(done)
        down = []
        with torch.cuda.stream(s_out):
            for a, b in bounds:
                host[a:b].copy_(dev[a:b], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s_out)
                down.append(e)
        if k + 1 < steps:
            for (a, b), e in zip(bounds, down):
                s_in.wait_event(e)
                with torch.cuda.stream(s_in):
                    dev[a:b].copy_(host[a:b], non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(s_in)
    end = torch.cuda.Event()
    end.record(s_out)
    comp.wait_event(end)
    return reports


def heat_solve(problem: HeatProblem, steps: int, config: SolveConfig = None, device=None):
    """Run ``steps`` implicit-Euler steps; returns (coefficients, [SolveReport])."""
    hs = HeatSolver(problem, config, device)
    hs.run(steps)
    return hs.coefficients(), hs.reports
