"""Jacobi-preconditioned CG on the B200 (drop-in for the reference ``pcg``).

Same signature, configuration, report and error behaviour as
``/root/reference/pkg/src/bspde/solver.py:20-117``.  The recurrence is the
reference's step for step (r0 = b - A x0; z = D^-1 r; p = z; loop: Ap,
pAp <= 0 -> IndefiniteOperatorError, alpha, x, r, z, beta, p, residual,
history, 1e3 divergence guard; stop on recursive ||r||/||b|| <= tol or
max_iter), executed as two fused sm_100a kernels per iteration:

* pass A (``sep_kernel<P, M_CGA>``): p_k = D^-1 r + beta p_{k-1} formed on
  the fly in shared memory (and stored to ring field k % P_RING), Ap_k,
  <p_k, Ap_k>;
* pass B (``cg_pass_b_kernel``): r -= alpha Ap, <r, D^-1 r>, <r, r>; every
  P_RING-th iteration also x += alpha_j p_j for the last P_RING iterations;

each finishing with a deterministic fixed-order reduction whose last CTA
runs the scalar update on the device.  Chunks of iterations are replayed as
one CUDA graph and the host polls the device state between chunks, so the
iteration count is exact (iterations past convergence are no-ops).
"""

from __future__ import annotations

import time
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .errors import (ConditioningWarning, ConfigurationError, DivergenceError,
                     IndefiniteOperatorError, ValidationError)


@dataclass
class SolveConfig:
    tol: float = 1e-8
    max_iter: int = 1000
    precond: str = "jacobi"  # "none" or "jacobi"
    coarse_init_factor: int = 0  # 0 disables coarse-grid initialization (problem.solve_problem)
    record_history: bool = False
    poll_every: int = 8  # CG iterations per CUDA-graph chunk between host polls

    def __post_init__(self):
        if self.tol <= 0:
            raise ValidationError(f"tol must be positive, got {self.tol}")
        if self.max_iter < 1:
            raise ValidationError(f"max_iter must be >= 1, got {self.max_iter}")
        if self.precond not in ("none", "jacobi"):
            raise ValidationError(f"unknown preconditioner {self.precond!r}")


@dataclass
class SolveReport:
    iterations: int
    relative_residual: float
    converged: bool
    wall_time: float
    history: list = field(default_factory=list)

    def history_csv(self):
        lines = ["iteration,residual"]
        lines += [f"{i},{r:.16e}" for i, r in enumerate(self.history)]
        return "\n".join(lines) + "\n"


class CgWork:
    """Device work vectors for one operator: r, the ring of R search
    directions (R = 4, or 2 when HBM is short: ``device.choose_ring``), Ap
    (also the heat RHS b: b is dead once r0 = b - A x0 is formed), scalar
    scratch, history.

    Allocated once and reused; nothing is allocated inside the CG loop."""

    def __init__(self, op, max_iter, ring=None):
        from .device import choose_ring

        lay = op.layout
        ring = ring or choose_ring(lay, op.device)
        self.r = lay.alloc(op.device)
        self.pring = lay.alloc_ring(op.device, ring)
        self.ap = lay.alloc(op.device)
        self.scratch = op.plan().scratch()
        self.history = None
        self.ensure_history(op, max_iter)

    def ensure_history(self, op, max_iter):
        import torch

        if self.history is None or self.history.numel() < max_iter + 1:
            self.history = torch.zeros(max_iter + 1, dtype=torch.float64, device=op.device)


def _work(op, max_iter) -> CgWork:
    w = getattr(op, "_cg_work", None)
    if w is None:
        w = CgWork(op, max_iter)
        op._cg_work = w
    return w


def _warn_diag(op, precond):
    if precond != "jacobi":
        return
    if np.any(op.data.diag_table() <= 0):
        op.jacobi_diagonal()  # emits ConditioningWarning with the node index


def report_from(rep, config, wall, history_dev):
    it = int(rep.iterations)
    if rep.status == N.BSPDE_CG_INDEFINITE:
        raise IndefiniteOperatorError(
            f"non-positive curvature p.Ap = {rep.last_pAp:.3e} at iteration {it}")
    if rep.status == N.BSPDE_CG_DIVERGED:
        raise DivergenceError(
            f"residual grew to {rep.residual:.3e} from {rep.residual0:.3e} at iteration {it}")
    rel = float(rep.relative_residual)
    hist = []
    if config.record_history:
        hist = [float(v) for v in history_dev[: it + 1].cpu().numpy()]
    return SolveReport(iterations=it, relative_residual=rel, converged=bool(rel <= config.tol),
                       wall_time=wall, history=hist)


def pcg_device(op, b_buf, x_buf, config: SolveConfig = None, has_x0=True, stream=None):
    """Solve ``A x = b`` on ghosted-slab device tensors; ``x_buf`` holds x0 on
    entry (if ``has_x0``) and the solution on return.  Returns SolveReport."""
    config = config or SolveConfig()
    t0 = time.perf_counter()
    _warn_diag(op, config.precond)
    w = _work(op, config.max_iter)
    w.ensure_history(op, config.max_iter)
    plan = op.plan(config.precond)
    rep = plan.pcg(b_buf, x_buf, w.r, w.pring, w.ap, w.scratch,
                   w.history if config.record_history else None, config.tol, config.max_iter,
                   config.record_history, has_x0, config.poll_every, stream)
    return report_from(rep, config, time.perf_counter() - t0, w.history)


def pcg(operator, rhs, config: SolveConfig = None, x0=None):
    """Solve ``operator.apply(c) = rhs``; returns ``(c, SolveReport)``.

    ``operator`` must be a ``b200`` operator (``make_operator(data, "b200")``);
    raises :class:`IndefiniteOperatorError` on non-positive curvature and
    :class:`DivergenceError` when the residual grows a thousandfold.
    """
    from .operator import B200Operator
    from .varcoef import B200StencilOperator

    config = config or SolveConfig()
    if isinstance(operator, B200StencilOperator):
        rhs = np.asarray(rhs, dtype=np.float64)
        if not np.all(np.isfinite(rhs)):
            raise ValidationError("right-hand side contains non-finite values")
        return operator.pcg(rhs.reshape(operator.data.cext), config, x0)
    if not isinstance(operator, B200Operator) and not hasattr(operator, "pcg_device"):
        raise ConfigurationError(
            "pcg here runs the B200 device solver; pass an operator from "
            "make_operator(data, 'b200') (host operators belong to the reference pcg)")
    rhs = np.asarray(rhs, dtype=np.float64)
    if not np.all(np.isfinite(rhs)):
        raise ValidationError("right-hand side contains non-finite values")
    if hasattr(operator, "pcg_device"):  # distributed operator
        return operator.pcg_host(rhs, config, x0)
    t0 = time.perf_counter()
    shape = operator.data.cext
    if rhs.shape != shape:
        rhs = rhs.reshape(shape)
    lay = operator.layout
    b_buf = lay.upload(rhs.reshape(lay.owned_shape), operator.device)
    if x0 is not None:
        x0 = np.asarray(x0, dtype=np.float64).reshape(lay.owned_shape)
        x_buf = lay.upload(x0, operator.device)
    else:
        x_buf = lay.alloc(operator.device)
    rep = pcg_device(operator, b_buf, x_buf, config, has_x0=x0 is not None)
    x = lay.download(x_buf).reshape(shape)
    rep.wall_time = time.perf_counter() - t0
    return x, rep
