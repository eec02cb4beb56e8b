"""GPU parity: the sm_100a path (through the C ABI) vs the reference (golden
fixtures) and the CPU oracle.

Bars: operator apply <= 1e-13 relative max; Jacobi diagonal
<= 1e-14; CG iteration counts within +-1 at tol 1e-10; solution coefficients
within 1e-10 relative L2 at CG tol 1e-13.  Between two correct
implementations that differ only in rounding, the coefficients drift by
~kappa*tol (measured: reference vs oracle 2.8e-10 at tol 1e-12 on C1), so the
looser tolerances are asserted at 1e-9 (tol 1e-12) and 1e-7 (tol 1e-10).
"""

import numpy as np
import pytest

from oracle import bspde_oracle as O
from paper_1904_03057_b200 import (BoxDomain, Grid, HeatProblem, HeatSolver,
                                   IndefiniteOperatorError, SolveConfig, assembled_rhs,
                                   build_system, heat_system, make_operator, mass_system, pcg)

pytestmark = pytest.mark.gpu

APPLY_TAGS = ["p1", "p2", "p3", "p4", "p5", "p3_heat", "p3_min", "p3_stiff", "p2_2d",
              "p1_1d", "p3_1d"]


def _data(meta, ndim):
    p, D, mu = int(meta[0]), meta[1], meta[2]
    step = tuple(meta[3:3 + ndim])
    ext = tuple(int(v) for v in meta[3 + ndim:3 + 2 * ndim])
    return build_system(BoxDomain(Grid(ext, step)), p, p, D, mu, []), ext, step, p, D, mu


def relmax(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


@pytest.mark.parametrize("tag", APPLY_TAGS)
def test_apply_and_diagonal_vs_reference(golden, cuda_device, tag):
    g = golden("apply.npz")
    c = g[f"{tag}_c"]
    data, *_ = _data(g[f"{tag}_meta"], c.ndim)
    op = make_operator(data, "b200")
    t = op.apply(c)
    assert t.shape == c.shape
    assert relmax(t, g[f"{tag}_t"]) < 1e-13
    np.testing.assert_allclose(op.jacobi_diagonal(), g[f"{tag}_diag"], rtol=1e-14, atol=1e-17)
    out = np.empty_like(c)
    assert op.apply(c, out=out) is out


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_rhs_vs_reference(golden, cuda_device, p):
    g = golden("rhs.npz")
    meta = g[f"p{p}_meta"]
    step = tuple(meta[1:4])
    ext = tuple(int(v) for v in meta[4:7])
    data = build_system(BoxDomain(Grid(ext, step)), p, p, 0.0, 1.0, [])
    t = assembled_rhs(data, p, g[f"p{p}_q"])
    assert relmax(t, g[f"p{p}_t"]) < 1e-13


@pytest.mark.parametrize("p,ext", [(3, (70, 45, 97)), (1, (33, 65, 31)), (2, (40, 33, 66)),
                                   (4, (37, 41, 35)), (5, (36, 34, 40)), (3, (300, 6, 6)),
                                   (3, (4, 70, 5))])
def test_apply_multi_tile_vs_oracle(cuda_device, p, ext):
    rng = np.random.default_rng(sum(ext) + p)
    step = (0.013, 0.021, 0.017)
    D, mu = 3e-4, 1.0
    data = build_system(BoxDomain(Grid(ext, step)), p, p, D, mu, [])
    ora = O.KronOperator(ext, step, p, D, mu)
    c = rng.normal(size=data.cext)
    op = make_operator(data, "b200")
    assert relmax(op.apply(c), ora.apply(c)) < 1e-13
    # mass apply with axpy through the device API
    lay = op.layout
    cb = lay.upload(c, op.device)
    fb = lay.upload(np.cos(c), op.device)
    ob = lay.alloc(op.device)
    op.mass_apply_device(cb, ob, fb, a=0.25)
    want = ora.mass_apply(c) + 0.25 * np.cos(c)
    assert relmax(lay.download(ob), want) < 1e-13


def _heat_op(h):
    p, N, hh, dt = int(h["meta"][0]), int(h["meta"][1]), h["meta"][2], h["meta"][3]
    return p, N, hh, dt


def test_heat16_steps_vs_reference(golden, cuda_device):
    h = golden("heat16.npz")
    p, N, hh, dt = _heat_op(h)
    prob = HeatProblem(Grid((N,) * 3, (hh,) * 3), p, dt, initial_coeffs=h["u0"],
                       source_coeffs=h["q"])
    hs = HeatSolver(prob, SolveConfig(tol=1e-10, max_iter=5000))
    its = [hs.step().iterations for _ in range(10)]
    ref = [int(v) for v in h["iters_tol1e-10"]]
    print("heat16 iterations gpu", its, "reference", ref)
    # ~235 iterations per step: the oracle itself (same recurrence, numpy
    # rounding) lands at +-1 of the reference here
    assert all(abs(a - b) <= 1 for a, b in zip(its, ref)), (its, ref)
    u = hs.coefficients()
    refu = h["u_final_tol1e-10"]
    assert np.linalg.norm(u - refu) / np.linalg.norm(refu) < 1e-7


def test_heat16_tol12_coefficients_vs_reference(golden, cuda_device):
    h = golden("heat16.npz")
    p, N, hh, dt = _heat_op(h)
    op = make_operator(heat_system(Grid((N,) * 3, (hh,) * 3), p, dt), "b200")
    x, rep = pcg(op, h["b1"], SolveConfig(tol=1e-12, max_iter=5000, record_history=True),
                 x0=h["u0"])
    ref = h["u1_tol1e-12"]
    assert np.linalg.norm(x - ref) / np.linalg.norm(ref) < 1e-9
    assert abs(rep.iterations - int(h["iters1_tol1e-12"][0])) <= 1
    x13, rep13 = pcg(op, h["b1"], SolveConfig(tol=1e-13, max_iter=5000), x0=h["u0"])
    ref = h["u1_tol1e-13"]
    assert np.linalg.norm(x13 - ref) / np.linalg.norm(ref) < 1e-10
    assert abs(rep13.iterations - int(h["iters1_tol1e-13"][0])) <= 1
    hist = np.array(rep.history)
    rh = h["history1_tol1e-12"]
    n = min(len(hist), len(rh))
    # trajectories agree to rounding drift relative to the initial residual
    assert float(np.abs(hist[:n] - rh[:n]).max()) < 1e-8 * rh[0]
    assert rep.converged and rep.relative_residual <= 1e-12


def test_heat64_C1_vs_reference(golden, cuda_device):
    """C1: 64^3, p=3, lambda=4, 10 steps -- reference CG counts
    [45, 45, 47, 50, 63, 77, 91, 112, 120, 129] within +-1."""
    h = golden("heat64.npz")
    p, N, hh, dt = _heat_op(h)
    inp = O.heat_inputs(64)  # identical to the reference's inputs (test_oracle)
    prob = HeatProblem(Grid((N,) * 3, (hh,) * 3), p, dt, initial_coeffs=inp["u0"],
                       source_coeffs=inp["q"])
    hs = HeatSolver(prob, SolveConfig(tol=1e-10, max_iter=5000))
    ora = O.KronOperator((N,) * 3, (hh,) * 3, p, dt, 1.0)
    F = ora.mass_apply(inp["q"])
    np.testing.assert_allclose(hs.op.layout.download(hs.F), F, rtol=0,
                               atol=1e-13 * np.abs(F).max())
    its = [hs.step().iterations for _ in range(10)]
    ref = [int(v) for v in h["iters_tol1e-10"]]
    assert all(abs(a - b) <= 1 for a, b in zip(its, ref)), (its, ref)
    refu = h["u_final_tol1e-10"]
    assert np.linalg.norm(hs.coefficients() - refu) / np.linalg.norm(refu) < 1e-7
    op = make_operator(heat_system(Grid((N,) * 3, (hh,) * 3), p, dt), "b200")
    assert relmax(op.apply(inp["u0"]), ora.apply(inp["u0"])) < 1e-13
    b1 = ora.mass_apply(inp["u0"]) + dt * F
    for tol, bar in ((1e-12, 1e-9), (1e-13, 1e-10)):
        x, rep = pcg(op, b1, SolveConfig(tol=tol, max_iter=5000), x0=inp["u0"])
        ref = h[f"u1_tol{tol:.0e}"]
        assert np.linalg.norm(x - ref) / np.linalg.norm(ref) < bar, tol
        assert abs(rep.iterations - int(h[f"iters1_tol{tol:.0e}"][0])) <= 1


def _smooth_rhs(ora, seed):
    """Galerkin RHS of a smooth source (b = M q): a physically meaningful
    right-hand side.  (With white-noise b the Jacobi-PCG residual of these
    mass-dominated systems grows >1e3x before converging, so the reference
    algorithm itself stops with DivergenceError -- see test_divergence_guard.)"""
    rng = np.random.default_rng(seed)
    axes = [np.linspace(0.0, 1.0, n) for n in ora.cext]
    Z, Y, X = np.meshgrid(*axes, indexing="ij")
    k = rng.uniform(1.0, 3.0, 3)
    q = np.cos(k[0] * np.pi * Z) * np.sin(k[1] * np.pi * Y + 0.3) + np.exp(-8 * (X - 0.4) ** 2)
    return ora.mass_apply(q)


def test_cg_vs_oracle_odd_shapes(cuda_device):
    # ragged tiles, odd x extent, p=2 and p=5, both preconditioners
    for p, ext, precond in [(2, (23, 37, 41), "jacobi"), (5, (20, 19, 33), "jacobi"),
                            (3, (25, 30, 27), "none")]:
        step = tuple(1.0 / (n - 1) for n in ext)
        data = build_system(BoxDomain(Grid(ext, step)), p, p, 0.01, 1.0, [])
        ora = O.KronOperator(ext, step, p, 0.01, 1.0)
        b = _smooth_rhs(ora, p)
        op = make_operator(data, "b200")
        cfg = SolveConfig(tol=1e-11, max_iter=3000, precond=precond, record_history=True)
        x, rep = pcg(op, b, cfg)
        xo, ro = O.pcg(ora.apply, ora.jacobi_diagonal, b, tol=1e-11, max_iter=3000,
                       precond=precond, record_history=True)
        assert abs(rep.iterations - ro["iterations"]) <= 1, (p, rep.iterations, ro["iterations"])
        # both solutions solve the system to the same (recursive) tolerance; the
        # edge coefficients of these mass-dominated systems are ill-conditioned,
        # so x itself agrees only to ~kappa*tol -- check the true residuals
        true_res = float(np.linalg.norm(b - ora.apply(x)) / np.linalg.norm(b))
        true_res_o = float(np.linalg.norm(b - ora.apply(xo)) / np.linalg.norm(b))
        # the true residual agrees with the oracle's: for the ill-conditioned p=5
        # case the recursive residual stagnates at ~1e-9 while the true one sits
        # at ~3.4e-7 in both implementations
        assert true_res < 3 * true_res_o + 1e-9, (true_res, true_res_o)
        # same outcome as the reference recurrence (the p=5 case stagnates at its
        # rounding floor ~1e-9 and stops at max_iter in both)
        assert rep.converged == bool(ro["converged"])
        assert rep.relative_residual < 10 * ro["relative_residual"] + 1e-12
        assert len(rep.history) == rep.iterations + 1


# (n, D, mu, seed): indefinite systems (negative absorption) on which the
# reference recurrence's recursive residual grows past 1e3 * res0 while every
# curvature p.Ap stays positive (min p.Ap / p.p ~1e-9 relative to the
# operator scale ~1e-3: far from the rounding level); found by a sweep of the
# oracle pcg over sizes, shifts and seeds.  The last residual ratio before
# the guard fires is 1.1e3 / 1.5e3 / 1.7e3.
DIVERGENT = [(6, 1.0, -20.0, 0), (8, 0.01, -1.0, 0), (7, 0.1, -0.2, 2)]


@pytest.mark.parametrize("case", DIVERGENT)
def test_divergence_guard(cuda_device, case):
    """A residual that grows past 1e3*res0 stops the solve with
    DivergenceError at the same iteration as the reference recurrence
    (solver.py:105-108; reference test pkg/tests/test_solver.py:206-218)."""
    import re

    from paper_1904_03057_b200 import DivergenceError

    n, D, mu, seed = case
    ext = (n, n, n)
    step = tuple(1.0 / (m - 1) for m in ext)
    data = build_system(BoxDomain(Grid(ext, step)), 3, 3, D, mu, [])
    ora = O.KronOperator(ext, step, 3, D, mu)
    b = np.random.default_rng(seed).normal(size=ora.cext)
    with pytest.raises(O.OracleDivergence) as eo:
        O.pcg(ora.apply, ora.jacobi_diagonal, b, tol=1e-10, max_iter=3000)
    it_o = int(re.search(r"iteration (\d+)", str(eo.value)).group(1))
    with pytest.raises(DivergenceError) as eg:
        pcg(make_operator(data, "b200"), b, SolveConfig(tol=1e-10, max_iter=3000))
    it_g = int(re.search(r"iteration (\d+)", str(eg.value)).group(1))
    assert it_g == it_o, (it_g, it_o)


def test_cg_edge_cases(cuda_device):
    ext, step = (12, 12, 12), (0.1, 0.1, 0.1)
    data = build_system(BoxDomain(Grid(ext, step)), 3, 3, 0.01, 1.0, [])
    op = make_operator(data, "b200")
    x, rep = pcg(op, np.zeros(data.cext))
    assert rep.iterations == 0 and rep.converged and not x.any()
    b = np.random.default_rng(0).normal(size=data.cext)
    x, rep = pcg(op, b, SolveConfig(tol=1e-14, max_iter=3))
    assert rep.iterations == 3 and not rep.converged
    # x0 == exact solution of a zero rhs -> zero residual, no iterations
    x, rep = pcg(op, np.zeros(data.cext), SolveConfig(), x0=np.zeros(data.cext))
    assert rep.iterations == 0
    # indefinite: negative absorption
    neg = build_system(BoxDomain(Grid(ext, step)), 3, 3, 0.0, -1.0, [])
    with pytest.raises(IndefiniteOperatorError):
        pcg(make_operator(neg, "b200"), b, SolveConfig(precond="none"))
    from paper_1904_03057_b200 import ValidationError
    bad = b.copy()
    bad[0, 0, 0] = np.nan
    with pytest.raises(ValidationError):
        pcg(op, bad)
    with pytest.raises(ValidationError):
        op.apply(np.ones((5, 5, 5)))


def test_determinism_bitwise(cuda_device):
    ext = (40, 50, 60)
    step = tuple(1.0 / (n - 1) for n in ext)
    data = build_system(BoxDomain(Grid(ext, step)), 3, 3, 1e-3, 1.0, [])
    b = np.random.default_rng(5).normal(size=data.cext)
    op = make_operator(data, "b200")
    x1, r1 = pcg(op, b, SolveConfig(tol=1e-10, record_history=True))
    x2, r2 = pcg(op, b, SolveConfig(tol=1e-10, record_history=True))
    assert np.array_equal(x1, x2) and r1.history == r2.history
    t1 = op.apply(b)
    assert np.array_equal(t1, op.apply(b))


@pytest.mark.slow
def test_c2_256_properties(cuda_device):
    """C2 (256^3): apply vs oracle, symmetry, and a converged heat step
    checked through its true residual (the oracle pcg is too slow here)."""
    import torch

    n = 256
    N = n - 2
    hh = 1.0 / (N - 1)
    dt = 4 * hh * hh
    g = Grid((N,) * 3, (hh,) * 3)
    op = make_operator(heat_system(g, 3, dt), "b200")
    ora = O.KronOperator((N,) * 3, (hh,) * 3, 3, dt, 1.0)
    rng = np.random.default_rng(256)
    u = rng.normal(size=op.data.cext)
    v = rng.normal(size=op.data.cext)
    Au = op.apply(u)
    assert relmax(Au, ora.apply(u)) < 1e-13
    Av = op.apply(v)
    assert abs(np.vdot(u, Av) - np.vdot(Au, v)) / abs(np.vdot(u, Av)) < 1e-12
    inp = O.heat_inputs(n)
    A_b = ora.mass_apply(inp["u0"]) + dt * ora.mass_apply(inp["q"])
    x, rep = pcg(op, A_b, SolveConfig(tol=1e-10, max_iter=5000), x0=inp["u0"])
    assert rep.converged
    true_res = np.linalg.norm(A_b - ora.apply(x)) / np.linalg.norm(A_b)
    assert true_res < 1e-9
    torch.cuda.empty_cache()


@pytest.mark.parametrize("case", [(3, (12, 12, 12), False), (3, (12, 12, 12), True),
                                  (2, (23, 37, 41), False), (5, (20, 19, 33), True)])
def test_cg_stepwise_vs_oracle(cuda_device, case):
    """One CG iteration through the step-wise ABI: every vector and scalar of
    the recurrence (solver.py:75-101) against the oracle."""
    import ctypes as C

    import torch

    from paper_1904_03057_b200.solver import _work

    p, ext, has_x0 = case
    step = tuple(1.0 / (n - 1) for n in ext)
    D, mu = 0.01, 1.0
    data = build_system(BoxDomain(Grid(ext, step)), p, p, D, mu, [])
    ora = O.KronOperator(ext, step, p, D, mu)
    rng = np.random.default_rng(7)
    b = rng.normal(size=data.cext)
    x0 = rng.normal(size=data.cext) if has_x0 else np.zeros(data.cext)
    op = make_operator(data, "b200")
    lay = op.layout
    plan = op.plan()
    w = _work(op, 10)
    bb = lay.upload(b, op.device)
    xb = lay.upload(x0, op.device)
    R = w.pring.shape[0]
    w.pring[R - 1].zero_()  # p_{-1}
    w.pring[0].fill_(np.nan)  # pass A must write every owned point of p_out
    plan.cg_setup(w.scratch, None, 1e-300, 100, False, has_x0)
    plan.cg_residual(bb, xb, w.r, w.scratch, 1)
    torch.cuda.synchronize()
    inv = 1.0 / ora.jacobi_diagonal()
    r0 = b - ora.apply(x0)
    assert relmax(lay.download(w.r), r0) < 1e-13
    st = w.scratch[:160].cpu().numpy().view(np.float64)
    rz0 = float(np.vdot(r0, inv * r0))
    assert abs(st[8] - rz0) / rz0 < 1e-12  # state.rz
    plan.cg_pass_a(xb, w.r, w.pring[R - 1], w.pring[0], w.ap, w.scratch, 1)
    torch.cuda.synchronize()
    p0 = inv * r0
    assert float(relmax(lay.download(w.pring[0]), p0)) < 1e-13  # p_k written by pass A
    assert np.array_equal(lay.download(xb), x0)  # nothing pending before iteration 0
    Ap = ora.apply(p0)
    assert relmax(lay.download(w.ap), Ap) < 1e-13
    st = w.scratch[:160].cpu().numpy().view(np.float64)
    pAp = float(np.vdot(p0, Ap))
    assert abs(st[11] - pAp) / pAp < 1e-12  # state.pAp
    alpha = rz0 / pAp
    assert abs(st[9] - alpha) / alpha < 1e-12  # state.alpha
    plan.cg_pass_b(w.r, w.ap, w.scratch, 1)
    torch.cuda.synchronize()
    x1 = x0 + alpha * p0
    r1 = r0 - alpha * Ap
    # x moves in the next pass A (or on the flush at the end of a solve)
    assert np.array_equal(lay.download(xb), x0)
    assert relmax(lay.download(w.r), r1) < 1e-12
    rep, active = plan.cg_read(w.scratch)
    assert rep.iterations == 1
    assert abs(rep.residual - np.linalg.norm(r1)) / np.linalg.norm(r1) < 1e-12
    state1 = w.scratch.clone()  # after iteration 0
    xe = xb.clone()
    plan.cg_flush_x(xe, w.pring, w.scratch)
    torch.cuda.synchronize()
    assert relmax(lay.download(xe), x1) < 1e-13
    plan.cg_flush_x(xe, w.pring, w.scratch)  # idempotent: nothing pending any more
    assert relmax(lay.download(xe), x1) < 1e-13
    # ... and pass A of iteration 1 (from the unflushed state) applies the same
    # update x1 = fl(x0 + fl(alpha p0)) bit for bit (forced active: the p = 5
    # case trips the divergence guard at iteration 1)
    w.scratch.copy_(state1)
    w.scratch[152:156].view(torch.int32)[0] = 1  # CgState.active
    plan.cg_pass_a(xb, w.r, w.pring[0], w.pring[1 % R], w.ap, w.scratch, 1)
    torch.cuda.synchronize()
    assert np.array_equal(lay.download(xb), lay.download(xe))


@pytest.mark.parametrize("iters,ring", [(1, 2), (2, 2), (3, 2), (5, 2), (8, 2), (3, 4), (9, 4)])
def test_deferred_x_update_is_bitwise_eager(cuda_device, iters, ring):
    """Pass A of iteration k applies x += alpha_{k-1} p_{k-1}; flushing after
    every pass B instead (x updated one pass A earlier) must give bit-identical
    x (the same stored roundings, solver.py:94), for both ring lengths."""
    import torch

    ext, p = (13, 12, 11), 3
    step = tuple(1.0 / (n - 1) for n in ext)
    data = build_system(BoxDomain(Grid(ext, step)), p, p, 0.01, 1.0, [])
    rng = np.random.default_rng(11)
    b = rng.normal(size=data.cext)
    x0 = rng.normal(size=data.cext)
    outs = []
    for eager in (False, True):
        op = make_operator(data, "b200")
        lay, plan = op.layout, op.plan()
        bb, xb = lay.upload(b, op.device), lay.upload(x0, op.device)
        r, ap = lay.alloc(op.device), lay.alloc(op.device)
        pring = lay.alloc_ring(op.device, ring)
        R = pring.shape[0]
        scratch = plan.scratch()
        plan.cg_setup(scratch, None, 1e-300, 100, False, True, p_ring=R)
        plan.cg_residual(bb, xb, r, scratch, 1)
        for k in range(iters):
            plan.cg_pass_a(xb, r, pring[(k - 1) % R], pring[k % R], ap, scratch, 1)
            plan.cg_pass_b(r, ap, scratch, 1)
            if eager:
                plan.cg_flush_x(xb, pring, scratch)
        plan.cg_flush_x(xb, pring, scratch)
        torch.cuda.synchronize()
        outs.append(lay.download(xb))
    assert np.array_equal(outs[0], outs[1])


def test_distributed_path_single_rank_matches_fused(cuda_device):
    """The z-slab driver (step-wise ABI, fuse=0, separate finalize kernels) on
    one rank reproduces the fused single-GPU solver bit for bit."""
    from paper_1904_03057_b200.distributed import DistributedOperator

    h_n = 24
    inp = O.heat_inputs(h_n)
    N, hh, dt = inp["N"], inp["h"], inp["dt"]
    data = heat_system(Grid((N,) * 3, (hh,) * 3), 3, dt)
    ora = O.KronOperator((N,) * 3, (hh,) * 3, 3, dt, 1.0)
    b = ora.mass_apply(inp["u0"]) + dt * ora.mass_apply(inp["q"])
    cfg = SolveConfig(tol=1e-10, max_iter=2000, record_history=True)
    x1, r1 = pcg(make_operator(data, "b200"), b, cfg, x0=inp["u0"])
    dop = DistributedOperator(data)
    x2, r2 = dop.pcg_host(b, cfg, x0=inp["u0"])
    assert r1.iterations == r2.iterations
    assert np.array_equal(x1, x2)
    assert r1.history == r2.history
    # operator apply through the slab path
    cb = dop.scatter(inp["u0"])
    ob = dop.layout.alloc(dop.device)
    dop.apply_device(cb, ob)
    assert relmax(dop.gather(ob), ora.apply(inp["u0"])) < 1e-13


# ---------------------------------------------------------------------------
# box-face Robin / penalty terms

FACE_TAGS = ["p1", "p2", "p3", "p4", "p5", "p3_all", "p2_2d", "p3_1d"]


@pytest.mark.parametrize("tag", FACE_TAGS)
def test_faces_apply_diag_rhs_vs_reference(golden, cuda_device, tag):
    """build_system(face_specs) -> b200 apply / Jacobi diagonal / assembled_rhs
    against the reference's OnTheFlyOperator and assembled_rhs."""
    g = golden("faces.npz")
    meta = g[f"{tag}_meta"]
    p, D, mu = int(meta[0]), float(meta[1]), float(meta[2])
    d = (len(meta) - 3) // 2
    step = tuple(float(v) for v in meta[3:3 + d])
    ext = tuple(int(v) for v in meta[3 + d:])
    specs = [(int(a), int(s), float(w), None if np.isnan(v) else float(v))
             for a, s, w, v in g[f"{tag}_faces"]]
    data = build_system(BoxDomain(Grid(ext, step)), p, p, D, mu, specs)
    op = make_operator(data, "b200")
    assert relmax(op.apply(g[f"{tag}_c"]), g[f"{tag}_t"]) < 1e-13
    assert relmax(op.jacobi_diagonal(), g[f"{tag}_diag"]) < 1e-13
    assert relmax(assembled_rhs(data, p, g[f"{tag}_q"]), g[f"{tag}_rhs"]) < 1e-13


@pytest.mark.parametrize("bc_kind", ["penalty", "mixed"])
def test_heat_with_faces_vs_oracle(cuda_device, bc_kind):
    """Implicit Euler with Robin / DirichletPenalty faces: CG counts (+-1) and
    coefficients against the oracle's composition (M + dt(K + W)) u = M u +
    dt F + dt G, at tol 1e-13 for the 1e-10 coefficient bar."""
    from paper_1904_03057_b200 import DirichletPenalty, Neumann, Robin, realize_bc

    inp = O.heat_inputs(20)
    N, hh, dt, p = inp["N"], inp["h"], inp["dt"], 3
    grid = Grid((N,) * 3, (hh,) * 3)
    if bc_kind == "penalty":
        bc = {"all": DirichletPenalty(0.2, epsilon=0.05)}
    else:
        bc = {"all": Neumann(), "x0": Robin(0.5), "y1": DirichletPenalty(1.0, epsilon=0.02),
              "z0": DirichletPenalty(-0.5, epsilon=0.1)}
    specs = realize_bc(bc, grid)
    for tol, steps in ((1e-10, 3), (1e-13, 1)):
        prob = HeatProblem(grid, p, dt, initial_coeffs=inp["u0"], source_coeffs=inp["q"], bc=bc)
        hs = HeatSolver(prob, SolveConfig(tol=tol, max_iter=5000))
        its = [hs.step().iterations for _ in range(steps)]
        u_ora, its_ora = O.heat_steps(N, hh, p, dt, inp["u0"], inp["q"], steps, tol=tol,
                                      faces=specs)
        print(bc_kind, tol, "gpu", its, "oracle", its_ora)
        # +-1 for ~100-iteration solves; these take 300-470
        # iterations and the rounding drift between two correct recurrences
        # grows with the count: +-0.5%
        assert all(abs(a - b) <= max(1, round(0.005 * b)) for a, b in zip(its, its_ora)), \
            (its, its_ora)
        u = hs.coefficients()
        rel = np.linalg.norm(u - u_ora) / np.linalg.norm(u_ora)
        assert rel < (1e-10 if tol == 1e-13 else 1e-7), rel


# ---------------------------------------------------------------------------
# B-spline field transforms on the GPU


def test_direct_transform_vs_reference(golden, cuda_device):
    """prefilter_kernel (all three extensions, p=2..5, 1-D/2-D/3-D, lines
    shorter than the causal-init horizon) against the reference."""
    from paper_1904_03057_b200.transform import direct_transform

    g = golden("transform.npz")
    n = 0
    for key in list(g.keys()):
        if not key.endswith("_x") or key.startswith("field"):
            continue
        tag = key[:-2]
        parts = tag.split("_")
        p = int(parts[1][1:])
        ext_mode = parts[2] if parts[2] in ("mirror", "replicate", "zero") else "mirror"
        c = direct_transform(g[key], p, ext_mode)
        assert relmax(c, g[f"{tag}_c"]) < 1e-13, tag
        n += 1
    assert n == 11


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_transform_field_and_sampling_vs_reference(golden, cuda_device, p):
    from paper_1904_03057_b200.transform import sample_solution, transform_field

    g = golden("transform.npz")
    grid = Grid((9, 10, 11), (0.1, 0.2, 0.15))
    ce = transform_field(g[f"field_p{p}_f"], grid, p)
    assert relmax(ce, g[f"field_p{p}_c"]) < 1e-13
    s = sample_solution(g[f"field_p{p}_c"], grid, p)
    assert relmax(s, g[f"field_p{p}_s"]) < 1e-14
    # interpolation: sampling the transform reproduces the samples
    assert relmax(s, g[f"field_p{p}_f"]) < 1e-10


def test_transform_2d_and_heat_ic(golden, cuda_device):
    from paper_1904_03057_b200.transform import sample_solution, transform_field

    g = golden("transform.npz")
    grid2 = Grid((12, 9), (0.5, 0.25))
    assert relmax(transform_field(g["field2d_p3_f"], grid2, 3), g["field2d_p3_c"]) < 1e-13
    assert relmax(sample_solution(g["field2d_p3_c"], grid2, 3), g["field2d_p3_s"]) < 1e-14
    # the heat16 initial condition via a callable, straight into the slab layout
    h = golden("heat16.npz")
    p, N, hh, dt = _heat_op(h)
    prob = HeatProblem(Grid((N,) * 3, (hh,) * 3), p, dt,
                       initial=lambda x, y, z: np.exp(-40 * ((x - .5) ** 2 + (y - .4) ** 2 +
                                                             (z - .6) ** 2)))
    hs = HeatSolver(prob)
    assert float(np.abs(hs.coefficients() - h["u0"]).max()) < 1e-14
    x = np.arange(N) * hh
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    ref = np.exp(-40 * ((X - .5) ** 2 + (Y - .4) ** 2 + (Z - .6) ** 2))
    assert float(np.abs(hs.node_values() - ref).max()) < 1e-10


def test_run_host_matches_device_stepping(golden, cuda_device):
    """HeatSolver.run_host (state in pinned host memory, overlapped chunked
    copies) gives bit-identical coefficients and counts to device stepping."""
    import torch

    h = golden("heat16.npz")
    p, N, hh, dt = _heat_op(h)
    grid = Grid((N,) * 3, (hh,) * 3)
    a = HeatSolver(HeatProblem(grid, p, dt, initial_coeffs=h["u0"], source_coeffs=h["q"]))
    its_a = [a.step().iterations for _ in range(3)]
    b = HeatSolver(HeatProblem(grid, p, dt, initial_coeffs=h["u0"], source_coeffs=h["q"]))
    host = torch.from_numpy(np.ascontiguousarray(h["u0"])).pin_memory()
    b.u.zero_()  # the input must come from host memory
    reps = b.run_host(host, 3, chunks=5)
    torch.cuda.synchronize()
    assert [r.iterations for r in reps] == its_a
    assert np.array_equal(host.numpy(), a.coefficients())
    assert np.array_equal(b.coefficients(), a.coefficients())


@pytest.mark.parametrize("p,ext,world", [(3, (30, 19, 33), 2), (3, (31, 20, 21), 3),
                                         (5, (32, 17, 19), 2), (1, (14, 12, 13), 2)])
def test_pass_a_ranges_on_emulated_slabs(cuda_device, p, ext, world):
    """Pass A split as the overlapped z-slab driver runs it (interior planes
    [p, nz-p) first, then the two p-plane boundary ranges, sums accumulated)
    on every slab of an emulated `world`-rank partition on ONE device, ghost
    planes filled from the neighbours by plain copies: Ap and p_k must equal
    the unsplit pass A bit for bit and match the global oracle; the summed
    <p,Ap> the global one."""
    import torch

    from paper_1904_03057_b200.device import NativePlan, SlabLayout
    from paper_1904_03057_b200.distributed import SlabPartition

    step = tuple(1.0 / (n - 1) for n in ext)
    data = build_system(BoxDomain(Grid(ext, step)), p, p, 0.01, 1.0, [])
    ora = O.KronOperator(ext, step, p, 0.01, 1.0)
    rng = np.random.default_rng(3)
    r_full = rng.normal(size=data.cext)
    q_full = rng.normal(size=data.cext)
    inv = 1.0 / ora.jacobi_diagonal()
    beta = 0.37
    p_full = inv * r_full + beta * q_full
    want_ap = ora.apply(p_full)
    nzg, ny, nx = data.dims3
    dots = []
    for rank in range(world):
        part = SlabPartition(nzg, world, rank)
        lo, hi = part.bounds()
        lay = SlabLayout(part.nz, ny, nx, ghost=p, z_offset=part.z_offset, nz_global=nzg)
        assert lay.nz > 2 * p
        plan = NativePlan(data, lay, cuda_device)

        def slab(full):
            buf = lay.alloc(cuda_device)
            glo, ghi = max(lo - p, 0), min(hi + p, nzg)
            src = torch.from_numpy(np.ascontiguousarray(full.reshape(nzg, ny, nx)[glo:ghi]))
            buf[glo - (lo - p):ghi - (lo - p), :, :nx] = src.to(cuda_device)
            return buf

        rb, qb = slab(r_full), slab(q_full)
        x0 = rng.normal(size=(hi - lo, ny, nx))
        outs = []
        for split in (False, True):
            scratch = plan.scratch()
            plan.cg_setup(scratch, None, 1e-300, 100, False, False)
            scratch[72:80].view(torch.float64)[0] = 0.61  # CgState.alpha (= alpha_{k-1})
            scratch[80:88].view(torch.float64)[0] = beta  # CgState.beta
            scratch[144:148].view(torch.int32)[0] = 1     # CgState.it: iteration k = 1
            scratch[152:156].view(torch.int32)[0] = 1     # CgState.active (18 doubles, it, max_iter)
            ap, pout = lay.alloc(cuda_device), lay.alloc(cuda_device)
            xb = lay.upload(x0, cuda_device)
            pout.fill_(float("nan"))
            if split:
                nz = lay.nz
                plan.cg_pass_a_range(xb, rb, qb, pout, ap, scratch, p, nz - 2 * p, False)
                plan.cg_pass_a_range(xb, rb, qb, pout, ap, scratch, 0, p, True)
                plan.cg_pass_a_range(xb, rb, qb, pout, ap, scratch, nz - p, p, True)
            else:
                plan.cg_pass_a(xb, rb, qb, pout, ap, scratch, 0)
            torch.cuda.synchronize()
            pair = scratch[:64].view(torch.float64).cpu().numpy()  # fuse = 0: (hi, lo) pairs
            outs.append((lay.download(ap), lay.download(pout), float(pair[0] + pair[4])))
            # x += alpha_{k-1} p_{k-1} on the owned planes, rounded as solver.py:94
            want_x = x0 + 0.61 * q_full.reshape(nzg, ny, nx)[lo:hi]
            assert np.array_equal(lay.download(xb), want_x)
        (a0, p0, d0), (a1, p1, d1) = outs
        assert np.array_equal(a0, a1) and np.array_equal(p0, p1)
        assert abs(d0 - d1) <= 2.3e-16 * abs(d0)  # double-double: the split does not round
        sl = (slice(lo, hi),)
        assert relmax(a1, want_ap.reshape(nzg, ny, nx)[sl].reshape(a1.shape)) < 1e-13
        assert relmax(p1, p_full.reshape(nzg, ny, nx)[sl].reshape(p1.shape)) < 1e-14
        dots.append(d1)
    want = float(np.vdot(p_full, want_ap))
    assert abs(sum(dots) - want) <= 1e-11 * abs(want)


def test_pass_a_range_rejects_bad_ranges(cuda_device):
    from paper_1904_03057_b200.errors import NativeLibraryError  # noqa: F401

    ext, p = (12, 12, 12), 3
    step = tuple(1.0 / (n - 1) for n in ext)
    data = build_system(BoxDomain(Grid(ext, step)), p, p, 0.01, 1.0, [])
    op = make_operator(data, "b200")
    lay, plan = op.layout, op.plan()
    r, q, o, ap = (lay.alloc(op.device) for _ in range(4))
    scratch = plan.scratch()
    for z0, cnt in [(-1, 2), (0, 0), (lay.nz - 1, 2)]:
        with pytest.raises(Exception, match="z range"):
            plan.cg_pass_a_range(o, r, q, o, ap, scratch, z0, cnt, False)


@pytest.mark.slow
@pytest.mark.parametrize("ncoef,p", [(930, 3), (512, 1), (512, 2), (512, 3), (512, 4), (512, 5)])
def test_full_size_windows_symmetry_and_true_residual(cuda_device, ncoef, p):
    """C3 at full size (930^3 coefficients, p = 3, lambda = 4) and the C4
    degree sweep (512^3, p = 1..5): the device apply of a random field
    against the oracle on output planes at both z ends and the middle (each
    plane spans the y/x edges) (<= 1e-13); <u,Av> = <Au,v>; and a heat
    step's PCG (tol 1e-10) checked through its true residual |b - A x| / |b|
    computed with the (window-verified) device apply."""
    import torch

    from paper_1904_03057_b200.solver import pcg_device
    from paper_1904_03057_b200.synthetic import IC, SOURCE, gaussian_coeffs, heat_c_inputs

    N, hh, dt = heat_c_inputs(ncoef, p)
    op = make_operator(heat_system(Grid((N,) * 3, (hh,) * 3), p, dt), "b200")
    ora = O.KronOperator((N,) * 3, (hh,) * 3, p, dt, 1.0)
    lay, dev = op.layout, op.device
    assert ora.cext == op.data.cext == (ncoef,) * 3
    gen = torch.Generator(device=dev).manual_seed(ncoef + p)
    u = lay.alloc(dev)
    lay.owned(u).copy_(torch.randn(lay.owned_shape, generator=gen, device=dev,
                                   dtype=torch.float64).reshape(lay.owned(u).shape))
    Au = lay.alloc(dev)
    op.apply_device(u, Au)
    torch.cuda.synchronize()
    own_u, own_Au = lay.owned(u), lay.owned(Au)
    for z0 in sorted({0, 1, 2, 5, ncoef // 2, ncoef - 3, ncoef - 1}):
        lo, hi = max(0, z0 - p), min(ncoef, z0 + p + 1)
        want = ora.apply_plane(own_u[lo:hi].cpu().numpy(), lo, z0)
        got = own_Au[z0].cpu().numpy()
        assert relmax(got, want) < 1e-13, z0
    v = lay.alloc(dev)
    lay.owned(v).copy_(1.0 + 0.1 * torch.randn(lay.owned_shape, generator=gen, device=dev,
                                               dtype=torch.float64).reshape(own_u.shape))
    Av = lay.alloc(dev)
    op.apply_device(v, Av)
    s1 = float((own_u * lay.owned(Av)).sum())
    s2 = float((own_Au * lay.owned(v)).sum())
    assert abs(s1 - s2) <= 1e-11 * max(abs(s1), 1.0), (s1, s2)
    del v, Av
    # one heat step: b = M u0 + dt M q, x0 = u0
    gaussian_coeffs(N, hh, p, device=dev, out=u, layout=lay, **IC)
    q = lay.alloc(dev)
    gaussian_coeffs(N, hh, p, device=dev, out=q, layout=lay, **SOURCE)
    F = lay.alloc(dev)
    op.mass_apply_device(q, F)
    b = lay.alloc(dev)
    op.mass_apply_device(u, b, F, a=dt)
    del q, F
    x = u.clone()
    rep = pcg_device(op, b, x, SolveConfig(tol=1e-10, max_iter=500), has_x0=True)
    assert rep.converged and rep.iterations <= 200, rep
    if (ncoef, p) == (930, 3):
        assert 10 <= rep.iterations <= 20, rep  # the bench's 14-15
    op.apply_device(x, Au)
    torch.cuda.synchronize()
    rt = torch.linalg.vector_norm(lay.owned(b) - own_Au) / torch.linalg.vector_norm(lay.owned(b))
    assert float(rt) < 2e-10, float(rt)
    del u, Au, b, x
    torch.cuda.empty_cache()


LARGE = [(256, 3), (512, 1), (512, 2), (512, 3), (512, 4), (512, 5), (930, 3)]


@pytest.mark.slow
@pytest.mark.parametrize("ncoef,p", LARGE)
def test_large_heat_step_vs_oracle_fixture(golden, cuda_device, ncoef, p):
    """C2 (256^3) and C4 (512^3, p = 1..5): heat step 1 (b = M u0 + dt F,
    x0 = u0) against the oracle recurrence run in the build container
    (tests/golden/make_large_golden.py): CG iteration counts within +-1 at
    tol 1e-10 and 1e-13 (BASELINE.json configs[1] / [3]; north_star), and at
    tol 1e-13 the coefficients within 1e-10 relative (||x|| and 4096 fixed
    sampled coefficients)."""
    import torch

    from paper_1904_03057_b200.solver import pcg_device
    from paper_1904_03057_b200.synthetic import IC, SOURCE, gaussian_coeffs, heat_c_inputs

    g = golden(f"large_{ncoef}_p{p}.npz")
    N, hh, dt = heat_c_inputs(ncoef, p)
    assert np.allclose(g["meta"], [ncoef, p, N, hh, dt], rtol=1e-15, atol=0)
    op = make_operator(heat_system(Grid((N,) * 3, (hh,) * 3), p, dt), "b200")
    lay, dev = op.layout, op.device
    idx = torch.from_numpy(g["idx"].astype(np.int64)).to(dev)

    def sample(buf):
        own = lay.owned(buf)
        return own[idx[:, 0], idx[:, 1], idx[:, 2]].cpu().numpy()

    u = lay.alloc(dev)
    gaussian_coeffs(N, hh, p, device=dev, out=u, layout=lay, **IC)
    assert relmax(sample(u), g["u0_sample"]) < 1e-13  # same inputs as the oracle run
    q = lay.alloc(dev)
    gaussian_coeffs(N, hh, p, device=dev, out=q, layout=lay, **SOURCE)
    F = lay.alloc(dev)
    op.mass_apply_device(q, F)
    del q
    b = lay.alloc(dev)
    op.mass_apply_device(u, b, F, a=dt)
    del F
    bn = float(torch.linalg.vector_norm(lay.owned(b)))
    # input check (the oracle run's b): <= 1e-13 at 256^3 / 512^3, 3.4e-13 at 930^3
    assert abs(bn - float(g["b_norm"])) <= 1e-12 * bn, (bn, float(g["b_norm"]))
    nmax = len(g["res_history"]) - 1  # the oracle run's last iteration
    final_tol = float(g["final_tol"]) if "final_tol" in g else 1e-13
    for tol, key in ((1e-10, "its_1e10"), (1e-13, "its_1e13")):
        if tol < final_tol:
            continue  # C3: the oracle ran to 1e-10 only (host-memory / time bound)
        x = u.clone()
        want = int(g[key])
        rep = pcg_device(op, b, x, SolveConfig(tol=tol, max_iter=nmax if want < 0 else 5000),
                         has_x0=True)
        if want < 0:  # the oracle stopped at its cap before tol (p >= 4 at 1e-13)
            assert rep.iterations == nmax
        else:
            assert abs(rep.iterations - want) <= 1, (tol, rep.iterations, want)
    # the final coefficients: 1e-10 at tol 1e-13; at tol
    # 1e-10 two correct solvers drift ~kappa * tol apart (C3 bar 1e-7)
    bar = 1e-10 if final_tol <= 1e-13 else 1e-7
    xs, xo = sample(x), g["x_sample"]
    assert np.linalg.norm(xs - xo) / np.linalg.norm(xo) < bar
    xn = float(torch.linalg.vector_norm(lay.owned(x)))
    assert abs(xn - float(g["x_norm"])) <= bar * xn
    del x, u, b
    torch.cuda.empty_cache()


@pytest.mark.parametrize("p,ext", [(1, (14, 15, 16)), (2, (17, 13, 20)), (3, (40, 50, 70)),
                                   (4, (19, 18, 17)), (5, (22, 21, 23))])
def test_fused_heat_residual_matches_rhs_then_residual(cuda_device, p, ext):
    """bspde_heat_residual (RHS fused into the first residual, b never
    stored) equals bspde_mass_apply + bspde_cg_residual bit for bit: r0 and
    the three initial sums (<b,b>, <r,D^-1 r>, <r,r>)."""
    import torch

    step = tuple(1.0 / (n - 1) for n in ext)
    dt = 4 * min(step) ** 2
    op = make_operator(heat_system(Grid(ext, step), p, dt), "b200")
    lay, plan, dev = op.layout, op.plan(), op.device
    rng = np.random.default_rng(p)
    u = lay.upload(rng.normal(size=op.data.cext), dev)
    F = lay.upload(rng.normal(size=op.data.cext), dev)
    outs = []
    for fused in (False, True):
        r = lay.alloc(dev)
        scratch = plan.scratch()
        plan.cg_setup(scratch, None, 1e-300, 10, False, True)
        if fused:
            plan.heat_residual(u, F, op.data.vol, dt, r, scratch, 1)
        else:
            b = lay.alloc(dev)
            op.mass_apply_device(u, b, F, a=dt)
            plan.cg_residual(b, u, r, scratch, 1)
        torch.cuda.synchronize()
        outs.append((lay.download(r), scratch[:24].cpu().numpy().view(np.float64).copy()))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])
