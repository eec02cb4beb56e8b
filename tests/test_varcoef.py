"""Variable-coefficient operator: host setup (CPU) and GPU parity vs the
reference (tests/golden/varcoef.npz from make_golden.py: var_cases)."""

import numpy as np
import pytest

from paper_1904_03057_b200 import BoxDomain, Grid, SolveConfig, build_system, make_operator, pcg
from paper_1904_03057_b200.gram import basis_extension, edge_width, trilinear_tables
from paper_1904_03057_b200.varcoef import VarSystemData

TAGS = ["v1", "v2", "v3", "v4", "v5", "v3p2", "v2p5", "v3f", "v2f", "v3p0", "v1p0"]
# v4, v5 stop at max_iter in the reference
CONVERGED = ["v1", "v2", "v3", "v3p2", "v2p5", "v3f", "v2f", "v3p0", "v1p0"]


def case(golden, tag):
    g = golden("varcoef.npz")
    meta = g[f"{tag}_meta"]
    nb, npar = int(meta[0]), int(meta[1])
    step = tuple(float(v) for v in meta[2:5])
    ext = tuple(int(v) for v in meta[5:8])
    return g, nb, npar, step, ext


def relmax(a, b):
    return float(np.abs(np.asarray(a) - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("tag", TAGS)
def test_trilinear_tables_vs_reference_bands(golden, tag):
    g, nb, npar, step, ext = case(golden, tag)
    ew = edge_width(nb)
    n = ext[2] + 2 * basis_extension(nb)
    for d in (0, 1):
        T = trilinear_tables(nb, npar, d)
        assert np.abs(T[ew] - g[f"{tag}_band{d}_interior"]).max() < 1e-15
        for pos, tab in zip(g[f"{tag}_band{d}_pos"], g[f"{tag}_band{d}_edges"]):
            c = pos if pos < ew else 2 * ew - (n - 1 - pos)
            assert np.abs(T[c] - tab).max() < 1e-15, (d, pos)


def test_variable_fields_build_var_system():
    dom = BoxDomain(Grid((9, 10, 11), (0.5, 1.0, 0.25)))
    shp = (11, 12, 13)
    d = build_system(dom, 3, 3, 1.0 + np.random.default_rng(0).random(shp), 1.0, [])
    assert isinstance(d, VarSystemData) and d.cext == (11, 12, 13)
    assert d.mfield.shape == shp and np.all(d.mfield == 1.0)
    df = build_system(dom, 3, 3, 1.0 + np.random.default_rng(0).random(shp), 1.0,
                      [(0, 0, 1.0, 2.0)])
    assert len(df.faces) == 1 and df.face_rhs().shape == d.cext
    d2 = build_system(BoxDomain(Grid((9, 10), (0.5, 1.0))), 3, 3,
                      1.0 + np.random.default_rng(0).random((11, 12)), 1.0, [])
    assert isinstance(d2, VarSystemData) and d2.cext == (11, 12)  # 2-D: unit leading axis


def _op(golden, tag):
    g, nb, npar, step, ext = case(golden, tag)
    specs = [(int(a), int(s), float(w), None if np.isnan(v) else float(v))
             for a, s, w, v in g.get(f"{tag}_faces", np.zeros((0, 4)))]
    data = build_system(BoxDomain(Grid(ext, step)), nb, npar, g[f"{tag}_D"], g[f"{tag}_mu"], specs)
    return g, make_operator(data, "b200")


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_varcoef_apply_and_diagonal_vs_reference(golden, cuda_device, tag):
    g, op = _op(golden, tag)
    assert relmax(op.apply(g[f"{tag}_c"]), g[f"{tag}_t"]) < 1e-13
    assert relmax(op.jacobi_diagonal(), g[f"{tag}_diag"]) < 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("tag", CONVERGED)
def test_varcoef_pcg_vs_reference(golden, cuda_device, tag):
    g, op = _op(golden, tag)
    x, rep = pcg(op, g[f"{tag}_b"], SolveConfig(tol=1e-12, max_iter=5000))
    ref_its = int(g[f"{tag}_its"][0])
    assert rep.converged
    # +-1 at ~100 iterations; these take 84-644: +-max(1, 0.5%)
    assert abs(rep.iterations - ref_its) <= max(1, round(0.005 * ref_its)), (rep.iterations, ref_its)
    ref = g[f"{tag}_x"]
    assert np.linalg.norm(x - ref) / np.linalg.norm(ref) < 1e-9


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["v3f", "v2f"])
def test_varcoef_face_rhs_vs_reference(golden, cuda_device, tag):
    from paper_1904_03057_b200 import assembled_rhs

    g, op = _op(golden, tag)
    t = assembled_rhs(op.data, op.data.n_b, np.zeros(op.data.cext))
    assert relmax(t, g[f"{tag}_facerhs"]) < 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["heatvar", "heatvarf"])
def test_heat_with_variable_conductivity_vs_reference(golden, cuda_device, tag):
    """HeatSolver with conductivity = kappa(x) (assembled-stencil solve, box
    mass RHS) against the reference composition, 2 steps at tol 1e-12."""
    from paper_1904_03057_b200 import (DirichletPenalty, HeatProblem, HeatSolver, Neumann, Robin,
                                       realize_bc)

    g = golden("varcoef.npz")
    p, n, dt = int(g[f"{tag}_meta"][0]), int(g[f"{tag}_meta"][1]), float(g[f"{tag}_meta"][2])
    grid = Grid((n,) * 3, (1.0 / (n - 1),) * 3)
    bc = None
    if tag == "heatvarf":  # the fixture's (0, 0, 50, 1.0), (2, 1, 0.5, None)
        bc = {"all": Neumann(), "x0": DirichletPenalty(1.0, epsilon=0.02), "z1": Robin(1.0)}
        specs = [(int(a), int(s_), float(w), None if np.isnan(v) else float(v))
                 for a, s_, w, v in g[f"{tag}_faces"]]
        assert realize_bc(bc, grid) == specs
    prob = HeatProblem(grid, p, dt, conductivity=g[f"{tag}_kappa"], bc=bc,
                       initial_coeffs=g[f"{tag}_u0"], source_coeffs=g[f"{tag}_q"])
    hs = HeatSolver(prob, SolveConfig(tol=1e-12, max_iter=5000))
    assert hs.sop is not None
    its = [hs.step().iterations for _ in range(2)]
    ref_its = [int(v) for v in g[f"{tag}_its"]]
    assert all(abs(a - b) <= max(1, round(0.005 * b)) for a, b in zip(its, ref_its)), (its, ref_its)
    ref = g[f"{tag}_u"][-1]
    # rounding drift between two correct solvers ~ kappa * tol: the penalty
    # face makes heatvarf much worse conditioned (~750 iterations)
    bar = 1e-8 if tag == "heatvarf" else 1e-9
    assert np.linalg.norm(hs.coefficients() - ref) / np.linalg.norm(ref) < bar


@pytest.mark.gpu
@pytest.mark.parametrize("p,ext", [(1, (40, 33, 35)), (2, (37, 41, 30)), (3, (64, 48, 72))])
def test_otf_matches_assembled_stencil(cuda_device, monkeypatch, p, ext):
    """The matrix-free operator (otf.cuh: the reference's on-the-fly
    algorithm, nothing stored) against the assembled stencil (stencil.cuh):
    two independent device implementations of the same variable-coefficient
    operator; apply <= 1e-13, Jacobi diagonal <= 1e-14, PCG counts +-1 and
    solutions 1e-10 at tol 1e-13.  Sizes with several x-y tiles, ragged
    tiles and every edge class."""
    import torch

    from paper_1904_03057_b200.gram import basis_extension

    step = tuple(1.0 / (n - 1) for n in ext)
    pe = [n + 2 * basis_extension(p) for n in ext]
    z, y, x = (np.linspace(0, 1, n) for n in pe)
    D = 0.01 * (1.0 + 0.5 * np.sin(3 * z)[:, None, None] * np.cos(2 * y)[None, :, None]
                * (1 + x[None, None, :]))
    mu = 1.0 + 0.2 * np.cos(5 * z)[:, None, None] * np.sin(2 * y + 1)[None, :, None] \
        * np.ones((1, 1, pe[2]))
    data = build_system(BoxDomain(Grid(ext, step)), p, p, D, mu, [])
    ops = {}
    for kind in ("otf", "stencil"):
        monkeypatch.setenv("BSPDE_VAR_STRATEGY", kind)
        ops[kind] = make_operator(data, "b200")
        assert ops[kind].kind == kind
    c = np.random.default_rng(p).normal(size=data.cext)
    t_o, t_s = ops["otf"].apply(c), ops["stencil"].apply(c)
    assert relmax(t_o, t_s) < 1e-13
    assert relmax(ops["otf"].jacobi_diagonal(), ops["stencil"].jacobi_diagonal()) < 1e-14
    b = ops["stencil"].apply(np.cos(np.linspace(0, 3, c.size)).reshape(c.shape))
    res = {k: pcg(op, b, SolveConfig(tol=1e-13, max_iter=3000)) for k, op in ops.items()}
    (xo, ro), (xs, rs) = res["otf"], res["stencil"]
    assert ro.converged and rs.converged
    assert abs(ro.iterations - rs.iterations) <= 1, (ro.iterations, rs.iterations)
    assert np.linalg.norm(xo - xs) / np.linalg.norm(xs) < 1e-10
    torch.cuda.empty_cache()


def test_otf_strategy_selection(monkeypatch):
    """Matrix-free for 3-D boxes without faces and n_b = n_p <= 3; the
    assembled stencil otherwise (faces, other degrees, 1-D / 2-D, masks)."""
    import ctypes as C

    from paper_1904_03057_b200 import varcoef

    class Lib:
        def __init__(self, ok):
            self.ok = ok

        def bspde_otf_supported(self, h):
            return self.ok

    class D:
        mask = None

    assert varcoef._var_strategy(D(), Lib(1), C.c_void_p()) == "otf"
    assert varcoef._var_strategy(D(), Lib(0), C.c_void_p()) == "stencil"
    monkeypatch.setenv("BSPDE_VAR_STRATEGY", "stencil")
    assert varcoef._var_strategy(D(), Lib(1), C.c_void_p()) == "stencil"
    monkeypatch.setenv("BSPDE_VAR_STRATEGY", "otf")
    from paper_1904_03057_b200.errors import ConfigurationError
    with pytest.raises(ConfigurationError):
        varcoef._var_strategy(D(), Lib(0), C.c_void_p())
    m = D()
    m.mask = object()
    monkeypatch.setenv("BSPDE_VAR_STRATEGY", "auto")
    assert varcoef._var_strategy(m, Lib(1), C.c_void_p()) == "stencil"
