"""1-D / 2-D variable-coefficient boxes and masks through the stencil
operator (unit leading axes) against reference fixtures
(tests/golden/lowdim.npz, make_golden.py ``lowdim``)."""

import os

import numpy as np
import pytest

from paper_1904_03057_b200.domain import BoxDomain, Grid, MaskDomain

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "lowdim.npz"))
G2 = Grid((14, 15), (0.5, 0.25))
CASES = {
    "b2v": (lambda: BoxDomain(Grid((13, 11), (0.3, 0.5))), 3, 2,
            [(0, 0, 0.7, None), (1, 1, 5.0, 1.5)]),
    "b1v": (lambda: BoxDomain(Grid((17,), (0.2,))), 2, 1, [(0, 1, 2.0, 0.5)]),
    "m2d": (lambda: MaskDomain(G2, GOLD["m2d_mask"]), 2, 1, [(0, 0, 3.0, 1.0)]),
    "m2d3": (lambda: MaskDomain(G2, GOLD["m2d3_mask"]), 3, 0, []),
    "m1d": (lambda: MaskDomain(Grid((17,), (0.25,)), GOLD["m1d_mask"]), 1, 1,
            [(0, 0, 2.0, 0.5)]),
}


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def _data(tag):
    from paper_1904_03057_b200 import build_system

    dom, nb, npar, specs = CASES[tag]
    return build_system(dom(), nb, npar, GOLD[f"{tag}_D"], GOLD[f"{tag}_mu"], specs)


def test_low_dim_systems_build_on_cpu():
    for tag in CASES:
        data = _data(tag)
        assert data.cext == GOLD[f"{tag}_c"].shape


@pytest.mark.gpu
@pytest.mark.parametrize("tag", list(CASES))
def test_apply_diag_rhs_pcg(tag):
    from paper_1904_03057_b200 import assembled_rhs, make_operator, pcg
    from paper_1904_03057_b200.solver import SolveConfig

    data = _data(tag)
    op = make_operator(data, "b200")
    assert rel(op.apply(GOLD[f"{tag}_c"]), GOLD[f"{tag}_t"]) <= 1e-13
    assert rel(op.jacobi_diagonal(), GOLD[f"{tag}_diag"]) <= 1e-14
    assert rel(assembled_rhs(data, data.n_b, GOLD[f"{tag}_q"]), GOLD[f"{tag}_rhs"]) <= 1e-13
    x, rep = pcg(op, GOLD[f"{tag}_b"], SolveConfig(tol=1e-10, max_iter=4000))
    its = int(GOLD[f"{tag}_its"][0])
    assert rep.converged and abs(rep.iterations - its) <= max(1, its // 100)
    assert rel(x, GOLD[f"{tag}_x"]) <= 1e-7


@pytest.mark.gpu
def test_heat_steps_on_2d_mask():
    from paper_1904_03057_b200 import DirichletPenalty, HeatProblem, HeatSolver
    from paper_1904_03057_b200.solver import SolveConfig

    prob = HeatProblem(grid=G2, degree=2, dt=0.02, conductivity=GOLD["heat2d_kappa"],
                       initial_coeffs=GOLD["heat2d_u0"], source_coeffs=GOLD["heat2d_q"],
                       bc=DirichletPenalty(1.0, 1.0 / 40.0), mask=GOLD["m2d_mask"])
    hs = HeatSolver(prob, SolveConfig(tol=1e-12, max_iter=5000))
    for k, its in enumerate(GOLD["heat2d_its"]):
        rep = hs.step()
        assert rep.converged and abs(rep.iterations - int(its)) <= max(1, int(its) // 100)
        assert rel(hs.coefficients(), GOLD["heat2d_u"][k]) <= 1e-9
