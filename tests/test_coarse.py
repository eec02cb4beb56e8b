"""Steady pipeline with coarse-grid initialisation against reference fixtures
(tests/golden/coarse.npz, make_golden.py ``coarse``; problem.py:374-482)."""

import os

import numpy as np
import pytest

from paper_1904_03057_b200.domain import BoxDomain, Grid, MaskDomain

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "coarse.npz"))


def specs():
    from paper_1904_03057_b200.boundary import DirichletPenalty, Robin
    from paper_1904_03057_b200.problem import ProblemSpec

    g1 = Grid((13, 14, 31), (1.0, 1.0, 1.0))
    g2 = Grid((11, 12, 13), (0.1, 0.08, 0.12))
    zz, yy, xx = np.meshgrid(*[g2.node_coordinates(a) for a in range(3)], indexing="ij")
    g3 = Grid((21, 17), (0.05, 0.06))
    yy2, xx2 = np.meshgrid(*[g3.node_coordinates(a) for a in range(2)], indexing="ij")
    return {
        "c2d": (ProblemSpec(domain=BoxDomain(g3), basis_degree=2, diffusion=0.8, absorption=1.0,
                            source=np.cos(3 * xx2) + yy2, bc={"all": DirichletPenalty(1.0, 1e-3)}),
                3),
        "c1": (ProblemSpec(domain=MaskDomain(g1, GOLD["c1_mask"]), basis_degree=1, diffusion=0.5,
                           absorption=0.0, source=GOLD["c1_src"],
                           bc=DirichletPenalty(20.0, 1e-3)), 3),
        "c3": (ProblemSpec(domain=BoxDomain(g2), basis_degree=3,
                           diffusion=1.0 + 0.3 * np.sin(4 * xx) * np.cos(3 * yy),
                           absorption=0.5 + zz, source=np.exp(-(xx - .5) ** 2 - yy),
                           bc=Robin(0.7)), 2),
    }


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


def test_spec_validation():
    from paper_1904_03057_b200.errors import ConfigurationError, ValidationError
    from paper_1904_03057_b200.problem import ProblemSpec

    g = Grid((6, 6, 6), (1.0, 1.0, 1.0))
    with pytest.raises(ValidationError):
        ProblemSpec(domain=BoxDomain(Grid((3, 3, 3), (1.0, 1.0, 1.0))), basis_degree=5)
    with pytest.raises(ValidationError):
        ProblemSpec(domain=BoxDomain(g), basis_degree=3, precision="f16")
    with pytest.raises(ConfigurationError):
        ProblemSpec(domain=BoxDomain(g), basis_degree=3, precision="f32")
    s = ProblemSpec(domain=BoxDomain(g), basis_degree=3)
    assert s.param_degree == 3 and s.source_degree == 3 and s.default_epsilon() == 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["c1", "c3", "c2d"])
def test_coarse_initialize_matches_reference(tag):
    from paper_1904_03057_b200.problem import coarse_initialize

    spec, factor = specs()[tag]
    x0, info = coarse_initialize(spec, factor)
    assert tuple(info["coarse_extents"]) == tuple(GOLD[f"{tag}_coarse_ext"])
    assert abs(info["coarse_iterations"] - int(GOLD[f"{tag}_coarse_its"][0])) <= 1
    # coarse solve to tol 1e-8: rounding differences scale with kappa * tol
    assert rel(x0, GOLD[f"{tag}_x0"]) <= 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["c1", "c3", "c2d"])
def test_solve_problem_with_coarse_init(tag):
    from paper_1904_03057_b200.problem import solve_problem
    from paper_1904_03057_b200.solver import SolveConfig

    spec, factor = specs()[tag]
    its_ref, its_ref0 = (int(v) for v in GOLD[f"{tag}_its"])
    sol = solve_problem(spec, SolveConfig(tol=1e-9, max_iter=4000, coarse_init_factor=factor))
    assert sol.report.converged
    # c2d (penalty weight 1e3 on every face) stops in a residual plateau: the
    # reference itself takes 94 or 96 iterations when its dot products are
    # perturbed by one rounding unit (5 of 6 seeds give 96;
    # tools/count_sensitivity.py c2d), so its bar is +-2
    bar = 2 if tag == "c2d" else max(1, its_ref // 100)
    assert abs(sol.report.iterations - its_ref) <= bar
    assert rel(sol.coeffs, GOLD[f"{tag}_coeffs"]) <= 1e-6
    assert rel(sol.samples, GOLD[f"{tag}_samples"]) <= 1e-6
    sol0 = solve_problem(spec, SolveConfig(tol=1e-9, max_iter=4000))
    assert abs(sol0.report.iterations - its_ref0) <= max(1, its_ref0 // 100)


IND = np.load(os.path.join(os.path.dirname(__file__), "golden", "indirect.npz"))


@pytest.mark.gpu
@pytest.mark.parametrize("tag", sorted({k.rsplit("_", 1)[0] for k in IND.keys()}))
def test_indirect_transform_matches_reference(tag):
    from paper_1904_03057_b200.transform import indirect_transform

    meta = IND[f"{tag}_meta"]
    first = IND[f"{tag}_first"]
    vals = indirect_transform(IND[f"{tag}_c"], int(meta[0]), IND[f"{tag}_pts"],
                              str(IND[f"{tag}_ext"][0]),
                              tuple(int(v) for v in first) if first.size else None,
                              step=tuple(meta[1:]))
    assert np.abs(vals - IND[f"{tag}_vals"]).max() <= 1e-13 * max(1.0, np.abs(IND[f"{tag}_vals"]).max())


def test_indirect_transform_rejects_points_outside_the_span():
    from paper_1904_03057_b200.errors import OutOfDomainError
    from paper_1904_03057_b200.transform import lattice_taps

    with pytest.raises(OutOfDomainError):
        lattice_taps(3, 0.5, np.array([0.0, 4.6]), 10)


@pytest.mark.parametrize("k", range(4))
def test_coarsen_mask_matches_reference(k):
    from paper_1904_03057_b200.problem import _coarsen_mask

    want = GOLD[f"cm{k}_coarse"]
    got = _coarsen_mask(GOLD[f"cm{k}_fine"], Grid(tuple(c + 1 for c in want.shape),
                                                  (1.0,) * want.ndim))
    assert np.array_equal(got, want)


L2 = np.load(os.path.join(os.path.dirname(__file__), "golden", "l2.npz"))


@pytest.mark.gpu
@pytest.mark.parametrize("tag", sorted({k.rsplit("_", 1)[0] for k in L2.keys()}))
def test_l2_prefilter_matches_reference(tag):
    from paper_1904_03057_b200.transform import transform_field

    meta = L2[f"{tag}_meta"]
    deg, dim = int(meta[0]), int(meta[1])
    shape = tuple(int(v) for v in meta[2:2 + dim])
    grid = Grid(shape, tuple(0.1 * (a + 1) for a in range(dim)))
    got = transform_field(L2[f"{tag}_samples"], grid, deg, prefilter="l2")
    # the folded Gram of the sampled beta^(2n+1) has condition 47 (n = 4) and
    # 116 (n = 5) per axis: pivoted LAPACK (reference) and the banded LU differ
    # by ~eps * cond^dim there
    assert rel(got, L2[f"{tag}_coeffs"]) <= (1e-13 if deg <= 3 else 1e-10)


def test_l2_factors_reject_short_lines():
    from paper_1904_03057_b200.errors import ValidationError
    from paper_1904_03057_b200.transform import l2_factors

    with pytest.raises(ValidationError):
        l2_factors(5, 5)
