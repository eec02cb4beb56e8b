"""Box-face Robin / penalty terms: host setup, oracle pinning, BC realization.

Golden fixtures (tests/golden/faces.npz) come from the reference's
build_system(face_specs) + OnTheFlyOperator / assembled_rhs
(make_golden.py: face_cases).  GPU parity lives in test_parity_gpu.py.
"""

import numpy as np
import pytest

from oracle import bspde_oracle as O
from paper_1904_03057_b200 import (BoxDomain, DirichletPenalty, Grid, Neumann, Robin,
                                   build_system, heat_system, realize_bc)
from paper_1904_03057_b200.errors import ConfigurationError, ValidationError

TAGS = ["p1", "p2", "p3", "p4", "p5", "p3_all", "p2_2d", "p3_1d"]


def case(golden, tag):
    g = golden("faces.npz")
    meta = g[f"{tag}_meta"]
    p, D, mu = int(meta[0]), float(meta[1]), float(meta[2])
    d = (len(meta) - 3) // 2
    step = tuple(float(v) for v in meta[3:3 + d])
    ext = tuple(int(v) for v in meta[3 + d:])
    specs = [(int(a), int(s), float(w), None if np.isnan(v) else float(v))
             for a, s, w, v in g[f"{tag}_faces"]]
    return g, p, D, mu, step, ext, specs


def relmax(a, b):
    return float(np.abs(np.asarray(a) - b).max() / max(np.abs(b).max(), 1e-300))


def dense_apply(data, c):
    """A c from this build's class tables (CPU, small sizes): the operator the
    kernels realize, with the face terms folded into the stiffness factors."""
    mats_m = [f.dense() for f in data.mass]
    mats_k = [f.dense() for f in data.stiff]
    c3 = np.asarray(c, dtype=float).reshape(data.dims3)

    def kron(mats, x):
        for ax, m in enumerate(mats):
            x = np.moveaxis(np.tensordot(m, np.moveaxis(x, ax, 0), axes=1), 0, ax)
        return x

    out = data.c_mass * kron(mats_m, c3)
    for a in range(3):
        if data.c_stiff[a] != 0.0:
            out = out + data.c_stiff[a] * kron([mats_k[b] if b == a else mats_m[b]
                                                for b in range(3)], c3)
    return out.reshape(data.cext)


@pytest.mark.parametrize("tag", TAGS)
def test_oracle_faces_vs_reference(golden, tag):
    g, p, D, mu, step, ext, specs = case(golden, tag)
    ora = O.KronOperator(ext, step, p, D, mu, faces=specs)
    assert relmax(ora.apply(g[f"{tag}_c"]), g[f"{tag}_t"]) < 1e-13
    assert relmax(ora.jacobi_diagonal(), g[f"{tag}_diag"]) < 1e-13
    rhs = ora.mass_apply(g[f"{tag}_q"]) + ora.face_rhs()
    assert relmax(rhs, g[f"{tag}_rhs"]) < 1e-13
    assert relmax(ora.face_rhs(), g[f"{tag}_facerhs"]) < 1e-13


@pytest.mark.parametrize("tag", TAGS)
def test_host_face_folding_vs_reference(golden, tag):
    """Class tables with the faces folded into K (what the kernels get)."""
    g, p, D, mu, step, ext, specs = case(golden, tag)
    data = build_system(BoxDomain(Grid(ext, step)), p, p, D, mu, specs)
    assert len(data.faces) == len(specs)
    assert relmax(dense_apply(data, g[f"{tag}_c"]), g[f"{tag}_t"]) < 1e-13
    assert relmax(data.expand_table(data.diag_table()), g[f"{tag}_diag"]) < 1e-13
    assert relmax(data.face_rhs(), g[f"{tag}_facerhs"]) < 1e-13


def test_faces_only_touch_edge_classes():
    grid = Grid((12, 12, 12), (0.1,) * 3)
    a = build_system(BoxDomain(grid), 3, 3, 0.5, 1.0, [])
    b = build_system(BoxDomain(grid), 3, 3, 0.5, 1.0, [(1, 0, 7.0, 1.0), (2, 1, 3.0, None)])
    for ax in range(3):
        ta, tb = a.stiff[ax].table, b.stiff[ax].table
        ew = a.stiff[ax].ew
        assert np.array_equal(ta[ew], tb[ew])  # interior taps unchanged
        changed = not np.array_equal(ta, tb)
        assert changed == (ax in (1, 2))
    assert np.array_equal(b.mass[1].table, a.mass[1].table)


def test_face_spec_validation():
    dom = BoxDomain(Grid((9, 9, 9), (0.1,) * 3))
    with pytest.raises(ValidationError):
        build_system(dom, 3, 3, 0.5, 1.0, [(3, 0, 1.0, None)])
    with pytest.raises(ValidationError):
        build_system(dom, 3, 3, 0.5, 1.0, [(0, 2, 1.0, None)])
    with pytest.raises(ValidationError):
        build_system(dom, 3, 3, 0.5, 1.0, [(0, 0, float("nan"), None)])
    with pytest.raises(ConfigurationError):  # faces ride on the diffusion factors
        build_system(dom, 3, 3, 0.0, 1.0, [(0, 0, 1.0, None)])


def test_realize_bc_rules():
    grid = Grid((5, 6, 7), (0.1, 0.2, 0.3))
    specs = realize_bc({"all": DirichletPenalty(20.0), "x0": Robin(0.5), "z1": Neumann()}, grid)
    assert specs[0] == (0, 0, 1.0, None)
    eps = 1e-4 * 0.1
    assert specs[1] == (0, 1, 1.0 / eps, 20.0)
    assert (2, 1) not in [(a, s) for a, s, _, _ in specs]
    assert len(specs) == 5
    assert realize_bc(Neumann(), grid) == []
    assert realize_bc(DirichletPenalty(1.0, epsilon=0.5), Grid((5, 5), (1.0, 1.0))) == [
        (0, 0, 2.0, 1.0), (0, 1, 2.0, 1.0), (1, 0, 2.0, 1.0), (1, 1, 2.0, 1.0)]
    with pytest.raises(ConfigurationError):
        realize_bc({"x0": Robin()}, grid)  # missing faces
    with pytest.raises(ConfigurationError):
        realize_bc({"all": Neumann(), "w0": Neumann()}, grid)
    with pytest.raises(ConfigurationError):
        realize_bc(Robin(gamma=0.0), grid)
    with pytest.raises(ConfigurationError):
        realize_bc(DirichletPenalty(1.0, epsilon=-1.0), grid)

    class Spec:  # the reference's ProblemSpec shape
        bc = Robin(2.0)
    Spec.grid = grid
    assert realize_bc(Spec())[0] == (0, 0, 0.25, None)


def test_heat_system_scales_face_weights_by_dt():
    grid = Grid((10, 10, 10), (0.1,) * 3)
    specs = [(0, 0, 4.0, 2.0)]
    d = heat_system(grid, 3, 0.01, face_specs=specs)
    assert d.faces[0].weight == pytest.approx(0.04)
    assert d.faces[0].rhs_weight == pytest.approx(0.08)
