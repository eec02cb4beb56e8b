"""Host-side system setup (class tables, scales, transforms) vs oracle/golden."""

import numpy as np
import pytest

from oracle import bspde_oracle as O
from paper_1904_03057_b200 import (BoxDomain, ConfigurationError, Grid, ValidationError,
                                   build_system, heat_system)
from paper_1904_03057_b200.transform import direct_transform, sample_solution, transform_field


def kron_from_system(data):
    """Assemble A from the product's class tables (host, small sizes)."""
    mats = []
    for a in range(3):
        mats.append((data.mass[a].dense(), data.stiff[a].dense()))
    (Mz, Kz), (My, Ky), (Mx, Kx) = mats
    A = data.c_mass * np.kron(np.kron(Mz, My), Mx)
    A += data.c_stiff[0] * np.kron(np.kron(Kz, My), Mx)
    A += data.c_stiff[1] * np.kron(np.kron(Mz, Ky), Mx)
    A += data.c_stiff[2] * np.kron(np.kron(Mz, My), Kx)
    return A


@pytest.mark.parametrize("p,ext,step", [(1, (5, 6, 7), (0.5, 1.0, 0.25)),
                                        (3, (6, 7, 8), (0.5, 1.0, 0.25)),
                                        (5, (8, 9, 8), (1.0, 0.5, 2.0)),
                                        (2, (9, 7), (0.5, 0.25)),
                                        (3, (11,), (0.3,))])
def test_system_tables_match_oracle(p, ext, step):
    D, mu = 0.37, 1.3
    data = build_system(BoxDomain(Grid(ext, step)), p, p, D, mu, [])
    ora = O.KronOperator(ext, step, p, D, mu)
    A = kron_from_system(data)
    Ad = ora.dense().toarray()
    assert np.abs(A - Ad).max() / np.abs(Ad).max() < 1e-14
    diag = data.expand_table(data.diag_table())
    np.testing.assert_allclose(diag, ora.jacobi_diagonal(), rtol=1e-14)
    inv = data.expand_table(data.inv_diag_table())
    np.testing.assert_allclose(inv, 1.0 / ora.jacobi_diagonal(), rtol=1e-14)
    assert np.all(data.expand_table(data.inv_diag_table("none")) == 1.0)


def test_constant_field_detection():
    dom = BoxDomain(Grid((8, 8, 8), (1.0,) * 3))
    shp = (10, 10, 10)
    data = build_system(dom, 3, 3, np.full(shp, 0.5), np.full(shp, 2.0), [])
    assert data.diffusion == 0.5 and data.absorption == 2.0
    f = np.full(shp, 0.5)
    f[3, 3, 3] = 0.6
    with pytest.raises(ConfigurationError):
        build_system(dom, 3, 3, f, np.full(shp, 2.0), [])
    # box-face terms are realized (tests/test_faces.py)
    assert len(build_system(dom, 3, 3, 1.0, 1.0, [(0, 0, 1.0, None)]).faces) == 1
    with pytest.raises(ValidationError):
        build_system(dom, 6, 3, 1.0, 1.0, [])


def test_heat_system_scales():
    g = Grid((20, 20, 20), (1 / 19,) * 3)
    dt = 4 / 19 ** 2
    d = heat_system(g, 3, dt)
    vol = (1 / 19) ** 3
    assert d.c_mass == pytest.approx(vol)
    assert d.c_stiff[0] == pytest.approx(vol * dt * 19 ** 2)


def test_transform_matches_reference(golden):
    h = golden("heat16.npz")
    p, N, hh = int(h["meta"][0]), int(h["meta"][1]), h["meta"][2]
    g = Grid((N,) * 3, (hh,) * 3)
    u0 = transform_field(lambda x, y, z: np.exp(-40 * ((x - .5) ** 2 + (y - .4) ** 2 +
                                                       (z - .6) ** 2)), g, p)
    np.testing.assert_allclose(u0, h["u0"], rtol=0, atol=1e-14)
    s = sample_solution(u0, g, p)
    x = g.node_coordinates(0)
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    np.testing.assert_allclose(s, np.exp(-40 * ((X - .5) ** 2 + (Y - .4) ** 2 + (Z - .6) ** 2)),
                               atol=1e-10)
    assert direct_transform(np.ones((5, 5)), 1).shape == (5, 5)
