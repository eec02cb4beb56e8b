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
    # a variable field selects the assembled-stencil operator (varcoef.py)
    from paper_1904_03057_b200.varcoef import VarSystemData

    assert isinstance(build_system(dom, 3, 3, f, np.full(shp, 2.0), []), VarSystemData)
    assert len(build_system(dom, 3, 3, f, np.full(shp, 2.0), [(0, 0, 1.0, None)]).faces) == 1
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


def test_transforms_need_the_gpu():
    """The product transforms run on the GPU only (no CPU fallback); degree
    <= 1 needs no prefilter and constants stay exact on the host."""
    import torch

    from paper_1904_03057_b200.errors import NativeLibraryError

    assert direct_transform(np.ones((5, 5)), 1).shape == (5, 5)
    g = Grid((5, 5, 5), (0.25,) * 3)
    assert np.all(transform_field(2.5, g, 3) == 2.5)
    if not torch.cuda.is_available():
        with pytest.raises(NativeLibraryError):
            direct_transform(np.ones((5, 5)), 3)
        with pytest.raises(NativeLibraryError):
            sample_solution(np.ones((7, 7, 7)), g, 3)
