"""Host setup: exact 1-D Gram factors vs the reference (golden) and KATs."""

import numpy as np
import pytest

from paper_1904_03057_b200.errors import ValidationError
from paper_1904_03057_b200.gram import (basis_extension, edge_width, gram_factor,
                                        min_axis_length, product_integral)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("N", ["small", 12])
def test_gram_matches_reference(golden, p, N):
    g = golden("gram.npz")
    N = p + 6 if N == "small" else N
    M = gram_factor(p, N, "mass").dense()
    K = gram_factor(p, N, "stiff").dense()
    np.testing.assert_allclose(M, g[f"M_p{p}_N{N}"], rtol=0, atol=2e-16)
    np.testing.assert_allclose(K, g[f"K_p{p}_N{N}"], rtol=0, atol=5e-16)


def test_p3_known_values():
    # SURVEY.md §8(a) known-answer rows (reference, unit step)
    M = gram_factor(3, 12, "mass").dense()
    K = gram_factor(3, 12, "stiff").dense()
    np.testing.assert_allclose(M[3, 0:7], np.array([1, 120, 1191, 2416, 1191, 120, 1]) / 5040,
                               rtol=1e-15)
    np.testing.assert_allclose(K[3, 0:7], np.array([-1, -24, -15, 80, -15, -24, -1]) / 120,
                               rtol=1e-15, atol=1e-17)
    np.testing.assert_allclose(M[0, 0:4], [0.00396825396825397, 0.02559523809523809,
                                           0.0119047619047619, 0.0001984126984127], rtol=1e-13)
    np.testing.assert_allclose(M[2, 0:6], [0.011904761904761902, 0.21071428571428572,
                                           0.47539682539682548, 0.23630952380952383,
                                           0.023809523809523808, 0.00019841269841269839],
                               rtol=1e-14)
    np.testing.assert_allclose(K[1, 0:5], [0.058333333333333336, 0.33333333333333337,
                                           -0.18333333333333346, -0.2, -0.008333333333333333],
                               rtol=1e-13)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_structure(p):
    N = 20
    M = gram_factor(p, N, "mass").dense()
    K = gram_factor(p, N, "stiff").dense()
    assert np.array_equal(M, M.T) and np.array_equal(K, K.T)
    # Neumann: constants are in the stiffness kernel; mass integrates the box
    assert np.abs(K.sum(axis=1)).max() < 1e-14
    assert M.sum() == pytest.approx(N - 1, rel=1e-14)
    # mirror symmetry of the edge rows
    assert np.array_equal(M, M[::-1, ::-1])
    assert np.all(np.linalg.eigvalsh(M) > 0)
    assert np.linalg.eigvalsh(K).min() > -1e-12


def test_edge_widths_and_extension():
    assert [basis_extension(p) for p in range(1, 6)] == [0, 1, 1, 2, 2]
    assert [edge_width(p) for p in range(1, 6)] == [1, 3, 3, 5, 5]


def test_too_short_axis():
    p = 3
    with pytest.raises(ValidationError):
        gram_factor(p, min_axis_length(p), "mass")
    gram_factor(p, min_axis_length(p) + 1, "mass")


def test_exact_integral_identities():
    from fractions import Fraction

    # int beta^3(x) beta^3(x-k) = beta^7(k): beta^7(0) = 151/315
    assert product_integral(3, 0, 0, 0, 0) == Fraction(151, 315)
    # grad-grad Gram of linear splines: [-1, 2, -1]
    assert [product_integral(1, 1, k, 1, 0) for k in (-1, 0, 1)] == [-1, 2, -1]


def test_taps_header_matches_factors():
    import os

    from paper_1904_03057_b200.gram import taps_header

    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "paper_1904_03057_b200", "csrc", "gram_taps.cuh")
    assert open(path).read() == taps_header()
    for p in range(1, 6):
        assert "kHostGramM" in taps_header() and f"struct GramTaps<{p}>" in taps_header()
        interior = gram_factor(p, 20, "mass").interior
        assert repr(float(interior[p])) in taps_header()
