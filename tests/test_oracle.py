"""Pin the CPU oracle to the reference's own outputs (golden fixtures).

The oracle (oracle/bspde_oracle.py) is the checker of every GPU parity test,
so it is validated first against fixtures generated from the reference
implementation (tests/golden/make_golden.py).
"""

import numpy as np
import pytest

from oracle import bspde_oracle as O

APPLY_TAGS = ["p1", "p2", "p3", "p4", "p5", "p3_heat", "p3_min", "p3_stiff", "p2_2d",
              "p1_1d", "p3_1d"]


def _op(meta, ndim):
    p, D, mu = int(meta[0]), meta[1], meta[2]
    step = tuple(meta[3:3 + ndim])
    ext = tuple(int(v) for v in meta[3 + ndim:3 + 2 * ndim])
    return O.KronOperator(ext, step, p, D, mu)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_oracle_gram_vs_reference(golden, p):
    g = golden("gram.npz")
    for N in (p + 6, 12):
        np.testing.assert_allclose(O.gram_1d(p, N, "mass"), g[f"M_p{p}_N{N}"], atol=1e-15)
        np.testing.assert_allclose(O.gram_1d(p, N, "stiff"), g[f"K_p{p}_N{N}"], atol=1e-15)


@pytest.mark.parametrize("tag", APPLY_TAGS)
def test_oracle_apply_vs_reference(golden, tag):
    g = golden("apply.npz")
    c, t = g[f"{tag}_c"], g[f"{tag}_t"]
    op = _op(g[f"{tag}_meta"], c.ndim)
    got = op.apply(c)
    assert np.abs(got - t).max() / np.abs(t).max() < 1e-13
    np.testing.assert_allclose(op.jacobi_diagonal(), g[f"{tag}_diag"], rtol=1e-14, atol=1e-16)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_oracle_rhs_vs_reference(golden, p):
    g = golden("rhs.npz")
    meta = g[f"p{p}_meta"]
    step = tuple(meta[1:4])
    ext = tuple(int(v) for v in meta[4:7])
    op = O.KronOperator(ext, step, p, 0.0, 1.0)
    t = g[f"p{p}_t"]
    got = op.mass_apply(g[f"p{p}_q"])
    assert np.abs(got - t).max() / np.abs(t).max() < 1e-13


def test_oracle_transform_vs_reference(golden):
    h = golden("heat16.npz")
    inp = O.heat_inputs(16)
    np.testing.assert_allclose(inp["u0"], h["u0"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(inp["q"], h["q"], rtol=0, atol=1e-13)


def test_oracle_heat16_vs_reference(golden):
    h = golden("heat16.npz")
    p, N, hh, dt = int(h["meta"][0]), int(h["meta"][1]), h["meta"][2], h["meta"][3]
    A = O.KronOperator((N,) * 3, (hh,) * 3, p, dt, 1.0)
    F = A.mass_apply(h["q"])
    np.testing.assert_allclose(F, h["F"], rtol=0, atol=1e-15 * np.abs(h["F"]).max() * 10)
    u, its = O.heat_steps(N, hh, p, dt, h["u0"], h["q"], 10)
    ref_its = list(h["iters_tol1e-10"])
    assert all(abs(a - b) <= 1 for a, b in zip(its, ref_its)), (its, ref_its)
    # coefficient parity: 1e-9 at tol 1e-12, 1e-10 at tol 1e-13
    for tol, bar in ((1e-12, 1e-9), (1e-13, 1e-10)):
        u1, rep = O.pcg(A.apply, A.jacobi_diagonal, h["b1"], tol=tol, max_iter=5000, x0=h["u0"])
        ref = h[f"u1_tol{tol:.0e}".replace("e-", "e-")]
        assert np.linalg.norm(u1 - ref) / np.linalg.norm(ref) < bar
        assert abs(rep["iterations"] - int(h[f"iters1_tol{tol:.0e}"][0])) <= 1


def test_oracle_pcg_guards():
    A = np.diag([1.0, -1.0, 2.0])
    with pytest.raises(O.OracleIndefinite):
        O.pcg(lambda c: A @ c, lambda: np.diag(A), np.ones(3), precond="none")
    x, rep = O.pcg(lambda c: A @ c, lambda: np.diag(A), np.zeros(3))
    assert rep["iterations"] == 0 and not x.any()


def test_oracle_c1_step1_vs_reference(golden):
    """C1 (64^3): the oracle's first heat step reproduces the reference
    solution to 1e-10 relative L2 at CG tol 1e-13."""
    h = golden("heat64.npz")
    inp = O.heat_inputs(64)
    N, hh, dt = inp["N"], inp["h"], inp["dt"]
    A = O.KronOperator((N,) * 3, (hh,) * 3, 3, dt, 1.0)
    b1 = A.mass_apply(inp["u0"]) + dt * A.mass_apply(inp["q"])
    u1, rep = O.pcg(A.apply, A.jacobi_diagonal, b1, tol=1e-13, max_iter=5000, x0=inp["u0"])
    ref = h["u1_tol1e-13"]
    assert np.linalg.norm(u1 - ref) / np.linalg.norm(ref) < 1e-10
    assert abs(rep["iterations"] - int(h["iters1_tol1e-13"][0])) <= 1


def test_oracle_direct_transform_vs_reference_fixtures(golden):
    """The oracle's mirror prefilter against the reference's direct_transform
    (tests/golden/transform.npz; replicate / zero are GPU-tested only)."""
    g = golden("transform.npz")
    for key in list(g.keys()):
        if key.endswith("_x") and "_mirror" in key:
            tag = key[:-2]
            p = int(tag.split("_")[1][1:])
            c = O.direct_transform(g[key], p)
            ref = g[f"{tag}_c"]
            assert float(np.abs(c - ref).max()) <= 1e-13 * float(np.abs(ref).max()), tag


def test_apply_plane_matches_full_apply():
    """The plane-window oracle used by the C3 (930^3) GPU check equals rows
    of the full oracle apply."""
    N = 20
    h = 1.0 / (N - 1)
    ora = O.KronOperator((N,) * 3, (h,) * 3, 3, 4 * h * h, 1.0)
    u = np.random.default_rng(0).normal(size=ora.cext)
    A = ora.apply(u)
    n0 = ora.cext[0]
    for z0 in (0, 1, 5, n0 - 2, n0 - 1):
        lo, hi = max(0, z0 - 3), min(n0, z0 + 4)
        w = ora.apply_plane(u[lo:hi], lo, z0)
        assert np.abs(w - A[z0]).max() <= 1e-14 * np.abs(A[z0]).max()
