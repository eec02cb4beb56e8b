"""Exact 1-D B-spline Gram factors (host setup, computed once per grid).

For constant diffusion ``D`` and absorption ``mu`` on a box domain without
face terms, the reference operator (``OnTheFlyOperator`` over
``build_system``, ``/root/reference/pkg/src/bspde/assembly.py:396-457``)
is exactly the Kronecker sum

    A = vol * [ mu * Mz(x)My(x)Mx
                + D * ( Kz(x)My(x)Mx / hz^2 + Mz(x)Ky(x)Mx / hy^2 + Mz(x)My(x)Kx / hx^2 ) ]

where ``Ma``/``Ka`` are the 1-D mass and stiffness Gram matrices of the
degree-p centered B-splines on the *extended* coefficient axis (length
``N + 2*ext``).  Each is banded (half-width p), symmetric, Toeplitz in the
interior and position dependent in the first/last ``ew = ext + fc`` rows
(``assembly.py:83-108``: ``trilinear_axis_band`` with ``edge_trilinear_table``
for ``i < ew`` and the mirrored table for ``i >= n - ew``).

The reference integrates the products with composite Gauss-Legendre
quadrature (``kernels.py:65-93``).  Here every entry is computed in exact
rational arithmetic (the B-spline pieces have rational coefficients and
the integration limits are half-integers), then rounded once to fp64, so
the factors are correctly rounded.  ``tests/test_gram.py`` pins them
against the reference's tables (golden fixtures) at <= 1e-15.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction
from functools import lru_cache

import numpy as np

from .errors import DegreeError, ValidationError

MAX_DEGREE = 5


# ---------------------------------------------------------------------------
# exact polynomial helpers (coefficient lists, lowest power first)


def _pmul(a, b):
    out = [Fraction(0)] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        if x == 0:
            continue
        for j, y in enumerate(b):
            out[i + j] += x * y
    return out


def _pshift(a, s):
    """Coefficients of q(x) = a(x - s)."""
    out = [Fraction(0)] * len(a)
    for k, c in enumerate(a):
        if c == 0:
            continue
        # (x - s)^k = sum_j C(k,j) x^j (-s)^(k-j)
        for j in range(k + 1):
            out[j] += c * math.comb(k, j) * (-s) ** (k - j)
    return out


def _pderiv(a):
    return [a[k] * k for k in range(1, len(a))] or [Fraction(0)]


def _pint(a, lo, hi):
    tot = Fraction(0)
    for k, c in enumerate(a):
        if c != 0:
            tot += c * (hi ** (k + 1) - lo ** (k + 1)) / (k + 1)
    return tot


@lru_cache(maxsize=None)
def bspline_pieces(p: int, deriv: int = 0):
    """Centered cardinal B-spline ``beta^p`` (or its derivative) as exact pieces.

    Returns a tuple of ``(lo, hi, coeffs)`` on the knot intervals
    ``[-(p+1)/2 + m, -(p+1)/2 + m + 1]``, using the truncated-power form
    ``beta^p(x) = 1/p! sum_k (-1)^k C(p+1,k) (x - a_k)_+^p``.
    """
    if not 0 <= p <= 2 * MAX_DEGREE + 1:
        raise DegreeError(f"degree {p} out of range")
    if deriv > p:
        raise ValidationError(f"order-{deriv} derivative of degree-{p} spline")
    a0 = Fraction(-(p + 1), 2)
    knots = [a0 + m for m in range(p + 2)]
    pieces = []
    for m in range(p + 1):
        poly = [Fraction(0)] * (p + 1)
        for k in range(m + 1):
            term = _pshift([Fraction(0)] * p + [Fraction(1)], knots[k])  # (x - a_k)^p
            coef = Fraction((-1) ** k * math.comb(p + 1, k), math.factorial(p))
            for j, c in enumerate(term):
                poly[j] += coef * c
        for _ in range(deriv):
            poly = _pderiv(poly)
        pieces.append((knots[m], knots[m + 1], tuple(poly)))
    return tuple(pieces)


def product_integral(p, d1, s1, d2, s2, lo=None, hi=None) -> Fraction:
    """Exact ``int_lo^hi D^d1 beta^p(x - s1) * D^d2 beta^p(x - s2) dx``."""
    s1 = Fraction(s1)
    s2 = Fraction(s2)
    tot = Fraction(0)
    for a1, b1, c1 in bspline_pieces(p, d1):
        for a2, b2, c2 in bspline_pieces(p, d2):
            a = max(a1 + s1, a2 + s2)
            b = min(b1 + s1, b2 + s2)
            if lo is not None:
                a = max(a, Fraction(lo))
            if hi is not None:
                b = min(b, Fraction(hi))
            if b <= a:
                continue
            prod = _pmul(_pshift(list(c1), s1), _pshift(list(c2), s2))
            tot += _pint(prod, a, b)
    return tot


# ---------------------------------------------------------------------------
# index conventions (reference: domain.py:222-224, assembly.py:37-44)


def basis_extension(p: int) -> int:
    """Extended-grid padding per side: ``ceil((p+1)/2) - 1``."""
    return max(int(math.ceil((p + 1) / 2.0)) - 1, 0)


def first_clean_position(p: int) -> int:
    return int(math.ceil((p + 1) / 2.0 - 1e-12))


def edge_width(p: int) -> int:
    """Number of position-dependent rows per axis end (``ew = ext + fc``)."""
    return basis_extension(p) + first_clean_position(p)


def min_axis_length(p: int) -> int:
    """Minimal number of cells per axis for non-interacting edge rows."""
    return int(math.ceil(first_clean_position(p) - 1 + (p + 1) / 2.0))


# ---------------------------------------------------------------------------
# 1-D Gram factors


@dataclass(frozen=True)
class GramFactor:
    """Banded symmetric 1-D Gram matrix in class form.

    ``table[c, k + p]`` is the entry ``G[i, i + k]`` of any row ``i`` of class
    ``c``; classes ``0..ew-1`` are the first rows, ``ew`` the interior
    (Toeplitz) row, ``ew+1..2ew`` the last rows (``2ew`` = row ``n-1``).
    """

    degree: int
    n: int  # extended axis length
    ew: int
    table: np.ndarray  # (2*ew + 1, 2*p + 1) float64

    @property
    def interior(self):
        return self.table[self.ew]

    def row_class(self, i):
        i = np.asarray(i)
        return np.where(i < self.ew, i,
                        np.where(i >= self.n - self.ew, 2 * self.ew - (self.n - 1 - i), self.ew))

    def dense(self) -> np.ndarray:
        p = self.degree
        G = np.zeros((self.n, self.n))
        cls = self.row_class(np.arange(self.n))
        for i in range(self.n):
            for k in range(-p, p + 1):
                j = i + k
                if 0 <= j < self.n:
                    G[i, j] = self.table[cls[i], k + p]
        return G

    def diagonal_by_class(self) -> np.ndarray:
        return self.table[:, self.degree].copy()

    def plus(self, add: np.ndarray) -> "GramFactor":
        """Factor with ``add`` (same class layout) added to its table."""
        table = self.table + add
        table.setflags(write=False)
        return GramFactor(degree=self.degree, n=self.n, ew=self.ew, table=table)


@lru_cache(maxsize=None)
def _exact_rows(p: int, deriv: int):
    """Interior taps and left edge rows (exact Fractions) for degree p."""
    ext = basis_extension(p)
    ew = edge_width(p)
    interior = tuple(product_integral(p, deriv, k, deriv, 0) for k in range(-p, p + 1))
    edge = []
    for i in range(ew):
        ci = i - ext
        row = []
        for k in range(-p, p + 1):
            j = i + k
            row.append(product_integral(p, deriv, j - ext, deriv, ci, lo=0)
                       if j >= 0 else Fraction(0))
        edge.append(tuple(row))
    return interior, tuple(edge)


def _check_degree(p):
    if not isinstance(p, (int, np.integer)) or not 1 <= p <= MAX_DEGREE:
        raise DegreeError(f"basis degree {p} not in 1..{MAX_DEGREE}")


@lru_cache(maxsize=None)
def gram_factor(p: int, num_nodes: int, kind: str) -> GramFactor:
    """Mass (``kind='mass'``) or stiffness (``'stiff'``) factor for one axis.

    ``num_nodes`` is the node count N of the axis; the factor acts on the
    extended axis of length ``N + 2*ext``.  Entries are in unit-grid
    coordinates (scale by h for mass, 1/h for stiffness).
    """
    _check_degree(p)
    if kind not in ("mass", "stiff"):
        raise ValidationError(f"unknown Gram kind {kind!r}")
    if num_nodes - 1 < min_axis_length(p):
        raise ValidationError(
            f"axis with {num_nodes} nodes too short for degree {p} edge tables")
    deriv = 1 if kind == "stiff" else 0
    ext = basis_extension(p)
    ew = edge_width(p)
    n = num_nodes + 2 * ext
    interior, edge = _exact_rows(p, deriv)
    table = np.zeros((2 * ew + 1, 2 * p + 1))
    for c in range(ew):
        table[c] = [float(v) for v in edge[c]]
        # right end mirrors the left one: G[n-1-i, n-1-i-k] = G[i, i+k]
        table[2 * ew - c] = [float(v) for v in edge[c][::-1]]
    table[ew] = [float(v) for v in interior]
    table.setflags(write=False)
    return GramFactor(degree=p, n=n, ew=ew, table=table)


def degenerate_factor(p: int, kind: str) -> GramFactor:
    """Unit factor for a padded (absent) axis: mass = identity, stiffness = 0."""
    table = np.zeros((1, 2 * p + 1))
    if kind == "mass":
        table[0, p] = 1.0
    table.setflags(write=False)
    return GramFactor(degree=p, n=1, ew=0, table=table)


# ---------------------------------------------------------------------------
# trilinear factors for variable coefficients (reference: kernels.py:96-173,
# assembly.py:83-108)


def multi_product_integral(factors, lo=None, hi=None) -> Fraction:
    """Exact ``int prod_f D^d_f beta^{p_f}(x - s_f) dx`` over ``[lo, hi]``."""
    pieces = []
    for deg, shift, deriv in factors:
        sh = Fraction(shift)
        pieces.append([(a + sh, b + sh, _pshift(list(c), sh))
                       for a, b, c in bspline_pieces(deg, deriv)])
    tot = Fraction(0)

    def rec(k, a, b, poly):
        nonlocal tot
        if k == len(pieces):
            if b > a:
                tot += _pint(poly, a, b)
            return
        for pa, pb, pc in pieces[k]:
            na, nb = max(a, pa), min(b, pb)
            if nb > na:
                rec(k + 1, na, nb, _pmul(poly, pc))

    lo_f = Fraction(lo) if lo is not None else Fraction(-10 ** 9)
    hi_f = Fraction(hi) if hi is not None else Fraction(10 ** 9)
    rec(0, lo_f, hi_f, [Fraction(1)])
    return tot


def param_reach(n_b: int, n_p: int) -> int:
    return (n_b + n_p + 1) // 2


@lru_cache(maxsize=None)
def _trilinear_exact(n_b: int, n_p: int, deriv: int):
    """Interior table and left edge tables (exact) of
    ``int D^d beta(x - a) D^d beta(x) beta_np(x - b)`` (a trial, b parameter
    offsets), edge rows integrated over ``[0, inf)`` at test position i - ext."""
    mw = param_reach(n_b, n_p)
    offs_a = range(-n_b, n_b + 1)
    offs_b = range(-mw, mw + 1)
    interior = tuple(tuple(multi_product_integral([(n_b, a, deriv), (n_b, 0, deriv), (n_p, b, 0)])
                           for b in offs_b) for a in offs_a)
    ext = basis_extension(n_b)
    edge = []
    for i in range(edge_width(n_b)):
        pos = i - ext
        edge.append(tuple(tuple(multi_product_integral(
            [(n_b, pos + a, deriv), (n_b, pos, deriv), (n_p, pos + b, 0)], lo=0)
            for b in offs_b) for a in offs_a))
    return interior, tuple(edge)


def trilinear_tables(n_b: int, n_p: int, deriv: int) -> np.ndarray:
    """Class tables ``(2ew+1, 2n_b+1, 2mw+1)``: classes 0..ew-1 = first rows,
    ew = interior, ew+1..2ew = last rows (the mirror image, sign +1 since
    both factors carry the same derivative)."""
    _check_degree(n_b)
    if not isinstance(n_p, (int, np.integer)) or not 0 <= n_p <= MAX_DEGREE:
        raise DegreeError(f"parameter degree {n_p} not in 0..{MAX_DEGREE}")
    interior, edge = _trilinear_exact(n_b, n_p, deriv)
    ew = edge_width(n_b)
    A, B = 2 * n_b + 1, 2 * param_reach(n_b, n_p) + 1
    t = np.zeros((2 * ew + 1, A, B))
    for c in range(ew):
        t[c] = [[float(v) for v in row] for row in edge[c]]
        t[2 * ew - c] = t[c][::-1, ::-1]
    t[ew] = [[float(v) for v in row] for row in interior]
    return t


# ---------------------------------------------------------------------------
# box-face (Robin / penalty) terms (reference: assembly.py:138-232)


def bspline_value(p: int, x) -> Fraction:
    """Exact ``beta^p(x)``."""
    x = Fraction(x)
    for lo, hi, coeffs in bspline_pieces(p, 0):
        if lo <= x < hi:
            return sum((c * x ** k for k, c in enumerate(coeffs)), Fraction(0))
    return Fraction(0)


def single_integral(p: int, s, lo=None, hi=None) -> Fraction:
    """Exact ``int_lo^hi beta^p(x - s) dx``."""
    s = Fraction(s)
    tot = Fraction(0)
    for a, b, coeffs in bspline_pieces(p, 0):
        a, b = a + s, b + s
        if lo is not None:
            a = max(a, Fraction(lo))
        if hi is not None:
            b = min(b, Fraction(hi))
        if b > a:
            tot += _pint(_pshift(list(coeffs), s), a, b)
    return tot


@lru_cache(maxsize=None)
def face_values(p: int) -> tuple:
    """``beta(u_face - pos_i)`` for the first ``ew`` extended positions of the
    low face (``face_point_values``, assembly.py:173-180); all later entries
    are zero and the high face is the mirror image."""
    _check_degree(p)
    ext = basis_extension(p)
    vals = tuple(bspline_value(p, ext - i) for i in range(edge_width(p)))
    assert bspline_value(p, ext - edge_width(p)) == 0
    return vals


def face_vector(p: int, num_nodes: int, side: int) -> np.ndarray:
    """Full-length face value vector (length ``num_nodes + 2*ext``)."""
    n = num_nodes + 2 * basis_extension(p)
    v = np.zeros(n)
    f = [float(x) for x in face_values(p)]
    if side == 0:
        v[: len(f)] = f
    else:
        v[n - len(f):] = f[::-1]
    return v


def face_table(p: int, side: int) -> np.ndarray:
    """Class-table addition (shape ``(2ew+1, 2p+1)``) of the rank-1 normal
    factor ``v v^T`` of one face (``make_face_term`` pair factors): rows of
    classes ``0..ew-1`` for the low face, ``ew+1..2ew`` for the high face."""
    ew = edge_width(p)
    v = face_values(p)
    add = np.zeros((2 * ew + 1, 2 * p + 1))
    for m in range(ew):
        for mm in range(ew):
            k = mm - m  # column offset of row m (low face)
            if abs(k) <= p:
                if side == 0:
                    add[m, k + p] = float(v[m] * v[mm])
                else:  # row n-1-m, column n-1-mm: offset m - mm
                    add[2 * ew - m, -k + p] = float(v[m] * v[mm])
    return add


@lru_cache(maxsize=None)
def surface_single_rows(p: int) -> tuple:
    """``int_0^inf beta(u - pos_i) du`` for the first ``ew`` positions
    (``surface_single_positions``, assembly.py:158-170); interior rows are 1."""
    ext = basis_extension(p)
    return tuple(single_integral(p, i - ext, lo=0) for i in range(edge_width(p)))


def surface_single_vector(p: int, num_nodes: int) -> np.ndarray:
    n = num_nodes + 2 * basis_extension(p)
    s = np.ones(n)
    rows = [float(x) for x in surface_single_rows(p)]
    s[: len(rows)] = rows
    s[n - len(rows):] = rows[::-1]
    return s


# ---------------------------------------------------------------------------
# per-cell tables for mask domains (reference: kernels.py:331-380)


def cell_offsets(p: int) -> tuple:
    """(lo, hi): node offsets j (spline centred at c + j) non-zero on cell
    (c, c + 1) (``cell_node_offsets``, kernels.py:331-336)."""
    half = Fraction(p + 1, 2)
    return math.floor(-half) + 1, math.ceil(1 + half) - 1


@lru_cache(maxsize=None)
def cell_trilinear(n_b: int, n_p: int, deriv: int) -> np.ndarray:
    """``T[j1, j2, b] = int_0^1 D^d beta(x - j1) D^d beta(x - j2) beta_np(x - b)``
    over the offsets of :func:`cell_offsets` (exact; kernels.py:340-355)."""
    (lo, hi), (plo, phi) = cell_offsets(n_b), cell_offsets(n_p)
    js, bs = range(lo, hi + 1), range(plo, phi + 1)
    return np.array([[[float(multi_product_integral(
        [(n_b, j1, deriv), (n_b, j2, deriv), (n_p, b, 0)], lo=0, hi=1)) for b in bs]
        for j2 in js] for j1 in js])


@lru_cache(maxsize=None)
def cell_bilinear(n1: int, n2: int) -> np.ndarray:
    """``R[j1, j2] = int_0^1 beta_n1(x - j1) beta_n2(x - j2)`` (kernels.py:359-371)."""
    (l1, h1), (l2, h2) = cell_offsets(n1), cell_offsets(n2)
    return np.array([[float(multi_product_integral([(n1, j1, 0), (n2, j2, 0)], lo=0, hi=1))
                      for j2 in range(l2, h2 + 1)] for j1 in range(l1, h1 + 1)])


@lru_cache(maxsize=None)
def cell_single(p: int) -> np.ndarray:
    """``S[j] = int_0^1 beta(x - j)`` (kernels.py:375-380)."""
    lo, hi = cell_offsets(p)
    return np.array([float(single_integral(p, j, lo=0, hi=1)) for j in range(lo, hi + 1)])


def face_normal_values(p: int) -> np.ndarray:
    """``beta(k - (fc - 1))`` for k = 0 .. 2 fc - 2: the values at a cell face
    of the splines whose support crosses it (assembly.py:676-681)."""
    fc = first_clean_position(p)
    return np.array([float(bspline_value(p, k - (fc - 1))) for k in range(2 * fc - 1)])


def taps_header() -> str:
    """C++ header with the exact interior taps (mass, stiffness) for p=1..5.

    Generated into ``csrc/gram_taps.cuh``: constexpr functions (immediates the
    kernels' fast paths fold in; measured faster than ``__constant__`` or
    kernel-parameter taps) and a host copy that ``bspde_plan_create`` checks
    the callers' interior table rows against.  ``tests/test_gram.py`` checks
    the committed header against ``gram_factor`` so the two cannot drift.
    """
    def fn(name, vals):
        body = " : ".join(f"k == {i} ? {repr(float(v))}" for i, v in enumerate(vals[:-1]))
        return (f"  __host__ __device__ static constexpr double {name}(int k) {{\n"
                f"    return {body} : {repr(float(vals[-1]))};\n  }}")

    rows_m, rows_k, spec = [], [], []
    for p in range(1, MAX_DEGREE + 1):
        im, _ = _exact_rows(p, 0)
        ik, _ = _exact_rows(p, 1)
        pad = [0.0] * (2 * MAX_DEGREE + 1 - len(im))
        rows_m.append(", ".join(repr(float(v)) for v in list(im) + pad))
        rows_k.append(", ".join(repr(float(v)) for v in list(ik) + pad))
        spec += [f"template <> struct GramTaps<{p}> {{", fn("M", im), fn("K", ik), "};"]
    lines = ["// generated by paper_1904_03057_b200/gram.py:taps_header() -- do not edit",
             "// exact interior taps G[i, i+k-p], k=0..2p, of the unit-step 1-D Gram",
             "// factors (mass: int b(x)b(x-k); stiffness: int b'(x)b'(x-k)), p = 1..5",
             "#pragma once", "",
             "// host copy (bspde_plan_create validates the interior table rows)",
             f"static const double kHostGramM[{MAX_DEGREE}][{2 * MAX_DEGREE + 1}] = {{"]
    lines += [f"    {{{r}}}," for r in rows_m]
    lines += ["};", f"static const double kHostGramK[{MAX_DEGREE}][{2 * MAX_DEGREE + 1}] = {{"]
    lines += [f"    {{{r}}}," for r in rows_k]
    lines += ["};", "", "template <int P> struct GramTaps;"]
    lines += spec
    return "\n".join(lines) + "\n"
