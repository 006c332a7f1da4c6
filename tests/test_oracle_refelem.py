"""Pins of the oracle reference element against closed forms and invariants
(DESIGN.md §"Oracle pins", rows 'LGL', 'cubature', 'triangle nodes', 'basis')."""
import json
import math
import os

import numpy as np
import pytest

from oracle import refelem as R

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _ev(s):
    return float(eval(s, {"sqrt": math.sqrt}))


def test_lgl_closed_forms():
    """LGL orders 1-3 in closed form."""
    with open(os.path.join(GOLD, "lgl_closed_forms.json")) as f:
        g = json.load(f)
    for p in (1, 2, 3):
        x, w = R.lgl(p)
        np.testing.assert_allclose(x, [_ev(s) for s in g[str(p)]["nodes"]], atol=1e-15)
        np.testing.assert_allclose(w, [_ev(s) for s in g[str(p)]["weights"]], atol=1e-15)


@pytest.mark.parametrize("p", range(1, 10))
def test_lgl_exactness(p):
    """LGL with p+1 points integrates x^k exactly for k <= 2p-1; nodes
    symmetric, endpoints +-1."""
    x, w = R.lgl(p)
    for k in range(2 * p):
        exact = 2.0 / (k + 1) if k % 2 == 0 else 0.0
        assert abs(np.sum(w * x ** k) - exact) < 1e-14
    assert x[0] == -1.0 and x[-1] == 1.0
    np.testing.assert_allclose(x, -x[::-1], atol=1e-15)
    # and NOT exact at degree 2p (the rule is Lobatto, not Gauss)
    assert abs(np.sum(w * x ** (2 * p)) - 2.0 / (2 * p + 1)) > 1e-6


@pytest.mark.parametrize("p", range(1, 10))
def test_triangle_cubature_moments(p):
    """Collapsed rule (O-4) exact to degree 2p+1: with u=(1+r)/2, v=(1+s)/2,
    int_T u^i v^j dr ds = 4 i! j! / (i+j+2)!  (closed form)."""
    r, s, w = R.tri_cubature(p)
    u, v = (1 + r) / 2, (1 + s) / 2
    f = math.factorial
    for i in range(2 * p + 2):
        for j in range(2 * p + 2 - i):
            exact = 4.0 * f(i) * f(j) / f(i + j + 2)
            assert abs(np.sum(w * u ** i * v ** j) - exact) < 2e-15, (i, j)
    assert np.all(w > 0) and np.all(r >= -1) and np.all(s >= -1) and np.all(r + s <= 1e-15)


@pytest.mark.parametrize("p", range(1, 10))
def test_triangle_nodes(p):
    """Blyth-Pozrikidis set (O1): Nt nodes; edge nodes are the LGL nodes;
    invariant under the 6 symmetries of the triangle; vertices included."""
    r, s = R.tri_nodes(p)
    Nt = (p + 1) * (p + 2) // 2
    assert len(r) == Nt
    lam1, lam2 = (1 + r) / 2, (1 + s) / 2
    lam0 = 1 - lam1 - lam2
    lg = (1 + R.lgl(p)[0]) / 2
    on_e = np.abs(lam2) < 1e-14
    np.testing.assert_allclose(np.sort(lam1[on_e]), lg, atol=1e-15)
    bary = np.stack([lam0, lam1, lam2], 1)
    key = lambda B: np.array(sorted(map(tuple, np.round(B, 12))))
    base = key(bary)
    for perm in [(1, 2, 0), (2, 0, 1), (1, 0, 2), (0, 2, 1), (2, 1, 0)]:
        np.testing.assert_allclose(key(bary[:, perm]), base, atol=1e-12)
    # Vandermonde well conditioned (<= ~362 at p=8)
    V = R.dubiner(p, r, s)[0]
    assert np.linalg.cond(V) < 1e3


def _poly_tri(p, rng):
    c = rng.uniform(-1, 1, (p + 1, p + 1))
    for a in range(p + 1):
        for b in range(p + 1):
            if a + b > p:
                c[a, b] = 0.0

    def f(r, s):
        return sum(c[a, b] * r ** a * s ** b for a in range(p + 1) for b in range(p + 1))

    def fr(r, s):
        return sum(a * c[a, b] * r ** (a - 1) * s ** b for a in range(1, p + 1) for b in range(p + 1))

    def fs(r, s):
        return sum(b * c[a, b] * r ** a * s ** (b - 1) for a in range(p + 1) for b in range(1, p + 1))
    return f, fr, fs


@pytest.mark.parametrize("p", range(1, 9))
def test_prism_basis_reproduces_polynomials(p):
    """Cardinal property and exact interpolation/differentiation of random
    polynomials in P_p(triangle) x P_p(t) at random points."""
    rng = np.random.default_rng(p)
    rst, _ = R.prism_nodes(p)
    val, _ = R.prism_basis(p, rst)
    np.testing.assert_allclose(val, np.eye(len(rst)), atol=1e-12)
    f, fr, fs = _poly_tri(p, rng)
    ct = rng.uniform(-1, 1, p + 1)
    g = lambda t: sum(ct[k] * t ** k for k in range(p + 1))
    gt = lambda t: sum(k * ct[k] * t ** (k - 1) for k in range(1, p + 1))
    u = f(rst[:, 0], rst[:, 1]) * g(rst[:, 2])
    pts = np.stack([rng.uniform(-1, 0, 20), rng.uniform(-1, 0, 20), rng.uniform(-1, 1, 20)], 1)
    pts[:, 1] = np.minimum(pts[:, 1], -pts[:, 0])
    v, grad = R.prism_basis(p, pts)
    r, s, t = pts.T
    np.testing.assert_allclose(v @ u, f(r, s) * g(t), atol=1e-11)
    np.testing.assert_allclose(grad[0] @ u, fr(r, s) * g(t), atol=1e-10)
    np.testing.assert_allclose(grad[1] @ u, fs(r, s) * g(t), atol=1e-10)
    np.testing.assert_allclose(grad[2] @ u, f(r, s) * gt(t), atol=1e-10)
    # partition of unity / derivative rows sum to zero
    np.testing.assert_allclose(v.sum(1), 1.0, atol=1e-12)
    np.testing.assert_allclose(grad.sum(2), 0.0, atol=1e-10)


def test_level_schedule():
    """P:534 rule ceil((P+1)/2) with strict-decrease guard."""
    want = {8: [8, 5, 3, 2, 1], 7: [7, 4, 3, 2, 1], 6: [6, 4, 3, 2, 1], 5: [5, 3, 2, 1],
            4: [4, 3, 2, 1], 3: [3, 2, 1], 2: [2, 1], 1: [1]}
    for p, s in want.items():
        assert R.level_schedule(p) == s
