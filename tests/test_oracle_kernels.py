"""Pins for the oracle's panel-pair integrals (oracle/kernels_q.c) -- CPU only.

Every check compares against something other than the oracle itself: a textbook closed form,
brute-force quadrature built on the textbook rectangle potential (tests/quadrature_ref.py),
Gauss's law, the far-field limit, or a symbolic antiderivative identity.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle as O
from tests import quadrature_ref as QR

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))


def test_self_term_textbook():
    ref = GOLD["self_term_unit_square"]["value"]
    for a in range(3):
        hi, lo = O.kappa_hilo(0, a, a, (0, 0, 0))
        assert abs((hi + lo) - ref) < 2e-16
    exact = (4.0 / 3.0) * (1 - np.sqrt(2.0)) + 4 * np.log(1 + np.sqrt(2.0))
    assert abs(ref - exact) < 1e-15


# touching / near pairs: outer adaptive quadrature of the textbook rectangle potential/field
NEAR = [
    (0, 2, 2, (0, 0, 1)), (0, 2, 2, (1, 0, 0)), (0, 2, 2, (1, 1, 1)),
    (0, 2, 1, (0, 0, 0)), (0, 2, 1, (0, 1, 0)), (0, 2, 1, (1, -1, 1)),
    (0, 0, 1, (1, -1, 0)), (0, 1, 0, (0, 1, -1)), (0, 0, 2, (1, 0, -1)),
    (1, 2, 2, (0, 0, -1)), (1, 2, 2, (1, 0, 1)), (1, 0, 0, (1, 1, 0)),
    (1, 2, 1, (0, 0, 0)), (1, 2, 1, (0, 1, 0)), (1, 2, 1, (1, 1, 0)),
    (1, 0, 1, (0, 0, 0)), (1, 1, 2, (0, 1, -1)), (1, 0, 2, (0, 1, 1)),
    (1, 2, 0, (-1, 0, 1)), (1, 1, 0, (1, 0, 1)),
]


@pytest.mark.parametrize("kind,alpha,beta,d", NEAR)
def test_near_pairs_vs_quadrature(kind, alpha, beta, d):
    ref = QR.kappa_quad(kind, alpha, beta, d, epsabs=1e-12, epsrel=1e-11)
    got = O.kappa(kind, alpha, beta, d)
    assert abs(got - ref) <= 1e-10 * max(1.0, abs(ref)), (got, ref)


def test_far_pairs_vs_gauss_legendre():
    rng = np.random.default_rng(7)
    n = 0
    for _ in range(200):
        kind, a, b = int(rng.integers(0, 2)), int(rng.integers(0, 3)), int(rng.integers(0, 3))
        d = rng.integers(-7, 8, 3)
        if np.linalg.norm(d) < 4:
            continue
        ref = QR.kappa_gl(kind, a, b, tuple(d), q=14)
        got = O.kappa(kind, a, b, tuple(int(v) for v in d))
        assert abs(got - ref) < 1e-14, (kind, a, b, d, got, ref)
        n += 1
    assert n > 100


def _box_surface(n):
    """Panels (axis, slot, outward sign) on the boundary of the box [0,n]^3 of voxels."""
    out = []
    for a in range(3):
        u, v = [x for x in range(3) if x != a]
        for p, s in ((0, -1), (n, +1)):
            for i in range(n):
                for j in range(n):
                    slot = [0, 0, 0]
                    slot[a], slot[u], slot[v] = p, i, j
                    out.append((a, tuple(slot), s))
    return out


def _flux(surface, src_axis, src_slot):
    tot = 0.0
    for a, slot, s in surface:
        d = tuple(slot[i] - src_slot[i] for i in range(3))
        tot += s * O.kappa(1, a, src_axis, d)
    return tot


def test_gauss_law_exact():
    """Σ_{closed surface} s_k E+_kl = -4π (inside), 0 (outside), -2π (on surface, PV)."""
    surf = _box_surface(3)
    g = GOLD["gauss_law"]
    inside = [(0, (1, 1, 1)), (1, (2, 1, 0)), (2, (0, 2, 1)), (0, (2, 0, 2))]
    outside = [(0, (4, 1, 1)), (2, (1, 1, -1)), (1, (-1, 5, 2)), (0, (-1, 0, 0))]
    on = [(0, (0, 1, 1)), (2, (0, 0, 3)), (1, (2, 3, 0)), (0, (3, 2, 2))]
    for ax, sl in inside:
        assert abs(_flux(surf, ax, sl) - g["inside"]) < 1e-12
    for ax, sl in outside:
        assert abs(_flux(surf, ax, sl) - g["outside"]) < 1e-12
    for ax, sl in on:
        assert abs(_flux(surf, ax, sl) - g["on_surface_pv"]) < 1e-12


def test_far_field_limit():
    """kappa_P -> 1/d and kappa_E+ -> -d_alpha/d^3 at large separation (point charges)."""
    for a, b in itertools.product(range(3), range(3)):
        D = np.array([151, -97, 203])
        cen = lambda ax, s: s + 0.5 - 0.5 * np.eye(3)[ax]
        r = cen(a, D) - cen(b, np.zeros(3))
        dist = np.linalg.norm(r)
        assert abs(O.kappa(0, a, b, D) * dist - 1.0) < 1e-5
        e = O.kappa(1, a, b, D)
        assert abs(e / (-r[a] / dist ** 3) - 1.0) < 1e-4


def test_reciprocity_and_parity():
    rng = np.random.default_rng(3)
    for _ in range(60):
        a, b = int(rng.integers(0, 3)), int(rng.integers(0, 3))
        d = tuple(int(v) for v in rng.integers(-4, 5, 3))
        md = tuple(-v for v in d)
        # P reciprocity: P^{ab}(D) = P^{ba}(-D)  (symmetric Galerkin matrix, Eq. 12 origin)
        assert abs(O.kappa(0, a, b, d) - O.kappa(0, b, a, md)) < 1e-14
    for _ in range(60):
        a = int(rng.integers(0, 3))
        d = np.array([int(v) for v in rng.integers(-4, 5, 3)])
        # parallel E+^{aa} is odd along a, even along the two other axes
        m = d.copy()
        m[a] = -m[a]
        assert abs(O.kappa(1, a, a, tuple(d)) + O.kappa(1, a, a, tuple(m))) < 1e-14
        u = (a + 1) % 3
        m = d.copy()
        m[u] = -m[u]
        assert abs(O.kappa(1, a, a, tuple(d)) - O.kappa(1, a, a, tuple(m))) < 1e-14


def test_coplanar_parallel_field_vanishes():
    for a in range(3):
        for d in [(1, 0, 0), (0, 2, 0), (3, -1, 0), (0, 0, 4)]:
            dd = list(d)
            dd[a] = 0
            assert abs(O.kappa(1, a, a, tuple(dd))) < 1e-30


@pytest.mark.slow
def test_antiderivatives_symbolic():
    """d^4F/da^2db^2 = 1/r and d^4H/da^2 db dc = 1/r (closed forms used by the oracle)."""
    sp = pytest.importorskip("sympy")
    a, b, c = sp.symbols("a b c", positive=True)
    r = sp.sqrt(a ** 2 + b ** 2 + c ** 2)
    F = ((b ** 2 - c ** 2) / 2 * a * sp.log(a + r) + (a ** 2 - c ** 2) / 2 * b * sp.log(b + r)
         - (a ** 2 + b ** 2 - 2 * c ** 2) * r / 6 - a * b * c * sp.atan(a * b / (c * r)))
    H = (a * b * c * sp.log(a + r) + (a ** 2 * b / 2 - b ** 3 / 6) * sp.log(c + r)
         + (a ** 2 * c / 2 - c ** 3 / 6) * sp.log(b + r) - b * c * r / 3
         + (-a ** 3 / 9 + a * b ** 2 / 6 + a * c ** 2 / 6) * sp.atan(b * c / (a * r))
         + (a ** 3 / 18 - a * b ** 2 / 3 + a * c ** 2 / 6) * sp.atan(a * c / (b * r))
         + (a ** 3 / 18 + a * b ** 2 / 6 - a * c ** 2 / 3) * sp.atan(a * b / (c * r)))
    dF = sp.diff(F, a, a, b, b)
    dH = sp.diff(H, a, a, b, c)
    for v in [(0.3, 0.7, 1.1), (2.0, 0.5, 0.9), (1.3, 2.2, 0.4)]:
        sub = {a: v[0], b: v[1], c: v[2]}
        inv = 1.0 / np.sqrt(sum(x * x for x in v))
        assert abs(float(dF.subs(sub)) - inv) < 1e-12
        assert abs(float(dH.subs(sub)) - inv) < 1e-12
