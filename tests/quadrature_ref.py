"""Brute-force panel-pair integrals for pinning the oracle (test helper, not the oracle).

Independent of oracle/kernels_q.c: the inner (source) integral uses the textbook potential /
field of a uniformly charged rectangle at a point, the outer (observer) integral is numerical
(scipy dblquad, or tensor Gauss-Legendre for separated pairs).  Unit voxel, 4πε0 = 1.
"""
import numpy as np
from scipy import integrate


def panel_rect(axis, slot):
    """(normal axis, plane coordinate, [(lo, hi)] for the two in-plane axes u<v)."""
    u, v = [a for a in range(3) if a != axis]
    return axis, float(slot[axis]), (u, float(slot[u]), float(slot[u]) + 1.0), \
        (v, float(slot[v]), float(slot[v]) + 1.0)


def _g(U, V, h):
    """Antiderivative of 1/R over the rectangle (textbook): U ln(V+R) + V ln(U+R) - h atan."""
    R = np.sqrt(U * U + V * V + h * h)
    t = 0.0
    if U != 0.0:
        vr = V + R if V >= 0 else (U * U + h * h) / (R - V)
        t += U * np.log(vr) if vr > 0 else 0.0
    if V != 0.0:
        ur = U + R if U >= 0 else (V * V + h * h) / (R - U)
        t += V * np.log(ur) if ur > 0 else 0.0
    if h != 0.0 and U != 0.0 and V != 0.0:
        t -= h * np.arctan(U * V / (h * R))
    return t


def rect_potential(p, src_axis, src_slot):
    """∬_src dS'/|p - r'| for a unit source panel (textbook closed form)."""
    n, z0, (u, u1, u2), (v, v1, v2) = panel_rect(src_axis, src_slot)
    h = p[n] - z0
    s = 0.0
    for i, uu in ((1, u2), (-1, u1)):
        for j, vv in ((1, v2), (-1, v1)):
            s += i * j * _g(uu - p[u], vv - p[v], h)
    return s


def rect_field_plus(p, obs_axis, src_axis, src_slot):
    """∂/∂p_obs_axis of rect_potential (field along +axis at p, sign-free gradient)."""
    n, z0, (u, u1, u2), (v, v1, v2) = panel_rect(src_axis, src_slot)
    h = p[n] - z0
    s = 0.0
    for i, uu in ((1, u2), (-1, u1)):
        for j, vv in ((1, v2), (-1, v1)):
            U, V = uu - p[u], vv - p[v]
            R = np.sqrt(U * U + V * V + h * h)
            if obs_axis == n:
                # d g/d h = -atan(UV/(hR))
                if h != 0.0 and U != 0.0 and V != 0.0:
                    s += i * j * (-np.arctan(U * V / (h * R)))
            elif obs_axis == u:
                # d g/d p_u = -d g/dU = -ln(V + R)
                vr = V + R if V >= 0 else (U * U + h * h) / (R - V)
                s += i * j * (-np.log(vr))
            else:
                ur = U + R if U >= 0 else (V * V + h * h) / (R - U)
                s += i * j * (-np.log(ur))
    return s


def kappa_quad(kind, alpha, beta, d, epsabs=1e-13, epsrel=1e-12):
    """Observer alpha-panel at slot d, source beta-panel at slot 0: outer dblquad."""
    n, z1, (u, u1, u2), (v, v1, v2) = panel_rect(alpha, d)
    src = (0, 0, 0)

    def f(y, x):
        p = [0.0, 0.0, 0.0]
        p[n] = z1
        p[u] = x
        p[v] = y
        if kind == 0:
            return rect_potential(p, beta, src)
        return rect_field_plus(p, alpha, beta, src)

    val, err = integrate.dblquad(f, u1, u2, v1, v2, epsabs=epsabs, epsrel=epsrel)
    return val


def kappa_gl(kind, alpha, beta, d, q=14):
    """Tensor Gauss-Legendre over both panels (for separated pairs only)."""
    x, w = np.polynomial.legendre.leggauss(q)
    x = 0.5 * (x + 1.0)
    w = 0.5 * w

    def pts(axis, slot):
        n, z0, (u, a0, a1), (v, b0, b1) = panel_rect(axis, slot)
        P = np.zeros((q, q, 3))
        P[..., n] = z0
        P[..., u] = (a0 + x)[:, None]
        P[..., v] = (b0 + x)[None, :]
        W = w[:, None] * w[None, :]
        return P.reshape(-1, 3), W.reshape(-1)

    po, wo = pts(alpha, d)
    ps, ws = pts(beta, (0, 0, 0))
    diff = po[:, None, :] - ps[None, :, :]
    r = np.sqrt((diff ** 2).sum(-1))
    if kind == 0:
        f = 1.0 / r
    else:
        f = -diff[..., alpha] / r ** 3  # d/d(obs_alpha) of 1/r
    return float(wo @ f @ ws)
