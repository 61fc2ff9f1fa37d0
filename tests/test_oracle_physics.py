"""Physics pins for the oracle's assembly / solve / extraction -- CPU only.

Independent of the oracle's own arithmetic: symmetry reductions with brute-force integrals,
scale invariance, Richardson extrapolation to the literature cube capacitance, the analytic
coated sphere, Gauss-law consequences, Maxwell-matrix invariants.
"""
import json
import os

import numpy as np
import pytest

import oracle as O
import voxgen
from tests import quadrature_ref as QR

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))
K = 4 * np.pi * O.EPS0


def _cap(st):
    p = O.enumerate_panels(st.label, st.eps, st.eps_out, st.dv)
    return p, O.solve_capacitance(p)


def test_one_voxel_symmetry_reduction():
    """All 6 panels equivalent -> uniform rho; C = 4πε0 Δv * 6/(P_self + P_opp + 4 P_edge)
    with the three integrals from textbook/brute force (not from the oracle)."""
    s = GOLD["self_term_unit_square"]["value"]
    opp = QR.kappa_quad(0, 2, 2, (0, 0, 1))
    edge = QR.kappa_quad(0, 2, 1, (0, 0, 0))
    ref = 6.0 / (s + opp + 4 * edge)
    dv = 1e-6
    st = voxgen.cube(1, dv)
    _, C = _cap(st)
    assert abs(C[0, 0] / (K * dv) - ref) < 1e-12
    assert abs(ref - 0.648818037184) < 1e-11


def test_cube_scale_invariance():
    """2^3 voxels of edge Δv == one voxel of edge 2Δv with a constant charge on each face."""
    _, C1 = _cap(voxgen.cube(1, 2e-6))
    _, C2 = _cap(voxgen.cube(2, 1e-6))
    assert abs(C2[0, 0] / C1[0, 0] - 1.0) < 1e-12


def test_cube_convergence_to_literature():
    """Galerkin C(n^3)/(4πε0 a) increases with n and extrapolates to 0.66068 (BASELINE)."""
    v = {}
    for n in (2, 4, 8):
        _, C = _cap(voxgen.cube(n, 1.0 / n))
        v[n] = C[0, 0] / K
    assert v[2] < v[4] < v[8] < GOLD["unit_cube_capacitance"]["value"]
    p = np.log2((v[4] - v[2]) / (v[8] - v[4]))
    rich = v[8] + (v[8] - v[4]) / (2 ** p - 1)
    assert abs(rich / GOLD["unit_cube_capacitance"]["value"] - 1) < 2e-3, (v, p, rich)


def test_conductor_block_spd():
    p = O.enumerate_panels(voxgen.sphere(4).label)
    A = O.assemble(p)
    assert np.abs(A - A.T).max() <= 1e-14 * np.abs(A).max()
    assert np.linalg.eigvalsh(A).min() > 0


def test_sphere_near_one():
    """Voxelised sphere capacitance -> 4πε0 R (BASELINE north_star): above 1 and within the
    staircase error (error * R ≈ 0.14-0.21 voxels); the exact survey values
    are pinned in test_oracle_survey_pins.py."""
    R = 8
    _, C = _cap(voxgen.sphere(R, dv=1.0))
    val = C[0, 0] / (K * R)
    assert 1.0 < val < 1.0 + 0.25 / R, val


def _two_blocks(eps_r=None):
    lab = np.zeros((6, 6, 10), np.int32)
    lab[2:4, 2:4, 1:3] = 1
    lab[2:4, 2:4, 6:9] = 2
    eps = np.ones(lab.shape)
    if eps_r:
        eps[1:5, 1:5, 3:6] = eps_r
    return voxgen.Structure(lab, eps, 1.0, 1e-6)


@pytest.mark.parametrize("eps_r", [None, 3.5])
def test_maxwell_invariants(eps_r):
    p, C = _cap(_two_blocks(eps_r))
    assert (np.diag(C) > 0).all()
    assert C[0, 1] < 0 and C[1, 0] < 0
    assert (C.sum(axis=1) > 0).all()
    asym = abs(C[0, 1] - C[1, 0]) / abs(C).max()
    assert asym < (1e-12 if eps_r is None else 2e-2)


def test_isolated_dielectric_neutral():
    """An isolated dielectric body carries no net (bound) charge: Σ A_k ρ_k = 0 (Gauss law +
    Eq. 7)."""
    lab = np.zeros((6, 6, 10), np.int32)
    lab[2:4, 2:4, 1:3] = 1
    eps = np.ones(lab.shape)
    eps[1:5, 2:5, 5:8] = 3.0
    p = O.enumerate_panels(lab, eps, 1.0, 1e-6)
    C, rho = O.solve_capacitance(p, return_rho=True)
    d = ~p.is_cond
    q = (rho[d, 0] * p.dv ** 2).sum()
    scale = (np.abs(rho[d, 0]) * p.dv ** 2).sum()
    assert abs(q) < 1e-10 * scale


def test_dielectric_row_sign_freedom():
    """Flipping a dielectric row's normal (s, ε_d <-> ε_b) leaves ρ unchanged (reading O7)."""
    st = _two_blocks(3.5)
    p = O.enumerate_panels(st.label, st.eps, 1.0, st.dv)
    C0, r0 = O.solve_capacitance(p, return_rho=True)
    d = np.nonzero(~p.is_cond)[0][::3]
    q = O.Panels(p.dims, p.dv, p.m, p.axis, p.slot, p.sign.copy(), p.cid, p.eps_d.copy(),
                 p.eps_b.copy())
    q.sign[d] *= -1
    q.eps_d[d], q.eps_b[d] = p.eps_b[d], p.eps_d[d]
    q = O.Panels(q.dims, q.dv, q.m, q.axis, q.slot, q.sign, q.cid, q.eps_d, q.eps_b)
    C1, r1 = O.solve_capacitance(q, return_rho=True)
    assert np.abs(r1 - r0).max() < 1e-10 * np.abs(r0).max()
    assert np.allclose(C0, C1, rtol=1e-12)


def test_coated_sphere_analytic():
    """C = 4πε0 εr rd rc/((rd - rc) + εr rc), within the staircase error."""
    rc, rd, er = 4, 8, 2.0
    st = voxgen.coated_sphere(rc, rd, er, dv=1.0)
    _, C = _cap(st)
    ana = er * rd * rc / ((rd - rc) + er * rc)
    assert abs(C[0, 0] / K / ana - 1) < 0.05


def test_permittivity_sweep():
    """P:155 sweep (εr 2 -> 2e7): C grows monotonically with εr, converges as εr -> ∞ (the
    shell becomes equipotential) to within the discretisation error of a conductor of the
    shell's shape, and the εr = 1 coating is invisible."""
    rc, rd = 2, 4
    _, Cbare_c = _cap(voxgen.sphere(rc, dv=1.0, n=2 * rd))
    _, Cbare_d = _cap(voxgen.sphere(rd, dv=1.0))
    vals = []
    for er in (1.0, 2.0, 20.0, 2e3, 2e5, 2e7):
        _, C = _cap(voxgen.coated_sphere(rc, rd, er, dv=1.0))
        vals.append(C[0, 0])
    assert abs(vals[0] / Cbare_c[0, 0] - 1) < 1e-12
    assert all(b > a for a, b in zip(vals, vals[1:]))
    assert abs(vals[-1] - vals[-2]) < 1e-4 * vals[-1]
    assert abs(vals[-1] / Cbare_d[0, 0] - 1) < 0.03


def test_precond_whole_domain_box_is_exact_inverse():
    """A single box covering a conductor-only domain makes R_BD = A^{-1} (S:434 idea), and
    R_D = Ī^{-1} on dielectric rows."""
    st = voxgen.random_structure(1)
    p = O.enumerate_panels(st.label, np.ones_like(st.eps), 1.0, st.dv)
    A = O.assemble(p)
    x = voxgen.seeded_vector(p.n, 0)
    z = O.precond_apply(p, A @ x, nv=(64, 64, 64), A=A)
    assert np.abs(z - x).max() < 1e-10 * np.abs(x).max()
    st = _two_blocks(3.5)
    p = O.enumerate_panels(st.label, st.eps, 1.0, st.dv)
    r = voxgen.seeded_vector(p.n, 1)
    z = O.precond_apply(p, r, nv=(2, 2, 2))
    d = ~p.is_cond
    assert np.allclose(z[d], r[d] / p.ibar[d], rtol=1e-15)
    # the conventional block-diagonal comparator: with one box holding every panel
    # (dielectric ones too) R = A^{-1}; with no dielectric panels it equals the proposed one
    A = O.assemble(p)
    x = voxgen.seeded_vector(p.n, 2)
    z = O.precond_apply(p, A @ x, nv=(64, 64, 64), A=A, conventional=True)
    assert np.abs(z - x).max() < 1e-9 * np.abs(x).max()
    st = _two_blocks()
    p = O.enumerate_panels(st.label, st.eps, 1.0, st.dv)
    r = voxgen.seeded_vector(p.n, 3)
    assert np.allclose(O.precond_apply(p, r, nv=(3, 3, 3)), O.precond_apply(p, r, nv=(3, 3, 3), conventional=True),
                       rtol=1e-13, atol=0)
