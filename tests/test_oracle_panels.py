"""Pins for the oracle's panel enumeration (a1) -- CPU only (S:60-64, S:77-79 ideas)."""
import os

import numpy as np
import pytest

import oracle as O
import voxgen


def _lab(shape, fill=0):
    return np.full(shape, fill, np.int32)


def test_single_voxel_six_panels():
    p = O.enumerate_panels(_lab((1, 1, 1), 1))
    assert p.n == 6 and p.n_cond == 6 and p.n_diel == 0
    # canonical order: x-panels (i=0 then 1), then y, then z; outward signs -, +
    assert list(p.axis) == [0, 0, 1, 1, 2, 2]
    assert list(p.sign) == [-1, 1, -1, 1, -1, 1]
    assert [tuple(s) for s in p.slot] == [(0, 0, 0), (1, 0, 0), (0, 0, 0), (0, 1, 0),
                                          (0, 0, 0), (0, 0, 1)]
    assert (p.fc == 1.0).all()


def test_bar_ten_panels():
    p = O.enumerate_panels(_lab((1, 1, 2), 1))  # 2 x 1 x 1 along x
    assert p.n == 10  # shared internal face is not a boundary


def test_dielectric_cube_24_outward():
    lab = _lab((4, 4, 4))
    lab[0, 0, 0] = 1  # a conductor far corner so m >= 1
    eps = np.ones((4, 4, 4))
    eps[2:4, 2:4, 2:4] = 3.0
    p = O.enumerate_panels(lab, eps)
    d = ~p.is_cond
    assert d.sum() == 24
    # outward normal: sign +1 exactly on the faces at the + side of the block
    for a in range(3):
        sel = d & (p.axis == a)
        assert set(zip(p.slot[sel, a].tolist(), p.sign[sel].tolist())) == {(2, -1), (4, 1)}
    assert np.allclose(p.eps_d[d], 3.0) and np.allclose(p.eps_b[d], 1.0)
    # Eq. (7): Ī = A(εd+εb)/(2ε0(εd-εb)), A = 1
    assert np.allclose(p.ibar[d], 4.0 / (2 * O.EPS0 * 2.0))


def test_canonical_order_and_closed_surface_parity():
    for seed in range(1, 6):
        st = voxgen.random_structure(seed)
        p = O.enumerate_panels(st.label, st.eps, st.eps_out, st.dv)
        key = p.axis.astype(np.int64) * 10 ** 9 + (p.slot[:, 2].astype(np.int64) * 10 ** 6
                                                   + p.slot[:, 1] * 10 ** 3 + p.slot[:, 0])
        assert (np.diff(key) > 0).all()
        for c in range(1, p.m + 1):
            for a in range(3):
                sel = (p.cid == c) & (p.axis == a)
                assert p.sign[sel].sum() == 0  # closed surface: as many + as - faces


def test_translation_invariance():
    st = voxgen.random_structure(3)
    p0 = O.enumerate_panels(st.label, st.eps)
    lab = np.pad(st.label, ((2, 1), (1, 0), (3, 2)))
    eps = np.pad(st.eps, ((2, 1), (1, 0), (3, 2)), constant_values=1.0)
    p1 = O.enumerate_panels(lab, eps)
    assert p0.n == p1.n
    assert (p1.slot - p0.slot == np.array([3, 1, 2])).all()
    assert (p0.sign == p1.sign).all() and (p0.cid == p1.cid).all()


def test_config_counts():
    # C2: plates 2*(2*32*32 + 4*32) conductor panels, slab side walls 4*32*4 dielectric
    st = voxgen.config("C2")
    p = O.enumerate_panels(st.label, st.eps)
    assert (p.n, p.n_cond, p.n_diel) == (4864, 4352, 512)
    fc_slab = p.fc[p.is_cond & (p.axis == 2) & ((p.slot[:, 2] == 1) | (p.slot[:, 2] == 5))]
    assert fc_slab.size == 2048 and (fc_slab == 4.0).all()
    st = voxgen.config("C1")
    assert O.enumerate_panels(st.label).n == 6 * 64


@pytest.mark.parametrize("case", ["neg", "gap_ids", "empty", "clash", "eps0", "epsnan"])
def test_input_errors(case):
    lab = _lab((3, 3, 3))
    eps = np.ones((3, 3, 3))
    if case == "neg":
        lab[0, 0, 0] = -1
    elif case == "gap_ids":
        lab[0, 0, 0] = 2
    elif case == "clash":
        lab[0, 0, 0] = 1
        lab[0, 0, 1] = 2
    elif case == "eps0":
        lab[1, 1, 1] = 1
        eps[0, 0, 0] = 0.0
    elif case == "epsnan":
        lab[1, 1, 1] = 1
        eps[0, 0, 0] = np.nan
    with pytest.raises(O.OracleInputError):
        O.enumerate_panels(lab, eps)


def test_coated_sphere_panel_counts_match_paper():
    """the coated sphere (r_c = 0.25 m, r_d = 0.5 m) at dv = 0.05 / 0.025 / 0.02 / 0.01 m
    has N_i voxels and N panels as printed (golden values, tests/golden/pins.json)."""
    import json
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))
    pin = g["coated_sphere_panel_counts"]
    for dv, ni, n in zip(pin["dv_m"], pin["N_i"], pin["N"]):
        rc, rd = pin["r_c_m"] / dv, pin["r_d_m"] / dv
        st = voxgen.coated_sphere(rc, rd, 2.0, dv=dv)
        assert st.label.size == ni
        p = O.enumerate_panels(st.label, st.eps, 1.0, st.dv)
        assert p.n == n, (dv, p.n, n)
