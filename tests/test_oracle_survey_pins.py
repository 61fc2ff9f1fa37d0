"""Survey-time reference values as oracle pins -- CPU only.

The values in ``golden/survey_values.json`` were computed at survey time, before this repo's
oracle existed, by two independent methods (SURVEY.md §8(c) pins table and "C2 reference
details"): 80-digit closed forms and fp64 closed forms / brute-force quadrature.  Pinning the
oracle's capacitances to them catches a dropped term, a wrong sign or a transposed operand
anywhere in the assembly (Eq. 4-7), the right-hand side or the extraction (Eq. 8):
each of those moves the 12th digit.  Tolerance: half a unit of the last quoted digit.
"""
import json
import os

import numpy as np
import pytest

import oracle as O
import voxgen

SV = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "survey_values.json")))
K = 4 * np.pi * O.EPS0


def _half_ulp(v, digits):
    """Half a unit of the last quoted decimal place of v (quoted with `digits` decimals)."""
    return 0.5 * 10.0 ** (-digits)


def _cap(st):
    p = O.enumerate_panels(st.label, st.eps, st.eps_out, st.dv)
    return p, O.solve_capacitance(p)


@pytest.mark.parametrize("key,n", [("one_voxel_cube", 1), ("cube_4", 4), ("cube_8_C1", 8)])
def test_cube_capacitance_survey_values(key, n):
    """Cube of n^3 voxels, edge a = 1 (Δv = 1/n): C / (4πε0 a) to 12 digits."""
    ref = SV[key]
    _, C = _cap(voxgen.cube(n, 1.0 / n))
    val = C[0, 0] / K
    assert abs(val - ref["value"]) <= _half_ulp(ref["value"], ref["digits"]) + 1e-14, (key, val)


def test_c1_farads():
    """BASELINE configs[0] in SI: a = 8 µm -> 5.862116e-16 F."""
    _, C = _cap(voxgen.config("C1"))
    assert abs(C[0, 0] / SV["cube_8_C1"]["farads_a_8um"] - 1) < 1e-6


def _quoted_decimals(v):
    s = repr(v)
    return len(s.split(".")[1]) if "." in s else 0


@pytest.mark.parametrize("R", [4, 6, 8, 12, pytest.param(16, marks=pytest.mark.slow)])
def test_sphere_survey_values(R):
    """Voxel-centre sphere of radius R in (2R)^3: panel count and C / (4πε0 R) as quoted
    (non-monotone in R, above 1: SURVEY.md §8(c))."""
    sv = SV["sphere"]
    i = sv["R"].index(R)
    p, C = _cap(voxgen.sphere(R, dv=1.0))
    assert p.n == sv["N"][i]
    val = C[0, 0] / (K * R)
    ref = sv["value"][i]
    assert abs(val - ref) <= 0.5 * 10.0 ** (-_quoted_decimals(ref)), (R, val, ref)


@pytest.mark.slow
def test_c2_matrix_survey_values():
    """C2 (two 32x32 plates + ε_r 4 slab): the full 2 x 2 Maxwell matrix in units of 4πε0 Δv
    and the SI entries (SURVEY.md §8(c) C2 reference details).  The survey's two independent
    runs agree to 12 significant digits, so the bar is 5e-12 relative.  Also the geometry's
    z-mirror symmetry (C12 = C21, C11 = C22) and the fringing excess over ε_r A / d
    (|C12| = 1.0714 ε_r A/d)."""
    sv = SV["C2"]
    st = voxgen.config("C2")
    p, C = _cap(st)
    assert (p.n, p.n_cond, p.n_diel) == (sv["N"], sv["N_c"], sv["N_d"])
    val = C / (K * st.dv)
    ref = np.array(sv["value"])
    assert np.abs(val - ref).max() <= 5e-12 * np.abs(ref).max(), (val, ref)
    assert abs(C[0, 1] - C[1, 0]) < 1e-12 * abs(C[0, 1])
    assert abs(C[0, 0] - C[1, 1]) < 5e-12 * abs(C[0, 0])
    par = 4.0 * O.EPS0 * (32 * st.dv) ** 2 / (4 * st.dv)
    assert abs(-C[0, 1] / par - 1.0714) < 5e-5
    assert abs(C[0, 0] / sv["farads"]["C11"] - 1) < 1e-9
    assert abs(C[0, 1] / sv["farads"]["C12"] - 1) < 1e-9
