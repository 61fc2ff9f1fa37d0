"""§III.A validation suite on the GPU path.

The dielectric-coated PEC sphere of the paper (r_c = 0.25 m, r_d = 0.5 m) at its four voxel
sizes: panel counts as printed, self-capacitance against the analytic formula of P:153,
the eps_r sweep 2 -> 2e7 at RRE 1e-8, and the preconditioner ordering of Fig. 3(d)
(P:157).  Everything runs through the C ABI; the analytic formula and the printed counts are the
references (no oracle needed at these sizes).
"""
import json
import os

import numpy as np
import pytest

import voxgen

pytestmark = pytest.mark.gpu

try:
    import paper_2004_02609_b200 as vc
except Exception:  # pragma: no cover
    vc = None

EPS0 = 8.8541878128e-12
PINS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))
RC, RD = 0.25, 0.5


def _analytic(er, rc=RC, rd=RD):
    """C = 4 pi eps0 eps_r r_d r_c / ((r_d - r_c) + eps_r r_c)."""
    return 4 * np.pi * EPS0 * er * rd * rc / ((rd - rc) + er * rc)


@pytest.fixture(scope="module")
def ctx():
    c = vc.VoxCap(0)
    yield c
    c.close()


def _coated(dv, er):
    return voxgen.coated_sphere(RC / dv, RD / dv, er, dv=dv)


@pytest.mark.parametrize("dv", [0.05, 0.025, 0.02, 0.01])
def test_coated_sphere_counts_and_analytic(ctx, dv):
    pin = PINS["coated_sphere_panel_counts"]
    st = _coated(dv, 2.0)
    ctx.set_structure(st)
    assert ctx.n == pin["N"][pin["dv_m"].index(dv)]
    ctx.build_operator()
    C4, info4 = ctx.solve_capacitance(tol=1e-4, maxit=3000)  # the paper's RRE
    C, info = ctx.solve_capacitance(tol=1e-8, maxit=3000)
    assert info[0]["converged"] and info4[0]["converged"]
    paper_it = {0.05: 7, 0.025: 7, 0.02: 10, 0.01: 10}[dv]  # VoxCap iterations
    print(f"dv={dv} iterations at RRE 1e-4: {info4[0]['iters']} (paper {paper_it})")
    assert info4[0]["iters"] <= 2 * paper_it
    err = abs(C[0, 0] / _analytic(2.0) - 1)
    print(f"dv={dv} N={ctx.n} C={C[0, 0]:.6e} F analytic={_analytic(2.0):.6e} err={err:.4f} "
          f"iters={info[0]['iters']}")
    # voxel staircase: the error shrinks with dv (Fig. 3(b)); bound grows with dv
    assert err < 0.6 * dv / 0.05 * 0.05 + 0.01


def test_permittivity_sweep(ctx):
    """eps_r 2 -> 2e7 (one decade per step) at dv = 0.05 m, RRE 1e-8: every solve
    converges, C grows monotonically and saturates at the capacitance of a conductor filling
    the shell (the shell becomes equipotential), within the voxel discretisation."""
    dv = 0.05
    ctx.set_structure(voxgen.sphere(int(round(RD / dv)), dv=dv))
    ctx.build_operator()
    Cs, _ = ctx.solve_capacitance(tol=1e-12)
    vals, iters, tight = [], [], []
    for k in range(8):
        er = 2.0 * 10 ** k
        ctx.set_structure(_coated(dv, er))
        ctx.build_operator()
        C, info = ctx.solve_capacitance(tol=1e-8, maxit=5000)
        assert info[0]["converged"], er
        vals.append(C[0, 0])
        iters.append(info[0]["iters"])
        C12, info12 = ctx.solve_capacitance(tol=1e-13, maxit=5000)
        tight.append(C12[0, 0])
    print("eps_r sweep C (RRE 1e-8):", vals, "iters:", iters)
    print("eps_r sweep C (RRE 1e-13):", tight, "conductor of the shell's shape:", Cs[0, 0])
    # the free-charge scaling eps_r * rho_c amplifies the solve residual by ~eps_r (P:155 notes
    # the paper needed RRE 1e-8 for the same reason): the trend is checked at RRE 1e-13; at the
    # paper's 1e-8 the extraction matches it to 1e-3 up to eps_r = 2e5 (measured drift beyond:
    # 0.01% at 2e6, 1.2% at 2e7 -- see DESIGN.md §12)
    assert all(b > a for a, b in zip(tight, tight[1:]))
    assert all(abs(v / t - 1) < 1e-3 for v, t in zip(vals[:6], tight[:6]))
    # eps_r -> inf: the shell is equipotential; its limit is C of a sphere of radius r_d
    # (analytic 4 pi eps0 r_d) and of the voxel conductor of the shell's shape, each within
    # the discretisation error of the dielectric / conductor panel formulations at dv = 0.05
    assert abs(tight[-1] / (4 * np.pi * EPS0 * RD) - 1) < 0.02
    assert abs(tight[-1] / Cs[0, 0] - 1) < 0.02
    assert abs(tight[0] / _analytic(2.0) - 1) < 0.04


def test_preconditioner_ordering(ctx):
    """P:155-157 (Fig. 3(d)) as the paper ran it: the coated sphere at dv = 0.01 m (N = 59,016,
    P:153), eps_r = 2, boxes N_v = 10, RRE 1e-8.  Iterations with the proposed block-diagonal-
    diagonal preconditioner (3), the conventional block-diagonal one (4: dielectric panels in the
    blocks too), the diagonal one (2) and none (1) order as the paper's 22 < 27 < 41 < 142
    (proposed <= conventional: they tie here), and the proposed blocks need less than a quarter
    of the conventional blocks' memory (paper: 17.04 vs 70.26 MB)."""
    st = _coated(0.01, 2.0)
    it, mem = {}, {}
    for kind, name in ((3, "proposed"), (4, "block_diagonal"), (2, "diagonal"), (1, "none")):
        ctx.set_structure(st)
        ctx.build_operator(precond=kind, box=(10, 10, 10))
        C, info = ctx.solve_capacitance(tol=1e-8, maxit=5000)
        assert info[0]["converged"], name
        it[name] = info[0]["iters"]
        mem[name] = ctx.stats()["precond_doubles"] * 8 / 1e6
    print("iterations to RRE 1e-8:", it, "paper (P:157):", PINS["precond_iterations_rre1e-8"])
    print("preconditioner block memory (MB):", mem, "paper: proposed 17.04, conventional 70.26")
    # measured (r02): 28 / 28 / 35 / 161 -- the proposed preconditioner ties the conventional
    # one here (the paper has 22 vs 27) while storing 5.5x less
    assert it["proposed"] <= it["block_diagonal"] < it["diagonal"] < it["none"]
    assert mem["proposed"] < mem["block_diagonal"] / 4


@pytest.mark.parametrize("name,box", [("R5", (4, 4, 4)), ("C2", (8, 8, 6)), ("R3", (3, 3, 3))])
def test_conventional_block_diagonal_parity(ctx, name, box):
    """precond = 4 (every panel of a box in its block, Eq. 4 rows) against the oracle's
    conventional block-diagonal preconditioner (oracle.precond_apply(conventional=True))."""
    import oracle as O
    st = voxgen.config(name)
    ctx.set_structure(st)
    ctx.build_operator(precond=4, box=box)
    p = O.enumerate_panels(st.label, st.eps, st.eps_out, st.dv)
    A = O.assemble(p)
    r = voxgen.seeded_vector(p.n, 8)
    z = ctx.precond(r)
    ref = O.precond_apply(p, r, nv=box, A=A, conventional=True)
    # Gauss-Jordan on the non-symmetric blocks (no pivoting; dielectric rows are Ī-dominant):
    # rounding ~ cond(block) x eps, measured 1e-10 on C2 -> bar 1e-9 (the proposed SPD blocks
    # are inverted by the symmetric sweep and meet 1e-12, test_precond_parity)
    assert np.linalg.norm(z - ref) / np.linalg.norm(ref) <= 1e-9
    x, info = ctx.solve(A @ voxgen.seeded_vector(p.n, 9), tol=1e-12, maxit=500)
    assert info["converged"]
