"""Reduced-grid dense parity of the C3 / C4 / C5 generators (last pins row:
"pinned on the same generator at reduced grids ... vs the dense oracle").

Each structure runs through exactly what ``bench.py`` times -- the default build (automatic
z mode, batch buffers kept when m >= 2) and ``vc_solve_capacitance``, which solves m >= 2
columns in lockstep pairs with batched matvecs -- and is compared with the dense oracle:
matvec (single column and the batched pair) rel-L2 <= 1e-10, capacitance <= 1e-6 (max entry)
at RRE 1e-12 (reading O19).  Both z modes are checked on the matvec.

  C3r: the C3 sphere generator at R = 16 (C3 / 4 per axis), conductor only, N = 4,872.
  C4r: the C4 meander pair on a 48 x 48 x 8 box over a 4-voxel ε_r 4.4 substrate, N = 6,542.
  C5r: the C5 crossing bus (2 + 2 lines, 2 x 2 voxels) in the three C5 layers, 32 x 32 x 16,
       N = 6,600, m = 4 (two lockstep pairs).
"""
import numpy as np
import pytest

import oracle as O
import voxgen

pytestmark = pytest.mark.gpu

try:
    import paper_2004_02609_b200 as vc
except Exception:  # pragma: no cover
    vc = None

_CACHE = {}


def _dense(name):
    if name not in _CACHE:
        st = voxgen.config(name)
        p = O.enumerate_panels(st.label, st.eps, st.eps_out, st.dv)
        A = O.assemble(p)
        _CACHE[name] = (st, p, A, O.solve_capacitance(p, A=A))
    return _CACHE[name]


@pytest.fixture(scope="module")
def ctx():
    c = vc.VoxCap(0)
    yield c
    c.close()


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("name", voxgen.REDUCED_NAMES)
def test_reduced_matvec_dense_parity(ctx, name):
    st, p, A, _ = _dense(name)
    ctx.set_structure(st)
    assert ctx.n == p.n and ctx.m == p.m
    g = ctx.panels()
    assert np.array_equal(g["slot"], p.slot) and np.array_equal(g["cid"], p.cid)
    X = np.stack([voxgen.seeded_vector(p.n, 40 + i) for i in range(2)], axis=1)
    R = A @ X
    for zmode in (0, 1, 2):
        ctx.build_operator(zmode=zmode)
        for i in range(2):
            assert _rel(ctx.matvec(X[:, i]), R[:, i]) <= 1e-10, (name, zmode, i)
        Y = ctx.matvec_batch(X)
        for i in range(2):
            assert _rel(Y[:, i], R[:, i]) <= 1e-10, (name, zmode, "batch", i)


@pytest.mark.parametrize("name", voxgen.REDUCED_NAMES)
def test_reduced_capacitance_dense_parity(ctx, name):
    """The bench's path (default build, lockstep pairs for m >= 2) at RRE 1e-12 vs the dense
    direct solve; Maxwell invariants (C_ii > 0, C_ij < 0, row sums >= 0 up to 1e-6)."""
    st, p, A, Cref = _dense(name)
    ctx.set_structure(st)
    ctx.build_operator()
    C, info = ctx.solve_capacitance(tol=1e-12, maxit=6000)
    assert all(i["converged"] for i in info), info
    err = np.abs(C - Cref).max() / np.abs(Cref).max()
    assert err <= 1e-6, (name, err, C, Cref)
    assert (np.diag(C) > 0).all()
    off = C - np.diag(np.diag(C))
    assert (off[~np.eye(p.m, dtype=bool)] < 0).all()
    assert (C.sum(axis=1) >= -1e-6 * np.abs(C).max()).all()
    print(name, "iters", [i["iters"] for i in info], "C rel err", err)
