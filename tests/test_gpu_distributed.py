"""Distributed (slab-partitioned) path on one GPU: W ranks as an in-process thread group.

Every rank runs the same kernels as a real multi-GPU run; only the transport differs (stream-
ordered peer copies instead of NCCL).  The partitioned matvec must be BITWISE equal to the
1-rank matvec (each pencil is transformed by the same plan, only its placement changes; SURVEY
§4 item 5); solves and capacitance agree to solver tolerance (dot products are summed over
ranks in a different order) and with the CPU oracle.
"""
import threading
import time

import numpy as np
import pytest

import oracle as O
import voxgen

pytestmark = pytest.mark.gpu

try:
    import paper_2004_02609_b200 as vc
except Exception:  # pragma: no cover
    vc = None


def _group(W, st, fn, timeout=600, **build):
    grp = vc.ThreadGroup(W)
    ctxs = [vc.VoxCap(0) for _ in range(W)]
    out, err = [None] * W, [None] * W

    def work(r):
        try:
            c = ctxs[r]
            c.init_distributed(r, W, group=grp)
            c.set_structure(st)
            c.build_operator(**build)
            out[r] = fn(c, r)
        except Exception as e:  # pragma: no cover - surfaced below
            err[r] = e

    th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(W)]
    for t in th:
        t.start()
    t0 = time.time()
    while any(t.is_alive() for t in th) and time.time() - t0 < timeout:
        # a rank that failed leaves its peers waiting at the next collective: surface it now
        for e in err:
            if e is not None:
                raise e
        time.sleep(0.05)
    assert not any(t.is_alive() for t in th), "distributed ranks hung"
    for c in ctxs:
        c.close()
    grp.close()
    for e in err:
        if e is not None:
            raise e
    return out


def _single(st, fn, **build):
    with vc.VoxCap(0) as c:
        c.set_structure(st)
        c.build_operator(**build)
        return fn(c)


CASES = [("R1", 2, 0), ("R2", 3, 0), ("R3", 2, 1), ("R3", 2, 2), ("R4", 4, 0), ("R5", 2, 1),
         ("C2", 2, 2), ("C2", 3, 1), ("sphere12", 2, 0), ("C1", 8, 0)]


def _st(name):
    return voxgen.sphere(12) if name == "sphere12" else voxgen.config(name)



@pytest.mark.parametrize("name,W,zmode", CASES)
def test_distributed_matvec_bitwise(name, W, zmode):
    st = _st(name)
    box = (4, 4, 4)
    n = _single(st, lambda c: c.n, box=box)
    x = voxgen.seeded_vector(n, 21)
    # (multi-rank builds generate every kernel block; mirror=False makes the 1-rank build do the same)
    y1 = _single(st, lambda c: c.matvec(x), box=box, zmode=zmode, mirror=False)
    res = _group(W, st, lambda c, r: (c.local_panels(), c.matvec(x[c.local_panels()])), box=box,
                 zmode=zmode)
    idx = np.concatenate([g for g, _ in res])
    assert np.array_equal(np.sort(idx), np.arange(n)), "ranks must partition the panels"
    yd = np.empty(n)
    for g, yl in res:
        yd[g] = yl
    assert np.array_equal(yd, y1)


@pytest.mark.parametrize("name,W", [("R5", 2), ("C2", 3)])
def test_distributed_precond(name, W):
    st = _st(name)
    box = (4, 4, 4)
    n = _single(st, lambda c: c.n, box=box)
    r = voxgen.seeded_vector(n, 5)
    z1 = _single(st, lambda c: c.precond(r), box=box)
    res = _group(W, st, lambda c, k: (c.local_panels(), c.precond(r[c.local_panels()])), box=box)
    zd = np.empty(n)
    for g, zl in res:
        zd[g] = zl
    assert np.array_equal(zd, z1)


@pytest.mark.parametrize("name,W", [("C1", 2), ("R2", 2), ("C2", 2), ("R4", 3)])
def test_distributed_capacitance(name, W):
    st = _st(name)
    C1, _ = _single(st, lambda c: c.solve_capacitance(tol=1e-12, maxit=4000))
    res = _group(W, st, lambda c, r: c.solve_capacitance(tol=1e-12, maxit=4000))
    p = O.enumerate_panels(st.label, st.eps, st.eps_out, st.dv)
    Cref = O.solve_capacitance(p)
    for C, info in res:
        assert all(i["converged"] for i in info)
        assert np.array_equal(C, res[0][0]), "every rank returns the same matrix"
        assert np.abs(C - C1).max() <= 1e-9 * np.abs(C1).max()
        assert np.abs(C - Cref).max() <= 1e-6 * np.abs(Cref).max()


def test_distributed_solve_matches_single():
    st = voxgen.config("R5")
    box = (4, 4, 4)
    n = _single(st, lambda c: c.n, box=box)
    b = voxgen.seeded_vector(n, 9)
    x1, _ = _single(st, lambda c: c.solve(b, tol=1e-12, maxit=2000), box=box)
    res = _group(2, st, lambda c, r: (c.local_panels(), c.solve(b[c.local_panels()], tol=1e-12,
                                                                maxit=2000)), box=box)
    xd = np.empty(n)
    for g, (xl, info) in res:
        assert info["converged"]
        xd[g] = xl
    assert np.linalg.norm(xd - x1) <= 1e-9 * np.linalg.norm(x1)


@pytest.mark.parametrize("name,W", [("C2", 2), ("C2", 3), ("R2", 2), ("C5r", 4)])
def test_distributed_batch_bitwise(name, W):
    """Batched matvecs (two columns per launch chain, NEXT-3) on W ranks: every column equals the
    1-rank single-column matvec bitwise (direct-z builds, where multi-rank batching applies)."""
    st = _st(name)
    n = _single(st, lambda c: c.n, zmode=2)
    X = np.stack([voxgen.seeded_vector(n, 31), voxgen.seeded_vector(n, 32)], axis=1)
    Y1 = np.stack([_single(st, lambda c: c.matvec(X[:, i]), zmode=2, mirror=False) for i in range(2)], axis=1)
    def fn(c, r):
        g = c.local_panels()
        c.reset_stats()
        Y = c.matvec_batch(np.ascontiguousarray(X[g]))
        s = c.stats()
        return g, Y, (s["n_matvec"], s["n_pass"][0])

    res = _group(W, st, fn, zmode=2)
    Yd = np.empty_like(Y1)
    for g, yl, cnt in res:
        Yd[g] = yl
        assert cnt == (2, 1), cnt  # both columns in one launch chain
    assert np.array_equal(Yd, Y1)


@pytest.mark.parametrize("W", [2, 8])
def test_distributed_full_size_c4_rows(W):
    """BASELINE C4 at full size split over W ranks (W = 8: one node's worth): the distributed
    matvec -- single and batched pair -- equals the 1-rank one bitwise."""
    st = voxgen.config("C4")
    n = _single(st, lambda c: c.n)
    x = voxgen.seeded_vector(n, 0)
    x2 = voxgen.seeded_vector(n, 1)
    y1 = _single(st, lambda c: c.matvec(x), mirror=False)
    y2 = _single(st, lambda c: c.matvec(x2), mirror=False)

    def fn(c, r):
        g = c.local_panels()
        return g, c.matvec(x[g]), c.matvec_batch(np.stack([x[g], x2[g]], axis=1))

    res = _group(W, st, fn, timeout=1200)
    yd, Yd = np.empty(n), np.empty((n, 2))
    for g, yl, Yl in res:
        yd[g] = yl
        Yd[g] = Yl
    assert np.array_equal(yd, y1)
    assert np.array_equal(Yd[:, 0], y1) and np.array_equal(Yd[:, 1], y2)


def test_nccl_transport_world1():
    """The NCCL transport on the one GPU a test box has (the NCCL code never ran):
    libnccl loads, a unique id is drawn, a world-1 communicator initialises, ncclAllReduce and a
    grouped ncclSend / ncclRecv (this rank as its own peer) move the right bytes, and a
    capacitance extraction through a context initialised with the NCCL transport equals the
    plain one bitwise."""
    st = voxgen.config("C2")
    C0, _ = _single(st, lambda c: c.solve_capacitance(tol=1e-10, maxit=4000))
    with vc.VoxCap(0) as c:
        c.init_distributed(0, 1, nccl_id=vc.nccl_unique_id())
        out = c.nccl_selftest()
        assert np.array_equal(out, [1, 2, 3, 4, 1, 2, 3, 4]), out
        c.set_structure(st)
        c.build_operator()
        C1, info = c.solve_capacitance(tol=1e-10, maxit=4000)
    assert all(i["converged"] for i in info)
    assert np.array_equal(C1, C0)
