"""Tucker-compressed kernel spectra (§II.C, Eq. 13) and their
install-time cache file (NEXT-4: P:119), through the C ABI.

The compression is an approximation, so the bar is the stated one carried through: with
tucker_digits = d every block's spectrum keeps ||X - X~||_F <= 10^-d ||X||_F (measured on the
device against the exact table, vc_get_tucker), and the matvec against the dense oracle (which
knows nothing of FFTs or Tucker) stays within 1e-10 relative L2 at d >= 10 -- the exact path's
parity bar -- and within a small multiple of 10^-d below that.  Capacitance at d = 10 within
1e-6 of the oracle's direct solve.  The cache file must reproduce the compressed tables
(to the rounding of its dv = 1 m normalisation, App. C), serve other voxel sizes, and a
corrupted file must be rebuilt, never trusted.
"""
import os

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
        _CACHE[name] = (st, p, A)
    return _CACHE[name]


@pytest.fixture(scope="module")
def ctx():
    c = vc.VoxCap(0)
    yield c
    c.close()


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("name", ["C2", "C4r", "C5r"])
def test_tucker_matvec_vs_dense_oracle(ctx, name):
    st, p, A = _dense(name)
    ctx.set_structure(st)
    X = np.stack([voxgen.seeded_vector(p.n, 60 + i) for i in range(2)], axis=1)
    R = A @ X
    errs = {}
    for d in (6, 8, 10, 12):
        ctx.build_operator(zmode=2, tucker_digits=d)
        tk = ctx.tucker()
        assert tk is not None and tk["nblk"] >= 1
        nkx, nq, ZU = tk["dims"]
        for (r1, r2), e in zip(tk["ranks"], tk["err"]):
            assert 1 <= r1 <= nkx and 1 <= r2 <= nq
            assert e <= 10.0 ** -d, (d, e)  # the HOSVD bound, measured against the exact table
        s = ctx.stats()
        assert s["tucker_err"] == max(tk["err"])
        y = ctx.matvec(X[:, 0])
        errs[d] = _rel(y, R[:, 0])
        Y = ctx.matvec_batch(X)
        assert np.array_equal(Y[:, 0], y)  # the batched launch rebuilds the same K rows
        assert _rel(Y[:, 1], R[:, 1]) <= max(1e-10, 20 * 10.0 ** -d)
        assert errs[d] <= max(1e-10, 20 * 10.0 ** -d), (d, errs[d])
    assert errs[10] <= 1e-10 and errs[12] <= 1e-10
    assert errs[6] > errs[12]  # the error follows the truncation
    print(name, {d: f"{e:.1e}" for d, e in errs.items()})


def test_tucker_capacitance_vs_oracle(ctx):
    st, p, A = _dense("C4r")
    Cref = O.solve_capacitance(p, A=A)
    ctx.set_structure(st)
    ctx.build_operator(zmode=2, tucker_digits=10)
    C, info = ctx.solve_capacitance(tol=1e-12)
    assert all(i["converged"] for i in info)
    assert np.abs(C - Cref).max() <= 1e-6 * np.abs(Cref).max()


def test_tucker_unsupported_and_bad_input(ctx):
    st = voxgen.config("C2")
    ctx.set_structure(st)
    with pytest.raises(vc.VoxCapError) as e:
        ctx.build_operator(zmode=1, tucker_digits=10)  # z-FFT mode: no Tucker P3
    assert e.value.code == "VC_ERR_UNSUPPORTED"
    with pytest.raises(vc.VoxCapError) as e:
        ctx.build_operator(zmode=2, tucker_digits=15)
    assert e.value.code == "VC_ERR_INPUT"
    ctx.build_operator(zmode=2)  # exact spectra again: no Tucker info
    assert ctx.tucker() is None
    assert ctx.stats()["tucker_err"] == 0.0


def test_tucker_cache_roundtrip(ctx, tmp_path):
    st = voxgen.config("C4r")
    ctx.set_structure(st)
    x = voxgen.seeded_vector(ctx.n, 7)
    d = str(tmp_path)
    ctx.build_operator(zmode=2, tucker_digits=10, tucker_cache=d)
    assert ctx.stats()["tucker_cache"] == 2  # written
    files = [f for f in os.listdir(d) if f.startswith("voxcap_tk_") and f.endswith(".bin")]
    assert len(files) == 1
    y1, tk1 = ctx.matvec(x), ctx.tucker()
    ctx.build_operator(zmode=2, tucker_digits=10, tucker_cache=d)
    assert ctx.stats()["tucker_cache"] == 1  # loaded: no generation, no FFTs, no compression
    y2, tk2 = ctx.matvec(x), ctx.tucker()
    # same ranks and errors; the cores went through the dv = 1 m normalisation of the file
    # (App. C scaling), so the matvec agrees to rounding
    assert tk1 == tk2 and _rel(y2, y1) <= 1e-14
    # another voxel size hits the same file (spectra scale as dv^3 / dv^2, App. C)
    st2 = voxgen.config("C4r")
    ctx.set_geometry(st2.label, st2.eps, st2.eps_out, dv=2.5 * st2.dv)
    ctx.build_operator(zmode=2, tucker_digits=10, tucker_cache=d)
    assert ctx.stats()["tucker_cache"] == 1
    y3 = ctx.matvec(x)
    ctx.build_operator(zmode=2, tucker_digits=10)
    assert ctx.stats()["tucker_cache"] == 0
    assert _rel(y3, ctx.matvec(x)) <= 1e-13
    ctx.set_structure(st)
    # another precision is another signature: a second file
    ctx.build_operator(zmode=2, tucker_digits=8, tucker_cache=d)
    assert ctx.stats()["tucker_cache"] == 2
    assert len([f for f in os.listdir(d) if f.endswith(".bin")]) == 2
    # a corrupted payload fails the checksum: rebuilt and rewritten, same bits as a fresh build
    path = os.path.join(d, files[0])
    raw = bytearray(open(path, "rb").read())
    raw[-100] ^= 0xFF
    open(path, "wb").write(bytes(raw))
    ctx.build_operator(zmode=2, tucker_digits=10, tucker_cache=d)
    assert ctx.stats()["tucker_cache"] == 2
    assert np.array_equal(ctx.matvec(x), y1)  # a fresh compression: the same bits as the first
    # an unwritable directory: the build still succeeds, the stat says the write failed
    ctx.build_operator(zmode=2, tucker_digits=10, tucker_cache=os.path.join(d, "missing", "dir"))
    assert ctx.stats()["tucker_cache"] == 3
    assert np.array_equal(ctx.matvec(x), y1)


def test_tucker_full_size_c4(ctx):
    """BASELINE configs[3] at full size: the compressed P3 against the exact one (the exact
    path is itself pinned to the oracle row by row in test_gpu_parity), resident table size."""
    st = voxgen.config("C4")
    ctx.set_structure(st)
    X = np.stack([voxgen.seeded_vector(ctx.n, 80 + i) for i in range(2)], axis=1)
    ctx.build_operator()
    exact_doubles = ctx.stats()["spectra_doubles"]
    Y0 = ctx.matvec_batch(X)
    ctx.build_operator(tucker_digits=10)
    s = ctx.stats()
    tk = ctx.tucker()
    assert s["spectra_doubles"] * 10 < exact_doubles, (s["spectra_doubles"], exact_doubles)
    assert max(tk["err"]) <= 1e-10
    Y = ctx.matvec_batch(X)
    for c in range(2):
        assert _rel(Y[:, c], Y0[:, c]) <= 1e-10
        assert np.array_equal(ctx.matvec(X[:, c]), Y[:, c])
    print("C4 tucker ranks", tk["ranks"], "resident doubles", s["spectra_doubles"], "exact", exact_doubles)


def test_tucker_distributed_slabs():
    """Several ranks (in-process thread group, the same kernels as one process per GPU): each rank
    compresses its own kx slab of the spectra, so the matvec is no longer bitwise the 1-rank one,
    but stays within the Tucker bound of the dense oracle; each rank's cache file is its own."""
    import threading
    st, p, A = _dense("C4r")
    x = voxgen.seeded_vector(p.n, 33)
    ref = A @ x
    W = 2
    grp = vc.ThreadGroup(W)
    ctxs = [vc.VoxCap(0) for _ in range(W)]
    out, err = [None] * W, [None] * W

    def work(r):
        try:
            c = ctxs[r]
            c.init_distributed(r, W, group=grp)
            c.set_structure(st)
            c.build_operator(zmode=2, tucker_digits=10)
            g = c.local_panels()
            out[r] = (g, c.matvec(x[g]), c.tucker())
        except Exception as e:  # pragma: no cover
            err[r] = e

    th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(W)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    assert not any(t.is_alive() for t in th), "distributed ranks hung"
    for c in ctxs:
        c.close()
    grp.close()
    for e in err:
        if e is not None:
            raise e
    y = np.empty(p.n)
    for g, yl, tk in out:
        y[g] = yl
        assert max(tk["err"]) <= 1e-10 and tk["dims"][0] > 0  # each rank: its own kx slab
    assert _rel(y, ref) <= 1e-10
