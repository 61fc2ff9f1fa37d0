"""NEXT-1 measurement (Eq. 13): how Tucker-compressible are the
stored kernel spectra, and what does compressing them do to the matvec?

For every block of the built operator's folded, phase-stripped spectrum table (vc_debug_get_spectra)
the truncated HOSVD (per-mode eigen-decomposition of the unfolding Gram matrices; discarded
energy <= eps^2 ||X||^2 / 3 per mode, so the relative Frobenius error is <= eps) gives the
multilinear ranks (r1, r2, r3) and the compressed size r1 r2 r3 + sum D_i r_i.  The compressed
table (all blocks at one eps) is then written back (vc_debug_set_spectra) and the matvec of a
seeded vector compared with the exact one (relative L2), which is the number that decides
whether a Tucker-compressed P3 could meet the 1e-10 matvec parity bar.

usage: python tools/tucker_ranks.py [--config C4] [--out gpurun_out/tucker_C4.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2004_02609_b200 as vc  # noqa: E402
import voxgen  # noqa: E402

EPS = (1e-4, 1e-6, 1e-8, 1e-10, 1e-12)


def blocks_of(raw, lay):
    """[block][kx][ky][w] views of the tile-major table (direct-z or z-FFT layout)."""
    KY, nt3, T, NW, nb, nkx = lay["KY"], lay["nt3"], lay["T3"], lay["NW"], lay["nblk"], lay["nkx"]
    if lay["zdirect"]:
        t = raw.reshape(KY, nt3, T, lay["RS1"])[..., : nb * NW].reshape(KY, nt3 * T, nb, NW)
        return [np.ascontiguousarray(t[:, :nkx, b, :].transpose(1, 0, 2)) for b in range(nb)]
    rc = raw.size // (KY * nt3)
    t = raw.reshape(KY, nt3, rc)[..., : nb * NW * T].reshape(KY, nt3, nb, NW, T)
    return [np.ascontiguousarray(t[:, :, b].transpose(1, 3, 0, 2).reshape(nt3 * T, KY, NW)[:nkx]) for b in range(nb)]


def write_back(raw, lay, blocks):
    KY, nt3, T, NW, nb, nkx = lay["KY"], lay["nt3"], lay["T3"], lay["NW"], lay["nblk"], lay["nkx"]
    out = raw.copy()
    if lay["zdirect"]:
        t = out.reshape(KY, nt3, T, lay["RS1"])
        v = t[..., : nb * NW].reshape(KY, nt3 * T, nb, NW)
        for b, X in enumerate(blocks):
            v[:, :nkx, b, :] = X.transpose(1, 0, 2)
        t[..., : nb * NW] = v.reshape(KY, nt3, T, nb * NW)
        return out
    rc = raw.size // (KY * nt3)
    t = out.reshape(KY, nt3, rc)
    v = t[..., : nb * NW * T].reshape(KY, nt3, nb, NW, T)
    for b, X in enumerate(blocks):
        pad = np.zeros((nt3 * T, KY, NW))
        pad[:nkx] = X
        v[:, :, b] = pad.reshape(nt3, T, KY, NW).transpose(2, 0, 3, 1)
    t[..., : nb * NW * T] = v.reshape(KY, nt3, nb * NW * T)
    return out


def mode_basis(X, mode):
    """Left singular vectors of the mode-`mode` unfolding (SVD of the unfolding itself: the Gram
    matrix would square the condition number and floor the error near 1e-8)."""
    Xm = np.moveaxis(X, mode, 0).reshape(X.shape[mode], -1)
    U, sv, _ = np.linalg.svd(Xm, full_matrices=False)
    return sv * sv, U


def hosvd(X, eps, bases):
    tot = float(np.sum(X * X))
    ranks, Us = [], []
    for (w, U) in bases:
        tail = np.cumsum(w[::-1])[::-1]  # tail[r] = energy discarded keeping r components
        r = len(w)
        for k in range(len(w) + 1):
            if k == len(w) or tail[k] <= eps * eps * tot / 3.0:
                r = max(k, 1)
                break
        ranks.append(r)
        Us.append(U[:, :r])
    core = np.einsum("abc,ai,bj,ck->ijk", X, Us[0], Us[1], Us[2], optimize=True)
    Xr = np.einsum("ijk,ai,bj,ck->abc", core, Us[0], Us[1], Us[2], optimize=True)
    err = float(np.sqrt(np.sum((Xr - X) ** 2) / max(tot, 1e-300)))
    size = int(np.prod(ranks) + sum(d * r for d, r in zip(X.shape, ranks)))
    return ranks, size, err, Xr


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    st = voxgen.config(a.config)
    ctx = vc.VoxCap(0)
    ctx.set_structure(st)
    ctx.build_operator()
    raw, lay = ctx.spectra()
    x = voxgen.seeded_vector(ctx.n, 0)
    y0 = ctx.matvec(x)
    blocks = blocks_of(raw, lay)
    assert np.array_equal(write_back(raw, lay, blocks), raw)  # the de-tiling round-trips exactly
    res = {"config": a.config, "layout": lay, "grid": list(ctx.grid()), "n": int(ctx.n),
           "table_doubles": int(raw.size), "blocks": []}
    t0 = time.time()
    recon = {e: [] for e in EPS}
    for b, X in enumerate(blocks):
        bases = [mode_basis(X, m) for m in range(3)]
        ent = {"block": b, "shape": list(X.shape), "eps": {}}
        for e in EPS:
            r, size, err, Xr = hosvd(X, e, bases)
            ent["eps"][str(e)] = {"ranks": r, "size": size, "cr": X.size / size, "rel_fro_err": err}
            recon[e].append(Xr)
        res["blocks"].append(ent)
        print("block", b, X.shape, {k: (v["ranks"], round(v["cr"], 1), "%.1e" % v["rel_fro_err"])
                                    for k, v in ent["eps"].items()}, flush=True)
    res["hosvd_s"] = time.time() - t0
    res["matvec"] = {}
    for e in EPS:
        ctx.set_spectra(write_back(raw, lay, recon[e]))
        y = ctx.matvec(x)
        rel = float(np.linalg.norm(y - y0) / np.linalg.norm(y0))
        tot = sum(bb["eps"][str(e)]["size"] for bb in res["blocks"])
        orig = sum(int(np.prod(bb["shape"])) for bb in res["blocks"])
        res["matvec"][str(e)] = {"rel_l2_vs_exact": rel, "compressed_doubles": tot, "cr_all_blocks": orig / tot}
        print("eps %.0e: matvec rel-L2 vs exact %.2e, CR %.1f (%d -> %d doubles)" % (e, rel, orig / tot, orig, tot),
              flush=True)
    ctx.set_spectra(raw)
    assert np.array_equal(ctx.matvec(x), y0)
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
