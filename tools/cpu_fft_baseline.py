"""Like-for-like CPU FFT baseline: one matvec of the same
five-pass dataflow the GPU runs, on the host cores with scipy.fft (workers = all cores) and numpy.

It times the dataflow, not the numbers: the kernel spectra are random real arrays of the shape
the GPU build stores (direct-z: n_K blocks x K_x x (M_y/2 + 1) x ZU offsets; z-FFT mode:
n_K x K_x x (M_y/2 + 1) x (M_z/2 + 1)), so no kernel generation is included.  The panel
geometry (slots, axes, kinds) is the real one, taken from the library's panel table.

  P1 scatter the panel values onto the active planes of each source grid, rfft along x
  P2 fft along y (zero-padded to M_y)
  P3 direct-z: sum over source planes of K(u(z_o - z_i)) Q(z_i) per output plane (numpy MACs on
     (k_y, k_x) slabs); z-FFT mode: fft along z, the 3 x n_f MAC, ifft along z
  P4 ifft along y, keep the field's rows
  P5 irfft along x, gather at the panels

Not the oracle and not the product: a reference timing on the same machine (bench.py reports it
next to the oracle's rows as `cpu_fft_baseline`).
"""
import os
import time

import numpy as np
import scipy.fft as sfft


def time_matvec(panels, grid, n_fields=6, zdirect=True, reps=1, seed=0):
    """panels: dict with axis int8[N], slot int32[N,3], cid int32[N] (library order);
    grid: (Mx, My, Mz).  Returns (seconds per matvec, threads)."""
    axis, slot, cid = panels["axis"], panels["slot"], panels["cid"]
    N = axis.size
    Mx, My, Mz = grid
    Kx = Mx // 2 + 1
    lo = slot.min(axis=0)
    rel = slot - lo
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(N)
    workers = os.cpu_count() or 1
    # source planes per orientation and output planes per field (C^a: conductor a-panels,
    # D^a: dielectric a-panels)
    src = [np.nonzero(axis == a)[0] for a in range(3)]
    fld = [np.nonzero((axis == a) & (cid > 0))[0] for a in range(3)] + \
          [np.nonzero((axis == a) & (cid == 0))[0] for a in range(3)]
    fld = [f for f in fld if f.size][:n_fields]
    zin = [np.unique(rel[s, 2]) for s in src]
    zout = [np.unique(rel[f, 2]) for f in fld]
    ey = int(rel[:, 1].max()) + 1
    ZU = int(max(z.max() for z in zin if z.size)) + 2
    nK = len(fld) * 3
    if zdirect:
        K = rng.standard_normal((nK, ZU, My // 2 + 1, Kx))
    else:
        K = rng.standard_normal((nK, Mz // 2 + 1, My // 2 + 1, Kx))
    t0 = time.perf_counter()
    for _ in range(reps):
        # P1 + P2
        Q = []
        for a in range(3):
            s = src[a]
            if not s.size:
                Q.append(None)
                continue
            planes = zin[a]
            g = np.zeros((planes.size, ey, Mx))
            jz = np.searchsorted(planes, rel[s, 2])
            g[jz, rel[s, 1], np.minimum(rel[s, 0], Mx - 1)] = x[s]
            gx = sfft.rfft(g, axis=2, workers=workers)
            Q.append(sfft.fft(gx, n=My, axis=1, workers=workers))
        # P3
        outs = []
        for fi, f in enumerate(fld):
            po = zout[fi]
            if zdirect:
                acc = np.zeros((po.size, My, Kx), np.complex128)
                for a in range(3):
                    if Q[a] is None:
                        continue
                    Kb = K[fi * 3 + a]
                    Kfull = np.concatenate([Kb, Kb[:, -2:0:-1, :]], axis=1)  # both ky signs
                    for jo, zo in enumerate(po):
                        for ji, zi in enumerate(zin[a]):
                            acc[jo] += Kfull[min(abs(int(zo) - int(zi)), ZU - 1)] * Q[a][ji]
            else:
                acc = None
                for a in range(3):
                    if Q[a] is None:
                        continue
                    qz = np.zeros((Mz, My, Kx), np.complex128)
                    qz[zin[a]] = Q[a]
                    qz = sfft.fft(qz, axis=0, workers=workers)
                    Kb = K[fi * 3 + a]
                    Kz = np.concatenate([Kb, Kb[-2:0:-1]], axis=0)
                    Kz = np.concatenate([Kz, Kz[:, -2:0:-1, :]], axis=1)
                    acc = Kz * qz if acc is None else acc + Kz * qz
                acc = sfft.ifft(acc, axis=0, workers=workers)[po]
            outs.append(acc)
        # P4 + P5 + gather
        y = np.zeros(N)
        for fi, f in enumerate(fld):
            g = sfft.ifft(outs[fi], axis=1, workers=workers)[:, :ey, :]
            r = sfft.irfft(g, n=Mx, axis=2, workers=workers)
            jz = np.searchsorted(zout[fi], rel[f, 2])
            y[f] = r[jz, rel[f, 1], np.minimum(rel[f, 0], Mx - 1)]
    return (time.perf_counter() - t0) / reps, workers
