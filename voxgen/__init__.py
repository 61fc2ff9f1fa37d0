"""Seeded synthetic voxel structures shaped like the paper's workloads.

This module holds NO arithmetic of the method (no panel rules, no kernels, no FFT, no
solver): it only produces voxel label / permittivity arrays and seeded right-hand vectors.
It is the one module both the CPU oracle (``oracle/``) and the CUDA path's tests/bench use.

Array conventions:
  * ``label``: int32 array of shape (Nz, Ny, Nx) (x fastest in memory); 0 = non-conductor,
    1..m = conductor id.
  * ``eps``: float64 array of the same shape, relative permittivity of each non-conductor
    voxel (ignored on conductor voxels); ``eps_out`` is the medium outside the box.

Configs C1..C5 follow BASELINE.json ``configs`` as concretised in SURVEY.md §8(d):
  C1 8^3 cube (P:147-style free-space conductor), C2 two plates + eps_r 4 slab, C3 voxelised
  sphere R=64 in 128^3, C4 two parallel meander lines over an eps_r 4.4 substrate
  (512x512x64; the paper's §III.E meander), C5 16x16 crossing bus in three
  dielectric layers (2048x2048x128; the paper's §III.D crossing bus).  R1..R5 are
  the small random parity structures of SURVEY.md §8(d).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "Structure", "cube", "plates_slab", "sphere", "coated_sphere", "meander", "crossing_bus",
    "random_structure", "config", "CONFIG_NAMES", "REDUCED_NAMES", "seeded_vector",
]


class Structure:
    """A voxelised structure: label, eps, eps_out, dv (metres) and a name."""

    def __init__(self, label, eps, eps_out=1.0, dv=1e-6, name=""):
        self.label = np.ascontiguousarray(label, dtype=np.int32)
        self.eps = np.ascontiguousarray(eps, dtype=np.float64)
        assert self.label.shape == self.eps.shape and self.label.ndim == 3
        self.eps_out = float(eps_out)
        self.dv = float(dv)
        self.name = name

    @property
    def dims(self):
        """(Nx, Ny, Nz)."""
        nz, ny, nx = self.label.shape
        return nx, ny, nz

    @property
    def m(self):
        return int(self.label.max())

    def __repr__(self):
        return f"Structure({self.name!r}, dims={self.dims}, m={self.m}, dv={self.dv})"


def _empty(nx, ny, nz, eps_fill=1.0):
    return np.zeros((nz, ny, nx), np.int32), np.full((nz, ny, nx), eps_fill, np.float64)


def cube(n=8, dv=1e-6):
    """C1: an n^3 conductor filling the whole box, free space (BASELINE configs[0])."""
    label, eps = _empty(n, n, n)
    label[:] = 1
    return Structure(label, eps, 1.0, dv, f"cube{n}")


def plates_slab(nx=32, ny=32, gap=4, eps_r=4.0, dv=1e-6):
    """C2: two nx*ny*1 plates separated by a ``gap``-voxel eps_r slab (BASELINE configs[1])."""
    nz = gap + 2
    label, eps = _empty(nx, ny, nz)
    label[0] = 1
    label[nz - 1] = 2
    eps[1:nz - 1] = eps_r
    return Structure(label, eps, 1.0, dv, "plates_slab")


def sphere(R=64, dv=1e-6, n=None):
    """C3: voxel-centre-inside sphere of radius R voxels centred in a (2R)^3 box (O16)."""
    n = 2 * R if n is None else n
    label, eps = _empty(n, n, n)
    c = np.arange(n) + 0.5 - n / 2.0
    zz, yy, xx = np.meshgrid(c, c, c, indexing="ij")
    label[(xx * xx + yy * yy + zz * zz) < R * R] = 1
    return Structure(label, eps, 1.0, dv, f"sphere{R}")


def coated_sphere(rc_vox, rd_vox, eps_r=2.0, dv=1.0, margin=0):
    """§III.A dielectric-coated PEC sphere: conductor radius rc, shell radius rd."""
    n = int(2 * rd_vox + 2 * margin)
    label, eps = _empty(n, n, n)
    c = np.arange(n) + 0.5 - n / 2.0
    zz, yy, xx = np.meshgrid(c, c, c, indexing="ij")
    d2 = xx * xx + yy * yy + zz * zz
    eps[d2 < rd_vox * rd_vox] = eps_r
    label[d2 < rc_vox * rc_vox] = 1
    return Structure(label, eps, 1.0, dv, f"coated_sphere{rc_vox}_{rd_vox}")


def meander(seed=0, nx=512, ny=512, nz=64, sub=16, eps_r=4.4, dv=1e-6,
            width=2, thick=2, pitch=4, run_pitch=12, run_min=400, run_max=500, edge=16):
    """C4: two parallel meander lines over a ``sub``-voxel eps_r substrate (P:238-257 shape).

    The pair follows a serpentine centre path: runs along x with lengths
    ``rng.integers(run_min, run_max)`` (clamped to the box), ``run_pitch`` apart in y, joined
    by U-turns.  Line 1 is the path offset by -pitch/2 and line 2 by +pitch/2 to the left of
    the direction of travel, so the two lines are ``pitch`` apart centre to centre everywhere
    and the U-turns nest.  Each line is a band ``width`` voxels wide and ``thick`` voxels thick
    lying on the substrate (z in [sub, sub+thick)).  The substrate leaves a one-voxel margin at
    the +x/+y walls.  ``edge`` is the clearance of the serpentine from the walls
    (16 at full size; the reduced parity grids use a smaller one).
    """
    rng = np.random.default_rng(seed)
    label, eps = _empty(nx, ny, nz)
    eps[:sub, : ny - 1, : nx - 1] = eps_r
    z0, z1 = sub, sub + thick
    lo_edge, hi_edge = edge, nx - edge - 1
    hw = width // 2
    x = lo_edge
    y = edge
    d = +1
    runs = []  # (x_start, x_end, y, direction)
    while y + edge < ny - edge:
        L = int(rng.integers(run_min, run_max))
        xe = min(max(x + d * L, lo_edge), hi_edge)
        runs.append((x, xe, y, d))
        x, y, d = xe, y + run_pitch, -d

    def band_h(cid, xa, xb, yc):
        label[z0:z1, yc - hw:yc + width - hw, min(xa, xb) - hw:max(xa, xb) + width - hw] = cid

    def band_v(cid, xc, ya, yb):
        label[z0:z1, min(ya, yb) - hw:max(ya, yb) + width - hw, xc - hw:xc + width - hw] = cid

    half = pitch // 2
    for cid, o in ((1, -half), (2, +half)):
        for r, (xs, xe, yc, dr) in enumerate(runs):
            # left of +x travel is +y, left of -x travel is -y; the vertical legs travel +y,
            # whose left is -x: a leg at centre x = X sits at X - o for this line.
            yl = yc + o * dr
            xa = xs - o if r > 0 else xs
            xb = xe - o if r + 1 < len(runs) else xe
            band_h(cid, xa, xb, yl)
            if r + 1 < len(runs):
                yn = runs[r + 1][2] + o * runs[r + 1][3]
                band_v(cid, xb, yl, yn)
    return Structure(label, eps, 1.0, dv, f"meander_s{seed}")


def crossing_bus(seed=0, nx=2048, ny=2048, nz=128, n_lines=16, w=4, dv=1e-6,
                 layers=((0, 40, 3.9), (40, 80, 7.0), (80, 127, 2.5)), edge=16, end=8, jitter=8):
    """C5: 16 lines along x in the lower layer crossing 16 lines along y in the upper layer,
    each w x w voxels, in three dielectric layers (eps_r 3.9 / 7.0 / 2.5) over x,y in
    [0, n-1) (one-voxel margin); seeded pitch and offsets (the §III.D crossing-bus shape,
    P:218).  ``edge`` / ``jitter`` (first-line offset and pitch jitter) and ``end`` (line-end
    clearance) are 16 / 8 / 8 at full size; the reduced parity grids use smaller ones."""
    rng = np.random.default_rng(seed)
    label, eps = _empty(nx, ny, nz)
    for z0, z1, e in layers:
        eps[z0:z1, : ny - 1, : nx - 1] = e
    zl = (layers[0][0] + layers[0][1]) // 2 - w // 2
    zu = (layers[1][0] + layers[1][1]) // 2 - w // 2
    span = min(nx, ny) - 2 * edge
    pitch = int(rng.integers(span // (n_lines + 1) - jitter, span // (n_lines + 1)))
    off_a = edge + int(rng.integers(0, jitter))
    off_b = edge + int(rng.integers(0, jitter))
    cid = 1
    for i in range(n_lines):
        y0 = off_a + i * pitch
        label[zl:zl + w, y0:y0 + w, end:nx - end - 1] = cid
        cid += 1
    for i in range(n_lines):
        x0 = off_b + i * pitch
        label[zu:zu + w, end:ny - end - 1, x0:x0 + w] = cid
        cid += 1
    return Structure(label, eps, 1.0, dv, f"crossing_bus_s{seed}")


def random_structure(seed, margin=None):
    """R1..R5 parity structures: grid from {6..12}x{6..12}x{4..8}; 1-3
    conductors (random boxes, >= 1 voxel apart); 0-2 dielectric boxes with eps_r ~ U(1.5, 10)
    that may touch conductors and each other.  Even seeds keep a one-voxel margin, odd seeds
    let dielectrics touch the walls (both padding rules, O11)."""
    rng = np.random.default_rng(1000 + seed)
    nx, ny = int(rng.integers(6, 13)), int(rng.integers(6, 13))
    nz = int(rng.integers(4, 9))
    margin = (seed % 2 == 0) if margin is None else margin
    label, eps = _empty(nx, ny, nz)
    n_die = int(rng.integers(0, 3))
    for _ in range(n_die):
        lo = [int(rng.integers(0, d - 1)) for d in (nz, ny, nx)]
        hi = [int(rng.integers(l + 1, d + 1)) for l, d in zip(lo, (nz, ny, nx))]
        if margin:
            lo = [max(l, 1) for l in lo]
            hi = [min(h, d - 1) for h, d in zip(hi, (nz, ny, nx))]
            if any(h <= l for l, h in zip(lo, hi)):
                continue
        eps[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]] = float(rng.uniform(1.5, 10.0))
    m_target = int(rng.integers(1, 4))
    cid = 0
    tries = 0
    while cid < m_target and tries < 200:
        tries += 1
        sz = [int(rng.integers(1, min(4, d) + 1)) for d in (nz, ny, nx)]
        lo = [int(rng.integers(0, d - s + 1)) for d, s in zip((nz, ny, nx), sz)]
        hi = [l + s for l, s in zip(lo, sz)]
        # keep >= 1 voxel from other conductors (touching conductors are an input error)
        zl, yl, xl = [max(l - 1, 0) for l in lo]
        zh, yh, xh = [h + 1 for h in hi]
        if label[zl:zh, yl:yh, xl:xh].any():
            continue
        cid += 1
        label[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]] = cid
    if cid == 0:
        label[nz // 2, ny // 2, nx // 2] = 1
    return Structure(label, eps, 1.0, 1e-6, f"R{seed}")


CONFIG_NAMES = ("C1", "C2", "C3", "C4", "C5")

# Reduced grids of the C3 / C4 / C5 generators, small enough for the dense oracle (SURVEY.md
# §8(c) last pins row: "pinned on the same generator at reduced grids").  C3r = C3 / 4 per
# axis; C4r = the C4 meander pair (2 x 2 lines, pitch 4, run pitch 12, three U-turns) on a
# 48 x 48 x 8 box with a 4-voxel eps_r 4.4 substrate; C5r = C5 / 64 in x, y,
# / 8 in z with 2 + 2 lines of 2 x 2 voxels in the same three layers.
REDUCED_NAMES = ("C3r", "C4r", "C5r")


def config(name, seed=0):
    """Structures for BASELINE.json configs[0..4] (SURVEY.md §8(d) concretisation)."""
    if name == "C1":
        return cube(8)
    if name == "C2":
        return plates_slab()
    if name == "C3":
        return sphere(64)
    if name == "C4":
        return meander(seed)
    if name == "C5":
        return crossing_bus(seed)
    if name == "C3r":
        return sphere(16)
    if name == "C4r":
        return meander(seed, 48, 48, 8, sub=4, run_min=24, run_max=32, edge=6)
    if name == "C5r":
        return crossing_bus(seed, 32, 32, 16, n_lines=2, w=2, edge=4, end=2, jitter=2,
                            layers=((0, 5, 3.9), (5, 10, 7.0), (10, 15, 2.5)))
    if name.startswith("R"):
        return random_structure(int(name[1:]))
    raise KeyError(name)


def seeded_vector(n, seed):
    """x ~ N(0, 1), float64, seeded (SURVEY.md §8(d) matvec inputs)."""
    return np.random.default_rng(seed).standard_normal(n)
