"""Pins for the oracle's preconditioner box assignment (``precond_boxes``) -- CPU only.

P:137 (§II.D): the bounding box is split into small boxes of N_vx x N_vy x N_vz voxels and
each block of R_BD holds the interactions of the panels in one small box.  The paper does not
say which box a face lying ON a box boundary joins; reading O9 assigns the
panel with slot s along axis a to box min(s // N_va, nbox_a - 1) (the face between voxels
s - 1 and s joins the box of voxel s; the top wall joins the last box).

Pins, none of which re-types the oracle's formula:
  * a hand-worked example (two conductors, anisotropic boxes, both boundary cases and the
    top-wall clamp) with every panel's box written out by hand;
  * a geometric membership property: the panel's centre point lies in its box's half-open
    voxel range on every axis (closed on the top wall), with anisotropic N_v on a non-cubic
    grid so a transposed box index or axis mix-up fails;
  * the paper's P:157 statement that the proposed (conductor-only) R_BD needs about a quarter
    of the memory of the conventional block-diagonal one (all panels blocked) on the coated
    sphere at Δv = 0.01 m, N_v = 10 (paper 17.04 vs 70.26 MB).
"""
import numpy as np

import oracle as O
import voxgen


def _hand_structure():
    # dims (nx, ny, nz) = (5, 3, 2); label is [z, y, x]
    lab = np.zeros((2, 3, 5), np.int32)
    lab[0, 1, 1:4] = 1          # bar: voxels x = 1..3, y = 1, z = 0
    lab[1, 0, 0] = 2            # single voxel x = 0, y = 0, z = 1 (no shared face with the bar)
    return lab


def test_precond_boxes_hand_worked():
    """N_v = (2, 2, 1) on a 5 x 3 x 2 grid: nbox = (3, 2, 2); box id = (bz*2 + by)*3 + bx.
    Worked by hand from P:137 + reading O9, in canonical panel order (axis-major, then k, j, i)."""
    p = O.enumerate_panels(_hand_structure())
    # slots (i, j, k) written out by hand
    slots = [
        # x-normal: bar -x end (1,1,0), bar +x end (4,1,0); voxel 2: -x wall (0,0,1), +x (1,0,1)
        (1, 1, 0), (4, 1, 0), (0, 0, 1), (1, 0, 1),
        # y-normal: bar j = 1 (i = 1..3), bar j = 2 (i = 1..3), voxel 2 j = 0 and j = 1
        (1, 1, 0), (2, 1, 0), (3, 1, 0), (1, 2, 0), (2, 2, 0), (3, 2, 0), (0, 0, 1), (0, 1, 1),
        # z-normal: bar k = 0, voxel 2 bottom (0,0,1), bar k = 1, voxel 2 top (0,0,2)
        (1, 1, 0), (2, 1, 0), (3, 1, 0), (0, 0, 1), (1, 1, 1), (2, 1, 1), (3, 1, 1), (0, 0, 2),
    ]
    assert p.n == 20
    assert np.array_equal(p.slot, np.array(slots, np.int32))
    # boxes by hand:
    #  (4,1,0) x-face: between voxel 3 (box x 1) and voxel 4 -> box x 2 (boundary face, O9)
    #  (1,2,0) y-face: between row 1 and row 2 -> box y 1; (1,0,1) x-face: 1 // 2 = 0
    #  (1,1,1) z-face: top of the bar = bottom of layer 1 -> box z 1
    #  (0,0,2) z-face: top wall, 2 // 1 = 2 clamped to nbox_z - 1 = 1
    boxes_xyz = [
        (0, 0, 0), (2, 0, 0), (0, 0, 1), (0, 0, 1),
        (0, 0, 0), (1, 0, 0), (1, 0, 0), (0, 1, 0), (1, 1, 0), (1, 1, 0), (0, 0, 1), (0, 0, 1),
        (0, 0, 0), (1, 0, 0), (1, 0, 0), (0, 0, 1), (0, 0, 1), (1, 0, 1), (1, 0, 1), (0, 0, 1),
    ]
    want = [(bz * 2 + by) * 3 + bx for bx, by, bz in boxes_xyz]
    got = O.precond_boxes(p, nv=(2, 2, 1))
    assert got.tolist() == want


def _centre(p):
    """Geometric centre of each panel in voxel units: the face plane along its own axis,
    mid-voxel along the other two."""
    c = p.slot.astype(np.float64) + 0.5
    ax = p.axis.astype(np.int64)
    c[np.arange(p.n), ax] -= 0.5
    return c


def test_precond_boxes_geometric_membership():
    """Every panel's centre lies inside its box: b_a N_va <= c_a < (b_a + 1) N_va per axis
    (c_a = N_a allowed on the top wall of the last box); anisotropic N_v on a non-cubic grid
    with dielectrics, so swapped axes or a transposed index would fail."""
    for seed in (1, 2, 3, 4):
        st = voxgen.random_structure(seed)
        p = O.enumerate_panels(st.label, st.eps, st.eps_out, st.dv)
        nv = (2, 3, 5)
        nbox = [-(-p.dims[a] // nv[a]) for a in range(3)]
        box = O.precond_boxes(p, nv)
        bx = box % nbox[0]
        by = (box // nbox[0]) % nbox[1]
        bz = box // (nbox[0] * nbox[1])
        assert (bz < nbox[2]).all()
        c = _centre(p)
        for a, b in enumerate((bx, by, bz)):
            lo, hi = b * nv[a], np.minimum((b + 1) * nv[a], p.dims[a])
            inside = (lo <= c[:, a]) & ((c[:, a] < hi) | ((c[:, a] == p.dims[a]) & (hi == p.dims[a])))
            assert inside.all(), (seed, a)


def _block_bytes(p, box, sel):
    _, counts = np.unique(box[sel], return_counts=True)
    return 8.0 * float((counts.astype(np.int64) ** 2).sum())


def test_precond_memory_quarter_of_conventional():
    """on the coated sphere (r_c = 0.25 m, r_d = 0.5 m, ε_r = 2, Δv = 0.01 m, N = 59,016
    (P:153), N_v = 10) the proposed R_BD (conductor panels only, reading O9) needs about a
    quarter of the memory of the conventional block-diagonal preconditioner whose blocks hold
    every panel in the box (paper: 17.04 MB vs 70.26 MB).  Dense fp64 blocks, MB = 1e6 B.
    Measured with this reading: 12.4 MB vs 68.8 MB (the conventional figure within 3% of the
    paper; the proposed one smaller than the paper's, DESIGN.md §3 O9)."""
    st = voxgen.coated_sphere(25, 50, 2.0, dv=0.01)
    p = O.enumerate_panels(st.label, st.eps, st.eps_out, st.dv)
    assert p.n == 59016
    box = O.precond_boxes(p, (10, 10, 10))
    prop = _block_bytes(p, box, p.is_cond) / 1e6
    conv = _block_bytes(p, box, np.ones(p.n, bool)) / 1e6
    assert abs(conv / 70.26 - 1) < 0.03, conv
    assert prop < conv / 4, (prop, conv)
