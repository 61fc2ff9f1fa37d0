"""VoxCap CPU oracle -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Plain definitions, no FFT, no circulants, no Tables VI-X.  Panel-pair
integrals come from ``kernels_q.c`` (binary128 closed forms, one corner sum per entry); the
dense algebra uses numpy / LAPACK as library primitives.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

__all__ = [
    "EPS0", "OracleInputError", "Panels", "build_lib", "kappa", "kappa_hilo", "kappa_batch",
    "enumerate_panels", "rows_of", "assemble", "matvec", "matvec_rows", "solve",
    "solve_capacitance", "capacitance_from_rho", "precond_boxes", "precond_apply",
]

EPS0 = 8.8541878128e-12  # F/m (reading O15)
FOUR_PI_EPS0 = 4.0 * np.pi * EPS0

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "kernels_q.c")
_SO = os.path.join(_HERE, "_liboracle_q.so")
_lock = threading.Lock()
_lib = None


class OracleInputError(ValueError):
    """Invalid voxel structure (mirrors the ABI's VC_ERR_INPUT cases)."""


# --------------------------------------------------------------------------------------------
# binary128 closed forms (oracle/kernels_q.c)
# --------------------------------------------------------------------------------------------
def build_lib(force=False):
    """Compile oracle/kernels_q.c (gcc, libquadmath, OpenMP).  Returns the .so path."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", tmp, _SRC,
                               "-lquadmath", "-lm"])
        os.replace(tmp, _SO)
    return _SO


def _get_lib():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build_lib())
            i32, i64, dbl = ctypes.c_int, ctypes.c_int64, ctypes.c_double
            lib.oq_kappa.restype = dbl
            lib.oq_kappa.argtypes = [i32, i32, i32, i64, i64, i64]
            lib.oq_kappa_hilo.restype = None
            lib.oq_kappa_hilo.argtypes = [i32, i32, i32, i64, i64, i64,
                                          ctypes.POINTER(dbl), ctypes.POINTER(dbl)]
            lib.oq_kappa_batch.restype = None
            lib.oq_kappa_batch.argtypes = [i64, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
            _lib = lib
    return _lib


def kappa(kind, alpha, beta, d):
    """Unit-voxel panel-pair integral (Δv = 1, 4πε0 = 1).

    kind 0: P (Eq. 5); kind 1: E+ (Eq. 6 along +alpha at the observer; App. A
    Eqs. 15-16).  ``alpha`` = observer (testing) panel normal, ``beta`` = source
    normal (0,1,2 = x,y,z); ``d`` = observer slot - source slot (integers, P:97 grids).
    """
    return _get_lib().oq_kappa(int(kind), int(alpha), int(beta), int(d[0]), int(d[1]),
                               int(d[2]))


def kappa_hilo(kind, alpha, beta, d):
    """kappa as an unevaluated double-double (hi, lo) -- binary128 rounded to 2 doubles."""
    hi, lo = ctypes.c_double(), ctypes.c_double()
    _get_lib().oq_kappa_hilo(int(kind), int(alpha), int(beta), int(d[0]), int(d[1]),
                             int(d[2]), ctypes.byref(hi), ctypes.byref(lo))
    return hi.value, lo.value


def kappa_batch(kind, alpha, beta, d):
    """Vectorised :func:`kappa` (OpenMP over entries)."""
    d = np.ascontiguousarray(d, dtype=np.int64).reshape(-1, 3)
    n = d.shape[0]
    kind = np.ascontiguousarray(np.broadcast_to(kind, (n,)), dtype=np.int32)
    alpha = np.ascontiguousarray(np.broadcast_to(alpha, (n,)), dtype=np.int32)
    beta = np.ascontiguousarray(np.broadcast_to(beta, (n,)), dtype=np.int32)
    out = np.empty(n, np.float64)
    if n:
        _get_lib().oq_kappa_batch(n, kind.ctypes.data, alpha.ctypes.data, beta.ctypes.data,
                                  d.ctypes.data, out.ctypes.data)
    return out


# --------------------------------------------------------------------------------------------
# panel enumeration (a1)
# --------------------------------------------------------------------------------------------
class Panels:
    """Boundary panels in canonical order (axis-major, then k, j, i with i fastest; O14).

    Fields (length N): axis int8 (0,1,2 = x,y,z); slot int32 [N,3] as (i,j,k) on the axis
    grid of P:97; sign int8 (+1 if the normal is +axis); cid int32 (1..m conductor, 0
    dielectric); eps_d, eps_b float64 (dielectric: the two sides per O7; conductor: eps_d = 0,
    eps_b = eps_r of the medium the normal points into); ibar float64 (Eq. 7, SI; 0 on
    conductor rows); fc float64 (free-charge factor O8; 0 on dielectric rows).
    """

    def __init__(self, dims, dv, m, axis, slot, sign, cid, eps_d, eps_b):
        self.dims = tuple(int(v) for v in dims)
        self.dv = float(dv)
        self.m = int(m)
        self.axis = axis
        self.slot = slot
        self.sign = sign
        self.cid = cid
        self.eps_d = eps_d
        self.eps_b = eps_b
        self.is_cond = cid > 0
        area = self.dv * self.dv
        with np.errstate(divide="ignore", invalid="ignore"):
            ib = area * (eps_d + eps_b) / (2.0 * EPS0 * (eps_d - eps_b))  # Eq. (7)
        self.ibar = np.where(self.is_cond, 0.0, ib)
        self.fc = np.where(self.is_cond, eps_b, 0.0)

    @property
    def n(self):
        return int(self.axis.shape[0])

    @property
    def n_cond(self):
        return int(self.is_cond.sum())

    @property
    def n_diel(self):
        return self.n - self.n_cond


def enumerate_panels(label, eps=None, eps_out=1.0, dv=1.0):
    """Classify every voxel face (P:47, P:53-57, P:97 grids, P:115 signs; readings O7, O8).

    ``label`` int array (Nz, Ny, Nx): 0 = non-conductor, 1..m = conductor id.  ``eps``:
    relative permittivity of non-conductor voxels (None = 1).  The face between voxel u and
    u + e_a (outside the box = non-conductor with ``eps_out``) is
      * a conductor panel if exactly one side is a conductor voxel: cid = that conductor,
        sign = +1 iff the conductor is on the lower side (outward normal +a), medium eps =
        eps of the other side;
      * a dielectric panel if neither side is a conductor and the permittivities differ:
        the d side is the non-background side if one side equals eps_out, else the higher-eps
        side; sign = +1 iff d is the lower side (normal from d into b).
    Two different conductors sharing a face is an input error.
    """
    label = np.asarray(label)
    if label.ndim != 3 or min(label.shape) <= 0:
        raise OracleInputError("label must be a non-empty 3-D array")
    if not dv > 0 or not np.isfinite(dv):
        raise OracleInputError("dv must be positive")
    if eps is None:
        eps = np.ones(label.shape)
    eps = np.asarray(eps, dtype=np.float64)
    if eps.shape != label.shape:
        raise OracleInputError("eps shape mismatch")
    label = label.astype(np.int64)
    if (label < 0).any():
        raise OracleInputError("negative label")
    m = int(label.max())
    if m == 0:
        raise OracleInputError("empty structure (no conductor)")
    present = np.unique(label[label > 0])
    if present.size != m or present[0] != 1:
        raise OracleInputError("conductor ids must be exactly 1..m")
    nonc = label == 0
    if not (np.isfinite(eps[nonc]).all() and (eps[nonc] > 0).all()):
        raise OracleInputError("eps must be finite and > 0")
    if not (np.isfinite(eps_out) and eps_out > 0):
        raise OracleInputError("eps_out must be finite and > 0")
    nz, ny, nx = label.shape
    cols = {k: [] for k in ("axis", "i", "j", "k", "sign", "cid", "eps_d", "eps_b")}
    for a, npax in ((0, 2), (1, 1), (2, 0)):  # x, y, z and the numpy axis they map to
        pad = [(0, 0)] * 3
        pad[npax] = (1, 1)
        lab = np.pad(label, pad, constant_values=0)
        ep = np.pad(np.where(label > 0, 0.0, eps), pad, constant_values=eps_out)
        sl_lo = [slice(None)] * 3
        sl_hi = [slice(None)] * 3
        sl_lo[npax] = slice(0, -1)
        sl_hi[npax] = slice(1, None)
        lo, hi = lab[tuple(sl_lo)], lab[tuple(sl_hi)]
        elo, ehi = ep[tuple(sl_lo)], ep[tuple(sl_hi)]
        cl, ch = lo > 0, hi > 0
        if (cl & ch & (lo != hi)).any():
            raise OracleInputError("two different conductors share a face")
        is_c = cl ^ ch
        is_d = (~cl) & (~ch) & (elo != ehi)
        d_lo = np.where(elo == eps_out, False, np.where(ehi == eps_out, True, elo > ehi))
        face = is_c | is_d
        kk, jj, ii = np.nonzero(face)  # lexicographic (k, j, i), i fastest (O14)
        fc_ = is_c[kk, jj, ii]
        cl_ = cl[kk, jj, ii]
        dl_ = d_lo[kk, jj, ii]
        lo_, hi_ = lo[kk, jj, ii], hi[kk, jj, ii]
        elo_, ehi_ = elo[kk, jj, ii], ehi[kk, jj, ii]
        sign = np.where(fc_, np.where(cl_, 1, -1), np.where(dl_, 1, -1))
        cid = np.where(fc_, np.where(cl_, lo_, hi_), 0)
        eps_d = np.where(fc_, 0.0, np.where(dl_, elo_, ehi_))
        eps_b = np.where(fc_, np.where(cl_, ehi_, elo_), np.where(dl_, ehi_, elo_))
        cols["axis"].append(np.full(kk.shape, a))
        cols["i"].append(ii)
        cols["j"].append(jj)
        cols["k"].append(kk)
        cols["sign"].append(sign)
        cols["cid"].append(cid)
        cols["eps_d"].append(eps_d)
        cols["eps_b"].append(eps_b)
    cat = {k: np.concatenate(v) for k, v in cols.items()}
    slot = np.stack([cat["i"], cat["j"], cat["k"]], axis=1).astype(np.int32)
    return Panels((nx, ny, nz), dv, m, cat["axis"].astype(np.int8), slot,
                  cat["sign"].astype(np.int8), cat["cid"].astype(np.int32),
                  cat["eps_d"].astype(np.float64), cat["eps_b"].astype(np.float64))


# --------------------------------------------------------------------------------------------
# dense assembly (Eq. 4)
# --------------------------------------------------------------------------------------------
def _keys(kind, alpha, beta, d):
    off = np.int64(1 << 15)
    return (((((kind.astype(np.int64) * 3 + alpha) * 3 + beta) << 48)
             | ((d[..., 0] + off) << 32) | ((d[..., 1] + off) << 16) | (d[..., 2] + off)))


def rows_of(p: Panels, rows, cols=None):
    """Dense rows A[rows, cols] of Eq. (4), SI units.

    Conductor row k:  A_kl = P_kl = Δv^3/(4πε0) kappa_P(α_k, β_l, t_k - s_l)   (Eq. 5)
    Dielectric row k: A_kl = s_k Δv^2/(4πε0) kappa_E+(α_k, β_l, t_k - s_l)     (Eq. 6)
                      + δ_kl Ī_k                                               (Eq. 7)
    Each distinct (kind, α, β, offset) is evaluated once (a pure function of those keys).
    """
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.arange(p.n) if cols is None else np.asarray(cols, dtype=np.int64)
    slot = p.slot.astype(np.int64)
    d = slot[rows][:, None, :] - slot[cols][None, :, :]
    kind = np.where(p.is_cond[rows], 0, 1)[:, None]
    alpha = p.axis[rows].astype(np.int64)[:, None]
    beta = p.axis[cols].astype(np.int64)[None, :]
    kind_b = np.broadcast_to(kind, d.shape[:2])
    key = _keys(kind_b, alpha, beta, d)
    uk, inv = np.unique(key.ravel(), return_inverse=True)
    off = np.int64(1 << 15)
    ud = np.stack([((uk >> 32) & 0xFFFF) - off, ((uk >> 16) & 0xFFFF) - off,
                   (uk & 0xFFFF) - off], axis=1)
    ukab = uk >> 48
    ukind, ualpha, ubeta = ukab // 9, (ukab // 3) % 3, ukab % 3
    vals = kappa_batch(ukind, ualpha, ubeta, ud)
    A = vals[inv].reshape(d.shape[:2])
    dv = p.dv
    scale = np.where(p.is_cond[rows], dv ** 3 / FOUR_PI_EPS0,
                     p.sign[rows].astype(np.float64) * dv ** 2 / FOUR_PI_EPS0)
    A *= scale[:, None]
    # Eq. (7): overlap term on the dielectric diagonal
    diag = (rows[:, None] == cols[None, :]) & (~p.is_cond[rows])[:, None]
    A[diag] += np.broadcast_to(p.ibar[rows][:, None], A.shape)[diag]
    return A


def assemble(p: Panels):
    """The dense N x N matrix of Eq. (4)."""
    return rows_of(p, np.arange(p.n))


def matvec(p: Panels, x, A=None):
    """y = ([0; Ī] + [P; E]) x  (Eq. 4)."""
    A = assemble(p) if A is None else A
    return A @ np.asarray(x, dtype=np.float64)


def matvec_rows(p: Panels, x, rows):
    """y[rows] of Eq. (4) without forming the full matrix (row-sampled parity, §8(c))."""
    return rows_of(p, rows) @ np.asarray(x, dtype=np.float64)


def solve(A, b):
    """Direct dense solve (LAPACK gesv)."""
    return np.linalg.solve(A, b)


def rhs(p: Panels):
    """V^j, j = 1..m: V_k = A_k Φ_k with unit potential on conductor j."""
    area = p.dv * p.dv
    B = np.zeros((p.n, p.m))
    for j in range(1, p.m + 1):
        B[p.cid == j, j - 1] = area
    return B


def capacitance_from_rho(p: Panels, rho):
    """C = V^T rho_c with free-charge scaling (Eq. 8; reading O8):
    C_ij = sum_{k in conductor i} A_k fc_k rho^j_k."""
    rho = np.asarray(rho).reshape(p.n, -1)
    area = p.dv * p.dv
    C = np.zeros((p.m, rho.shape[1]))
    for i in range(1, p.m + 1):
        sel = p.cid == i
        C[i - 1] = (area * p.fc[sel])[None, :] @ rho[sel]
    return C


def solve_capacitance(p: Panels, A=None, return_rho=False):
    """Maxwell capacitance matrix (farads): m unit-potential solves + Eq. (8)."""
    A = assemble(p) if A is None else A
    rho = solve(A, rhs(p))
    C = capacitance_from_rho(p, rho)
    return (C, rho) if return_rho else C


# --------------------------------------------------------------------------------------------
# block-diagonal-diagonal preconditioner (Eq. 14)
# --------------------------------------------------------------------------------------------
def precond_boxes(p: Panels, nv=(10, 10, 10)):
    """Box id of every panel: box_a = min(slot_a // N_va, nbox_a - 1) (reading O9:
    faces on the top boundary join the last box)."""
    nbox = [max(1, -(-p.dims[a] // nv[a])) for a in range(3)]
    b = [np.minimum(p.slot[:, a] // nv[a], nbox[a] - 1) for a in range(3)]
    return (b[2] * nbox[1] + b[1]) * nbox[0] + b[0]


def precond_apply(p: Panels, r, nv=(10, 10, 10), A=None, conventional=False):
    """z = R r with R = [R_BD; R_D] (Eq. 14; reading O9).

    R_BD: for every box, the inverse of the dense block of conductor-panel interactions
    inside the box (Eq. 5 entries); R_D = Ī^{-1} on dielectric rows.

    conventional=True: the "conventional block-diagonal preconditioner" the paper compares
    against: every panel of a box, conductor and dielectric, in its block, whose
    entries are the rows of Eq. (4) restricted to the box; no separate diagonal part."""
    A = assemble(p) if A is None else A
    r = np.asarray(r, dtype=np.float64)
    z = np.zeros_like(r)
    box = precond_boxes(p, nv)
    sel = np.ones(p.n, bool) if conventional else p.is_cond
    if not conventional:
        diel = ~p.is_cond
        z[diel] = r[diel] / p.ibar[diel]
    for b in np.unique(box[sel]):
        idx = np.nonzero(sel & (box == b))[0]
        blk = A[np.ix_(idx, idx)]
        z[idx] = np.linalg.inv(blk) @ r[idx]
    return z
