"""voxcap-b200: ctypes binding of libvoxcap.so (include/voxcap.h).

Argument marshalling only -- every step of the hot path (panel indexing, kernel generation,
FFT matvec, preconditioner, GMRES, capacitance) runs in the library's CUDA kernels.  There is no
CPU fallback: importing works without a GPU, but creating a :class:`VoxCap` context requires the
built library and a CUDA device, and raises otherwise.

Host arrays are numpy; device vectors may be passed as CUDA torch tensors (float64,
contiguous), in which case work is ordered on the current torch stream of that device.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = ["VoxCap", "VoxCapError", "lib_path", "load_library", "EXPORTS", "BuildOpts",
           "SolveOpts", "SolveInfo", "Stats", "ThreadGroup", "nccl_unique_id", "plan_slabs"]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_NAME = "libvoxcap.so"

# every symbol include/voxcap.h declares
EXPORTS = ("vc_create", "vc_set_geometry", "vc_get_sizes", "vc_get_panels", "vc_build_operator",
           "vc_get_grid", "vc_matvec", "vc_matvec_batch", "vc_precond", "vc_solve", "vc_solve_capacitance",
           "vc_set_timing", "vc_get_stats", "vc_reset_stats", "vc_debug_kernel_entries",
           "vc_debug_fft", "vc_last_error", "vc_version", "vc_destroy", "vc_init_distributed",
           "vc_nccl_unique_id", "vc_group_create", "vc_group_destroy", "vc_get_local_panels",
           "vc_plan_slabs", "vc_debug_get_spectra", "vc_debug_set_spectra",
           "vc_debug_nccl_selftest", "vc_get_tucker")

STATUS = {0: "VC_OK", 1: "VC_ERR_INPUT", 2: "VC_ERR_STATE", 3: "VC_ERR_OOM", 4: "VC_ERR_CUDA",
          5: "VC_ERR_NCCL", 6: "VC_NOT_CONVERGED", 7: "VC_ERR_UNSUPPORTED"}


class VoxCapError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        self.code = STATUS.get(status, str(status))
        super().__init__(f"{self.code}: {msg}")


class BuildOpts(ctypes.Structure):
    _fields_ = [("pad", ctypes.c_int32 * 3), ("box", ctypes.c_int32 * 3),
                ("precond", ctypes.c_int32), ("zmode", ctypes.c_int32),
                ("no_mirror", ctypes.c_int32), ("no_batch", ctypes.c_int32),
                ("reuse_tables", ctypes.c_int32), ("tucker_digits", ctypes.c_int32),
                ("tucker_pad_", ctypes.c_int32), ("tucker_cache", ctypes.c_char_p),
                ("reserved", ctypes.c_int32 * 2)]


class SolveOpts(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("restart", ctypes.c_int32), ("maxit", ctypes.c_int32),
                ("x0_is_guess", ctypes.c_int32), ("reserved", ctypes.c_int32 * 5)]


class SolveInfo(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("rre_prec", ctypes.c_double), ("rre_true", ctypes.c_double)]

    def as_dict(self):
        return {"iters": self.iters, "converged": bool(self.converged),
                "rre_prec": self.rre_prec, "rre_true": self.rre_true}


class Stats(ctypes.Structure):
    _fields_ = [("n_matvec", ctypes.c_int64), ("ms_matvec", ctypes.c_double),
                ("n_pass", ctypes.c_int64 * 5), ("ms_pass", ctypes.c_double * 5),
                ("bytes_pass", ctypes.c_double * 5), ("bytes_matvec", ctypes.c_double),
                ("ms_setup", ctypes.c_double), ("ms_precond_build", ctypes.c_double),
                ("gpu_launches", ctypes.c_int64), ("ms_kgen", ctypes.c_double),
                ("ms_kfft", ctypes.c_double), ("ms_geometry", ctypes.c_double),
                ("ms_comm", ctypes.c_double), ("bytes_moved", ctypes.c_double * 5),
                ("precond_doubles", ctypes.c_int64), ("spectra_doubles", ctypes.c_int64),
                ("tucker_cache", ctypes.c_int64), ("tucker_err", ctypes.c_double)]

    def as_dict(self):
        return {"n_matvec": self.n_matvec, "ms_matvec": self.ms_matvec,
                "n_pass": list(self.n_pass), "ms_pass": list(self.ms_pass),
                "bytes_pass": list(self.bytes_pass), "bytes_matvec": self.bytes_matvec,
                "bytes_moved": list(self.bytes_moved),
                "ms_setup": self.ms_setup, "ms_precond_build": self.ms_precond_build,
                "gpu_launches": self.gpu_launches, "ms_kgen": self.ms_kgen,
                "ms_kfft": self.ms_kfft, "ms_geometry": self.ms_geometry,
                "ms_comm": self.ms_comm, "precond_doubles": self.precond_doubles,
                "spectra_doubles": self.spectra_doubles, "tucker_cache": self.tucker_cache,
                "tucker_err": self.tucker_err}


def lib_path():
    # VOXCAP_LIB: an alternative in-tree build of the same library (A/B timing of build
    # variants; tools/ only)
    return os.environ.get("VOXCAP_LIB") or os.path.join(_HERE, _LIB_NAME)


_lib = None


def load_library(build_if_missing=False):
    """Load libvoxcap.so (raises if absent; never falls back to anything else)."""
    global _lib
    if _lib is not None:
        return _lib
    p = lib_path()
    if not os.path.exists(p):
        if build_if_missing:
            from .build import build
            build()
        else:
            raise VoxCapError(4, f"{p} not built: run `python -m paper_2004_02609_b200.build`")
    lib = ctypes.CDLL(p)
    vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    P = ctypes.POINTER
    sig = {
        "vc_create": [P(vp), ctypes.c_int, vp],
        "vc_set_geometry": [vp, i32, i32, i32, dbl, vp, vp, dbl, i32],
        "vc_get_sizes": [vp, P(i64), P(i64), P(i64), P(i32)],
        "vc_get_panels": [vp, vp, vp, vp, vp, vp, vp],
        "vc_build_operator": [vp, P(BuildOpts)],
        "vc_get_grid": [vp, vp],
        "vc_matvec": [vp, vp, vp, i32],
        "vc_precond": [vp, vp, vp, i32],
        "vc_solve": [vp, vp, vp, P(SolveOpts), P(SolveInfo), i32],
        "vc_solve_capacitance": [vp, vp, P(SolveOpts), vp],
        "vc_set_timing": [vp, i32],
        "vc_matvec_batch": [vp, i32, vp, vp, i32],
        "vc_get_stats": [vp, P(Stats)],
        "vc_reset_stats": [vp],
        "vc_debug_kernel_entries": [vp, i32, vp, vp, vp, vp, vp],
        "vc_debug_fft": [vp, i32, i32, vp, i32],
        "vc_debug_get_spectra": [vp, P(i64), vp, vp],
        "vc_debug_set_spectra": [vp, i64, vp],
        "vc_debug_nccl_selftest": [vp, vp],
        "vc_get_tucker": [vp, vp, vp, vp, vp],
        "vc_init_distributed": [vp, i32, i32, i32, vp],
        "vc_nccl_unique_id": [vp],
        "vc_group_create": [i32, P(vp)],
        "vc_get_local_panels": [vp, P(i64), vp],
        "vc_plan_slabs": [i32, i32, i32, i32, i32, i32, i32, vp, vp],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    lib.vc_last_error.argtypes = [vp]
    lib.vc_last_error.restype = ctypes.c_char_p
    lib.vc_version.argtypes = []
    lib.vc_version.restype = ctypes.c_char_p
    lib.vc_destroy.argtypes = [vp]
    lib.vc_destroy.restype = None
    lib.vc_group_destroy.argtypes = [vp]
    lib.vc_group_destroy.restype = None
    _lib = lib
    return lib


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if isinstance(a, np.ndarray) else ctypes.c_void_p(a.data_ptr())


def _is_cuda_tensor(a):
    return hasattr(a, "is_cuda") and a.is_cuda


def nccl_unique_id():
    """128-byte NCCL unique id (rank 0 draws it; the caller broadcasts it)."""
    buf = (ctypes.c_uint8 * 128)()
    st = load_library().vc_nccl_unique_id(buf)
    if st != 0:
        raise VoxCapError(st, "vc_nccl_unique_id failed (libnccl.so.2 not loadable?)")
    return bytes(buf)


def plan_slabs(world, ny, lo_y, ey, box_y, kx, tile):
    """Slab boundaries (host only): (ya, kxa), each world + 1 int32 (see include/voxcap.h)."""
    ya = np.zeros(world + 1, np.int32)
    kxa = np.zeros(world + 1, np.int32)
    st = load_library().vc_plan_slabs(world, ny, lo_y, ey, box_y, kx, tile, _ptr(ya), _ptr(kxa))
    if st != 0:
        raise VoxCapError(st, "vc_plan_slabs: invalid arguments")
    return ya, kxa


class ThreadGroup:
    """In-process group of `world` ranks (transport 1): each member context must be driven by its
    own Python thread (ctypes releases the GIL during library calls)."""

    def __init__(self, world):
        self._lib = load_library()
        self.world = int(world)
        self.handle = ctypes.c_void_p()
        st = self._lib.vc_group_create(self.world, ctypes.byref(self.handle))
        if st != 0:
            raise VoxCapError(st, "vc_group_create failed")

    def close(self):
        if self.handle.value:
            self._lib.vc_group_destroy(self.handle)
            self.handle = ctypes.c_void_p()


class VoxCap:
    """One context = one device (+ stream).  Methods mirror the C ABI one to one."""

    def __init__(self, device=0, stream=None):
        self._lib = load_library()
        self._ctx = ctypes.c_void_p()
        self._tstream = None
        if stream is None:
            try:
                import torch
                if torch.cuda.is_available():
                    # the context's own stream, known to torch so device-tensor calls can be
                    # fenced against torch's current stream (see _fence_in / _fence_out)
                    self._tstream = torch.cuda.Stream(device)
                    stream = self._tstream.cuda_stream
            except ImportError:
                stream = None
        st = self._lib.vc_create(ctypes.byref(self._ctx), int(device),
                                 ctypes.c_void_p(stream) if stream else None)
        if st != 0:
            raise VoxCapError(st, "vc_create failed (no CUDA device?)")
        self.device = device
        self.n = 0
        self.m = 0

    # -- plumbing ------------------------------------------------------------------------
    def _check(self, st, allow=(0,)):
        if st not in allow:
            raise VoxCapError(st, self._lib.vc_last_error(self._ctx).decode())
        return st

    def close(self):
        if getattr(self, "_ctx", None) and self._ctx.value:
            self._lib.vc_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @staticmethod
    def version():
        return load_library().vc_version().decode()

    # -- distribution --------------------------------------------------------------------
    def init_distributed(self, rank, world, nccl_id=None, group=None):
        """Join a group of `world` ranks: NCCL (nccl_id = 128 bytes from nccl_unique_id(), one
        process per GPU) or an in-process ThreadGroup."""
        if group is not None:
            st = self._lib.vc_init_distributed(self._ctx, int(rank), int(world), 1, group.handle)
        else:
            buf = (ctypes.c_uint8 * 128).from_buffer_copy(bytes(nccl_id))
            st = self._lib.vc_init_distributed(self._ctx, int(rank), int(world), 0, buf)
        self._check(st)
        self.rank, self.world = int(rank), int(world)
        return self

    def local_panels(self):
        """Global canonical indices of this rank's panels (the layout of local vectors)."""
        n = ctypes.c_int64()
        self._check(self._lib.vc_get_local_panels(self._ctx, ctypes.byref(n), None))
        out = np.empty(n.value, np.int64)
        self._check(self._lib.vc_get_local_panels(self._ctx, ctypes.byref(n), _ptr(out)))
        return out

    # -- geometry ------------------------------------------------------------------------
    def set_geometry(self, label, eps=None, eps_out=1.0, dv=1e-6):
        """label (Nz, Ny, Nx) int32 (numpy, or CUDA torch tensor), eps same shape float64."""
        on_dev = _is_cuda_tensor(label)
        if on_dev:
            lab = label.contiguous()
            ep = None if eps is None else eps.contiguous()
            assert str(lab.dtype) == "torch.int32"
            self._fence_in(*[t for t in (lab, ep) if t is not None])
        else:
            lab = np.ascontiguousarray(label, dtype=np.int32)
            ep = None if eps is None else np.ascontiguousarray(eps, dtype=np.float64)
        nz, ny, nx = lab.shape
        self._keep = (lab, ep)
        self._check(self._lib.vc_set_geometry(self._ctx, nx, ny, nz, float(dv), _ptr(lab),
                                              None if ep is None else _ptr(ep), float(eps_out),
                                              1 if on_dev else 0))
        n, nc, nd, m = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
        self._check(self._lib.vc_get_sizes(self._ctx, ctypes.byref(n), ctypes.byref(nc),
                                           ctypes.byref(nd), ctypes.byref(m)))
        self.n, self.n_cond, self.n_diel, self.m = n.value, nc.value, nd.value, m.value
        return self

    def set_structure(self, st):
        """Convenience: a voxgen.Structure-like object (label, eps, eps_out, dv)."""
        return self.set_geometry(st.label, st.eps, st.eps_out, st.dv)

    def panels(self):
        n = self.n
        out = {"axis": np.empty(n, np.int8), "slot": np.empty((n, 3), np.int32),
               "sign": np.empty(n, np.int8), "cid": np.empty(n, np.int32),
               "eps_d": np.empty(n, np.float64), "eps_b": np.empty(n, np.float64)}
        self._check(self._lib.vc_get_panels(self._ctx, *[_ptr(out[k]) for k in
                                                         ("axis", "slot", "sign", "cid",
                                                          "eps_d", "eps_b")]))
        return out

    # -- operator ------------------------------------------------------------------------
    def build_operator(self, pad=None, box=None, precond=3, zmode=0, mirror=True, batch=True,
                       reuse_tables=False, tucker_digits=0, tucker_cache=None):
        """zmode: 0 automatic, 1 z-FFT (3-D circulant), 2 direct z-convolution; mirror=False
        generates every kernel block (no x<->y transposes); tucker_digits=d > 0 keeps the
        direct-z spectra Tucker-compressed to relative error 10^-d, with the
        compressed tables cached in directory `tucker_cache`."""
        o = BuildOpts()
        o.tucker_digits = int(tucker_digits)
        self._tk_cache = None if tucker_cache is None else os.fsencode(tucker_cache)
        o.tucker_cache = self._tk_cache
        o.zmode = int(zmode)
        o.no_mirror = 0 if mirror else 1
        o.no_batch = 0 if batch else 1
        o.reuse_tables = 1 if reuse_tables else 0
        if pad is not None:
            for a in range(3):
                o.pad[a] = int(pad[a])
        if box is not None:
            for a in range(3):
                o.box[a] = int(box[a])
        o.precond = int(precond)
        self._check(self._lib.vc_build_operator(self._ctx, ctypes.byref(o)))
        return self

    def grid(self):
        m3 = (ctypes.c_int32 * 3)()
        self._check(self._lib.vc_get_grid(self._ctx, m3))
        return tuple(m3)

    def _fence_in(self, *tensors):
        """Order the context stream after torch's current stream (inputs are ready)."""
        if self._tstream is not None:
            import torch
            self._tstream.wait_stream(torch.cuda.current_stream(self.device))
            for t in tensors:
                t.record_stream(self._tstream)

    def _fence_out(self):
        """Order torch's current stream after the context stream (outputs are ready)."""
        if self._tstream is not None:
            import torch
            torch.cuda.current_stream(self.device).wait_stream(self._tstream)

    def _vec_call(self, fn, x, out=None):
        if _is_cuda_tensor(x):
            import torch
            x = x.contiguous()
            y = torch.empty_like(x) if out is None else out
            self._fence_in(x, y)
            self._check(fn(self._ctx, _ptr(x), _ptr(y), 1))
            self._fence_out()
            return y
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x) if out is None else out
        self._check(fn(self._ctx, _ptr(x), _ptr(y), 0))
        return y

    def matvec(self, x, out=None):
        """y = ([0; Ī] + [P; E]) x (Eq. 4)."""
        return self._vec_call(self._lib.vc_matvec, x, out)

    def matvec_batch(self, X):
        """Y[:, c] = A X[:, c] for the columns of an (n, nb) array (NEXT-3 batched matvec)."""
        if _is_cuda_tensor(X):
            import torch
            Xc = X.t().contiguous()  # column c contiguous
            Y = torch.empty_like(Xc)
            self._fence_in(Xc, Y)
            self._check(self._lib.vc_matvec_batch(self._ctx, int(Xc.shape[0]), _ptr(Xc), _ptr(Y), 1))
            self._fence_out()
            return Y.t()
        Xc = np.ascontiguousarray(np.asarray(X, dtype=np.float64).T)
        Y = np.empty_like(Xc)
        self._check(self._lib.vc_matvec_batch(self._ctx, int(Xc.shape[0]), _ptr(Xc), _ptr(Y), 0))
        return Y.T

    def precond(self, r, out=None):
        return self._vec_call(self._lib.vc_precond, r, out)

    @staticmethod
    def _sopts(tol, restart, maxit, guess=False):
        o = SolveOpts()
        o.tol = float(tol or 0)
        o.restart = int(restart or 0)
        o.maxit = int(maxit or 0)
        o.x0_is_guess = 1 if guess else 0
        return o

    def solve(self, b, tol=1e-4, restart=35, maxit=2000, x0=None):
        o = self._sopts(tol, restart, maxit, x0 is not None)
        info = SolveInfo()
        on_dev = _is_cuda_tensor(b)
        if on_dev:
            import torch
            b = b.contiguous()
            x = torch.zeros_like(b) if x0 is None else x0.clone()
            self._fence_in(b, x)
            st = self._lib.vc_solve(self._ctx, _ptr(b), _ptr(x), ctypes.byref(o),
                                    ctypes.byref(info), 1)
            self._fence_out()
        else:
            b = np.ascontiguousarray(b, dtype=np.float64)
            x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64)
            st = self._lib.vc_solve(self._ctx, _ptr(b), _ptr(x), ctypes.byref(o),
                                    ctypes.byref(info), 0)
        self._check(st, allow=(0, 6))
        return x, info.as_dict()

    def solve_capacitance(self, tol=1e-4, restart=35, maxit=2000):
        """Maxwell capacitance matrix (m x m, farads) and per-column solve info."""
        o = self._sopts(tol, restart, maxit)
        C = np.zeros((self.m, self.m), np.float64)
        infos = (SolveInfo * max(1, self.m))()
        st = self._lib.vc_solve_capacitance(self._ctx, _ptr(C), ctypes.byref(o), infos)
        self._check(st, allow=(0, 6))
        return C, [infos[i].as_dict() for i in range(self.m)]

    # -- instrumentation / test hooks -----------------------------------------------------
    def set_timing(self, detail=True):
        self._check(self._lib.vc_set_timing(self._ctx, 1 if detail else 0))

    def stats(self):
        s = Stats()
        self._check(self._lib.vc_get_stats(self._ctx, ctypes.byref(s)))
        return s.as_dict()

    def reset_stats(self):
        self._check(self._lib.vc_reset_stats(self._ctx))

    def kernel_entries(self, kind, alpha, beta, d):
        """Device kernel-entry generator in unit-voxel units (test hook)."""
        d = np.ascontiguousarray(d, dtype=np.int32).reshape(-1, 3)
        n = d.shape[0]
        kind = np.ascontiguousarray(np.broadcast_to(kind, (n,)), dtype=np.int32)
        alpha = np.ascontiguousarray(np.broadcast_to(alpha, (n,)), dtype=np.int32)
        beta = np.ascontiguousarray(np.broadcast_to(beta, (n,)), dtype=np.int32)
        out = np.empty(n, np.float64)
        self._check(self._lib.vc_debug_kernel_entries(self._ctx, n, _ptr(kind), _ptr(alpha),
                                                      _ptr(beta), _ptr(d), _ptr(out)))
        return out

    def spectra(self):
        """Folded kernel-spectrum table (test hook): (raw float64 array, layout dict)."""
        n = ctypes.c_int64()
        lay = np.zeros(8, np.int32)
        self._check(self._lib.vc_debug_get_spectra(self._ctx, ctypes.byref(n), _ptr(lay), None))
        out = np.empty(n.value, np.float64)
        self._check(self._lib.vc_debug_get_spectra(self._ctx, ctypes.byref(n), _ptr(lay), _ptr(out)))
        keys = ("zdirect", "nblk", "NW", "T3", "nt3", "KY", "RS1", "nkx")
        return out, dict(zip(keys, (int(v) for v in lay)))

    def tucker(self):
        """Tucker-compressed spectra of the last build: ranks (r1, r2) and measured relative
        error per block, dims (nkx, nq, ZU); None when the build kept exact spectra."""
        nb = ctypes.c_int32()
        ranks = np.zeros(32, np.int32)
        err = np.zeros(16)
        dims = np.zeros(3, np.int32)
        st = self._lib.vc_get_tucker(self._ctx, ctypes.byref(nb), _ptr(ranks), _ptr(err), _ptr(dims))
        if st == 2:
            return None
        self._check(st)
        n = nb.value
        return {"nblk": n, "ranks": ranks[: 2 * n].reshape(n, 2).tolist(), "err": err[:n].tolist(),
                "dims": dims.tolist()}

    def nccl_selftest(self):
        """NCCL transport self-test (test hook): allreduce + grouped send/recv to self."""
        out = np.zeros(8)
        self._check(self._lib.vc_debug_nccl_selftest(self._ctx, _ptr(out)))
        return out

    def spectra_layout(self):
        """Layout of the kernel-spectrum table (no copy): zdirect, nblk, NW, T3, nt3, KY, RS1, nkx."""
        n = ctypes.c_int64()
        lay = np.zeros(8, np.int32)
        self._check(self._lib.vc_debug_get_spectra(self._ctx, ctypes.byref(n), _ptr(lay), None))
        keys = ("zdirect", "nblk", "NW", "T3", "nt3", "KY", "RS1", "nkx")
        return dict(zip(keys, (int(v) for v in lay)))

    def set_spectra(self, table):
        """Overwrite the kernel-spectrum table (test hook; same length and layout)."""
        a = np.ascontiguousarray(table, dtype=np.float64)
        self._check(self._lib.vc_debug_set_spectra(self._ctx, a.size, _ptr(a)))

    def fft(self, data, inverse=False):
        """Device batched FFT along the last axis (test hook); complex128 in, complex128 out."""
        a = np.ascontiguousarray(data, dtype=np.complex128).copy()
        L = a.shape[-1]
        nl = a.size // L
        self._check(self._lib.vc_debug_fft(self._ctx, L, nl, _ptr(a), 1 if inverse else -1))
        return a
