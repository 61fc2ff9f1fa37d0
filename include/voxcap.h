/*
 * voxcap.h -- C ABI of libvoxcap.so, the B200-native (sm_100a) hot path of VoxCap
 * (Wang, Qian, White, Yucel, arXiv 2004.02609, "VoxCap: FFT-Accelerated and Tucker-Enhanced
 * Capacitance Extraction Simulator for Voxelized Structures").
 *
 * Citations: P:L = line L of the paper text, with its section/equation.
 *
 * The library solves the Galerkin system of Eq. (4)
 *        [V; 0] = ([0; Ī] + [P; E]) [rho_c; rho_d]
 * for conductor panels (potential rows, Eq. 5) and dielectric-interface panels
 * (normal-field rows, Eq. 6, plus the overlap diagonal Ī of Eq. 7), with the
 * matrix-vector product evaluated by FFTs on the voxel-panel grids (Eqs. 9-12),
 * restarted GMRES with the block-diagonal-diagonal preconditioner (Eq. 14,
 * P:131-139), and extracts the Maxwell capacitance matrix C = V^T rho_c (Eq. 8).
 *
 * Conventions (all calls):
 *   * Units are SI; eps0 = 8.8541878128e-12 F/m.
 *   * Voxel arrays are nz*ny*nx, x fastest.  label: 0 = non-conductor, 1..m = conductor id.
 *   * Panel vectors (x, y, b, rho, r, z) are in canonical panel order: axis-major (x-, y-,
 *     then z-normal panels), then slot (k, j, i) lexicographic with i fastest; conductor and
 *     dielectric panels interleaved (reading O14).  Slot (i,j,k) of an a-normal
 *     panel is its position on the a-grid of P:97: the face between voxel (slot - e_a) and
 *     voxel (slot).
 *   * on_device = 1: pointers are device pointers on the context's device, and work is
 *     ordered on the context's stream (no host synchronisation beyond what the call needs);
 *     on_device = 0: host pointers, the call copies in/out and returns when results are
 *     on the host.
 *   * Ownership: the caller owns every buffer it passes; the library copies what it keeps.
 *     The context owns all device state until vc_destroy.  Calls on one context are not
 *     thread-safe; distinct contexts are independent.
 *   * Errors: every call returns a vc_status; VC_OK = 0.  On error the context keeps its last
 *     valid state (a failed vc_set_geometry leaves no geometry) and vc_last_error() returns a
 *     message.  CUDA errors map to VC_ERR_CUDA (the context should then be destroyed).
 */
#ifndef VOXCAP_H
#define VOXCAP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    VC_OK = 0,
    VC_ERR_INPUT = 1,       /* invalid argument or geometry (dims <= 0, dv <= 0, label < 0,
                               ids not exactly 1..m, m = 0, eps <= 0 / non-finite, two
                               conductors sharing a face, null pointer, grid too large)     */
    VC_ERR_STATE = 2,       /* call out of order (e.g. matvec before build_operator)        */
    VC_ERR_OOM = 3,         /* device allocation failed                                    */
    VC_ERR_CUDA = 4,        /* CUDA runtime / kernel error                                 */
    VC_ERR_NCCL = 5,        /* reserved for the multi-GPU path                             */
    VC_NOT_CONVERGED = 6,   /* GMRES hit maxit; the best iterate is returned                */
    VC_ERR_UNSUPPORTED = 7  /* valid but unsupported request (padded FFT size > 4096 along x
                               or y, > 256 along z)                                          */
} vc_status;

typedef struct vc_ctx vc_ctx;

/* Build options for vc_build_operator.  Zero-initialise and set what you need; zero fields
 * take the defaults noted. */
typedef struct {
    int32_t pad[3];         /* FFT grid size per axis (power of two >= the exactness bound of
                               DESIGN.md reading O11); 0 = smallest valid power of two        */
    int32_t box[3];         /* preconditioner box N_vx, N_vy, N_vz; 0 = 10    */
    int32_t precond;        /* 0 = default = 3; 1 = none; 2 = diagonal only (Ī^{-1} on
                               dielectric rows, 1/P_kk on conductor rows); 3 = the paper's
                               block-diagonal-diagonal (Eq. 14); 4 = the
                               conventional block-diagonal comparator of P:155-157 (every
                               panel of a box in its block, Eq. 4 rows; one rank only)          */
    int32_t zmode;          /* z direction of the matvec: 0 = automatic, 1 = z-FFT
                               (3-D circulant, Eq. 11), 2 = direct z-convolution on the x/y
                               spectra (exact; cheaper when panels occupy few z-planes)       */
    int32_t no_mirror;      /* 0 = default: with a square x/y FFT grid on one rank, blocks that
                               are x<->y mirrors of another (P^{yy} of P^{xx}, ...) are
                               transposed from it instead of generated; 1 =
                               generate every block (bitwise comparisons with multi-rank runs) */
    int32_t no_batch;       /* 0 = default: on one rank with m >= 2 conductors, keep pass buffers
                               for 2 columns so vc_solve_capacitance runs its m solves in
                               lockstep with batched matvecs; 1 = one
                               column at a time (less memory)                                 */
    int32_t reuse_tables;   /* 1: keep the kernel spectra and preconditioner near-field tables
                               from the previous build when their signature (grid, z mode,
                               kernel blocks, tile layout, rank slab, dv, boxes, variants) is
                               unchanged -- they do not depend on panel positions or on the
                               permittivities (kept in HBM instead of an
                               install-time file); 0 = default: always regenerate            */
    int32_t tucker_digits;  /* d > 0: keep the direct-z kernel spectra Tucker-compressed (P:121-129,
                               Eq. 13): per block X ~ S x1 U1 x2 U2 with
                               ||X - X~||_F <= 10^-d ||X||_F, and P3 rebuilds every tile's kernel
                               rows from U1 and W = S x2 U2 on the FP64 tensor cores; the exact
                               table is freed after compression.  Needs the direct-z P3 (zmode 0
                               choosing it, or 2): VC_ERR_UNSUPPORTED otherwise.  0 = default:
                               exact spectra.  d in 1..15.                                    */
    int32_t tucker_pad_;    /* (alignment; must be 0)                                         */
    const char* tucker_cache; /* with tucker_digits > 0: a directory holding the install-time
                               cache of compressed tables:
                               the build loads voxcap_tk_<signature>.bin when it exists and is
                               valid (no kernel generation, no FFTs, no compression), otherwise
                               builds, compresses and writes it (atomically).  The signature
                               covers grid, window, rank slab, dv, kernel blocks, z offsets and
                               digits.  NULL = no cache.                                      */
    int32_t reserved[2];
} vc_build_opts;

/* Solve options.  Zero fields take the paper's defaults. */
typedef struct {
    double tol;             /* relative residual of the preconditioned system; 0 = 1e-4      */
    int32_t restart;        /* GMRES restart length; 0 = 35                                  */
    int32_t maxit;          /* max total iterations; 0 = 2000                                */
    int32_t x0_is_guess;    /* vc_solve: 1 = x holds the initial guess, 0 = start from 0     */
    int32_t reserved[5];
} vc_solve_opts;

typedef struct {
    int32_t iters;          /* GMRES iterations (matvecs) performed                          */
    int32_t converged;      /* 1 if rre_prec <= tol                                          */
    double rre_prec;        /* ||R(b - A x)|| / ||R b|| at exit (preconditioned)      */
    double rre_true;        /* ||b - A x|| / ||b|| at exit (unpreconditioned, recomputed)     */
} vc_solve_info;

/* Instrumentation (CUDA events on the context stream, accumulated since the last reset). */
typedef struct {
    int64_t n_matvec;       /* matvecs executed                                             */
    double  ms_matvec;      /* total device time of the matvec kernel chain                 */
    int64_t n_pass[5];      /* launches of FFT passes P1..P5                                */
    double  ms_pass[5];     /* device time per pass (only when timing_detail = 1)            */
    double  bytes_pass[5];  /* algorithmic bytes per launch of each pass  */
    double  bytes_matvec;   /* algorithmic bytes of one matvec                               */
    double  ms_setup;       /* device time of the last build_operator                        */
    double  ms_precond_build;
    int64_t gpu_launches;   /* kernels launched by the library since the last reset          */
    double  ms_kgen;        /* last build: kernel-entry generation (octant + fill)           */
    double  ms_kfft;        /* last build: 3-D FFT of the kernels + phase strip / fold        */
    double  ms_geometry;    /* last vc_set_geometry (panel indexing), device time            */
    double  ms_comm;        /* all-to-all time inside matvecs (world > 1, timing_detail = 1)  */
    double  bytes_moved[5]; /* algorithmic bytes of all launches of each pass since the reset:
                               a batched launch of nb columns counts nb x its per-column arrays
                               and the P3 kernel spectra once (vc_matvec_batch)              */
    int64_t precond_doubles;/* last build: doubles of the stored (unique) preconditioner blocks
                               (the memory P:157 compares; 0 for precond 1 / 2)              */
    int64_t spectra_doubles;/* last build: doubles of the resident kernel tables P3 reads (exact
                               table, or the Tucker U1 / W fragment tables)                   */
    int64_t tucker_cache;   /* last build: 0 no cache, 1 loaded from the cache file, 2 written,
                               3 could not be written                                        */
    double  tucker_err;     /* last build: max over blocks of the measured relative Frobenius
                               error of the Tucker-compressed spectra (0 when exact)          */
} vc_stats;

/* Create a context on CUDA device `cuda_device`.  `cuda_stream` is a cudaStream_t to order
 * work on, or NULL for a stream owned by the context.  *out receives the context. */
vc_status vc_create(vc_ctx** out, int cuda_device, void* cuda_stream);

/* ---- Multi-GPU (one context per rank and GPU) -------------------------------
 * The padded FFT grid is split in slabs: rank r owns a contiguous range of preconditioner box
 * rows along y for the spatial passes (scatter + x-FFT, x-IFFT + gather, preconditioner, Krylov
 * vectors) and a contiguous range of kx tiles for the spectral passes (y- and z-FFTs, kernel
 * MAC, kernel spectra).  Each matvec does two all-to-all transposes; GMRES dot products and the
 * capacitance columns are summed over ranks.
 *
 * vc_init_distributed: join a group of `world` (1..8) ranks as rank `rank`; call after
 *   vc_create and before vc_set_geometry.  transport 0 = NCCL (one process per GPU): comm_id
 *   points to the 128-byte ncclUniqueId that rank 0 drew with vc_nccl_unique_id and the caller
 *   broadcast (libnccl.so.2 is loaded at this call; VC_ERR_NCCL if it cannot be).  transport 1 =
 *   in-process thread group: comm_id is the handle from vc_group_create(world); each of the
 *   `world` contexts must then be driven by its own host thread, making the same calls in the
 *   same order (collective calls: vc_set_geometry, vc_build_operator, vc_matvec, vc_solve,
 *   vc_solve_capacitance).  Every rank passes the whole voxel structure to vc_set_geometry.
 * With world > 1, the vectors of vc_matvec / vc_precond / vc_solve are this rank's LOCAL panels
 * (canonical order restricted to the rank; see vc_get_local_panels); vc_get_sizes and
 * vc_get_panels stay global, and vc_solve_capacitance returns the full matrix on every rank. */
vc_status vc_init_distributed(vc_ctx* ctx, int32_t rank, int32_t world, int32_t transport,
                              const void* comm_id);
/* Draw an NCCL unique id (128 bytes) into out; VC_ERR_NCCL if libnccl cannot be loaded. */
vc_status vc_nccl_unique_id(void* out);
/* In-process thread group of `world` ranks (transport 1); destroy after all its contexts. */
vc_status vc_group_create(int32_t world, void** group);
void vc_group_destroy(void* group);
/* Host-only (no device needed): the slab boundaries vc_build_operator uses for `world` ranks.
 * Rows: the slot rows [lo_y, lo_y + ey) of the FFT window (ny voxel rows, preconditioner box
 * height box_y) -> ya[0..world] window-relative row boundaries (rank r owns [ya[r], ya[r+1]),
 * whole box rows each).  Columns: kx in [0, kx) in tiles of `tile` -> kxa[0..world].  Both
 * arrays are caller-allocated with world + 1 entries. */
vc_status vc_plan_slabs(int32_t world, int32_t ny, int32_t lo_y, int32_t ey, int32_t box_y,
                        int32_t kx, int32_t tile, int32_t* ya, int32_t* kxa);
/* After vc_build_operator: number of panels this rank owns and (if global_index != NULL) their
 * global canonical indices, ascending.  world = 1: all panels. */
vc_status vc_get_local_panels(const vc_ctx* ctx, int64_t* n_local, int64_t* global_index);

/* Voxel structure (§II.A; §II.B grids).  Copies label[nz*ny*nx] (int32) and eps_r
 * [nz*ny*nx] (float64, relative permittivity of non-conductor voxels; NULL = all 1.0; values
 * on conductor voxels are ignored).  eps_r_outside is the medium outside the box.  dv_m is the
 * voxel edge in metres.  Runs the panel-indexing kernels (DESIGN.md a1): conductor panels are
 * faces with exactly one conductor side; dielectric panels are non-conductor faces whose two
 * permittivities differ (normal and (eps_d, eps_b) per reading O7).  Errors: VC_ERR_INPUT as
 * listed in vc_status. */
vc_status vc_set_geometry(vc_ctx* ctx, int32_t nx, int32_t ny, int32_t nz, double dv_m,
                          const int32_t* label, const double* eps_r, double eps_r_outside,
                          int32_t on_device);

/* Panel counts after vc_set_geometry: N, N_c, N_d and the number of conductors m.  Any
 * output pointer may be NULL. */
vc_status vc_get_sizes(const vc_ctx* ctx, int64_t* n_panels, int64_t* n_cond, int64_t* n_diel,
                       int32_t* m_conductors);

/* Copy the panel table (canonical order) to caller-allocated host arrays of length N (slot:
 * 3N, (i,j,k) per panel).  axis 0/1/2 = x/y/z normal; sign +1 = normal along +axis; cid
 * 1..m conductor, 0 dielectric; eps_d/eps_b per reading O7 (conductor panels: eps_d = 0,
 * eps_b = eps_r of the medium its normal points into, the free-charge factor of Eq. 8).  Any
 * pointer may be NULL. */
vc_status vc_get_panels(const vc_ctx* ctx, int8_t* axis, int32_t* slot, int8_t* sign,
                        int32_t* cid, double* eps_d, double* eps_b);

/* Plan the FFT grid, generate the kernel entries (Eqs. 5-6 closed forms near, Gauss-Legendre
 * far, scaled by dv^3 / dv^2 (App. C)), transform them into phase-stripped, parity-
 * folded real spectra (Eqs. 11-12), and build the preconditioner (Eq. 14).  opts may be NULL. */
vc_status vc_build_operator(vc_ctx* ctx, const vc_build_opts* opts);

/* FFT grid chosen by vc_build_operator (M_x, M_y, M_z). */
vc_status vc_get_grid(const vc_ctx* ctx, int32_t* m3);

/* y = ([0; Ī] + [P; E]) x   (Eq. 4; Eqs. 9-11).  x, y: N doubles (world > 1:
 * this rank's n_local entries). */
vc_status vc_matvec(vc_ctx* ctx, const double* x, double* y, int32_t on_device);

/* Y = A X for nb columns (the matvec of vc_matvec per column): X, Y are
 * column-major n x nb (column c at x + c * n, n = N or this rank's n_local), host or device.
 * Columns are processed up to two per launch chain when the build kept batch buffers
 * (vc_build_opts.no_batch = 0, one rank, m >= 2): every pass runs once for the pair and P3
 * reads each kernel-spectrum tile once for both; each column's result is bitwise equal to
 * vc_matvec on it.  nb = 0 is a no-op; nb < 0 or NULL vectors: VC_ERR_INPUT. */
vc_status vc_matvec_batch(vc_ctx* ctx, int32_t nb, const double* x, double* y, int32_t on_device);

/* z = R r with R the preconditioner chosen at build time (Eq. 14). */
vc_status vc_precond(vc_ctx* ctx, const double* r, double* z, int32_t on_device);

/* Solve A x = b by left-preconditioned restarted GMRES (Eq. 14).  info may be NULL.
 * Returns VC_NOT_CONVERGED (with the best iterate in x) if maxit is reached. */
vc_status vc_solve(vc_ctx* ctx, const double* b, double* x, const vc_solve_opts* opts,
                   vc_solve_info* info, int32_t on_device);

/* Maxwell capacitance matrix (Eq. 8): for each conductor j a unit-potential solve
 * with V_k = A_k on conductor j's panels, then C_ij = sum_{k in i} A_k * fc_k * rho^j_k with
 * fc_k the relative permittivity next to panel k (free-charge scaling).  C: m*m host
 * doubles, row-major, farads.  per_column: m entries or NULL.  Returns VC_NOT_CONVERGED if
 * any column did not converge (C is still filled). */
vc_status vc_solve_capacitance(vc_ctx* ctx, double* C, const vc_solve_opts* opts,
                               vc_solve_info* per_column);

/* Instrumentation: timing_detail = 1 records CUDA events around every matvec and every pass
 * (ms_matvec, ms_pass, ms_comm); 0 records none.  Nothing waits on the device inside a
 * matvec: the events are queued and resolved when vc_get_stats or vc_reset_stats is called
 * (those two calls wait for the last timed matvec).  vc_get_stats copies the counters;
 * vc_reset_stats zeroes them. */
vc_status vc_set_timing(vc_ctx* ctx, int32_t timing_detail);
vc_status vc_get_stats(const vc_ctx* ctx, vc_stats* out);
vc_status vc_reset_stats(vc_ctx* ctx);

/* Test hooks (documented, stable): evaluate the device kernel-entry generator for n offsets
 * (kind 0 = P, 1 = E+; alpha = observer normal, beta = source normal; d = observer slot -
 * source slot, 3n int32) in unit-voxel units (dv = 1, 4*pi*eps0 = 1), results to host out[n];
 * and run the device batched FFT on host data (n_lines lines of length L, interleaved
 * re/im doubles, in place; dir -1 forward, +1 inverse unnormalised). */
vc_status vc_debug_kernel_entries(vc_ctx* ctx, int32_t n, const int32_t* kind,
                                  const int32_t* alpha, const int32_t* beta, const int32_t* d,
                                  double* out);
vc_status vc_debug_fft(vc_ctx* ctx, int32_t L, int32_t n_lines, double* data, int32_t dir);
/* Test hook (documented, stable): the folded, phase-stripped kernel spectra of the built operator
 * (Eqs. 11-12 after App. B folding; DESIGN.md §6 "R").  layout[8] receives {zdirect, nblk, NW,
 * T3, nt3, KY, RS1, nkx}: the table is [KY][nt3][...] tiles of rchunk doubles; direct-z tiles are
 * [T3][RS1] with row = block * NW + u (NW = ZU z offsets, last row zero), z-FFT tiles are
 * [block][NW = Mz/2 + 1][T3].  *n receives the table length in doubles.  vc_debug_get_spectra
 * copies it to host `out` (NULL: sizes only); vc_debug_set_spectra overwrites it from host `in`
 * (n doubles; VC_ERR_INPUT on a length mismatch) -- used to measure what a compressed (e.g.
 * Tucker) spectrum does to the matvec.  VC_ERR_STATE before vc_build_operator. */
vc_status vc_debug_get_spectra(vc_ctx* ctx, int64_t* n, int32_t* layout, double* out);
/* Test hook: NCCL transport self-test on a context initialised with transport 0 -- an
 * ncclAllReduce of {1,2,3,4} and a grouped ncclSend / ncclRecv of four doubles with this rank as
 * its own peer (works on a world-1 communicator, i.e. on one GPU).  out[8] host doubles:
 * out[0..3] = world x {1,2,3,4}, out[4..7] = the received {world x 1..4}.  VC_ERR_STATE without
 * an NCCL communicator, VC_ERR_NCCL on a failing call. */
vc_status vc_debug_nccl_selftest(vc_ctx* ctx, double* out);
vc_status vc_debug_set_spectra(vc_ctx* ctx, int64_t n, const double* in);
/* Tucker-compressed spectra of the last build (vc_build_opts.tucker_digits > 0): *nblk blocks;
 * ranks[2 * nblk] = (r1, r2) per block (kx mode, |ky| mode; the z-offset mode is kept full);
 * err[nblk] = measured relative Frobenius error per block (as stored in the cache file when it
 * was loaded); dims[3] = (nkx, nq, ZU).  Any output pointer may be NULL; arrays hold at least 16
 * blocks.  VC_ERR_STATE if the build kept exact spectra. */
vc_status vc_get_tucker(const vc_ctx* ctx, int32_t* nblk, int32_t* ranks, double* err, int32_t* dims);

/* Last error message of the context ("" if none).  Valid until the next call on ctx. */
const char* vc_last_error(const vc_ctx* ctx);

/* Library version string. */
const char* vc_version(void);

void vc_destroy(vc_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* VOXCAP_H */
