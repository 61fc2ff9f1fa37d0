// ctx.h -- host-side context of libvoxcap (one per device / stream).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/voxcap.h"

namespace vc {

// Owning, grow-only device buffer: alloc() reuses the allocation when it is large enough, so
// repeated extractions of same-sized problems never call cudaMalloc / cudaFree (cudaFree
// synchronises the device) after the first one.  reset() releases the memory.
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0, cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { reset(); }
    void reset() {
        if (p) cudaFree(p);
        p = nullptr;
        n = cap = 0;
    }
    cudaError_t alloc(size_t count) {
        if (p && count <= cap) {
            n = count;
            return cudaSuccess;
        }
        reset();
        if (count == 0) return cudaSuccess;
        cudaError_t e = cudaMalloc(&p, count * sizeof(T));
        if (e == cudaSuccess) n = cap = count;
        else p = nullptr;
        return e;
    }
    T* get() const { return p; }
    size_t bytes() const { return n * sizeof(T); }
};

// Grow-only pinned host array (page-locked, so device -> host copies run at full speed and
// truly asynchronously); the host mirrors of the panel table.
template <class T>
struct PinnedVec {
    T* p = nullptr;
    size_t n = 0, cap = 0;
    PinnedVec() = default;
    PinnedVec(const PinnedVec&) = delete;
    PinnedVec& operator=(const PinnedVec&) = delete;
    ~PinnedVec() {
        if (p) cudaFreeHost(p);
    }
    cudaError_t resize(size_t count) {
        if (count > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            cap = n = 0;
            cudaError_t e = cudaMallocHost(&p, std::max<size_t>(1, count) * sizeof(T));
            if (e != cudaSuccess) {
                p = nullptr;
                return e;
            }
            cap = count;
        }
        n = count;
        return cudaSuccess;
    }
    T* data() { return p; }
    const T* data() const { return p; }
    size_t size() const { return n; }
    T& operator[](size_t i) { return p[i]; }
    const T& operator[](size_t i) const { return p[i]; }
};

struct PanelsDev {
    DevBuf<int8_t> axis, sign, info;  // info bit0: dielectric row, bit1: sign < 0
    DevBuf<int32_t> si, sj, sk, cid;
    DevBuf<double> eps_d, eps_b, ibar, fc;
    DevBuf<int32_t> slotmap[3];  // per orientation: slot -> panel index or -1
};

// Output field of the FFT matvec: C^alpha (kind 0, conductor rows) or D^alpha (kind 1).
struct Field {
    int kind, axis;
    int ext[3];  // slot extent relative to the window origin, per axis
};

struct Precond;  // precond.cu
struct Comm;     // comm.cu

// Tucker-compressed direct-z kernel spectra (Eq. 13; tucker.cu).
// Block b's table X_b[kx][q][u] (this rank's kx, q = |ky|, z offset u) is kept as
//   X_b ~ S_b x1 U1_b x2 U2_b      (U1_b: nkx x r1, U2_b: nq x r2 orthonormal; S_b: r1 x r2 x ZU)
// and P3 reconstructs the K rows of every tile on the fly from two resident tables:
//   U1f [kx tile][block][kc][32]        DMMA A fragments of U1_b (8 kx x 4 ranks per kc)
//   Wf  [q][block][nc][kc][32]          DMMA B fragments of W_b[q] = S_b x2 U2_b[q] (4 ranks x 8 u)
struct Tucker {
    bool on = false;
    int digits = 0;          // relative Frobenius error <= 10^-digits per block
    int nblk = 0, nkx = 0, nq = 0, ZU = 0;
    std::vector<int> r1, r2;  // multilinear ranks (mode kx, mode q); mode u is kept full
    std::vector<double> err;  // measured relative Frobenius error of the reconstructed block
    int nkc[16] = {}, u1o[16] = {}, wo[16] = {};  // per block: rank chunks, fragment offsets
    int nc = 0;               // 8-wide u chunks
    int u1t = 0, wq = 0;      // doubles per U1f kx tile / per Wf q
    int cache = 0;            // 0 no cache file, 1 loaded (NEXT-4 hit), 2 written, 3 write failed
    int kind[16] = {};        // block kind (0 = P, 1 = E): the file holds cores at dv = 1 m, scaled
    double dv = 0;            // by dv^3 (P) / dv^2 (E) when loaded (App. C)
    DevBuf<double> U1f, Wf;
    DevBuf<double> U1, U2, S;   // factors (column-major per block: [b][k][i]) and cores
    DevBuf<double> R, vb, st, part, t1, w, errs;  // build scratch
    int64_t resident() const { return (int64_t)(U1f.n + Wf.n); }
};

constexpr int kMaxRanks = 8;  // one NVLink box

// This rank's panels (canonical order restricted to the rank) and its slot maps
struct PanelsLocal {
    DevBuf<int8_t> info;
    DevBuf<double> ibar, fc;
    DevBuf<int32_t> cid;
    DevBuf<int32_t> slotmap[3];  // slot -> local index or -1 (only own rows are looked up)
    DevBuf<int64_t> gidx;        // local -> global index
};

// Matvec timing (vc_set_timing): every timed matvec records its events from a grow-only pool
// and queues a record; nothing waits on the device inside a matvec.  The records are resolved
// (one event synchronise for the whole batch) when the stats are read or reset, or when the
// queue reaches kMaxRecs.
struct Timing {
    static constexpr int kEvPerMv = 16;   // [0] start, [1..5] pass starts, [6..10] pass ends,
                                          // [11] end, [12..15] all-to-all brackets
    static constexpr int kMaxRecs = 4096;
    bool on = false;      // per-matvec events (ms_matvec)
    bool detail = false;  // per-pass events (ms_pass, ms_comm)
    std::vector<cudaEvent_t> pool;
    struct Rec { int base; int nb; bool det; bool comm; };
    std::vector<Rec> recs;
    int used = 0;
};

}  // namespace vc

struct vc_ctx {
    int device = 0;
    // ---- distribution (vc_init_distributed; world = 1 otherwise) ----
    int rank = 0, world = 1;
    vc::Comm* comm = nullptr;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // several ranks: the exchanges run on their own stream, chunk by chunk, so each source's /
    // field's all-to-all overlaps the transform of the next; events [0..8]
    // "chunk produced" (compute stream), [9..17] "chunk exchanged" (comm stream)
    cudaStream_t cstream = nullptr;
    // host mirror of the panel arrays (h_axis .. h_cid): copied on its own stream after the
    // panel emit, so vc_set_geometry does not wait for it; readers call vc::mirror_wait
    cudaStream_t mstream = nullptr;
    cudaEvent_t mev = nullptr;
    cudaEvent_t cev[18] = {};
    bool cev_ok = false;
    std::string err;

    // ---- geometry (vc_set_geometry) ----
    bool has_geom = false;
    int nx = 0, ny = 0, nz = 0;
    double dv = 0, eps_out = 1;
    int64_t N = 0, Nc = 0, Nd = 0;
    int m = 0;
    vc::PanelsDev pan;
    // [kind][orientation][0 = min, 1 = max][axis]; min > max when no such panels
    int ext[2][3][2][3];
    // host mirror of the panel table (structure-only work: preconditioner boxes)
    vc::PinnedVec<int8_t> h_axis;
    vc::PinnedVec<int32_t> h_si, h_sj, h_sk, h_cid;
    vc::PinnedVec<char> pc_stage;  // pinned staging of the preconditioner uploads

    // ---- operator (vc_build_operator) ----
    bool has_op = false;
    int M[3] = {0, 0, 0}, Kx = 0;
    int lo[3] = {0, 0, 0};
    int ext_in[3][3];  // per source orientation beta: slot extents (0 = no beta panels)
    int nf = 0;
    vc::Field f[6];
    int blk[6][3];  // kernel spectrum index for (field, beta), -1 = none
    int nblk = 0;
    size_t blk_stride = 0;  // doubles per folded spectrum
    vc::DevBuf<double> Rt;  // folded, phase-stripped, scaled kernel spectra
    vc::Tucker tk;          // Tucker-compressed form of Rt (vc_build_opts.tucker_digits)
    vc::DevBuf<double2> tw;  // twiddles exp(-2 pi i n / kTabN)
    std::vector<double> kt_key;  // signature of the kernel tables in Rt / pcTab (reuse_tables)
    bool tables_reused = false;
    vc::DevBuf<double2> bufA, bufB, bufC;  // X1/X4, X2, X3 (nbmax column copies each)
    int nbmax = 1;                          // columns one batched matvec may carry (NEXT-3)
    int lgtk = 2;                           // log2 of P2's kx tile width (one-rank X1 layout)
    int lgt4 = 1;                           // log2 of P4's kx tile width (X3 layout)
    size_t colA = 0, colB = 0, colC = 0;    // per-column strides of bufA / bufB / bufC
    size_t colS = 0;                        // per-column stride of bufS (several ranks)
    size_t offB[3], offC[6];
    int T3 = 1, nt3 = 1;   // P3 tile width and kx-tile count (tile-major X2 / R layouts)
    bool zdirect = false;  // P3 direct-z mode (operator.cu k_p3m)
    int ZU = 0;            // z offsets u per kernel block (direct-z)
    int rs1 = 0;           // direct-z: K rows per kx in a tile (nblk * ZU + one zero row)
    // k_p3m tables: A offsets [KC][MCT][32] (uint16 row | sign << 15, padded to an even count)
    // then output rows [MCT * 8] (int32 f | plane << 4, -1 = padding)
    vc::DevBuf<int32_t> p3m_tab;
    int p3m_nzt = 0, p3m_kc = 0, p3m_mct = 0;  // stacked padded planes, column / row chunks
    int p3m_nst = 2;                           // k_p3m ring depth
    int p3m_nneg = 0, p3m_oddmask = 0;         // negated odd-block rows (count, block bitmask)
    size_t p3m_negoff = 0;                     // their row offsets in p3m_tab (int32)
    int p3m_zoff[3] = {0, 0, 0};               // first stacked position of each source
    std::vector<int32_t> h_planes;     // host copy of the plane lists
    size_t rchunk = 0;     // doubles of R per P3 tile
    int ZL = 0, nzin[3] = {0, 0, 0}, nzout[6] = {0, 0, 0, 0, 0, 0};  // active z-plane counts
    vc::DevBuf<int32_t> planes;  // plane lists + inverse maps (operator.cu)
    double bytes_pass[5] = {0, 0, 0, 0, 0};
    double bytes_k3 = 0;  // the kernel-spectrum share of bytes_pass[2] (read once per P3 launch)
    int precond_kind = 3;
    int box[3] = {10, 10, 10};
    vc::Precond* pc = nullptr;
    // partition (operator_build): window-relative row slabs and kx slabs of every rank
    int ya[vc::kMaxRanks + 1] = {}, kxa[vc::kMaxRanks + 1] = {};
    int nr[vc::kMaxRanks][9] = {};  // rows of rank p for source b (0..2) / field f (3 + f)
    int64_t NL = 0;                 // panels owned by this rank
    int own_Nv = 10, own_nb = 1, own_b0 = 0, own_nbr = 1;  // box-row ownership (row_owner_abs)
    vc::PanelsLocal lp;
    std::vector<int64_t> h_gidx;    // local -> global
    vc::DevBuf<double2> bufS;       // all-to-all send blocks (peers only)
    std::vector<const void*> a2a_send[2];
    std::vector<void*> a2a_recv[2];
    std::vector<size_t> a2a_sb[2], a2a_rb[2];
    size_t offS1[vc::kMaxRanks][3] = {}, offR1[vc::kMaxRanks][3] = {};
    size_t offS2[vc::kMaxRanks][6] = {}, offR2[vc::kMaxRanks][6] = {};

    // ---- reusable scratch (grow-only; see DevBuf) ----
    vc::DevBuf<double2> kG;            // kernel-spectra build grid
    vc::DevBuf<double> kKo;            // kernel octant table
    // near-field P entries for the preconditioner blocks, cut from the octant tables of the
    // kernel build (same generator, no re-evaluation): [pair][iz][iy][ix], |t| <= box
    vc::DevBuf<double> pcTab;
    std::vector<cudaEvent_t> kev;  // kernel-table build: 4 events per block
    int kev_n = 0;
    int pcTabDim[3] = {0, 0, 0};
    int pcPair[3][3] = {{-1, -1, -1}, {-1, -1, -1}, {-1, -1, -1}};
    vc::DevBuf<double> cap_b, cap_rho, cap_part, cap_col;  // capacitance columns
    vc::DevBuf<double> io_in, io_out;  // host-vector calls
    vc::DevBuf<int32_t> in_label;      // host voxel inputs
    vc::DevBuf<double> in_eps;
    vc::DevBuf<unsigned char> geo_flags;    // panel indexing temporaries
    vc::DevBuf<int> geo_pres, geo_ext;
    vc::DevBuf<int64_t> geo_tiles, geo_total;

    // ---- solver work ----
    vc::DevBuf<double> work;  // Krylov basis + temporaries
    size_t work_n = 0;
    vc::DevBuf<double> partial;
    vc::DevBuf<double> dvec;  // small device vector (dots)
    double* h_pinned = nullptr;  // pinned host scratch (dots)
    double* h_pinned_multi = nullptr;  // pinned host scratch of the lockstep solver
    vc::DevBuf<unsigned> ticket;  // last-block ticket of the fused multi-dot
    cudaEvent_t arn_ev[2] = {};   // pipelined Arnoldi: coefficients of step j landed on the host
    bool arn_ev_ok = false;
    cudaEvent_t mc_ev[2] = {};   // lockstep solver: coefficients of the step in parity slot p landed
    bool mc_ev_ok = false;

    // ---- instrumentation ----
    vc_stats stats{};
    vc::Timing timing;
};

namespace vc {
// Host-side phase trace (stderr) when the environment variable VC_TRACE is set.
struct HostTrace {
    bool on;
    const char* tag;
    std::chrono::steady_clock::time_point t0, t;
    explicit HostTrace(const char* tg) : on(getenv("VC_TRACE") != nullptr), tag(tg) {
        t0 = t = std::chrono::steady_clock::now();
    }
    void mark(const char* what) {
        if (!on) return;
        const auto n = std::chrono::steady_clock::now();
        fprintf(stderr, "[vc %s] %-28s %8.3f ms (total %8.3f)\n", tag, what,
                std::chrono::duration<double, std::milli>(n - t).count(),
                std::chrono::duration<double, std::milli>(n - t0).count());
        t = n;
    }
};
// error helpers
inline vc_status set_err(vc_ctx* c, vc_status s, const std::string& msg) {
    c->err = msg;
    return s;
}
#define VC_CUDA(c, expr)                                                                    \
    do {                                                                                    \
        cudaError_t _e = (expr);                                                            \
        if (_e != cudaSuccess)                                                              \
            return vc::set_err((c), _e == cudaErrorMemoryAllocation ? VC_ERR_OOM : VC_ERR_CUDA, \
                               std::string(#expr) + ": " + cudaGetErrorString(_e));        \
    } while (0)

// entry points implemented in the .cu files
vc_status geometry_build(vc_ctx* c, const int32_t* d_label, const double* d_eps);
vc_status operator_build(vc_ctx* c, const vc_build_opts* o);
vc_status matvec_dev(vc_ctx* c, const double* d_x, double* d_y);
// y_c = A x_c for c < nb with one launch per pass (kernel spectra read once per P3 tile for all
// columns); nb <= ctx->nbmax, else (or in z-FFT mode) column by column
vc_status matvec_batch_dev(vc_ctx* c, int nb, const double* const* d_x, double* const* d_y);
// preconditioner host bookkeeping (boxes, signatures, unique blocks, tiles), separable so that
// vc_build_operator can run it on a helper thread beside the kernel-table build
struct PcPlan;
PcPlan* pc_plan_new();
void pc_plan_free(PcPlan* p);
void pc_plan_compute(const vc_ctx* c, const int32_t box_in[3], int64_t N, PcPlan& P, bool all_panels = false);
vc_status precond_build(vc_ctx* c, const int32_t box[3], int kind, const PcPlan* pre = nullptr);
vc_status precond_apply_dev(vc_ctx* c, const double* d_r, double* d_z);
// z_q = R r_q for nc columns (two at once share each R row read)
vc_status precond_apply_multi_dev(vc_ctx* c, int nc, const double* const* d_r, double* const* d_z);
void precond_free(vc_ctx* c);
vc_status solve_dev(vc_ctx* c, const double* d_b, double* d_x, const vc_solve_opts* o,
                    vc_solve_info* info);
vc_status capacitance_dev(vc_ctx* c, double* h_C, const vc_solve_opts* o, vc_solve_info* info);
vc_status debug_kernel_entries(vc_ctx* c, int n, const int32_t* kind, const int32_t* a,
                               const int32_t* b, const int32_t* d, double* out);
vc_status debug_fft(vc_ctx* c, int L, int nl, double* data, int dir);
vc_status partition_build(vc_ctx* c);  // operator.cu: slabs, local panels, local slot maps
void kernel_table_times(vc_ctx* c);
vc_status timing_resolve(vc_ctx* c);  // fold queued matvec timing records into c->stats
int row_owner_abs(const vc_ctx* c, int yabs);
void plan_kx_slabs(int W, int Kx, int T3, int* kxa);
int row_owner_plan(int W, int Nv, int nb, int b0, int nbr, int yabs);
void plan_row_slabs(int W, int ny, int lo, int EY, int Nv, int* ya, int* nb, int* b0, int* nbr);
// tucker.cu
vc_status tucker_compress(vc_ctx* c);
vc_status tucker_from_cache(vc_ctx* c);
bool tucker_try_load(vc_ctx* c, const char* dir, const std::vector<double>& key);
void tucker_save(vc_ctx* c, const char* dir, const std::vector<double>& key);
// comm.cu
vc_status comm_nccl_unique_id(void* out, std::string& err);
void* group_create(int world);
void group_destroy(void* g);
vc_status comm_init(vc_ctx* c, int rank, int world, int transport, const void* id);
void comm_free(vc_ctx* c);
vc_status comm_alltoall(vc_ctx* c, const std::vector<const void*>& send, const std::vector<size_t>& sb,
                        const std::vector<void*>& recv, const std::vector<size_t>& rb,
                        cudaStream_t st = nullptr /* nullptr: the context stream */);
vc_status comm_allreduce(vc_ctx* c, double* d, int n);
vc_status comm_nccl_selftest(vc_ctx* c, double* out);
inline void count_launch(vc_ctx* c, int k = 1) { c->stats.gpu_launches += k; }
}  // namespace vc

namespace vc {
// the host panel mirror is complete (its copies were enqueued by geometry_build); thread-safe
inline void mirror_wait(const vc_ctx* c) {
    if (c->mev) cudaEventSynchronize(c->mev);
}
}  // namespace vc
