// mv.cuh -- the matvec launch descriptor shared by the pass kernels (operator.cu) and the P3
// direct-z DMMA kernel (p3m.cu), plus small launch helpers.
#pragma once

#include <cuda.h>

#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "ctx.h"

namespace vc {

constexpr int kMaxRows = 256;  // P3 direct-z: max stacked output rows
constexpr int kMaxB = 2;    // columns per batched matvec (NEXT-3; one rank, direct-z mode)

struct MV {
    int Mx, My, Mz, Kx;
    int lo[3];
    int G[3][3];       // slot-grid dims [orientation][axis]
    int ext_in[3][3];  // [beta][axis]
    int nf;
    int fkind[6], faxis[6];
    int ext_out[6][3];
    const int32_t* slotmap[3];
    const double* x;
    double* y;
    // batched matvec (blockIdx.z / P3 thread group = column c): x, y and the pass buffers of
    // column c are xs[c], ys[c] and the column-0 buffers + c * col{A,B,C} (one rank only)
    int nb;
    const double* xs[kMaxB];
    double* ys[kMaxB];
    int64_t colA, colB, colC;
    int64_t colS;  // several ranks: per-column stride of the peer send blocks (bufS)
    const int8_t* info;
    const double* ibar;
    double2* X2[3];
    double2* X3[6];
    // distribution: rank r owns window rows [ya[r], ya[r+1]) of the spatial
    // passes (P1, P5) and kx columns [kxa[r], kxa[r+1]) of the spectral passes (P2-P4).  The
    // x-transformed planes travel as blocks [source][plane][own rows][dest kx] (P1 -> P2) and
    // [field][plane][dest rows][own kx] (P4 -> P5); the self block is written in place.
    int W, rank;
    // several ranks, chunked exchange: P1 / P2 run for the sources [s0, s1),
    // P4 / P5 for the fields [f0, f1); one launch for all: s0 = 0, s1 = 3, f0 = 0, f1 = nf
    int s0, s1, f0, f1;
    int ya[kMaxRanks + 1], kxa[kMaxRanks + 1];
    int nr[kMaxRanks][9];  // rows of rank p within source b's (0..2) / field f's (3+f) extent
    int kx0, nkx;          // this rank's kx slab
    int lgtk;              // one rank: X1 is kx-tile-major with 2^lgtk kx per tile (= P2's width)
    int lgt4;              // X3 is kx-tile-major with P4's tile width 2^lgt4: [f][plane][tile][ky][t]
    double2* S1[kMaxRanks][3];
    const double2* R1[kMaxRanks][3];
    double2* S2[kMaxRanks][6];
    const double2* R2[kMaxRanks][6];
    const double* Rt;       // tile-major: [q][kx-tile][block][kz'][t], rchunk doubles per tile
    int rchunk;
    int T3, lgT3;           // P3 tile width (power of two) and its log2
    int blk[6][3];
    int nblk;
    const double2* tw;
    // active z-planes (window-relative) of each source orientation / output field: only planes
    // holding panels are transformed along x and y and stored
    const int32_t* planes;  // [9][ZL] lists, then [9][ZL] inverse maps (plane -> index or -1)
    int ZL;
    int nzin[3], nzout[6];
    // P3 direct-z mode (k_p3m): K rows per kx in the tile-major table (rs1 =
    // nblk * ZU + 1 zero row) and the DMMA fragment tables (vc_ctx::p3m_tab)
    int zdirect, ZU, rs1;
    // X2 tile chunk layout [tile][side][plane][t]: per-source arrays (z-FFT mode: x2nz = nzin[b],
    // x2zo = 0) or one stacked-plane array shared by the three sources (direct-z: x2nz = sum of
    // nzin, x2zo[b] = planes of the sources before b)
    int x2nz[3], x2zo[3];
    const int32_t* p3m_tab;
    int p3m_nzt, p3m_kc, p3m_mct;  // stacked padded planes, 4-column chunks, 8-row chunks
    int p3m_nst;                   // k_p3m ring depth
    // odd (E^{z.}) block rows whose negated copies k_p3m writes per tile (row offsets b * ZU + u)
    int p3m_nneg, p3m_oddmask;
    const int32_t* p3m_neg;
    // Tucker-compressed spectra (tucker.cu; vc::Tucker): k_p3m<TK> rebuilds each tile's K rows
    // from U1f (per kx tile, tk_u1t doubles) and Wf (per q, tk_wq doubles) instead of reading Rt
    int tk;
    const double* tk_u1;
    const double* tk_w;
    int tk_u1t, tk_wq, tk_nc, tk_items;
    int tk_nkc[16], tk_u1o[16], tk_wo[16];
};

__device__ __forceinline__ int zlist(const MV& mv, int g, int j) { return mv.planes[g * mv.ZL + j]; }
// rank owning window row y / kx column k (slabs are contiguous; W <= 8)
__device__ __forceinline__ int row_owner(const MV& mv, int y) {
    int p = 0;
    while (y >= mv.ya[p + 1]) ++p;
    return p;
}
__device__ __forceinline__ int kx_owner(const MV& mv, int k) {
    int q = 0;
    while (k >= mv.kxa[q + 1]) ++q;
    return q;
}


// ---- launch helpers ---------------------------------------------------------------------
template <class K>
inline cudaError_t prep(K kern, size_t smem) {
    // all-shared carveout: the FFT passes are shared-memory-resident, so more CTAs per SM
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e) return e;
    // the limit is a process-wide function attribute: contexts of one process (ranks of a
    // thread group) launch with different sizes, so always grant the device maximum (a
    // per-launch value would race) -- occupancy follows the actual launch size
    if (smem > 48 * 1024) return grant_max_dyn_smem(kern, max_dyn_smem());
    return cudaSuccess;
}

// prep() plus an L1-friendly carveout: the shared-memory share of the unified L1 / shared array
// is set to what the kernel's resident CTAs need (register / thread limits included), not the
// maximum, so that the rest stays L1 for the twiddle table and the other cached loads (the FFT
// passes read twiddles through L1; with an all-shared carveout they came from L2).  Falls back to
// the all-shared carveout if the smaller one would lose a CTA per SM.  VC_CARVE=0 disables it.
template <class K>
inline cudaError_t prep_fit(K kern, int nthr, size_t smem) {
    cudaError_t e = prep(kern, smem);
    if (e) return e;
    static const bool on = !(getenv("VC_CARVE") && !atoi(getenv("VC_CARVE")));
    if (!on) return cudaSuccess;
    int nb_max = 0, dev = 0, smsm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb_max, kern, nthr, smem);
    if (e || nb_max <= 0) return e;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smsm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaFuncAttributes fa;
    if ((e = cudaFuncGetAttributes(&fa, kern))) return e;
    const double need = (double)nb_max * ((double)smem + fa.sharedSizeBytes + 1024.0);
    const int pct = std::min(100, (int)std::ceil(100.0 * need / std::max(1, smsm)) + 1);
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct))) return e;
    int nb2 = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb2, kern, nthr, smem);
    if (e || nb2 < nb_max) return cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    return cudaSuccess;
}

template <class K>
inline int persistent_grid(K kern, int nthr, size_t smem, int ntiles) {
    int per_sm = 0, nsm = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nthr, smem);
    return std::max(1, std::min(ntiles, std::max(1, per_sm) * nsm));
}

// ---- P3 direct-z (p3m.cu) -----------------------------------------------------------------
constexpr int kMmaT = 8;       // P3 direct-z tile width (kx per tile)
constexpr int kMmaSplit = 2;   // warps per kx (row-chunk halves)
constexpr int kMmaMC = 8;      // row chunks (8 rows each) per pass: C fragments in registers
constexpr int kP3mMaxStages = 6;
// ring depth that fits shared memory for a shape (0 or 1: the shape cannot run direct-z)
int p3m_stages(int rs1, int nzp, int kc, int mct, bool neg);
size_t p3m_smem(int rs1, int nzp, int kc, int mct, int nst, bool neg);
// Tucker P3: (block, u chunk) items per warp held in registers, and the ring depth that fits
constexpr int kTkItems = 6;
int p3m_tk_stages(int rs1, int nzp, int kc, int mct, int u1t, int wq, bool neg);
cudaError_t launch_p3m(const MV& mv, cudaStream_t st);

}  // namespace vc
