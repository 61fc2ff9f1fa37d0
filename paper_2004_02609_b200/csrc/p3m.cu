// p3m.cu -- P3 of the direct-z matvec on FP64 tensor cores (Eqs. 10-12).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "ctx.h"
#include "mv.cuh"

namespace vc {

// ---------------------------------------------------------------------------------------
// P3, direct-z mode: FFT along x and y only, direct convolution along z.
//   out^f(kx, ky, z_o) = sum_b sum_{z_i} K^{f b}(kx, ky, z_o - z_i) Q^b(kx, ky, z_i)
// with K the x/y-transformed, phase-stripped kernel at the geometric z offset (SURVEY App. B
// applied to x and y only).  Exact like the z-FFT form (no circulant along z at all), and for
// layered structures whose panels occupy few z-planes it costs sum_{f,b} n_out(f) n_in(b)
// complex-by-real MACs per (kx, ky) instead of 3 + n_f z-FFTs.  K is stored on the z-parity
// octant u = (|2 dz + s2| - |s2|) / 2 (s2 = 2 (c_a,z - c_b,z)): even in z except the E^{z.}
// blocks (odd); E^{x.}, E^{y.} carry the factor i (odd along x / y) and E^{y.} the ky sign.
//
// Per (kx, |ky|) the whole P3 is one small real matrix product on FP64 tensor cores (DMMA,
// mma.sync m8n8k4 f64):  C[r][n] = sum_c A[r][c] B[c][n], with
//   r = output row (field f_r, plane z_r), all fields stacked, padded to 8-row chunks;
//   c = input column = stacked plane position (sources one after another, each padded to an
//       even count, the total to a multiple of 4; padding planes hold zeros), 4-column chunks;
//   A[r][c] = K^{f_r b_c}(kx, |ky|, u(z_r - z_c)) (+- for the odd E^{z.} blocks; 0 where the
//             block is absent or for padding) -- the Toeplitz blocks, gathered from the staged
//             K rows through a host-built offset table (vc_ctx::p3m_tab, int16: row | sign);
//   B[c][n] = Q(kx, ky_side, c) re / im of batch column col, n = (col, side, re / im): the 8
//             right-hand sides that share K (both ky signs share the folded spectrum; a
//             single-column launch duplicates column 0).
// Tiles are T = 8 adjacent kx x one |ky| pair.  CTA = 16 warps, one per (kx, half of the row
// chunks); thread 0 also streams each tile into an NST-deep shared-memory ring (full / empty
// mbarriers, no CTA-wide barrier): the K rows ([t][row], one contiguous chunk) with
// cp.async.bulk, the X2 rows ([side][plane][t] per column, 128-byte rows) with 2-D TMA tensor
// copies under the 128-byte swizzle, side 1 shifted by 4 rows, so that a B fragment (4 planes x
// 2 sides of one kx) touches 8 distinct 16-byte bank groups.  The A offsets of a warp are
// tile-invariant and live in registers when its rows fit one pass.
// ---------------------------------------------------------------------------------------

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// X2 stage: 4 (column, side) regions of 128-byte rows (side 1 starts 4 rows early), each a
// whole number of 1024-byte swizzle atoms
__host__ __device__ constexpr int p3m_xregion(int nzp) { return ((nzp + 4) * 128 + 1023) & ~1023; }
// K rows of a stage: [t][rs1], then (neg: odd E^{z.} blocks present) their negated copies at
// row index 8 rs1 + t rs1 + (block row), so that every A entry is a plain shared load
__host__ __device__ constexpr int p3m_kbytes(int rs1, bool neg) { return (8 * kMmaT * rs1 * (neg ? 2 : 1) + 1023) & ~1023; }
static size_t p3m_fixed(int kc, int mct) {  // tables + barriers + k-split exchange (after the stages)
    return 16 * (size_t)mct * 8 + 2 * (size_t)kc * mct * 32 + 4 * (size_t)mct * 8 + 16 * kP3mMaxStages + 64 +
           (mct <= kMmaMC ? (size_t)kMmaT * mct * 32 * 16 : 0);
}
int p3m_stages(int rs1, int nzp, int kc, int mct, bool neg) {
    const size_t st = (size_t)p3m_kbytes(rs1, neg) + 4 * (size_t)p3m_xregion(nzp);
    const size_t avail = 227 * 1024 - 1024 - p3m_fixed(kc, mct);
    return (int)std::min<size_t>(kP3mMaxStages, avail / st);
}
size_t p3m_smem(int rs1, int nzp, int kc, int mct, int nst, bool neg) {
    return 1024 + (size_t)nst * ((size_t)p3m_kbytes(rs1, neg) + 4 * (size_t)p3m_xregion(nzp)) + p3m_fixed(kc, mct);
}
// Tucker P3 (TK): a stage's first region holds the tile's U1 fragments, then (rebuilt in place)
// its K rows; the W fragments of the current q sit after the stages; no k-split exchange buffer
// (K rows in shared memory use the odd stride rs1 | 1: the rebuilt rows of 8 kx land in distinct
// banks)
__host__ __device__ constexpr int p3m_tk_region(int rs1, int u1t, bool neg) {
    return ((8 * u1t > 8 * kMmaT * (rs1 | 1) * (neg ? 2 : 1) ? 8 * u1t : 8 * kMmaT * (rs1 | 1) * (neg ? 2 : 1)) + 1023) &
           ~1023;
}
static size_t p3m_tk_fixed(int kc, int mct, int wq) {
    return (((size_t)8 * wq + 15) & ~(size_t)15) + 16 * (size_t)mct * 8 + 2 * (size_t)kc * mct * 32 +
           4 * (size_t)mct * 8 + 16 * kP3mMaxStages + 64 + 16 * (size_t)kMmaT * kMmaSplit * kTkItems + 16;
}
static size_t p3m_tk_smem(int rs1, int nzp, int kc, int mct, int u1t, int wq, int nst, bool neg) {
    return 1024 + (size_t)nst * ((size_t)p3m_tk_region(rs1, u1t, neg) + 4 * (size_t)p3m_xregion(nzp)) +
           p3m_tk_fixed(kc, mct, wq);
}
int p3m_tk_stages(int rs1, int nzp, int kc, int mct, int u1t, int wq, bool neg) {
    const size_t st = (size_t)p3m_tk_region(rs1, u1t, neg) + 4 * (size_t)p3m_xregion(nzp);
    const size_t fx = 1024 + p3m_tk_fixed(kc, mct, wq);
    if (fx >= 227 * 1024) return 0;
    return (int)std::min<size_t>(2, (227 * 1024 - fx) / st);
}

// A entry: row index | sign << 15 (odd E^{z.} blocks at negative offsets).  The Tucker P3 (PL)
// writes negated copies of the odd rows when it rebuilds them (p3m_kbytes), so its entries are
// plain row indices (measured: for the exact table, negating the rows in shared memory per tile
// costs more than the sign flips it saves, 0.529 -> 0.543 ms per C4 pair launch)
template <bool PL>
__device__ __forceinline__ double p3m_aval(const double* __restrict__ kt, unsigned e16) {
    if constexpr (PL) return kt[e16];
    const double v = kt[e16 & 0x7fff];
    return __longlong_as_double(__double_as_longlong(v) ^ ((long long)(e16 & 0x8000) << 48));
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
        ::"r"(smem_u32(dst)), "l"(tm), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// KS (k-split, all row chunks in one pass): the two warps of a kx share the column chunks
// instead of the rows and exchange partial sums through shared memory (a 64-thread named
// barrier per pair), each storing half of the row chunks.  Measured on C4 (pair launch):
// 0.61 ms vs 0.54 ms for the row split, so KS is off unless VC_P3M_KS=1 (A/B).
// Tucker P3: the K-row items k = 0..NI-1 of this warp (item = warp + 16 k = (block, u chunk)),
// C = U1 W[q] on the tensor cores as NI interleaved accumulation chains over the rank chunks
template <int NI>
__device__ __forceinline__ void tk_rebuild(double (&cr)[kTkItems][2], const double* __restrict__ u1s,
                                           const double* __restrict__ wsm, const int4* __restrict__ it4, int nkc,
                                           int lane) {
    int ao[NI], bo[NI];
#pragma unroll
    for (int k = 0; k < NI; ++k) {
        const int4 d = it4[k * kMmaT * kMmaSplit];
        ao[k] = d.x + lane;
        bo[k] = d.y + lane;
        cr[k][0] = cr[k][1] = 0.0;
    }
    for (int kc = 0; kc < nkc; ++kc) {
        double a[NI], bv[NI];
#pragma unroll
        for (int k = 0; k < NI; ++k) {
            a[k] = u1s[ao[k] + kc * 32];
            bv[k] = wsm[bo[k] + kc * 32];
        }
#pragma unroll
        for (int k = 0; k < NI; ++k) dmma884(cr[k][0], cr[k][1], a[k], bv[k]);
    }
}

// TK (Tucker-compressed spectra, tucker.cu): the stage carries the tile's U1 fragments instead
// of its K rows; every warp first rebuilds (block, u chunk) items of K = U1 W[q] on the tensor
// cores (W[q] resident in shared memory, reloaded by the producer when q changes: each CTA walks
// one contiguous, q-major range of tiles), a CTA barrier, the K rows are written over the U1
// fragments, a second barrier, then the MAC runs unchanged.
template <int MC, int KCM, bool KS, bool TK>
__global__ void __launch_bounds__(kMmaT * kMmaSplit * 32, 1)
    k_p3m(const __grid_constant__ CUtensorMap tmx0, const __grid_constant__ CUtensorMap tmx1, MV mv) {
    constexpr int T = kMmaT, NW = kMmaT * kMmaSplit, NTHR = NW * 32;
    extern __shared__ __align__(1024) uint8_t smraw[];
    // 1024-byte alignment for the 128B-swizzle TMA boxes, computed on the shared-window address
    // so that the pointers stay shared-space (LDS, not generic loads)
    uint8_t* const sm = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nkx = mv.nkx, My = mv.My;
    const int nt3 = (nkx + T - 1) / T;
    const int ntiles = nt3 * (My / 2 + 1);
    const int nb = mv.nb, nzp = mv.p3m_nzt, KC = mv.p3m_kc, MCT = mv.p3m_mct, RS1 = mv.rs1;
    const int NST = mv.p3m_nst;
    const int RC = T * RS1;
    const bool NEG = TK && mv.p3m_nneg > 0;
    const int KB = TK ? p3m_tk_region(RS1, mv.tk_u1t, NEG) : p3m_kbytes(RS1, NEG);
    const int XR = p3m_xregion(nzp), SB = KB + 4 * XR;  // stage bytes
    const int lg4 = mv.lgt4;
    const int nt4 = (nkx + (1 << lg4) - 1) >> lg4;
    const int WB = TK ? ((8 * mv.tk_wq + 15) & ~15) : 0;  // W[q] fragments (TK)
    double* const wsm = reinterpret_cast<double*>(sm + (size_t)NST * SB);
    longlong2* const rdesc = reinterpret_cast<longlong2*>(sm + (size_t)NST * SB + WB);  // [MCT * 8]
    uint16_t* const atab = reinterpret_cast<uint16_t*>(rdesc + MCT * 8);             // [KC][MCT][32]
    int* const rtab = reinterpret_cast<int*>(atab + ((KC * MCT * 32 + 1) & ~1));     // [MCT * 8]
    uint64_t* const full = reinterpret_cast<uint64_t*>(rtab + ((MCT * 8 + 1) & ~1));
    uint64_t* const empty = full + kP3mMaxStages;
    uint64_t* const wbar = empty + kP3mMaxStages;  // TK: W[q] landed
    // TK: per (item k, warp) the tile-invariant offsets {U1 fragment, W fragment, K row of the
    // chunk, u left in the chunk} of the warp's (block, u chunk) items, [k][warp]
    int4* const tki = reinterpret_cast<int4*>((reinterpret_cast<uintptr_t>(wbar + 2) + 15) & ~(uintptr_t)15);
    double2* const xch = reinterpret_cast<double2*>(empty + kP3mMaxStages);  // KS: [T][MCT][32]
    const int KS1 = TK ? (RS1 | 1) : RS1;  // K row stride in shared memory
    if (TK)
        for (int e = threadIdx.x; e < kTkItems * NW; e += NTHR) {
            const int k = e / NW, w = e % NW;
            const int item = w + k * NW;
            int4 v = make_int4(0, 0, 0, 0);
            if (item < mv.tk_items) {
                const int b = item / mv.tk_nc, ncc = item - b * mv.tk_nc;
                v = make_int4(mv.tk_u1o[b], mv.tk_wo[b] + ncc * mv.tk_nkc[b] * 32, b * mv.ZU + 8 * ncc,
                              (mv.ZU - 8 * ncc) | ((mv.p3m_oddmask >> b & 1) << 16));
            }
            tki[e] = v;
        }
    {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(mv.p3m_tab);
        uint32_t* dst = reinterpret_cast<uint32_t*>(atab);
        const int na = KC * MCT * 16;  // uint16 pairs
        for (int e = threadIdx.x; e < na; e += NTHR) dst[e] = src[e];
        for (int e = threadIdx.x; e < MCT * 8; e += NTHR) rtab[e] = (int)src[na + e];
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        if (TK) mbar_init(wbar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    // output rows, once per CTA: X3 offset of the row's plane relative to X3[0] (x = -1:
    // padding row) and the i-factor / ky-sign flags
    for (int r = threadIdx.x; r < MCT * 8; r += NTHR) {
        const int fj = rtab[r];
        longlong2 d = make_longlong2(-1, 0);
        if (fj >= 0) {
            const int f = fj & 15, jo = fj >> 4;
            const bool ifac = mv.fkind[f] == 1 && mv.faxis[f] != 2;  // E^{x.}, E^{y.}: R holds Im(K)
            const bool oddy = ifac && mv.faxis[f] == 1;              // odd along y: ky < 0 side
            d.x = (long long)(mv.X3[f] - mv.X3[0]) + (((long long)jo * nt4 * My) << lg4);
            d.y = (ifac ? 1 : 0) | (oddy ? 2 : 0);
        }
        rdesc[r] = d;
    }
    __syncthreads();
    // producer: thread 0 streams the tiles, NST - 1 ahead of its own compute; before refilling
    // a stage it waits until all warps released that stage's previous tile
    const unsigned kbytes = TK ? (unsigned)(8 * mv.tk_u1t) : (unsigned)(8 * RC), xbox = (unsigned)(128 * (nzp + 4));
    // tiles of this CTA: strided over the grid, or (TK) one contiguous q-major range, so that
    // W[q] changes only every nt3 tiles
    const int tbeg = TK ? (int)((long long)ntiles * blockIdx.x / gridDim.x) : 0;
    const int tend = TK ? (int)((long long)ntiles * (blockIdx.x + 1) / gridDim.x) : ntiles;
    auto tile_of = [&](int j) { return TK ? tbeg + j : (int)blockIdx.x + j * (int)gridDim.x; };
    // producer state of the next issue (tile, stage, round): no runtime divisions per tile
    const int tstride = TK ? 1 : (int)gridDim.x;
    int ptl = tile_of(0), ps = 0, pround = 0;
    auto load = [&](int tl, int s) {  // tile tl into stage s (the stage is free)
        uint8_t* st = sm + (size_t)s * SB;
        mbar_arrive_expect_tx(&full[s], kbytes + (unsigned)(2 * nb) * xbox);
        if (TK) bulk_g2s(st, mv.tk_u1 + (size_t)(tl % nt3) * mv.tk_u1t, kbytes, &full[s]);
        else bulk_g2s(st, mv.Rt + (size_t)tl * RC, kbytes, &full[s]);
        // side 0: rows [row0, row0 + nzp + 4) (the last 4 land in the region's slack); side 1:
        // rows [row0 + nzp - 4, row0 + 2 nzp), so its plane p sits in region row p + 4
        const int row0 = tl * 2 * nzp;
        tma_load_2d(st + KB, &tmx0, 0, row0, &full[s]);
        tma_load_2d(st + KB + XR, &tmx0, 0, row0 + nzp - 4, &full[s]);
        if (nb > 1) {
            tma_load_2d(st + KB + 2 * XR, &tmx1, 0, row0, &full[s]);
            tma_load_2d(st + KB + 3 * XR, &tmx1, 0, row0 + nzp - 4, &full[s]);
        }
    };
    auto issue = [&](int j) {  // this CTA's j-th tile into stage j % NST (j issued in order)
        const int tl = ptl;
        if (tl >= tend) return;
        const int s = ps;
        ptl += tstride;
        if (++ps == NST) ps = 0;
        if (j >= NST) mbar_wait(&empty[s], (pround - 1) & 1);
        if (ps == 0) ++pround;
        load(tl, s);
    };

    auto wissue = [&](int j) {  // TK: W fragments of tile j's q (all blocks, one bulk copy)
        const int q = tile_of(j) / nt3;
        mbar_arrive_expect_tx(wbar, (unsigned)(8 * mv.tk_wq));
        bulk_g2s(wsm, mv.tk_w + (size_t)q * mv.tk_wq, (unsigned)(8 * mv.tk_wq), wbar);
    };
    const bool producer = threadIdx.x == 0;
    if (producer) {
        if (TK && tbeg < tend) wissue(0);
        for (int j = 0; j < NST - 1; ++j) issue(j);
    }
    const int t = warp & (T - 1), half = warp / T;
    const int h0 = (MCT + 1) >> 1;  // row chunks stored by (!KS: computed by) the first half
    const int mlo = KS ? 0 : (half ? h0 : 0), mhi = KS ? MCT : (half ? MCT : h0);
    const int kh = (KC + 1) >> 1;   // KS: column chunks of the first half
    const int klo = KS ? (half ? kh : 0) : 0, khi = KS ? (half ? KC : kh) : KC;
    const int slo = half ? h0 : 0, shi = half ? MCT : h0;  // KS: row chunks this warp stores
    // this lane's B element (k = lane % 4, n = lane / 4 = (column, side, re / im)) of column
    // chunk kc: stacked plane p = 4 kc + lane % 4 in 128-byte row p (side 0) or p + 4 (side 1)
    // of its region, 16-byte chunk t swizzled by the row (SWIZZLE_128B: chunk ^= row & 7)
    const int bcol = min((lane >> 4) & 1, nb - 1), bside = (lane >> 3) & 1, breim = (lane >> 2) & 1;
    const int brow0 = (lane & 3) + 4 * bside;  // row of chunk 0; chunk kc adds 4 kc rows
    const int boff0 = KB + (bcol * 2 + bside) * XR + brow0 * 128 + breim * 8;
    // (brow0 + 4 kc) & 7 = (brow0 + 4 (kc & 1)) & 7: the swizzled t alternates with kc parity
    const int bsw0 = (t ^ (brow0 & 7)) << 4, bsw1 = (t ^ ((brow0 + 4) & 7)) << 4;
    // A offsets of the whole tile in registers when the warp's rows fit one pass and KC <= KCM
    // (measured: guarded loops over the template bounds beat exact-count instantiations)
    const int nkw = khi - klo;  // column chunks of this warp
    const bool fast = mhi - mlo <= MC && nkw <= KCM;
    uint32_t ar[KCM][(MC + 1) / 2];
    if (fast) {
#pragma unroll
        for (int k = 0; k < KCM; ++k)
#pragma unroll
            for (int m = 0; m < MC; m += 2) {
                const int kk = klo + k;
                const uint32_t lo = k < nkw && mlo + m < mhi ? atab[(kk * MCT + mlo + m) * 32 + lane] : 0u;
                const uint32_t hi = k < nkw && mlo + m + 1 < mhi ? atab[(kk * MCT + mlo + m + 1) * 32 + lane] : 0u;
                ar[k][m / 2] = lo | hi << 16;
            }
    }
    const int ocol = (lane & 3) >> 1, oside = lane & 1;  // this lane's C columns (see below)
    double2* const X3c = mv.X3[0] + ocol * mv.colC;
    int qprev = -1, nwl = 0;  // TK: q of the resident W, W loads waited for
    // consumer state: tile, stage and phase, and the tile's (q, x tile) advanced without divisions
    int tl = tile_of(0), s = 0, sph = 0;
    int q = tl / nt3, xti = tl - q * nt3;
    const int dq = tstride / nt3, dxt = tstride - dq * nt3;
    for (int it = 0; tl < tend; ++it) {
        if (producer) issue(it + NST - 1);
        mbar_wait(&full[s], sph);
        const uint8_t* stg = sm + (size_t)s * SB;
        if constexpr (TK) {
            if (q != qprev) {
                mbar_wait(wbar, nwl & 1);
                ++nwl;
                qprev = q;
            }
            // K rows of the tile: item = (block, 8-wide u chunk), C[t][u] = sum_i U1[t][i] W[i][u];
            // a warp's items (warp, warp + 16, ...) run as interleaved chains (uniform rank chunks)
            const double* u1s = reinterpret_cast<const double*>(stg);
            double cr[kTkItems][2];
            const int nit = max(0, (mv.tk_items - warp + NW - 1) / NW);
            const int4* it4 = tki + warp;  // item k at it4[k * NW]
            const int nkc = mv.tk_nkc[0];
            switch (nit) {
                case 1: tk_rebuild<1>(cr, u1s, wsm, it4, nkc, lane); break;
                case 2: tk_rebuild<2>(cr, u1s, wsm, it4, nkc, lane); break;
                case 3: tk_rebuild<3>(cr, u1s, wsm, it4, nkc, lane); break;
                case 4: tk_rebuild<4>(cr, u1s, wsm, it4, nkc, lane); break;
                case 5: tk_rebuild<5>(cr, u1s, wsm, it4, nkc, lane); break;
                case 6: tk_rebuild<6>(cr, u1s, wsm, it4, nkc, lane); break;
                default: break;
            }
            __syncwarp();
            asm volatile("bar.sync 15, %0;\n" ::"n"(NTHR) : "memory");  // U1 and W reads done
            const int tn = tile_of(it + 1);
            if (producer && tn < tend && tn / nt3 != q) wissue(it + 1);
            double* kw = reinterpret_cast<double*>(sm + (size_t)s * SB);
            const int uo = 2 * (lane & 3), ko = (lane >> 2) * KS1 + uo;
#pragma unroll
            for (int k = 0; k < kTkItems; ++k) {
                if (k < nit) {
                    const int4 d = it4[k * NW];
                    const int rem = d.w & 0xffff;
                    if (uo < rem) kw[d.z + ko] = cr[k][0];
                    if (uo + 1 < rem) kw[d.z + ko + 1] = cr[k][1];
                    if (d.w >> 16) {  // odd block: the negated copy too
                        if (uo < rem) kw[8 * KS1 + d.z + ko] = -cr[k][0];
                        if (uo + 1 < rem) kw[8 * KS1 + d.z + ko + 1] = -cr[k][1];
                    }
                }
            }
            if (threadIdx.x < T) kw[threadIdx.x * KS1 + RS1 - 1] = 0.0;  // the zero row
            __syncwarp();
            asm volatile("bar.sync 15, %0;\n" ::"n"(NTHR) : "memory");  // K rows complete
        }
        const double* __restrict__ kt_ = reinterpret_cast<const double*>(stg) + t * KS1;
        const uint8_t* xb_ = stg + boff0;
        const int kx = xti * T + t;
        const int nside = (q == 0 || 2 * q == My) ? 1 : 2;
        const bool store = kx < nkx && ocol < nb && oside < nside;
        const int64_t oofs = ((int64_t)(kx >> lg4) * My + (oside ? My - q : q)) << lg4 | (kx & ((1 << lg4) - 1));
        for (int mc0 = mlo; mc0 < mhi; mc0 += MC) {
            double c[MC][2];
#pragma unroll
            for (int m = 0; m < MC; ++m) c[m][0] = c[m][1] = 0.0;
            if (fast && mc0 + MC <= mhi) {  // all MC row chunks: no per-chunk guards
#pragma unroll
                for (int k = 0; k < KCM; ++k) {
                    if (k >= nkw) break;
                    const int kk = klo + k;
                    const double bv = *reinterpret_cast<const double*>(xb_ + kk * 512 + ((kk & 1) ? bsw1 : bsw0));
#pragma unroll
                    for (int m = 0; m < MC; ++m)
                        dmma884(c[m][0], c[m][1], p3m_aval<TK>(kt_, (ar[k][m / 2] >> (16 * (m & 1))) & 0xffff), bv);
                }
            } else if (fast) {
#pragma unroll
                for (int k = 0; k < KCM; ++k) {
                    if (k >= nkw) break;
                    const int kk = klo + k;
                    const double bv = *reinterpret_cast<const double*>(xb_ + kk * 512 + ((kk & 1) ? bsw1 : bsw0));
#pragma unroll
                    for (int m = 0; m < MC; ++m)
                        if (mc0 + m < mhi)
                            dmma884(c[m][0], c[m][1], p3m_aval<TK>(kt_, (ar[k][m / 2] >> (16 * (m & 1))) & 0xffff), bv);
                }
            } else {
                for (int kc = klo; kc < khi; ++kc) {
                    const double bv = *reinterpret_cast<const double*>(xb_ + kc * 512 + ((kc & 1) ? bsw1 : bsw0));
                    const uint16_t* at = atab + (kc * MCT + mc0) * 32 + lane;
#pragma unroll
                    for (int m = 0; m < MC; ++m)
                        if (mc0 + m < mhi) dmma884(c[m][0], c[m][1], p3m_aval<TK>(kt_, at[m * 32]), bv);
                }
            }
            if (mc0 + MC >= mhi) {  // last read of this stage: release it to the producer
                if (TK) fence_proxy_async();  // K rows were written here (generic proxy)
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }
            if (KS) {  // exchange the partial sums of the row chunks the partner warp stores
                double2* xo = xch + (size_t)t * MCT * 32 + lane;
#pragma unroll
                for (int m = 0; m < MC; ++m)
                    if (m < MCT && (m < slo || m >= shi)) xo[m * 32] = make_double2(c[m][0], c[m][1]);
                asm volatile("bar.sync %0, 64;\n" ::"r"(1 + t) : "memory");
#pragma unroll
                for (int m = 0; m < MC; ++m)
                    if (m >= slo && m < shi) {
                        const double2 v = xo[m * 32];
                        c[m][0] += v.x;
                        c[m][1] += v.y;
                    }
                asm volatile("bar.sync %0, 64;\n" ::"r"(1 + t) : "memory");  // buffer reused next tile
            }
            // C fragment: row lane / 4 of the chunk, right-hand sides n = 2 (lane % 4) + {0, 1} =
            // (column (lane % 4) / 2, side lane % 2, re / im)
            if (store) {
#pragma unroll
                for (int m = 0; m < MC; ++m) {
                    if (mc0 + m >= mhi) break;
                    if (KS && (m < slo || m >= shi)) continue;
                    const longlong2 d = rdesc[(mc0 + m) * 8 + (lane >> 2)];
                    if (d.x < 0) continue;
                    double2 a = make_double2(c[m][0], c[m][1]);
                    if (d.y & 1) {  // times i; the odd-in-y blocks flip sign on the ky < 0 side
                        a = ((d.y & 2) && oside) ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
                    }
                    X3c[d.x + oofs] = a;
                }
            }
        }
        if (mhi <= mlo) {  // no rows for this half: still release the stage
            if (TK) fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        tl += tstride;
        q += dq;
        xti += dxt;
        if (xti >= nt3) {
            xti -= nt3;
            ++q;
        }
        if (++s == NST) {
            s = 0;
            sph ^= 1;
        }
    }
}

// TMA descriptor of one column's X2 (direct-z layout: rows of 8 kx x complex128 = 128 bytes)
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static cudaError_t p3m_tensor_map(CUtensorMap* tm, const double2* base, uint64_t rows, int box_rows) {
    static PFN_encodeTiled enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
        enc = reinterpret_cast<PFN_encodeTiled>(fn);
    }
    const cuuint64_t dims[2] = {16, rows};           // doubles per row, rows
    const cuuint64_t strides[1] = {128};             // bytes between rows
    const cuuint32_t box[2] = {16, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double2*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_p3m(const MV& mv, cudaStream_t st) {
    const int nt3 = (mv.nkx + kMmaT - 1) / kMmaT;
    const int ntiles = nt3 * (mv.My / 2 + 1);
    if (ntiles == 0 || mv.p3m_mct == 0) return cudaSuccess;
    const bool tk = mv.tk != 0;
    const int nst = mv.p3m_nst;
    const size_t smem = tk ? p3m_tk_smem(mv.rs1, mv.p3m_nzt, mv.p3m_kc, mv.p3m_mct, mv.tk_u1t, mv.tk_wq, nst,
                                         mv.p3m_nneg > 0)
                           : p3m_smem(mv.rs1, mv.p3m_nzt, mv.p3m_kc, mv.p3m_mct, nst, false);
    if (nst < 2 || smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    // X2 of each column as a 2-D tensor of 128-byte rows, boxes of nzp + 4 rows.  The maps depend
    // only on the buffers and the shape, so they are encoded once and cached (per host thread:
    // the ranks of a thread group launch concurrently)
    const uint64_t rows = (uint64_t)ntiles * 2 * mv.p3m_nzt;
    struct TmKey {
        const void* b0;
        const void* b1;
        uint64_t rows;
        int box;
    };
    struct TmEnt {
        TmKey k;
        CUtensorMap tm[2];
    };
    thread_local TmEnt cache[4];
    thread_local int cache_n = 0, cache_next = 0;
    const TmKey key = {mv.X2[0], mv.X2[0] + (mv.nb > 1 ? mv.colB : 0), rows, mv.p3m_nzt + 4};
    const CUtensorMap* tm = nullptr;
    for (int i = 0; i < cache_n && !tm; ++i)
        if (!memcmp(&cache[i].k, &key, sizeof key)) tm = cache[i].tm;
    if (!tm) {
        TmEnt& en = cache[cache_next];
        cache_next = (cache_next + 1) % 4;
        cache_n = std::min(cache_n + 1, 4);
        memset(&en.k, 0, sizeof en.k);
        for (int c = 0; c < 2; ++c) {
            cudaError_t e = p3m_tensor_map(&en.tm[c], c ? static_cast<const double2*>(key.b1) : mv.X2[0], rows,
                                           mv.p3m_nzt + 4);
            if (e) return e;
        }
        en.k = key;
        tm = en.tm;
    }
    // k-split (KS) when all row chunks fit one pass; else row halves in balanced passes
    static const bool ks_env = getenv("VC_P3M_KS") && atoi(getenv("VC_P3M_KS"));
    const bool ks = mv.p3m_mct <= kMmaMC && ks_env && !tk;
    const int npass = ks ? 1 : (((mv.p3m_mct + 1) >> 1) + kMmaMC - 1) / kMmaMC;
    const int mc = ks ? mv.p3m_mct : (((mv.p3m_mct + 1) >> 1) + npass - 1) / npass;
    const int kw = ks ? (mv.p3m_kc + 1) >> 1 : mv.p3m_kc;  // column chunks per warp
    const int kcm = kw <= 4 ? 4 : kw <= 8 ? 8 : kw <= 10 ? 10 : kw <= 12 ? 12 : 16;
    constexpr int NT = kMmaT * kMmaSplit * 32;
    cudaError_t e = cudaSuccess;
    // one CTA per SM (16 warps, shared memory sized for the ring): the grid is the SM count
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int grid = std::max(1, std::min(ntiles, nsm));
#define VC_P3M_K2(M, KK, KSV, TKV)                                                             \
    {                                                                                          \
        static bool granted = false; /* process-wide attribute: grant the maximum once */      \
        if (!granted) {                                                                        \
            e = prep(k_p3m<M, KK, KSV, TKV>, 227 * 1024);                                      \
            if (e) return e;                                                                   \
            granted = true;                                                                    \
        }                                                                                      \
        k_p3m<M, KK, KSV, TKV><<<grid, NT, smem, st>>>(tm[0], tm[1], mv);                      \
    }
#define VC_P3M_K(M, KK)                                                                        \
    case KK:                                                                                   \
        if (tk) VC_P3M_K2(M, KK, false, true)                                                  \
        else if (ks) VC_P3M_K2(M, KK, true, false) else VC_P3M_K2(M, KK, false, false)        \
        break;
#define VC_P3M_CASE(M)                                                                         \
    case M:                                                                                    \
        switch (kcm) { VC_P3M_K(M, 4) VC_P3M_K(M, 8) VC_P3M_K(M, 10) VC_P3M_K(M, 12)         \
                       VC_P3M_K(M, 16)                                                        \
                       default: return cudaErrorInvalidValue; }                                \
        break;
    switch (mc) {
        VC_P3M_CASE(1) VC_P3M_CASE(2) VC_P3M_CASE(3) VC_P3M_CASE(4)
        VC_P3M_CASE(5) VC_P3M_CASE(6) VC_P3M_CASE(7) VC_P3M_CASE(8)
        default: return cudaErrorInvalidValue;
    }
#undef VC_P3M_CASE
#undef VC_P3M_K
#undef VC_P3M_K2
    return cudaGetLastError();
}


}  // namespace vc
