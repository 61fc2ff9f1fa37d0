// operator.cu -- FFT-accelerated Galerkin matvec (DESIGN.md a2-a8; Eqs. 9-12).
//
// Data flow of one matvec (all complex128, kx fastest, window origin lo = min panel slot):
//   P1  x  --scatter + R2C along x (two real lines per complex FFT)-->  X1[b][z<ez][y<ey][kx]
//   P2  X1 --C2C along y, zero-padded to My, times phi-bar_b,y-->        X2[b][z<ez][ky][kx]
//   P3  X2 --C2C along z, times phi-bar_b,z; MAC with the folded real spectra R^{f,b};
//           times i (E blocks) and phi_f,z; inverse C2C along z, pruned-->  X3[f][z<ez_f][ky][kx]
//   P4  X3 --times phi_f,y; inverse C2C along y, pruned-->             X4[f][z][y<ey_f][kx]
//   P5  X4 --times phi_f,x; C2R along x (two lines per complex FFT); gather at the f-panels:
//           y_k = C^a[slot_k] (conductor rows) or s_k D^a[slot_k] + Ī_k x_k (dielectric rows)
// K^{ab}(k) = phi_a(k) R^{ab}(k) conj(phi_b(k)), phi_g(k) = exp(2 pi i sum_c kt_c cg_c / M_c),
// R real for P blocks and i*real for E blocks, even / odd (E along a) in each kt_c, so only the
// octant 0 <= kt_c <= M_c/2 is stored; R^{yx} = R^{xy} (Eq. 12 after phase stripping).
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "ctx.h"
#include "fft.cuh"
#include "kgen.cuh"
#include "mv.cuh"

namespace vc {

// ---- tile-size choices (compile-time functions of the FFT length) -----------------------
constexpr int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
// x passes (contiguous lines): T pencils of length L per CTA with NT threads (one stage-0
// radix-16 butterfly per thread) and 32 KB of shared memory (L <= 2048), so ~6 CTAs per SM
// overlap their load, transform and store phases.  y passes (strided, pencil = one kx column)
// keep 4 adjacent kx per CTA (64-byte row segments; measured faster than 2).
template <int L> struct FX {
    static constexpr int T = clampi(2048 / L, 1, 64);
    static constexpr int NT = clampi(T * L / 16, 64, 256);
    // register caps (measured on C4): P1 best at <= 96 (5 CTAs/SM), P5 at <= 128 (no spills)
    static constexpr int MINB = 65536 / (NT * 96) < 1 ? 1 : 65536 / (NT * 96);
#ifndef VC_P5_REGS
#define VC_P5_REGS 128
#endif
    static constexpr int MINB5 = 65536 / (NT * VC_P5_REGS) < 1 ? 1 : 65536 / (NT * VC_P5_REGS);
};
// Tile widths the host layout code must agree with (X1 is tiled by P2's width, X3 by P4's):
// operator_build sizes and indexes those arrays through these two functions only.
constexpr int p2_tile(int L) { return clampi(4096 / L, 2, 32); }  // FY<L>::T
constexpr int kP2Ahead = 2 * 148;  // P2's L2 prefetch distance in blocks (two resident CTAs per SM)
constexpr int kP4KB = 32;                                          // P4's shared KB per stage
constexpr int p4_tile(int L) { return clampi(kP4KB * 64 / L, 1, 32); }  // FYS<L, kP4KB>::T
#ifndef VC_P2_MINB
#define VC_P2_MINB 0  // 0: no minimum-blocks bound (nvcc then caps P2 at 120 registers; an
                      // explicit 1 lets it take 142 and halves the CTAs per SM: 0.32 -> 0.48 ms)
#endif
template <int L> struct FY {
    static constexpr int T = p2_tile(L);  // >= 2 adjacent kx: 32-byte row segments
    // 256 threads; 512 at L = 4096 (C5), where a CTA holds 2 pencils of 4096: one stage-0
    // butterfly per thread (P2's bulk-fed stage 0) and 16 warps on the one CTA per SM
    static constexpr int NT = L >= 4096 ? 512 : 256;
    static constexpr int MINB2 = VC_P2_MINB;  // P2's register cap (launch bounds)
};
template <int L> struct TX { static constexpr int T = FX<L>::T; };
template <int L> struct TY { static constexpr int T = FY<L>::T; };
constexpr int kNT = 256;
constexpr int kNT3 = 256;  // P3 threads per CTA
constexpr int kMaxLz = 256;  // largest z FFT length (P3 keeps whole z-pencils in shared memory)

__device__ __forceinline__ int ktil(int k, int M) { return k <= M / 2 ? k : k - M; }

// ---------------------------------------------------------------------------------------
// P1: scatter + forward R2C along x
// ---------------------------------------------------------------------------------------
// D: multi-rank (slab-partitioned) build; D = false compiles out the owner lookups
template <int L, bool D>
__global__ void __launch_bounds__(FX<L>::NT, FX<L>::MINB) k_p1(MV mv) {
    constexpr int T = TX<L>::T;
    extern __shared__ double2 sm[];
    const int beta = blockIdx.y + mv.s0;
    const int ex = mv.ext_in[beta][0];
    if (ex == 0) return;
    const int nrow = mv.nr[mv.rank][beta];  // own rows of this source grid
    // rows are paired (two real lines per complex FFT) at absolute slot rows (2m, 2m + 1), so a
    // slab split changes no pairing and the partitioned matvec stays bitwise equal (local row
    // l = 2q - s is the real part, l + 1 the imaginary part)
    const int s = (mv.lo[1] + mv.ya[mv.rank]) & 1;
    const int nyp = (nrow + s + 1) >> 1;
    const int nch = (nyp + T - 1) / T;
    if (nch == 0) return;
    const int j = blockIdx.x / nch, ch = blockIdx.x % nch;
    if (j >= mv.nzin[beta]) return;
    const int z = zlist(mv, beta, j);
    const int32_t* __restrict__ smap = mv.slotmap[beta];
    const int Gx = mv.G[beta][0], Gy = mv.G[beta][1];
    const int64_t zrow =
        ((int64_t)(z + mv.lo[2]) * Gy + mv.lo[1] + mv.ya[mv.rank]) * Gx + mv.lo[0];
    const double* __restrict__ x = mv.xs[blockIdx.z];
    // branch-free (predicated loads, selects), so the unrolled stage-0 loop issues all its
    // slot-map loads, then all its x loads, instead of one dependent pair at a time
    auto ld0 = [&](int t, int n) -> double2 {
        const int q = ch * T + t;
        const int l0 = 2 * q - s;
        const bool ok = q < nyp && n < ex;
        const bool v0 = ok && l0 >= 0, v1 = ok && l0 + 1 < nrow;
        const int64_t r0 = zrow + (int64_t)l0 * Gx + n;
        const int32_t e0 = v0 ? __ldg(smap + r0) : -1;
        const int32_t e1 = v1 ? __ldg(smap + r0 + Gx) : -1;
        // (predicated, not clamped to x[0]: a rank may own no panels, x == nullptr)
        const double a = e0 >= 0 ? __ldg(x + (e0 & kSlotIdx)) : 0.0;
        const double b = e1 >= 0 ? __ldg(x + (e1 & kSlotIdx)) : 0.0;
        return make_double2(a, b);
    };
    auto sts = [&](int t, int p, double2 v) { sm[smi<L, T, false>(t, p)] = v; };
    fft_run<L, T, FX<L>::NT, false, false>(sm, ld0, sts, mv.tw);
    __syncthreads();
    constexpr int K = L / 2 + 1;
    const bool ph = beta != 0;  // c_beta,x = 1/2 for y- and z-normal panels
    double2* const S1self = mv.S1[0][beta] + blockIdx.z * mv.colA;
    for (int u = threadIdx.x; u < T * K; u += FX<L>::NT) {
        const int t = u / K, k = u % K;
        const int q = ch * T + t;
        if (q >= nyp) continue;
        const double2 zk = sm[smi<L, T, false>(t, Plan<L>::pos(k))];
        const double2 zm = sm[smi<L, T, false>(t, Plan<L>::pos((L - k) & (L - 1)))];
        double2 A = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
        double2 B = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
        if (ph) {
            const double2 w = half_phase(mv.tw, k, L, -1);
            A = cmul(A, w);
            B = cmul(B, w);
        }
        const int qd = D ? kx_owner(mv, k) : 0;
        const int k0 = D ? mv.kxa[qd] : 0;
        const int nk = D ? mv.kxa[qd + 1] - k0 : mv.nkx;
        const int l0 = 2 * q - s;
        if (D) {
            double2* o = mv.S1[qd][beta] + blockIdx.z * (qd == mv.rank ? mv.colA : mv.colS) +
                         ((int64_t)j * nrow + l0) * nk + (k - k0);
            if (l0 >= 0) o[0] = A;
            if (l0 + 1 < nrow) o[nk] = B;
        } else {  // one rank: [plane][kx tile][row][kx % tk], so P2 reads each tile contiguously
            const int tk = 1 << mv.lgtk, ntk = (nk + tk - 1) >> mv.lgtk;
            const int rowtk = nrow << mv.lgtk;  // elements of one kx tile of the plane
            double2* o = S1self + (int64_t)j * ntk * rowtk + ((k >> mv.lgtk) * rowtk + l0 * tk + (k & (tk - 1)));
            if (l0 >= 0) o[0] = A;
            if (l0 + 1 < nrow) o[tk] = B;
        }
    }
}

// ---------------------------------------------------------------------------------------
// P2: forward C2C along y (zero-padded input), times conj(phi_beta,y)
// ---------------------------------------------------------------------------------------
template <int L, bool D>
#if VC_P2_MINB > 0
__global__ void __launch_bounds__(FY<L>::NT, FY<L>::MINB2) k_p2(MV mv) {
#else
__global__ void __launch_bounds__(FY<L>::NT) k_p2(MV mv) {
#endif
    constexpr int T = TY<L>::T;
    extern __shared__ double2 sm[];
    const int beta = blockIdx.y + mv.s0;
    const int ex = mv.ext_in[beta][0], ey = mv.ext_in[beta][1], ez = mv.ext_in[beta][2];
    if (ex == 0) return;
    const int nkx = mv.nkx;  // own kx slab (local column kx)
    const int ntile = (nkx + T - 1) / T;
    if (ntile == 0) return;
    // direct-z: the planes of one kx tile are adjacent blocks (their X2 elements share sectors)
    const int nzb = mv.nzin[beta];
    if (nzb == 0) return;
    // planes fastest in the grid when X2 elements of adjacent planes share a sector (direct-z, or
    // a one-kx P3 tile: C5), so the CTAs writing the two halves of a sector run together and L2
    // merges them before eviction (kx fastest otherwise)
    const bool jfast = mv.zdirect || mv.T3 == 1;
    const int j = jfast ? blockIdx.x % nzb : blockIdx.x / ntile;
    const int tile = jfast ? blockIdx.x / nzb : blockIdx.x % ntile;
    if (j >= nzb || tile >= ntile) return;
    (void)ez;
    // X2 tile-major for P3, q = |ky| (ky <= L/2: side 0): [q][kx / T3][side][plane][kx % T3],
    // plane = x2zo + j of x2nz (z-FFT mode: per source; direct-z: the stacked sources, each
    // padded to an even count, zero padding planes)
    double2* __restrict__ out = mv.X2[beta] + blockIdx.z * mv.colB;
    const int nt3 = (nkx + mv.T3 - 1) >> mv.lgT3;
    const bool ph = beta != 1;  // c_beta,y = 1/2 for x- and z-normal panels
    // (!D) tile `tile` of plane j: T adjacent kx of all ey rows, contiguous
    const double2* const in0 = mv.R1[0][beta] + blockIdx.z * mv.colA + (int64_t)j * ntile * ey * T;
    auto ld0 = [&](int t, int n) -> double2 {
        const int kx = tile * T + t;
        if (n >= ey || kx >= nkx) return czero();
        if (!D) return in0[((int64_t)tile * ey + n) * T + t];  // kx-tile-major X1 (one rank)
        const int p = row_owner(mv, n);  // row n arrived from rank p
        return mv.R1[p][beta][blockIdx.z * mv.colA + ((int64_t)j * mv.nr[p][beta] + (n - mv.ya[p])) * nkx + kx];
    };
    // element (q, kx tile, side, plane, kx % T3): the side and q strides are CTA constants and the
    // kx / plane part is fixed per butterfly, so a store costs one 64-bit multiply-add
    const int64_t x2ss = (int64_t)mv.x2nz[beta] << mv.lgT3, x2sq = 2 * nt3 * x2ss;
    double2* const outj = out + ((int64_t)(mv.x2zo[beta] + j) << mv.lgT3);
    auto stN = [&](int t, int p, double2 v) {
        const int kx = tile * T + t;
        if (kx >= nkx) return;
        const int k = Plan<L>::freq(p);
        if (ph) v = cmul(v, half_phase(mv.tw, ktil(k, L), L, -1));
        const int side = k > L / 2, qq = side ? L - k : k;
        double2* o = outj + ((kx >> mv.lgT3) * 2 * x2ss + (kx & (mv.T3 - 1))) + qq * x2sq + (side ? x2ss : 0);
        o[0] = v;
        if (mv.zdirect && j == nzb - 1) {  // zero the padding planes up to the next source's
            const int pad = (beta < 2 ? mv.x2zo[beta + 1] : mv.x2nz[beta]) - mv.x2zo[beta] - nzb;
            for (int e = 1; e <= pad; ++e) o[e << mv.lgT3] = czero();
        }
    };
    // one rank (BULK): the tile's rows are one contiguous block of X1 ([row][t], P2's tile layout),
    // fetched with a single bulk copy into the FFT buffer; stage 0 reads it from there (all loads,
    // a barrier, then the stores: fft_stage0_aliased), so no global load waits in registers
    constexpr bool BULK = !D && Plan<L>::NS >= 2 && T * (L / Plan<L>::radix(0)) == FY<L>::NT;
    if constexpr (BULK) {
        __shared__ uint64_t p2bar;
        const unsigned bytes = (unsigned)(16 * T * ey);
        if (threadIdx.x == 0) {
            mbar_init(&p2bar, 1);
            fence_mbar_init();
            mbar_arrive_expect_tx(&p2bar, bytes);
            bulk_g2s(sm, in0 + (int64_t)tile * ey * T, bytes, &p2bar);
            // the block that takes this CTA's slot next (launch order, kP2Ahead blocks on) finds
            // its input in L2: X1 is read once, so the prefetch adds no traffic
            const int bn = blockIdx.x + kP2Ahead;
            const int jn = jfast ? bn % nzb : bn / ntile, tn = jfast ? bn / nzb : bn % ntile;
            if (jn < nzb && tn < ntile)
                bulk_prefetch_l2(mv.R1[0][beta] + blockIdx.z * mv.colA + ((int64_t)jn * ntile + tn) * ey * T, bytes);
        }
        __syncthreads();  // (the barrier is initialised before anyone waits on it)
        mbar_wait(&p2bar, 0);
        const double2* __restrict__ inb = sm;
        auto lds0 = [&](int t, int n) -> double2 {
            const int kx = tile * T + t;
            return (n < ey && kx < nkx) ? inb[n * T + t] : czero();
        };
        fft_stage0_aliased<L, T, FY<L>::NT, false, true, true>(sm, lds0, mv.tw);
        fft_run_from1<L, T, FY<L>::NT, false, true, true>(sm, stN, mv.tw);
    } else {
        fft_run<L, T, FY<L>::NT, false, true, 0, true>(sm, ld0, stN, mv.tw);
    }
}

// ---------------------------------------------------------------------------------------
// P4, staged: persistent CTAs walk tiles (plane, T adjacent kx); each tile's input pencils are
// prefetched with cp.async (16 B per copy, zero-filled outside the data) into the other half of
// a two-stage shared-memory ring while the CTA transforms the current tile in place, so global
// loads stay in flight through the FFT stages (the unstaged kernel waits on them): C4 P4 0.266
// -> 0.198 ms.  (The same staging of P2, whose input is half zero padding, measured slower than
// the unstaged P2, which skips the padding loads altogether, and a staged P5 was slower than the
// unstaged one (its gather epilogue dominates): both stay unstaged.)
// ---------------------------------------------------------------------------------------
template <int L, int KB = 32> struct FYS {  // KB: shared memory per stage
    static constexpr int T = clampi(KB * 64 / L, 1, 32);
    static constexpr int NT = clampi(T * L / 16, 64, 256);
};

template <int L, int KB, bool D>
__global__ void __launch_bounds__(FYS<L, KB>::NT) k_p4s(MV mv) {
    constexpr int T = FYS<L, KB>::T, NT = FYS<L, KB>::NT;
    extern __shared__ __align__(16) double2 sm[];  // [2][L][T]
    const int nkx = mv.nkx;
    const int ntx = (nkx + T - 1) / T;
    int G = 0;
    for (int f = mv.f0; f < mv.f1; ++f) G += mv.nzout[f];  // fields [f0, f1)
    const int nt1 = G * ntx;  // tiles per column
    const int ntiles = nt1 * mv.nb;
    auto decode = [&](int tl, int& f, int& j, int& xt) {
        tl %= nt1;
        xt = tl % ntx;
        int g = tl / ntx;
        f = mv.f0;
        while (g >= mv.nzout[f]) g -= mv.nzout[f++];
        j = g;
    };
    // BULK: the tile's block arrives by one cp.async.bulk (mbarrier per stage) in its plain
    // [ky][t] layout, and stage 0 reads it from there (fft_stage0_aliased), instead of L T / NT
    // swizzled 16-byte cp.async copies per thread
    constexpr bool BULK = Plan<L>::NS >= 2 && T * (L / Plan<L>::radix(0)) == NT;
    __shared__ uint64_t p4bar[2];
    if (BULK) {
        if (threadIdx.x == 0) {
            mbar_init(&p4bar[0], 1);
            mbar_init(&p4bar[1], 1);
            fence_mbar_init();
        }
        __syncthreads();
    }
    auto prefetch = [&](int tl, int stg) {
        if (BULK && threadIdx.x != 0) return;  // (one thread issues the bulk copy: only it decodes)
        int f, j, xt;
        decode(tl, f, j, xt);
        // kx-tile-major X3: the tile's T kx x L ky are one contiguous block
        const double2* in = mv.X3[f] + (tl / nt1) * mv.colC + ((int64_t)j * ntx + xt) * L * T;
        double2* dst = sm + stg * L * T;
        if constexpr (BULK) {
            mbar_arrive_expect_tx(&p4bar[stg], (unsigned)(16 * L * T));
            bulk_g2s(dst, in, (unsigned)(16 * L * T), &p4bar[stg]);
            return;
        }
        for (int e = threadIdx.x; e < L * T; e += NT) {
            const int n = e / T, t = e % T;
            const bool valid = xt * T + t < nkx;
            cp_async16(dst + smi<L, T, true, true>(t, n), valid ? in + e : in, valid);
        }
        cp_async_commit();
    };
    if ((int)blockIdx.x < ntiles) prefetch(blockIdx.x, 0);
    int it = 0;
    for (int tl = blockIdx.x; tl < ntiles; tl += gridDim.x, ++it) {
        const int stg = it & 1;
        if (tl + (int)gridDim.x < ntiles) prefetch(tl + gridDim.x, stg ^ 1);
        else if (!BULK) cp_async_commit();
        if constexpr (BULK) {
            mbar_wait(&p4bar[stg], (it >> 1) & 1);
        } else {
            cp_async_wait<1>();
            __syncthreads();
        }
        int f, j, xt;
        decode(tl, f, j, xt);
        const int eyo = mv.ext_out[f][1];
        const bool ph = mv.faxis[f] != 1;
        double2* buf = sm + stg * L * T;
        auto lds = [&](int t, int n) {
            double2 v = buf[smi<L, T, true, true>(t, n)];
            if (ph) v = cmul(v, half_phase(mv.tw, ktil(n, L), L, +1));
            return v;
        };
        // one rank: X4 row-pair blocked [plane][row pair][2][kx] (P5's pairs at absolute rows
        // (2m, 2m + 1)): row yy sits at row yy + s5 of the plane's 2 np rows. A tile one kx wide
        // (T = 1, M_y >= 2048: C5) would write 16-byte half sectors there, so it keeps the
        // row-pair interleaved [plane][row pair][kx][2] (a pair's two rows fill one sector)
        constexpr bool IL = T == 1;
        const int s5 = mv.lo[1] & 1;
        double2* const o4 =
            D ? nullptr
              : mv.S2[0][f] + (tl / nt1) * mv.colA + ((int64_t)j * (((mv.nr[0][3 + f] + s5 + 1) >> 1) * 2) + s5) * nkx;
        auto stN = [&](int t, int p, double2 v) {
            const int kx = xt * T + t;
            const int yy = Plan<L>::freq(p);
            if (kx < nkx && yy < eyo) {
                if (D) {
                    const int pr = row_owner(mv, yy);  // row yy goes to rank pr for P5
                    const int y0 = mv.ya[pr];
                    mv.S2[pr][f][(tl / nt1) * (pr == mv.rank ? mv.colA : mv.colS) +
                                 ((int64_t)j * mv.nr[pr][3 + f] + (yy - y0)) * nkx + kx] = v;
                } else if (IL) {
                    o4[(((int64_t)((yy + s5) >> 1) * nkx + kx) << 1 | ((yy + s5) & 1)) - (int64_t)s5 * nkx] = v;
                } else {
                    o4[(int64_t)yy * nkx + kx] = v;
                }
            }
        };
        if constexpr (BULK) {
            auto lds0 = [&](int t, int n) {
                double2 v = (xt * T + t < nkx) ? buf[n * T + t] : czero();  // plain [ky][t]
                if (ph) v = cmul(v, half_phase(mv.tw, ktil(n, L), L, +1));
                return v;
            };
            fft_stage0_aliased<L, T, NT, true, true, true>(buf, lds0, mv.tw);
            fft_run_from1<L, T, NT, true, true, true>(buf, stN, mv.tw);
            fence_proxy_async();  // this stage is refilled by the async proxy next
        } else {
            fft_run<L, T, NT, true, true, 0, true>(buf, lds, stN, mv.tw);
        }
        __syncthreads();
    }
    if (!BULK) cp_async_wait<0>();
}

// ---------------------------------------------------------------------------------------
// P3: forward z FFT of the three source fields, orientation-block MAC (Eqs. 10-12), inverse z
//   One tile = T adjacent kx x the ky pair {q, My - q} (the two share every folded spectrum
//   row, so each R element is read from HBM once).  Persistent, TMA-fed: each CTA walks tiles
//   with stride gridDim.x.  A tile's inputs are contiguous by construction -- P2 writes X2
//   tile-major ([q][tile][side][plane][t] per source) and the build stores R tile-major
//   ([q][tile][block][kz'][t]) -- so one elected thread fetches the next tile with four
//   cp.async.bulk copies (three sources + R) into the other half of a two-stage shared-memory
//   ring while the CTA transforms the current one.  One buffer [L][W] holds the 6T forward
//   pencils, then (after the MAC has pulled its inputs into registers) the NF*2T output
//   pencils, which are inverse-transformed together.
//   Phase algebra (App. B): out^a = phi_a sum_b R^{ab} phibar_b Q^b.  Along z, c_x = c_y = 1/2
//   and c_z = 0, so phi_a,z phibar_b,z is 1 for a, b both in {x, y} or both z, phi_z-bar for
//   (a = z, b in {x, y}) and phi_z for (a in {x, y}, b = z): one complex multiply per source
//   (Q^z) and one per z-field, instead of one per (field, source).  The parity sign of the
//   odd E blocks and the factor i are common to all sources of a field and applied once.
//   (A warp-register variant -- one lane group per pencil, four-step FFT in registers -- was
//   measured at 1.7x this kernel's time on C4: ~230 registers/thread capped residency at one
//   CTA per SM.)
// ---------------------------------------------------------------------------------------
template <int L, int NF>
struct P3T {
    static constexpr int T = clampi(256 / L, 1, 16) * (NF <= 3 ? 2 : 1);
    static constexpr int W = (NF <= 3 ? 6 : 2 * NF) * T;  // buffer width (pencils)
};
// host mirror of P3T<L, NF>::T (the tile width also fixes the X2 / R tiled layouts)
inline int p3_tile(int Mz, int nf) { return clampi(256 / Mz, 1, 16) * (nf <= 3 ? 2 : 1); }

// NS: stages of the TMA ring.  NS = 2 prefetches the next tile while the current one is
// transformed (one CTA per SM: the stages fill shared memory); NS = 1 refills the single stage
// as soon as the MAC has read it (overlapping the inverse z-FFT and the stores), small enough
// for two CTAs per SM that overlap each other.
template <int L, int NF, int NS = 2>
__global__ void __launch_bounds__(kNT3) k_p3(MV mv) {
    constexpr int T = P3T<L, NF>::T;
    constexpr int W = P3T<L, NF>::W;
    constexpr int T2 = 2 * T;
    constexpr int KZ = L / 2 + 1;
    constexpr int NI = (L * T2 + kNT3 - 1) / kNT3;  // MAC items per thread
    extern __shared__ __align__(16) double2 sm[];
    const int Kx = mv.nkx, My = mv.My;  // own kx slab
    const int nz0 = mv.nzin[0], nz1 = mv.nzin[1], nz2 = mv.nzin[2];
    const int XS = T2 * (nz0 + nz1 + nz2);          // double2 per stage
    const int RC = mv.rchunk;                       // doubles per stage (even)
    double2* buf = sm;                              // [L][W] transform buffer
    double2* ph = buf + L * W;                      // [L] exp(-i pi kt / L)
    double2* xin = ph + L;                          // [NS][XS] staged X2 tiles
    double* rin = reinterpret_cast<double*>(xin + NS * XS);  // [NS][RC] staged R tiles
    // [9][ZS] plane -> index / -1; rows padded to L + 2 so that the three sources' (fields') rows
    // start in different banks (lanes of one warp read several rows at the same z)
    constexpr int ZS = L + 2;
    int16_t* zmap = reinterpret_cast<int16_t*>(rin + NS * RC);
    uint64_t* bar = reinterpret_cast<uint64_t*>(zmap + ((9 * ZS + 3) & ~3));  // [2]
    __shared__ int fmeta[NF][4];                    // kind | alpha << 1, R offsets of b0..b2
    const int xo1 = T2 * nz0, xo2 = T2 * (nz0 + nz1);
    const int ntile = (Kx + T - 1) / T;
    const int ntiles = ntile * (My / 2 + 1);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    if (threadIdx.x < NF) {
        const int f = threadIdx.x;
        fmeta[f][0] = mv.fkind[f] | (mv.faxis[f] << 1);
        for (int b = 0; b < 3; ++b) fmeta[f][1 + b] = mv.blk[f][b] < 0 ? -1 : mv.blk[f][b] * KZ * T;
    }
    for (int k = threadIdx.x; k < L; k += kNT3) ph[k] = half_phase(mv.tw, ktil(k, L), L, -1);
    for (int e = threadIdx.x; e < 9 * L; e += kNT3) {
        const int g = e / L, z = e % L;
        zmap[g * ZS + z] = (int16_t)(z < mv.ZL ? mv.planes[(9 + g) * mv.ZL + z] : -1);
    }
    __syncthreads();
    // tile order: kx tiles fastest, or (X3 one kx wide, lgt4 = 0: C5) |ky| fastest, so that the
    // CTAs writing adjacent ky of one X3 sector run together and L2 merges the halves
    const int nq = My / 2 + 1;
    const bool qfast = mv.lgt4 == 0;
    auto qt_of = [&](int tl) { return qfast ? (tl % nq) * ntile + tl / nq : tl; };  // X2 / R block
    auto issue = [&](int tl, int s) {  // one thread: fetch tile tl (block q * ntile + tile) into stage s
        const size_t qt = (size_t)qt_of(tl);
        mbar_arrive_expect_tx(&bar[s], (unsigned)(16 * XS + 8 * RC));
        if (nz0) bulk_g2s(xin + s * XS, mv.X2[0] + qt * T2 * nz0, 16u * T2 * nz0, &bar[s]);
        if (nz1) bulk_g2s(xin + s * XS + xo1, mv.X2[1] + qt * T2 * nz1, 16u * T2 * nz1, &bar[s]);
        if (nz2) bulk_g2s(xin + s * XS + xo2, mv.X2[2] + qt * T2 * nz2, 16u * T2 * nz2, &bar[s]);
        bulk_g2s(rin + s * RC, mv.Rt + qt * RC, 8u * RC, &bar[s]);
    };
    if (threadIdx.x == 0 && (int)blockIdx.x < ntiles) issue(blockIdx.x, 0);
    unsigned par0 = 0, par1 = 0;
    int it = 0;
    for (int tl = blockIdx.x; tl < ntiles; tl += gridDim.x, ++it) {
        const int s = NS == 1 ? 0 : (it & 1);
        if (NS == 2 && threadIdx.x == 0 && tl + (int)gridDim.x < ntiles) {
            fence_proxy_async();
            issue(tl + gridDim.x, s ^ 1);
        }
        if (s == 0) { mbar_wait(&bar[0], par0); par0 ^= 1; }
        else { mbar_wait(&bar[1], par1); par1 ^= 1; }
        const double2* xs = xin + s * XS;
        const double* rs = rin + s * RC;
        const int qt = qt_of(tl);
        const int q = qt / ntile, tile = qt % ntile;
        const int nside = (q == 0 || 2 * q == My) ? 1 : 2;
        // forward z-FFT of pencils pp = beta * 2T + side * T + t (zero-padded to L)
        auto ld0 = [&](int pp, int n) -> double2 {
            const int t = pp % T, side = (pp / T) & 1, beta = pp / T2;
            const int jz = zmap[beta * ZS + n];
            if (side >= nside || tile * T + t >= Kx || jz < 0) return czero();
            const int nzb = beta == 0 ? nz0 : (beta == 1 ? nz1 : nz2);
            const int xo = beta == 0 ? 0 : (beta == 1 ? xo1 : xo2);
            return xs[xo + (side * nzb + jz) * T + t];
        };
        auto sti = [&](int pp, int p, double2 v) { buf[p * W + pp] = v; };
        fft_run<L, W, kNT3, false, true>(buf, ld0, sti, mv.tw, 3 * T2);
        __syncthreads();
        // MAC: item u = k * 2T + c (c = side * T + t); inputs to registers, outputs in place
        double2 qv[NI][3];
#pragma unroll
        for (int ii = 0; ii < NI; ++ii) {
            const int u = threadIdx.x + ii * kNT3;
            if (u < L * T2) {
                const int k = u / T2, c = u % T2;
                const double2* row = buf + Plan<L>::pos(k) * W + c;
                qv[ii][0] = row[0];
                qv[ii][1] = row[T2];
                qv[ii][2] = row[2 * T2];
            }
        }
        __syncthreads();
#pragma unroll
        for (int ii = 0; ii < NI; ++ii) {
            const int u = threadIdx.x + ii * kNT3;
            if (u >= L * T2) break;
            const int k = u / T2, c = u % T2;
            const int side = c / T, t = c % T;
            const int kt = ktil(k, L);
            const int kzp = kt < 0 ? -kt : kt;
            const double2 phb = ph[k];                 // phibar_z = exp(-i pi kt / L)
            const double2 qx = qv[ii][0], qy = qv[ii][1];
            const double2 qz = cmulc(qv[ii][2], phb);  // phi_z Q^z
            const double* rrow = rs + kzp * T + t;
            double2* orow = buf + k * W + c;
            const bool live = side < nside;
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                const int km = fmeta[f][0], o0 = fmeta[f][1], o1 = fmeta[f][2], o2 = fmeta[f][3];
                const int kind = km & 1, alpha = km >> 1;
                // out = phibar_z^[a = z] * (R^{a x} Qx + R^{a y} Qy + R^{a z} phi_z Qz)
                double2 a = czero();
                if (o0 >= 0) {
                    const double r = rrow[o0];
                    a.x = fma(r, qx.x, a.x);
                    a.y = fma(r, qx.y, a.y);
                }
                if (o1 >= 0) {
                    const double r = rrow[o1];
                    a.x = fma(r, qy.x, a.x);
                    a.y = fma(r, qy.y, a.y);
                }
                if (o2 >= 0) {
                    const double r = rrow[o2];
                    a.x = fma(r, qz.x, a.x);
                    a.y = fma(r, qz.y, a.y);
                }
                if (alpha == 2) a = cmul(a, phb);
                if (kind == 1) {
                    // E blocks: R stores Im(K), odd along alpha; sign from the octant fold
                    const bool neg = (alpha == 1 && side == 1) || (alpha == 2 && kt < 0);
                    a = neg ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
                }
                orow[f * T2] = live ? a : czero();
            }
        }
        __syncthreads();
        if (NS == 1 && threadIdx.x == 0 && tl + (int)gridDim.x < ntiles) {
            // the stage is consumed (forward FFT and MAC done): refill it during the inverse
            fence_proxy_async();
            issue(tl + gridDim.x, 0);
        }
        auto ldo = [&](int pp, int n) { return buf[n * W + pp]; };
        auto sto = [&](int pp, int p, double2 v) {
            const int f = pp / T2, c = pp % T2;
            const int side = c / T, t = c % T;
            const int kx = tile * T + t;
            const int jz = zmap[(3 + f) * ZS + Plan<L>::freq(p)];
            if (side < nside && kx < Kx && jz >= 0)
                mv.X3[f][((((int64_t)jz * ((Kx + (1 << mv.lgt4) - 1) >> mv.lgt4) + (kx >> mv.lgt4)) * My +
                           (side ? My - q : q)) << mv.lgt4) | (kx & ((1 << mv.lgt4) - 1))] = v;
        };
        fft_run<L, W, kNT3, true, true>(buf, ldo, sto, mv.tw, NF * T2);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------
// P5: times phi_f,x, C2R along x (two lines per complex FFT), gather + dielectric terms
// ---------------------------------------------------------------------------------------
// bytes of P5's staged input block (T row pairs x nk kx x 2 rows, complex), 128-byte rounded
__host__ __device__ constexpr size_t p5_inbytes(int L, int T, int nk) {
    return ((size_t)32 * T * nk > (size_t)16 * L * T ? ((size_t)32 * T * nk + 127) & ~(size_t)127 : (size_t)16 * L * T);
}
// P5's stage-0 input at line position n from the two rows' spectra A, B at kx = k (k = n, or
// L - n with the conjugates: the rows are real): Z = A' + i B' with A' = A phi (phi the half
// phase, ph) and Im A' dropped at the self-conjugate k.  Both rows share phi, so off those two k
// Z = (A + i B) phi, or (conj A + i conj B) conj phi: one complex product instead of two.
template <int L>
__device__ __forceinline__ double2 p5_combine(double2 A, double2 B, int k, bool lo, bool ph,
                                              const double2* __restrict__ tw) {
    if (k == 0 || 2 * k == L) {
        if (ph) {
            const double2 w = half_phase(tw, k, L, +1);
            A = cmul(A, w);
            B = cmul(B, w);
        }
        return make_double2(A.x, B.x);
    }
    if (!lo) {
        A.y = -A.y;
        B.y = -B.y;
    }
    double2 Z = make_double2(A.x - B.y, A.y + B.x);
    if (ph) {
        double2 w = half_phase(tw, k, L, +1);
        if (!lo) w.y = -w.y;
        Z = cmul(Z, w);
    }
    return Z;
}
template <int L, bool D, bool IL = false>  // IL: X4 row-pair interleaved (one rank, lgt4 = 0)
__global__ void __launch_bounds__(FX<L>::NT, FX<L>::MINB5) k_p5(MV mv) {
    constexpr int T = TX<L>::T;
    extern __shared__ double2 sm[];
    const int f = blockIdx.y + mv.f0;
    if (f >= mv.nf) return;
    const int kind = mv.fkind[f], alpha = mv.faxis[f];
    const int exo = mv.ext_out[f][0];
    const int nrow = mv.nr[mv.rank][3 + f];  // own rows of this field
    const int s = (mv.lo[1] + mv.ya[mv.rank]) & 1;  // absolute row pairing, as in P1
    const int nyp = (nrow + s + 1) >> 1;
    const int nch = (nyp + T - 1) / T;
    if (nch == 0) return;
    const int j = blockIdx.x / nch, ch = blockIdx.x % nch;
    if (j >= mv.nzout[f]) return;
    const int z = zlist(mv, 3 + f, j);
    const bool ph = alpha != 0;
    constexpr bool x4il = !D && IL;  // P4's tile one kx wide: X4 row-pair interleaved
    auto At = [&](int yrow, int k, bool v) -> double2 {
        int qd = 0, nk = mv.nkx, k0 = 0;
        if (D) {
            qd = kx_owner(mv, k);  // column k arrived from rank qd
            k0 = mv.kxa[qd];
            nk = mv.kxa[qd + 1] - k0;
        }
        const int rr = yrow + s;  // one rank: row-pair blocked (interleaved: x4il) X4 (see P4)
        const double2* src =
            D ? mv.R2[qd][f] + blockIdx.z * mv.colA + ((int64_t)j * nrow + yrow) * nk + (k - k0)
              : mv.R2[0][f] + blockIdx.z * mv.colA +
                    (x4il ? (((int64_t)j * nyp + (rr >> 1)) * nk + k) << 1 | (rr & 1)
                          : ((int64_t)j * nyp * 2 + rr) * nk + k);
        return v ? __ldg(src) : czero();
    };
    auto ld0 = [&](int t, int n) -> double2 {
        const int q = ch * T + t;
        const int l0 = 2 * q - s;
        const bool ok = q < nyp;
        const bool has0 = ok && l0 >= 0, has1 = ok && l0 + 1 < nrow;
        const bool lo = 2 * n <= L;
        const int k = lo ? n : L - n;
        const double2 A = At(has0 ? l0 : 0, k, has0), B = At(has1 ? l0 + 1 : 0, k, has1);
        return p5_combine<L>(A, B, k, lo, ph, mv.tw);
    };
    // the last stage goes to shared memory; the gather then walks each output line with
    // consecutive lanes on consecutive slots (coalesced slot-map reads and y writes; the panel
    // kind and the dielectric sign come folded into the slot-map entry, common.cuh kSlot*).
    // The 2T slot-map lines are fetched with cp.async before the FFT, so the gather does not
    // wait on them.
    const int32_t* __restrict__ smap = mv.slotmap[alpha];
    const int Gx = mv.G[alpha][0], Gy = mv.G[alpha][1];
    const int64_t zrow =
        ((int64_t)(z + mv.lo[2]) * Gy + mv.lo[1] + mv.ya[mv.rank]) * Gx + mv.lo[0];
    // one rank (BULK): the CTA's T row pairs of X4 are one contiguous block ([pair][2][kx], P4's
    // row-pair blocked layout: consecutive kx of a row are adjacent, so stage 0's reads are
    // conflict-free), fetched with a single bulk copy into the FFT buffer itself;
    // stage 0 reads it from there (fft_stage0_aliased: all loads, a barrier, then the stores), so
    // no global load sits in a thread's registers while the transform waits on it
    constexpr bool BULK = !D && Plan<L>::NS >= 2 && T * (L / Plan<L>::radix(0)) == FX<L>::NT;
    const int nk1 = mv.nkx;
    int32_t* const ss = reinterpret_cast<int32_t*>(
        reinterpret_cast<uint8_t*>(sm) + (BULK ? p5_inbytes(L, T, nk1) : sizeof(double2) * L * T));  // [2T][L]
    __shared__ uint64_t p5bar;
    if (BULK) {
        const int nqc = min(T, nyp - ch * T);
        const unsigned bytes = (unsigned)(32 * nk1 * nqc);
        if (threadIdx.x == 0) {
            mbar_init(&p5bar, 1);
            fence_mbar_init();
            mbar_arrive_expect_tx(&p5bar, bytes);
            bulk_g2s(sm, mv.R2[0][f] + blockIdx.z * mv.colA + (((int64_t)j * nyp + ch * T) * nk1 << 1), bytes,
                     &p5bar);
        }
        __syncthreads();  // (the barrier is initialised before anyone waits on it)
    }
    for (int r = 0; r < 2 * T; ++r) {
        const int q = ch * T + (r >> 1), l = 2 * q - s + (r & 1);
        if (q >= nyp || l < 0 || l >= nrow) continue;
        const int32_t* srow = smap + zrow + (int64_t)l * Gx;
        for (int n = threadIdx.x; n < exo; n += FX<L>::NT) cp_async4(ss + r * L + n, srow + n);
    }
    cp_async_commit();
    auto sts = [&](int t, int p, double2 v) { sm[smi<L, T, false>(t, p)] = v; };
    if constexpr (BULK) {
        // the same values as ld0 / At, read from the staged block [pair t][row][kx]
        const double2* __restrict__ inb = sm;
        auto As = [&](int t, int row, int k, bool v) -> double2 {
            return v ? inb[x4il ? (t * nk1 + k) * 2 + row : (t * 2 + row) * nk1 + k] : czero();
        };
        auto lds0 = [&](int t, int n) -> double2 {
            const int q = ch * T + t;
            const int l0 = 2 * q - s;
            const bool ok = q < nyp;
            const bool has0 = ok && l0 >= 0, has1 = ok && l0 + 1 < nrow;
            const bool lo = 2 * n <= L;
            const int k = lo ? n : L - n;
            const double2 A = As(t, 0, k, has0), B = As(t, 1, k, has1);
            return p5_combine<L>(A, B, k, lo, ph, mv.tw);
        };
        mbar_wait(&p5bar, 0);
        fft_stage0_aliased<L, T, FX<L>::NT, true>(sm, lds0, mv.tw);
        fft_run_from1<L, T, FX<L>::NT, true>(sm, sts, mv.tw);
    } else {
        fft_run<L, T, FX<L>::NT, true, false>(sm, ld0, sts, mv.tw);
    }
    cp_async_wait<0>();
    __syncthreads();
    const int32_t want = kind ? kSlotDiel : 0;
    double* __restrict__ y = mv.ys[blockIdx.z];
    constexpr int NI = (L + FX<L>::NT - 1) / FX<L>::NT;  // slots per thread and line (exo <= L)
#pragma unroll 1
    for (int r = 0; r < 2 * T; ++r) {
        const int t = r >> 1, half = r & 1;
        const int q = ch * T + t;
        const int l = 2 * q - s + half;
        if (q >= nyp || l < 0 || l >= nrow) continue;
        int32_t e[NI];
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const int n = threadIdx.x + i * FX<L>::NT;
            e[i] = n < exo ? ss[r * L + n] : -1;
        }
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const int n = threadIdx.x + i * FX<L>::NT;
            if (e[i] < 0 || (e[i] & kSlotDiel) != want) continue;
            const double2 v = sm[smi<L, T, false>(t, Plan<L>::pos(n))];
            const double val = half ? v.y : v.x;
            const int p = e[i] & kSlotIdx;
            // dielectric rows: y was initialised to Ī x by k_yinit (Eq. 7); the field term is
            // added without reading anything back (each panel appears in exactly one slot map,
            // so the reduction has no contention and the thread never waits on it)
            if (kind == 0) y[p] = val;
            else atomicAdd(y + p, (e[i] & kSlotNeg) ? -val : val);
        }
    }
}

// ---------------------------------------------------------------------------------------
// setup kernels: kernel-entry grid (a2), in-place 3-D C2C FFT, spectrum extraction (a3)
// ---------------------------------------------------------------------------------------
__global__ void k_twiddles(double2* tw) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= kTabN) return;
    double s, c;
    sincospi(-2.0 * n / (double)kTabN, &s, &c);
    tw[n] = make_double2(c, s);
}

// Cyclic index n on an M-grid -> signed geometric offset t (doubled, 2t) of the representative
// slot difference minimising |delta + s|, s2 = 2 s in {-1, 0, 1}.  The tie of
// s = 0 at n = M/2 is taken as +M/2 (odd kernels are zeroed there by the caller).
__device__ __forceinline__ int rep_t2(int n, int M, int s2) {
    int d;
    if (s2 > 0) d = n < M / 2 ? n : n - M;
    else if (s2 < 0) d = n <= M / 2 ? n : n - M;
    else d = n <= M / 2 ? n : n - M;
    return 2 * d + s2;
}

// a2 on the parity octant: Ko[iz][iy][ix] = kappa at the non-negative geometric offset
// |t| = i (s = 0) or i + 1/2 (s = +-1/2) per axis.  P blocks are even in every component of t,
// E^{a.} blocks odd along a and even otherwise (Table VIII), so the
// full cyclic grid follows from this octant with signs.
__device__ __forceinline__ int oct_D(int i, int alpha, int beta, int a) {
    const int s2 = c2(alpha, a) - c2(beta, a);
    // |t| = i (s2 = 0) or i + 1/2; slot offset D = t - s
    return s2 == 0 ? i : (s2 > 0 ? i : i + 1);
}
// symxy (zz blocks, Ox == Oy): z-normal pairs are symmetric under x <-> y, so only ix <= iy is
// evaluated and written to both (ix, iy) and (iy, ix)
__global__ void k_kgen_oct(double* Ko, int Ox, int Oy, int Oz, int kind, int alpha, int beta,
                           double scale, int symxy) {
    const int64_t tot = (int64_t)Ox * Oy * Oz;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int i[3] = {(int)(idx % Ox), (int)((idx / Ox) % Oy), (int)(idx / ((int64_t)Ox * Oy))};
        if (symxy && i[0] > i[1]) continue;
        const double v = scale * kappa(kind, alpha, beta, oct_D(i[0], alpha, beta, 0),
                                       oct_D(i[1], alpha, beta, 1), oct_D(i[2], alpha, beta, 2));
        Ko[idx] = v;
        if (symxy && i[0] != i[1]) Ko[((int64_t)i[2] * Oy + i[0]) * Ox + i[1]] = v;
    }
}

// preconditioner near-field table: the near corner |t| < T of a P block's octant, evaluated
// directly (the same kernel for generated and mirrored blocks, so both builds agree bitwise)
// All P pairs in one launch (blockIdx.y = pair; the near-field closed forms are long-latency,
// six small launches in sequence cost 6x one).
struct CornerPairs {
    int n, alpha[6], beta[6], slot[6];
};
__global__ void k_kgen_corner(double* __restrict__ Tb0, int Tx, int Ty, int Tz, int Ox, int Oy,
                              int Oz, CornerPairs cp, double scale) {
    const int n = Tx * Ty * Tz;
    const int alpha = cp.alpha[blockIdx.y], beta = cp.beta[blockIdx.y];
    double* __restrict__ Tb = Tb0 + (size_t)cp.slot[blockIdx.y] * n;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
        const int ix = e % Tx, iy = (e / Tx) % Ty, iz = e / (Tx * Ty);
        Tb[e] = (ix < Ox && iy < Oy && iz < Oz)
                    ? scale * kappa(0, alpha, beta, oct_D(ix, alpha, beta, 0), oct_D(iy, alpha, beta, 1),
                                    oct_D(iz, alpha, beta, 2))
                    : 0.0;
    }
}

// x <-> y mirror blocks (square x/y window, one rank): swapping the x and y axes maps the
// (a, b) panel pair to (s(a), s(b)), s = (x y), and the kernel at offset (Dx, Dy, Dz) to the
// kernel at (Dy, Dx, Dz) -- e.g. P^{yy}(Dx, Dy, Dz) = P^{xx}(Dy, Dx, Dz), E^{zy} likewise from
// E^{zx} -- so the folded, phase-stripped spectrum of the mirror block is the kx <-> ky
// transpose of the original's (the strip phases and the parity octants swap with the axes):
//   R_dst(kx, ky, w) = R_src(ky, kx, w), w = kz' (z-FFT mode) or u (direct-z mode)
// Index of R(kx, |ky|, block, w) in the tile-major table: z-FFT mode [block][kz'][t] per tile;
// direct-z mode (RS1 > 0) [t][block * NW + u] with RS1 doubles per kx (k_p3m reads one kx's
// rows contiguously; the last row of each kx is the zero row)
__host__ __device__ __forceinline__ int64_t rt_idx(int ky, int kx, int blk, int NW, int w, int lgT3,
                                                   int nt3, int RC, int RS1) {
    const int64_t base = ((int64_t)ky * nt3 + (kx >> lgT3)) * RC;
    const int t = kx & ((1 << lgT3) - 1);
    return RS1 ? base + (int64_t)t * RS1 + (int64_t)blk * NW + w
               : base + ((int64_t)blk * NW + w) * (1 << lgT3) + t;
}

__global__ void k_rt_mirror(double* R, int K, int NW, int src, int dst, int lgT3, int RC, int RS1) {
    const int T3 = 1 << lgT3, nt3 = (K + T3 - 1) >> lgT3;
    const int64_t tot = (int64_t)K * K * NW;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int kx = (int)(idx % K);
        const int w = (int)((idx / K) % NW);
        const int ky = (int)(idx / ((int64_t)K * NW));
        R[rt_idx(ky, kx, dst, NW, w, lgT3, nt3, RC, RS1)] = R[rt_idx(kx, ky, src, NW, w, lgT3, nt3, RC, RS1)];
    }
}

// full cyclic grid (real part of G) from the octant table, with the parity signs
__global__ void k_kfill(double2* G, const double* __restrict__ Ko, int Mx, int My, int Mz, int Ox,
                        int Oy, int kind, int alpha, int beta) {
    const int64_t tot = (int64_t)Mx * My * Mz;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int n[3] = {(int)(idx % Mx), (int)((idx / Mx) % My), (int)(idx / ((int64_t)Mx * My))};
        const int M[3] = {Mx, My, Mz};
        int o[3];
        double sg = 1.0;
        bool zero = false;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int s2 = c2(alpha, a) - c2(beta, a);
            const int t2 = rep_t2(n[a], M[a], s2);
            const int at2 = t2 < 0 ? -t2 : t2;
            o[a] = s2 == 0 ? at2 / 2 : (at2 - 1) / 2;
            if (kind == 1 && a == alpha) {
                if (t2 < 0) sg = -sg;
                if (s2 == 0 && 2 * n[a] == M[a]) zero = true;  // unresolvable odd tie
            }
        }
        const double v = zero ? 0.0 : sg * Ko[((int64_t)o[2] * Oy + o[1]) * Ox + o[0]];
        G[idx] = make_double2(v, 0.0);
    }
}

// direct-z mode: x/y-cyclic grid G[u][y][x] (real part) from the octant table Ko[u][oy][ox],
// with the x / y parity signs (the z parity is applied in k_p3d)
__global__ void k_kfill2d(double2* G, const double* __restrict__ Ko, int Mx, int My, int ZU,
                          int Ox, int Oy, int kind, int alpha, int beta) {
    const int64_t tot = (int64_t)Mx * My * ZU;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int n[2] = {(int)(idx % Mx), (int)((idx / Mx) % My)};
        const int u = (int)(idx / ((int64_t)Mx * My));
        const int M[2] = {Mx, My};
        int o[2];
        double sg = 1.0;
        bool zero = false;
#pragma unroll
        for (int a = 0; a < 2; ++a) {
            const int s2 = c2(alpha, a) - c2(beta, a);
            const int t2 = rep_t2(n[a], M[a], s2);
            const int at2 = t2 < 0 ? -t2 : t2;
            o[a] = s2 == 0 ? at2 / 2 : (at2 - 1) / 2;
            if (kind == 1 && a == alpha) {
                if (t2 < 0) sg = -sg;
                if (s2 == 0 && 2 * n[a] == M[a]) zero = true;  // unresolvable odd tie
            }
        }
        const double v = zero ? 0.0 : sg * Ko[((int64_t)u * Oy + o[1]) * Ox + o[0]];
        G[idx] = make_double2(v, 0.0);
    }
}

// direct-z mode: x/y-transformed, phase-stripped kernel, tile-major for k_p3d:
//   R[(ky' * nt3 + kx / T3) * RC + (blk * ZU + u) * T3 + kx % T3]; Re (P, E^{z.}) or Im (E^{x.},
//   E^{y.}) part; kx local to [kx0, kx0 + nkx)
__global__ void k_extract2d(const double2* __restrict__ G, double* __restrict__ R, int Mx, int My,
                            int ZU, int kx0, int nkx, int kind, int alpha, int beta,
                            const double2* __restrict__ tw, int blk, int lgT3, int RC, int RS1) {
    const int KY = My / 2 + 1;
    const int T3 = 1 << lgT3;
    const int nt3 = (nkx + T3 - 1) >> lgT3;
    const int64_t tot = (int64_t)nkx * KY * ZU;
    const int s2x = c2(alpha, 0) - c2(beta, 0), s2y = c2(alpha, 1) - c2(beta, 1);
    const bool im = kind == 1 && alpha != 2;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int kx = (int)(idx % nkx);
        const int u = (int)((idx / nkx) % ZU);
        const int ky = (int)(idx / ((int64_t)nkx * ZU));
        double2 v = G[((int64_t)u * My + ky) * Mx + kx0 + kx];
        v = cmul(v, half_phase(tw, (kx0 + kx) * s2x, Mx, -1));
        v = cmul(v, half_phase(tw, ky * s2y, My, -1));
        R[rt_idx(ky, kx, blk, ZU, u, lgT3, nt3, RC, RS1)] = im ? v.y : v.x;
    }
}

// in-place C2C FFT of contiguous lines: data[line][L]
template <int L, bool INV>
__global__ void __launch_bounds__(FX<L>::NT) k_fft_lines(double2* data, int64_t nlines,
                                                   const double2* __restrict__ tw) {
    constexpr int T = TX<L>::T;
    extern __shared__ double2 sm[];
    const int64_t l0 = (int64_t)blockIdx.x * T;
    auto ld0 = [&](int t, int n) -> double2 {
        return l0 + t < nlines ? data[(l0 + t) * L + n] : czero();
    };
    auto stN = [&](int t, int p, double2 v) {
        if (l0 + t < nlines) data[(l0 + t) * L + Plan<L>::freq(p)] = v;
    };
    fft_run<L, T, FX<L>::NT, INV, false>(sm, ld0, stN, tw);
}

// in-place C2C FFT along a strided axis: element n of column c in batch b at
// data[b*bs + n*es + c], columns c in [0, ncols) contiguous.
template <int L>
__global__ void __launch_bounds__(FY<L>::NT) k_fft_strided(double2* data, int64_t es, int64_t ncols,
                                                     int64_t bs, const double2* __restrict__ tw) {
    constexpr int T = TY<L>::T;
    extern __shared__ double2 sm[];
    const int64_t ntile = (ncols + T - 1) / T;
    const int64_t b = blockIdx.x / ntile, c0 = (blockIdx.x % ntile) * T;
    double2* base = data + b * bs + c0;
    auto ld0 = [&](int t, int n) -> double2 {
        return c0 + t < ncols ? base[n * es + t] : czero();
    };
    auto stN = [&](int t, int p, double2 v) {
        if (c0 + t < ncols) base[(int64_t)Plan<L>::freq(p) * es + t] = v;
    };
    fft_run<L, T, FY<L>::NT, false, true, 0, true>(sm, ld0, stN, tw);
}

// Direct-z kernel table in two fused passes (replacing fill -> C2C x -> C2C y -> extract):
// x stage: the cyclic x/y kernel rows are built from the octant table on the fly (the parity
// signs of k_kfill2d), two real rows per complex FFT, split R2C -> Gx[u][y][kx < Mx/2 + 1];
// y stage: C2C along y of this rank's kx columns only, phase-stripped and folded straight into
// the tile-major table (the store of k_extract2d).  Half the x work, a quarter of the y work
// and two fewer passes over the grid.
template <int L>
__global__ void __launch_bounds__(FX<L>::NT) k_kx_r2c(double2* __restrict__ Gx,
                                                    const double* __restrict__ Ko, int My, int ZU,
                                                    int Ox, int Oy, int kind, int alpha, int beta,
                                                    const double2* __restrict__ tw) {
    constexpr int T = TX<L>::T, K = L / 2 + 1, NT = FX<L>::NT;
    extern __shared__ double2 sm[];
    const int npair = My / 2;
    const int64_t npen = (int64_t)ZU * npair;
    const int64_t pair0 = (int64_t)blockIdx.x * T;
    // x part of the octant mapping per column n, once per CTA: o_x | parity sign (bit 30) |
    // unresolvable odd tie (bit 31, value 0)
    int32_t* const xt = reinterpret_cast<int32_t*>(sm + L * T);
    {
        const int s2 = c2(alpha, 0) - c2(beta, 0);
        for (int n = threadIdx.x; n < L; n += NT) {
            const int t2 = rep_t2(n, L, s2);
            const int at2 = t2 < 0 ? -t2 : t2;
            int e = s2 == 0 ? at2 / 2 : (at2 - 1) / 2;
            if (kind == 1 && alpha == 0) {
                if (t2 < 0) e |= 1 << 30;
                if (s2 == 0 && 2 * n == L) e |= (int)(1u << 31);
            }
            xt[n] = e;
        }
        __syncthreads();
    }
    auto val = [&](int nx, int ny, int u) -> double {
        const int s2 = c2(alpha, 1) - c2(beta, 1);
        const int t2 = rep_t2(ny, My, s2);
        const int at2 = t2 < 0 ? -t2 : t2;
        const int oy = s2 == 0 ? at2 / 2 : (at2 - 1) / 2;
        bool neg = false, zero = false;
        if (kind == 1 && alpha == 1) {
            neg = t2 < 0;
            zero = s2 == 0 && 2 * ny == My;  // unresolvable odd tie
        }
        const int e = xt[nx];
        neg ^= (e >> 30) & 1;
        zero |= e < 0;
        const double v = Ko[((int64_t)u * Oy + oy) * Ox + (e & 0x3fffffff)];
        return zero ? 0.0 : (neg ? -v : v);
    };
    auto ld0 = [&](int t, int n) -> double2 {
        const int64_t pp = pair0 + t;
        if (pp >= npen) return czero();
        const int u = (int)(pp / npair), q = (int)(pp % npair);
        return make_double2(val(n, 2 * q, u), val(n, 2 * q + 1, u));
    };
    const SmAcc<L, T, false, false> sts{sm};
    fft_run<L, T, NT, false, false>(sm, ld0, sts, tw);
    __syncthreads();
    for (int e = threadIdx.x; e < T * K; e += NT) {
        const int t = e / K, k = e % K;
        const int64_t pp = pair0 + t;
        if (pp >= npen) continue;
        const int u = (int)(pp / npair), q = (int)(pp % npair);
        const double2 zk = sm[smi<L, T, false>(t, Plan<L>::pos(k))];
        const double2 zm = sm[smi<L, T, false>(t, Plan<L>::pos((L - k) & (L - 1)))];
        double2* o = Gx + ((int64_t)u * My + 2 * q) * K + k;
        o[0] = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
        o[K] = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
    }
}

template <int L>
__global__ void __launch_bounds__(FY<L>::NT) k_ky_extract(double* __restrict__ R,
                                                        const double2* __restrict__ Gx, int Mx,
                                                        int ZU, int kx0, int nkx, int kind,
                                                        int alpha, int beta,
                                                        const double2* __restrict__ tw, int blk,
                                                        int lgT3, int RC, int RS1) {
    constexpr int T = TY<L>::T;
    extern __shared__ double2 sm[];
    const int Kx = Mx / 2 + 1;
    const int ntile = (nkx + T - 1) / T;
    const int u = blockIdx.x / ntile, tile = blockIdx.x % ntile;
    const int T3 = 1 << lgT3, nt3 = (nkx + T3 - 1) >> lgT3;
    const int s2x = c2(alpha, 0) - c2(beta, 0), s2y = c2(alpha, 1) - c2(beta, 1);
    const bool im = kind == 1 && alpha != 2;
    const double2* __restrict__ col = Gx + (int64_t)u * L * Kx + kx0;
    auto ld0 = [&](int t, int n) -> double2 {
        const int kxl = tile * T + t;
        return kxl < nkx ? col[(int64_t)n * Kx + kxl] : czero();
    };
    auto stN = [&](int t, int p, double2 v) {
        const int kxl = tile * T + t;
        const int ky = Plan<L>::freq(p);
        if (kxl >= nkx || 2 * ky > L) return;
        v = cmul(v, half_phase(tw, (kx0 + kxl) * s2x, Mx, -1));
        v = cmul(v, half_phase(tw, ky * s2y, L, -1));
        R[rt_idx(ky, kxl, blk, ZU, u, lgT3, nt3, RC, RS1)] = im ? v.y : v.x;
    };
    fft_run<L, T, FY<L>::NT, false, true, 0, true>(sm, ld0, stN, tw);
}

// Folded spectrum of block `blk`, tile-major for P3:
//   R[(ky' * nt3 + kx / T3) * RC + blk * KZ * T3 + kz' * T3 + kx % T3]
//     = {Re | Im}(K^(kx, ky', kz') exp(-2 pi i k.(c_a - c_b) / M)) * scale
//   (kx local to this rank's slab [kx0, kx0 + nkx))
__global__ void k_extract(const double2* __restrict__ G, double* __restrict__ R, int Mx, int My,
                          int Mz, int kx0, int nkx, int kind, int alpha, int beta, double scale,
                          const double2* __restrict__ tw, int blk, int lgT3, int RC) {
    const int KY = My / 2 + 1, KZ = Mz / 2 + 1;
    const int T3 = 1 << lgT3;
    const int nt3 = (nkx + T3 - 1) >> lgT3;
    const int Kx = nkx;
    const int64_t tot = (int64_t)Kx * KY * KZ;
    const int s2x = c2(alpha, 0) - c2(beta, 0), s2y = c2(alpha, 1) - c2(beta, 1),
              s2z = c2(alpha, 2) - c2(beta, 2);
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int kx = (int)(idx % Kx);
        const int kz = (int)((idx / Kx) % KZ);
        const int ky = (int)(idx / ((int64_t)Kx * KZ));
        double2 v = G[((int64_t)kz * My + ky) * Mx + kx0 + kx];
        v = cmul(v, half_phase(tw, (kx0 + kx) * s2x, Mx, -1));
        v = cmul(v, half_phase(tw, ky * s2y, My, -1));
        v = cmul(v, half_phase(tw, kz * s2z, Mz, -1));
        R[((int64_t)ky * nt3 + (kx >> lgT3)) * RC + ((int64_t)blk * KZ + kz) * T3 + (kx & (T3 - 1))] =
            (kind == 0 ? v.x : v.y) * scale;
    }
}

// y = [0; Ī] x (Eq. 4's overlap diagonal, Eq. 7): dielectric rows start at Ī_k x_k, conductor
// rows at 0; P5 then stores the conductor rows and adds the field term of the dielectric rows
__global__ void k_yinit(double* __restrict__ y, const double* __restrict__ x,
                        const double* __restrict__ ibar, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        y[i] = ibar[i] * x[i];  // ibar = 0 on conductor rows
}

// active-plane flags: has[g][z] = 1 if source orientation g < 3 (field f: g = 3 + f) has a panel
// on window plane z (benign racy stores of the value 1)
__global__ void k_plane_flags(int64_t n, const int8_t* __restrict__ axis, const int32_t* __restrict__ sk,
                              const int32_t* __restrict__ cid, int lo2, int ZL,
                              const int* __restrict__ fidx, char* __restrict__ has) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int a = axis[p], z = sk[p] - lo2;
        has[(int64_t)a * ZL + z] = 1;
        has[(int64_t)(3 + fidx[(cid[p] == 0 ? 3 : 0) + a]) * ZL + z] = 1;
    }
}

__global__ void k_zero(double* y, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        y[i] = 0.0;
}

__global__ void k_debug_kappa(int n, const int32_t* kind, const int32_t* a, const int32_t* b,
                              const int32_t* d, double* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = kappa(kind[i], a[i], b[i], d[3 * i], d[3 * i + 1], d[3 * i + 2]);
}

// ---------------------------------------------------------------------------------------
// launchers (compile-time FFT length dispatch)
// ---------------------------------------------------------------------------------------

#define VC_DISPATCH_L(L, ...)                                       \
    switch (L) {                                                    \
        case 8: { constexpr int LL = 8; __VA_ARGS__; } break;       \
        case 16: { constexpr int LL = 16; __VA_ARGS__; } break;     \
        case 32: { constexpr int LL = 32; __VA_ARGS__; } break;     \
        case 64: { constexpr int LL = 64; __VA_ARGS__; } break;     \
        case 128: { constexpr int LL = 128; __VA_ARGS__; } break;   \
        case 256: { constexpr int LL = 256; __VA_ARGS__; } break;   \
        case 512: { constexpr int LL = 512; __VA_ARGS__; } break;   \
        case 1024: { constexpr int LL = 1024; __VA_ARGS__; } break; \
        case 2048: { constexpr int LL = 2048; __VA_ARGS__; } break; \
        case 4096: { constexpr int LL = 4096; __VA_ARGS__; } break; \
        default: return cudaErrorInvalidValue;                      \
    }

static cudaError_t launch_p1(const MV& mv, cudaStream_t st) {
    int maxch = 0, maxz = 0;
    for (int b = 0; b < 3; ++b) { maxz = std::max(maxz, mv.nzin[b]); }
    VC_DISPATCH_L(mv.Mx, {
        constexpr int T = TX<LL>::T;
        for (int b = 0; b < 3; ++b) maxch = std::max(maxch, ((mv.nr[mv.rank][b] + 2) / 2 + T - 1) / T);
        const size_t smem = sizeof(double2) * LL * T;
        auto kern = mv.W > 1 ? k_p1<LL, true> : k_p1<LL, false>;
        cudaError_t e = prep_fit(kern, FX<LL>::NT, smem);
        if (e) return e;
        dim3 grid(std::max(1, maxch * maxz), mv.s1 - mv.s0, mv.nb);  // sources [s0, s1)
        kern<<<grid, FX<LL>::NT, smem, st>>>(mv);
    });
    return cudaGetLastError();
}
template <int LL, int KB>
static cudaError_t launch_p4s_t(const MV& mv, cudaStream_t st) {
    constexpr int T = FYS<LL, KB>::T, NT = FYS<LL, KB>::NT;
    static_assert(T == p4_tile(LL), "X3 layout (operator_build, p4_tile) and P4's tile disagree");
    int G = 0;
    for (int f = mv.f0; f < mv.f1; ++f) G += mv.nzout[f];
    const size_t smem = sizeof(double2) * 2 * LL * T;
    auto kern = mv.W > 1 ? k_p4s<LL, KB, true> : k_p4s<LL, KB, false>;
    cudaError_t e = prep_fit(kern, NT, smem);
    if (e) return e;
    const int ntiles = G * ((mv.nkx + T - 1) / T) * mv.nb;
    if (ntiles == 0) return cudaSuccess;
    kern<<<persistent_grid(kern, NT, smem, ntiles), NT, smem, st>>>(mv);
    return cudaSuccess;
}
static cudaError_t launch_p4s(const MV& mv, cudaStream_t st) {
    cudaError_t e;
    VC_DISPATCH_L(mv.My, { e = launch_p4s_t<LL, kP4KB>(mv, st); if (e) return e; });
    return cudaGetLastError();
}
static cudaError_t launch_p2(const MV& mv, cudaStream_t st) {
    int maxz = 0;
    for (int b = 0; b < 3; ++b) maxz = std::max(maxz, mv.nzin[b]);
    VC_DISPATCH_L(mv.My, {
        constexpr int T = TY<LL>::T;
        const size_t smem = sizeof(double2) * LL * T;
        auto kern = mv.W > 1 ? k_p2<LL, true> : k_p2<LL, false>;
        cudaError_t e = prep_fit(kern, FY<LL>::NT, smem);
        if (e) return e;
        dim3 grid(std::max(1, ((mv.nkx + T - 1) / T) * maxz), mv.s1 - mv.s0, mv.nb);  // sources [s0, s1)
        kern<<<grid, FY<LL>::NT, smem, st>>>(mv);
    });
    return cudaGetLastError();
}
template <int L, int NF>
static size_t p3_smem(const MV& mv, int ns) {
    constexpr int W = P3T<L, NF>::W, T = P3T<L, NF>::T;
    const size_t XS = (size_t)2 * T * (mv.nzin[0] + mv.nzin[1] + mv.nzin[2]);
    return sizeof(double2) * ((size_t)L * W + L + ns * XS) + sizeof(double) * ns * (size_t)mv.rchunk +
           sizeof(int16_t) * ((9 * (L + 2) + 3) & ~3) + 2 * sizeof(uint64_t);
}
template <int L, int NF, int NS>
static cudaError_t launch_p3_ns(const MV& mv, cudaStream_t st, size_t smem) {
    constexpr int T = P3T<L, NF>::T;
    cudaError_t e = prep(k_p3<L, NF, NS>, smem);
    if (e) return e;
    int per_sm = 0, nsm = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_p3<L, NF, NS>, kNT3, smem);
    const int ntiles = ((mv.nkx + T - 1) / T) * (mv.My / 2 + 1);
    if (ntiles == 0) return cudaSuccess;
    const int grid = std::max(1, std::min(ntiles, std::max(1, per_sm) * nsm));
    k_p3<L, NF, NS><<<grid, kNT3, smem, st>>>(mv);
    return cudaSuccess;
}
template <int L, int NF>
static cudaError_t launch_p3_t(const MV& mv, cudaStream_t st) {
    // one stage when that lets two CTAs share an SM (VC_P3_NS forces 1 or 2: A/B)
    static const int ns_env = getenv("VC_P3_NS") ? atoi(getenv("VC_P3_NS")) : 0;
    const size_t s1 = p3_smem<L, NF>(mv, 1), s2 = p3_smem<L, NF>(mv, 2);
    const int ns = ns_env == 1 || ns_env == 2 ? ns_env : (s1 <= 112 * 1024 && s2 > 112 * 1024 ? 1 : 2);
    const size_t smem = ns == 1 ? s1 : s2;
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    return ns == 1 ? launch_p3_ns<L, NF, 1>(mv, st, smem) : launch_p3_ns<L, NF, 2>(mv, st, smem);
}
template <int L>
static cudaError_t launch_p3_l(const MV& mv, cudaStream_t st) {
    switch (mv.nf) {
        case 1: return launch_p3_t<L, 1>(mv, st);
        case 2: return launch_p3_t<L, 2>(mv, st);
        case 3: return launch_p3_t<L, 3>(mv, st);
        case 4: return launch_p3_t<L, 4>(mv, st);
        case 5: return launch_p3_t<L, 5>(mv, st);
        case 6: return launch_p3_t<L, 6>(mv, st);
        default: return cudaErrorInvalidValue;
    }
}
static bool p3m_batched(const MV& mv) { return mv.zdirect != 0; }
static cudaError_t launch_p3(const MV& mv, cudaStream_t st) {
    if (mv.nb > 1 && !p3m_batched(mv)) {
        // column by column (z-FFT mode, or the batched tile does not fit one CTA)
        for (int c = 0; c < mv.nb; ++c) {
            MV m1 = mv;
            m1.nb = 1;
            for (int b = 0; b < 3; ++b) m1.X2[b] += c * mv.colB;
            for (int f = 0; f < 6; ++f) m1.X3[f] += c * mv.colC;
            const cudaError_t e = launch_p3(m1, st);
            if (e) return e;
        }
        return cudaSuccess;
    }
    if (mv.zdirect) return launch_p3m(mv, st);
    cudaError_t e;
    switch (mv.Mz) {  // kMaxLz: the [L][W] pencil buffer must fit one CTA's shared memory
        case 8: e = launch_p3_l<8>(mv, st); break;
        case 16: e = launch_p3_l<16>(mv, st); break;
        case 32: e = launch_p3_l<32>(mv, st); break;
        case 64: e = launch_p3_l<64>(mv, st); break;
        case 128: e = launch_p3_l<128>(mv, st); break;
        case 256: e = launch_p3_l<256>(mv, st); break;
        default: return cudaErrorInvalidValue;
    }
    if (e) return e;
    return cudaGetLastError();
}

static cudaError_t launch_p5(const MV& mv, cudaStream_t st) {
    int maxz = 0, maxch = 0;
    for (int f = 0; f < mv.nf; ++f) maxz = std::max(maxz, mv.nzout[f]);
    VC_DISPATCH_L(mv.Mx, {
        constexpr int T = TX<LL>::T;
        for (int f = 0; f < mv.nf; ++f) maxch = std::max(maxch, ((mv.nr[mv.rank][3 + f] + 2) / 2 + T - 1) / T);
        // FFT buffer (one rank: the staged input block, which may be a little larger) + slot lines
        const size_t smem = (mv.W > 1 ? sizeof(double2) * LL * T : p5_inbytes(LL, T, mv.nkx)) +
                            sizeof(int32_t) * 2 * T * LL;
        auto kern = mv.W > 1 ? k_p5<LL, true> : mv.lgt4 == 0 ? k_p5<LL, false, true> : k_p5<LL, false>;
        cudaError_t e = prep_fit(kern, FX<LL>::NT, smem);
        if (e) return e;
        dim3 grid(std::max(1, maxch * maxz), mv.f1 - mv.f0, mv.nb);  // fields [f0, f1)
        kern<<<grid, FX<LL>::NT, smem, st>>>(mv);
    });
    return cudaGetLastError();
}
static cudaError_t launch_fft_lines(double2* d, int L, int64_t nlines, bool inv,
                                    const double2* tw, cudaStream_t st) {
    VC_DISPATCH_L(L, {
        constexpr int T = TX<LL>::T;
        const size_t smem = sizeof(double2) * LL * T;
        const unsigned grid = (unsigned)((nlines + T - 1) / T);
        if (inv) {
            cudaError_t e = prep(k_fft_lines<LL, true>, smem);
            if (e) return e;
            k_fft_lines<LL, true><<<grid, FX<LL>::NT, smem, st>>>(d, nlines, tw);
        } else {
            cudaError_t e = prep(k_fft_lines<LL, false>, smem);
            if (e) return e;
            k_fft_lines<LL, false><<<grid, FX<LL>::NT, smem, st>>>(d, nlines, tw);
        }
    });
    return cudaGetLastError();
}
static cudaError_t launch_kx_r2c(double2* Gx, const double* Ko, int Mx, int My, int ZU, int Ox,
                                 int Oy, int kind, int alpha, int beta, const double2* tw,
                                 cudaStream_t st) {
    VC_DISPATCH_L(Mx, {
        constexpr int T = TX<LL>::T;
        const size_t smem = sizeof(double2) * LL * T + sizeof(int32_t) * LL;  // + x table
        cudaError_t e = prep(k_kx_r2c<LL>, smem);
        if (e) return e;
        const unsigned grid = (unsigned)(((int64_t)ZU * (My / 2) + T - 1) / T);
        k_kx_r2c<LL><<<grid, FX<LL>::NT, smem, st>>>(Gx, Ko, My, ZU, Ox, Oy, kind, alpha, beta, tw);
    });
    return cudaGetLastError();
}
static cudaError_t launch_ky_extract(double* R, const double2* Gx, int Mx, int My, int ZU, int kx0,
                                     int nkx, int kind, int alpha, int beta, const double2* tw,
                                     int blk, int lgT3, int RC, int RS1, cudaStream_t st) {
    VC_DISPATCH_L(My, {
        constexpr int T = TY<LL>::T;
        const size_t smem = sizeof(double2) * LL * T;
        cudaError_t e = prep(k_ky_extract<LL>, smem);
        if (e) return e;
        const unsigned grid = (unsigned)(ZU * ((nkx + T - 1) / T));
        if (grid) k_ky_extract<LL><<<grid, FY<LL>::NT, smem, st>>>(R, Gx, Mx, ZU, kx0, nkx, kind, alpha,
                                                                 beta, tw, blk, lgT3, RC, RS1);
    });
    return cudaGetLastError();
}

static cudaError_t launch_fft_strided(double2* d, int L, int64_t es, int64_t ncols,
                                      int64_t nbatch, int64_t bs, const double2* tw,
                                      cudaStream_t st) {
    VC_DISPATCH_L(L, {
        constexpr int T = TY<LL>::T;
        const size_t smem = sizeof(double2) * LL * T;
        cudaError_t e = prep(k_fft_strided<LL>, smem);
        if (e) return e;
        const unsigned grid = (unsigned)(((ncols + T - 1) / T) * nbatch);
        k_fft_strided<LL><<<grid, FY<LL>::NT, smem, st>>>(d, es, ncols, bs, tw);
    });
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// planning and build (vc_build_operator)
// ---------------------------------------------------------------------------------------
// ---- slab planning (host only; also exported as vc_plan_slabs for tests) -----------------
// Spectral: rank q owns kx tiles [q nt / W, (q + 1) nt / W) of width T3.
void plan_kx_slabs(int W, int Kx, int T3, int* kxa) {
    const int nt = (Kx + T3 - 1) / T3;
    for (int q = 0; q <= W; ++q) kxa[q] = std::min(Kx, (int)((int64_t)q * nt / W) * T3);
    kxa[W] = Kx;
}
// Spatial: the preconditioner box rows (along y, box height Nv) that the window rows
// [lo, lo + EY) touch are split into W contiguous ranges; a slot row belongs to the rank of
// its box row (the top row ny joins the last box, as in the preconditioner).
int row_owner_plan(int W, int Nv, int nb, int b0, int nbr, int yabs) {
    const int br = std::min(std::max(yabs, 0) / Nv, nb - 1) - b0;
    int p = 0;
    while (p + 1 < W && (int64_t)(p + 1) * nbr / W <= br) ++p;
    return p;
}
void plan_row_slabs(int W, int ny, int lo, int EY, int Nv, int* ya, int* nb_out, int* b0_out,
                    int* nbr_out) {
    const int nb = std::max(1, (ny + Nv - 1) / Nv);
    const int b0 = std::min(lo / Nv, nb - 1);
    const int nbr = std::min((lo + EY - 1) / Nv, nb - 1) - b0 + 1;
    ya[0] = 0;
    int p = 1;
    for (int y = 0; y < EY && p < W; ++y)
        while (p < W && row_owner_plan(W, Nv, nb, b0, nbr, lo + y) >= p) ya[p++] = y;
    for (; p <= W; ++p) ya[p] = EY;
    *nb_out = nb;
    *b0_out = b0;
    *nbr_out = nbr;
}

static int next_pow2(int v) {
    int p = 8;
    while (p < v) p *= 2;
    return p;
}

vc_status operator_build(vc_ctx* c, const vc_build_opts* o) {
    if (c->world > 1) mirror_wait(c);  // the slab bookkeeping reads the host panel mirror
    cudaStream_t st = c->stream;
    HostTrace tr("operator");
    // window origin and per-orientation extents
    int lo[3] = {INT32_MAX, INT32_MAX, INT32_MAX};
    bool has[2][3] = {{false, false, false}, {false, false, false}};
    for (int kind = 0; kind < 2; ++kind)
        for (int a = 0; a < 3; ++a) {
            if (c->ext[kind][a][0][0] > c->ext[kind][a][1][0]) continue;
            has[kind][a] = true;
            for (int t = 0; t < 3; ++t) lo[t] = std::min(lo[t], c->ext[kind][a][0][t]);
        }
    // centre extents (doubled) of each (kind, orientation) class along each axis
    auto cmin2 = [&](int kind, int a, int t) { return 2 * c->ext[kind][a][0][t] + c2(a, t); };
    auto cmax2 = [&](int kind, int a, int t) { return 2 * c->ext[kind][a][1][t] + c2(a, t); };
    int req[3] = {8, 8, 8};
    for (int t = 0; t < 3; ++t) {
        for (int kr = 0; kr < 2; ++kr)
            for (int al = 0; al < 3; ++al) {
                if (!has[kr][al]) continue;
                for (int ks = 0; ks < 2; ++ks)
                    for (int be = 0; be < 3; ++be) {
                        if (!has[ks][be]) continue;
                        // largest |centre offset| (doubled) between rows (kr,al) and cols (ks,be)
                        const int L2 = std::max(cmax2(kr, al, t) - cmin2(ks, be, t),
                                                cmax2(ks, be, t) - cmin2(kr, al, t));
                        const int s2 = c2(al, t) - c2(be, t);
                        int r;
                        if (s2 != 0) r = L2 + 1;            // half-integer offsets: M >= 2L + 1
                        else r = L2 + ((kr == 1 && al == t) ? 1 : 0);  // integer: 2L (+1 if odd)
                        req[t] = std::max(req[t], r);
                    }
            }
        int extmax = 0;
        for (int kind = 0; kind < 2; ++kind)
            for (int a = 0; a < 3; ++a)
                if (has[kind][a]) extmax = std::max(extmax, c->ext[kind][a][1][t] - lo[t] + 1);
        req[t] = std::max(req[t], extmax);
    }
    int M[3];
    for (int t = 0; t < 3; ++t) {
        M[t] = next_pow2(req[t]);
        if (o && o->pad[t]) {
            if (o->pad[t] < req[t] || (o->pad[t] & (o->pad[t] - 1)) || o->pad[t] < 8)
                return set_err(c, VC_ERR_INPUT, "pad must be a power of two >= 8 and >= the exactness bound " + std::to_string(req[t]));
            M[t] = o->pad[t];
        }
        if (M[t] > kMaxL) return set_err(c, VC_ERR_UNSUPPORTED, "padded FFT size > 4096 along an axis");
        if (t == 2 && M[t] > kMaxLz)
            return set_err(c, VC_ERR_UNSUPPORTED, "padded FFT size along z > 256 (P3 shared-memory pencils)");
    }
    for (int t = 0; t < 3; ++t) {
        c->M[t] = M[t];
        c->lo[t] = lo[t];
    }
    c->Kx = M[0] / 2 + 1;
    const int Kx = c->Kx, My = M[1], Mz = M[2];
    // source orientations (any panel kind) and output fields
    for (int b = 0; b < 3; ++b) {
        int hi[3] = {-1, -1, -1};
        for (int kind = 0; kind < 2; ++kind)
            if (has[kind][b])
                for (int t = 0; t < 3; ++t) hi[t] = std::max(hi[t], c->ext[kind][b][1][t]);
        for (int t = 0; t < 3; ++t) c->ext_in[b][t] = hi[t] < 0 ? 0 : hi[t] - lo[t] + 1;
    }
    c->nf = 0;
    for (int kind = 0; kind < 2; ++kind)
        for (int a = 0; a < 3; ++a) {
            if (!has[kind][a]) continue;
            Field& F = c->f[c->nf++];
            F.kind = kind;
            F.axis = a;
            for (int t = 0; t < 3; ++t) F.ext[t] = c->ext[kind][a][1][t] - lo[t] + 1;
        }
    // kernel blocks: (field, beta); P^{ab} and P^{ba} share one spectrum (Eq. 12)
    int pblk[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) pblk[a][b] = -1;
    struct BlkDef { int kind, alpha, beta; };
    std::vector<BlkDef> defs;
    for (int f = 0; f < c->nf; ++f)
        for (int b = 0; b < 3; ++b) {
            c->blk[f][b] = -1;
            if (c->ext_in[b][0] == 0) continue;
            const int kind = c->f[f].kind, a = c->f[f].axis;
            if (kind == 0) {
                const int lo_ = std::min(a, b), hi_ = std::max(a, b);
                if (pblk[lo_][hi_] < 0) {
                    pblk[lo_][hi_] = (int)defs.size();
                    defs.push_back({0, lo_, hi_});
                }
                c->blk[f][b] = pblk[lo_][hi_];
            } else {
                c->blk[f][b] = (int)defs.size();
                defs.push_back({1, a, b});
            }
        }
    for (int f = c->nf; f < 6; ++f)
        for (int b = 0; b < 3; ++b) c->blk[f][b] = -1;
    c->nblk = (int)defs.size();
    c->blk_stride = (size_t)Kx * (My / 2 + 1) * (Mz / 2 + 1);
    // active z-planes: a plane of source orientation b (output field f) is transformed along x
    // and y only if it holds b-panels (f-panels); empty planes are zero and never touched
    {
        int ZL = 1;
        for (int b = 0; b < 3; ++b) ZL = std::max(ZL, c->ext_in[b][2]);
        for (int f = 0; f < c->nf; ++f) ZL = std::max(ZL, c->f[f].ext[2]);
        int fidx[2][3] = {{-1, -1, -1}, {-1, -1, -1}};
        for (int f = 0; f < c->nf; ++f) fidx[c->f[f].kind][c->f[f].axis] = f;
        // plane occupancy on the device (one flag per (source or field, plane)), read back as
        // 9 ZL bytes: no host loop over the panels (round 2)
        std::vector<char> has(9 * (size_t)ZL, 0);
        {
            DevBuf<char> dh;
            DevBuf<int> dfi;
            VC_CUDA(c, dh.alloc(has.size()));
            VC_CUDA(c, cudaMemsetAsync(dh.p, 0, has.size(), st));
            VC_CUDA(c, dfi.alloc(6));
            int fl[6];
            for (int q = 0; q < 6; ++q) fl[q] = fidx[q / 3][q % 3];
            VC_CUDA(c, cudaMemcpyAsync(dfi.p, fl, sizeof fl, cudaMemcpyHostToDevice, st));
            if (c->N)
                k_plane_flags<<<(unsigned)std::min<int64_t>((c->N + 255) / 256, 148 * 8), 256, 0, st>>>(
                    c->N, c->pan.axis.p, c->pan.sk.p, c->pan.cid.p, lo[2], ZL, dfi.p, dh.p);
            count_launch(c);
            VC_CUDA(c, cudaMemcpyAsync(has.data(), dh.p, has.size(), cudaMemcpyDeviceToHost, st));
            VC_CUDA(c, cudaStreamSynchronize(st));
        }
        std::vector<int32_t> hp(18 * (size_t)ZL, -1);
        for (int g = 0; g < 9; ++g) {
            int n = 0;
            for (int z = 0; z < ZL; ++z)
                if (has[(size_t)g * ZL + z]) {
                    hp[(size_t)g * ZL + n] = z;
                    hp[(size_t)(9 + g) * ZL + z] = n;
                    ++n;
                }
            if (g < 3) c->nzin[g] = n;
            else c->nzout[g - 3] = n;
        }
        c->ZL = ZL;
        c->h_planes = hp;
        VC_CUDA(c, c->planes.alloc(hp.size()));
        VC_CUDA(c, cudaMemcpyAsync(c->planes.p, hp.data(), 4 * hp.size(), cudaMemcpyHostToDevice, st));
        VC_CUDA(c, cudaStreamSynchronize(st));
    }
    // P3 mode: direct z-convolution when the layered structure makes it cheaper than the
    // z-FFTs (complex-by-real MACs vs a radix-2 estimate of 3 + n_f transforms of length Mz)
    {
        double mac = 0;
        int nrows = 0;
        for (int f = 0; f < c->nf; ++f) {
            for (int b = 0; b < 3; ++b)
                if (c->blk[f][b] >= 0) mac += (double)c->nzout[f] * c->nzin[b];
            nrows += c->nzout[f];
        }
        // k_p3m columns: stacked plane positions, each source padded to an even count (X2
        // sectors never straddle two sources) and the total to a multiple of 4
        int zoff[3], nzp = 0;
        for (int b = 0; b < 3; ++b) {
            zoff[b] = nzp;
            nzp += (c->nzin[b] + 1) & ~1;
        }
        nzp = (nzp + 3) & ~3;
        const double fft = 0.6 * (3 + c->nf) * 5.0 * Mz * ilog2c(Mz);
        const int zmode = o ? o->zmode : 0;
        if (zmode < 0 || zmode > 2) return set_err(c, VC_ERR_INPUT, "zmode must be 0, 1 or 2");
        // k_p3m: stacked rows in 8-row chunks, split into balanced passes of <= kMmaMC chunks
        const int mct0 = (nrows + 7) / 8, npass = std::max(1, (mct0 + kMmaMC - 1) / kMmaMC);
        const int mct = npass * ((mct0 + npass - 1) / npass), kc = nzp / 4;
        const int rs1 = std::max(1, c->nblk) * c->ZL + 1;
        // ring depth: 2 measured fastest on C4 (0.538 / 0.546 / 0.550 / 0.559 ms for 2 / 3 / 4 / 5
        // stages per pair launch); VC_P3M_NST overrides it (A/B), bounded by what fits
        // odd (E^{z.}) blocks: k_p3m keeps negated copies of their rows so that no A entry
        // carries a sign (the A offsets are plain uint16 row indices, negated rows at 8 ks1 + row)
        int oddmask = 0;
        for (int f = 0; f < c->nf; ++f)
            if (c->f[f].kind == 1 && c->f[f].axis == 2)
                for (int b = 0; b < 3; ++b)
                    if (c->blk[f][b] >= 0) oddmask |= 1 << c->blk[f][b];
        const bool tkb = o && o->tucker_digits > 0;
        const int ks1 = tkb ? (rs1 | 1) : rs1;  // K row stride in shared memory
        const int nst_fit = p3m_stages(rs1, nzp, kc, mct, false);
        const int nst = std::min(nst_fit, getenv("VC_P3M_NST") ? std::max(2, atoi(getenv("VC_P3M_NST"))) : 2);
        c->zdirect = nrows <= kMaxRows && nzp > 0 && nzp + 4 <= 256 && rs1 <= 0x7fff && 9 * ks1 <= 0xffff &&
                     nst_fit >= 2 &&
                     (zmode == 2 || (zmode == 0 && 4.0 * mac <= fft));
        if (zmode == 2 && !c->zdirect)
            return set_err(c, VC_ERR_UNSUPPORTED, "direct-z mode: too many output planes or input planes");
        const int tkd = o ? o->tucker_digits : 0;
        if (tkd < 0 || tkd > 14) return set_err(c, VC_ERR_INPUT, "tucker_digits must be 0..14");
        if (tkd > 0 && !c->zdirect)
            return set_err(c, VC_ERR_UNSUPPORTED, "Tucker-compressed spectra need the direct-z P3 (zmode 0 choosing it, or 2)");
        c->ZU = c->ZL;
        c->rs1 = c->zdirect ? rs1 : 0;
        c->p3m_nzt = c->p3m_kc = c->p3m_mct = 0;
        auto plane = [&](int g, int j) { return c->h_planes[(size_t)g * c->ZL + j]; };
        if (c->zdirect) {
            // DMMA fragment tables of k_p3m (see the kernel): A[r][c] = K^{f_r b_c}(u(z_r - z_c)),
            // uint16 row | sign << 15, [KC][MCT][32]; then the output rows (f | plane << 4)
            std::vector<int32_t> rows(8 * (size_t)mct, -1), cols(nzp, -1);
            int r = 0;
            for (int f = 0; f < c->nf; ++f)
                for (int j = 0; j < c->nzout[f]; ++j) rows[r++] = f | j << 4;
            for (int b = 0; b < 3; ++b)
                for (int j = 0; j < c->nzin[b]; ++j) cols[zoff[b] + j] = b << 16 | j;
            const int zero_row = rs1 - 1;
            std::vector<uint16_t> at;
            at.reserve((size_t)kc * mct * 32 + 1);
            for (int k = 0; k < kc; ++k)
                for (int m = 0; m < mct; ++m)
                    for (int l = 0; l < 32; ++l) {
                        const int rr = m * 8 + l / 4, cc = k * 4 + l % 4;
                        uint16_t e = (uint16_t)zero_row;
                        if (rows[rr] >= 0 && cols[cc] >= 0) {
                            const int f = rows[rr] & 15, jo = rows[rr] >> 4;
                            const int b = cols[cc] >> 16, ji = cols[cc] & 0xffff;
                            const int bk = c->blk[f][b];
                            if (bk >= 0) {
                                const int s2 = c2(c->f[f].axis, 2) - c2(b, 2);
                                const int g2 = 2 * plane(3 + f, jo) + s2 - 2 * plane(b, ji);
                                const int u = ((g2 < 0 ? -g2 : g2) - (s2 != 0)) >> 1;
                                if (u < 0 || u >= c->ZU) return set_err(c, VC_ERR_INPUT, "direct-z offset out of range");
                                const bool odd = c->f[f].kind == 1 && c->f[f].axis == 2;
                                // Tucker P3: negated copy at 8 ks1 + row; exact table: sign bit
                                e = tkb ? (uint16_t)((odd && g2 < 0 ? 8 * ks1 : 0) + bk * c->ZU + u)
                                        : (uint16_t)((bk * c->ZU + u) | (odd && g2 < 0 ? 0x8000 : 0));
                            }
                        }
                        at.push_back(e);
                    }
            if (at.size() & 1) at.push_back(0);
            std::vector<int32_t> negs;
            for (int b = 0; b < c->nblk; ++b)
                if (oddmask >> b & 1)
                    for (int u = 0; u < c->ZU; ++u) negs.push_back(b * c->ZU + u);
            std::vector<int32_t> tab(at.size() / 2 + rows.size() + negs.size());
            memcpy(tab.data(), at.data(), 2 * at.size());
            memcpy(tab.data() + at.size() / 2, rows.data(), 4 * rows.size());
            memcpy(tab.data() + at.size() / 2 + rows.size(), negs.data(), 4 * negs.size());
            c->p3m_nneg = (int)negs.size();
            c->p3m_oddmask = oddmask;
            c->p3m_negoff = at.size() / 2 + rows.size();
            c->p3m_nzt = nzp;
            c->p3m_nst = nst;
            c->p3m_kc = kc;
            c->p3m_mct = mct;
            for (int b = 0; b < 3; ++b) c->p3m_zoff[b] = zoff[b];
            VC_CUDA(c, c->p3m_tab.alloc(tab.size()));
            VC_CUDA(c, cudaMemcpyAsync(c->p3m_tab.p, tab.data(), 4 * tab.size(), cudaMemcpyHostToDevice, st));
            VC_CUDA(c, cudaStreamSynchronize(st));
        }
    }
    tr.mark("plans");
    // P3 tile width and the tile-major spectrum layout (one contiguous chunk per P3 tile)
    c->T3 = c->zdirect ? kMmaT : p3_tile(Mz, c->nf);
    plan_kx_slabs(c->world, Kx, c->T3, c->kxa);
    const int kx0 = c->kxa[c->rank], nkx = c->kxa[c->rank + 1] - kx0;
    c->nt3 = (nkx + c->T3 - 1) / c->T3;
    // direct-z: [t][block * ZU + u] plus one zero row per kx (k_p3m's absent / padding entries)
    c->rchunk = c->zdirect ? (size_t)c->T3 * c->rs1
                           : ((size_t)std::max(1, c->nblk) * (Mz / 2 + 1) * c->T3 + 1) & ~(size_t)1;
    VC_CUDA(c, c->tw.alloc(kTabN));
    k_twiddles<<<(kTabN + 255) / 256, 256, 0, st>>>(c->tw.p);
    count_launch(c);
    // kernel-table reuse (as a device-resident cache): the spectra and the
    // preconditioner near-field tables depend only on this signature -- grid, z mode, blocks,
    // tile layout, rank slab, dv, boxes and the build variants -- not on where the panels are or
    // on the permittivities, so with vc_build_opts.reuse_tables a rebuild on the same signature
    // keeps the tables already in HBM
    std::vector<double> key = {(double)M[0], (double)M[1], (double)M[2], (double)c->zdirect,
                               (double)c->ZU, (double)c->T3, (double)c->rchunk, (double)nkx,
                               (double)kx0, (double)c->world, (double)c->rank, c->dv,
                               (double)c->box[0], (double)c->box[1], (double)c->box[2],
                               (double)(o && o->no_mirror),
                               (double)(getenv("VC_KT_LEGACY") && atoi(getenv("VC_KT_LEGACY")))};
    for (const BlkDef& d : defs) {
        key.push_back(d.kind);
        key.push_back(d.alpha);
        key.push_back(d.beta);
    }
    const size_t rt_n = std::max<size_t>(1, c->rchunk * (size_t)(My / 2 + 1) * c->nt3);
    // Tucker-compressed spectra (NEXT-1) and their cache file (NEXT-4, keyed without the
    // preconditioner boxes, which the spectra do not depend on)
    Tucker& TK = c->tk;
    TK.on = o && o->tucker_digits > 0;
    TK.cache = 0;
    TK.err.clear();
    std::vector<double> tk_key;
    bool tk_hit = false;
    if (TK.on) {
        TK.digits = o->tucker_digits;
        TK.nblk = c->nblk;
        TK.nkx = nkx;
        TK.nq = My / 2 + 1;
        TK.ZU = c->ZU;
        TK.dv = c->dv;
        for (int i = 0; i < c->nblk && i < 16; ++i) TK.kind[i] = defs[i].kind;
        // the spectra scale as dv^3 (P) / dv^2 (E) (App. C): the file is independent of dv
        tk_key = {1.0 /* format */, (double)M[0], (double)M[1], (double)M[2], (double)c->ZU, (double)nkx,
                  (double)kx0, (double)c->world, (double)c->rank, (double)TK.digits,
                  (double)(o && o->no_mirror)};
        for (const BlkDef& d : defs) {
            tk_key.push_back(d.kind);
            tk_key.push_back(d.alpha);
            tk_key.push_back(d.beta);
        }
        tk_hit = tucker_try_load(c, o->tucker_cache, tk_key);
    }
    const bool reuse = !TK.on && o && o->reuse_tables && key == c->kt_key && c->Rt.p && c->Rt.n == rt_n;
    c->kt_key.clear();
    c->tables_reused = reuse;
    if (tk_hit) {
        c->Rt.reset();  // the compressed tables come from the cache file: no exact table at all
    } else {
        VC_CUDA(c, c->Rt.alloc(rt_n));
        if (!reuse) VC_CUDA(c, cudaMemsetAsync(c->Rt.p, 0, c->Rt.bytes(), st));
    }
    // spectra (a2 on the parity octant -> full cyclic grid -> 3-D FFT -> phase strip + fold)
    {
        // no host synchronisation in this loop: the preconditioner's host bookkeeping (next in
        // vc_build_operator) overlaps the kernel-table work; per-block event pairs are read
        // once the build is complete (kernel_table_times)
        if (c->kev.size() < 4 * (size_t)std::max(1, c->nblk)) {
            const size_t n0 = c->kev.size();
            c->kev.resize(4 * (size_t)std::max(1, c->nblk));
            for (size_t e = n0; e < c->kev.size(); ++e) VC_CUDA(c, cudaEventCreate(&c->kev[e]));
        }
        c->kev_n = (reuse || tk_hit) ? 0 : c->nblk;
        DevBuf<double2>& G = c->kG;
        DevBuf<double>& Ko = c->kKo;
        const bool zd = c->zdirect;
        // z-FFT mode: full 3-D cyclic grid; direct-z mode: x/y-cyclic grid x ZU octant z offsets
        const int MZ = zd ? c->ZU : M[2];
        const int64_t tot = (int64_t)M[0] * M[1] * MZ;
        const int Ox = M[0] / 2 + 1, Oy = M[1] / 2 + 1, Oz = zd ? c->ZU : M[2] / 2 + 1;
        const int64_t otot = (int64_t)Ox * Oy * Oz;
        if (!reuse && !tk_hit) {
            VC_CUDA(c, G.alloc(tot));
            VC_CUDA(c, Ko.alloc(otot));
        }
        // preconditioner near-field tables: one per P pair, |t| <= box along each axis
        for (int a = 0; a < 3; ++a) c->pcTabDim[a] = c->box[a] + 1;
        const int tvol = c->pcTabDim[0] * c->pcTabDim[1] * c->pcTabDim[2];
        int npair = 0;
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) c->pcPair[a][b] = -1;
        for (int i = 0; i < c->nblk; ++i)
            if (defs[i].kind == 0) {
                c->pcPair[defs[i].alpha][defs[i].beta] = c->pcPair[defs[i].beta][defs[i].alpha] = npair;
                ++npair;
            }
        VC_CUDA(c, c->pcTab.alloc((size_t)std::max(1, npair) * tvol));
        const double fpe = 4.0 * kPi * kEps0;
        if (!reuse) {
        // x <-> y mirror pairs (k_rt_mirror): with a square x/y window on one rank, a block whose
        // mirror was listed earlier is transposed from it instead of generated + transformed
        const bool mirror_ok = M[0] == M[1] && c->world == 1 && !(o && o->no_mirror);
        auto sig = [](int a) { return a == 0 ? 1 : (a == 1 ? 0 : 2); };
        std::vector<int> mirror_of(c->nblk, -1);
        if (mirror_ok)
            for (int i = 0; i < c->nblk; ++i) {
                int ma = sig(defs[i].alpha), mb = sig(defs[i].beta);
                if (defs[i].kind == 0 && ma > mb) std::swap(ma, mb);  // P pairs stored with a <= b
                if (ma == defs[i].alpha && mb == defs[i].beta) continue;
                for (int j = 0; j < i; ++j)
                    if (mirror_of[j] < 0 && defs[j].kind == defs[i].kind && defs[j].alpha == ma &&
                        defs[j].beta == mb) {
                        mirror_of[i] = j;
                        break;
                    }
            }
        const int NW = zd ? c->ZU : Mz / 2 + 1;
        // direct-z: fused kernel-table stages (VC_KT_LEGACY=1: the fill / FFT / extract chain)
        const bool fused_kt = !(getenv("VC_KT_LEGACY") && atoi(getenv("VC_KT_LEGACY")));
        {   // preconditioner near-field tables of every P pair, evaluated directly (one launch)
            CornerPairs cp{};
            for (int i = 0; i < c->nblk; ++i)
                if (defs[i].kind == 0) {
                    cp.alpha[cp.n] = defs[i].alpha;
                    cp.beta[cp.n] = defs[i].beta;
                    cp.slot[cp.n] = c->pcPair[defs[i].alpha][defs[i].beta];
                    ++cp.n;
                }
            if (cp.n) {
                k_kgen_corner<<<dim3((tvol + 127) / 128, cp.n), 128, 0, st>>>(
                    c->pcTab.p, c->pcTabDim[0], c->pcTabDim[1], c->pcTabDim[2], Ox, Oy, Oz, cp,
                    c->dv * c->dv * c->dv / fpe);
                count_launch(c);
            }
        }
        for (int pass = 0; pass < (tk_hit ? 0 : 2); ++pass)
        for (int i = 0; i < c->nblk; ++i) {
            const BlkDef& d = defs[i];
            if ((mirror_of[i] >= 0) != (pass == 1)) continue;
            const double scale = (d.kind == 0 ? c->dv * c->dv * c->dv : c->dv * c->dv) / fpe /
                                 ((double)M[0] * M[1] * (zd ? 1 : M[2]));
            cudaEvent_t* ev = c->kev.data() + 4 * (size_t)i;
            if (mirror_of[i] >= 0) {
                VC_CUDA(c, cudaEventRecord(ev[0], st));
                VC_CUDA(c, cudaEventRecord(ev[1], st));
                VC_CUDA(c, cudaEventRecord(ev[2], st));
                const int64_t mt = (int64_t)Kx * Kx * NW;
                k_rt_mirror<<<(int)std::min<int64_t>((mt + 255) / 256, 148 * 32), 256, 0, st>>>(
                    c->Rt.p, Kx, NW, mirror_of[i], i, ilog2c(c->T3), (int)c->rchunk, c->rs1);
                count_launch(c);
                VC_CUDA(c, cudaEventRecord(ev[3], st));
                continue;
            }
            VC_CUDA(c, cudaEventRecord(ev[0], st));
            const int oblocks = (int)std::min<int64_t>((otot + 127) / 128, 148 * 64);
            k_kgen_oct<<<oblocks, 128, 0, st>>>(Ko.p, Ox, Oy, Oz, d.kind, d.alpha, d.beta, scale,
                                                d.alpha == 2 && d.beta == 2 && Ox == Oy);
            if (zd && fused_kt) {  // fused x / y stages (k_kx_r2c, k_ky_extract)
                VC_CUDA(c, launch_kx_r2c(G.p, Ko.p, M[0], M[1], MZ, Ox, Oy, d.kind, d.alpha, d.beta,
                                         c->tw.p, st));
                VC_CUDA(c, cudaEventRecord(ev[1], st));
                VC_CUDA(c, cudaEventRecord(ev[2], st));
                VC_CUDA(c, launch_ky_extract(c->Rt.p, G.p, M[0], M[1], MZ, kx0, nkx, d.kind, d.alpha,
                                             d.beta, c->tw.p, i, ilog2c(c->T3), (int)c->rchunk, c->rs1, st));
                VC_CUDA(c, cudaEventRecord(ev[3], st));
                count_launch(c, 3);
                continue;
            }
            const int gblocks = (int)std::min<int64_t>((tot + 255) / 256, 148 * 64);
            if (zd)
                k_kfill2d<<<gblocks, 256, 0, st>>>(G.p, Ko.p, M[0], M[1], MZ, Ox, Oy, d.kind, d.alpha, d.beta);
            else
                k_kfill<<<gblocks, 256, 0, st>>>(G.p, Ko.p, M[0], M[1], M[2], Ox, Oy, d.kind, d.alpha, d.beta);
            VC_CUDA(c, cudaEventRecord(ev[1], st));
            VC_CUDA(c, launch_fft_lines(G.p, M[0], (int64_t)M[1] * MZ, false, c->tw.p, st));
            VC_CUDA(c, launch_fft_strided(G.p, M[1], M[0], M[0], MZ, (int64_t)M[0] * M[1], c->tw.p, st));
            if (!zd)
                VC_CUDA(c, launch_fft_strided(G.p, M[2], (int64_t)M[0] * M[1], (int64_t)M[0] * M[1], 1, 0, c->tw.p, st));
            VC_CUDA(c, cudaEventRecord(ev[2], st));
            const int64_t etot = (int64_t)std::max(1, nkx) * (My / 2 + 1) * (zd ? c->ZU : Mz / 2 + 1);
            const int eblocks = (int)std::max<int64_t>(1, std::min<int64_t>((etot + 255) / 256, 148 * 32));
            if (zd)
                k_extract2d<<<eblocks, 256, 0, st>>>(G.p, c->Rt.p, M[0], M[1], c->ZU, kx0, nkx, d.kind,
                                                     d.alpha, d.beta, c->tw.p, i, ilog2c(c->T3),
                                                     (int)c->rchunk, c->rs1);
            else
                k_extract<<<eblocks, 256, 0, st>>>(G.p, c->Rt.p, M[0], M[1], M[2], kx0, nkx, d.kind, d.alpha,
                                                   d.beta, 1.0, c->tw.p, i, ilog2c(c->T3),
                                                   (int)c->rchunk);
            VC_CUDA(c, cudaEventRecord(ev[3], st));
            count_launch(c, 6);
        }
        // the build grid is the largest transient (C5: 69 GB): keep it for reuse only when
        // small, so that the pass buffers allocated next fit beside the kernel tables
        if (G.bytes() > ((size_t)8 << 30)) {
            G.reset();
            Ko.reset();
        }
        }  // !reuse
        VC_CUDA(c, cudaGetLastError());
        if (!TK.on) c->kt_key = key;
    }
    tr.mark("kernel tables enqueued");
    if (TK.on) {
        vc_status ts = tk_hit ? tucker_from_cache(c) : tucker_compress(c);
        if (ts != VC_OK) return ts;
        if (tk_hit) {
            TK.cache = 1;
        } else {
            c->Rt.reset();  // P3 reads the compressed tables only
            if (o->tucker_cache && *o->tucker_cache) tucker_save(c, o->tucker_cache, tk_key);
        }
        tr.mark("tucker tables");
    }
    // ---- spatial partition: rank p owns a contiguous range of preconditioner
    // box rows along y, so every R_BD block stays on one rank; window row y -> rank (monotone)
    int EY = 1;
    for (int b = 0; b < 3; ++b) EY = std::max(EY, c->ext_in[b][1]);
    for (int f = 0; f < c->nf; ++f) EY = std::max(EY, c->f[f].ext[1]);
    const int W = c->world, rk = c->rank;
    {
        plan_row_slabs(W, c->ny, lo[1], EY, c->box[1], c->ya, &c->own_nb, &c->own_b0, &c->own_nbr);
        c->own_Nv = c->box[1];
        for (int q = 0; q < W; ++q) {
            auto cnt = [&](int e) { return std::max(0, std::min(c->ya[q + 1], e) - c->ya[q]); };
            for (int b = 0; b < 3; ++b) c->nr[q][b] = cnt(c->ext_in[b][1]);
            for (int f = 0; f < 6; ++f) c->nr[q][3 + f] = f < c->nf ? cnt(c->f[f].ext[1]) : 0;
        }
    }
    // ---- pass buffers.  A: P1 -> P2 blocks [sender][source][plane][rows][own kx] (recv 1),
    // later P4 -> P5 blocks [sender][field][plane][own rows][sender kx] (recv 2); S: blocks for
    // peers (send 1, later send 2); B: X2 tile-major; C: X3.
    auto nkxq = [&](int q) { return c->kxa[q + 1] - c->kxa[q]; };
    c->lgtk = ilog2c(p2_tile(My));  // FY<My>::T, P2's kx tile width
    c->lgt4 = ilog2c(p4_tile(My));  // FYS<My, kP4KB>::T, P4's
    size_t nR1 = 0, nR2 = 0, nS1 = 0, nS2 = 0, nBt = 0, nC = 0;
    for (int p = 0; p < W; ++p)
        for (int b = 0; b < 3; ++b) {
            c->offR1[p][b] = nR1;
            // one rank: kx-tile-major X1 padded to whole P2 tiles
            const size_t nkxp = W == 1 ? (size_t)((nkx + (1 << c->lgtk) - 1) >> c->lgtk) << c->lgtk : nkx;
            nR1 += (size_t)c->nzin[b] * c->nr[p][b] * nkxp;
        }
    for (int q = 0; q < W; ++q)
        for (int f = 0; f < c->nf; ++f) {
            c->offR2[q][f] = nR2;
            // one rank: row-pair blocked (P5 pairs rows at absolute (2m, 2m+1))
            const int s5 = c->lo[1] & 1;
            nR2 += (size_t)c->nzout[f] * nkxq(q) *
                   (W == 1 ? (size_t)2 * ((c->nr[rk][3 + f] + s5 + 1) >> 1) : (size_t)c->nr[rk][3 + f]);
        }
    for (int q = 0; q < W; ++q)
        for (int b = 0; b < 3; ++b) {
            c->offS1[q][b] = nS1;
            if (q != rk) nS1 += (size_t)c->nzin[b] * c->nr[rk][b] * nkxq(q);
        }
    for (int p = 0; p < W; ++p)
        for (int f = 0; f < c->nf; ++f) {
            c->offS2[p][f] = nS2;
            if (p != rk) nS2 += (size_t)c->nzout[f] * c->nr[p][3 + f] * nkx;
        }
    for (int b = 0; b < 3; ++b) {
        // tile-major, padded; direct-z: one stacked-plane array for the three sources (k_p3m)
        c->offB[b] = c->zdirect ? 0 : nBt;
        if (!c->zdirect || b == 0)
            nBt += (size_t)(My / 2 + 1) * c->nt3 * 2 * (c->zdirect ? c->p3m_nzt : c->nzin[b]) * c->T3;
    }
    for (int f = 0; f < c->nf; ++f) {
        c->offC[f] = nC;
        nC += (size_t)c->nzout[f] * My * ((size_t)((nkx + (1 << c->lgt4) - 1) >> c->lgt4) << c->lgt4);
    }
    // batched matvec (NEXT-3): one rank and at least two conductors; as many column copies of
    // the pass buffers as the free memory comfortably holds (<= kMaxB)
    c->colA = std::max<size_t>(1, std::max(nR1, nR2));
    c->colB = std::max<size_t>(1, nBt);
    c->colC = std::max<size_t>(1, nC);
    // (several ranks too, round 2: the pass kernels offset every block by the column, the
    // all-to-alls run per column and the lockstep solver sums its dot products over ranks).
    // Multi-rank batching needs the direct-z P3 (z-FFT mode runs P3 column by column anyway).
    c->colS = W > 1 ? std::max<size_t>(1, std::max(nS1, nS2)) : 0;
    c->nbmax = 1;
    const int nbw = std::min(kMaxB, c->m);
    const bool want_batch = c->m >= 2 && !(o && o->no_batch) && (W == 1 || c->zdirect);
    if (want_batch && c->bufA.cap >= c->colA * nbw && c->bufB.cap >= c->colB * nbw &&
        c->bufC.cap >= c->colC * nbw && c->bufS.cap >= c->colS * nbw) {
        c->nbmax = nbw;  // the buffers already hold nbw columns (no memory query: it can stall
                         // behind the kernel-table work just enqueued)
    } else if (want_batch) {
        size_t fr = 0, totm = 0;
        cudaMemGetInfo(&fr, &totm);
        const size_t percol = sizeof(double2) * (c->colA + c->colB + c->colC + c->colS);
        const size_t have = c->bufA.bytes() + c->bufB.bytes() + c->bufC.bytes() + c->bufS.bytes();
        while (c->nbmax < std::min(kMaxB, c->m) && (c->nbmax + 1) * percol <= (fr + have) / 3) ++c->nbmax;
    }
    VC_CUDA(c, c->bufA.alloc(c->colA * c->nbmax));
    VC_CUDA(c, c->bufB.alloc(c->colB * c->nbmax));
    VC_CUDA(c, c->bufC.alloc(c->colC * c->nbmax));
    if (W > 1) VC_CUDA(c, c->bufS.alloc(c->colS * c->nbmax));
    else c->bufS.reset();
    // all-to-all block tables (bytes; the self block is written in place by P1 / P4)
    for (int e = 0; e < 2; ++e) {
        c->a2a_send[e].assign(W, nullptr);
        c->a2a_recv[e].assign(W, nullptr);
        c->a2a_sb[e].assign(W, 0);
        c->a2a_rb[e].assign(W, 0);
    }
    for (int q = 0; q < W && W > 1; ++q) {
        size_t s1 = 0, r1 = 0, s2 = 0, r2 = 0;
        for (int b = 0; b < 3; ++b) {
            s1 += (size_t)c->nzin[b] * c->nr[rk][b] * nkxq(q);
            r1 += (size_t)c->nzin[b] * c->nr[q][b] * nkx;
        }
        for (int f = 0; f < c->nf; ++f) {
            s2 += (size_t)c->nzout[f] * c->nr[q][3 + f] * nkx;
            r2 += (size_t)c->nzout[f] * c->nr[rk][3 + f] * nkxq(q);
        }
        c->a2a_send[0][q] = c->bufS.p + c->offS1[q][0];
        c->a2a_recv[0][q] = c->bufA.p + c->offR1[q][0];
        c->a2a_send[1][q] = c->bufS.p + c->offS2[q][0];
        c->a2a_recv[1][q] = c->bufA.p + (c->nf ? c->offR2[q][0] : 0);
        if (q != rk) {
            c->a2a_sb[0][q] = 16 * s1;
            c->a2a_rb[0][q] = 16 * r1;
            c->a2a_sb[1][q] = 16 * s2;
            c->a2a_rb[1][q] = 16 * r2;
        }
    }
    {
        vc_status ps = partition_build(c);
        if (ps != VC_OK) return ps;
    }
    // algorithmic bytes of this rank's share of each pass: complex128 reads +
    // writes of the pass arrays, kernel spectra read once, panel vectors and slot maps once.
    const double cb = 16.0;
    double slots = 0, nX1 = 0, nX1r = 0, nB = 0, nX4 = 0, nX4r = 0;
    for (int b = 0; b < 3; ++b) {
        slots += (double)c->ext_in[b][0] * c->nr[rk][b] * c->nzin[b];
        nX1 += (double)c->nzin[b] * c->nr[rk][b] * Kx;         // P1 writes (own rows, all kx)
        nX1r += (double)c->nzin[b] * c->ext_in[b][1] * nkx;    // P2 reads (all rows, own kx)
        nB += (double)c->nzin[b] * My * nkx;
    }
    double slots_out = 0;
    for (int f = 0; f < c->nf; ++f) {
        slots_out += (double)c->f[f].ext[0] * c->nr[rk][3 + f] * c->nzout[f];
        nX4 += (double)c->nzout[f] * c->f[f].ext[1] * nkx;    // P4 writes
        nX4r += (double)c->nzout[f] * c->nr[rk][3 + f] * Kx;  // P5 reads
    }
    const double NL = (double)c->NL;
    double ndl = (double)c->Nd;  // one rank: every dielectric panel
    if (W > 1) {
        ndl = 0;
        for (int64_t i = 0; i < c->NL; ++i) ndl += c->h_cid[c->h_gidx[i]] == 0;
    }
    c->bytes_pass[0] = cb * nX1 + 4.0 * slots + 8.0 * NL;
    c->bytes_pass[1] = cb * (nX1r + nB);
    c->bytes_k3 = TK.on ? 8.0 * (double)TK.resident()
                        : 8.0 * (double)nkx * (My / 2 + 1) * (c->zdirect ? c->ZU : Mz / 2 + 1) * c->nblk;
    c->stats.spectra_doubles = TK.on ? TK.resident() : (int64_t)c->Rt.n;
    c->stats.tucker_cache = TK.cache;
    double tkerr = 0;
    for (double e : TK.err) tkerr = std::max(tkerr, e);
    c->stats.tucker_err = TK.on ? tkerr : 0.0;
    c->bytes_pass[2] = cb * (nB + (double)nC) + c->bytes_k3;
    c->bytes_pass[3] = cb * ((double)nC + nX4);
    c->bytes_pass[4] = cb * nX4r + 4.0 * slots_out + 8.0 * NL + (8.0 + 8.0 + 1.0) * ndl + 1.0 * NL;
    double tot = 0;
    for (int p = 0; p < 5; ++p) {
        c->stats.bytes_pass[p] = c->bytes_pass[p];
        tot += c->bytes_pass[p];
    }
    c->stats.bytes_matvec = tot;
    tr.mark("buffers + partition + bytes");
    return VC_OK;
}

// rank owning absolute slot row yabs (along y): by preconditioner box row, contiguous ranges
int row_owner_abs(const vc_ctx* c, int yabs) {
    return row_owner_plan(c->world, c->own_Nv, c->own_nb, c->own_b0, c->own_nbr, yabs);
}

__global__ void k_local_panels(int64_t nl, const int64_t* __restrict__ gidx,
                               const int8_t* __restrict__ info, const double* __restrict__ ibar,
                               const double* __restrict__ fc, const int32_t* __restrict__ cid,
                               const int8_t* __restrict__ axis, const int32_t* __restrict__ si,
                               const int32_t* __restrict__ sj, const int32_t* __restrict__ sk,
                               int8_t* __restrict__ linfo, double* __restrict__ libar,
                               double* __restrict__ lfc, int32_t* __restrict__ lcid,
                               int32_t* __restrict__ sm0, int32_t* __restrict__ sm1,
                               int32_t* __restrict__ sm2, int nx, int ny) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nl;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = gidx[i];
        linfo[i] = info[g];
        libar[i] = ibar[g];
        lfc[i] = fc[g];
        lcid[i] = cid[g];
        const int a = axis[g];
        const int gx = nx + (a == 0), gy = ny + (a == 1);
        int32_t* sm = a == 0 ? sm0 : (a == 1 ? sm1 : sm2);
        const int inf = info[g];  // same encoding as the global map (common.cuh kSlot*)
        sm[((int64_t)sk[g] * gy + sj[g]) * gx + si[g]] =
            (int32_t)i | ((inf & 1) ? kSlotDiel : 0) | ((inf & 3) == 3 ? kSlotNeg : 0);
    }
}

// This rank's panels: canonical order restricted to the panels whose slot row it owns, and
// slot maps to local indices (world = 1: the global arrays are used as they are).
vc_status partition_build(vc_ctx* c) {
    mirror_wait(c);
    c->h_gidx.clear();
    if (c->world == 1) {
        c->NL = c->N;
        return VC_OK;
    }
    for (int64_t p = 0; p < c->N; ++p)
        if (row_owner_abs(c, c->h_sj[p]) == c->rank) c->h_gidx.push_back(p);
    c->NL = (int64_t)c->h_gidx.size();
    const int64_t nl = c->NL;
    cudaStream_t st = c->stream;
    PanelsLocal& L = c->lp;
    VC_CUDA(c, L.gidx.alloc(std::max<int64_t>(1, nl)));
    VC_CUDA(c, L.info.alloc(std::max<int64_t>(1, nl)));
    VC_CUDA(c, L.ibar.alloc(std::max<int64_t>(1, nl)));
    VC_CUDA(c, L.fc.alloc(std::max<int64_t>(1, nl)));
    VC_CUDA(c, L.cid.alloc(std::max<int64_t>(1, nl)));
    for (int a = 0; a < 3; ++a) {
        const size_t n = (size_t)(c->nx + (a == 0)) * (c->ny + (a == 1)) * (c->nz + (a == 2));
        VC_CUDA(c, L.slotmap[a].alloc(n));
        VC_CUDA(c, cudaMemsetAsync(L.slotmap[a].p, 0xff, 4 * n, st));
    }
    if (nl) {
        VC_CUDA(c, cudaMemcpyAsync(L.gidx.p, c->h_gidx.data(), 8 * nl, cudaMemcpyHostToDevice, st));
        const PanelsDev& P = c->pan;
        k_local_panels<<<(unsigned)std::min<int64_t>((nl + 255) / 256, 148 * 8), 256, 0, st>>>(
            nl, L.gidx.p, P.info.p, P.ibar.p, P.fc.p, P.cid.p, P.axis.p, P.si.p, P.sj.p, P.sk.p,
            L.info.p, L.ibar.p, L.fc.p, L.cid.p, L.slotmap[0].p, L.slotmap[1].p, L.slotmap[2].p,
            c->nx, c->ny);
        count_launch(c);
    }
    VC_CUDA(c, cudaStreamSynchronize(st));
    VC_CUDA(c, cudaGetLastError());
    return VC_OK;
}

static MV make_mv(vc_ctx* c, const double* x, double* y) {
    MV mv;
    memset(&mv, 0, sizeof(mv));
    mv.Mx = c->M[0];
    mv.My = c->M[1];
    mv.Mz = c->M[2];
    mv.Kx = c->Kx;
    const bool loc = c->world > 1;
    for (int t = 0; t < 3; ++t) mv.lo[t] = c->lo[t];
    for (int a = 0; a < 3; ++a) {
        mv.G[a][0] = c->nx + (a == 0);
        mv.G[a][1] = c->ny + (a == 1);
        mv.G[a][2] = c->nz + (a == 2);
        for (int t = 0; t < 3; ++t) mv.ext_in[a][t] = c->ext_in[a][t];
        mv.slotmap[a] = loc ? c->lp.slotmap[a].p : c->pan.slotmap[a].p;
        mv.X2[a] = c->bufB.p + c->offB[a];
    }
    mv.nf = c->nf;
    for (int f = 0; f < 6; ++f) {
        for (int b = 0; b < 3; ++b) mv.blk[f][b] = c->blk[f][b];
        if (f < c->nf) {
            mv.fkind[f] = c->f[f].kind;
            mv.faxis[f] = c->f[f].axis;
            for (int t = 0; t < 3; ++t) mv.ext_out[f][t] = c->f[f].ext[t];
            mv.X3[f] = c->bufC.p + c->offC[f];
        }
    }
    mv.x = x;
    mv.y = y;
    mv.nb = 1;
    mv.xs[0] = x;
    mv.ys[0] = y;
    mv.colA = (int64_t)c->colA;
    mv.colB = (int64_t)c->colB;
    mv.colC = (int64_t)c->colC;
    mv.colS = (int64_t)c->colS;
    mv.info = loc ? c->lp.info.p : c->pan.info.p;
    mv.ibar = loc ? c->lp.ibar.p : c->pan.ibar.p;
    mv.Rt = c->Rt.p;
    mv.rchunk = (int)c->rchunk;
    mv.T3 = c->T3;
    mv.lgT3 = ilog2c(c->T3);
    mv.nblk = c->nblk;
    mv.tw = c->tw.p;
    mv.planes = c->planes.p;
    mv.ZL = c->ZL;
    mv.zdirect = c->zdirect;
    mv.ZU = c->ZU;
    mv.rs1 = c->rs1;
    mv.tk = c->tk.on ? 1 : 0;
    if (mv.tk) {
        const Tucker& T = c->tk;
        mv.tk_u1 = T.U1f.p;
        mv.tk_w = T.Wf.p;
        mv.tk_u1t = T.u1t;
        mv.tk_wq = T.wq;
        mv.tk_nc = T.nc;
        mv.tk_items = T.nblk * T.nc;
        for (int b = 0; b < 16; ++b) {
            mv.tk_nkc[b] = b < T.nblk ? T.nkc[b] : 0;
            mv.tk_u1o[b] = b < T.nblk ? T.u1o[b] : 0;
            mv.tk_wo[b] = b < T.nblk ? T.wo[b] : 0;
        }
    }
    for (int b = 0; b < 3; ++b) {
        mv.x2nz[b] = c->zdirect ? c->p3m_nzt : c->nzin[b];
        mv.x2zo[b] = c->zdirect ? c->p3m_zoff[b] : 0;
    }
    mv.p3m_tab = c->p3m_tab.p;
    mv.s0 = 0;
    mv.s1 = 3;
    mv.f0 = 0;
    mv.f1 = c->nf;
    mv.p3m_nneg = c->zdirect ? c->p3m_nneg : 0;
    mv.p3m_oddmask = c->p3m_oddmask;
    mv.p3m_neg = c->p3m_tab.p + c->p3m_negoff;
    mv.p3m_nzt = c->p3m_nzt;
    mv.p3m_kc = c->p3m_kc;
    mv.p3m_mct = c->p3m_mct;
    mv.p3m_nst = c->p3m_nst;
    for (int b = 0; b < 3; ++b) mv.nzin[b] = c->nzin[b];
    for (int f = 0; f < 6; ++f) mv.nzout[f] = f < c->nf ? c->nzout[f] : 0;
    const int W = c->world, r = c->rank;
    mv.W = W;
    mv.rank = r;
    for (int q = 0; q <= kMaxRanks; ++q) {
        mv.ya[q] = q <= W ? c->ya[q] : INT32_MAX;
        mv.kxa[q] = q <= W ? c->kxa[q] : INT32_MAX;
    }
    for (int q = 0; q < W; ++q)
        for (int g = 0; g < 9; ++g) mv.nr[q][g] = c->nr[q][g];
    mv.lgtk = c->lgtk;
    mv.lgt4 = c->lgt4;
    mv.kx0 = c->kxa[r];
    mv.nkx = c->kxa[r + 1] - c->kxa[r];
    for (int q = 0; q < W; ++q) {
        for (int b = 0; b < 3; ++b) {
            mv.S1[q][b] = q == r ? c->bufA.p + c->offR1[r][b] : c->bufS.p + c->offS1[q][b];
            mv.R1[q][b] = c->bufA.p + c->offR1[q][b];
        }
        for (int f = 0; f < c->nf; ++f) {
            mv.S2[q][f] = q == r ? c->bufA.p + c->offR2[r][f] : c->bufS.p + c->offS2[q][f];
            mv.R2[q][f] = c->bufA.p + c->offR2[q][f];
        }
    }
    return mv;
}

static vc_status matvec_run(vc_ctx* c, const MV& mv);

vc_status matvec_batch_dev(vc_ctx* c, int nb, const double* const* d_x, double* const* d_y) {
    for (int c0 = 0; c0 < nb; c0 += c->nbmax) {
        const int n1 = std::min(c->nbmax, nb - c0);
        if (n1 == 1) {
            vc_status s = matvec_dev(c, d_x[c0], d_y[c0]);
            if (s) return s;
            continue;
        }
        MV mv = make_mv(c, d_x[c0], d_y[c0]);
        mv.nb = n1;
        for (int i = 0; i < n1; ++i) {
            mv.xs[i] = d_x[c0 + i];
            mv.ys[i] = d_y[c0 + i];
        }
        vc_status s = matvec_run(c, mv);
        if (s) return s;
    }
    return VC_OK;
}

vc_status matvec_dev(vc_ctx* c, const double* d_x, double* d_y) {
    return matvec_run(c, make_mv(c, d_x, d_y));
}

// Accumulate the queued matvec timing records into c->stats (one wait for the newest event).
vc_status timing_resolve(vc_ctx* c) {
    Timing& T = c->timing;
    if (T.recs.empty()) return VC_OK;
    VC_CUDA(c, cudaEventSynchronize(T.pool[T.recs.back().base + 11]));
    float ms = 0;
    for (const Timing::Rec& r : T.recs) {
        const cudaEvent_t* ev = T.pool.data() + r.base;
        VC_CUDA(c, cudaEventElapsedTime(&ms, ev[0], ev[11]));
        c->stats.ms_matvec += ms;
        if (r.det) {
            for (int p = 0; p < 5; ++p) {
                VC_CUDA(c, cudaEventElapsedTime(&ms, ev[1 + p], ev[6 + p]));
                c->stats.ms_pass[p] += ms;
            }
            if (r.comm)
                for (int e = 0; e < 2; ++e) {
                    VC_CUDA(c, cudaEventElapsedTime(&ms, ev[12 + e], ev[14 + e]));
                    c->stats.ms_comm += ms;
                }
        }
    }
    T.recs.clear();
    T.used = 0;
    return VC_OK;
}

// Several ranks: the two all-to-alls are split by source (after P1) and by field
// (after P4) and run on the comm stream, so each chunk's exchange overlaps the transforms of the
// chunks after it: P1(b) -> a2a(b) || P1(b + 1); P2(b) waits for a2a(b) only; the same for
// P4(f) -> a2a(f) -> P5(f).  The arithmetic is that of the one-launch passes (each pencil is
// transformed by the same plan), so the partitioned matvec stays bitwise equal to one rank's.
static vc_status a2a_chunk(vc_ctx* c, int e, int g, int col, cudaStream_t cs) {
    const int W = c->world, rk = c->rank, nkx = c->kxa[rk + 1] - c->kxa[rk];
    std::vector<const void*> sp(W, nullptr);
    std::vector<void*> rp(W, nullptr);
    std::vector<size_t> sb(W, 0), rb(W, 0);
    for (int q = 0; q < W; ++q) {
        if (q == rk) continue;
        const int nkq = c->kxa[q + 1] - c->kxa[q];
        if (e == 0) {  // source g: [sender][source][plane][rows][dest kx] blocks
            sp[q] = c->bufS.p + c->offS1[q][g] + (size_t)col * c->colS;
            rp[q] = c->bufA.p + c->offR1[q][g] + (size_t)col * c->colA;
            sb[q] = 16 * (size_t)c->nzin[g] * c->nr[rk][g] * nkq;
            rb[q] = 16 * (size_t)c->nzin[g] * c->nr[q][g] * nkx;
        } else {  // field g: [field][plane][dest rows][own kx] blocks
            sp[q] = c->bufS.p + c->offS2[q][g] + (size_t)col * c->colS;
            rp[q] = c->bufA.p + c->offR2[q][g] + (size_t)col * c->colA;
            sb[q] = 16 * (size_t)c->nzout[g] * c->nr[q][3 + g] * nkx;
            rb[q] = 16 * (size_t)c->nzout[g] * c->nr[rk][3 + g] * nkq;
        }
    }
    return comm_alltoall(c, sp, sb, rp, rb, cs);
}

static vc_status matvec_chunked(vc_ctx* c, const MV& mv, const cudaEvent_t* ev, bool det) {
    cudaStream_t st = c->stream;
    if (!c->cstream) VC_CUDA(c, cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
    if (!c->cev_ok) {
        for (auto& e : c->cev) VC_CUDA(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->cev_ok = true;
    }
    cudaStream_t cs = c->cstream;
    cudaEvent_t* made = c->cev;      // [0..8]: chunk produced on the compute stream
    cudaEvent_t* moved = c->cev + 9; // [9..17]: chunk exchanged on the comm stream
    // the comm stream starts after everything before this matvec (its buffers' previous users)
    VC_CUDA(c, cudaEventRecord(made[8], st));
    VC_CUDA(c, cudaStreamWaitEvent(cs, made[8], 0));
    for (int ph = 0; ph < 2; ++ph) {  // ph 0: P1 -> a2a #1 -> P2; ph 1: P4 -> a2a #2 -> P5
        const int ng = ph == 0 ? 3 : c->nf;
        const int pa = ph == 0 ? 0 : 3, pb = ph == 0 ? 1 : 4;  // producing / consuming pass
        if (ph == 1) {  // P3 between the phases
            if (det) VC_CUDA(c, cudaEventRecord(ev[1 + 2], st));
            VC_CUDA(c, launch_p3(mv, st));
            if (det) VC_CUDA(c, cudaEventRecord(ev[6 + 2], st));
        }
        if (det) VC_CUDA(c, cudaEventRecord(ev[1 + pa], st));
        if (det) VC_CUDA(c, cudaEventRecord(ev[12 + ph], cs));
        for (int g = 0; g < ng; ++g) {
            MV m = mv;
            if (ph == 0) { m.s0 = g; m.s1 = g + 1; } else { m.f0 = g; m.f1 = g + 1; }
            VC_CUDA(c, ph == 0 ? launch_p1(m, st) : launch_p4s(m, st));
            VC_CUDA(c, cudaEventRecord(made[g], st));
            VC_CUDA(c, cudaStreamWaitEvent(cs, made[g], 0));
            for (int i = 0; i < mv.nb; ++i) {  // one exchange per batch column
                vc_status s = a2a_chunk(c, ph, g, i, cs);
                if (s) return s;
            }
            VC_CUDA(c, cudaEventRecord(moved[g], cs));
        }
        if (det) VC_CUDA(c, cudaEventRecord(ev[6 + pa], st));
        if (det) VC_CUDA(c, cudaEventRecord(ev[14 + ph], cs));
        if (det) VC_CUDA(c, cudaEventRecord(ev[1 + pb], st));
        for (int g = 0; g < ng; ++g) {
            MV m = mv;
            if (ph == 0) { m.s0 = g; m.s1 = g + 1; } else { m.f0 = g; m.f1 = g + 1; }
            VC_CUDA(c, cudaStreamWaitEvent(st, moved[g], 0));
            VC_CUDA(c, ph == 0 ? launch_p2(m, st) : launch_p5(m, st));
        }
        if (det) VC_CUDA(c, cudaEventRecord(ev[6 + pb], st));
    }
    return VC_OK;
}

static vc_status matvec_run(vc_ctx* c, const MV& mv) {
    cudaStream_t st = c->stream;
    Timing& T = c->timing;
    const cudaEvent_t* ev = nullptr;
    if (T.on) {
        if ((int)T.recs.size() >= Timing::kMaxRecs) {
            vc_status s = timing_resolve(c);
            if (s) return s;
        }
        while ((int)T.pool.size() < T.used + Timing::kEvPerMv) {
            cudaEvent_t e;
            VC_CUDA(c, cudaEventCreate(&e));
            T.pool.push_back(e);
        }
        T.recs.push_back({T.used, mv.nb, T.detail, c->world > 1});
        ev = T.pool.data() + T.used;
        T.used += Timing::kEvPerMv;
    }
    const bool det = ev && T.detail;
    if (ev) VC_CUDA(c, cudaEventRecord(ev[0], st));
    for (int i = 0; i < mv.nb; ++i)
        k_yinit<<<std::max<int64_t>(1, std::min<int64_t>((c->NL + 255) / 256, 1184)), 256, 0, st>>>(
            mv.ys[i], mv.xs[i], mv.ibar, c->NL);
    cudaError_t (*launch[5])(const MV&, cudaStream_t) = {launch_p1, launch_p2, launch_p3,
                                                         launch_p4s, launch_p5};
    if (c->world == 1) {
        for (int p = 0; p < 5; ++p) {
            if (det) VC_CUDA(c, cudaEventRecord(ev[1 + p], st));
            VC_CUDA(c, launch[p](mv, st));
            if (det) VC_CUDA(c, cudaEventRecord(ev[6 + p], st));
        }
    } else {
        vc_status s = matvec_chunked(c, mv, ev, det);
        if (s) return s;
    }
    if (ev) VC_CUDA(c, cudaEventRecord(ev[11], st));
    count_launch(c, (c->world > 1 ? 7 + 2 * c->nf : 5) + mv.nb);  // (chunked: 3 + 3 + 1 + 2 nf)
    c->stats.n_matvec += mv.nb;
    for (int p = 0; p < 5; ++p) {
        c->stats.n_pass[p] += 1;
        // a batched P3 launch reads the kernel spectra once for its columns (z-FFT mode and
        // oversized tiles run P3 column by column: nb reads)
        const bool shared_k = p == 2 && mv.nb > 1 && p3m_batched(mv);
        c->stats.bytes_moved[p] += mv.nb * c->bytes_pass[p] - (shared_k ? (mv.nb - 1) * c->bytes_k3 : 0.0);
    }
    return VC_OK;
}

// device times of the last kernel-table build (call after the stream has drained)
void kernel_table_times(vc_ctx* c) {
    float t_kgen = 0, t_fft = 0, ms = 0;
    for (int i = 0; i < c->kev_n; ++i) {
        const cudaEvent_t* ev = c->kev.data() + 4 * (size_t)i;
        if (cudaEventElapsedTime(&ms, ev[0], ev[1]) == cudaSuccess) t_kgen += ms;
        if (cudaEventElapsedTime(&ms, ev[1], ev[3]) == cudaSuccess) t_fft += ms;
    }
    c->stats.ms_kgen = t_kgen;
    c->stats.ms_kfft = t_fft;
}

vc_status debug_kernel_entries(vc_ctx* c, int n, const int32_t* kind, const int32_t* a,
                               const int32_t* b, const int32_t* d, double* out) {
    DevBuf<int32_t> dk, da, db, dd;
    DevBuf<double> dout;
    VC_CUDA(c, dk.alloc(n));
    VC_CUDA(c, da.alloc(n));
    VC_CUDA(c, db.alloc(n));
    VC_CUDA(c, dd.alloc(3 * (size_t)n));
    VC_CUDA(c, dout.alloc(n));
    cudaStream_t st = c->stream;
    VC_CUDA(c, cudaMemcpyAsync(dk.p, kind, 4 * (size_t)n, cudaMemcpyHostToDevice, st));
    VC_CUDA(c, cudaMemcpyAsync(da.p, a, 4 * (size_t)n, cudaMemcpyHostToDevice, st));
    VC_CUDA(c, cudaMemcpyAsync(db.p, b, 4 * (size_t)n, cudaMemcpyHostToDevice, st));
    VC_CUDA(c, cudaMemcpyAsync(dd.p, d, 12 * (size_t)n, cudaMemcpyHostToDevice, st));
    k_debug_kappa<<<(n + 127) / 128, 128, 0, st>>>(n, dk.p, da.p, db.p, dd.p, dout.p);
    count_launch(c);
    VC_CUDA(c, cudaMemcpyAsync(out, dout.p, 8 * (size_t)n, cudaMemcpyDeviceToHost, st));
    VC_CUDA(c, cudaStreamSynchronize(st));
    VC_CUDA(c, cudaGetLastError());
    return VC_OK;
}

vc_status debug_fft(vc_ctx* c, int L, int nl, double* data, int dir) {
    if (L < 8 || L > kMaxL || (L & (L - 1))) return set_err(c, VC_ERR_INPUT, "L must be a power of two in [8, 4096]");
    cudaStream_t st = c->stream;
    if (!c->tw.p) {
        VC_CUDA(c, c->tw.alloc(kTabN));
        k_twiddles<<<(kTabN + 255) / 256, 256, 0, st>>>(c->tw.p);
        count_launch(c);
    }
    DevBuf<double2> d;
    VC_CUDA(c, d.alloc((size_t)L * nl));
    VC_CUDA(c, cudaMemcpyAsync(d.p, data, 16 * (size_t)L * nl, cudaMemcpyHostToDevice, st));
    VC_CUDA(c, launch_fft_lines(d.p, L, nl, dir > 0, c->tw.p, st));
    count_launch(c);
    VC_CUDA(c, cudaMemcpyAsync(data, d.p, 16 * (size_t)L * nl, cudaMemcpyDeviceToHost, st));
    VC_CUDA(c, cudaStreamSynchronize(st));
    return VC_OK;
}

}  // namespace vc
