// tucker.cu -- Tucker-compressed direct-z kernel spectra (§II.C,
// Eq. 13) and their install-time cache file (NEXT-4: P:119).
//
// The paper stores each Toeplitz tensor compressed as a Tucker core times factor matrices and
// restores it before every convolution.  Here the compressed object is the folded, phase-
// stripped direct-z spectrum table of each kernel block, X_b[kx][q][u] (this
// rank's kx, q = |ky|, z offset u), which is what P3 reads:
//   X_b ~ S_b x1 U1_b x2 U2_b,   U1_b: nkx x r1 and U2_b: nq x r2 with orthonormal columns,
//                                S_b = X_b x1 U1_b^T x2 U2_b^T  (r1 x r2 x ZU; the short u mode
//                                is kept full).
// Factors: truncated column-pivoted Gram-Schmidt on each mode unfolding (greedy: the fibre of
// largest residual norm joins the basis, re-orthogonalised twice, and the residual is deflated
// in place), stopped when the residual energy -- summed directly from the deflated unfolding,
// not by subtraction -- is <= (10^-d)^2 / 2 of ||X_b||^2.  The two projections then leave
// ||X_b - X~_b||_F <= 10^-d ||X_b||_F (HOSVD error bound: the mode errors add in squares); the
// error actually reached is measured against the exact table before it is freed.  This is the
// paper's truncated HOSVD (Eq. 13) with a rank-revealing QR in place of the SVD: it reaches the
// same bound with a few more ranks and needs no eigen-solver.
//
// P3 (p3m.cu, TK instantiation) rebuilds every tile's kernel rows on the FP64 tensor cores:
//   K_b[kx][u] = sum_i U1_b[kx][i] W_b[q][i][u],  W_b[q] = S_b x2 U2_b[q]  (r1 x ZU),
// from two resident fragment tables (ctx.h vc::Tucker): U1f, the DMMA A fragments of 8 kx x 4
// ranks, streamed per tile; and Wf, the B fragments of W_b[q] for all blocks, loaded into shared
// memory once per q (the Tucker P3 walks its tiles q-major in contiguous ranges).
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ctx.h"
#include "mv.cuh"

namespace vc {

namespace {

constexpr int kTkNT = 256;
constexpr int kTkMaxRank = 192;

// tile-major direct-z table index (operator.cu rt_idx, T3 = kMmaT): [q][kx tile][t][b * ZU + u]
__device__ __forceinline__ int64_t tk_rt(int q, int kx, int b, int u, int ZU, int nt3, int RS1) {
    return (((int64_t)q * nt3 + (kx >> 3)) * kMmaT + (kx & 7)) * RS1 + (int64_t)b * ZU + u;
}

// dense copy [b][kx][q][u] of every block of the tile-major table
__global__ void k_tk_gather(double* __restrict__ R, const double* __restrict__ Rt, int nkx, int nq, int ZU,
                            int nt3, int RS1, int nblk) {
    const int64_t per = (int64_t)nkx * nq * ZU, tot = per * nblk;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(e / per);
        const int64_t r = e - b * per;
        const int kx = (int)(r / ((int64_t)nq * ZU));
        const int q = (int)((r / ZU) % nq), u = (int)(r % ZU);
        R[e] = Rt[tk_rt(q, kx, b, u, ZU, nt3, RS1)];
    }
}

// block-wide reductions over kTkNT threads: sum, and (max, smallest index of the max)
__device__ double blk_sum(double v, double* sh) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0;
    for (int w = 0; w < kTkNT / 32; ++w) s += sh[w];
    return s;
}
__device__ void blk_argmax(double& m, long long& a, double* shm, long long* sha) {
    for (int o = 16; o; o >>= 1) {
        const double m2 = __shfl_xor_sync(0xffffffffu, m, o);
        const long long a2 = __shfl_xor_sync(0xffffffffu, a, o);
        if (m2 > m || (m2 == m && a2 < a)) {
            m = m2;
            a = a2;
        }
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
        shm[threadIdx.x >> 5] = m;
        sha[threadIdx.x >> 5] = a;
    }
    __syncthreads();
    m = shm[0];
    a = sha[0];
    for (int w = 1; w < kTkNT / 32; ++w)
        if (shm[w] > m || (shm[w] == m && sha[w] < a)) {
            m = shm[w];
            a = sha[w];
        }
}

// Per block state st[4 b + {0: done, 1: basis size, 2: final rank, 3: ||X_b||^2}].
// One greedy step on every unfinished block, part 1: deflate the residual unfolding by the
// newest basis vector v (R_j -= v (v . R_j) for every column j; skipped at step 0) and compute
// the new column energies; each CTA leaves (max energy, its column, energy sum) in part.
// Element (i, j) of block b's unfolding sits at R[b * blkN + i * sI + (j / ZU) * sJ + j % ZU].
__global__ void __launch_bounds__(kTkNT) k_tk_cols(double* __restrict__ R, int64_t blkN, int I, int64_t J, int ZU,
                                                   int64_t sI, int64_t sJ, const double* __restrict__ vb,
                                                   const double* __restrict__ st, double* __restrict__ part) {
    extern __shared__ double v[];  // [I]
    __shared__ double shm[kTkNT / 32];
    __shared__ long long sha[kTkNT / 32];
    const int b = blockIdx.y;
    if (st[4 * b] != 0.0) return;
    const bool upd = st[4 * b + 1] > 0.5;
    if (upd)
        for (int i = threadIdx.x; i < I; i += kTkNT) v[i] = vb[(int64_t)b * I + i];
    __syncthreads();
    double* Rb = R + b * blkN;
    double mx = -1.0, sum = 0.0;
    long long arg = 0;
    for (int64_t j = blockIdx.x * (int64_t)kTkNT + threadIdx.x; j < J; j += (int64_t)gridDim.x * kTkNT) {
        double* col = Rb + (j / ZU) * sJ + (j % ZU);
        double w = 0.0;
        if (upd)
            for (int i = 0; i < I; ++i) w = fma(v[i], col[i * sI], w);
        double e = 0.0;
        for (int i = 0; i < I; ++i) {
            double r = col[i * sI];
            if (upd) {
                r = fma(-v[i], w, r);
                col[i * sI] = r;
            }
            e = fma(r, r, e);
        }
        sum += e;
        if (e > mx) {
            mx = e;
            arg = j;
        }
    }
    __shared__ double shs[kTkNT / 32];
    const double s = blk_sum(sum, shs);
    blk_argmax(mx, arg, shm, sha);
    if (threadIdx.x == 0) {
        double* p = part + ((int64_t)b * gridDim.x + blockIdx.x) * 3;
        p[0] = mx;
        p[1] = (double)arg;
        p[2] = s;
    }
}

// Part 2 (one CTA per block): stop when the residual energy is <= tol2 ||X_b||^2 (or nothing is
// left, or the rank cap is reached); else the pivot column, normalised, re-orthogonalised twice
// against the basis (classical Gram-Schmidt), becomes basis vector `it` (U[b][it][:]) and the v
// that part 1 deflates with next.
__global__ void __launch_bounds__(kTkNT) k_tk_pivot(const double* __restrict__ R, int64_t blkN, int I, int ZU,
                                                    int64_t sI, int64_t sJ, double* __restrict__ U, int rmax,
                                                    double* __restrict__ vb, double* __restrict__ st,
                                                    const double* __restrict__ part, int nparts, double tol2) {
    extern __shared__ double v[];  // [I] + h[rmax]
    double* h = v + I;
    __shared__ double shm[kTkNT / 32];
    __shared__ long long sha[kTkNT / 32];
    __shared__ double shs[kTkNT / 32];
    const int b = blockIdx.x;
    double* sb = st + 4 * b;
    if (sb[0] != 0.0) return;
    const int it = (int)sb[1];
    double mx = -1.0, sum = 0.0;
    long long arg = 0;
    for (int p = threadIdx.x; p < nparts; p += kTkNT) {
        const double* pp = part + ((int64_t)b * nparts + p) * 3;
        sum += pp[2];
        const long long a = (long long)pp[1];
        if (pp[0] > mx || (pp[0] == mx && a < arg)) {
            mx = pp[0];
            arg = a;
        }
    }
    sum = blk_sum(sum, shs);
    blk_argmax(mx, arg, shm, sha);
    const double norm2 = it == 0 ? sum : sb[3];
    const int cap = min(rmax, I);
    if (sum <= tol2 * norm2 || !(mx > 0.0) || it >= cap) {
        __syncthreads();
        if (threadIdx.x == 0) {
            sb[0] = 1.0;
            sb[2] = (double)it;
            if (it == 0) sb[3] = sum;
        }
        return;
    }
    const double* col = R + b * blkN + (arg / ZU) * sJ + (arg % ZU);
    const double inv = 1.0 / sqrt(mx);
    for (int i = threadIdx.x; i < I; i += kTkNT) v[i] = col[i * sI] * inv;
    __syncthreads();
    double* Ub = U + (int64_t)b * rmax * I;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int pass = 0; pass < 2; ++pass) {
        for (int k = warp; k < it; k += kTkNT / 32) {
            double d = 0.0;
            for (int i = lane; i < I; i += 32) d = fma(Ub[(int64_t)k * I + i], v[i], d);
            for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
            if (lane == 0) h[k] = d;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < I; i += kTkNT) {
            double s = v[i];
            for (int k = 0; k < it; ++k) s = fma(-h[k], Ub[(int64_t)k * I + i], s);
            v[i] = s;
        }
        __syncthreads();
    }
    double nn = 0.0;
    for (int i = threadIdx.x; i < I; i += kTkNT) nn = fma(v[i], v[i], nn);
    nn = blk_sum(nn, shs);
    const double sc = nn > 0.0 ? 1.0 / sqrt(nn) : 0.0;
    for (int i = threadIdx.x; i < I; i += kTkNT) {
        const double x = v[i] * sc;
        Ub[(int64_t)it * I + i] = x;
        vb[(int64_t)b * I + i] = x;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        sb[1] = (double)(it + 1);
        if (it == 0) sb[3] = sum;
    }
}

struct TkDims {
    int r1[16], r2[16];
};

// T1[b][i][q * ZU + u] = sum_kx U1[b][i][kx] X[b][kx][q][u] (mode-1 projection), 8 ranks per CTA row
__global__ void __launch_bounds__(kTkNT) k_tk_t1(double* __restrict__ T1, const double* __restrict__ X,
                                                 const double* __restrict__ U1, int r1max, int nkx, int64_t J,
                                                 TkDims d) {
    const int b = blockIdx.z, i0 = blockIdx.y * 8;
    if (i0 >= d.r1[b]) return;
    const int nr = min(8, d.r1[b] - i0);
    const double* Xb = X + (int64_t)b * nkx * J;
    const double* Ub = U1 + ((int64_t)b * r1max + i0) * nkx;
    for (int64_t j = blockIdx.x * (int64_t)kTkNT + threadIdx.x; j < J; j += (int64_t)gridDim.x * kTkNT) {
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int kx = 0; kx < nkx; ++kx) {
            const double x = Xb[(int64_t)kx * J + j];
#pragma unroll
            for (int r = 0; r < 8; ++r)
                if (r < nr) acc[r] = fma(__ldg(Ub + (int64_t)r * nkx + kx), x, acc[r]);
        }
        for (int r = 0; r < nr; ++r) T1[((int64_t)b * r1max + i0 + r) * J + j] = acc[r];
    }
}

// S[b][i][j][u] = sum_q U2[b][j][q] T1[b][i][q][u] (core), one (i, u) per thread, 8 ranks j per CTA row
__global__ void __launch_bounds__(kTkNT) k_tk_core(double* __restrict__ S, const double* __restrict__ T1,
                                                   const double* __restrict__ U2, int r1max, int r2max, int nq,
                                                   int ZU, TkDims d) {
    const int b = blockIdx.z, j0 = blockIdx.y * 8;
    if (j0 >= d.r2[b]) return;
    const int nr = min(8, d.r2[b] - j0);
    const int64_t J = (int64_t)nq * ZU;
    const int64_t n = (int64_t)d.r1[b] * ZU;
    for (int64_t e = blockIdx.x * (int64_t)kTkNT + threadIdx.x; e < n; e += (int64_t)gridDim.x * kTkNT) {
        const int i = (int)(e / ZU), u = (int)(e % ZU);
        const double* t = T1 + ((int64_t)b * r1max + i) * J + u;
        const double* Ub = U2 + ((int64_t)b * r2max + j0) * nq;
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int q = 0; q < nq; ++q) {
            const double x = t[(int64_t)q * ZU];
#pragma unroll
            for (int r = 0; r < 8; ++r)
                if (r < nr) acc[r] = fma(__ldg(Ub + (int64_t)r * nq + q), x, acc[r]);
        }
        for (int r = 0; r < nr; ++r) S[(((int64_t)b * r1max + i) * r2max + j0 + r) * ZU + u] = acc[r];
    }
}

struct TkFrag {
    int nblk, nc;
    int nkc[16], u1o[16], wo[16], r1[16], r2[16];
};

__device__ __forceinline__ int tk_block_of(const TkFrag& f, int r, const int* off) {
    int b = 0;
    while (b + 1 < f.nblk && r >= off[b + 1]) ++b;
    return b;
}

// Wf[q][wo[b] + (nc * nkc_b + kc) * 32 + lane] = W_b[q][i = 4 kc + lane % 4][u = 8 nc + lane / 4]
// with W_b[q][i][u] = sum_j U2[b][j][q] S[b][i][j][u]   (0 outside r1 x ZU)
__global__ void k_tk_wfrag(double* __restrict__ Wf, const double* __restrict__ S, const double* __restrict__ U2,
                           int r1max, int r2max, int nq, int ZU, int wq, TkFrag f) {
    const int64_t tot = (int64_t)nq * wq;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int q = (int)(e / wq), r = (int)(e % wq);
        const int b = tk_block_of(f, r, f.wo);
        const int rr = r - f.wo[b], lane = rr & 31, kc = (rr >> 5) % f.nkc[b], ncc = (rr >> 5) / f.nkc[b];
        const int i = 4 * kc + (lane & 3), u = 8 * ncc + (lane >> 2);
        double v = 0.0;
        if (i < f.r1[b] && u < ZU) {
            const double* s = S + (((int64_t)b * r1max + i) * r2max) * ZU + u;
            const double* Ub = U2 + (int64_t)b * r2max * nq + q;
            for (int j = 0; j < f.r2[b]; ++j) v = fma(Ub[(int64_t)j * nq], s[(int64_t)j * ZU], v);
        }
        Wf[e] = v;
    }
}

// U1f[xt][u1o[b] + kc * 32 + lane] = U1[b][i = 4 kc + lane % 4][kx = 8 xt + lane / 4]
__global__ void k_tk_u1frag(double* __restrict__ U1f, const double* __restrict__ U1, int r1max, int nkx, int nt3,
                            int u1t, TkFrag f) {
    const int64_t tot = (int64_t)nt3 * u1t;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int xt = (int)(e / u1t), r = (int)(e % u1t);
        const int b = tk_block_of(f, r, f.u1o);
        const int rr = r - f.u1o[b], lane = rr & 31, kc = rr >> 5;
        const int i = 4 * kc + (lane & 3), kx = 8 * xt + (lane >> 2);
        U1f[e] = (i < f.r1[b] && kx < nkx) ? U1[((int64_t)b * r1max + i) * nkx + kx] : 0.0;
    }
}

// ||X_b - X~_b||^2 and ||X_b||^2 per block (errs[2 b], errs[2 b + 1]), X~ rebuilt from the
// fragment tables exactly as P3 does (same products, other summation order)
__global__ void __launch_bounds__(kTkNT) k_tk_err(double* __restrict__ errs, const double* __restrict__ Rt,
                                                  const double* __restrict__ U1f, const double* __restrict__ Wf,
                                                  int nkx, int nq, int ZU, int nt3, int RS1, int u1t, int wq,
                                                  TkFrag f) {
    __shared__ double sh[kTkNT / 32];
    const int b = blockIdx.y;
    const int64_t per = (int64_t)nkx * nq * ZU;
    double d2 = 0.0, x2 = 0.0;
    for (int64_t e = blockIdx.x * (int64_t)kTkNT + threadIdx.x; e < per; e += (int64_t)gridDim.x * kTkNT) {
        const int kx = (int)(e / ((int64_t)nq * ZU)), q = (int)((e / ZU) % nq), u = (int)(e % ZU);
        const double* a = U1f + (int64_t)(kx >> 3) * u1t + f.u1o[b] + 4 * (kx & 7);
        const double* w = Wf + (int64_t)q * wq + f.wo[b] + (int64_t)(u >> 3) * f.nkc[b] * 32 + 4 * (u & 7);
        double k = 0.0;
        for (int kc = 0; kc < f.nkc[b]; ++kc)
            for (int l = 0; l < 4; ++l) k = fma(a[kc * 32 + l], w[kc * 32 + l], k);
        const double x = Rt[tk_rt(q, kx, b, u, ZU, nt3, RS1)];
        d2 = fma(k - x, k - x, d2);
        x2 = fma(x, x, x2);
    }
    d2 = blk_sum(d2, sh);
    x2 = blk_sum(x2, sh);
    if (threadIdx.x == 0) {
        atomicAdd(errs + 2 * b, d2);
        atomicAdd(errs + 2 * b + 1, x2);
    }
}

int grid_for(int64_t n, int per = kTkNT) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + per - 1) / per, 148 * 16));
}

// greedy rank-revealing basis of one mode for every block: U[b][k][i] (rmax columns reserved)
vc_status tk_mode(vc_ctx* c, int mode, int rmax, double tol2, std::vector<int>& rank) {
    Tucker& T = c->tk;
    cudaStream_t st = c->stream;
    const int nkx = T.nkx, nq = T.nq, ZU = T.ZU, nb = T.nblk;
    const int64_t blkN = (int64_t)nkx * nq * ZU;
    const int I = mode == 1 ? nkx : nq;
    const int64_t J = mode == 1 ? (int64_t)nq * ZU : (int64_t)nkx * ZU;
    const int64_t sI = mode == 1 ? (int64_t)nq * ZU : ZU, sJ = mode == 1 ? ZU : (int64_t)nq * ZU;
    DevBuf<double>& U = mode == 1 ? T.U1 : T.U2;
    VC_CUDA(c, U.alloc((size_t)nb * rmax * I));
    VC_CUDA(c, cudaMemsetAsync(U.p, 0, U.bytes(), st));
    VC_CUDA(c, T.vb.alloc((size_t)nb * I));
    VC_CUDA(c, T.st.alloc(4 * (size_t)nb));
    VC_CUDA(c, cudaMemsetAsync(T.st.p, 0, T.st.bytes(), st));
    const int nparts = (int)std::min<int64_t>((J + kTkNT - 1) / kTkNT, 296);
    VC_CUDA(c, T.part.alloc((size_t)nb * nparts * 3));
    k_tk_gather<<<grid_for(blkN * nb), kTkNT, 0, st>>>(T.R.p, c->Rt.p, nkx, nq, ZU, c->nt3, c->rs1, nb);
    count_launch(c);
    const size_t smc = 8 * (size_t)I, smp = 8 * ((size_t)I + rmax);
    if (smp > 48 * 1024) {
        VC_CUDA(c, cudaFuncSetAttribute(k_tk_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smc));
        VC_CUDA(c, cudaFuncSetAttribute(k_tk_pivot, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smp));
    }
    std::vector<double> hs(4 * (size_t)nb);
    for (int it = 0; it <= std::min(rmax, I); ++it) {
        k_tk_cols<<<dim3(nparts, nb), kTkNT, smc, st>>>(T.R.p, blkN, I, J, ZU, sI, sJ, T.vb.p, T.st.p, T.part.p);
        k_tk_pivot<<<nb, kTkNT, smp, st>>>(T.R.p, blkN, I, ZU, sI, sJ, U.p, rmax, T.vb.p, T.st.p, T.part.p, nparts,
                                           tol2);
        count_launch(c, 2);
        if (it % 8 == 7 || it == std::min(rmax, I)) {
            VC_CUDA(c, cudaMemcpyAsync(hs.data(), T.st.p, 8 * hs.size(), cudaMemcpyDeviceToHost, st));
            VC_CUDA(c, cudaStreamSynchronize(st));
            bool all = true;
            for (int b = 0; b < nb; ++b) all = all && hs[4 * b] != 0.0;
            if (all) break;
        }
    }
    VC_CUDA(c, cudaGetLastError());
    rank.assign(nb, 0);
    for (int b = 0; b < nb; ++b) {
        rank[b] = hs[4 * b] != 0.0 ? (int)hs[4 * b + 2] : (int)hs[4 * b + 1];
        if (rank[b] < 1) rank[b] = 1;  // a zero block keeps one (zero) basis vector
    }
    return VC_OK;
}

uint64_t fnv1a(const void* p, size_t n, uint64_t h = 1469598103934665603ull) {
    const unsigned char* s = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) {
        h ^= s[i];
        h *= 1099511628211ull;
    }
    return h;
}

std::string tk_path(const char* dir, const std::vector<double>& key) {
    char name[64];
    snprintf(name, sizeof name, "voxcap_tk_%016llx.bin", (unsigned long long)fnv1a(key.data(), 8 * key.size()));
    std::string d(dir);
    if (!d.empty() && d.back() != '/') d += '/';
    return d + name;
}

constexpr char kMagic[8] = {'V', 'X', 'T', 'K', '0', '0', '0', '1'};

}  // namespace

// Layout of the fragment tables from the ranks (host), allocation, and the device kernels that
// fill them from U1, U2 and S; checks that the Tucker P3 fits shared memory.
static vc_status tk_tables(vc_ctx* c) {
    Tucker& T = c->tk;
    cudaStream_t st = c->stream;
    const int nb = T.nblk;
    T.nc = (T.ZU + 7) / 8;
    int u1 = 0, w = 0;
    int r1max = 1, r2max = 1;
    // one rank-chunk count for all blocks (the smaller ranks padded with zero fragments): P3
    // runs the (block, u chunk) items of a warp as interleaved DMMA chains of equal length
    int nkcu = 1;
    for (int b = 0; b < nb; ++b) nkcu = std::max(nkcu, (T.r1[b] + 3) / 4);
    for (int b = 0; b < nb; ++b) {
        T.nkc[b] = nkcu;
        T.u1o[b] = u1;
        T.wo[b] = w;
        u1 += T.nkc[b] * 32;
        w += T.nc * T.nkc[b] * 32;
        r1max = std::max(r1max, T.r1[b]);
        r2max = std::max(r2max, T.r2[b]);
    }
    T.u1t = u1;
    T.wq = w;
    if (nb * T.nc > kMmaT * kMmaSplit * kTkItems)
        return set_err(c, VC_ERR_UNSUPPORTED, "Tucker P3: too many (block, u chunk) items per tile");
    if (p3m_tk_stages(c->rs1, c->p3m_nzt, c->p3m_kc, c->p3m_mct, T.u1t, T.wq, c->p3m_nneg > 0) < 2)
        return set_err(c, VC_ERR_UNSUPPORTED, "Tucker P3: the ranks need more shared memory than a CTA has "
                                              "(use fewer digits)");
    TkFrag f{};
    f.nblk = nb;
    f.nc = T.nc;
    for (int b = 0; b < nb; ++b) {
        f.nkc[b] = T.nkc[b];
        f.u1o[b] = T.u1o[b];
        f.wo[b] = T.wo[b];
        f.r1[b] = T.r1[b];
        f.r2[b] = T.r2[b];
    }
    VC_CUDA(c, T.U1f.alloc((size_t)c->nt3 * T.u1t));
    VC_CUDA(c, T.Wf.alloc((size_t)T.nq * T.wq));
    // U1 / U2 / S are stored with the per-mode maximum rank as stride (tk_pack / tk_load)
    k_tk_u1frag<<<grid_for((int64_t)c->nt3 * T.u1t), kTkNT, 0, st>>>(T.U1f.p, T.U1.p, r1max, T.nkx, c->nt3, T.u1t, f);
    k_tk_wfrag<<<grid_for((int64_t)T.nq * T.wq), kTkNT, 0, st>>>(T.Wf.p, T.S.p, T.U2.p, r1max, r2max, T.nq, T.ZU,
                                                                  T.wq, f);
    count_launch(c, 2);
    VC_CUDA(c, cudaGetLastError());
    return VC_OK;
}

// repack a [b][rmax][n] factor to stride rnew <= rmax (through a temporary: the ranges overlap)
static vc_status tk_repack(vc_ctx* c, DevBuf<double>& U, int nb, int rmax, int rnew, int64_t n) {
    if (rnew == rmax) return VC_OK;
    DevBuf<double> tmp;
    VC_CUDA(c, tmp.alloc((size_t)nb * rnew * n));
    for (int b = 0; b < nb; ++b)
        VC_CUDA(c, cudaMemcpyAsync(tmp.p + (int64_t)b * rnew * n, U.p + (int64_t)b * rmax * n, 8 * (size_t)rnew * n,
                                   cudaMemcpyDeviceToDevice, c->stream));
    VC_CUDA(c, cudaMemcpyAsync(U.p, tmp.p, tmp.bytes(), cudaMemcpyDeviceToDevice, c->stream));
    VC_CUDA(c, cudaStreamSynchronize(c->stream));  // tmp is freed on return
    U.n = (size_t)nb * rnew * n;
    return VC_OK;
}

bool tucker_try_load(vc_ctx* c, const char* dir, const std::vector<double>& key) {
    Tucker& T = c->tk;
    if (!dir || !*dir) return false;
    const std::string path = tk_path(dir, key);
    FILE* fp = fopen(path.c_str(), "rb");
    if (!fp) return false;
    bool ok = false;
    do {
        char mg[8];
        uint64_t kn = 0;
        if (fread(mg, 1, 8, fp) != 8 || memcmp(mg, kMagic, 8) != 0) break;
        if (fread(&kn, 8, 1, fp) != 1 || kn != key.size()) break;
        std::vector<double> k2(kn);
        if (fread(k2.data(), 8, kn, fp) != kn || k2 != key) break;
        int32_t hd[5];
        if (fread(hd, 4, 5, fp) != 5) break;
        if (hd[0] != T.nblk || hd[1] != T.nkx || hd[2] != T.nq || hd[3] != T.ZU || hd[4] != T.digits) break;
        const int nb = T.nblk;
        std::vector<int32_t> rk(2 * nb);
        std::vector<double> er(nb);
        if (fread(rk.data(), 4, 2 * nb, fp) != (size_t)(2 * nb) || fread(er.data(), 8, nb, fp) != (size_t)nb) break;
        int r1m = 1, r2m = 1;
        bool bad = false;
        for (int b = 0; b < nb; ++b) {
            if (rk[2 * b] < 1 || rk[2 * b] > T.nkx || rk[2 * b + 1] < 1 || rk[2 * b + 1] > T.nq) bad = true;
            r1m = std::max(r1m, (int)rk[2 * b]);
            r2m = std::max(r2m, (int)rk[2 * b + 1]);
        }
        if (bad) break;
        // payload: U1 [b][r1m][nkx], U2 [b][r2m][nq], S [b][r1m][r2m][ZU] (maximum-rank strides)
        const size_t n1 = (size_t)nb * r1m * T.nkx, n2 = (size_t)nb * r2m * T.nq, n3 = (size_t)nb * r1m * r2m * T.ZU;
        std::vector<double> pay(n1 + n2 + n3);
        uint64_t cs = 0;
        if (fread(pay.data(), 8, pay.size(), fp) != pay.size() || fread(&cs, 8, 1, fp) != 1) break;
        if (cs != fnv1a(pay.data(), 8 * pay.size())) break;
        if (T.U1.alloc(n1) || T.U2.alloc(n2) || T.S.alloc(n3)) break;
        // cores are stored for dv = 1 m: scale by dv^3 (P blocks) / dv^2 (E blocks) (App. C)
        for (int b = 0; b < nb; ++b) {
            const double sc = T.kind[b] == 0 ? T.dv * T.dv * T.dv : T.dv * T.dv;
            double* sb = pay.data() + n1 + n2 + (size_t)b * r1m * r2m * T.ZU;
            for (size_t e = 0; e < (size_t)r1m * r2m * T.ZU; ++e) sb[e] *= sc;
        }
        cudaStream_t cs_ = c->stream;
        if (cudaMemcpyAsync(T.U1.p, pay.data(), 8 * n1, cudaMemcpyHostToDevice, cs_) ||
            cudaMemcpyAsync(T.U2.p, pay.data() + n1, 8 * n2, cudaMemcpyHostToDevice, cs_) ||
            cudaMemcpyAsync(T.S.p, pay.data() + n1 + n2, 8 * n3, cudaMemcpyHostToDevice, cs_) ||
            cudaStreamSynchronize(cs_))
            break;
        T.r1.resize(nb);
        T.r2.resize(nb);
        for (int b = 0; b < nb; ++b) {
            T.r1[b] = rk[2 * b];
            T.r2[b] = rk[2 * b + 1];
        }
        T.err = er;
        ok = true;
    } while (false);
    fclose(fp);
    return ok;
}

static int tk_write(vc_ctx* c, const char* dir, const std::vector<double>& key, int r1m, int r2m) {
    Tucker& T = c->tk;
    const int nb = T.nblk;
    const size_t n1 = (size_t)nb * r1m * T.nkx, n2 = (size_t)nb * r2m * T.nq, n3 = (size_t)nb * r1m * r2m * T.ZU;
    std::vector<double> pay(n1 + n2 + n3);
    if (cudaMemcpyAsync(pay.data(), T.U1.p, 8 * n1, cudaMemcpyDeviceToHost, c->stream) ||
        cudaMemcpyAsync(pay.data() + n1, T.U2.p, 8 * n2, cudaMemcpyDeviceToHost, c->stream) ||
        cudaMemcpyAsync(pay.data() + n1 + n2, T.S.p, 8 * n3, cudaMemcpyDeviceToHost, c->stream) ||
        cudaStreamSynchronize(c->stream))
        return 3;
    for (int b = 0; b < nb; ++b) {  // cores at dv = 1 m (App. C scaling, undone when loaded)
        const double sc = T.kind[b] == 0 ? T.dv * T.dv * T.dv : T.dv * T.dv;
        double* sb = pay.data() + n1 + n2 + (size_t)b * r1m * r2m * T.ZU;
        for (size_t e = 0; e < (size_t)r1m * r2m * T.ZU; ++e) sb[e] /= sc;
    }
    const std::string path = tk_path(dir, key);
    const std::string tmp = path + ".tmp" + std::to_string((long long)(uintptr_t)c);
    FILE* fp = fopen(tmp.c_str(), "wb");
    if (!fp) return 3;
    const uint64_t kn = key.size();
    const int32_t hd[5] = {nb, T.nkx, T.nq, T.ZU, T.digits};
    std::vector<int32_t> rk(2 * nb);
    for (int b = 0; b < nb; ++b) {
        rk[2 * b] = T.r1[b];
        rk[2 * b + 1] = T.r2[b];
    }
    const uint64_t cs = fnv1a(pay.data(), 8 * pay.size());
    bool ok = fwrite(kMagic, 1, 8, fp) == 8 && fwrite(&kn, 8, 1, fp) == 1 &&
              fwrite(key.data(), 8, kn, fp) == kn && fwrite(hd, 4, 5, fp) == 5 &&
              fwrite(rk.data(), 4, rk.size(), fp) == rk.size() && fwrite(T.err.data(), 8, nb, fp) == (size_t)nb &&
              fwrite(pay.data(), 8, pay.size(), fp) == pay.size() && fwrite(&cs, 8, 1, fp) == 1;
    ok = (fclose(fp) == 0) && ok;
    if (!ok || rename(tmp.c_str(), path.c_str()) != 0) {
        remove(tmp.c_str());
        return 3;
    }
    return 2;
}

// Compress the exact table c->Rt (direct-z layout) block by block on the device; fills the
// factors, cores, fragment tables and measured errors.  The caller frees Rt afterwards.
vc_status tucker_compress(vc_ctx* c) {
    Tucker& T = c->tk;
    cudaStream_t st = c->stream;
    const int nb = T.nblk, nkx = T.nkx, nq = T.nq, ZU = T.ZU;
    const double eps = pow(10.0, -T.digits);
    const double tol2 = eps * eps / 2.0;
    const int64_t blkN = (int64_t)nkx * nq * ZU;
    VC_CUDA(c, T.R.alloc((size_t)nb * blkN));
    const int rm1 = std::min(nkx, kTkMaxRank), rm2 = std::min(nq, kTkMaxRank);
    std::vector<int> r1, r2;
    vc_status s = tk_mode(c, 1, rm1, tol2, r1);
    if (s) return s;
    s = tk_mode(c, 2, rm2, tol2, r2);
    if (s) return s;
    T.r1 = r1;
    T.r2 = r2;
    int r1m = 1, r2m = 1;
    for (int b = 0; b < nb; ++b) {
        r1m = std::max(r1m, r1[b]);
        r2m = std::max(r2m, r2[b]);
    }
    // factors to their maximum-rank strides
    s = tk_repack(c, T.U1, nb, rm1, r1m, nkx);
    if (s) return s;
    s = tk_repack(c, T.U2, nb, rm2, r2m, nq);
    if (s) return s;
    TkDims d{};
    for (int b = 0; b < nb; ++b) {
        d.r1[b] = r1[b];
        d.r2[b] = r2[b];
    }
    // core: T1 = X x1 U1^T, S = T1 x2 U2^T (X densely re-gathered: the mode passes deflated R)
    k_tk_gather<<<grid_for(blkN * nb), kTkNT, 0, st>>>(T.R.p, c->Rt.p, nkx, nq, ZU, c->nt3, c->rs1, nb);
    const int64_t J = (int64_t)nq * ZU;
    VC_CUDA(c, T.t1.alloc((size_t)nb * r1m * J));
    VC_CUDA(c, T.S.alloc((size_t)nb * r1m * r2m * ZU));
    VC_CUDA(c, cudaMemsetAsync(T.S.p, 0, T.S.bytes(), st));
    k_tk_t1<<<dim3(grid_for(J), (r1m + 7) / 8, nb), kTkNT, 0, st>>>(T.t1.p, T.R.p, T.U1.p, r1m, nkx, J, d);
    k_tk_core<<<dim3(grid_for((int64_t)r1m * ZU), (r2m + 7) / 8, nb), kTkNT, 0, st>>>(T.S.p, T.t1.p, T.U2.p, r1m,
                                                                                     r2m, nq, ZU, d);
    count_launch(c, 3);
    VC_CUDA(c, cudaGetLastError());
    s = tk_tables(c);
    if (s) return s;
    // measured error of the tables P3 will use, against the exact table
    VC_CUDA(c, T.errs.alloc(2 * (size_t)nb));
    VC_CUDA(c, cudaMemsetAsync(T.errs.p, 0, T.errs.bytes(), st));
    TkFrag f{};
    f.nblk = nb;
    f.nc = T.nc;
    for (int b = 0; b < nb; ++b) {
        f.nkc[b] = T.nkc[b];
        f.u1o[b] = T.u1o[b];
        f.wo[b] = T.wo[b];
        f.r1[b] = r1[b];
        f.r2[b] = r2[b];
    }
    k_tk_err<<<dim3(grid_for(blkN), nb), kTkNT, 0, st>>>(T.errs.p, c->Rt.p, T.U1f.p, T.Wf.p, nkx, nq, ZU, c->nt3,
                                                        c->rs1, T.u1t, T.wq, f);
    count_launch(c);
    std::vector<double> e(2 * (size_t)nb);
    VC_CUDA(c, cudaMemcpyAsync(e.data(), T.errs.p, 8 * e.size(), cudaMemcpyDeviceToHost, st));
    VC_CUDA(c, cudaStreamSynchronize(st));
    T.err.assign(nb, 0.0);
    for (int b = 0; b < nb; ++b) T.err[b] = e[2 * b + 1] > 0 ? sqrt(e[2 * b] / e[2 * b + 1]) : 0.0;
    // build scratch is the size of the exact table: release it
    T.R.reset();
    T.t1.reset();
    T.part.reset();
    return VC_OK;
}

// After a cache hit: fragment tables from the loaded factors and cores.
vc_status tucker_from_cache(vc_ctx* c) { return tk_tables(c); }

// Write the cache file (after tucker_compress); sets T.cache to 2 (written) or 3 (failed).
void tucker_save(vc_ctx* c, const char* dir, const std::vector<double>& key) {
    Tucker& T = c->tk;
    int r1m = 1, r2m = 1;
    for (int b = 0; b < T.nblk; ++b) {
        r1m = std::max(r1m, T.r1[b]);
        r2m = std::max(r2m, T.r2[b]);
    }
    T.cache = tk_write(c, dir, key, r1m, r2m);
}

}  // namespace vc
