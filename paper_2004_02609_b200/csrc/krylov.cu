// krylov.cu -- restarted GMRES with left preconditioning (Eq. 14) and the capacitance
// extraction of Eq. (8).  DESIGN.md a11 / a12.
//
// Orthogonalisation is classical Gram-Schmidt applied twice (CGS2) so each Arnoldi step is two
// fused multi-dot passes + two multi-axpy passes over the basis; all reductions are two-level
// and fixed-order (deterministic).  The (restart+1) x restart Hessenberg least-squares problem
// is tiny and is updated with Givens rotations on the host, one 3*(restart+1)-double device ->
// host copy per iteration.
#include <algorithm>
#include <deque>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "ctx.h"

namespace vc {

namespace {

constexpr int kMaxBasis = 64;  // restart + 1 <= 64
constexpr int kMaxCols = 2;    // lockstep columns (= the batched matvec's kMaxB)
constexpr int kRedBlocks = 296;
constexpr int kRedNT = 256;

// out[i] = sum_n V[i][n] * w[n], i < nv.  Grid (chunk, vector group of kDotG): each block
// accumulates kDotG dots over a grid-stride range of n (kDotG registers, no predicated slots
// for absent vectors), writes per-block partials, and the last block to finish (ticket) sums
// them in a fixed order -- one launch, deterministic.
constexpr int kDotG = 8;
__global__ void __launch_bounds__(kRedNT) k_multidot(const double* __restrict__ V, int64_t ldv, int nv,
                                                     const double* __restrict__ w, int64_t n,
                                                     double* __restrict__ partial,
                                                     unsigned* __restrict__ ticket,
                                                     double* __restrict__ out) {
    const int g0 = blockIdx.y * kDotG;
    const int ng = min(kDotG, nv - g0);
    double acc[kDotG];
#pragma unroll
    for (int i = 0; i < kDotG; ++i) acc[i] = 0.0;
    const double* __restrict__ Vg = V + (int64_t)g0 * ldv;
#pragma unroll 2
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const double wk = w[k];
        if (ng == kDotG) {
#pragma unroll
            for (int i = 0; i < kDotG; ++i) acc[i] = fma(Vg[i * ldv + k], wk, acc[i]);
        } else {
#pragma unroll
            for (int i = 0; i < kDotG; ++i)
                if (i < ng) acc[i] = fma(Vg[i * ldv + k], wk, acc[i]);
        }
    }
    __shared__ double s[kRedNT / 32][kDotG];
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < kDotG; ++i) {
        double v = acc[i];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) s[wp][i] = v;
    }
    __syncthreads();
    if (threadIdx.x < ng) {
        double v = 0.0;
        for (int q = 0; q < kRedNT / 32; ++q) v += s[q][threadIdx.x];
        partial[(int64_t)blockIdx.x * nv + g0 + threadIdx.x] = v;
    }
    __threadfence();
    __shared__ bool last;
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x * gridDim.y - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    // warp per vector, lanes stride over the block partials, fixed-order shuffle tree
    for (int i = wp; i < nv; i += kRedNT / 32) {
        double v = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) v += __ldcg(partial + (int64_t)b * nv + i);
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) out[i] = v;
    }
    if (threadIdx.x == 0) *ticket = 0u;
}

// Two lockstep columns in one launch each (blockIdx.z = column; same nv for both): the same
// per-column arithmetic as k_multidot / k_multiaxpy / k_scale_by_norm (identical summation order,
// so the lockstep solver stays bitwise equal to the one-column solver), half the launches and a
// fuller grid.  Per-column partials and tickets.
struct Cols2 {
    const double* V[2];
    const double* w[2];
    double* out[2];  // dots: outputs; axpy: the updated vectors
    const double* h[2];
    double* d[2];    // k_gs_fused: the dots of the updated vectors
};
__global__ void __launch_bounds__(kRedNT) k_multidot2(Cols2 cc, int64_t ldv, int nv, int64_t n,
                                                      double* __restrict__ partial,
                                                      unsigned* __restrict__ ticket) {
    const int z = blockIdx.z;
    const int g0 = blockIdx.y * kDotG;
    const int ng = min(kDotG, nv - g0);
    double* __restrict__ part = partial + (size_t)z * kRedBlocks * kMaxBasis;
    const double* __restrict__ w = cc.w[z];
    double acc[kDotG];
#pragma unroll
    for (int i = 0; i < kDotG; ++i) acc[i] = 0.0;
    const double* __restrict__ Vg = cc.V[z] + (int64_t)g0 * ldv;
#pragma unroll 2
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const double wk = w[k];
        if (ng == kDotG) {
#pragma unroll
            for (int i = 0; i < kDotG; ++i) acc[i] = fma(Vg[i * ldv + k], wk, acc[i]);
        } else {
#pragma unroll
            for (int i = 0; i < kDotG; ++i)
                if (i < ng) acc[i] = fma(Vg[i * ldv + k], wk, acc[i]);
        }
    }
    __shared__ double s[kRedNT / 32][kDotG];
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < kDotG; ++i) {
        double v = acc[i];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) s[wp][i] = v;
    }
    __syncthreads();
    if (threadIdx.x < ng) {
        double v = 0.0;
        for (int q = 0; q < kRedNT / 32; ++q) v += s[q][threadIdx.x];
        part[(int64_t)blockIdx.x * nv + g0 + threadIdx.x] = v;
    }
    __threadfence();
    __shared__ bool last;
    if (threadIdx.x == 0) last = atomicAdd(ticket + z, 1u) == gridDim.x * gridDim.y - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int i = wp; i < nv; i += kRedNT / 32) {
        double v = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) v += __ldcg(part + (int64_t)b * nv + i);
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) cc.out[z][i] = v;
    }
    if (threadIdx.x == 0) ticket[z] = 0u;
}

__global__ void k_multiaxpy2(Cols2 cc, int64_t ldv, int nv, int64_t n, double sgn) {
    const int z = blockIdx.z;
    __shared__ double hs[kMaxBasis];
    if (threadIdx.x < nv) hs[threadIdx.x] = cc.h[z][threadIdx.x];
    __syncthreads();
    const double* __restrict__ V = cc.V[z];
    double* __restrict__ w = cc.out[z];
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int i = 0; i < nv; ++i) acc = fma(hs[i], V[i * ldv + k], acc);
        w[k] = fma(sgn, acc, w[k]);
    }
}

// CGS2's middle passes in one basis pass (blockIdx.z = column): w <- w - V h (in place, the
// arithmetic of k_multiaxpy / k_multiaxpy2: ascending fma chain, then fma(-1, acc, w)) and the
// second projection's dots d = V^T w from the same V values, held in registers (NVB >= nv
// vectors per thread), reduced per block and then in a fixed order by the last block (ticket),
// as k_multidot2 does.  Replaces a multi-axpy + multi-dot pair: one read of V and w instead of
// two (measured in DESIGN.md §7 "GMRES").
template <int NVB, int NT>
__global__ void __launch_bounds__(NT) k_gs_fused(Cols2 cc, int64_t ldv, int nv, int64_t n,
                                                     double* __restrict__ partial,
                                                     unsigned* __restrict__ ticket) {
    const int z = blockIdx.z;
    __shared__ double hs[NVB];
    if (threadIdx.x < NVB) hs[threadIdx.x] = threadIdx.x < nv ? cc.h[z][threadIdx.x] : 0.0;
    __syncthreads();
    const double* __restrict__ V = cc.V[z];
    double* __restrict__ w = cc.out[z];
    double* __restrict__ part = partial + (size_t)z * kRedBlocks * kMaxBasis;
    double acc[NVB];
#pragma unroll
    for (int i = 0; i < NVB; ++i) acc[i] = 0.0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        double v[NVB];  // the row's V values stay in registers
#pragma unroll
        for (int i = 0; i < NVB; ++i) v[i] = i < nv ? V[i * ldv + k] : 0.0;
        double a = 0.0;
#pragma unroll
        for (int i = 0; i < NVB; ++i)
            if (i < nv) a = fma(hs[i], v[i], a);
        const double w1 = fma(-1.0, a, w[k]);
        w[k] = w1;
#pragma unroll
        for (int i = 0; i < NVB; ++i) acc[i] = fma(v[i], w1, acc[i]);
    }
    __shared__ double s[NT / 32][NVB];
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < NVB; ++i) {
        if (i >= nv) break;
        double v = acc[i];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) s[wp][i] = v;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nv; i += NT) {
        double v = 0.0;
        for (int q = 0; q < NT / 32; ++q) v += s[q][i];
        part[(int64_t)blockIdx.x * nv + i] = v;
    }
    __threadfence();
    __shared__ bool last;
    if (threadIdx.x == 0) last = atomicAdd(ticket + z, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int i = wp; i < nv; i += NT / 32) {
        double v = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) v += __ldcg(part + (int64_t)b * nv + i);
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) cc.d[z][i] = v;
    }
    if (threadIdx.x == 0) ticket[z] = 0u;
}
// nv above this: the separate multi-axpy + multi-dot kernels (VC_GS_FUSED=<max nv> overrides for
// A/B runs; 0 = never fused)
constexpr int kGsFusedMaxNV = 32;
inline int gs_fused_max() {
    static const int v = getenv("VC_GS_FUSED") ? std::min(kGsFusedMaxNV, atoi(getenv("VC_GS_FUSED"))) : kGsFusedMaxNV;
    return v;
}

// w_z <- w_z - V_z h_z and d_z = V_z^T w_z for nc <= 2 columns (k_gs_fused)
cudaError_t launch_gs_fused(const Cols2& cc, int64_t n, int nv, int nc, double* partial, unsigned* ticket,
                            cudaStream_t st) {
    // registers sized to the basis in steps of 4 vectors; from 28 vectors on (> 140 registers)
    // 128-thread blocks, twice as many (the partials of <= 32 vectors x 592 blocks still fit)
    const dim3 g(kRedBlocks, 1, nc), g2(2 * kRedBlocks, 1, nc);
    switch ((nv + 3) / 4) {
#define VC_GSF(K)                                                                              \
    case K:                                                                                    \
        if (4 * K >= 28) k_gs_fused<4 * K, 128><<<g2, 128, 0, st>>>(cc, n, nv, n, partial, ticket); \
        else k_gs_fused<4 * K, kRedNT><<<g, kRedNT, 0, st>>>(cc, n, nv, n, partial, ticket);   \
        break;
        VC_GSF(1) VC_GSF(2) VC_GSF(3) VC_GSF(4) VC_GSF(5) VC_GSF(6) VC_GSF(7) VC_GSF(8)
#undef VC_GSF
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// CGS2's last pass with the norm: w <- w - V h (the arithmetic of k_multiaxpy / k_multiaxpy2) and
// d[z][0] = ||w||^2 (per-block partials, then a fixed-order sum by the last block), in place of
// a multi-axpy and a one-vector multi-dot (one read of w fewer, one launch fewer)
__global__ void __launch_bounds__(kRedNT) k_axpy_norm(Cols2 cc, int64_t ldv, int nv, int64_t n,
                                                      double* __restrict__ partial,
                                                      unsigned* __restrict__ ticket) {
    const int z = blockIdx.z;
    __shared__ double hs[kMaxBasis];
    if (threadIdx.x < nv) hs[threadIdx.x] = cc.h[z][threadIdx.x];
    __syncthreads();
    const double* __restrict__ V = cc.V[z];
    double* __restrict__ w = cc.out[z];
    double* __restrict__ part = partial + (size_t)z * kRedBlocks * kMaxBasis;
    double acc2 = 0.0;
    // two grid-stride elements per trip (their basis loads interleaved: twice the loads in
    // flight), each with the one-element arithmetic in the same order, so the result is unchanged
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += 2 * gs) {
        const int64_t k2 = k + gs < n ? k + gs : k;
        double accA = 0.0, accB = 0.0;
#pragma unroll 4
        for (int i = 0; i < nv; ++i) {
            const double va = V[i * ldv + k], vb = V[i * ldv + k2];
            accA = fma(hs[i], va, accA);
            accB = fma(hs[i], vb, accB);
        }
        const double wA = fma(-1.0, accA, w[k]);
        w[k] = wA;
        acc2 = fma(wA, wA, acc2);
        if (k2 != k) {
            const double wB = fma(-1.0, accB, w[k2]);
            w[k2] = wB;
            acc2 = fma(wB, wB, acc2);
        }
    }
    __shared__ double s[kRedNT / 32];
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    for (int o = 16; o; o >>= 1) acc2 += __shfl_xor_sync(0xffffffffu, acc2, o);
    if (lane == 0) s[wp] = acc2;
    __syncthreads();
    if (threadIdx.x == 0) {
        double v = 0.0;
        for (int q = 0; q < kRedNT / 32; ++q) v += s[q];
        part[blockIdx.x] = v;
    }
    __threadfence();
    __shared__ bool last;
    if (threadIdx.x == 0) last = atomicAdd(ticket + z, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (wp == 0) {
        double v = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) v += __ldcg(part + b);
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) cc.d[z][0] = v;
    }
    if (threadIdx.x == 0) ticket[z] = 0u;
}

// out[z] = w[z] / sqrt(*h[z])
__global__ void k_scale_by_norm2(Cols2 cc, int64_t n) {
    const int z = blockIdx.z;
    const double s = 1.0 / sqrt(*cc.h[z]);
    const double* __restrict__ src = cc.w[z];
    double* __restrict__ dst = cc.out[z];
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x)
        dst[k] = src[k] * s;
}

// w -= sum_i h[i] V[i]   (h on the device)
__global__ void k_multiaxpy(double* __restrict__ w, const double* __restrict__ V, int64_t ldv,
                            int nv, const double* __restrict__ h, int64_t n, double sgn) {
    __shared__ double hs[kMaxBasis];
    if (threadIdx.x < nv) hs[threadIdx.x] = h[threadIdx.x];
    __syncthreads();
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int i = 0; i < nv; ++i) acc = fma(hs[i], V[i * ldv + k], acc);
        w[k] = fma(sgn, acc, w[k]);
    }
}

// dst = src / sqrt(*nrm2)
__global__ void k_scale_by_norm(double* __restrict__ dst, const double* __restrict__ src,
                                const double* __restrict__ nrm2, int64_t n) {
    const double s = 1.0 / sqrt(*nrm2);
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x)
        dst[k] = src[k] * s;
}

// y = a*x + b*y  (y is not read when b == 0: it may hold stale non-finite data)
__global__ void k_axpby(double* __restrict__ y, const double* __restrict__ x, double a, double b,
                        int64_t n) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x)
        y[k] = b == 0.0 ? a * x[k] : fma(a, x[k], b * y[k]);
}

// b_k = dv^2 on the panels of conductor j (V_k = A_k Phi_k)
__global__ void k_rhs(double* __restrict__ b, const int32_t* __restrict__ cid, int j, double area,
                      int64_t n) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x)
        b[k] = cid[k] == j ? area : 0.0;
}

// partial[i * nb + blk] = sum over conductor-i panels in block blk of A fc rho  (Eq. 8)
__global__ void k_cap_partial(const double* __restrict__ rho, const int32_t* __restrict__ cid,
                              const double* __restrict__ fc, double area, int64_t n, int m,
                              double* __restrict__ partial) {
    // one pass per conductor i = blockIdx.y + 1
    const int i = blockIdx.y + 1;
    double acc = 0.0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x)
        if (cid[k] == i) acc = fma(area * fc[k], rho[k], acc);
    __shared__ double s[kRedNT / 32];
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double v = 0.0;
        for (int q = 0; q < kRedNT / 32; ++q) v += s[q];
        partial[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = v;
    }
}

__global__ void k_cap_final(const double* __restrict__ partial, int nb, int m,
                            double* __restrict__ out) {
    const int i = threadIdx.x;
    if (i >= m) return;
    double v = 0.0;
    for (int q = 0; q < nb; ++q) v += partial[(int64_t)i * nb + q];
    out[i] = v;
}

inline unsigned grid_for(int64_t n) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8));
}

}  // namespace

struct Krylov {
    vc_ctx* c;
    int64_t n;
    double *V, *w, *t, *r, *b, *x;  // V: (m+1) x n
    int m;
    vc_status ensure(int restart) {
        m = restart;
        const size_t need = (size_t)(m + 1 + 5) * n;
        if (c->work_n < need) {
            VC_CUDA(c, c->work.alloc(need));
            c->work_n = need;
        }
        if (c->partial.n < (size_t)kRedBlocks * kMaxBasis) VC_CUDA(c, c->partial.alloc((size_t)kRedBlocks * kMaxBasis));
        if (c->dvec.n < 8 * kMaxBasis) VC_CUDA(c, c->dvec.alloc(8 * kMaxBasis));
        if (c->ticket.n < 2) {
            VC_CUDA(c, c->ticket.alloc(2));
            VC_CUDA(c, cudaMemsetAsync(c->ticket.p, 0, 2 * sizeof(unsigned), c->stream));
        }
        if (!c->h_pinned) VC_CUDA(c, cudaMallocHost(&c->h_pinned, 8 * 8 * kMaxBasis));
        V = c->work.p;
        w = V + (size_t)(m + 1) * n;
        t = w + n;
        r = t + n;
        b = r + n;
        x = b + n;
        return VC_OK;
    }
    // out[0..nv) = V[0..nv) . vec, summed over ranks (world > 1)
    vc_status dots(const double* Vb, int nv, const double* vec, double* out) {
        const dim3 grid(kRedBlocks, (nv + kDotG - 1) / kDotG);
        k_multidot<<<grid, kRedNT, 0, c->stream>>>(Vb, n, nv, vec, n, c->partial.p, c->ticket.p, out);
        count_launch(c, 1);
        return comm_allreduce(c, out, nv);
    }
    // CGS2 middle passes: t -= V[0..nv) h (device), then d = V[0..nv) . t, summed over ranks
    vc_status fused(int nv, const double* h, double* d) {
        if (nv > gs_fused_max()) {
            k_multiaxpy<<<grid_for(n), 256, 0, c->stream>>>(t, V, n, nv, h, n, -1.0);
            count_launch(c, 1);
            return dots(V, nv, t, d);
        }
        Cols2 cc{};
        cc.V[0] = V;
        cc.out[0] = t;
        cc.h[0] = h;
        cc.d[0] = d;
        VC_CUDA(c, launch_gs_fused(cc, n, nv, 1, c->partial.p, c->ticket.p, c->stream));
        count_launch(c, 1);
        return comm_allreduce(c, d, nv);
    }
    // t -= V[0..nv) h (device), then d[0] = ||t||^2, summed over ranks
    vc_status axpy_norm(int nv, const double* h, double* d) {
        Cols2 cc{};
        cc.V[0] = V;
        cc.out[0] = t;
        cc.h[0] = h;
        cc.d[0] = d;
        k_axpy_norm<<<dim3(kRedBlocks, 1, 1), kRedNT, 0, c->stream>>>(cc, n, nv, n, c->partial.p, c->ticket.p);
        VC_CUDA(c, cudaGetLastError());
        count_launch(c, 1);
        return comm_allreduce(c, d, 1);
    }
    vc_status norm2_host(const double* vec, double* out) {
        vc_status s = dots(vec, 1, vec, c->dvec.p);
        if (s) return s;
        VC_CUDA(c, cudaMemcpyAsync(c->h_pinned, c->dvec.p, 8, cudaMemcpyDeviceToHost, c->stream));
        VC_CUDA(c, cudaStreamSynchronize(c->stream));
        *out = std::sqrt(c->h_pinned[0]);
        return VC_OK;
    }
    // dst = R A src
    vc_status op(const double* src, double* dst, double* tmp) {
        vc_status s = matvec_dev(c, src, tmp);
        if (s) return s;
        return precond_apply_dev(c, tmp, dst);
    }
};

vc_status solve_dev(vc_ctx* c, const double* d_b, double* d_x, const vc_solve_opts* o,
                    vc_solve_info* info) {
    const double tol = (o && o->tol > 0) ? o->tol : 1e-4;
    const int restart = (o && o->restart > 0) ? std::min(o->restart, kMaxBasis - 1) : 35;
    const int maxit = (o && o->maxit > 0) ? o->maxit : 2000;
    const bool guess = o && o->x0_is_guess;
    Krylov K{c, c->NL};
    vc_status s = K.ensure(restart);
    if (s) return s;
    cudaStream_t st = c->stream;
    const int64_t n = c->NL;
    const unsigned gn = grid_for(n);
    VC_CUDA(c, cudaMemcpyAsync(K.b, d_b, 8 * n, cudaMemcpyDeviceToDevice, st));
    if (guess) VC_CUDA(c, cudaMemcpyAsync(K.x, d_x, 8 * n, cudaMemcpyDeviceToDevice, st));
    else VC_CUDA(c, cudaMemsetAsync(K.x, 0, 8 * n, st));
    // ||R b||
    if ((s = precond_apply_dev(c, K.b, K.r))) return s;
    double nrb = 0, nb = 0;
    if ((s = K.norm2_host(K.r, &nrb))) return s;
    if ((s = K.norm2_host(K.b, &nb))) return s;
    int iters = 0;
    double rre = 1.0;
    bool converged = false;
    std::vector<double> H((size_t)(restart + 1) * restart), cs(restart), sn(restart), g(restart + 1), y(restart);
    if (nrb == 0.0) {
        converged = true;
        rre = 0.0;
    }
    while (!converged && iters < maxit) {
        // r = R (b - A x)
        if (iters == 0 && !guess) {
            // x = 0: r = R b (already in K.r)
        } else {
            if ((s = matvec_dev(c, K.x, K.w))) return s;
            k_axpby<<<gn, 256, 0, st>>>(K.w, K.b, 1.0, -1.0, n);  // w = b - A x
            count_launch(c);
            if ((s = precond_apply_dev(c, K.w, K.r))) return s;
        }
        double beta = 0;
        if ((s = K.norm2_host(K.r, &beta))) return s;
        rre = beta / nrb;
        if (rre <= tol) {
            converged = true;
            break;
        }
        k_axpby<<<gn, 256, 0, st>>>(K.V, K.r, 1.0 / beta, 0.0, n);  // V0 = r / beta
        count_launch(c);
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = beta;
        int jend = 0;
        // Arnoldi step j on the device: w = R A v_j, CGS2 against v_0..v_j (coefficients in
        // device slot j % 2), v_{j+1} = w / ||w||, coefficients copied to pinned host slot j % 2.
        // The host Givens update of step j runs while the device already executes step j + 1
        // (the next step needs only device data), so the convergence test lags one step: at
        // most one extra Arnoldi step per restart cycle, never a wrong iterate.
        auto enqueue = [&](int j) -> vc_status {
            double* vj = K.V + (size_t)j * n;
            double* vn = K.V + (size_t)(j + 1) * n;
            vc_status e;
            if ((e = K.op(vj, K.t, K.w))) return e;
            double* dh = c->dvec.p + (size_t)(j & 1) * 3 * kMaxBasis;
            if ((e = K.dots(K.V, j + 1, K.t, dh))) return e;
            if ((e = K.fused(j + 1, dh, dh + kMaxBasis))) return e;
            if ((e = K.axpy_norm(j + 1, dh + kMaxBasis, dh + 2 * kMaxBasis))) return e;
            k_scale_by_norm<<<gn, 256, 0, st>>>(vn, K.t, dh + 2 * kMaxBasis, n);
            count_launch(c, 1);
            VC_CUDA(c, cudaMemcpyAsync(c->h_pinned + (size_t)(j & 1) * 3 * kMaxBasis, dh,
                                       8 * 3 * kMaxBasis, cudaMemcpyDeviceToHost, st));
            VC_CUDA(c, cudaEventRecord(c->arn_ev[j & 1], st));
            return VC_OK;
        };
        if (!c->arn_ev_ok) {
            for (auto& e : c->arn_ev) VC_CUDA(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            c->arn_ev_ok = true;
        }
        int queued = 0;  // Arnoldi steps enqueued in this cycle
        const int it0 = iters;
        if (restart > 0 && iters < maxit) {
            if ((s = enqueue(0))) return s;
            queued = 1;
        }
        // The prefetch of step j + 1 is skipped when the residual history predicts that step j
        // converges (geometric extrapolation rre_j ~ rre_{j-1}^2 / rre_{j-2} within 2x of tol):
        // a wrong guess costs one host round trip, a right one saves a wasted Arnoldi step.
        double r_prev = 0.0, r_prev2 = 0.0;
        for (int j = 0; j < queued; ++j) {
            const bool can = queued < restart && it0 + queued < maxit;
            const bool near = j >= 2 && r_prev2 > 0.0 && r_prev * (r_prev / r_prev2) <= 2.0 * tol;
            if (can && !near) {
                if ((s = enqueue(queued))) return s;
                ++queued;
            }
            VC_CUDA(c, cudaEventSynchronize(c->arn_ev[j & 1]));
            ++iters;
            const double* hh = c->h_pinned + (size_t)(j & 1) * 3 * kMaxBasis;
            double* Hj = H.data() + (size_t)j * (restart + 1);  // column j
            for (int i = 0; i <= j; ++i) Hj[i] = hh[i] + hh[kMaxBasis + i];
            Hj[j + 1] = std::sqrt(hh[2 * kMaxBasis]);
            for (int i = 0; i < j; ++i) {
                const double a = Hj[i], bb = Hj[i + 1];
                Hj[i] = cs[i] * a + sn[i] * bb;
                Hj[i + 1] = -sn[i] * a + cs[i] * bb;
            }
            const double a = Hj[j], bb = Hj[j + 1];
            const double den = std::hypot(a, bb);
            cs[j] = den > 0 ? a / den : 1.0;
            sn[j] = den > 0 ? bb / den : 0.0;
            Hj[j] = den;
            Hj[j + 1] = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            rre = std::fabs(g[j + 1]) / nrb;
            jend = j + 1;
            if (rre <= tol || !(rre == rre)) break;
            r_prev2 = r_prev;
            r_prev = rre;
            if (queued == j + 1 && queued < restart && it0 + queued < maxit) {  // prefetch skipped
                if ((s = enqueue(queued))) return s;
                ++queued;
            }
        }
        // y = H^{-1} g (upper triangular), x += V y
        for (int i = jend - 1; i >= 0; --i) {
            double v = g[i];
            for (int k = i + 1; k < jend; ++k) v -= H[(size_t)k * (restart + 1) + i] * y[k];
            y[i] = v / H[(size_t)i * (restart + 1) + i];
        }
        VC_CUDA(c, cudaMemcpyAsync(c->dvec.p + 6 * kMaxBasis, y.data(), 8 * jend, cudaMemcpyHostToDevice, st));
        k_multiaxpy<<<gn, 256, 0, st>>>(K.x, K.V, n, jend, c->dvec.p + 6 * kMaxBasis, n, 1.0);
        count_launch(c);
        if (rre <= tol) converged = true;
        if (!(rre == rre)) break;
    }
    // true residual ||b - A x|| / ||b||
    if ((s = matvec_dev(c, K.x, K.w))) return s;
    k_axpby<<<gn, 256, 0, st>>>(K.w, K.b, 1.0, -1.0, n);
    count_launch(c);
    double nr = 0;
    if ((s = K.norm2_host(K.w, &nr))) return s;
    VC_CUDA(c, cudaMemcpyAsync(d_x, K.x, 8 * n, cudaMemcpyDeviceToDevice, st));
    VC_CUDA(c, cudaStreamSynchronize(st));
    if (info) {
        info->iters = iters;
        info->converged = converged ? 1 : 0;
        info->rre_prec = rre;
        info->rre_true = nb > 0 ? nr / nb : 0.0;
    }
    return converged ? VC_OK : set_err(c, VC_NOT_CONVERGED, "GMRES did not reach tol within maxit");
}

// Lockstep GMRES for ncol <= kMaxB right-hand sides: every column runs
// the same restarted, left-preconditioned GMRES with CGS2 as solve_dev (identical kernels and
// arithmetic per column), but each step's matvecs -- the Arnoldi products R A v_j of the columns
// in a cycle and the restart residuals b - A x of the others -- go through one batched matvec,
// so P3 reads each kernel tile once for all columns.  One host synchronisation per step (the
// Givens updates of all columns).  d_b, d_x: ncol device vectors of n.
vc_status solve_multi_dev(vc_ctx* c, int ncol, const double* const* d_b, double* const* d_x,
                          const vc_solve_opts* o, vc_solve_info* info) {
    const double tol = (o && o->tol > 0) ? o->tol : 1e-4;
    const int restart = (o && o->restart > 0) ? std::min(o->restart, kMaxBasis - 1) : 35;
    const int maxit = (o && o->maxit > 0) ? o->maxit : 2000;
    const int64_t n = c->NL;
    cudaStream_t st = c->stream;
    const unsigned gn = grid_for(n);
    const size_t per = (size_t)(restart + 1 + 5) * n;
    if (c->work_n < per * ncol) {
        VC_CUDA(c, c->work.alloc(per * ncol));
        c->work_n = per * ncol;
    }
    if (c->partial.n < (size_t)kRedBlocks * kMaxBasis * kMaxCols)
        VC_CUDA(c, c->partial.alloc((size_t)kRedBlocks * kMaxBasis * kMaxCols));
    if (c->dvec.n < (size_t)8 * kMaxBasis * kMaxCols) VC_CUDA(c, c->dvec.alloc((size_t)8 * kMaxBasis * kMaxCols));
    if (c->ticket.n < 2) {
        VC_CUDA(c, c->ticket.alloc(2));
        VC_CUDA(c, cudaMemsetAsync(c->ticket.p, 0, 2 * sizeof(unsigned), st));
    }
    if (!c->h_pinned_multi) VC_CUDA(c, cudaMallocHost(&c->h_pinned_multi, sizeof(double) * 8 * kMaxBasis * kMaxCols));
    if (!c->h_pinned) VC_CUDA(c, cudaMallocHost(&c->h_pinned, 8 * 8 * kMaxBasis));
    struct Col {
        Krylov K;
        double *dh, *hp;
        std::vector<double> H, cs, sn, g, y;
        double nrb = 0, nb = 0, rre = 1, nr = 0;
        int iters = 0, j = 0, phase = 0;  // phase 0: restart residual, 1: Arnoldi, 2: done
        double r_prev = 0, r_prev2 = 0;    // residual history (speculation guard)
        bool converged = false;
    };
    std::vector<Col> col(ncol);
    vc_status s;
    for (int i = 0; i < ncol; ++i) {
        Col& C = col[i];
        C.K.c = c;
        C.K.n = n;
        C.K.m = restart;
        C.K.V = c->work.p + per * i;
        C.K.w = C.K.V + (size_t)(restart + 1) * n;
        C.K.t = C.K.w + n;
        C.K.r = C.K.t + n;
        C.K.b = C.K.r + n;
        C.K.x = C.K.b + n;
        C.dh = c->dvec.p + (size_t)8 * kMaxBasis * i;
        C.hp = c->h_pinned_multi + (size_t)8 * kMaxBasis * i;
        C.H.assign((size_t)(restart + 1) * restart, 0.0);
        C.cs.assign(restart, 0.0);
        C.sn.assign(restart, 0.0);
        C.g.assign(restart + 1, 0.0);
        C.y.assign(restart, 0.0);
        VC_CUDA(c, cudaMemcpyAsync(C.K.b, d_b[i], 8 * n, cudaMemcpyDeviceToDevice, st));
        VC_CUDA(c, cudaMemsetAsync(C.K.x, 0, 8 * n, st));
        if ((s = precond_apply_dev(c, C.K.b, C.K.r))) return s;  // x = 0: r = R b
        if ((s = C.K.norm2_host(C.K.r, &C.nrb))) return s;
        if ((s = C.K.norm2_host(C.K.b, &C.nb))) return s;
        if (C.nrb == 0.0) {
            C.converged = true;
            C.rre = 0.0;
            C.phase = 2;
        } else {  // first cycle: V0 = r / ||r||
            k_axpby<<<gn, 256, 0, st>>>(C.K.V, C.K.r, 1.0 / C.nrb, 0.0, n);
            count_launch(c);
            C.g[0] = C.nrb;
            C.phase = 1;
        }
    }
    auto finish_cycle = [&](Col& C) -> vc_status {  // y = H^{-1} g, x += V y
        const int jend = C.j;
        for (int i = jend - 1; i >= 0; --i) {
            double v = C.g[i];
            for (int k = i + 1; k < jend; ++k) v -= C.H[(size_t)k * (restart + 1) + i] * C.y[k];
            C.y[i] = v / C.H[(size_t)i * (restart + 1) + i];
        }
        if (jend > 0) {
            VC_CUDA(c, cudaMemcpyAsync(C.dh + 6 * kMaxBasis, C.y.data(), 8 * jend, cudaMemcpyHostToDevice, st));
            k_multiaxpy<<<gn, 256, 0, st>>>(C.K.x, C.K.V, n, jend, C.dh + 6 * kMaxBasis, n, 1.0);
            count_launch(c);
        }
        return VC_OK;
    };
    // A step = one batched matvec + the per-column work after it, for a list of (column, phase,
    // j) entries; its coefficients land in parity slot `par` of each column's device / pinned
    // scratch (3 * kMaxBasis doubles each) and an event marks them.  While step s is in flight
    // the next Arnoldi step of the same columns is enqueued speculatively (its input v_{j+1} is
    // produced on the device), unless a column may leave phase 1 (cycle end, maxit, predicted
    // convergence); entries of a speculative step whose column changed state are discarded.
    struct Ent { int col, phase, j; };
    struct Step { std::vector<Ent> ent; int par; };
    std::deque<Step> q;
    int par = 0;
    if (!c->mc_ev_ok) {
        for (auto& e : c->mc_ev) VC_CUDA(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->mc_ev_ok = true;
    }
    std::vector<const double*> ins;
    std::vector<double*> outs;
    auto enqueue_step = [&](std::vector<Ent> ents) -> vc_status {
        Step S{std::move(ents), par};
        par ^= 1;
        const int sl = S.par * 3 * kMaxBasis;
        vc_status e;
        ins.clear();
        outs.clear();
        for (const Ent& en : S.ent) {
            Col& C = col[en.col];
            ins.push_back(en.phase == 1 ? C.K.V + (size_t)en.j * n : C.K.x);
            outs.push_back(C.K.w);
        }
        if ((e = matvec_batch_dev(c, (int)S.ent.size(), ins.data(), outs.data()))) return e;
        {  // t = R w for the Arnoldi columns, in one apply
            const double* pr[kMaxCols];
            double* pz[kMaxCols];
            int np = 0;
            for (const Ent& en : S.ent)
                if (en.phase == 1) {
                    pr[np] = col[en.col].K.w;
                    pz[np++] = col[en.col].K.t;
                }
            if (np && (e = precond_apply_multi_dev(c, np, pr, pz))) return e;
        }
        // both columns in Arnoldi at the same j: the CGS2 kernels run once for the pair
        static const bool pair_ok = !(getenv("VC_GS_PAIR") && !atoi(getenv("VC_GS_PAIR")));
        const bool pair = pair_ok && S.ent.size() == 2 && S.ent[0].phase == 1 &&
                          S.ent[1].phase == 1 && S.ent[0].j == S.ent[1].j;
        if (pair) {
            Col &A = col[S.ent[0].col], &B = col[S.ent[1].col];
            const int nv = S.ent[0].j + 1;
            double *ha = A.dh + sl, *hb = B.dh + sl;
            auto cc = [&](const double* v0, const double* v1, const double* w0, const double* w1,
                          double* o0, double* o1, const double* h0, const double* h1) {
                Cols2 qq;
                qq.V[0] = v0; qq.V[1] = v1; qq.w[0] = w0; qq.w[1] = w1;
                qq.out[0] = o0; qq.out[1] = o1; qq.h[0] = h0; qq.h[1] = h1;
                return qq;
            };
            const dim3 gd(kRedBlocks, (nv + kDotG - 1) / kDotG, 2), ga(gn, 1, 2);
            // several ranks: each column's partial dots are summed over ranks (as K.dots does)
            auto sum_ranks = [&](int off, int cnt) -> vc_status {
                if (c->world == 1) return VC_OK;
                vc_status e2 = comm_allreduce(c, ha + off, cnt);
                return e2 ? e2 : comm_allreduce(c, hb + off, cnt);
            };
            k_multidot2<<<gd, kRedNT, 0, st>>>(cc(A.K.V, B.K.V, A.K.t, B.K.t, ha, hb, nullptr, nullptr),
                                               n, nv, n, c->partial.p, c->ticket.p);
            if ((e = sum_ranks(0, nv))) return e;
            if (nv <= gs_fused_max()) {  // t -= V h1 and h2 = V^T t in one basis pass
                Cols2 f = cc(A.K.V, B.K.V, nullptr, nullptr, A.K.t, B.K.t, ha, hb);
                f.d[0] = ha + kMaxBasis;
                f.d[1] = hb + kMaxBasis;
                VC_CUDA(c, launch_gs_fused(f, n, nv, 2, c->partial.p, c->ticket.p, st));
            } else {
                k_multiaxpy2<<<ga, 256, 0, st>>>(cc(A.K.V, B.K.V, nullptr, nullptr, A.K.t, B.K.t, ha, hb),
                                                 n, nv, n, -1.0);
                k_multidot2<<<gd, kRedNT, 0, st>>>(cc(A.K.V, B.K.V, A.K.t, B.K.t, ha + kMaxBasis,
                                                      hb + kMaxBasis, nullptr, nullptr),
                                                   n, nv, n, c->partial.p, c->ticket.p);
            }
            if ((e = sum_ranks(kMaxBasis, nv))) return e;
            {  // t -= V h2 and ||t||^2 in one pass
                Cols2 f = cc(A.K.V, B.K.V, nullptr, nullptr, A.K.t, B.K.t, ha + kMaxBasis, hb + kMaxBasis);
                f.d[0] = ha + 2 * kMaxBasis;
                f.d[1] = hb + 2 * kMaxBasis;
                k_axpy_norm<<<dim3(kRedBlocks, 1, 2), kRedNT, 0, st>>>(f, n, nv, n, c->partial.p, c->ticket.p);
            }
            if ((e = sum_ranks(2 * kMaxBasis, 1))) return e;
            k_scale_by_norm2<<<ga, 256, 0, st>>>(cc(nullptr, nullptr, A.K.t, B.K.t,
                                                    A.K.V + (size_t)nv * n, B.K.V + (size_t)nv * n,
                                                    ha + 2 * kMaxBasis, hb + 2 * kMaxBasis),
                                                 n);
            count_launch(c, nv <= gs_fused_max() ? 4 : 5);
        } else {
            for (const Ent& en : S.ent) {
                Col& C = col[en.col];
                Krylov& K = C.K;
                double* dh = C.dh + sl;
                if (en.phase == 1) {  // CGS2 of w' = R A v_j against v_0..v_j, as in solve_dev
                    const int j = en.j;
                    if ((e = K.dots(K.V, j + 1, K.t, dh))) return e;
                    if ((e = K.fused(j + 1, dh, dh + kMaxBasis))) return e;
                    if ((e = K.axpy_norm(j + 1, dh + kMaxBasis, dh + 2 * kMaxBasis))) return e;
                    k_scale_by_norm<<<gn, 256, 0, st>>>(K.V + (size_t)(j + 1) * n, K.t, dh + 2 * kMaxBasis, n);
                    count_launch(c, 1);
                } else {  // restart residual r = R (b - A x)
                    k_axpby<<<gn, 256, 0, st>>>(K.w, K.b, 1.0, -1.0, n);
                    count_launch(c);
                    if ((e = precond_apply_dev(c, K.w, K.r))) return e;
                    if ((e = K.dots(K.r, 1, K.r, dh + 2 * kMaxBasis))) return e;
                }
            }
        }
        for (const Ent& en : S.ent)
            VC_CUDA(c, cudaMemcpyAsync(col[en.col].hp + sl, col[en.col].dh + sl, 8 * 3 * kMaxBasis,
                                       cudaMemcpyDeviceToHost, st));
        VC_CUDA(c, cudaEventRecord(c->mc_ev[S.par], st));
        q.push_back(std::move(S));
        return VC_OK;
    };
    auto near = [&](const Col& C) {  // residual history predicts convergence at the next step
        return C.r_prev2 > 0.0 && C.r_prev * (C.r_prev / C.r_prev2) <= 2.0 * tol;
    };
    for (;;) {
        if (q.empty()) {
            std::vector<Ent> ents;
            for (int i = 0; i < ncol; ++i)
                if (col[i].phase != 2) ents.push_back({i, col[i].phase, col[i].j});
            if (ents.empty()) break;
            if ((s = enqueue_step(std::move(ents)))) return s;
        }
        if (q.size() == 1) {  // speculative next Arnoldi step of the same columns
            bool spec = true;
            std::vector<Ent> nxt;
            int nact = 0;
            for (int i = 0; i < ncol; ++i) nact += col[i].phase != 2;
            for (const Ent& en : q.front().ent) {
                const Col& C = col[en.col];
                if (en.phase != 1 || en.j + 1 >= restart || C.iters + 1 >= maxit || near(C)) {
                    spec = false;
                    break;
                }
                nxt.push_back({en.col, 1, en.j + 1});
            }
            if (spec && (int)nxt.size() == nact && (s = enqueue_step(std::move(nxt)))) return s;
        }
        Step F = std::move(q.front());
        q.pop_front();
        VC_CUDA(c, cudaEventSynchronize(c->mc_ev[F.par]));
        for (const Ent& en : F.ent) {
            Col& C = col[en.col];
            if (C.phase != en.phase || (en.phase == 1 && C.j != en.j)) continue;  // stale
            const double* hh = C.hp + F.par * 3 * kMaxBasis;
            if (C.phase == 1) {
                const int j = C.j;
                ++C.iters;
                double* Hj = C.H.data() + (size_t)j * (restart + 1);
                for (int qq = 0; qq <= j; ++qq) Hj[qq] = hh[qq] + hh[kMaxBasis + qq];
                Hj[j + 1] = std::sqrt(hh[2 * kMaxBasis]);
                for (int qq = 0; qq < j; ++qq) {
                    const double a = Hj[qq], bb = Hj[qq + 1];
                    Hj[qq] = C.cs[qq] * a + C.sn[qq] * bb;
                    Hj[qq + 1] = -C.sn[qq] * a + C.cs[qq] * bb;
                }
                const double a = Hj[j], bb = Hj[j + 1];
                const double den = std::hypot(a, bb);
                C.cs[j] = den > 0 ? a / den : 1.0;
                C.sn[j] = den > 0 ? bb / den : 0.0;
                Hj[j] = den;
                Hj[j + 1] = 0.0;
                C.g[j + 1] = -C.sn[j] * C.g[j];
                C.g[j] = C.cs[j] * C.g[j];
                C.rre = std::fabs(C.g[j + 1]) / C.nrb;
                C.r_prev2 = C.r_prev;
                C.r_prev = C.rre;
                C.j = j + 1;
                const bool nan = !(C.rre == C.rre);
                if (C.rre <= tol || C.j == restart || C.iters >= maxit || nan) {
                    if ((s = finish_cycle(C))) return s;
                    C.r_prev = C.r_prev2 = 0.0;
                    if (C.rre <= tol) {
                        C.converged = true;
                        C.phase = 2;
                    } else if (C.iters >= maxit || nan) {
                        C.phase = 2;
                    } else {
                        C.phase = 0;
                    }
                }
            } else {
                const double beta = std::sqrt(hh[2 * kMaxBasis]);
                C.rre = beta / C.nrb;
                if (C.rre <= tol) {
                    C.converged = true;
                    C.phase = 2;
                } else {
                    k_axpby<<<gn, 256, 0, st>>>(C.K.V, C.K.r, 1.0 / beta, 0.0, n);
                    count_launch(c);
                    std::fill(C.g.begin(), C.g.end(), 0.0);
                    C.g[0] = beta;
                    C.j = 0;
                    C.phase = 1;
                }
            }
        }
    }
    // true residuals ||b - A x|| / ||b|| (one batched matvec)
    ins.clear();
    outs.clear();
    for (int i = 0; i < ncol; ++i) {
        ins.push_back(col[i].K.x);
        outs.push_back(col[i].K.w);
    }
    if ((s = matvec_batch_dev(c, ncol, ins.data(), outs.data()))) return s;
    bool all = true;
    for (int i = 0; i < ncol; ++i) {
        Col& C = col[i];
        k_axpby<<<gn, 256, 0, st>>>(C.K.w, C.K.b, 1.0, -1.0, n);
        count_launch(c);
        if ((s = C.K.norm2_host(C.K.w, &C.nr))) return s;
        VC_CUDA(c, cudaMemcpyAsync(d_x[i], C.K.x, 8 * n, cudaMemcpyDeviceToDevice, st));
        if (info) {
            info[i].iters = C.iters;
            info[i].converged = C.converged ? 1 : 0;
            info[i].rre_prec = C.rre;
            info[i].rre_true = C.nb > 0 ? C.nr / C.nb : 0.0;
        }
        all = all && C.converged;
    }
    VC_CUDA(c, cudaStreamSynchronize(st));
    return all ? VC_OK : set_err(c, VC_NOT_CONVERGED, "GMRES did not reach tol within maxit");
}

vc_status capacitance_dev(vc_ctx* c, double* h_C, const vc_solve_opts* o, vc_solve_info* info) {
    cudaStream_t st = c->stream;
    const int64_t n = c->NL;
    const int m = c->m;
    const int32_t* cid = c->world > 1 ? c->lp.cid.p : c->pan.cid.p;
    const double* fc = c->world > 1 ? c->lp.fc.p : c->pan.fc.p;
    DevBuf<double>&b = c->cap_b, &rho = c->cap_rho, &part = c->cap_part, &col = c->cap_col;
    // columns in lockstep groups of up to nbmax (batched matvecs, NEXT-3), else one by one
    const int G = std::max(1, std::min(std::min(c->nbmax, kMaxCols), m));
    VC_CUDA(c, b.alloc(std::max<int64_t>(1, n) * G));
    VC_CUDA(c, rho.alloc(std::max<int64_t>(1, n) * G));
    const unsigned nb = 148;
    VC_CUDA(c, part.alloc((size_t)nb * m));
    VC_CUDA(c, col.alloc(m));
    std::vector<double> hp(m);
    const double area = c->dv * c->dv;
    vc_status worst = VC_OK;
    for (int j0 = 1; j0 <= m; j0 += G) {
        const int ng = std::min(G, m - j0 + 1);
        const double* bs[kMaxCols];
        double* xs[kMaxCols];
        for (int q = 0; q < ng; ++q) {
            bs[q] = b.p + (size_t)q * n;
            xs[q] = rho.p + (size_t)q * n;
            k_rhs<<<grid_for(n), 256, 0, st>>>(b.p + (size_t)q * n, cid, j0 + q, area, n);
            count_launch(c);
        }
        vc_solve_info inf[kMaxCols] = {};
        vc_status s = ng > 1 ? solve_multi_dev(c, ng, bs, xs, o, inf)
                             : solve_dev(c, bs[0], xs[0], o, &inf[0]);
        if (s != VC_OK && s != VC_NOT_CONVERGED) return s;
        if (s == VC_NOT_CONVERGED) worst = s;
        for (int q = 0; q < ng; ++q) {
            const int j = j0 + q;
            if (info) info[j - 1] = inf[q];
            dim3 g(nb, m);
            k_cap_partial<<<g, kRedNT, 0, st>>>(xs[q], cid, fc, area, n, m, part.p);
            k_cap_final<<<1, std::max(32, ((m + 31) / 32) * 32), 0, st>>>(part.p, nb, m, col.p);
            count_launch(c, 2);
            if ((s = comm_allreduce(c, col.p, m))) return s;
            VC_CUDA(c, cudaMemcpyAsync(hp.data(), col.p, 8 * (size_t)m, cudaMemcpyDeviceToHost, st));
            VC_CUDA(c, cudaStreamSynchronize(st));
            for (int i = 0; i < m; ++i) h_C[(size_t)i * m + (j - 1)] = hp[i];
        }
    }
    return worst == VC_OK ? VC_OK : set_err(c, worst, "some capacitance columns did not converge");
}

}  // namespace vc
