// panels.cu -- a1 panel indexing on the GPU (P:47, P:53-57, P:97 grids, P:115 signs).
//
// The face space is the concatenation of the three axis grids of P:97 in canonical order
// (x-normal grid (Nx+1) x Ny x Nz, then y, then z; within a grid k, j, i with i fastest), so an
// exclusive scan of the per-face "is a panel" flag gives every panel its canonical index
// (reading O14) directly.  Three passes: count per tile -> scan of tile sums -> emit.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "ctx.h"

namespace vc {

namespace {

constexpr int kTile = 2048;  // faces per CTA
constexpr int kNT = 256;

// exact division of 32-bit unsigned values by a fixed divisor (round-up multiplier, shift =
// ceil(log2 d)): the face-index decomposition is 3-4 divisions per face, and 64-bit division is a
// long software sequence (k_count / k_emit were division-bound)
struct FDiv {
    uint32_t d, m, s;
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        return (uint32_t)(((uint64_t)__umulhi(n, m) + n) >> s);
    }
};
static FDiv fdiv_make(uint32_t d) {
    uint32_t s = 0;
    while ((1ull << s) < d) ++s;
    return {d, (uint32_t)((((1ull << 32) * ((1ull << s) - d)) / d) + 1), s};
}

struct Geo {
    int nx, ny, nz;
    bool fast;        // every axis grid has < 2^32 faces: 32-bit FDiv decomposition
    FDiv gx[3], gy[3];
    int64_t F[3];     // faces per axis grid
    int64_t Foff[3];  // offset of each axis grid in the face space
    double eps_out;
    const int32_t* label;
    const double* eps;
};

struct FaceInfo {
    int type;   // 0 none, 1 conductor, 2 dielectric, 3 clash
    int sign;   // +1 / -1
    int cid;    // conductor id (conductor panels)
    double ed, eb;
};

__device__ __forceinline__ void face_coords(const Geo& g, int64_t f, int& a, int& i, int& j,
                                            int& k) {
    a = f < g.Foff[1] ? 0 : (f < g.Foff[2] ? 1 : 2);
    if (g.fast) {  // (selects, not g.gx[a]: a dynamic index would copy the parameters to local memory)
        const uint32_t r = (uint32_t)(f - (a == 0 ? 0 : (a == 1 ? g.Foff[1] : g.Foff[2])));
        const FDiv dx = a == 0 ? g.gx[0] : (a == 1 ? g.gx[1] : g.gx[2]);
        const FDiv dy = a == 0 ? g.gy[0] : (a == 1 ? g.gy[1] : g.gy[2]);
        const uint32_t r1 = dx.div(r), r2 = dy.div(r1);
        i = (int)(r - r1 * dx.d);
        j = (int)(r1 - r2 * dy.d);
        k = (int)r2;
        return;
    }
    int64_t r = f - g.Foff[a];
    const int gx = g.nx + (a == 0), gy = g.ny + (a == 1);
    i = (int)(r % gx);
    r /= gx;
    j = (int)(r % gy);
    k = (int)(r / gy);
}

// Classification rules: SURVEY §8(a) a1 / DESIGN.md readings O7, O8.
__device__ __forceinline__ FaceInfo classify(const Geo& g, int a, int i, int j, int k) {
    int li = i, lj = j, lk = k;  // lower voxel = slot - e_a
    if (a == 0) li--;
    else if (a == 1) lj--;
    else lk--;
    const bool lo_in = li >= 0 && lj >= 0 && lk >= 0;
    const bool hi_in = i < g.nx && j < g.ny && k < g.nz;
    int lab_lo = 0, lab_hi = 0;
    double e_lo = g.eps_out, e_hi = g.eps_out;
    if (lo_in) {
        const int64_t v = ((int64_t)lk * g.ny + lj) * g.nx + li;
        lab_lo = g.label[v];
        if (lab_lo == 0) e_lo = g.eps ? g.eps[v] : 1.0;
    }
    if (hi_in) {
        const int64_t v = ((int64_t)k * g.ny + j) * g.nx + i;
        lab_hi = g.label[v];
        if (lab_hi == 0) e_hi = g.eps ? g.eps[v] : 1.0;
    }
    FaceInfo fi{0, 1, 0, 0.0, 0.0};
    const bool cl = lab_lo > 0, ch = lab_hi > 0;
    if (cl && ch) {
        if (lab_lo != lab_hi) fi.type = 3;
        return fi;
    }
    if (cl || ch) {
        fi.type = 1;
        fi.sign = cl ? 1 : -1;       // outward normal from the conductor
        fi.cid = cl ? lab_lo : lab_hi;
        fi.ed = 0.0;
        fi.eb = cl ? e_hi : e_lo;    // medium the normal points into (free-charge factor)
        return fi;
    }
    if (e_lo != e_hi) {
        bool d_lo;
        if (e_lo == g.eps_out) d_lo = false;
        else if (e_hi == g.eps_out) d_lo = true;
        else d_lo = e_lo > e_hi;
        fi.type = 2;
        fi.sign = d_lo ? 1 : -1;     // normal from the d side into the b side
        fi.ed = d_lo ? e_lo : e_hi;
        fi.eb = d_lo ? e_hi : e_lo;
    }
    return fi;
}

struct Flags {
    int min_label, max_label;
    int bad_eps, clash;
};

__global__ void k_validate(int64_t nvox, const int32_t* __restrict__ label,
                           const double* __restrict__ eps, Flags* fl) {
    int mn = INT32_MAX, mx = INT32_MIN, bad = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvox;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int l = label[v];
        mn = min(mn, l);
        mx = max(mx, l);
        if (l == 0 && eps) {
            const double e = eps[v];
            if (!(e > 0.0) || !isfinite(e)) bad = 1;
        }
    }
    for (int o = 16; o; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&fl->min_label, mn);
        atomicMax(&fl->max_label, mx);
        if (bad) atomicOr(&fl->bad_eps, 1);
    }
}

__global__ void k_presence(int64_t nvox, const int32_t* __restrict__ label, int* present) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvox;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int l = label[v];
        if (l > 0) present[l] = 1;
    }
}

__global__ void k_count(Geo g, int64_t Ftot, int64_t* tile_sum, Flags* fl) {
    const int64_t base = (int64_t)blockIdx.x * kTile;
    int cnt = 0, clash = 0;
    for (int t = threadIdx.x; t < kTile; t += kNT) {
        const int64_t f = base + t;
        if (f >= Ftot) break;
        int a, i, j, k;
        face_coords(g, f, a, i, j, k);
        const FaceInfo fi = classify(g, a, i, j, k);
        cnt += (fi.type == 1 || fi.type == 2);
        clash |= fi.type == 3;
    }
    __shared__ int s[kNT / 32];
    for (int o = 16; o; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        clash |= __shfl_xor_sync(0xffffffffu, clash, o);
    }
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = cnt;
    if ((threadIdx.x & 31) == 0 && clash) atomicOr(&fl->clash, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t tot = 0;
        for (int w = 0; w < kNT / 32; ++w) tot += s[w];
        tile_sum[blockIdx.x] = tot;
    }
}

// exclusive scan of n tile sums in place (single CTA, sequential chunks of 1024)
__global__ void k_scan_tiles(int64_t* v, int64_t n, int64_t* total) {
    __shared__ int64_t s[1024];
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < n; base += 1024) {
        const int64_t idx = base + threadIdx.x;
        const int64_t x = idx < n ? v[idx] : 0;
        s[threadIdx.x] = x;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            int64_t y = threadIdx.x >= o ? s[threadIdx.x - o] : 0;
            __syncthreads();
            s[threadIdx.x] += y;
            __syncthreads();
        }
        if (idx < n) v[idx] = carry + s[threadIdx.x] - x;
        __syncthreads();
        if (threadIdx.x == 1023) carry += s[1023];
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

struct Out {
    int8_t *axis, *sign, *info;
    int32_t *si, *sj, *sk, *cid;
    double *ed, *eb, *ibar, *fc;
    int32_t* slotmap[3];
    double area_over_2eps0;
    int* ext;  // [kind][orient][min/max][axis] flattened, 36 ints; [36] conductor-panel count
};

__global__ void k_emit(Geo g, int64_t Ftot, const int64_t* __restrict__ tile_off, Out o) {
    const int64_t base = (int64_t)blockIdx.x * kTile;
    constexpr int PER = kTile / kNT;  // faces per thread, contiguous
    __shared__ int64_t warp_tot[kNT / 32];
    // panel extents: reduced in shared memory, then one global atomic per value and block (a
    // global atomic per panel serialised ~4.6M updates on 36 addresses: 3.2 ms on C4)
    __shared__ int sext[37];
    if (threadIdx.x < 36) sext[threadIdx.x] = (threadIdx.x % 6) < 3 ? INT32_MAX : INT32_MIN;
    if (threadIdx.x == 36) sext[36] = 0;
    // pass 1: one panel bit per face (the face info is recomputed for the panels in pass 2, so
    // no per-face state stays live across the scan: 131 -> fewer registers, more CTAs per SM)
    unsigned bits = 0;
    int a_t = 2;  // axis of the thread's first face (faces past the end: a valid axis)
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int64_t f = base + (int64_t)threadIdx.x * PER + q;
        if (f < Ftot) {
            int a, i, j, k;
            face_coords(g, f, a, i, j, k);
            if (q == 0) a_t = a;
            const FaceInfo fq = classify(g, a, i, j, k);
            bits |= (unsigned)(fq.type == 1 || fq.type == 2) << q;
        }
    }
    const int local = __popc(bits);
    // block exclusive scan of per-thread counts
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int incl = local;
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    int64_t woff = 0;
    for (int x = 0; x < w; ++x) woff += warp_tot[x];
    int64_t p = tile_off[blockIdx.x] + woff + incl - local;
    // panel extents of the thread's axis grid (a_t = axis of its first face) in registers;
    // one warp reduction (redux.sync) and a few shared atomics per warp instead of seven
    // shared atomics per panel on 36 addresses (contended: 0.93 ms for C4's 766k panels)
    int emin[2][3], emax[2][3], ncond = 0;
#pragma unroll
    for (int d = 0; d < 2; ++d)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            emin[d][c] = INT32_MAX;
            emax[d][c] = INT32_MIN;
        }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int64_t f = base + (int64_t)threadIdx.x * PER + q;
        if (f >= Ftot) break;
        int a, iq, jq, kq;
        face_coords(g, f, a, iq, jq, kq);
        const int64_t r = f - (a == 0 ? 0 : (a == 1 ? g.Foff[1] : g.Foff[2]));
        int32_t* const sm_a = a == 0 ? o.slotmap[0] : (a == 1 ? o.slotmap[1] : o.slotmap[2]);
        if (bits >> q & 1) {
            const FaceInfo fq = classify(g, a, iq, jq, kq);
            const bool diel = fq.type == 2;
            ncond += diel ? 0 : 1;
            o.axis[p] = (int8_t)a;
            o.sign[p] = (int8_t)fq.sign;
            o.info[p] = (int8_t)((diel ? 1 : 0) | (fq.sign < 0 ? 2 : 0));
            o.si[p] = iq;
            o.sj[p] = jq;
            o.sk[p] = kq;
            o.cid[p] = diel ? 0 : fq.cid;
            o.ed[p] = fq.ed;
            o.eb[p] = fq.eb;
            // Eq. (7): Ī = A (eps_d + eps_b) / (2 eps0 (eps_d - eps_b)); conductor rows 0
            o.ibar[p] = diel ? o.area_over_2eps0 * (fq.ed + fq.eb) / (fq.ed - fq.eb) : 0.0;
            o.fc[p] = diel ? 0.0 : fq.eb;
            sm_a[r] = (int32_t)p | (diel ? kSlotDiel : 0) | (diel && fq.sign < 0 ? kSlotNeg : 0);
            if (a == a_t) {  // the thread's axis: extents in registers, reduced per warp below
#pragma unroll
                for (int d = 0; d < 2; ++d)  // (static indices: the arrays stay in registers)
                    if ((d == 1) == diel) {
                        emin[d][0] = min(emin[d][0], iq);
                        emin[d][1] = min(emin[d][1], jq);
                        emin[d][2] = min(emin[d][2], kq);
                        emax[d][0] = max(emax[d][0], iq);
                        emax[d][1] = max(emax[d][1], jq);
                        emax[d][2] = max(emax[d][2], kq);
                    }
            } else {  // a thread straddling two axis grids (at most two per grid boundary)
                int* e = sext + ((diel ? 1 : 0) * 3 + a) * 6;
                atomicMin(e + 0, iq);
                atomicMin(e + 1, jq);
                atomicMin(e + 2, kq);
                atomicMax(e + 3, iq);
                atomicMax(e + 4, jq);
                atomicMax(e + 5, kq);
            }
            ++p;
        } else {
            sm_a[r] = -1;
        }
    }
    {
        // warps whose threads share one axis reduce in registers; a mixed warp (straddling an
        // axis grid boundary) falls back to shared atomics per lane
        const unsigned full = 0xffffffffu;
        const bool uni = __all_sync(full, __shfl_sync(full, a_t, 0) == a_t);
        const int nc = __reduce_add_sync(full, ncond);
        if (lane == 0 && nc) atomicAdd(&sext[36], nc);
#pragma unroll
        for (int d = 0; d < 2; ++d)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                int* e = sext + (d * 3 + a_t) * 6;
                if (uni) {
                    const int vmin = __reduce_min_sync(full, emin[d][c]);
                    const int vmax = __reduce_max_sync(full, emax[d][c]);
                    if (lane == 0 && vmin != INT32_MAX) {
                        atomicMin(e + c, vmin);
                        atomicMax(e + 3 + c, vmax);
                    }
                } else if (emin[d][c] != INT32_MAX) {
                    atomicMin(e + c, emin[d][c]);
                    atomicMax(e + 3 + c, emax[d][c]);
                }
            }
    }
    __syncthreads();
    if (threadIdx.x == 36 && sext[36]) atomicAdd(o.ext + 36, sext[36]);
    if (threadIdx.x < 36) {
        const int v = sext[threadIdx.x];
        if ((threadIdx.x % 6) < 3) {
            if (v != INT32_MAX) atomicMin(o.ext + threadIdx.x, v);
        } else if (v != INT32_MIN) {
            atomicMax(o.ext + threadIdx.x, v);
        }
    }
}

}  // namespace

vc_status geometry_build(vc_ctx* c, const int32_t* d_label, const double* d_eps) {
    mirror_wait(c);  // the previous geometry's mirror copies are done before anything is reused
    const int64_t nvox = (int64_t)c->nx * c->ny * c->nz;
    cudaStream_t st = c->stream;
    HostTrace tr("geometry");
    DevBuf<unsigned char>& flb = c->geo_flags;
    VC_CUDA(c, flb.alloc(sizeof(Flags)));
    struct { Flags* p; } fl{reinterpret_cast<Flags*>(flb.p)};
    Flags h0{INT32_MAX, INT32_MIN, 0, 0};
    VC_CUDA(c, cudaMemcpyAsync(fl.p, &h0, sizeof(Flags), cudaMemcpyHostToDevice, st));
    const int vblocks = (int)std::min<int64_t>((nvox + 255) / 256, 148 * 16);
    k_validate<<<vblocks, 256, 0, st>>>(nvox, d_label, d_eps, fl.p);
    count_launch(c);
    Flags hf;
    VC_CUDA(c, cudaMemcpyAsync(&hf, fl.p, sizeof(Flags), cudaMemcpyDeviceToHost, st));
    VC_CUDA(c, cudaStreamSynchronize(st));
    if (hf.min_label < 0) return set_err(c, VC_ERR_INPUT, "label < 0");
    if (hf.max_label <= 0) return set_err(c, VC_ERR_INPUT, "empty structure: no conductor voxel");
    if (hf.bad_eps) return set_err(c, VC_ERR_INPUT, "eps_r must be finite and > 0");
    tr.mark("validate");
    const int m = hf.max_label;
    {
        DevBuf<int>& pres = c->geo_pres;
        VC_CUDA(c, pres.alloc((size_t)m + 1));
        VC_CUDA(c, cudaMemsetAsync(pres.p, 0, sizeof(int) * (m + 1), st));
        k_presence<<<vblocks, 256, 0, st>>>(nvox, d_label, pres.p);
        count_launch(c);
        std::vector<int> hp(m + 1);
        VC_CUDA(c, cudaMemcpyAsync(hp.data(), pres.p, sizeof(int) * (m + 1), cudaMemcpyDeviceToHost, st));
        VC_CUDA(c, cudaStreamSynchronize(st));
        for (int i = 1; i <= m; ++i)
            if (!hp[i]) return set_err(c, VC_ERR_INPUT, "conductor ids must be exactly 1..m (missing " + std::to_string(i) + ")");
    }
    tr.mark("presence");
    Geo g;
    g.nx = c->nx;
    g.ny = c->ny;
    g.nz = c->nz;
    g.F[0] = (int64_t)(c->nx + 1) * c->ny * c->nz;
    g.F[1] = (int64_t)c->nx * (c->ny + 1) * c->nz;
    g.F[2] = (int64_t)c->nx * c->ny * (c->nz + 1);
    g.Foff[0] = 0;
    g.Foff[1] = g.F[0];
    g.Foff[2] = g.F[0] + g.F[1];
    const int64_t Ftot = g.F[0] + g.F[1] + g.F[2];
    g.fast = true;
    for (int a = 0; a < 3; ++a) {
        g.fast = g.fast && g.F[a] < (int64_t(1) << 32);
        g.gx[a] = fdiv_make((uint32_t)(c->nx + (a == 0)));
        g.gy[a] = fdiv_make((uint32_t)(c->ny + (a == 1)));
    }
    g.eps_out = c->eps_out;
    g.label = d_label;
    g.eps = d_eps;
    const int64_t ntiles = (Ftot + kTile - 1) / kTile;
    DevBuf<int64_t>&tiles = c->geo_tiles, &total = c->geo_total;
    VC_CUDA(c, tiles.alloc(ntiles));
    VC_CUDA(c, total.alloc(1));
    k_count<<<(unsigned)ntiles, kNT, 0, st>>>(g, Ftot, tiles.p, fl.p);
    k_scan_tiles<<<1, 1024, 0, st>>>(tiles.p, ntiles, total.p);
    count_launch(c, 2);
    int64_t N = 0;
    VC_CUDA(c, cudaMemcpyAsync(&N, total.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    VC_CUDA(c, cudaMemcpyAsync(&hf, fl.p, sizeof(Flags), cudaMemcpyDeviceToHost, st));
    VC_CUDA(c, cudaStreamSynchronize(st));
    if (hf.clash) return set_err(c, VC_ERR_INPUT, "two different conductors share a face");
    tr.mark("count + scan");
    if (N > kSlotIdx) return set_err(c, VC_ERR_UNSUPPORTED, "more than 2^29 panels");

    PanelsDev& P = c->pan;
    VC_CUDA(c, P.axis.alloc(N));
    VC_CUDA(c, P.sign.alloc(N));
    VC_CUDA(c, P.info.alloc(N));
    VC_CUDA(c, P.si.alloc(N));
    VC_CUDA(c, P.sj.alloc(N));
    VC_CUDA(c, P.sk.alloc(N));
    VC_CUDA(c, P.cid.alloc(N));
    VC_CUDA(c, P.eps_d.alloc(N));
    VC_CUDA(c, P.eps_b.alloc(N));
    VC_CUDA(c, P.ibar.alloc(N));
    VC_CUDA(c, P.fc.alloc(N));
    for (int a = 0; a < 3; ++a) VC_CUDA(c, P.slotmap[a].alloc(g.F[a]));
    DevBuf<int>& ext = c->geo_ext;
    VC_CUDA(c, ext.alloc(37));
    std::vector<int> hext(37, 0);
    for (int q = 0; q < 6; ++q)
        for (int t = 0; t < 6; ++t) hext[q * 6 + t] = t < 3 ? INT32_MAX : INT32_MIN;
    VC_CUDA(c, cudaMemcpyAsync(ext.p, hext.data(), 37 * sizeof(int), cudaMemcpyHostToDevice, st));
    Out o;
    o.axis = P.axis.p;
    o.sign = P.sign.p;
    o.info = P.info.p;
    o.si = P.si.p;
    o.sj = P.sj.p;
    o.sk = P.sk.p;
    o.cid = P.cid.p;
    o.ed = P.eps_d.p;
    o.eb = P.eps_b.p;
    o.ibar = P.ibar.p;
    o.fc = P.fc.p;
    for (int a = 0; a < 3; ++a) o.slotmap[a] = P.slotmap[a].p;
    o.area_over_2eps0 = c->dv * c->dv / (2.0 * kEps0);
    o.ext = ext.p;
    tr.mark("allocs");
    k_emit<<<(unsigned)ntiles, kNT, 0, st>>>(g, Ftot, tiles.p, o);
    count_launch(c);
    VC_CUDA(c, cudaMemcpyAsync(hext.data(), ext.p, 37 * sizeof(int), cudaMemcpyDeviceToHost, st));
    // host mirror of the structural fields, on the mirror stream: only its readers (the
    // preconditioner plan, vc_get_panels, the slab partition) wait for it (vc::mirror_wait)
    if (!c->mstream) {
        VC_CUDA(c, cudaStreamCreateWithFlags(&c->mstream, cudaStreamNonBlocking));
        VC_CUDA(c, cudaEventCreateWithFlags(&c->mev, cudaEventDisableTiming));
    }
    VC_CUDA(c, cudaEventRecord(c->mev, st));
    VC_CUDA(c, cudaStreamWaitEvent(c->mstream, c->mev, 0));
    VC_CUDA(c, c->h_axis.resize(N));
    VC_CUDA(c, c->h_si.resize(N));
    VC_CUDA(c, c->h_sj.resize(N));
    VC_CUDA(c, c->h_sk.resize(N));
    VC_CUDA(c, c->h_cid.resize(N));
    cudaStream_t ms = c->mstream;
    VC_CUDA(c, cudaMemcpyAsync(c->h_axis.data(), P.axis.p, N, cudaMemcpyDeviceToHost, ms));
    VC_CUDA(c, cudaMemcpyAsync(c->h_si.data(), P.si.p, N * 4, cudaMemcpyDeviceToHost, ms));
    VC_CUDA(c, cudaMemcpyAsync(c->h_sj.data(), P.sj.p, N * 4, cudaMemcpyDeviceToHost, ms));
    VC_CUDA(c, cudaMemcpyAsync(c->h_sk.data(), P.sk.p, N * 4, cudaMemcpyDeviceToHost, ms));
    VC_CUDA(c, cudaMemcpyAsync(c->h_cid.data(), P.cid.p, N * 4, cudaMemcpyDeviceToHost, ms));
    VC_CUDA(c, cudaEventRecord(c->mev, ms));
    VC_CUDA(c, cudaStreamSynchronize(st));
    VC_CUDA(c, cudaGetLastError());
    for (int kind = 0; kind < 2; ++kind)
        for (int a = 0; a < 3; ++a)
            for (int t = 0; t < 3; ++t) {
                c->ext[kind][a][0][t] = hext[(kind * 3 + a) * 6 + t];
                c->ext[kind][a][1][t] = hext[(kind * 3 + a) * 6 + 3 + t];
            }
    tr.mark("emit + host mirrors");
    const int64_t Nc = hext[36];  // counted in k_emit
    c->N = N;
    c->Nc = Nc;
    c->Nd = N - Nc;
    c->m = m;
    return VC_OK;
}

}  // namespace vc
