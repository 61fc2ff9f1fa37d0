#include <cstdio>
// precond.cu -- block-diagonal-diagonal preconditioner (Eq. 14; DESIGN.md a9/a10).
//
// R_BD: the bounding box is split into boxes of Nvx x Nvy x Nvz voxels; every box's
// conductor panels (reading O9; a panel belongs to box min(slot_a / Nv_a, nbox_a - 1)) form a
// dense block of Eq. (5) interactions, which is inverted.  Boxes whose panel configurations are
// identical up to translation share one inverted block ("only unique blocks are
// stored").  R_D = Ī^{-1} on dielectric rows.
// Structure (box assignment, signatures, dedup) is host C++; block entries, inversion and the
// apply are CUDA kernels.
#include <algorithm>
#include <cstring>
#include <unordered_map>

#include "ctx.h"
#include "kgen.cuh"

namespace vc {

struct Precond {
    int kind = 3;
    int nbox = 0, nuniq = 0;
    int max_n = 0;
    DevBuf<int32_t> box_start, box_n, box_uid;  // per non-empty box
    DevBuf<int32_t> ubox_start, ubox_list;       // boxes of each unique block (CSR)
    DevBuf<int32_t> btile_b, btile_r0;           // per-box apply tiles (box, first row)
    int nbtile = 0;
    DevBuf<int32_t> stile_b, stile_r0;           // symmetric-apply tiles (box, first of kPsRows rows)
    int nstile = 0;
    DevBuf<int32_t> tile_u, tile_r0, tile_q0;    // apply tiles: (unique block, first row, first box)
    int ntile = 0;
    DevBuf<int32_t> panel_ids;                   // conductor panels sorted by box
    DevBuf<int64_t> uniq_off;                    // offset of each unique block (doubles)
    DevBuf<int32_t> uniq_n, uniq_list_off;
    DevBuf<int32_t> uniq_axis, uniq_slot;        // local panel descriptors (3 ints per slot)
    DevBuf<double> blocks;                       // inverted blocks, row-major
    DevBuf<double> diag_inv;                     // per panel: 1/Ī (diel), 1/P_kk (diag-only)
    int64_t block_doubles = 0;
};

namespace {

struct PcTab {
    const double* t;
    int dim[3];
    int pair[3][3];
};

// Block entries P_kl of Eq. (5): looked up in the near-field tables the kernel build cut from
// its octant tables (the same device generator, already scaled by dv^3 / (4 pi eps0)).  Octant
// index per axis of the signed slot offset d: |t| = |d + s| with s = c_a - c_b (App. B).
__global__ void k_pc_fill(const int32_t* __restrict__ un, const int64_t* __restrict__ uoff,
                          const int32_t* __restrict__ ulist, const int32_t* __restrict__ uaxis,
                          const int32_t* __restrict__ uslot, double* __restrict__ blocks,
                          PcTab tab) {
    const int u = blockIdx.y;
    const int n = un[u];
    const int64_t nn = (int64_t)n * n;
    double* B = blocks + uoff[u];
    const int l0 = ulist[u];
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nn;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(e / n), j = (int)(e % n);
        const int ai = uaxis[l0 + i], aj = uaxis[l0 + j];
        const int dx = uslot[3 * (l0 + i)] - uslot[3 * (l0 + j)];
        const int dy = uslot[3 * (l0 + i) + 1] - uslot[3 * (l0 + j) + 1];
        const int dz = uslot[3 * (l0 + i) + 2] - uslot[3 * (l0 + j) + 2];
        const int d[3] = {dx, dy, dz};
        int o[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int s2 = c2(ai, a) - c2(aj, a);
            const int t2 = 2 * d[a] + s2;
            o[a] = ((t2 < 0 ? -t2 : t2) - (s2 != 0)) >> 1;
        }
        B[e] = tab.t[(size_t)tab.pair[ai][aj] * tab.dim[0] * tab.dim[1] * tab.dim[2] +
                     ((size_t)o[2] * tab.dim[1] + o[1]) * tab.dim[0] + o[0]];
    }
}

// Conventional block-diagonal blocks (vc_build_opts.precond = 4; the comparator of P:155-157):
// every panel of a box, conductor rows from Eq. (5), dielectric rows from Eq. (6) with the Ī of
// Eq. (7) on the diagonal -- the same rows as the operator (Eq. 4) restricted to the box.  One
// block per box (no dedup: a dielectric row also depends on its permittivities), entries from the
// device closed forms (kgen.cuh kappa), scaled like the operator.
__global__ void k_pc_fill_conv(const int32_t* __restrict__ bn, const int64_t* __restrict__ uoff,
                               const int32_t* __restrict__ bstart, const int32_t* __restrict__ pids,
                               const int8_t* __restrict__ axis, const int32_t* __restrict__ si,
                               const int32_t* __restrict__ sj, const int32_t* __restrict__ sk,
                               const int8_t* __restrict__ info, const double* __restrict__ ibar,
                               double pscale, double escale, double* __restrict__ blocks) {
    const int b = blockIdx.y;
    const int n = bn[b], s0 = bstart[b];
    const int64_t nn = (int64_t)n * n;
    double* B = blocks + uoff[b];
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nn;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(e / n), j = (int)(e % n);
        const int pi = pids[s0 + i], pj = pids[s0 + j];
        const bool diel = info[pi] & 1;
        double v = kappa(diel ? 1 : 0, axis[pi], axis[pj], si[pi] - si[pj], sj[pi] - sj[pj], sk[pi] - sk[pj]);
        if (diel) {
            v *= (info[pi] & 2) ? -escale : escale;  // s_k
            if (i == j) v += ibar[pi];               // Eq. (7)
        } else {
            v *= pscale;
        }
        B[e] = v;
    }
}

// In-place Gauss-Jordan inverse of an SPD block (no pivoting needed), one CTA (32 x 16
// threads) per unique block.  The block is worked on in shared memory when it fits (copied in
// and out once), else in global memory (L2-resident); the 2-D thread layout avoids index
// divisions in the n^2 update of every pivot step.
__global__ void __launch_bounds__(512) k_pc_invert(const int32_t* __restrict__ un,
                                                   const int64_t* __restrict__ uoff,
                                                   double* __restrict__ blocks, int smem_elems,
                                                   int sweep_elems, int symmetrize) {
    extern __shared__ double sh[];
    const int u = blockIdx.x;
    const int n = un[u];
    if ((int64_t)n * (n + 1) / 2 + n <= sweep_elems) return;  // done by k_pc_sweep
    double* G = blocks + uoff[u];
    double* rowk = sh;
    double* colk = sh + n;
    const bool in_smem = (int64_t)n * n + 2 * n <= smem_elems;
    double* A = in_smem ? sh + 2 * n : G;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 columns x 16 rows
    if (in_smem) {
        for (int64_t e = threadIdx.x; e < (int64_t)n * n; e += blockDim.x) A[e] = G[e];
    }
    for (int k = 0; k < n; ++k) {
        __syncthreads();
        const double ip = 1.0 / A[(int64_t)k * n + k];
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            rowk[j] = j == k ? ip : A[(int64_t)k * n + j] * ip;
            colk[j] = A[(int64_t)j * n + k];
        }
        __syncthreads();
        for (int i = ty; i < n; i += 16) {
            double* Ai = A + (int64_t)i * n;
            const double ci = colk[i];
            for (int j = tx; j < n; j += 32) {
                if (i == k) Ai[j] = rowk[j];
                else if (j == k) Ai[j] = -ci * ip;
                else Ai[j] = fma(-ci, rowk[j], Ai[j]);
            }
        }
    }
    __syncthreads();
    if (symmetrize) {  // SPD block: make the inverse exactly symmetric (k_pc_apply_sym reads R^T)
        for (int64_t e = threadIdx.x; e < (int64_t)n * n; e += blockDim.x) {
            const int i = (int)(e / n), j = (int)(e % n);
            if (i < j) {
                const double v = 0.5 * (A[(int64_t)i * n + j] + A[(int64_t)j * n + i]);
                A[(int64_t)i * n + j] = v;
                A[(int64_t)j * n + i] = v;
            }
        }
        __syncthreads();
    }
    if (in_smem) {
        for (int64_t e = threadIdx.x; e < (int64_t)n * n; e += blockDim.x) G[e] = A[e];
    }
}

// Symmetric inverse by the sweep operator (Goodnight's SWEEP), one CTA per unique block whose
// packed lower triangle fits in shared memory.  Sweeping pivot k with d = a_kk:
//   a_kk <- -1/d,  a_ik = a_ki <- a_ik / d,  a_ij <- a_ij - a_ik a_kj / d   (i, j != k)
// keeps the matrix symmetric at every step (so half the storage and half the updates of the
// Gauss-Jordan kernel above), and sweeping every pivot of an SPD block (no pivoting needed)
// leaves -A^{-1}.  Packed index of (i >= j): i (i + 1) / 2 + j.  Warps take rows, lanes columns.
__global__ void __launch_bounds__(1024) k_pc_sweep(const int32_t* __restrict__ un,
                                                  const int64_t* __restrict__ uoff,
                                                  double* __restrict__ blocks, int smem_elems) {
    extern __shared__ double sh[];
    const int n = un[blockIdx.x];
    const int64_t np = (int64_t)n * (n + 1) / 2;
    if (np + n > smem_elems) return;  // left to k_pc_invert (global-memory path)
    double* G = blocks + uoff[blockIdx.x];
    double* P = sh;
    double* ck = sh + np;
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = wp; i < n; i += nw) {
        const int base = i * (i + 1) / 2;
        for (int j = lane; j <= i; j += 32) P[base + j] = G[(int64_t)i * n + j];
    }
    for (int k = 0; k < n; ++k) {
        __syncthreads();
        const int bk = k * (k + 1) / 2;
        for (int i = threadIdx.x; i < n; i += blockDim.x)
            ck[i] = i >= k ? P[i * (i + 1) / 2 + k] : P[bk + i];
        __syncthreads();
        const double id = 1.0 / ck[k];
        for (int i = wp; i < n; i += nw) {
            const int base = i * (i + 1) / 2;
            const double ci = ck[i], cid = ci * id;
            if (i == k) {
                for (int j = lane; j < k; j += 32) P[base + j] = ck[j] * id;
                if (lane == 0) P[base + k] = -id;
            } else {
                for (int j = lane; j <= i; j += 32)
                    P[base + j] = j == k ? cid : fma(-cid, ck[j], P[base + j]);
            }
        }
    }
    __syncthreads();
    for (int i = wp; i < n; i += nw) {
        const int base = i * (i + 1) / 2;
        for (int j = lane; j <= i; j += 32) {
            const double v = -P[base + j];
            G[(int64_t)i * n + j] = v;
            G[(int64_t)j * n + i] = v;
        }
    }
}

// z = R_D r on all rows (dielectric: r/Ī; conductor: r * diag_inv (diag-only) or 0)
__global__ void k_pc_diag(int64_t N, const double* __restrict__ r, const double* __restrict__ dinv,
                          double* __restrict__ z) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x)
        z[i] = r[i] * dinv[i];
}

// z_b = R_u r_b grouped by unique block: a CTA holds kPcRows rows of R_u in shared memory and
// applies them to every box b that uses R_u (each R element read once per apply; 8 lanes per
// row, shuffle-reduced)
constexpr int kPcRows = 32;
constexpr int kPcBoxes = 8;  // boxes per CTA (a block shared by many boxes is split over CTAs)
__global__ void __launch_bounds__(256) k_pc_apply_grouped(
    const int32_t* __restrict__ tile_u, const int32_t* __restrict__ tile_r0,
    const int32_t* __restrict__ tile_q0,
    const int32_t* __restrict__ un, const int64_t* __restrict__ uoff,
    const int32_t* __restrict__ ubs, const int32_t* __restrict__ ubl,
    const int32_t* __restrict__ bstart, const int32_t* __restrict__ pids,
    const double* __restrict__ blocks, const double* __restrict__ r, double* __restrict__ z) {
    extern __shared__ double sh[];
    const int u = tile_u[blockIdx.x], r0 = tile_r0[blockIdx.x];
    const int n = un[u];
    const int rows = min(kPcRows, n - r0);
    double* Rt = sh;              // [rows][n]
    double* rb = sh + kPcRows * n;  // [n]
    const double* R = blocks + uoff[u] + (int64_t)r0 * n;
    for (int e = threadIdx.x; e < rows * n; e += blockDim.x) Rt[e] = R[e];
    const int row = threadIdx.x >> 3, part = threadIdx.x & 7;
    const int q1 = min(ubs[u + 1], ubs[u] + tile_q0[blockIdx.x] + kPcBoxes);
    for (int q = ubs[u] + tile_q0[blockIdx.x]; q < q1; ++q) {
        const int b = ubl[q];
        const int s0 = bstart[b];
        __syncthreads();
        for (int j = threadIdx.x; j < n; j += blockDim.x) rb[j] = r[pids[s0 + j]];
        __syncthreads();
        double acc = 0.0;
        if (row < rows)
            for (int j = part; j < n; j += 8) acc = fma(Rt[row * n + j], rb[j], acc);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        acc += __shfl_xor_sync(0xffffffffu, acc, 4);
        if (part == 0 && row < rows) z[pids[s0 + r0 + row]] = acc;
    }
}

// z_b = R_u r_b with one CTA per (box, 32 rows): r_b gathered once into shared memory, each
// warp takes rows and reads them straight from the block table (L2-resident: the unique blocks
// of C4 total ~13 MB), lanes strided over the columns, shuffle-reduced.  No R staging and no
// per-box serial loop, so every box's latency overlaps (measured against the grouped kernel).
// NC columns (the lockstep solver's pair): each R row read once for all of them.
constexpr int kPbRows = 32;
struct PcCols {
    const double* r[2];
    double* z[2];
};
template <int NC>
__global__ void __launch_bounds__(256) k_pc_apply_box(
    const int32_t* __restrict__ tb, const int32_t* __restrict__ tr0,
    const int32_t* __restrict__ bstart, const int32_t* __restrict__ bn,
    const int32_t* __restrict__ buid, const int64_t* __restrict__ uoff,
    const int32_t* __restrict__ pids, const double* __restrict__ blocks, PcCols cols) {
    extern __shared__ double rb[];  // [NC][n]
    const int b = tb[blockIdx.x], r0 = tr0[blockIdx.x];
    const int n = bn[b], s0 = bstart[b];
    const double* __restrict__ R = blocks + uoff[buid[b]];
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const int p = pids[s0 + j];
#pragma unroll
        for (int q = 0; q < NC; ++q) rb[q * n + j] = cols.r[q][p];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int r1 = min(n, r0 + kPbRows);
    for (int row = r0 + w; row < r1; row += nw) {
        const double* __restrict__ Rr = R + (int64_t)row * n;
        double acc[NC];
#pragma unroll
        for (int q = 0; q < NC; ++q) acc[q] = 0.0;
#pragma unroll 8
        for (int j = lane; j < n; j += 32) {
            const double rv = __ldg(Rr + j);
#pragma unroll
            for (int q = 0; q < NC; ++q) acc[q] = fma(rv, rb[q * n + j], acc[q]);
        }
#pragma unroll
        for (int q = 0; q < NC; ++q) {
            for (int o = 16; o; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
            if (lane == 0) cols.z[q][pids[s0 + row]] = acc[q];
        }
    }
}

// Symmetric blocks (the proposed R_BD: SPD blocks inverted by the symmetric sweep, so R = R^T
// exactly): thread per row, z_row = sum_j R[j][row] r_j reads R column-wise, i.e. row j of the
// stored block across consecutive threads -- coalesced, no shuffle reduction -- with r_j
// broadcast from shared memory.  CTA = (box, kPsRows rows); all columns of the box in one pass.
constexpr int kPsRows = 128;
template <int NC>
__global__ void __launch_bounds__(kPsRows) k_pc_apply_sym(
    const int32_t* __restrict__ tb, const int32_t* __restrict__ tr0,
    const int32_t* __restrict__ bstart, const int32_t* __restrict__ bn,
    const int32_t* __restrict__ buid, const int64_t* __restrict__ uoff,
    const int32_t* __restrict__ pids, const double* __restrict__ blocks, PcCols cols) {
    extern __shared__ double rb[];  // [NC][n]
    const int b = tb[blockIdx.x], r0 = tr0[blockIdx.x];
    const int n = bn[b], s0 = bstart[b];
    const double* __restrict__ R = blocks + uoff[buid[b]];
    for (int j = threadIdx.x; j < n; j += kPsRows) {
        const int p = pids[s0 + j];
#pragma unroll
        for (int q = 0; q < NC; ++q) rb[q * n + j] = cols.r[q][p];
    }
    __syncthreads();
    const int row = r0 + threadIdx.x;
    if (row >= n) return;
    double acc[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) acc[q] = 0.0;
    const double* __restrict__ Rc = R + row;
#pragma unroll 4
    for (int j = 0; j < n; ++j) {
        const double rv = __ldg(Rc + (int64_t)j * n);
#pragma unroll
        for (int q = 0; q < NC; ++q) acc[q] = fma(rv, rb[q * n + j], acc[q]);
    }
    const int p = pids[s0 + row];
#pragma unroll
    for (int q = 0; q < NC; ++q) cols.z[q][p] = acc[q];
}

// per-panel diagonal of R: 1/Ī on dielectric rows; conductor rows 1 (none), 1/P_self
// (diagonal-only option) or 0 (their block of R_BD writes them)
__global__ void k_pc_dinv(int64_t n, const int32_t* __restrict__ cid, const double* __restrict__ ibar,
                          int kind, double pself, double* __restrict__ dinv) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (kind == 4) dinv[i] = 0.0;  // every row lies in a box block
        else if (cid[i] == 0) dinv[i] = kind == 1 ? 1.0 : 1.0 / ibar[i];
        else dinv[i] = kind == 1 ? 1.0 : (kind == 2 ? 1.0 / pself : 0.0);
    }
}


}  // namespace

void precond_free(vc_ctx* c) {
    delete c->pc;
    c->pc = nullptr;
}

// Host bookkeeping of the block-diagonal preconditioner: boxes of the conductor panels,
// their canonical signatures and the unique blocks (hash-first dedup), the per-box and
// grouped-apply tile lists.  Pure host work on the immutable panel mirrors, so
// vc_build_operator runs it on a helper thread beside the kernel-table build (one rank).
struct PcPlan {
    int nbox = 0, maxn = 0;
    int64_t total = 0;
    std::vector<int32_t> bcount, bstart, sorted, buid, un, ulist_off, uaxis, uslot;
    std::vector<int64_t> uoff;
};

void pc_plan_compute(const vc_ctx* c, const int32_t box_in[3], int64_t N, PcPlan& P, bool all_panels) {
    mirror_wait(c);  // reads the host panel mirror
    auto G = [&](int64_t i) { return c->world > 1 ? c->h_gidx[i] : i; };  // local -> global
    int nv[3], nb[3];
    const int dims[3] = {c->nx, c->ny, c->nz};
    for (int a = 0; a < 3; ++a) {
        nv[a] = box_in[a] > 0 ? box_in[a] : 10;
        nb[a] = std::max(1, (dims[a] + nv[a] - 1) / nv[a]);
    }
    // box of every conductor panel; stable counting sort by box
    std::vector<int64_t> pbox;
    std::vector<int32_t> cond;
    cond.reserve(c->Nc);
    for (int64_t i = 0; i < N; ++i)
        if (all_panels || c->h_cid[G(i)] > 0) cond.push_back((int32_t)i);  // local indices
    // dense box table (the box grid is small: (N_x/N_v)(N_y/N_v)(N_z/N_v) entries)
    std::vector<int32_t> box_index((size_t)nb[0] * nb[1] * nb[2], -1);
    std::vector<int64_t> box_keys;
    std::vector<int32_t> pb(cond.size());
    for (size_t q = 0; q < cond.size(); ++q) {
        const int64_t p = G(cond[q]);
        const int s[3] = {c->h_si[p], c->h_sj[p], c->h_sk[p]};
        int64_t bx[3];
        for (int a = 0; a < 3; ++a) bx[a] = std::min<int64_t>(s[a] / nv[a], nb[a] - 1);
        const int64_t key = (bx[2] * nb[1] + bx[1]) * nb[0] + bx[0];
        int32_t& bi = box_index[key];
        if (bi < 0) {
            bi = (int32_t)box_keys.size();
            box_keys.push_back(key);
        }
        pb[q] = bi;
    }
    const int nbox = (int)box_keys.size();
    std::vector<int32_t> bcount(nbox, 0), bstart(nbox + 1, 0);
    for (int32_t b : pb) bcount[b]++;
    for (int b = 0; b < nbox; ++b) bstart[b + 1] = bstart[b] + bcount[b];
    std::vector<int32_t> sorted(cond.size()), fillp(bstart.begin(), bstart.end() - 1);
    for (size_t q = 0; q < cond.size(); ++q) sorted[fillp[pb[q]]++] = cond[q];
    // signatures (axis + slot relative to the box origin, canonical order) -> unique blocks:
    // a 64-bit hash per box, full comparison against the stored signature on a hash match
    std::unordered_map<uint64_t, std::vector<int32_t>> by_hash;  // hash -> unique ids
    std::vector<int32_t> buid(nbox), un, ulist_off, uaxis, uslot;
    std::vector<int64_t> uoff;
    int64_t total = 0;
    int maxn = 0;
    for (int b = 0; b < nbox; ++b) {
        const int64_t key = box_keys[b];
        const int64_t bx = key % nb[0], by = (key / nb[0]) % nb[1], bz = key / ((int64_t)nb[0] * nb[1]);
        const int org[3] = {(int)(bx * nv[0]), (int)(by * nv[1]), (int)(bz * nv[2])};
        const int n = bcount[b];
        auto sig_at = [&](int q, int t) -> int32_t {  // t: 0 axis, 1..3 slot - origin
            const int64_t p = G(sorted[bstart[b] + q]);
            return t == 0 ? c->h_axis[p] : (t == 1 ? c->h_si[p] - org[0] : (t == 2 ? c->h_sj[p] - org[1] : c->h_sk[p] - org[2]));
        };
        uint64_t h = 1469598103934665603ull ^ (uint64_t)n;
        for (int q = 0; q < n; ++q)
            for (int t = 0; t < 4; ++t) {
                h ^= (uint32_t)sig_at(q, t);
                h *= 1099511628211ull;
            }
        int id = -1;
        auto& cand = by_hash[all_panels ? (uint64_t)b : h];  // conventional blocks: no dedup
        for (int u : cand) {
            if (un[u] != n) continue;
            bool same = true;
            const int l0 = ulist_off[u];
            for (int q = 0; q < n && same; ++q)
                same = uaxis[l0 + q] == sig_at(q, 0) && uslot[3 * (l0 + q)] == sig_at(q, 1) &&
                       uslot[3 * (l0 + q) + 1] == sig_at(q, 2) && uslot[3 * (l0 + q) + 2] == sig_at(q, 3);
            if (same) {
                id = u;
                break;
            }
        }
        if (id < 0) {
            id = (int)un.size();
            un.push_back(n);
            ulist_off.push_back((int32_t)uaxis.size());
            uoff.push_back(total);
            total += (int64_t)n * n;
            maxn = std::max(maxn, n);
            for (int q = 0; q < n; ++q) {
                uaxis.push_back(sig_at(q, 0));
                uslot.push_back(sig_at(q, 1));
                uslot.push_back(sig_at(q, 2));
                uslot.push_back(sig_at(q, 3));
            }
            cand.push_back(id);
        }
        buid[b] = id;
    }
    P.nbox = nbox;
    P.maxn = maxn;
    P.total = total;
    P.bcount = std::move(bcount);
    P.bstart = std::move(bstart);
    P.sorted = std::move(sorted);
    P.buid = std::move(buid);
    P.un = std::move(un);
    P.ulist_off = std::move(ulist_off);
    P.uaxis = std::move(uaxis);
    P.uslot = std::move(uslot);
    P.uoff = std::move(uoff);
}

vc_status precond_build(vc_ctx* c, const int32_t box_in[3], int kind, const PcPlan* pre) {
    if (!c->pc) c->pc = new Precond();  // kept across builds: its buffers are grow-only
    Precond* pc = c->pc;
    pc->kind = kind;
    pc->nbox = pc->nuniq = pc->max_n = 0;
    pc->block_doubles = 0;
    c->stats.precond_doubles = 0;
    cudaStream_t st = c->stream;
    HostTrace tr("precond");
    const int64_t N = c->NL;  // this rank's panels (boxes never straddle ranks)
    const double fpe = 4.0 * kPi * kEps0;
    const double pscale = c->dv * c->dv * c->dv / fpe;
    // diagonal part (on the device, from the rank's panel arrays)
    // self term of a unit square (textbook), used only for the diagonal-only option
    const double pself = pscale * ((4.0 / 3.0) * (1.0 - std::sqrt(2.0)) + 4.0 * std::log(1.0 + std::sqrt(2.0)));
    VC_CUDA(c, pc->diag_inv.alloc(std::max<int64_t>(1, N)));
    if (N) {
        const bool loc = c->world > 1;
        k_pc_dinv<<<(unsigned)std::min<int64_t>((N + 255) / 256, 148 * 8), 256, 0, st>>>(
            N, loc ? c->lp.cid.p : c->pan.cid.p, loc ? c->lp.ibar.p : c->pan.ibar.p, kind, pself,
            pc->diag_inv.p);
        count_launch(c);
    }
    tr.mark("diagonal");
    if (kind != 3 && kind != 4) {
        VC_CUDA(c, cudaStreamSynchronize(st));
        return VC_OK;
    }
    const bool conv = kind == 4;
    if (conv && c->world > 1)
        return set_err(c, VC_ERR_UNSUPPORTED, "the conventional block-diagonal preconditioner runs on one rank");
    PcPlan own;
    if (!pre || conv) pc_plan_compute(c, box_in, N, own, conv);
    const PcPlan& P = (pre && !conv) ? *pre : own;
    const int nbox = P.nbox, maxn = P.maxn;
    const int64_t total = P.total;
    const std::vector<int32_t>&bcount = P.bcount, &bstart = P.bstart, &sorted = P.sorted,
                          &buid = P.buid, &un = P.un, &ulist_off = P.ulist_off,
                          &uaxis = P.uaxis, &uslot = P.uslot;
    const std::vector<int64_t>& uoff = P.uoff;
    tr.mark("signatures");
    if (tr.on) {
        double f3 = 0;
        int big = 0;
        for (int n : un) {
            f3 += (double)n * n * n;
            big += (size_t)n * n + 2 * n > 26 * 1024;
        }
        fprintf(stderr, "[vc precond] boxes %d unique %zu max_n %d sum n^3 %.3g (%d not in smem)\n",
                nbox, un.size(), maxn, f3, big);
    }
    if ((size_t)maxn * (kPcRows + 1) * sizeof(double) > 220 * 1024)
        return set_err(c, VC_ERR_UNSUPPORTED, "preconditioner block too large (" + std::to_string(maxn) + " panels in one box); use smaller boxes");
    pc->nbox = nbox;
    pc->nuniq = (int)un.size();
    pc->max_n = maxn;
    pc->block_doubles = total;
    c->stats.precond_doubles = total;
    VC_CUDA(c, pc->box_start.alloc(std::max(1, nbox)));
    VC_CUDA(c, pc->box_n.alloc(std::max(1, nbox)));
    VC_CUDA(c, pc->box_uid.alloc(std::max(1, nbox)));
    VC_CUDA(c, pc->panel_ids.alloc(std::max<size_t>(1, sorted.size())));
    VC_CUDA(c, pc->uniq_off.alloc(std::max<size_t>(1, uoff.size())));
    VC_CUDA(c, pc->uniq_n.alloc(std::max<size_t>(1, un.size())));
    VC_CUDA(c, pc->uniq_list_off.alloc(std::max<size_t>(1, un.size())));
    VC_CUDA(c, pc->uniq_axis.alloc(std::max<size_t>(1, uaxis.size())));
    VC_CUDA(c, pc->uniq_slot.alloc(std::max<size_t>(1, uslot.size())));
    VC_CUDA(c, pc->blocks.alloc(std::max<int64_t>(1, total)));
    // uploads are gathered into one host staging area and sent from pinned memory in one batch
    // of async copies (a pageable cudaMemcpyAsync synchronises the stream first: sixteen of them
    // serialised the host behind the kernel tables)
    std::vector<char> stage;
    std::vector<std::pair<void*, std::pair<size_t, size_t>>> ups;  // dst, (offset, bytes)
    auto up = [&](void* d, const void* h, size_t bytes) {
        if (bytes) {
            const size_t off = (stage.size() + 15) & ~(size_t)15;
            stage.resize(off + bytes);
            memcpy(stage.data() + off, h, bytes);
            ups.push_back({d, {off, bytes}});
        }
        return cudaSuccess;
    };
    VC_CUDA(c, up(pc->box_start.p, bstart.data(), 4 * nbox));
    VC_CUDA(c, up(pc->box_n.p, bcount.data(), 4 * nbox));
    VC_CUDA(c, up(pc->box_uid.p, buid.data(), 4 * nbox));
    {   // unique block -> its boxes (CSR) and the grouped-apply tiles
        const int nu = (int)un.size();
        std::vector<int32_t> ubs(nu + 1, 0), ubl(nbox), fillq;
        for (int b = 0; b < nbox; ++b) ubs[buid[b] + 1]++;
        for (int u = 0; u < nu; ++u) ubs[u + 1] += ubs[u];
        fillq.assign(ubs.begin(), ubs.end() - 1);
        for (int b = 0; b < nbox; ++b) ubl[fillq[buid[b]]++] = b;
        std::vector<int32_t> tu, tr, tq;
        for (int u = 0; u < nu; ++u)
            for (int r0 = 0; r0 < un[u]; r0 += kPcRows)
                for (int q0 = 0; q0 < ubs[u + 1] - ubs[u]; q0 += kPcBoxes) {
                    tu.push_back(u);
                    tr.push_back(r0);
                    tq.push_back(q0);
                }
        pc->ntile = (int)tu.size();
        std::vector<int32_t> bt, br;
        for (int b = 0; b < nbox; ++b)
            for (int r0 = 0; r0 < bcount[b]; r0 += kPbRows) {
                bt.push_back(b);
                br.push_back(r0);
            }
        pc->nbtile = (int)bt.size();
        std::vector<int32_t> sb, sr;
        for (int b = 0; b < nbox; ++b)
            for (int r0 = 0; r0 < bcount[b]; r0 += kPsRows) {
                sb.push_back(b);
                sr.push_back(r0);
            }
        pc->nstile = (int)sb.size();
        VC_CUDA(c, pc->stile_b.alloc(std::max<size_t>(1, sb.size())));
        VC_CUDA(c, pc->stile_r0.alloc(std::max<size_t>(1, sr.size())));
        VC_CUDA(c, up(pc->stile_b.p, sb.data(), 4 * sb.size()));
        VC_CUDA(c, up(pc->stile_r0.p, sr.data(), 4 * sr.size()));
        VC_CUDA(c, pc->btile_b.alloc(std::max<size_t>(1, bt.size())));
        VC_CUDA(c, pc->btile_r0.alloc(std::max<size_t>(1, br.size())));
        VC_CUDA(c, up(pc->btile_b.p, bt.data(), 4 * bt.size()));
        VC_CUDA(c, up(pc->btile_r0.p, br.data(), 4 * br.size()));
        VC_CUDA(c, pc->ubox_start.alloc(nu + 1));
        VC_CUDA(c, pc->ubox_list.alloc(std::max(1, nbox)));
        VC_CUDA(c, pc->tile_u.alloc(std::max<size_t>(1, tu.size())));
        VC_CUDA(c, pc->tile_r0.alloc(std::max<size_t>(1, tr.size())));
        VC_CUDA(c, pc->tile_q0.alloc(std::max<size_t>(1, tq.size())));
        VC_CUDA(c, up(pc->tile_q0.p, tq.data(), 4 * tq.size()));
        VC_CUDA(c, up(pc->ubox_start.p, ubs.data(), 4 * (nu + 1)));
        VC_CUDA(c, up(pc->ubox_list.p, ubl.data(), 4 * nbox));
        VC_CUDA(c, up(pc->tile_u.p, tu.data(), 4 * tu.size()));
        VC_CUDA(c, up(pc->tile_r0.p, tr.data(), 4 * tr.size()));
    }
    VC_CUDA(c, up(pc->panel_ids.p, sorted.data(), 4 * sorted.size()));
    VC_CUDA(c, up(pc->uniq_off.p, uoff.data(), 8 * uoff.size()));
    VC_CUDA(c, up(pc->uniq_n.p, un.data(), 4 * un.size()));
    VC_CUDA(c, up(pc->uniq_list_off.p, ulist_off.data(), 4 * ulist_off.size()));
    VC_CUDA(c, up(pc->uniq_axis.p, uaxis.data(), 4 * uaxis.size()));
    VC_CUDA(c, up(pc->uniq_slot.p, uslot.data(), 4 * uslot.size()));
    VC_CUDA(c, c->pc_stage.resize(std::max<size_t>(1, stage.size())));
    if (!stage.empty()) memcpy(c->pc_stage.data(), stage.data(), stage.size());
    for (const auto& u : ups)
        VC_CUDA(c, cudaMemcpyAsync(u.first, c->pc_stage.data() + u.second.first, u.second.second,
                                   cudaMemcpyHostToDevice, st));
    if (pc->nuniq > 0) {
        dim3 g(std::max(1, std::min(64, (maxn * maxn + 255) / 256)), pc->nuniq);
        PcTab tab;
        tab.t = c->pcTab.p;
        for (int a = 0; a < 3; ++a) {
            tab.dim[a] = c->pcTabDim[a];
            for (int b = 0; b < 3; ++b) tab.pair[a][b] = c->pcPair[a][b];
        }
        if (conv) {  // one block per box, all panels, Eq. (4) rows; Gauss-Jordan (not symmetric)
            dim3 gb(std::max(1, std::min(64, (maxn * maxn + 255) / 256)), nbox);
            k_pc_fill_conv<<<gb, 256, 0, st>>>(pc->box_n.p, pc->uniq_off.p, pc->box_start.p, pc->panel_ids.p,
                                               c->pan.axis.p, c->pan.si.p, c->pan.sj.p, c->pan.sk.p,
                                               c->pan.info.p, c->pan.ibar.p, pscale,
                                               c->dv * c->dv / fpe, pc->blocks.p);
            const size_t cap = (size_t)max_dyn_smem() - 1024;
            const size_t sh = std::min(cap, sizeof(double) * ((size_t)maxn * maxn + 2 * maxn));
            if (sh > 48 * 1024) VC_CUDA(c, grant_max_dyn_smem(k_pc_invert, max_dyn_smem()));
            k_pc_invert<<<pc->nuniq, 512, sh, st>>>(pc->uniq_n.p, pc->uniq_off.p, pc->blocks.p,
                                                    (int)(sh / sizeof(double)), 0, 0);
            count_launch(c, 2);
            VC_CUDA(c, cudaGetLastError());
            VC_CUDA(c, cudaStreamSynchronize(st));
            return VC_OK;
        }
        k_pc_fill<<<g, 256, 0, st>>>(pc->uniq_n.p, pc->uniq_off.p, pc->uniq_list_off.p,
                                     pc->uniq_axis.p, pc->uniq_slot.p, pc->blocks.p, tab);
        // sweep (packed, shared memory) for every block it fits; Gauss-Jordan in global memory
        // (L2-resident) for the rest
        const size_t cap = (size_t)max_dyn_smem() - 1024;
        const size_t sw = std::min(cap, sizeof(double) * ((size_t)maxn * (maxn + 1) / 2 + maxn));
        if (sw > 48 * 1024) VC_CUDA(c, grant_max_dyn_smem(k_pc_sweep, max_dyn_smem()));
        k_pc_sweep<<<pc->nuniq, 1024, sw, st>>>(pc->uniq_n.p, pc->uniq_off.p, pc->blocks.p,
                                               (int)(sw / sizeof(double)));
        if ((size_t)maxn * (maxn + 1) / 2 + maxn > sw / sizeof(double)) {
            const size_t sh = 2 * sizeof(double) * maxn;
            k_pc_invert<<<pc->nuniq, 512, sh, st>>>(pc->uniq_n.p, pc->uniq_off.p, pc->blocks.p,
                                                    (int)(sh / sizeof(double)),
                                                    (int)(sw / sizeof(double)), 1);
            count_launch(c);
        }
        count_launch(c, 2);
    }
    if (tr.on) {
        cudaStreamSynchronize(st);
        tr.mark("uploads + fill + invert");
    }
    VC_CUDA(c, cudaStreamSynchronize(st));
    VC_CUDA(c, cudaGetLastError());
    return VC_OK;
}

// VC_PC_ROWWARP=1: the warp-per-row apply for symmetric blocks too (A/B of k_pc_apply_sym)
static bool pc_rowwarp() {
    static const bool v = getenv("VC_PC_ROWWARP") && atoi(getenv("VC_PC_ROWWARP"));
    return v;
}

vc_status precond_apply_multi_dev(vc_ctx* c, int nc, const double* const* d_r, double* const* d_z) {
    Precond* pc = c->pc;
    if (!pc) return set_err(c, VC_ERR_STATE, "no preconditioner");
    static const bool grouped = getenv("VC_PC_GROUPED") != nullptr;
    if (nc != 2 || pc->kind < 3 || grouped || pc->nbtile == 0) {
        for (int q = 0; q < nc; ++q) {
            vc_status s = precond_apply_dev(c, d_r[q], d_z[q]);
            if (s) return s;
        }
        return VC_OK;
    }
    cudaStream_t st = c->stream;
    const int64_t N = c->NL;
    PcCols cols{};
    for (int q = 0; q < 2; ++q) {
        k_pc_diag<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((N + 255) / 256, 148 * 8)), 256, 0, st>>>(N, d_r[q], pc->diag_inv.p, d_z[q]);
        cols.r[q] = d_r[q];
        cols.z[q] = d_z[q];
    }
    if (pc->kind == 3 && pc->nstile > 0 && !pc_rowwarp())
        k_pc_apply_sym<2><<<pc->nstile, kPsRows, 2 * sizeof(double) * (size_t)pc->max_n, st>>>(
            pc->stile_b.p, pc->stile_r0.p, pc->box_start.p, pc->box_n.p, pc->box_uid.p,
            pc->uniq_off.p, pc->panel_ids.p, pc->blocks.p, cols);
    else
        k_pc_apply_box<2><<<pc->nbtile, 256, 2 * sizeof(double) * (size_t)pc->max_n, st>>>(
            pc->btile_b.p, pc->btile_r0.p, pc->box_start.p, pc->box_n.p, pc->box_uid.p,
            pc->uniq_off.p, pc->panel_ids.p, pc->blocks.p, cols);
    count_launch(c, 3);
    VC_CUDA(c, cudaGetLastError());
    return VC_OK;
}

vc_status precond_apply_dev(vc_ctx* c, const double* d_r, double* d_z) {
    Precond* pc = c->pc;
    if (!pc) return set_err(c, VC_ERR_STATE, "no preconditioner");
    cudaStream_t st = c->stream;
    const int64_t N = c->NL;
    k_pc_diag<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((N + 255) / 256, 148 * 8)), 256, 0, st>>>(N, d_r, pc->diag_inv.p, d_z);
    count_launch(c);
    static const bool grouped = getenv("VC_PC_GROUPED") != nullptr;
    if (pc->kind >= 3 && !grouped && pc->nbtile > 0) {
        PcCols cols{};
        cols.r[0] = d_r;
        cols.z[0] = d_z;
        if (pc->kind == 3 && pc->nstile > 0 && !pc_rowwarp())
            k_pc_apply_sym<1><<<pc->nstile, kPsRows, sizeof(double) * (size_t)pc->max_n, st>>>(
                pc->stile_b.p, pc->stile_r0.p, pc->box_start.p, pc->box_n.p, pc->box_uid.p,
                pc->uniq_off.p, pc->panel_ids.p, pc->blocks.p, cols);
        else
            k_pc_apply_box<1><<<pc->nbtile, 256, sizeof(double) * (size_t)pc->max_n, st>>>(
                pc->btile_b.p, pc->btile_r0.p, pc->box_start.p, pc->box_n.p, pc->box_uid.p,
                pc->uniq_off.p, pc->panel_ids.p, pc->blocks.p, cols);
        count_launch(c);
    } else if (pc->kind >= 3 && pc->ntile > 0) {
        const size_t sh = sizeof(double) * (size_t)(kPcRows + 1) * pc->max_n;
        if (sh > 48 * 1024)
            VC_CUDA(c, grant_max_dyn_smem(k_pc_apply_grouped, max_dyn_smem()));
        k_pc_apply_grouped<<<pc->ntile, 256, sh, st>>>(
            pc->tile_u.p, pc->tile_r0.p, pc->tile_q0.p, pc->uniq_n.p, pc->uniq_off.p, pc->ubox_start.p,
            pc->ubox_list.p, pc->box_start.p, pc->panel_ids.p, pc->blocks.p, d_r, d_z);
        count_launch(c);
    }
    VC_CUDA(c, cudaGetLastError());
    return VC_OK;
}

}  // namespace vc

namespace vc {
PcPlan* pc_plan_new() { return new PcPlan(); }
void pc_plan_free(PcPlan* p) { delete p; }
}  // namespace vc
