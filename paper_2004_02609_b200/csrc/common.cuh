// common.cuh -- shared device/host helpers of libvoxcap (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace vc {

constexpr double kPi = 3.14159265358979323846264338327950288;
constexpr double kEps0 = 8.8541878128e-12;  // F/m (reading O15)
constexpr int kMaxL = 4096;                 // largest FFT length per axis
constexpr int kTabN = 2 * kMaxL;            // twiddle table: exp(-2 pi i n / kTabN)
// slot-map entries (slot -> panel): -1 = no panel, else the panel index in bits 0-28 with the
// row kind folded in, so the gather of P5 needs no per-panel info load: bit 30 = dielectric
// panel, bit 29 = its normal points along -axis (reading O7)
constexpr int32_t kSlotDiel = 1 << 30, kSlotNeg = 1 << 29, kSlotIdx = (1 << 29) - 1;
// Grant kernel `k` the largest dynamic shared memory the device allows next to its static
// shared memory.  The limit is a process-wide function attribute: contexts of one process
// (ranks of a thread group) launch with different sizes, so a per-launch value would race.
template <class K>
inline cudaError_t grant_max_dyn_smem(K k, int optin);
// opt-in shared memory per CTA of the current device (queried once per device)
inline int max_dyn_smem() {
    static int v[16] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 16) dev = 0;
    if (!v[dev]) {
        int x = 0;
        cudaDeviceGetAttribute(&x, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        v[dev] = x > 0 ? x : 48 * 1024;
    }
    return v[dev];
}
template <class K>
inline cudaError_t grant_max_dyn_smem(K k, int optin) {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, k);
    if (e) return e;
    return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                optin - (int)fa.sharedSizeBytes);
}

// Half-integer centre offsets of the a-normal panel grids, doubled (c_x = (0,1/2,1/2) ...;
// P:97 grids, Table VII P:331-341 in the S = c_beta - c_alpha form).
__host__ __device__ constexpr int c2(int normal, int axis) { return normal == axis ? 0 : 1; }

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 czero() { return make_double2(0.0, 0.0); }

// exp(-2 pi i n / kTabN) for n in [0, kTabN); inverse direction uses the conjugate.
template <bool INV>
__device__ __forceinline__ double2 twiddle(const double2* __restrict__ tw, int n) {
    double2 w = __ldg(tw + n);
    return INV ? cconj(w) : w;
}

// Half-shift phase exp(sgn * i pi kt / M) for a signed frequency kt in [-M/2, M/2]
// (sgn = -1: phi-bar, sgn = +1: phi; SURVEY App. B / DESIGN.md "spectra").
__device__ __forceinline__ double2 half_phase(const double2* __restrict__ tw, int kt, int M, int sgn) {
    // exp(-2 pi i |kt| / (2M)) = tw[|kt| * kTabN / (2M)]
    int a = kt < 0 ? -kt : kt;
    double2 w = __ldg(tw + a * (kTabN / (2 * M)));  // = exp(-i pi |kt| / M)
    // want exp(sgn * i pi kt / M): if sgn*kt > 0 -> conj(w), else w
    bool pos = (sgn > 0) == (kt > 0);
    return (kt != 0 && pos) ? cconj(w) : w;
}

// 8-byte global -> shared asynchronous copy (LDGSTS) and completion wait
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
// 16-byte global -> shared asynchronous copy, zero-filling when !valid (src-size 0)
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// ---- TMA bulk copies (cp.async.bulk, SASS UBLKCP) completing on a shared-memory mbarrier ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// make the initialised barriers visible to the async (TMA) proxy
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
// order this thread's earlier generic-proxy shared accesses before later async-proxy writes
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
// arrive (count 1) and add `bytes` to the barrier's expected transaction count
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes) : "memory");
}
// global -> shared bulk copy of `bytes` (multiple of 16, both addresses 16-B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// L2 prefetch of `bytes` (multiple of 16) at a 16-B aligned global address
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
// plain arrive (count 1)
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// wait until the barrier phase with parity `par` has completed
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned par) {
    asm volatile(
        "{\n .reg .pred P1;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        " @!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(par)
        : "memory");
}

}  // namespace vc
