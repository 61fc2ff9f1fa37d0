// fft.cuh -- batched in-shared-memory fp64 FFT building blocks (sm_100a).
//
// A length-L (power of two, 8..4096) transform is done as NS = ceil(log2 L / 4) in-place
// decimation-in-frequency radix-R stages (R = 2^bits, bits <= 4, spread evenly), each stage a
// register-resident R-point DFT followed by the inter-stage twiddle.  T independent pencils are
// transformed together; the caller supplies load/store functors, so the first stage can read
// straight from global memory (zero-padded input, strided pencils) and the last stage can write
// straight to global memory at the digit-reversed position -> frequency map, with shared memory
// only between stages (layout [element][pencil], pencil fastest, so lanes of a warp hit
// consecutive 16-byte words).
#pragma once
#include "common.cuh"

namespace vc {

constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n / 2); }

// MB: largest radix exponent per stage (4: radix <= 16, the default; 3: radix <= 8, more stages
// but fewer registers per thread)
template <int L, int MB = 4>
struct Plan {
    static_assert(L >= 2 && (L & (L - 1)) == 0 && L <= kMaxL, "L must be a power of two");
    static constexpr int B = ilog2c(L);
    static constexpr int NS = (B + MB - 1) / MB;
    __host__ __device__ static constexpr int bits(int s) { return B / NS + (s < B % NS ? 1 : 0); }
    __host__ __device__ static constexpr int radix(int s) { return 1 << bits(s); }
    __host__ __device__ static constexpr int lc(int s) {
        int r = L;
        for (int i = 0; i < s; ++i) r >>= bits(i);
        return r;
    }
    // storage position p (after all DIF stages) -> frequency k
    __host__ __device__ static constexpr int freq(int p) {
        int k = 0, mul = 1;
        for (int s = 0; s < NS; ++s) {
            int S = lc(s) / radix(s);
            int m = (p / S) % radix(s);
            k += m * mul;
            mul *= radix(s);
        }
        return k;
    }
    // frequency k -> storage position p
    __host__ __device__ static constexpr int pos(int k) {
        int p = 0;
        for (int s = 0; s < NS; ++s) {
            int R = radix(s);
            p += (k % R) * (lc(s) / R);
            k /= R;
        }
        return p;
    }
};

__host__ __device__ constexpr int hipow2(int m) {
    int h = 1;
    while (h * 2 <= m) h *= 2;
    return h;
}

template <int R>
__device__ __forceinline__ constexpr int bitrev(int i) {
    int r = 0;
    for (int b = 1; b < R; b <<= 1) {
        r = (r << 1) | (i & 1);
        i >>= 1;
    }
    return r;
}

// Multiply by w_16^k16 (forward: exp(-2 pi i k16/16)), k16 a compile-time constant after
// unrolling; trivial angles become adds / swaps.
template <bool INV>
__device__ __forceinline__ double2 rot16(double2 v, int k16) {
    constexpr double C1 = 0.92387953251128675613;  // cos(pi/8)
    constexpr double S1 = 0.38268343236508977173;  // sin(pi/8)
    constexpr double H = 0.70710678118654752440;   // sqrt(1/2)
    double c, s;  // w = c - i s (forward)
    switch (k16 & 15) {
        case 0: return v;
        case 4: return INV ? make_double2(-v.y, v.x) : make_double2(v.y, -v.x);
        case 8: return make_double2(-v.x, -v.y);
        case 12: return INV ? make_double2(v.y, -v.x) : make_double2(-v.y, v.x);
        case 1: c = C1; s = S1; break;
        case 2: c = H; s = H; break;
        case 3: c = S1; s = C1; break;
        case 5: c = -S1; s = C1; break;
        case 6: c = -H; s = H; break;
        case 7: c = -C1; s = S1; break;
        case 9: c = -C1; s = -S1; break;
        case 10: c = -H; s = -H; break;
        case 11: c = -S1; s = -C1; break;
        case 13: c = S1; s = -C1; break;
        case 14: c = H; s = -H; break;
        default: c = C1; s = -S1; break;  // 15
    }
    if (INV) s = -s;
    // (vx + i vy)(c - i s)
    return make_double2(fma(v.x, c, v.y * s), fma(v.y, c, -v.x * s));
}

// In-register R-point DFT (DIF radix-2 butterflies); on return register i holds frequency
// bitrev_R(i).
template <int R, bool INV>
__device__ __forceinline__ void reg_dft(double2 (&v)[R]) {
#pragma unroll
    for (int half = R / 2; half >= 1; half /= 2) {
#pragma unroll
        for (int g = 0; g < R; g += 2 * half) {
#pragma unroll
            for (int j = 0; j < half; ++j) {
                double2 a = v[g + j], b = v[g + j + half];
                v[g + j] = cadd(a, b);
                v[g + j + half] = rot16<INV>(csub(a, b), j * (16 / (2 * half)));
            }
        }
    }
}

// Shared-memory index of (pencil t, position p): PF -> [pos][pencil], else [pencil][pos].
// The low 3 bits of the index (8 complex = one 128-byte bank row) are XOR-swizzled with bits
// 3-5, 6-8 and 9-11, so that the access patterns of a quarter-warp -- 8 consecutive aligned
// elements (stages with S >= 8), and the strided patterns of the last radix-8 stage (S = 1) and
// of digit-reversed frequency reads -- hit 8 distinct bank groups (unswizzled, these were 2- to
// 8-way conflicts: 27M extra wavefronts in k_p1<1024> on C4).  PF = false always swizzles; PF
// layouts swizzle only with SWZ (P3's buffers are filled by bulk copies in the plain layout).
__host__ __device__ constexpr int swz8(int i) { return i ^ (((i >> 3) ^ (i >> 6) ^ (i >> 9)) & 7); }
template <int L, int T, bool PF, bool SWZ = false>
__device__ __forceinline__ int smi(int t, int p) {
    if constexpr (PF) return SWZ ? swz8(p * T + t) : p * T + t;
    else return t * L + swz8(p);
}

// Shared-memory accessor in the smi layout.  fft_stage recognises it and addresses the R legs of
// a butterfly as smi(t, base) ^ c_j with c_j a compile-time constant: the leg offsets j*S occupy
// bits disjoint from base (base = g*Lc + b, b < S, j*S < Lc) and from t, and both the layout and
// swz8 are XOR-linear over disjoint bit fields, so one XOR per element replaces the full index
// and swizzle arithmetic.
template <int L, int T, bool PF, bool SWZ>
struct SmAcc {
    double2* sm;
    __device__ __forceinline__ static int idx(int t, int p) { return smi<L, T, PF, SWZ>(t, p); }
    __device__ __forceinline__ double2 operator()(int t, int p) const { return sm[smi<L, T, PF, SWZ>(t, p)]; }
    __device__ __forceinline__ void operator()(int t, int p, double2 v) const { sm[smi<L, T, PF, SWZ>(t, p)] = v; }
    // index offset of a position displacement d with disjoint bits (see above)
    __host__ __device__ static constexpr int off(int d) {
        return PF ? (SWZ ? swz8(d * T) : d * T) : swz8(d);
    }
    // index of (t, p + d) from idx(t, p): XOR for the swizzled layouts (T a power of two there),
    // plain addition for the unswizzled [pos][pencil] layout (T may be any width, e.g. P3's)
    __device__ __forceinline__ static int at(int i0, int d) {
        static_assert(!(PF && SWZ) || (T & (T - 1)) == 0, "swizzled layouts need a power-of-two width");
        if constexpr (PF && !SWZ) return i0 + d * T;
        else return i0 ^ off(d);
    }
};
template <class X> struct IsSmAcc { static constexpr bool value = false; };
template <int L, int T, bool PF, bool SWZ> struct IsSmAcc<SmAcc<L, T, PF, SWZ>> {
    static constexpr bool value = true;
};
template <class X> struct Bare { using type = X; };
template <class X> struct Bare<X&> { using type = X; };
template <class X> struct Bare<const X&> { using type = X; };
template <class X> struct Bare<const X> { using type = X; };

// One DIF stage s of the length-L transform over T pencils with NT threads.
//   ld(t, p) -> double2 : element at storage position p of pencil t (stage input)
//   st(t, p, v)         : write element at position p of pencil t (stage output)
//   PF = true : consecutive lanes take consecutive pencils (strided-axis passes)
//   PF = false: consecutive lanes take consecutive butterflies of one pencil (contiguous lines)
//   Tn (<= T): pencils actually transformed (the shared-memory layout keeps stride T)
//   TB > 0 (PF only): Tn is a multiple of the compile-time pencil block TB; lanes take
//       consecutive pencils within a block, so no division by the run-time Tn is needed
template <int L, int T, int NT, bool INV, bool PF, int s, int TB = 0, int MB = 4, class LD, class ST>
__device__ __forceinline__ void fft_stage(LD&& ld, ST&& st, const double2* __restrict__ tw,
                                          const int Tn = T) {
    constexpr int R = Plan<L, MB>::radix(s);
    constexpr int Lc = Plan<L, MB>::lc(s);
    constexpr int S = Lc / R;
    constexpr int TW = kTabN / Lc;
    const int NB = Tn * (L / R);
#pragma unroll 1
    for (int u = threadIdx.x; u < NB; u += NT) {
        int t, rest;
        if constexpr (PF && TB > 0) {
            const int v = u / TB;
            rest = v % (L / R);
            t = (v / (L / R)) * TB + u % TB;
        } else {
            t = PF ? u % Tn : u / (L / R);
            rest = PF ? u / Tn : u % (L / R);
        }
        const int b = rest % S;
        const int g = rest / S;
        const int base = g * Lc + b;
        using LDT = typename Bare<LD>::type;
        using STT = typename Bare<ST>::type;
        double2 v[R];
        if constexpr (IsSmAcc<LDT>::value) {
            const int i0 = LDT::idx(t, base);
#pragma unroll
            for (int j = 0; j < R; ++j) v[j] = ld.sm[LDT::at(i0, j * S)];
        } else {
#pragma unroll
            for (int j = 0; j < R; ++j) v[j] = ld(t, base + j * S);
        }
        reg_dft<R, INV>(v);
        if (S > 1) {
            // inter-stage twiddles w_Lc^{b m}: one table load, powers by squaring/products
            // (measured: R-1 table loads instead made the HBM-bound passes 15-20% slower)
            double2 wp[R];
            wp[0] = make_double2(1.0, 0.0);
            wp[1] = twiddle<INV>(tw, b * TW);
#pragma unroll
            for (int m = 2; m < R; ++m) {
                const int hb = hipow2(m);  // highest power of two <= m
                wp[m] = (m == hb) ? cmul(wp[m / 2], wp[m / 2]) : cmul(wp[hb], wp[m - hb]);
            }
            if constexpr (IsSmAcc<STT>::value) {
                const int i0 = STT::idx(t, base);
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    const int m = bitrev<R>(i);
                    st.sm[STT::at(i0, m * S)] = m == 0 ? v[i] : cmul(v[i], wp[m]);
                }
            } else {
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    const int m = bitrev<R>(i);
                    st(t, base + m * S, m == 0 ? v[i] : cmul(v[i], wp[m]));
                }
            }
        } else if constexpr (IsSmAcc<STT>::value) {
            const int i0 = STT::idx(t, base);
#pragma unroll
            for (int i = 0; i < R; ++i) st.sm[STT::at(i0, bitrev<R>(i) * S)] = v[i];
        } else {
#pragma unroll
            for (int i = 0; i < R; ++i) st(t, base + bitrev<R>(i) * S, v[i]);
        }
    }
}

// Stage 0 of a PF = false transform whose input sits in (and may alias) the shared buffer:
// every point of the thread's butterfly is read through ld(t, p) into registers, then a CTA
// barrier (the caller's input region may overlap the FFT layout), then the DFT, inter-stage
// twiddles and stores of fft_stage into the smi layout.  One butterfly per thread.
template <int L, int T, int NT, bool INV, bool PF = false, bool SWZ = false, class LD>
__device__ __forceinline__ void fft_stage0_aliased(double2* sm, LD&& ld, const double2* __restrict__ tw) {
    constexpr int R = Plan<L>::radix(0);
    constexpr int S = L / R;
    constexpr int TW = kTabN / L;
    static_assert(T * (L / R) == NT, "one stage-0 butterfly per thread");
    // (as fft_stage: PF -> consecutive lanes on consecutive pencils)
    const int t = PF ? threadIdx.x % T : threadIdx.x / S, b = PF ? threadIdx.x / T : threadIdx.x % S;
    double2 v[R];
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = ld(t, b + j * S);
    __syncthreads();
    reg_dft<R, INV>(v);
    using A = SmAcc<L, T, PF, SWZ>;
    const int i0 = A::idx(t, b);
    if constexpr (S > 1) {
        double2 wp[R];
        wp[0] = make_double2(1.0, 0.0);
        wp[1] = twiddle<INV>(tw, b * TW);
#pragma unroll
        for (int m = 2; m < R; ++m) {
            const int hb = hipow2(m);
            wp[m] = (m == hb) ? cmul(wp[m / 2], wp[m / 2]) : cmul(wp[hb], wp[m - hb]);
        }
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int m = bitrev<R>(i);
            sm[A::at(i0, m * S)] = m == 0 ? v[i] : cmul(v[i], wp[m]);
        }
    } else {
#pragma unroll
        for (int i = 0; i < R; ++i) sm[A::at(i0, bitrev<R>(i) * S)] = v[i];
    }
}

// Stages 1 .. NS-1 of a PF = false transform (after fft_stage0_aliased; leading barrier
// included), the last writing through stN.
template <int L, int T, int NT, bool INV, bool PF = false, bool SWZ = false, class ST>
__device__ __forceinline__ void fft_run_from1(double2* sm, ST&& stN, const double2* __restrict__ tw) {
    constexpr int NS = Plan<L>::NS;
    const SmAcc<L, T, PF, SWZ> lds{sm}, sts{sm};
    __syncthreads();
    if constexpr (NS == 2) {
        fft_stage<L, T, NT, INV, PF, 1>(lds, stN, tw);
    } else if constexpr (NS == 3) {
        fft_stage<L, T, NT, INV, PF, 1>(lds, sts, tw);
        __syncthreads();
        fft_stage<L, T, NT, INV, PF, 2>(lds, stN, tw);
    } else {
        static_assert(NS == 4, "2 <= NS <= 4");
        fft_stage<L, T, NT, INV, PF, 1>(lds, sts, tw);
        __syncthreads();
        fft_stage<L, T, NT, INV, PF, 2>(lds, sts, tw);
        __syncthreads();
        fft_stage<L, T, NT, INV, PF, 3>(lds, stN, tw);
    }
}

// Full transform: stage 0 reads through `ld0`, the last stage writes through `stN`, and the
// intermediate stages use shared memory `sm` (layout smi<L,T,PF>).  If NS == 1 the single
// stage goes ld0 -> stN.  No trailing __syncthreads().
template <int L, int T, int NT, bool INV, bool PF, int TB = 0, bool SWZ = false, int MB = 4,
          class LD, class ST>
__device__ __forceinline__ void fft_run(double2* sm, LD&& ld0, ST&& stN,
                                        const double2* __restrict__ tw, const int Tn = T) {
    constexpr int NS = Plan<L, MB>::NS;
    const SmAcc<L, T, PF, SWZ> lds{sm}, sts{sm};
    if constexpr (NS == 1) {
        fft_stage<L, T, NT, INV, PF, 0, TB, MB>(ld0, stN, tw, Tn);
    } else if constexpr (NS == 2) {
        fft_stage<L, T, NT, INV, PF, 0, TB, MB>(ld0, sts, tw, Tn);
        __syncthreads();
        fft_stage<L, T, NT, INV, PF, 1, TB, MB>(lds, stN, tw, Tn);
    } else if constexpr (NS == 3) {
        fft_stage<L, T, NT, INV, PF, 0, TB, MB>(ld0, sts, tw, Tn);
        __syncthreads();
        fft_stage<L, T, NT, INV, PF, 1, TB, MB>(lds, sts, tw, Tn);
        __syncthreads();
        fft_stage<L, T, NT, INV, PF, 2, TB, MB>(lds, stN, tw, Tn);
    } else {
        static_assert(NS == 4, "L <= 4096 with radix >= 8");
        fft_stage<L, T, NT, INV, PF, 0, TB, MB>(ld0, sts, tw, Tn);
        __syncthreads();
        fft_stage<L, T, NT, INV, PF, 1, TB, MB>(lds, sts, tw, Tn);
        __syncthreads();
        fft_stage<L, T, NT, INV, PF, 2, TB, MB>(lds, sts, tw, Tn);
        __syncthreads();
        fft_stage<L, T, NT, INV, PF, 3, TB, MB>(lds, stN, tw, Tn);
    }
}

}  // namespace vc
