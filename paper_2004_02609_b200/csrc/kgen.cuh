// kgen.cuh -- device evaluation of the VoxCap panel-pair integrals (DESIGN.md a2).
//
// kappa(kind, alpha, beta, D) in unit-voxel units (dv = 1, 4 pi eps0 = 1) for an observer
// (testing) alpha-normal panel at slot D and a beta-normal source panel at slot 0 (P:97 grids):
//   kind 0: P = \int\int 1/|r - r'|                                    (Eq. 5)
//   kind 1: E+ = d/d(observer alpha coordinate) of the same integral   (Eq. 6)
// Near pairs (centre distance < 4 voxels): fp64 closed forms with cancellation-safe x + r,
//   parallel P : second-difference corner sum of F (antiderivative of [29]; reading O1)
//   parallel E : the same corner sum of -dF/dz reduced to a z ln(a+r) + b z ln(b+r)
//                + a b atan(ab/(z r)) - z r (terms that cancel in the corner sum dropped);
//                E(coplanar) = 0 (reading O4)
//   orthogonal P: corner sum of H (reading O1);  orthogonal E: corner sum of dH/dc reduced to
//                a b ln(a+r) + (a^2-c^2)/2 ln(b+r) - a c atan(ab/(c r)) - b r/2
//   exact zeros on touching orthogonal pairs take the one-sided limit (reading O5): a -> +eta,
//   b -> sign(sibling b) eta, c -> sign(sibling c) eta.
// Far pairs: Gauss-Legendre (triangle rule on shared axes), q per axis from the distance band
//   (reading O6): P q = 6 (d < 5), 5 (< 15), 4 (< 50), 3; E q = 7 (< 5), 6 (< 10),
//   5 (< 20), 4 (< 50), 3 (measured triangle-rule error at q = 3, d = 50: 5e-13 of 1/d^2).
// These formulas are written independently of the CPU oracle (which follows Eqs. 15/16
// verbatim in binary128); the parity tests compare the two.
#pragma once
#include "common.cuh"

namespace vc {

static __constant__ double kGLx[7][8] = {
    {-0.28867513459481287, 0.28867513459481287, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {-0.3872983346207417, 0.0, 0.3872983346207417, 0.0, 0.0, 0.0, 0.0, 0.0},
    {-0.4305681557970263, -0.16999052179242813, 0.16999052179242813, 0.4305681557970263, 0.0, 0.0, 0.0, 0.0},
    {-0.453089922969332, -0.26923465505284155, 0.0, 0.26923465505284155, 0.453089922969332, 0.0, 0.0, 0.0},
    {-0.46623475710157597, -0.33060469323313224, -0.11930959304159845, 0.11930959304159845, 0.33060469323313224, 0.46623475710157597, 0.0, 0.0},
    {-0.4745539561713793, -0.37076559279969723, -0.2029225756886986, 0.0, 0.2029225756886986, 0.37076559279969723, 0.4745539561713793, 0.0},
    {-0.4801449282487681, -0.39833323870681336, -0.2627662049581645, -0.09171732124782489, 0.09171732124782489, 0.2627662049581645, 0.39833323870681336, 0.4801449282487681},
};
static __constant__ double kGLw[7][8] = {
    {0.5, 0.5, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {0.27777777777777785, 0.4444444444444444, 0.27777777777777785, 0.0, 0.0, 0.0, 0.0, 0.0},
    {0.17392742256872679, 0.3260725774312732, 0.3260725774312732, 0.17392742256872679, 0.0, 0.0, 0.0, 0.0},
    {0.11846344252809464, 0.23931433524968315, 0.28444444444444433, 0.23931433524968315, 0.11846344252809464, 0.0, 0.0, 0.0},
    {0.08566224618958514, 0.18038078652406936, 0.23395696728634552, 0.23395696728634552, 0.18038078652406936, 0.08566224618958514, 0.0, 0.0},
    {0.06474248308443487, 0.13985269574463843, 0.19091502525255935, 0.20897959183673465, 0.19091502525255935, 0.13985269574463843, 0.06474248308443487, 0.0},
    {0.05061426814518853, 0.11119051722668721, 0.15685332293894344, 0.18134189168918083, 0.18134189168918083, 0.15685332293894344, 0.11119051722668721, 0.05061426814518853},
};

constexpr double kEta = 1e-30;  // one-sided-limit nudge (reading O5)

// x + r with r = sqrt(x^2 + rest2), cancellation-free for x < 0.
__device__ __forceinline__ double xpr(double x, double r, double rest2) {
    return x >= 0.0 ? x + r : rest2 / (r - x);
}

// ---- parallel -------------------------------------------------------------------------
__device__ __forceinline__ double F_par(double a, double b, double z) {
    const double a2 = a * a, b2 = b * b, z2 = z * z;
    const double r = sqrt(a2 + b2 + z2);
    if (r == 0.0) return 0.0;
    double s = -(a2 + b2 - 2.0 * z2) * r * (1.0 / 6.0);
    const double ca = 0.5 * (b2 - z2) * a;
    if (ca != 0.0) s += ca * log(xpr(a, r, b2 + z2));
    const double cb = 0.5 * (a2 - z2) * b;
    if (cb != 0.0) s += cb * log(xpr(b, r, a2 + z2));
    const double abz = a * b * z;
    if (abz != 0.0) s -= abz * atan(a * b / (z * r));
    return s;
}

// -dF/dz up to terms that cancel in the corner sum (z != 0)
__device__ __forceinline__ double G_par(double a, double b, double z) {
    const double a2 = a * a, b2 = b * b, z2 = z * z;
    const double r = sqrt(a2 + b2 + z2);
    double s = -z * r;
    if (a != 0.0) s += a * z * log(xpr(a, r, b2 + z2));
    if (b != 0.0) s += b * z * log(xpr(b, r, a2 + z2));
    if (a != 0.0 && b != 0.0) s += a * b * atan(a * b / (z * r));
    return s;
}

// observer in-plane offsets (Du, Dv), normal offset Dn (observer minus source)
static __device__ double kappa_par_cf(int kind, int Du, int Dv, int Dn) {
    if (kind == 1 && Dn == 0) return 0.0;  // coplanar: field normal to the plane vanishes (O4)
    const double a[3] = {-(double)Du - 1.0, -(double)Du, 1.0 - (double)Du};
    const double b[3] = {-(double)Dv - 1.0, -(double)Dv, 1.0 - (double)Dv};
    const double w[3] = {-1.0, 2.0, -1.0};
    const double z = -(double)Dn;
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        double si = 0.0;
#pragma unroll
        for (int j = 0; j < 3; ++j)
            si += w[j] * (kind == 0 ? F_par(a[i], b[j], z) : G_par(a[i], b[j], z));
        s += w[i] * si;
    }
    return s;
}

// ---- orthogonal (observer normal -> z, source normal -> y, other axis -> x) ---------------
__device__ __forceinline__ double H_orth(double a, double b, double c) {
    const double a2 = a * a, b2 = b * b, c2 = c * c;
    const double r = sqrt(a2 + b2 + c2);
    double s = a * b * c * log(xpr(a, r, b2 + c2));
    s += (0.5 * a2 * b - b2 * b * (1.0 / 6.0)) * log(xpr(c, r, a2 + b2));
    s += (0.5 * a2 * c - c2 * c * (1.0 / 6.0)) * log(xpr(b, r, a2 + c2));
    s -= b * c * r * (1.0 / 3.0);
    s += a * (-a2 * (1.0 / 9.0) + (b2 + c2) * (1.0 / 6.0)) * atan(b * c / (a * r));
    s += a * (a2 * (1.0 / 18.0) - b2 * (1.0 / 3.0) + c2 * (1.0 / 6.0)) * atan(a * c / (b * r));
    s += a * (a2 * (1.0 / 18.0) + b2 * (1.0 / 6.0) - c2 * (1.0 / 3.0)) * atan(a * b / (c * r));
    return s;
}

__device__ __forceinline__ double G_orth(double a, double b, double c) {
    const double a2 = a * a, b2 = b * b, c2 = c * c;
    const double r = sqrt(a2 + b2 + c2);
    double s = a * b * log(xpr(a, r, b2 + c2));
    s += 0.5 * (a2 - c2) * log(xpr(b, r, a2 + c2));
    s -= a * c * atan(a * b / (c * r));
    s -= 0.5 * b * r;
    return s;
}

__device__ __forceinline__ double sgn_nz(double v) { return v > 0.0 ? 1.0 : -1.0; }

static __device__ double kappa_orth_cf(int kind, int Dg, int Db, int Da) {
    double a[3] = {-(double)Dg - 1.0, -(double)Dg, 1.0 - (double)Dg};
    const double w[3] = {-1.0, 2.0, -1.0};
    double b[2] = {-(double)Db, -(double)Db - 1.0};
    double c[2] = {1.0 - (double)Da, -(double)Da};
#pragma unroll
    for (int i = 0; i < 3; ++i)
        if (a[i] == 0.0) a[i] = kEta;
    if (b[0] == 0.0) b[0] = sgn_nz(b[1]) * kEta;
    if (b[1] == 0.0) b[1] = sgn_nz(b[0]) * kEta;
    if (c[0] == 0.0) c[0] = sgn_nz(c[1]) * kEta;
    if (c[1] == 0.0) c[1] = sgn_nz(c[0]) * kEta;
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        double si = 0.0;
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int l = 0; l < 2; ++l) {
                // P: (-1)^{m+l+1} (1-based) ; E: (-1)^{m+l}
                const double sg = ((m + l) & 1) ? 1.0 : -1.0;
                si += kind == 0 ? sg * H_orth(a[i], b[m], c[l]) : -sg * G_orth(a[i], b[m], c[l]);
            }
        s += w[i] * si;
    }
    return s;
}

// ---- far field: Gauss-Legendre with the triangle rule on shared axes --------------------
// Along an axis both unit panels span, the double integral over [x0,x0+1] x [0,1] of g(x - x')
// equals \int_{-1}^{1} (1 - |s|) g(D + s) ds; split at the kink, each half gets q GL points with
// weights w (1 - x).  Parallel pairs share both in-plane axes ((2q)^2 points instead of q^4);
// orthogonal pairs share the third axis and keep one GL axis on each panel (2q^3 points).
template <int A, int B, int Q, int KIND>
__device__ double kappa_gl(double d0x, double d0y, double d0z) {
    const double* X = kGLx[Q - 2];  // offsets from 1/2 of the [0,1] nodes
    const double* W = kGLw[Q - 2];
    double acc = 0.0;
    if constexpr (A == B) {
        constexpr int U = A == 0 ? 1 : 0, V = A == 2 ? 1 : 2;
#pragma unroll 1
        for (int i = 0; i < 2 * Q; ++i) {
            const int ki = i % Q;
            const double xi = (i < Q ? 1.0 : -1.0) * (0.5 + X[ki]);
            const double wi = W[ki] * (0.5 - X[ki]);
            double e[3] = {d0x, d0y, d0z};
            e[U] += xi;
            double accj = 0.0;
#pragma unroll
            for (int j = 0; j < 2 * Q; ++j) {
                const int kj = j % Q;
                double f[3] = {e[0], e[1], e[2]};
                f[V] += (j < Q ? 1.0 : -1.0) * (0.5 + X[kj]);
                const double r2 = f[0] * f[0] + f[1] * f[1] + f[2] * f[2];
                const double ri = rsqrt(r2);
                const double v = KIND == 0 ? ri : -f[A] * ri * ri * ri;
                accj = fma(W[kj] * (0.5 - X[kj]), v, accj);
            }
            acc = fma(wi, accj, acc);
        }
    } else {
        constexpr int G = 3 - A - B;
#pragma unroll 1
        for (int i = 0; i < 2 * Q; ++i) {
            const int ki = i % Q;
            const double wi = W[ki] * (0.5 - X[ki]);
            double e[3] = {d0x, d0y, d0z};
            e[G] += (i < Q ? 1.0 : -1.0) * (0.5 + X[ki]);
#pragma unroll 1
            for (int j = 0; j < Q; ++j) {
                double f0[3] = {e[0], e[1], e[2]};
                f0[B] += X[j];  // observer extent along beta
                double acck = 0.0;
#pragma unroll
                for (int k = 0; k < Q; ++k) {
                    double f[3] = {f0[0], f0[1], f0[2]};
                    f[A] -= X[k];  // source extent along alpha
                    const double r2 = f[0] * f[0] + f[1] * f[1] + f[2] * f[2];
                    const double ri = rsqrt(r2);
                    const double v = KIND == 0 ? ri : -f[A] * ri * ri * ri;
                    acck = fma(W[k], v, acck);
                }
                acc = fma(wi * W[j], acck, acc);
            }
        }
    }
    return acc;
}

template <int A, int B, int KIND>
__device__ double kappa_gl_q(int q, double dx, double dy, double dz) {
    switch (q) {
        case 2: return kappa_gl<A, B, 2, KIND>(dx, dy, dz);
        case 3: return kappa_gl<A, B, 3, KIND>(dx, dy, dz);
        case 4: return kappa_gl<A, B, 4, KIND>(dx, dy, dz);
        case 5: return kappa_gl<A, B, 5, KIND>(dx, dy, dz);
        case 6: return kappa_gl<A, B, 6, KIND>(dx, dy, dz);
        default: return kappa_gl<A, B, 7, KIND>(dx, dy, dz);
    }
}

template <int KIND>
__device__ double kappa_gl_dispatch(int alpha, int beta, int q, double dx, double dy, double dz) {
    switch (alpha * 3 + beta) {
        case 0: return kappa_gl_q<0, 0, KIND>(q, dx, dy, dz);
        case 1: return kappa_gl_q<0, 1, KIND>(q, dx, dy, dz);
        case 2: return kappa_gl_q<0, 2, KIND>(q, dx, dy, dz);
        case 3: return kappa_gl_q<1, 0, KIND>(q, dx, dy, dz);
        case 4: return kappa_gl_q<1, 1, KIND>(q, dx, dy, dz);
        case 5: return kappa_gl_q<1, 2, KIND>(q, dx, dy, dz);
        case 6: return kappa_gl_q<2, 0, KIND>(q, dx, dy, dz);
        case 7: return kappa_gl_q<2, 1, KIND>(q, dx, dy, dz);
        default: return kappa_gl_q<2, 2, KIND>(q, dx, dy, dz);
    }
}

// orders per distance band (reading O6); q = 2 far out (round 2): worst error against the
// binary128 oracle over 150 random directions per band (relative to 1/d resp. 1/d^2): P 2.4e-12
// at d in [300, 350), 8.3e-13 in [400, 450); E 1.4e-12 in [450, 500), 9.3e-13 in [500, 600) --
// so q = 2 from d = 400 (P) and 500 (E), >= 2x inside the 2e-12 entry bar, for 56-70% fewer 1/r
// evaluations on those entries
__device__ __forceinline__ int gl_order(int kind, double dist) {
    if (kind == 0) return dist < 5.0 ? 6 : dist < 15.0 ? 5 : dist < 50.0 ? 4 : dist < 400.0 ? 3 : 2;
    return dist < 5.0 ? 7 : dist < 10.0 ? 6 : dist < 20.0 ? 5 : dist < 50.0 ? 4 : dist < 500.0 ? 3 : 2;
}

constexpr double kNearFar = 4.0;

// The entry generator: unit-voxel kappa for slot offset D = (observer slot - source slot).
static __device__ double kappa(int kind, int alpha, int beta, int Dx, int Dy, int Dz) {
    const int D[3] = {Dx, Dy, Dz};
    const double dx = Dx + 0.5 * (c2(alpha, 0) - c2(beta, 0));
    const double dy = Dy + 0.5 * (c2(alpha, 1) - c2(beta, 1));
    const double dz = Dz + 0.5 * (c2(alpha, 2) - c2(beta, 2));
    const double dist = sqrt(dx * dx + dy * dy + dz * dz);
    if (dist < kNearFar) {
        if (alpha == beta) {
            const int n = alpha, u = (n + 1) % 3, v = (n + 2) % 3;
            return kappa_par_cf(kind, D[u], D[v], D[n]);
        }
        const int g = 3 - alpha - beta;
        return kappa_orth_cf(kind, D[g], D[beta], D[alpha]);
    }
    const int q = gl_order(kind, dist);
    return kind == 0 ? kappa_gl_dispatch<0>(alpha, beta, q, dx, dy, dz)
                     : kappa_gl_dispatch<1>(alpha, beta, q, dx, dy, dz);
}

}  // namespace vc
