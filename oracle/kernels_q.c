/*
 * oracle/kernels_q.c -- TEST INFRASTRUCTURE ONLY (CPU oracle; never on the product path).
 *
 * Panel-pair integrals of the VoxCap Galerkin system, evaluated in IEEE binary128
 * (__float128, libquadmath) so that the oracle's entries are exact to ~1e-25 relative at
 * every distance that occurs on the BASELINE grids.  No switch to quadrature, no tables,
 * no blocking: one closed-form corner sum per entry, as the paper defines it.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load this library.  It shares no code, header or constant with paper_2004_02609_b200/.
 *
 * Units: unit voxel (Δv = 1) and 4πε0 = 1.  The physical entries are
 *     P_kl = Δv^3/(4πε0) * kappa_P,   E_kl = Δv^2/(4πε0) * kappa_E        (App. C)
 *
 * Geometry (§II.B, App. A): an alpha-panel at integer slot t lies in the
 * plane {x_alpha = t_alpha} and spans [t_u, t_u+1] along the two other axes u.  The entry
 * for testing (observer) panel alpha at slot t and source panel beta at slot s depends only
 * on D = t - s; the source is placed at slot 0 and the observer at slot D.
 *
 *  kind 0 (P, Eq. 5):  kappa = \int_{S_t}\int_{S_s} 1/|r - r'| dS' dS
 *     parallel  : sum_{k,m=1..4} (-1)^{k+m} F(a_k, b_m, z)              (closed form of [29],
 *                 the antiderivative with d^4F/da^2 db^2 = 1/r; reading O1 of DESIGN.md)
 *     orthogonal: sum_{k,m,l} (-1)^{k+m+l+1} H(a_k, b_m, c_l)           (d^4H/da^2 db dc = 1/r;
 *                 reading O1; not printed in the paper, which cites [29])
 *  kind 1 (E+, Eq. 6 with the derivative taken along +alpha at the observer):
 *     parallel  : -(Eq. 15)                       (sign reading O2)
 *     orthogonal: +(Eq. 16 with its first bracket term read as b(3a^2-b^2)/(6 r))
 *                                                 (misprint reading O3)
 *     E+(D = 0, alpha = beta) := 0                (principal value; the jump is carried by
 *                                                  Eq. 7's overlap term; reading O4)
 *  Zeros on touching orthogonal pairs: a zero b_m takes the sign of its sibling b, a zero c_l
 *  the sign of its sibling c, a zero a_k is +0 -- realised as a nudge of 1e-30, far below the
 *  binary128 resolution of every term (reading O5: the one-sided limit with the source moved
 *  off the observer's plane and outside its extent).
 */
#include <quadmath.h>
#include <stdint.h>
#include <stdlib.h>

typedef __float128 Q;

static const Q EPS = 1e-37Q; /* the paper's regulariser epsilon */
static const Q ETA = 1e-30Q; /* one-sided-limit nudge for exact zeros (reading O5) */

/* x + r with r = sqrt(x^2 + rest2), without cancellation for x < 0. */
static Q xpr(Q x, Q r, Q rest2) {
    if (x >= 0) return x + r;
    return rest2 / (r - x);
}

/* ---- parallel potential antiderivative F (A.1 reading of [29]) ----------------------- */
static Q F_par(Q a, Q b, Q z) {
    Q a2 = a * a, b2 = b * b, z2 = z * z;
    Q r = sqrtq(a2 + b2 + z2);
    Q s = 0;
    Q ca = (b2 - z2) / 2 * a;          /* (b^2 - z^2)/2 * a * ln(a + r) */
    if (ca != 0) s += ca * logq(xpr(a, r, b2 + z2));
    Q cb = (a2 - z2) / 2 * b;          /* (a^2 - z^2)/2 * b * ln(b + r) */
    if (cb != 0) s += cb * logq(xpr(b, r, a2 + z2));
    s -= (a2 + b2 - 2 * z2) * r / 6;
    if (a != 0 && b != 0 && z != 0)    /* a b z atan(ab/(z r)); 0 when z = 0 */
        s -= a * b * z * atanq(a * b / (z * r));
    return s;
}

/* ---- Eq. (15) bracket, verbatim; z already carries +epsilon ------------- */
static Q eq15(Q a, Q b, Q z) {
    Q a2 = a * a, b2 = b * b, z2 = z * z;
    Q r = sqrtq(a2 + b2 + z2);
    Q apr = xpr(a, r, b2 + z2), bpr = xpr(b, r, a2 + z2);
    Q t = 0;
    t += 0.5Q * a * z * (b2 - z2) / (apr * r + EPS);
    t -= a * z * logq(apr + EPS);
    t += 0.5Q * b * z * (a2 - z2) / (bpr * r + EPS);
    t -= b * z * logq(bpr + EPS);
    t += 2 * z * r / 3;
    t -= z * ((a2 + b2 - 2 * z2) / (6 * r));
    t -= a * b * atanq(a * b / (z * r));
    {
        Q num = a * b * z * (a * b / (r * r * r) + a * b / (z2 * r));
        Q den = a2 * b2 / (z2 * r * r) + 1;
        t += num / den;
    }
    return t;
}

/* ---- orthogonal potential antiderivative H (A.2 reading) ---------------------------- */
static Q H_orth(Q a, Q b, Q c) {
    Q a2 = a * a, b2 = b * b, c2 = c * c;
    Q r = sqrtq(a2 + b2 + c2);
    Q s = 0;
    s += a * b * c * logq(xpr(a, r, b2 + c2));
    s += (a2 * b / 2 - b2 * b / 6) * logq(xpr(c, r, a2 + b2));
    s += (a2 * c / 2 - c2 * c / 6) * logq(xpr(b, r, a2 + c2));
    s -= b * c * r / 3;
    s += (-a2 * a / 9 + a * b2 / 6 + a * c2 / 6) * atanq(b * c / (a * r));
    s += (a2 * a / 18 - a * b2 / 3 + a * c2 / 6) * atanq(a * c / (b * r));
    s += (a2 * a / 18 + a * b2 / 6 - a * c2 / 3) * atanq(a * b / (c * r));
    return s;
}

/* ---- Eq. (16) bracket, first term read as b(3a^2-b^2)/(6 r) (reading O3) */
static Q eq16(Q a, Q b, Q c) {
    Q a2 = a * a, b2 = b * b, c2 = c * c;
    Q r = sqrtq(a2 + b2 + c2), r2 = r * r;
    Q apr = xpr(a, r, b2 + c2), bpr = xpr(b, r, a2 + c2);
    Q t = 0;
    t += b * (3 * a2 - b2) / (6 * r);
    t += ((3 * a2 * c2 - c2 * c2) + 3 * (a2 - c2) * (r2 + b * r) * logq(bpr + EPS))
         / (6 * r * (bpr + EPS));
    t += a * b * c2 / (r * apr);
    t += a * b * logq(apr + EPS);
    t -= b * (r2 + c2) / (3 * r);
    t -= a2 * a2 * b / (6 * r * (a2 + c2));
    t -= a2 * b2 * b / (2 * r * (b2 + c2));
    t += a * c / 2 * (a * b * c * (r2 + c2) / (r * (a2 + c2) * (b2 + c2))
                      - 2 * atanq(a * b / (c * r) + EPS));
    return t;
}

static Q sgnq(Q x) { return x > 0 ? 1 : (x < 0 ? -1 : 0); }

/* kappa for one (kind, alpha, beta, D).  Axes 0,1,2 = x,y,z. */
static Q kappa_q(int kind, int alpha, int beta, const int64_t D[3]) {
    if (alpha == beta) {
        int n = alpha, u = (n + 1) % 3, v = (n + 2) % 3;
        /* observer [D_u, D_u+1] x [D_v, D_v+1] at z1 = D_n; source [0,1]^2 at z2 = 0 */
        Q xs1 = (Q)D[u], xe1 = xs1 + 1, xs2 = 0, xe2 = 1;
        Q ys1 = (Q)D[v], ye1 = ys1 + 1, ys2 = 0, ye2 = 1;
        Q a[4] = {xs2 - xe1, xe2 - xe1, xe2 - xs1, xs2 - xs1};
        Q b[4] = {ys2 - ye1, ye2 - ye1, ye2 - ys1, ys2 - ys1};
        Q z = 0 - (Q)D[n];
        Q s = 0;
        if (kind == 0) {
            for (int k = 0; k < 4; ++k)
                for (int m = 0; m < 4; ++m)
                    s += (((k + m) & 1) ? -1 : 1) * F_par(a[k], b[m], z);
            return s;
        }
        if (D[0] == 0 && D[1] == 0 && D[2] == 0) return 0; /* reading O4 */
        for (int k = 0; k < 4; ++k)
            for (int m = 0; m < 4; ++m)
                s += (((k + m) & 1) ? -1 : 1) * eq15(a[k], b[m], z + EPS);
        return -s; /* E+ = -Eq.(15): reading O2 */
    }
    /* orthogonal: observer normal alpha -> z, source normal beta -> y, other axis -> x */
    int g = 3 - alpha - beta;
    Q xs1 = (Q)D[g], xe1 = xs1 + 1, xs2 = 0, xe2 = 1;
    Q ys1 = (Q)D[beta], ye1 = ys1 + 1, y2 = 0;
    Q z1 = (Q)D[alpha], zs2 = 0, ze2 = 1;
    Q a[4] = {xs2 - xe1, xe2 - xe1, xe2 - xs1, xs2 - xs1};
    Q b[2] = {y2 - ys1, y2 - ye1};
    Q c[2] = {ze2 - z1, zs2 - z1};
    for (int k = 0; k < 4; ++k) if (a[k] == 0) a[k] = ETA;
    for (int m = 0; m < 2; ++m) if (b[m] == 0) b[m] = sgnq(b[1 - m]) * ETA;
    for (int l = 0; l < 2; ++l) if (c[l] == 0) c[l] = sgnq(c[1 - l]) * ETA;
    Q s = 0;
    for (int k = 0; k < 4; ++k)
        for (int m = 0; m < 2; ++m)
            for (int l = 0; l < 2; ++l) {
                int sg = (k + m + l) & 1; /* (-1)^{k+m+l} with 0-based = (-1)^{k+m+l+3} 1-based */
                if (kind == 0) {
                    /* (-1)^{k+m+l+1} (1-based) == (-1)^{k+m+l} (0-based) */
                    s += (sg ? -1 : 1) * H_orth(a[k], b[m], c[l]);
                } else {
                    /* (-1)^{k+m+l} (1-based) == -(-1)^{k+m+l} (0-based) */
                    s += (sg ? 1 : -1) * eq16(a[k], b[m], c[l]);
                }
            }
    return s;
}

/* ---- exported API (ctypes) ---------------------------------------------------------- */
double oq_kappa(int kind, int alpha, int beta, int64_t dx, int64_t dy, int64_t dz) {
    int64_t D[3] = {dx, dy, dz};
    return (double)kappa_q(kind, alpha, beta, D);
}

/* Same value rounded to double, also returning the low part (value - (double)value) so
 * tests can check extended-precision agreement. */
void oq_kappa_hilo(int kind, int alpha, int beta, int64_t dx, int64_t dy, int64_t dz,
                   double* hi, double* lo) {
    int64_t D[3] = {dx, dy, dz};
    Q v = kappa_q(kind, alpha, beta, D);
    double h = (double)v;
    *hi = h;
    *lo = (double)(v - (Q)h);
}

void oq_kappa_batch(int64_t n, const int32_t* kind, const int32_t* alpha,
                    const int32_t* beta, const int64_t* d, double* out) {
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i) {
        int64_t D[3] = {d[3 * i], d[3 * i + 1], d[3 * i + 2]};
        out[i] = (double)kappa_q(kind[i], alpha[i], beta[i], D);
    }
}
