// Matern covariance, Eq. (3) of PAPER.md:185-191,
//     C(h) = sigma2 / (2^(nu-1) Gamma(nu)) * (h/ell)^nu * K_nu(h/ell),   C(0) = sigma2,
// with the modified Bessel function K_nu evaluated on the device by
//   * Temme's series for |mu| <= 1/2, x <= 2 (N. M. Temme, J. Comput. Phys. 19 (1975)),
//   * Steed's continued fraction CF2 (Thompson & Barnett) for x > 2,
//   * upward recurrence K_{mu+k+1} = K_{mu+k-1} + 2 (mu+k)/x K_{mu+k}  (DLMF 10.29.1).
// Half-integer nu in {1/2, 3/2, 5/2} use the exact reductions of Eq. (3) (DLMF 10.49.12):
//   e^-x, (1+x) e^-x, (1+x+x^2/3) e^-x with x = h/ell (reading R1).
// __host__ __device__ so the same code is unit-tested on the CPU (tests/test_host_kernels.py).
#pragma once
#include <math.h>

#ifdef __CUDACC__
#define HD __host__ __device__ __forceinline__
#else
#define HD inline
#endif

// 1/Gamma(z) = sum_k c_k z^k  (Abramowitz & Stegun 6.1.34), used for Temme's gamma_1, gamma_2.
HD void hcov_temme_gammas(double mu, double *gam1, double *gam2, double *gampl, double *gammi)
{
    const double c[27] = {0.0,
        1.0, 0.5772156649015329, -0.6558780715202538, -0.0420026350340952, 0.1665386113822915,
        -0.0421977345555443, -0.0096219715278770, 0.0072189432466630, -0.0011651675918591,
        -0.0002152416741149, 0.0001280502823882, -0.0000201348547807, -0.0000012504934821,
        0.0000011330272320, -0.0000002056338417, 0.0000000061160950, 0.0000000050020075,
        -0.0000000011812746, 0.0000000001043427, 0.0000000000077823, -0.0000000000036968,
        0.0000000000005100, -0.0000000000000206, -0.0000000000000054, 0.0000000000000014,
        0.0000000000000001};
    // 1/Gamma(1+mu) = sum_k c_k mu^(k-1); 1/Gamma(1-mu) = sum_k c_k (-mu)^(k-1)
    double m2 = mu * mu;
    double g1 = 0.0, g2 = 0.0;       // g1 = -(c2 + c4 m2 + ...), g2 = c1 + c3 m2 + ...
    for (int k = 26; k >= 2; k -= 2) g1 = g1 * m2 + c[k];
    for (int k = 25; k >= 1; k -= 2) g2 = g2 * m2 + c[k];
    *gam1 = -g1;
    *gam2 = g2;
    // 1/Gamma(1+mu) = gam2 - mu*gam1 ; 1/Gamma(1-mu) = gam2 + mu*gam1
    *gampl = g2 + mu * g1;
    *gammi = g2 - mu * g1;
}

// exp(x) * K_mu(x), exp(x) * K_{mu+1}(x) for |mu| <= 1/2, x > 0.
HD void hcov_besselk_mu(double mu, double x, double *kmu_s, double *kmu1_s)
{
    const double EPS = 1e-17;
    const double PI = 3.141592653589793;
    if (x <= 2.0) {
        double x2 = 0.5 * x;
        double pimu = PI * mu;
        double fact = (fabs(pimu) < 1e-15) ? 1.0 : pimu / sin(pimu);
        double d = -log(x2);
        double e = mu * d;
        double fact2 = (fabs(e) < 1e-15) ? 1.0 : sinh(e) / e;
        double gam1, gam2, gampl, gammi;
        hcov_temme_gammas(mu, &gam1, &gam2, &gampl, &gammi);
        double ff = fact * (gam1 * cosh(e) + gam2 * fact2 * d);
        double sum = ff;
        double ee = exp(e);
        double p = 0.5 * ee / gampl;
        double q = 0.5 / (ee * gammi);
        double c = 1.0;
        double dd = x2 * x2;
        double sum1 = p;
        for (int i = 1; i < 500; ++i) {
            double di = (double)i;
            ff = (di * ff + p + q) / (di * di - mu * mu);
            c *= dd / di;
            p /= (di - mu);
            q /= (di + mu);
            double del = c * ff;
            sum += del;
            double del1 = c * (p - di * ff);
            sum1 += del1;
            if (fabs(del) < fabs(sum) * EPS) break;
        }
        double ex = exp(x);
        *kmu_s = sum * ex;
        *kmu1_s = sum1 * (2.0 / x) * ex;
    } else {
        double b = 2.0 * (1.0 + x);
        double d = 1.0 / b;
        double h = d, delh = d;
        double q1 = 0.0, q2 = 1.0;
        double a1 = 0.25 - mu * mu;
        double q = a1, c = a1;
        double a = -a1;
        double s = 1.0 + q * delh;
        for (int i = 1; i < 100000; ++i) {
            double di = (double)i;
            a -= 2.0 * di;
            c = -a * c / (di + 1.0);
            double qnew = (q1 - b * q2) / a;
            q1 = q2;
            q2 = qnew;
            q += c * qnew;
            b += 2.0;
            d = 1.0 / (b + a * d);
            delh = (b * d - 1.0) * delh;
            h += delh;
            double dels = q * delh;
            s += dels;
            if (fabs(dels / s) < EPS) break;
        }
        double kmu = sqrt(PI / (2.0 * x)) / s;   // scaled by e^x
        *kmu_s = kmu;
        *kmu1_s = kmu * (mu + x + 0.5 - a1 * h) / x;
    }
}

// exp(x) * K_nu(x), nu >= 0, x > 0.
HD double hcov_besselk_scaled(double nu, double x)
{
    int nl = (int)floor(nu + 0.5);
    double mu = nu - (double)nl;          // |mu| <= 1/2
    double k0, k1;
    hcov_besselk_mu(mu, x, &k0, &k1);     // K_mu, K_{mu+1} (scaled)
    for (int i = 1; i <= nl; ++i) {       // K_{mu+i+1} = K_{mu+i-1} + 2(mu+i)/x K_{mu+i}
        double k2 = k0 + 2.0 * (mu + (double)i) / x * k1;
        k0 = k1;
        k1 = k2;
    }
    return k0;                            // K_{mu+nl} = K_nu
}

HD double hcov_besselk(double nu, double x) { return exp(-x) * hcov_besselk_scaled(nu, x); }

// General nu: g(t) = x^nu K_nu(x) e^x with t = log x is analytic in t (singularities at
// Im t = +-pi), so a piecewise Chebyshev interpolant in t converges geometrically.  The table is
// built once per theta on the host from the series / continued fraction above (same accuracy,
// ~1e-16 interpolation error at degree 11 on intervals of width 0.32) and replaces ~100 divisions
// per entry by one Clenshaw recurrence.  Outside [KTAB_X0, KTAB_X1] the direct evaluation is used.
#define KTAB_NI 64
#define KTAB_NC 12
#define KTAB_X0 9.5367431640625e-07   /* 2^-20 */
#define KTAB_X1 745.0

// Matern parameters preprocessed once per theta.
struct MaternParams {
    double sigma2, inv_ell, nu, nugget;
    double pre;      // sigma2 * 2^(1-nu) / Gamma(nu)
    int kind;        // 0: nu=1/2, 1: nu=3/2, 2: nu=5/2, 3: general
    const double *tab;   // device: KTAB_NI x KTAB_NC Chebyshev coefficients of g (kind 3), or null
    double t0, inv_w;    // log(KTAB_X0), intervals per unit t
};

inline MaternParams hcov_matern_params(double sigma2, double ell, double nu, double nugget)
{
    MaternParams p;
    p.sigma2 = sigma2; p.inv_ell = 1.0 / ell; p.nu = nu; p.nugget = nugget;
    p.kind = (nu == 0.5) ? 0 : (nu == 1.5) ? 1 : (nu == 2.5) ? 2 : 3;
    p.pre = sigma2 * exp((1.0 - nu) * log(2.0) - lgamma(nu));
    p.tab = nullptr;
    p.t0 = log(KTAB_X0);
    p.inv_w = KTAB_NI / (log(KTAB_X1) - log(KTAB_X0));
    return p;
}

// Host: Chebyshev coefficients (KTAB_NI x KTAB_NC, row per interval) of g on each interval.
inline void hcov_matern_table(double nu, double *coef)
{
    const double PI = 3.141592653589793;
    const double t0 = log(KTAB_X0), w = (log(KTAB_X1) - t0) / KTAB_NI;
    const int N = KTAB_NC;
    for (int i = 0; i < KTAB_NI; ++i) {
        double f[KTAB_NC];
        for (int j = 0; j < N; ++j) {
            const double sj = cos(PI * (j + 0.5) / N);
            const double t = t0 + w * (i + 0.5 * (sj + 1.0));
            const double x = exp(t);
            f[j] = exp(nu * t) * hcov_besselk_scaled(nu, x);
        }
        for (int k = 0; k < N; ++k) {
            double sum = 0.0;
            for (int j = 0; j < N; ++j) sum += f[j] * cos(PI * k * (j + 0.5) / N);
            coef[i * N + k] = (k == 0 ? 1.0 : 2.0) * sum / N;
        }
    }
}

HD double hcov_matern_tab(const MaternParams &p, double x, double lx)
{
    const double u = (lx - p.t0) * p.inv_w;
    int i = (int)u;
    if (i > KTAB_NI - 1) i = KTAB_NI - 1;
    const double s = 2.0 * (u - i) - 1.0, s2 = 2.0 * s;
    const double *c = p.tab + i * KTAB_NC;
    double b1 = 0.0, b2 = 0.0;
#pragma unroll
    for (int k = KTAB_NC - 1; k >= 1; --k) {
        const double b0 = fma(s2, b1, c[k] - b2);
        b2 = b1;
        b1 = b0;
    }
    const double g = fma(s, b1, c[0] - b2);
    return p.pre * g * exp(-x);
}

// C(h), h >= 0 (Eq. (3)); no nugget.
HD double hcov_matern(const MaternParams &p, double h)
{
    if (h == 0.0) return p.sigma2;
    double x = h * p.inv_ell;
    switch (p.kind) {
    case 0: return p.sigma2 * exp(-x);
    case 1: return p.sigma2 * (1.0 + x) * exp(-x);
    case 2: return p.sigma2 * (1.0 + x + x * x * (1.0 / 3.0)) * exp(-x);
    default: {
        if (x > 740.0) return 0.0;
        double lx = log(x);
        if (p.tab && x >= KTAB_X0) return hcov_matern_tab(p, x, lx);
        return p.pre * exp(p.nu * lx - x) * hcov_besselk_scaled(p.nu, x);
    }
    }
}

// Covariance entry between internal positions a and b with coordinates (xa,ya), (xb,yb).
// Phantom positions (padding, NaN coordinates) form an identity block.
HD double hcov_cov_entry(const MaternParams &p, double xa, double ya, double xb, double yb, bool same)
{
    if (isnan(xa) || isnan(xb)) return same ? 1.0 : 0.0;
    double dx = xa - xb, dy = ya - yb;
    double c = hcov_matern(p, sqrt(dx * dx + dy * dy));
    if (same) c += p.nugget;
    return c;
}
