/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU code.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this.  It shares no code with paper_1709_08625_b200/ (the CUDA path).
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md):
 *   Eq. (3), PAPER.md:185-191 (Sec. 2.1 "Matern covariance functions"):
 *       C(h; theta) = sigma^2 / (2^(nu-1) Gamma(nu)) * (h/ell)^nu * K_nu(h/ell),   C(0) = sigma^2.
 *   K_nu, the modified Bessel function of the second kind, from its integral representation
 *       K_nu(x) = int_0^inf exp(-x cosh t) cosh(nu t) dt          (DLMF 10.32.9)
 *   evaluated by the trapezoid rule.  This is deliberately a different algorithm from the
 *   device code (series + continued fraction), see DESIGN.md "Oracle".
 *   Half-integer nu in {1/2, 3/2, 5/2}: Eq. (3) reduces exactly (DLMF 10.47.9 / 10.49.12) to
 *       e^-x, (1+x) e^-x, (1 + x + x^2/3) e^-x  with x = h/ell   (reading R1 in DESIGN.md:
 *   Eq. (3) literally; PAPER.md:205-208 prints the same forms with argument sqrt(2 nu) h/ell).
 *   The dense matrix entries follow Eq. (1)'s definition C_ij = C(s_i - s_j; theta)
 *    plus the nugget tau^2 on the diagonal (listing).
 */
#include <math.h>
#include <stdint.h>

/* exp(x) * K_nu(x) by the trapezoid rule on int_0^inf exp(-x (cosh t - 1)) cosh(nu t) dt.
 * Step h = min(0.05, 0.5/sqrt(x)): near t = 0 the integrand is ~exp(-x t^2/2), whose
 * trapezoid error is ~exp(-2 pi^2/(x h^2)) <= e^-79.  The sum stops once t is past the integrand's maximum and the term is
 * below 1e-18 of the running sum (double-exponential decay). */
double oracle_besselk_scaled(double nu, double x)
{
    const double h = fmin(0.05, 0.5 / sqrt(x));
    /* c = cosh(t) - 1, sh = sinh(t), e = exp(nu t), advanced by the addition theorems
     * cosh(t+h) = cosh t cosh h + sinh t sinh h, sinh(t+h) = sinh t cosh h + cosh t sinh h. */
    const double ch1 = 2.0 * sinh(0.5 * h) * sinh(0.5 * h);   /* cosh h - 1 */
    const double chh = 1.0 + ch1, shh = sinh(h), eh = exp(nu * h);
    double c = 0.0, sh = 0.0, e = 1.0;
    double sum = 0.5;                        /* t = 0 term: exp(0) cosh(0) / 2 */
    /* integrand maximum (for the stopping rule): where x sinh t = nu */
    double tpk = asinh(nu / x);
    for (int k = 1; k < 200000; ++k) {
        double t = k * h;
        double c2 = c * chh + ch1 + sh * shh;
        double s2 = sh * chh + (c + 1.0) * shh;
        c = c2; sh = s2; e *= eh;
        /* exp(-x (cosh t - 1)) * cosh(nu t) = exp(-x c) * (e + 1/e) / 2 */
        double f = exp(-x * c) * 0.5 * (e + 1.0 / e);
        sum += f;
        if (t > tpk && f < 1e-18 * sum) break;
    }
    return h * sum;
}

double oracle_besselk(double nu, double x)
{
    return exp(-x) * oracle_besselk_scaled(nu, x);
}

/* Eq. (3). Closed forms at nu in {1/2,3/2,5/2}, integral otherwise. */
double oracle_matern(double h, double sigma2, double ell, double nu)
{
    if (h == 0.0) return sigma2;
    double x = h / ell;
    if (nu == 0.5) return sigma2 * exp(-x);
    if (nu == 1.5) return sigma2 * (1.0 + x) * exp(-x);
    if (nu == 2.5) return sigma2 * (1.0 + x + x * x / 3.0) * exp(-x);
    /* sigma^2 2^(1-nu)/Gamma(nu) x^nu e^-x [e^x K_nu(x)] */
    double lg = lgamma(nu);
    double pre = exp((1.0 - nu) * log(2.0) - lg + nu * log(x) - x);
    if (pre == 0.0) return 0.0;
    return sigma2 * pre * oracle_besselk_scaled(nu, x);
}

/* Same, forcing the integral representation (used by the pins that compare the
 * integral against the closed forms). */
double oracle_matern_integral(double h, double sigma2, double ell, double nu)
{
    if (h == 0.0) return sigma2;
    double x = h / ell;
    double lg = lgamma(nu);
    double pre = exp((1.0 - nu) * log(2.0) - lg + nu * log(x) - x);
    if (pre == 0.0) return 0.0;
    return sigma2 * pre * oracle_besselk_scaled(nu, x);
}

/* Euclidean distance |s_i - s_j| of dim-dimensional points (dim = 2, or 3 for the 3-D variant,
 * PAPER.md:684-686), s: n x dim row-major. */
static double dist_ij(const double *s, int dim, int64_t i, int64_t j)
{
    double h2 = 0.0;
    for (int k = 0; k < dim; ++k) {
        double d = s[dim * i + k] - s[dim * j + k];
        h2 += d * d;
    }
    return sqrt(h2);
}

/* Dense covariance, EXTERNAL order, full symmetric n x n row-major:
 *   C_ij = C(|s_i - s_j|; theta) + nugget * [i == j].     s: n x dim row-major. */
void oracle_cov_dense(int64_t n, int dim, const double *s, double sigma2, double ell, double nu,
                      double nugget, double *C)
{
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = 0; j <= i; ++j) {
            double c = oracle_matern(dist_ij(s, dim, i, j), sigma2, ell, nu);
            if (i == j) c += nugget;
            C[i * n + j] = c;
            C[j * n + i] = c;
        }
    }
}

/* Selected entries C_{rows[a], cols[b]} (external indices), out: nr x nc row-major.
 * Used for sampled-column checks at oracle-infeasible n. */
void oracle_cov_entries(int64_t n, int dim, const double *s, double sigma2, double ell, double nu,
                        double nugget, const int64_t *rows, int64_t nr,
                        const int64_t *cols, int64_t nc, double *out)
{
    (void)n;
    #pragma omp parallel for schedule(static)
    for (int64_t a = 0; a < nr; ++a)
        for (int64_t b = 0; b < nc; ++b) {
            int64_t i = rows[a], j = cols[b];
            double c = oracle_matern(dist_ij(s, dim, i, j), sigma2, ell, nu);
            if (i == j) c += nugget;
            out[a * nc + b] = c;
        }
}
