// Host build of the device Matern / K_nu code (paper_1709_08625_b200/csrc/matern.cuh) for CPU tests.
#include <cstdint>
#include "../../paper_1709_08625_b200/csrc/matern.cuh"

extern "C" {
double host_besselk(double nu, double x) { return hcov_besselk(nu, x); }
// C(h) with the direct series / continued fraction (tab = 0) or the Chebyshev table (tab = 1)
void host_matern(double sigma2, double ell, double nu, const double *h, int64_t n, int tab, double *out)
{
    MaternParams p = hcov_matern_params(sigma2, ell, nu, 0.0);
    static double coef[KTAB_NI * KTAB_NC];
    if (tab && p.kind == 3) {
        hcov_matern_table(nu, coef);
        p.tab = coef;
    }
    for (int64_t i = 0; i < n; ++i) out[i] = hcov_matern(p, h[i]);
}
}
