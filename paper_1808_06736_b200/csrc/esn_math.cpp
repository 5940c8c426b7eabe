// esn_math.cpp -- host-side kernel mathematics for the B200 NUFFT core.
//
// Parameter recipe, 5-smooth fine-grid sizes, Gauss-Legendre quadrature,
// the phase-winding phi-hat correction and the piecewise-polynomial fit of
// the ES kernel.  These run once per plan on the host (microseconds) and feed
// device tables; they restate the published algorithm of arXiv 1808.06736
// as specified by the reference package (citations: /root/reference/pkg/src/
// esnufft/<file>:<line>).
#include "esn_internal.h"

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <vector>

namespace esn {

static const double kGammaSafety = 0.976;  // kernel.py:37

static double decay_rate(double sigma) {  // kernel.py:86-89
    const double g = kGammaSafety;
    return g * std::sqrt(1.0 - 1.0 / sigma - (1.0 / (g * g) - 1.0) / (4.0 * sigma * sigma));
}

static bool sigma_ok(double s) { return s == 2.0 || s == 1.25; }

int params_for_width(int w, double sigma, esn_kernel_params *out) {
    // kernel.py:98-107 + validation of KernelParams.__post_init__ (:61-77)
    if (!sigma_ok(sigma)) return fail(ESN_BAD_TOLERANCE, "sigma %g unsupported; choose one of (2.0, 1.25)", sigma);
    if (w < 2 || w > 16) return fail(ESN_BAD_TOLERANCE, "kernel width %d outside [2, 16]", w);
    double beta = (sigma == 2.0) ? 2.30 * w : kGammaSafety * M_PI * w * (1.0 - 1.0 / (2.0 * sigma));
    out->w = w;
    out->beta = beta;
    out->sigma = sigma;
    out->gamma = beta / (M_PI * w * (1.0 - 1.0 / (2.0 * sigma)));
    out->p_quad = (int)std::ceil(1.5 * w + 2);
    return ESN_SUCCESS;
}

int select_params(double tol, double sigma, esn_kernel_params *out) {
    // kernel.py:110-131: w = ceil(log10(1/tol)) + 1 clamped to [2, 16]
    if (!(tol >= 1e-15 && tol <= 1e-1) || std::isnan(tol))
        return fail(ESN_BAD_TOLERANCE, "tolerance %g outside supported range [1e-15, 0.1]", tol);
    if (!sigma_ok(sigma)) return fail(ESN_BAD_TOLERANCE, "sigma %g unsupported; choose one of (2.0, 1.25)", sigma);
    double digits = std::log10(1.0 / tol);
    if (sigma != 2.0) digits = digits / (decay_rate(sigma) / decay_rate(2.0));
    int w = (int)std::ceil(digits) + 1;
    w = std::min(std::max(w, 2), 16);
    return params_for_width(w, sigma, out);
}

double class_tolerance(int w, double sigma) {  // kernel.py:134-143
    double digits = (double)(w - 1);
    if (sigma != 2.0) digits = digits * (decay_rate(sigma) / decay_rate(2.0));
    return std::pow(10.0, -digits);
}

int64_t next_smooth(int64_t n) {  // grid.py:34-58
    if (n <= 1) return 1;
    int64_t best = INT64_MAX;
    for (int64_t p2 = 1;; p2 *= 2) {
        for (int64_t p23 = p2;; p23 *= 3) {
            int64_t v = p23;
            while (v < n) v *= 5;
            best = std::min(best, v);
            if (p23 >= n) break;
        }
        if (p2 >= n) break;
    }
    return best;
}

void gauss_legendre(int n, double *x, double *wts) {
    // kernel.py:167-203: Newton iteration on the Legendre three-term
    // recurrence from cos(pi (i + 3/4) / (n + 1/2)); sorted ascending.
    if (n == 1) {
        x[0] = 0.0;
        wts[0] = 2.0;
        return;
    }
    std::vector<double> xs(n), pn(n), pm(n);
    for (int i = 0; i < n; ++i) xs[i] = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    auto legendre = [&](void) {
        for (int i = 0; i < n; ++i) {
            double p0 = 1.0, p1 = xs[i];
            for (int k = 2; k <= n; ++k) {
                double p2 = ((2 * k - 1) * xs[i] * p1 - (k - 1) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            pn[i] = p1;
            pm[i] = p0;
        }
    };
    for (int it = 0; it < 100; ++it) {
        legendre();
        double mx = 0.0;
        for (int i = 0; i < n; ++i) {
            double dp = n * (xs[i] * pn[i] - pm[i]) / (xs[i] * xs[i] - 1.0);
            double dx = pn[i] / dp;
            xs[i] -= dx;
            mx = std::max(mx, std::fabs(dx));
        }
        if (mx < 1e-15) break;
    }
    legendre();
    std::vector<int> order(n);
    for (int i = 0; i < n; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int a, int b) { return xs[a] < xs[b]; });
    for (int i = 0; i < n; ++i) {
        int o = order[i];
        double dp = n * (xs[o] * pn[o] - pm[o]) / (xs[o] * xs[o] - 1.0);
        x[i] = xs[o];
        wts[i] = 2.0 / ((1.0 - xs[o] * xs[o]) * dp * dp);
    }
}

static double es_eval(double z, double beta) {  // kernel.py:146-158
    if (std::fabs(z) > 1.0) return 0.0;
    return std::exp(beta * (std::sqrt(1.0 - z * z) - 1.0));
}

// Positive half of the 2p-node rule, with a_j = w_j phi(q_j) (kernel.py:206-231).
static void positive_quad(const esn_kernel_params &p, std::vector<double> &q, std::vector<double> &a) {
    int n2 = 2 * p.p_quad;
    std::vector<double> x(n2), w(n2);
    gauss_legendre(n2, x.data(), w.data());
    q.assign(x.begin() + p.p_quad, x.end());
    a.resize(p.p_quad);
    for (int j = 0; j < p.p_quad; ++j) a[j] = w[p.p_quad + j] * es_eval(q[j], p.beta);
}

void kernel_ft(const esn_kernel_params &p, double alpha, int64_t nk, const double *k, double *out) {
    // kernel.py:213-231
    std::vector<double> q, a;
    positive_quad(p, q, a);
    for (int64_t i = 0; i < nk; ++i) {
        double s = 0.0;
        for (size_t j = 0; j < q.size(); ++j) s += std::cos(alpha * k[i] * q[j]) * a[j];
        out[i] = 2.0 * alpha * s;
    }
}

int fseries_correction(const esn_kernel_params &p, int64_t n, int64_t nmodes, double *out) {
    // kernel.py:234-288: p_k = h / psi_hat(k), psi_hat by p_quad complex
    // exponentials advanced by phase winding (cumulative products restarted
    // every 1024 modes from z^1024 powers).
    if (nmodes < 1 || n < nmodes)
        return fail(ESN_SIZE_ERROR, "need 1 <= num_modes <= n, got num_modes=%lld, n=%lld",
                    (long long)nmodes, (long long)n);
    const double alpha = M_PI * p.w / (double)n;
    std::vector<double> q, a;
    positive_quad(p, q, a);
    const int P = (int)q.size();
    for (int j = 0; j < P; ++j) a[j] *= 2.0 * alpha;
    const int64_t kmax = nmodes / 2;
    std::vector<std::complex<double>> z(P), zc(P), ph(P, 1.0), cur(P);
    for (int j = 0; j < P; ++j) {
        z[j] = std::exp(std::complex<double>(0.0, alpha * q[j]));
        zc[j] = z[j];
        for (int s = 0; s < 10; ++s) zc[j] = zc[j] * zc[j];  // z^1024
    }
    std::vector<double> psi(kmax + 1);
    const int64_t chunk = 1024;
    for (int64_t s = 0; s <= kmax; s += chunk) {
        int64_t m = std::min(chunk, kmax + 1 - s);
        for (int j = 0; j < P; ++j) cur[j] = ph[j];
        for (int64_t r = 0; r < m; ++r) {
            if (r > 0)
                for (int j = 0; j < P; ++j) cur[j] = cur[j] * z[j];
            double acc = 0.0;
            for (int j = 0; j < P; ++j) acc += cur[j].real() * a[j];
            psi[s + r] = acc;
        }
        for (int j = 0; j < P; ++j) ph[j] = ph[j] * zc[j];
    }
    for (int64_t k = 0; k <= kmax; ++k)
        if (!(psi[k] > 0.0))
            return fail(ESN_INTERNAL_ERROR, "kernel transform non-positive at mode %lld (w=%d, p_quad=%d)",
                        (long long)k, p.w, p.p_quad);
    const double h = 2.0 * M_PI / (double)n;
    for (int64_t i = 0; i < nmodes; ++i) {
        int64_t k = i - nmodes / 2;
        out[i] = h / psi[k < 0 ? -k : k];
    }
    return ESN_SUCCESS;
}

// Real least squares  min || A c - b ||  by Householder QR (A is m x n, row
// major, m >= n).  The complex collocation system of the reference is
// symmetric about the real axis, so its solution is real; stacking
// [Re A; Im A] c = [Re b; Im b] gives the same minimiser over real c.
static void lstsq_qr(int m, int n, std::vector<double> A, std::vector<double> b, double *c) {
    for (int k = 0; k < n; ++k) {
        double nrm = 0.0;
        for (int i = k; i < m; ++i) nrm += A[i * n + k] * A[i * n + k];
        nrm = std::sqrt(nrm);
        if (nrm == 0.0) continue;
        double alpha = A[k * n + k] > 0 ? -nrm : nrm;
        std::vector<double> v(m - k);
        for (int i = k; i < m; ++i) v[i - k] = A[i * n + k];
        v[0] -= alpha;
        double vv = 0.0;
        for (double e : v) vv += e * e;
        if (vv == 0.0) continue;
        for (int j = k; j < n; ++j) {
            double s = 0.0;
            for (int i = k; i < m; ++i) s += v[i - k] * A[i * n + j];
            s = 2.0 * s / vv;
            for (int i = k; i < m; ++i) A[i * n + j] -= s * v[i - k];
        }
        double s = 0.0;
        for (int i = k; i < m; ++i) s += v[i - k] * b[i];
        s = 2.0 * s / vv;
        for (int i = k; i < m; ++i) b[i] -= s * v[i - k];
    }
    for (int k = n - 1; k >= 0; --k) {
        double s = b[k];
        for (int j = k + 1; j < n; ++j) s -= A[k * n + j] * c[j];
        c[k] = s / A[k * n + k];
    }
}

int piecewise_poly(const esn_kernel_params &p, double *coeffs, double *residual_out) {
    // kernel.py:322-367: per piece m, degree w+3 in the local coordinate t
    // (z = center_m + t / w), collocated on 2(w+4) corner-clustered points
    // of the unit square boundary, rows weighted by 1/sqrt(d + 0.5/w) with d
    // the distance to the nearer kernel endpoint.
    const int w = p.w, deg = w + 3, nc = deg + 1, npts = 2 * nc;
    std::vector<std::complex<double>> tb(npts);
    for (int i = 0; i < npts; ++i) {
        double u = 2.0 * M_PI * (i + 0.5) / npts;
        double th = u - 0.25 * std::sin(4.0 * u);
        double cs = std::cos(th), sn = std::sin(th);
        tb[i] = std::complex<double>(cs, sn) / std::max(std::fabs(cs), std::fabs(sn));
    }
    double residual = 0.0;
    std::vector<std::complex<double>> V(npts * nc);
    for (int i = 0; i < npts; ++i) {
        std::complex<double> pw = 1.0;
        for (int j = nc - 1; j >= 0; --j) {  // highest degree first
            V[i * nc + j] = pw;
            pw *= tb[i];
        }
    }
    for (int m = 0; m < w; ++m) {
        const double center = -1.0 + (2.0 * m + 1.0) / w;
        std::vector<double> A(2 * npts * nc), b(2 * npts);
        std::vector<std::complex<double>> fb(npts);
        for (int i = 0; i < npts; ++i) {
            std::complex<double> zb = center + tb[i] / (double)w;
            fb[i] = std::exp(p.beta * (std::sqrt(1.0 - zb * zb) - 1.0));
            double d = std::min(std::abs(zb - 1.0), std::abs(zb + 1.0));
            double wt = 1.0 / std::sqrt(d + 0.5 / w);
            for (int j = 0; j < nc; ++j) {
                A[i * nc + j] = wt * V[i * nc + j].real();
                A[(npts + i) * nc + j] = wt * V[i * nc + j].imag();
            }
            b[i] = wt * fb[i].real();
            b[npts + i] = wt * fb[i].imag();
        }
        double *cm = coeffs + (size_t)m * nc;
        lstsq_qr(2 * npts, nc, A, b, cm);
        for (int i = 0; i < npts; ++i) {
            std::complex<double> v = 0.0;
            for (int j = 0; j < nc; ++j) v += V[i * nc + j] * cm[j];
            residual = std::max(residual, std::abs(v - fb[i]));
        }
    }
    if (residual_out) *residual_out = residual;
    double limit = std::max(class_tolerance(w, p.sigma), 1000.0 * 2.220446049250313e-16);
    if (residual > limit)
        return fail(ESN_INTERNAL_ERROR, "piecewise kernel fit failed for w=%d: collocation residual %.3e exceeds %.3e",
                    w, residual, limit);
    return ESN_SUCCESS;
}

}  // namespace esn
