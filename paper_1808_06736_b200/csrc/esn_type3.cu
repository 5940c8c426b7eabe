// esn_type3.cu -- the device pieces of the type-3 transform around the
// composed spread + type 2 (transforms.py:267-351):
//   * pre-phase: c_j e^{i sum_d s0_d (x_dj - x0_d)} (conjugated input for
//     isign < 0) and the rescaled source coordinates (x_dj - x0_d) / gamma_d;
//   * inner targets: (2 pi / n_d) gamma_d (s_dk - s0_d);
//   * the per-target correction prod_d (2 pi / n_d) / psi-hat_d(gamma_d (s_dk
//     - s0_d)) with psi-hat by the Gauss-Legendre rule of kernel_ft
//     (kernel.py:211-229), times the post-phase e^{i sum_d x0_d s_dk}, then
//     the final conjugation for isign < 0;
//   * the centring permutation of the spread grid (fftshift).
// One thread per point / target; float64 throughout (the reference's type 3
// is float64 only).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <vector>

#include "esn_internal.h"

namespace esn {

struct T3Geo {
    int dim;
    double x0[3], s0[3], gamma[3], n[3];
};

__global__ void k_type3_prephase(T3Geo g, int64_t M, const double *x, const double *y, const double *z, int conj,
                                 const double2 *cin, double2 *cout, double *xr, double *yr, double *zr) {
    const double *xs[3] = {x, y, z};
    double *rs[3] = {xr, yr, zr};
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x) {
        double ph = 0.0;
        bool shifted = false;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            if (d >= g.dim) break;
            const double xt = g.x0[d] != 0.0 ? xs[d][j] - g.x0[d] : xs[d][j];
            rs[d][j] = xt / g.gamma[d];
            if (g.s0[d] != 0.0) {  // (unfused multiply-add, as numpy)
                ph = shifted ? __dadd_rn(ph, __dmul_rn(g.s0[d], xt)) : __dmul_rn(g.s0[d], xt);
                shifted = true;
            }
        }
        double2 c = cin[j];
        if (conj) c.y = -c.y;
        if (shifted) {
            double sn, cs;
            sincos(ph, &sn, &cs);
            c = make_double2(c.x * cs - c.y * sn, c.x * sn + c.y * cs);
        }
        cout[j] = c;
    }
}

__global__ void k_type3_targets(T3Geo g, int64_t K, const double *s1, const double *s2, const double *s3,
                                double *t1, double *t2, double *t3) {
    const double *ss[3] = {s1, s2, s3};
    double *ts[3] = {t1, t2, t3};
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < K; k += (int64_t)gridDim.x * blockDim.x)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            if (d >= g.dim) break;
            const double st = g.s0[d] != 0.0 ? ss[d][k] - g.s0[d] : ss[d][k];
            ts[d][k] = (2.0 * M_PI / g.n[d]) * g.gamma[d] * st;
        }
}

constexpr int kMaxQuad = 64;  // positive Gauss-Legendre nodes of kernel_ft (p_quad <= 64)

struct T3Quad {
    int nq;
    double alpha[3];
    double q[kMaxQuad], a[kMaxQuad];  // nodes, weights * phi(node)
};

__global__ void k_type3_correct(T3Geo g, T3Quad qd, int64_t K, const double *s1, const double *s2, const double *s3,
                                int conj, double2 *out) {
    const double *ss[3] = {s1, s2, s3};
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < K; k += (int64_t)gridDim.x * blockDim.x) {
        double2 v = out[k];
        double post = 0.0;
        bool shifted = false;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            if (d >= g.dim) break;
            const double sd = ss[d][k];
            const double st = g.s0[d] != 0.0 ? sd - g.s0[d] : sd;
            // psi-hat(gamma (s - s0)) = 2 alpha sum_j a_j cos(alpha gamma (s - s0) q_j)
            const double arg = qd.alpha[d] * (g.gamma[d] * st);
            double acc = 0.0;
            for (int i = 0; i < qd.nq; ++i) acc = fma(qd.a[i], cos(arg * qd.q[i]), acc);
            const double f = (2.0 * M_PI / g.n[d]) / (2.0 * qd.alpha[d] * acc);
            v.x *= f;
            v.y *= f;
            if (g.x0[d] != 0.0) {
                post = shifted ? __dadd_rn(post, __dmul_rn(g.x0[d], sd)) : __dmul_rn(g.x0[d], sd);
                shifted = true;
            }
        }
        if (shifted) {
            double sn, cs;
            sincos(post, &sn, &cs);
            v = make_double2(v.x * cs - v.y * sn, v.x * sn + v.y * cs);
        }
        if (conj) v.y = -v.y;
        out[k] = v;
    }
}

// numpy fftshift in every dimension: out[k] = in[(k - n//2) mod n]
__global__ void k_fftshift(int dim, int n1, int n2, int n3, const double2 *in, double2 *out) {
    const int64_t total = (int64_t)n1 * n2 * n3;
    const int h1 = n1 / 2, h2 = dim > 1 ? n2 / 2 : 0, h3 = dim > 2 ? n3 / 2 : 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int i1 = (int)(i % n1);
        const int64_t r = i / n1;
        const int i2 = (int)(r % n2);
        const int i3 = (int)(r / n2);
        int j1 = i1 - h1;
        if (j1 < 0) j1 += n1;
        int j2 = i2 - h2;
        if (j2 < 0) j2 += n2;
        int j3 = i3 - h3;
        if (j3 < 0) j3 += n3;
        out[i] = in[((int64_t)j3 * n2 + j2) * n1 + j1];
    }
}

static int blocks_for(int64_t n) {
    int64_t b = (n + 255) / 256;
    const int64_t cap = (int64_t)device_sm_count() * 16;
    if (b > cap) b = cap;
    return b < 1 ? 1 : (int)b;
}

static int make_geo(int dim, const double *x0, const double *s0, const double *gamma, const int64_t *n, T3Geo *g) {
    if (dim < 1 || dim > 3) return fail(ESN_SIZE_ERROR, "dimension must be 1, 2, or 3");
    g->dim = dim;
    for (int d = 0; d < 3; ++d) {
        g->x0[d] = d < dim && x0 ? x0[d] : 0.0;
        g->s0[d] = d < dim && s0 ? s0[d] : 0.0;
        g->gamma[d] = d < dim && gamma ? gamma[d] : 1.0;
        g->n[d] = d < dim && n ? (double)n[d] : 1.0;
        if (d < dim && !(g->gamma[d] > 0.0)) return fail(ESN_SIZE_ERROR, "type-3 gamma must be positive");
        if (d < dim && n && n[d] < 1) return fail(ESN_SIZE_ERROR, "type-3 grid size must be positive");
    }
    return ESN_SUCCESS;
}

}  // namespace esn

using namespace esn;

extern "C" {

int esn_type3_prephase(int dim, int64_t M, const double *x, const double *y, const double *z, const double *x0,
                       const double *s0, const double *gamma, int conj, const void *c_in, void *c_out, double *xr,
                       double *yr, double *zr, void *stream) {
    T3Geo g;
    int rc = make_geo(dim, x0, s0, gamma, nullptr, &g);
    if (rc) return rc;
    if (M < 0) return fail(ESN_SIZE_ERROR, "negative point count");
    if (M == 0) return ESN_SUCCESS;
    const double *xs[3] = {x, y, z};
    double *rs[3] = {xr, yr, zr};
    for (int d = 0; d < dim; ++d)
        if (!xs[d] || !rs[d]) return fail(ESN_SIZE_ERROR, "coordinate array %d missing", d + 1);
    if (!c_in || !c_out) return fail(ESN_SIZE_ERROR, "null strength array");
    k_type3_prephase<<<blocks_for(M), 256, 0, (cudaStream_t)stream>>>(g, M, x, y, z, conj, (const double2 *)c_in,
                                                                      (double2 *)c_out, xr, yr, zr);
    ESN_CUDA_TRY(cudaGetLastError());
    return ESN_SUCCESS;
}

int esn_type3_targets(int dim, int64_t K, const double *s1, const double *s2, const double *s3, const double *s0,
                      const double *gamma, const int64_t *n, double *t1, double *t2, double *t3, void *stream) {
    T3Geo g;
    int rc = make_geo(dim, nullptr, s0, gamma, n, &g);
    if (rc) return rc;
    if (K < 0) return fail(ESN_SIZE_ERROR, "negative target count");
    if (K == 0) return ESN_SUCCESS;
    const double *ss[3] = {s1, s2, s3};
    double *ts[3] = {t1, t2, t3};
    for (int d = 0; d < dim; ++d)
        if (!ss[d] || !ts[d]) return fail(ESN_SIZE_ERROR, "target array %d missing", d + 1);
    k_type3_targets<<<blocks_for(K), 256, 0, (cudaStream_t)stream>>>(g, K, s1, s2, s3, t1, t2, t3);
    ESN_CUDA_TRY(cudaGetLastError());
    return ESN_SUCCESS;
}

int esn_type3_correct(int dim, int64_t K, const double *s1, const double *s2, const double *s3, const double *x0,
                      const double *s0, const double *gamma, const int64_t *n, const esn_kernel_params *kp, int conj,
                      void *out, void *stream) {
    T3Geo g;
    int rc = make_geo(dim, x0, s0, gamma, n, &g);
    if (rc) return rc;
    if (!kp) return fail(ESN_SIZE_ERROR, "null kernel parameters");
    if (K < 0) return fail(ESN_SIZE_ERROR, "negative target count");
    if (K == 0) return ESN_SUCCESS;
    const double *ss[3] = {s1, s2, s3};
    for (int d = 0; d < dim; ++d)
        if (!ss[d]) return fail(ESN_SIZE_ERROR, "target array %d missing", d + 1);
    if (!out) return fail(ESN_SIZE_ERROR, "null output array");
    // kernel_ft's rule: the positive half of a 2 p_quad Gauss-Legendre rule
    // on [-1, 1], weights times phi at the nodes (kernel.py:211-229)
    const int nq2 = 2 * kp->p_quad;
    if (kp->p_quad < 1 || kp->p_quad > kMaxQuad) return fail(ESN_SIZE_ERROR, "p_quad %d out of range", kp->p_quad);
    std::vector<double> q(nq2), w(nq2);
    if ((rc = esn_gauss_legendre(nq2, q.data(), w.data()))) return rc;
    T3Quad qd{};
    qd.nq = kp->p_quad;
    for (int i = 0; i < qd.nq; ++i) {
        const double z = q[kp->p_quad + i];
        const double a = 1.0 - z * z;
        qd.q[i] = z;
        qd.a[i] = w[kp->p_quad + i] * (a > 0.0 ? std::exp(kp->beta * (std::sqrt(a) - 1.0)) : 0.0);
    }
    for (int d = 0; d < 3; ++d) qd.alpha[d] = d < dim ? M_PI * kp->w / (double)n[d] : 1.0;
    k_type3_correct<<<blocks_for(K), 256, 0, (cudaStream_t)stream>>>(g, qd, K, s1, s2, s3, conj, (double2 *)out);
    ESN_CUDA_TRY(cudaGetLastError());
    return ESN_SUCCESS;
}

int esn_fftshift(int dim, const int64_t *n, const void *in, void *out, void *stream) {
    if (dim < 1 || dim > 3 || !n) return fail(ESN_SIZE_ERROR, "dimension must be 1, 2, or 3");
    int nn[3] = {1, 1, 1};
    for (int d = 0; d < dim; ++d) {
        if (n[d] < 1 || n[d] > INT_MAX) return fail(ESN_SIZE_ERROR, "invalid grid shape");
        nn[d] = (int)n[d];
    }
    if (!in || !out || in == out) return fail(ESN_SIZE_ERROR, "fftshift needs distinct input and output arrays");
    const int64_t total = (int64_t)nn[0] * nn[1] * nn[2];
    k_fftshift<<<blocks_for(total), 256, 0, (cudaStream_t)stream>>>(dim, nn[0], nn[1], nn[2], (const double2 *)in,
                                                                   (double2 *)out);
    ESN_CUDA_TRY(cudaGetLastError());
    return ESN_SUCCESS;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// One-shot host-buffer type 3 (the esnufftpy nufft{1,2,3}d3 analog,
// bindings/src/esnufftpy/__init__.py:155-215 over transforms.py:267-351):
// geometry on the host (min / max of the host arrays, as
// plan_type3_geometry), then the device composition prephase -> spreader
// plan -> fftshift -> inner type-2 plan -> correction.
namespace {

double axis_shift(double vmin, double vmax) {  // transforms.py:233-242
    const double mid = 0.5 * (vmin + vmax);
    if (mid == 0.0) return 0.0;
    const double before = std::max(std::fabs(vmin), std::fabs(vmax));
    const double after = 0.5 * (vmax - vmin);
    return 2.0 * after < before ? mid : 0.0;
}

struct DevBuf {
    void *p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    int alloc(size_t bytes) {
        if (cudaMalloc(&p, bytes ? bytes : 16) != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            return fail(ESN_RESOURCE_ERROR, "device allocation of %zu bytes failed", bytes);
        }
        return ESN_SUCCESS;
    }
};

struct PlanGuard {
    esn_plan p = nullptr;
    ~PlanGuard() {
        if (p) esn_plan_destroy(p);
    }
};

struct StreamGuard {
    cudaStream_t s = nullptr;
    ~StreamGuard() {
        if (s) cudaStreamDestroy(s);
    }
};

int nufft_type3_host(int dim, int64_t M, const double *const *xs, const void *c, int isign, double tol, int64_t K,
                     const double *const *ss, void *f, const esn_opts *opts) {
    // argument misuse -> SIZE_ERROR before any core work
    if (M < 0 || K < 0) return fail(ESN_SIZE_ERROR, "negative point or target count");
    if (isign != 1 && isign != -1) return fail(ESN_SIZE_ERROR, "isign must be +1 or -1");
    if ((M > 0 && !c) || (K > 0 && !f)) return fail(ESN_SIZE_ERROR, "null array argument");
    for (int d = 0; d < dim; ++d) {
        if (M > 0 && !xs[d]) return fail(ESN_SIZE_ERROR, "coordinate array %d missing", d + 1);
        if (K > 0 && !ss[d]) return fail(ESN_SIZE_ERROR, "target array %d missing", d + 1);
    }
    esn_opts o;
    if (opts) o = *opts; else esn_default_opts(&o);
    o.dtype = ESN_F64;  // the reference's type 3 is float64
    o.stream = nullptr;
    o.timing = 0;
    esn_kernel_params kp;
    int rc;
    if (o.params) kp = *o.params;
    else if ((rc = esn_select_params(tol, o.sigma, &kp))) return rc;
    if (K == 0) return ESN_SUCCESS;
    // finiteness (transforms.py:282-296)
    const double2 *ch = reinterpret_cast<const double2 *>(c);
    for (int d = 0; d < dim; ++d) {
        for (int64_t j = 0; j < M; ++j)
            if (!std::isfinite(xs[d][j])) return fail(ESN_DATA_ERROR, "non-finite coordinate in dimension %d", d + 1);
        for (int64_t k = 0; k < K; ++k)
            if (!std::isfinite(ss[d][k])) return fail(ESN_DATA_ERROR, "non-finite target in dimension %d", d + 1);
    }
    for (int64_t j = 0; j < M; ++j)
        if (!std::isfinite(ch[j].x) || !std::isfinite(ch[j].y))
            return fail(ESN_DATA_ERROR, "non-finite strength at index %lld", (long long)j);
    // geometry (plan_type3_geometry, transforms.py:245-264)
    double x0[3] = {0, 0, 0}, s0[3] = {0, 0, 0}, gam[3] = {1, 1, 1};
    int64_t n[3] = {1, 1, 1};
    for (int d = 0; d < dim; ++d) {
        double xmn = 0, xmx = 0, smn = 0, smx = 0;
        if (M > 0) {
            xmn = xmx = xs[d][0];
            for (int64_t j = 1; j < M; ++j) { xmn = std::min(xmn, xs[d][j]); xmx = std::max(xmx, xs[d][j]); }
        }
        smn = smx = ss[d][0];
        for (int64_t k = 1; k < K; ++k) { smn = std::min(smn, ss[d][k]); smx = std::max(smx, ss[d][k]); }
        x0[d] = M > 0 ? axis_shift(xmn, xmx) : 0.0;
        s0[d] = axis_shift(smn, smx);
        double xh = 0.0, sh = 0.0;
        for (int64_t j = 0; j < M; ++j) xh = std::max(xh, std::fabs(xs[d][j] - x0[d]));
        for (int64_t k = 0; k < K; ++k) sh = std::max(sh, std::fabs(ss[d][k] - s0[d]));
        const double se = sh > 0.0 ? sh : 1.0;
        const int64_t want = std::max<int64_t>((int64_t)std::ceil((2.0 * o.sigma / M_PI) * xh * se) + kp.w, 2 * kp.w);
        if ((rc = esn_next_smooth(want, &n[d]))) return rc;
        gam[d] = (double)n[d] / (2.0 * o.sigma * se);
    }
    int64_t inner[3] = {1, 1, 1};
    if ((rc = esn_fine_grid_sizes(dim, n, o.sigma, kp.w, inner))) return rc;
    int64_t G = 1, Gi = 1;
    for (int d = 0; d < dim; ++d) { G *= n[d]; Gi *= inner[d]; }
    if (G + Gi > o.max_grid_values)
        return fail(ESN_RESOURCE_ERROR, "type-3 grids need %lld complex values, over the cap of %lld",
                    (long long)(G + Gi), (long long)o.max_grid_values);
    // device buffers
    StreamGuard sg;
    ESN_CUDA_TRY(cudaStreamCreateWithFlags(&sg.s, cudaStreamNonBlocking));
    o.stream = sg.s;
    o.params = &kp;
    DevBuf dx, dc, dcph, dxr, ds, dt, dgrid, db, dout;
    if ((rc = dx.alloc(sizeof(double) * dim * M)) || (rc = dc.alloc(16 * M)) || (rc = dcph.alloc(16 * M)) ||
        (rc = dxr.alloc(sizeof(double) * dim * M)) || (rc = ds.alloc(sizeof(double) * dim * K)) ||
        (rc = dt.alloc(sizeof(double) * dim * K)) || (rc = dgrid.alloc(16 * G)) || (rc = db.alloc(16 * G)) ||
        (rc = dout.alloc(16 * K)))
        return rc;
    double *px[3] = {nullptr, nullptr, nullptr}, *pr[3] = {nullptr, nullptr, nullptr};
    double *ps[3] = {nullptr, nullptr, nullptr}, *pt[3] = {nullptr, nullptr, nullptr};
    for (int d = 0; d < dim; ++d) {
        px[d] = (double *)dx.p + d * M;
        pr[d] = (double *)dxr.p + d * M;
        ps[d] = (double *)ds.p + d * K;
        pt[d] = (double *)dt.p + d * K;
        if (M > 0) ESN_CUDA_TRY(cudaMemcpyAsync(px[d], xs[d], sizeof(double) * M, cudaMemcpyHostToDevice, sg.s));
        ESN_CUDA_TRY(cudaMemcpyAsync(ps[d], ss[d], sizeof(double) * K, cudaMemcpyHostToDevice, sg.s));
    }
    if (M > 0) ESN_CUDA_TRY(cudaMemcpyAsync(dc.p, c, 16 * M, cudaMemcpyHostToDevice, sg.s));
    const int conj = isign < 0;
    if ((rc = esn_type3_prephase(dim, M, px[0], px[1], px[2], x0, s0, gam, conj, dc.p, dcph.p, pr[0], pr[1], pr[2],
                                 sg.s)))
        return rc;
    {
        PlanGuard sp;
        esn_opts os = o;
        os.check_bounds = 0;
        if ((rc = esn_spreader_create(dim, n, 1, &os, &sp.p))) return rc;
        if ((rc = esn_plan_setpts(sp.p, M, ESN_F64, pr[0], pr[1], pr[2]))) return rc;
        if ((rc = esn_plan_spread(sp.p, dcph.p, dgrid.p))) return rc;
        if ((rc = esn_plan_check(sp.p, nullptr))) return rc;
    }
    if ((rc = esn_fftshift(dim, n, dgrid.p, db.p, sg.s))) return rc;
    if ((rc = esn_type3_targets(dim, K, ps[0], ps[1], ps[2], s0, gam, n, pt[0], pt[1], pt[2], sg.s))) return rc;
    {
        PlanGuard p2;
        esn_opts o2 = o;
        o2.check_bounds = 0;
        if ((rc = esn_plan_create(2, dim, n, 1, 1, tol, &o2, &p2.p))) return rc;
        if ((rc = esn_plan_setpts(p2.p, K, ESN_F64, pt[0], pt[1], pt[2]))) return rc;
        if ((rc = esn_plan_execute(p2.p, dout.p, db.p))) return rc;
        if ((rc = esn_plan_check(p2.p, nullptr))) return rc;
    }
    if ((rc = esn_type3_correct(dim, K, ps[0], ps[1], ps[2], x0, s0, gam, n, &kp, conj, dout.p, sg.s))) return rc;
    ESN_CUDA_TRY(cudaMemcpyAsync(f, dout.p, 16 * K, cudaMemcpyDeviceToHost, sg.s));
    ESN_CUDA_TRY(cudaStreamSynchronize(sg.s));
    return ESN_SUCCESS;
}

}  // namespace

extern "C" {

int esn_nufft1d3(int64_t M, const double *x, const void *c, int isign, double tol, int64_t K, const double *s,
                 void *f, const esn_opts *opts) {
    const double *xs[3] = {x, nullptr, nullptr}, *ss[3] = {s, nullptr, nullptr};
    return nufft_type3_host(1, M, xs, c, isign, tol, K, ss, f, opts);
}
int esn_nufft2d3(int64_t M, const double *x, const double *y, const void *c, int isign, double tol, int64_t K,
                 const double *s, const double *t, void *f, const esn_opts *opts) {
    const double *xs[3] = {x, y, nullptr}, *ss[3] = {s, t, nullptr};
    return nufft_type3_host(2, M, xs, c, isign, tol, K, ss, f, opts);
}
int esn_nufft3d3(int64_t M, const double *x, const double *y, const double *z, const void *c, int isign, double tol,
                 int64_t K, const double *s, const double *t, const double *u, void *f, const esn_opts *opts) {
    const double *xs[3] = {x, y, z}, *ss[3] = {s, t, u};
    return nufft_type3_host(3, M, xs, c, isign, tol, K, ss, f, opts);
}

}  // extern "C"
