/*
 * esn_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C + OpenMP) of the reference esnufft hot loops:
 * coordinate fold, 16x4x4 stable bin sort, subproblem spreading with serial
 * periodic add-back, and the interpolation gather.  It is the parity checker
 * for the CUDA path and the timed CPU baseline ("kind": "port") of bench.py.
 * Nothing in paper_1808_06736_b200/ may link, import or call this file;
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm use it.
 *
 * Every routine cites the reference file:line it restates (paths relative to
 * /root/reference/pkg/src/esnufft/).  Arithmetic is written in the same
 * operation order as the reference's numba loops and compiled with
 * -ffp-contract=off so that, for identical inputs, the spread/interp results
 * are bit-identical to the reference (pinned by tests/test_oracle_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TWO_PI (2.0 * M_PI)
#define BOX_FAST 16 /* grid.py:21 */
#define BOX_SLOW 4  /* grid.py:22 */

static int nthreads_or_all(int threads) {
#ifdef _OPENMP
    return threads > 0 ? threads : omp_get_num_procs();
#else
    (void)threads;
    return 1;
#endif
}

/* grid.py:152-168 (fold_coords) + spreadinterp.py:90-101 (build_point_set).
 * np.mod(x, 2pi) == fmod(x, 2pi) (+2pi when the signs differ); an exact 2pi
 * wraps to 0; then g = fold * (n / 2pi), pulled back when g >= n.
 * Returns the first non-finite index (or -1); *first_oob receives the first
 * index with |x| > 3pi (or -1). */
int64_t esno_grid_coords(int64_t m, const double *x, int64_t n, double *g,
                         int64_t *first_oob) {
    const double scale = (double)n / TWO_PI;
    const double limit = 3.0 * M_PI; /* grid.py:29 */
    int64_t bad = -1, oob = -1;
    for (int64_t i = 0; i < m; ++i) {
        double v = x[i];
        if (!isfinite(v)) {
            if (bad < 0) bad = i;
            g[i] = 0.0;
            continue;
        }
        if (oob < 0 && fabs(v) > limit) oob = i;
        double r = fmod(v, TWO_PI);
        if (r != 0.0 && ((r < 0.0) != (TWO_PI < 0.0))) r += TWO_PI;
        if (r == 0.0) r = 0.0; /* numpy returns +0 with the divisor's sign */
        if (r >= TWO_PI) r = 0.0;
        double gg = r * scale;
        if (gg >= (double)n) gg -= (double)n;
        g[i] = gg;
    }
    if (first_oob) *first_oob = oob;
    return bad;
}

/* grid.py:185-199 (_box_indices): flat 16x4x4 box index per point. */
void esno_box_indices(int dim, int64_t m, const double *const *g,
                      const int64_t *n, int64_t *boxes, int64_t *counts) {
    int64_t shape[3] = {BOX_FAST, BOX_SLOW, BOX_SLOW};
    for (int d = 0; d < dim; ++d) counts[d] = (n[d] + shape[d] - 1) / shape[d];
    for (int64_t i = 0; i < m; ++i) {
        int64_t flat = 0, stride = 1;
        for (int d = 0; d < dim; ++d) {
            int64_t b = (int64_t)g[d][i]; /* astype(int64) truncates; g >= 0 */
            b = b / shape[d];
            if (b < 0) b = 0;
            if (b > counts[d] - 1) b = counts[d] - 1;
            flat += b * stride;
            stride *= counts[d];
        }
        boxes[i] = flat;
    }
}

/* grid.py:202-222: stable counting sort of keys in [0, nkeys).  The
 * reference's threaded path (grid.py:224-253) yields the identical
 * permutation, so one stable pass is the whole contract. */
void esno_stable_counting_sort(int64_t m, const int64_t *keys, int64_t nkeys,
                               int64_t *perm) {
    int64_t *start = (int64_t *)calloc((size_t)nkeys + 1, sizeof(int64_t));
    for (int64_t i = 0; i < m; ++i) start[keys[i] + 1]++;
    for (int64_t b = 0; b < nkeys; ++b) start[b + 1] += start[b];
    for (int64_t i = 0; i < m; ++i) perm[start[keys[i]]++] = i;
    free(start);
}

/* grid.py:202-254 (bin_sort) for the reference 16x4x4 boxes. */
void esno_bin_sort(int dim, int64_t m, const double *const *g, const int64_t *n,
                   int64_t *perm, int64_t *boxes) {
    int64_t counts[3] = {1, 1, 1};
    esno_box_indices(dim, m, g, n, boxes, counts);
    int64_t nk = 1;
    for (int d = 0; d < dim; ++d) nk *= counts[d];
    esno_stable_counting_sort(m, boxes, nk, perm);
}

/* spreadinterp.py:117-120 (_base_indices): footprint origin per point. */
void esno_base_indices(int64_t m, const double *g, int w, int64_t *base) {
    for (int64_t i = 0; i < m; ++i) base[i] = (int64_t)floor(g[i] - 0.5 * w + 1.0);
}

/* spreadinterp.py:313-336 (_row). */
static inline int64_t kernel_row(double g, int w, const double *coeffs,
                                 double beta, int use_exact, double *row) {
    int64_t i0 = (int64_t)floor(g - 0.5 * w + 1.0);
    if (use_exact) {
        double step = 2.0 / w;
        double z = step * ((double)i0 - g);
        for (int m = 0; m < w; ++m) {
            double a = 1.0 - z * z;
            if (a < 0.0) a = 0.0;
            row[m] = exp(beta * (sqrt(a) - 1.0));
            z += step;
        }
    } else {
        double t = 2.0 * ((double)i0 - g) + ((double)w - 1.0);
        int deg1 = w + 4;
        for (int m = 0; m < w; ++m) {
            const double *cm = coeffs + (size_t)m * deg1;
            double v = cm[0];
            for (int q = 1; q < deg1; ++q) v = v * t + cm[q];
            row[m] = v;
        }
    }
    return i0;
}

typedef struct {
    int64_t start, stop, lo[3], ext[3];
} subprob_t;

/* spreadinterp.py:123-150 (partition_subproblems). */
static int64_t partition(int dim, int64_t m, const double *const *g,
                         const int64_t *perm, int w, int64_t cap,
                         subprob_t **out) {
    int64_t ns = (m + cap - 1) / cap;
    subprob_t *s = (subprob_t *)calloc((size_t)(ns > 0 ? ns : 1), sizeof(subprob_t));
    for (int64_t k = 0; k < ns; ++k) {
        s[k].start = k * cap;
        s[k].stop = (k + 1) * cap < m ? (k + 1) * cap : m;
        for (int d = 0; d < 3; ++d) { s[k].lo[d] = 0; s[k].ext[d] = 1; }
        for (int d = 0; d < dim; ++d) {
            int64_t lo = INT64_MAX, hi = INT64_MIN;
            for (int64_t q = s[k].start; q < s[k].stop; ++q) {
                int64_t b = (int64_t)floor(g[d][perm[q]] - 0.5 * w + 1.0);
                if (b < lo) lo = b;
                if (b > hi) hi = b;
            }
            s[k].lo[d] = lo;
            s[k].ext[d] = hi - lo + w;
        }
    }
    *out = s;
    return ns;
}

/* spreadinterp.py:339-392 (_spread_sub_{1,2,3}d) into a private cuboid. */
static void spread_sub(int dim, const double *const *g, const double *c,
                       const int64_t *perm, const subprob_t *sp, int w,
                       const double *coeffs, double beta, int use_exact,
                       double *loc) {
    double r1[16], r2[16], r3[16];
    for (int64_t s = sp->start; s < sp->stop; ++s) {
        int64_t j = perm[s];
        double cre = c[2 * j], cim = c[2 * j + 1];
        if (dim == 1) {
            int64_t b = kernel_row(g[0][j], w, coeffs, beta, use_exact, r1) - sp->lo[0];
            for (int m = 0; m < w; ++m) {
                loc[2 * (b + m)] += cre * r1[m];
                loc[2 * (b + m) + 1] += cim * r1[m];
            }
        } else if (dim == 2) {
            int64_t b1 = kernel_row(g[0][j], w, coeffs, beta, use_exact, r1) - sp->lo[0];
            int64_t b2 = kernel_row(g[1][j], w, coeffs, beta, use_exact, r2) - sp->lo[1];
            int64_t s1 = sp->ext[0];
            for (int m2 = 0; m2 < w; ++m2) {
                double are = cre * r2[m2], aim = cim * r2[m2];
                int64_t base = (b2 + m2) * s1 + b1;
                for (int m1 = 0; m1 < w; ++m1) {
                    loc[2 * (base + m1)] += are * r1[m1];
                    loc[2 * (base + m1) + 1] += aim * r1[m1];
                }
            }
        } else {
            int64_t b1 = kernel_row(g[0][j], w, coeffs, beta, use_exact, r1) - sp->lo[0];
            int64_t b2 = kernel_row(g[1][j], w, coeffs, beta, use_exact, r2) - sp->lo[1];
            int64_t b3 = kernel_row(g[2][j], w, coeffs, beta, use_exact, r3) - sp->lo[2];
            int64_t s1 = sp->ext[0], s2 = sp->ext[1];
            for (int m3 = 0; m3 < w; ++m3) {
                double a3re = cre * r3[m3], a3im = cim * r3[m3];
                int64_t plane = (b3 + m3) * s2;
                for (int m2 = 0; m2 < w; ++m2) {
                    double are = a3re * r2[m2], aim = a3im * r2[m2];
                    int64_t base = (plane + b2 + m2) * s1 + b1;
                    for (int m1 = 0; m1 < w; ++m1) {
                        loc[2 * (base + m1)] += are * r1[m1];
                        loc[2 * (base + m1) + 1] += aim * r1[m1];
                    }
                }
            }
        }
    }
}

static inline int64_t pmod(int64_t a, int64_t n) {
    int64_t r = a % n;
    return r < 0 ? r + n : r;
}

/* spreadinterp.py:395-428 (_add_back_{1,2,3}d), serial and in order. */
static void add_back(int dim, const subprob_t *sp, const double *loc,
                     const int64_t *n, double *grid) {
    int64_t s1 = sp->ext[0], s2 = dim > 1 ? sp->ext[1] : 1, s3 = dim > 2 ? sp->ext[2] : 1;
    int64_t n1 = n[0], n2 = dim > 1 ? n[1] : 1;
    for (int64_t q3 = 0; q3 < s3; ++q3) {
        int64_t gp = dim > 2 ? pmod(sp->lo[2] + q3, n[2]) * n2 * n1 : 0;
        for (int64_t q2 = 0; q2 < s2; ++q2) {
            int64_t gb = gp + (dim > 1 ? pmod(sp->lo[1] + q2, n[1]) * n1 : 0);
            int64_t lb = (q3 * s2 + q2) * s1;
            for (int64_t q1 = 0; q1 < s1; ++q1) {
                int64_t gi = gb + pmod(sp->lo[0] + q1, n1);
                grid[2 * gi] += loc[2 * (lb + q1)];
                grid[2 * gi + 1] += loc[2 * (lb + q1) + 1];
            }
        }
    }
}

/* spreadinterp.py:187-256 (spread).  grid (interleaved complex, C order
 * (n_d..n_1)) is zeroed here.  Returns 0. */
int esno_spread(int dim, int64_t m, const double *const *g, const int64_t *perm,
                const double *c, const int64_t *n, int w, const double *coeffs,
                double beta, int use_exact, int64_t cap, int threads,
                double *grid) {
    int64_t total = 1;
    for (int d = 0; d < dim; ++d) total *= n[d];
    memset(grid, 0, (size_t)total * 2 * sizeof(double));
    if (m == 0) return 0;
    subprob_t *subs = NULL;
    int64_t ns = partition(dim, m, g, perm, w, cap, &subs);
    double **locs = (double **)calloc((size_t)ns, sizeof(double *));
    int nt = nthreads_or_all(threads);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
    for (int64_t k = 0; k < ns; ++k) {
        int64_t vol = subs[k].ext[0] * subs[k].ext[1] * subs[k].ext[2];
        locs[k] = (double *)calloc((size_t)vol * 2, sizeof(double));
        spread_sub(dim, g, c, perm, &subs[k], w, coeffs, beta, use_exact, locs[k]);
    }
    for (int64_t k = 0; k < ns; ++k) {
        add_back(dim, &subs[k], locs[k], n, grid);
        free(locs[k]);
    }
    free(locs);
    free(subs);
    return 0;
}

/* spreadinterp.py:259-306 + 431-507 (interp, _interp_block_*): output in
 * original point order. */
int esno_interp(int dim, int64_t m, const double *const *g, const int64_t *perm,
                const double *grid, const int64_t *n, int w,
                const double *coeffs, double beta, int use_exact, int64_t cap,
                int threads, double *out) {
    if (m == 0) return 0;
    int64_t nblocks = (m + cap - 1) / cap;
    if (nblocks < 1) nblocks = 1;
    int nt = nthreads_or_all(threads);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
    for (int64_t blk = 0; blk < nblocks; ++blk) {
        /* np.linspace(0, m, nblocks + 1, dtype=int64) edges */
        int64_t s0 = (int64_t)((double)m * (double)blk / (double)nblocks);
        int64_t s1e = (int64_t)((double)m * (double)(blk + 1) / (double)nblocks);
        if (blk == nblocks - 1) s1e = m;
        double r1[16], r2[16], r3[16];
        int64_t ix1[16], ix2[16], ix3[16];
        for (int64_t s = s0; s < s1e; ++s) {
            int64_t j = perm[s];
            double are = 0.0, aim = 0.0;
            int64_t i1 = kernel_row(g[0][j], w, coeffs, beta, use_exact, r1);
            for (int q = 0; q < w; ++q) {
                int64_t i = i1 + q;
                ix1[q] = i < 0 ? i + n[0] : (i >= n[0] ? i - n[0] : i);
            }
            if (dim == 1) {
                for (int q = 0; q < w; ++q) {
                    are += r1[q] * grid[2 * ix1[q]];
                    aim += r1[q] * grid[2 * ix1[q] + 1];
                }
            } else {
                int64_t i2 = kernel_row(g[1][j], w, coeffs, beta, use_exact, r2);
                for (int q = 0; q < w; ++q) {
                    int64_t i = i2 + q;
                    ix2[q] = i < 0 ? i + n[1] : (i >= n[1] ? i - n[1] : i);
                }
                if (dim == 2) {
                    for (int q2 = 0; q2 < w; ++q2) {
                        int64_t base = ix2[q2] * n[0];
                        double pre = 0.0, pim = 0.0;
                        for (int q1 = 0; q1 < w; ++q1) {
                            pre += r1[q1] * grid[2 * (base + ix1[q1])];
                            pim += r1[q1] * grid[2 * (base + ix1[q1]) + 1];
                        }
                        are += r2[q2] * pre;
                        aim += r2[q2] * pim;
                    }
                } else {
                    int64_t i3 = kernel_row(g[2][j], w, coeffs, beta, use_exact, r3);
                    for (int q = 0; q < w; ++q) {
                        int64_t i = i3 + q;
                        ix3[q] = i < 0 ? i + n[2] : (i >= n[2] ? i - n[2] : i);
                    }
                    for (int q3 = 0; q3 < w; ++q3) {
                        int64_t plane = ix3[q3] * n[1] * n[0];
                        double p3re = 0.0, p3im = 0.0;
                        for (int q2 = 0; q2 < w; ++q2) {
                            int64_t base = plane + ix2[q2] * n[0];
                            double p2re = 0.0, p2im = 0.0;
                            for (int q1 = 0; q1 < w; ++q1) {
                                p2re += r1[q1] * grid[2 * (base + ix1[q1])];
                                p2im += r1[q1] * grid[2 * (base + ix1[q1]) + 1];
                            }
                            p3re += r2[q2] * p2re;
                            p3im += r2[q2] * p2im;
                        }
                        are += r3[q3] * p3re;
                        aim += r3[q3] * p3im;
                    }
                }
            }
            out[2 * j] = are;
            out[2 * j + 1] = aim;
        }
    }
    return 0;
}

/* oracle.py:52-88 (_sum1/_sum2/_sum3): O(M N) direct sums, ascending j. */
int esno_direct(int dim, int64_t m, const double *const *x, const double *c,
                int64_t nk, const double *const *s, double isign, int threads,
                double *out) {
    int nt = nthreads_or_all(threads);
#pragma omp parallel for schedule(static) num_threads(nt)
    for (int64_t a = 0; a < nk; ++a) {
        double are = 0.0, aim = 0.0;
        for (int64_t j = 0; j < m; ++j) {
            double ph = s[0][a] * x[0][j];
            if (dim > 1) ph = ph + s[1][a] * x[1][j];
            if (dim > 2) ph = ph + s[2][a] * x[2][j];
            ph = isign * ph;
            double co = cos(ph), si = sin(ph);
            are += c[2 * j] * co - c[2 * j + 1] * si;
            aim += c[2 * j] * si + c[2 * j + 1] * co;
        }
        out[2 * a] = are;
        out[2 * a + 1] = aim;
    }
    return 0;
}

int esno_num_procs(void) { return nthreads_or_all(0); }
