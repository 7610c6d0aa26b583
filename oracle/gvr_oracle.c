/* Plain-C FP64 restatement of the reference render path (TEST INFRASTRUCTURE ONLY).
 * See gvr_oracle.h for the contract and how parity of this port is pinned.
 *
 * Every function follows the reference line by line (same formulas, same
 * evaluation order, same tie-breaks); citations are into /root/reference/proj.
 */
#define _GNU_SOURCE
#include "gvr_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static __thread char g_err[256];

const char* gvro_last_error(void) { return g_err; }

static int fail(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return 1;
}

#define BEHIND_CAMERA_EPS 1e-4 /* include/gvr/tracer.hpp:28 */

/* ------------------------------------------------------------------ 3x3 helpers */

/* y = M x, sums in column order like Eigen's (shim) product. */
static void mat_vec(const double* m, const double* x, double* y) {
    for (int i = 0; i < 3; ++i) {
        double acc = 0.0;
        for (int k = 0; k < 3; ++k) acc += m[3 * i + k] * x[k];
        y[i] = acc;
    }
}

static void mat_mul(const double* a, const double* b, double* c) {
    double t[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double acc = 0.0;
            for (int k = 0; k < 3; ++k) acc += a[3 * i + k] * b[3 * k + j];
            t[3 * i + j] = acc;
        }
    memcpy(c, t, sizeof t);
}

static void transpose3(const double* a, double* t) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) t[3 * j + i] = a[3 * i + j];
}

static double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

static double det3(const double* m) {
    return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
           m[2] * (m[3] * m[7] - m[4] * m[6]);
}

/* 3x3 inverse by cofactors (Eigen 3x3 path). */
static void inverse3(const double* m, double* inv) {
#define M(i, j) m[3 * (i) + (j)]
    const double c00 = M(1, 1) * M(2, 2) - M(1, 2) * M(2, 1);
    const double c10 = M(1, 2) * M(2, 0) - M(1, 0) * M(2, 2);
    const double c20 = M(1, 0) * M(2, 1) - M(1, 1) * M(2, 0);
    const double det = M(0, 0) * c00 + M(0, 1) * c10 + M(0, 2) * c20;
    const double id = 1.0 / det;
    inv[0] = c00 * id;
    inv[3] = c10 * id;
    inv[6] = c20 * id;
    inv[1] = (M(0, 2) * M(2, 1) - M(0, 1) * M(2, 2)) * id;
    inv[4] = (M(0, 0) * M(2, 2) - M(0, 2) * M(2, 0)) * id;
    inv[7] = (M(0, 1) * M(2, 0) - M(0, 0) * M(2, 1)) * id;
    inv[2] = (M(0, 1) * M(1, 2) - M(0, 2) * M(1, 1)) * id;
    inv[5] = (M(0, 2) * M(1, 0) - M(0, 0) * M(1, 2)) * id;
    inv[8] = (M(0, 0) * M(1, 1) - M(0, 1) * M(1, 0)) * id;
#undef M
}

/* Smallest eigenvalue of the symmetric matrix read from the lower triangle
 * (Eigen's SelfAdjointEigenSolver reads the lower triangle), cyclic Jacobi. */
static double min_eigenvalue_lower(const double* m) {
    double a[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) a[3 * i + j] = i >= j ? m[3 * i + j] : m[3 * j + i];
    for (int sweep = 0; sweep < 100; ++sweep) {
        const double off = a[1] * a[1] + a[2] * a[2] + a[5] * a[5];
        if (off <= 2.2250738585072014e-308) break;
        for (int p = 0; p < 3; ++p)
            for (int q = p + 1; q < 3; ++q) {
                const double apq = a[3 * p + q];
                if (apq == 0.0) continue;
                const double theta = (a[3 * q + q] - a[3 * p + p]) / (2 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1));
                const double c = 1 / sqrt(t * t + 1), s = t * c;
                for (int k = 0; k < 3; ++k) {
                    const double akp = a[3 * k + p], akq = a[3 * k + q];
                    a[3 * k + p] = c * akp - s * akq;
                    a[3 * k + q] = s * akp + c * akq;
                }
                for (int k = 0; k < 3; ++k) {
                    const double apk = a[3 * p + k], aqk = a[3 * q + k];
                    a[3 * p + k] = c * apk - s * aqk;
                    a[3 * q + k] = s * apk + c * aqk;
                }
            }
    }
    double mn = a[0];
    if (a[4] < mn) mn = a[4];
    if (a[8] < mn) mn = a[8];
    return mn;
}

static int all_finite(const double* v, long n) {
    for (long i = 0; i < n; ++i)
        if (!isfinite(v[i])) return 0;
    return 1;
}

/* ------------------------------------------------------------------ validation */

/* GaussianScene::validate / GaussianKernel::validate (src/types.cpp:17-42). */
static int validate_scene(int K, int D, double tau, const double* centers, const double* inv_cov,
                          const double* attr) {
    if (tau < 0.0 || !isfinite(tau)) return fail("tau must be finite and >= 0");
    for (int k = 0; k < K; ++k) {
        const double* s = inv_cov + 9 * (long)k;
        if (!all_finite(centers + 3 * (long)k, 3) || !all_finite(s, 9) ||
            !all_finite(attr + (long)D * k, D)) {
            snprintf(g_err, sizeof g_err, "kernel has non-finite values (kernel %d)", k);
            return 1;
        }
        double scale = 0.0, asym = 0.0;
        for (int i = 0; i < 9; ++i)
            if (fabs(s[i]) > scale) scale = fabs(s[i]);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                const double d = fabs(s[3 * i + j] - s[3 * j + i]);
                if (d > asym) asym = d;
            }
        if (scale != 0.0 && !(asym <= 1e-6 * scale)) {
            snprintf(g_err, sizeof g_err, "inv_cov is not symmetric (kernel %d)", k);
            return 1;
        }
        if (min_eigenvalue_lower(s) <= 0.0) {
            snprintf(g_err, sizeof g_err, "inv_cov is not positive-definite (kernel %d)", k);
            return 1;
        }
    }
    return 0;
}

/* Camera::validate (src/types.cpp:44-63). */
static int validate_camera(const gvro_camera* c) {
    if (!all_finite(c->rotation, 9) || !all_finite(c->translation, 3))
        return fail("camera extrinsics have non-finite values");
    double rt[9], rtr[9];
    transpose3(c->rotation, rt);
    mat_mul(rt, c->rotation, rtr);
    double worst = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            const double d = fabs(rtr[3 * i + j] - (i == j ? 1.0 : 0.0));
            if (d > worst) worst = d;
        }
    if (worst > 1e-6) return fail("camera rotation is not orthonormal");
    if (fabs(det3(c->rotation) - 1.0) > 1e-6) return fail("camera rotation determinant is not +1");
    if (!(c->focal > 0.0) || !isfinite(c->focal)) return fail("camera focal length must be > 0");
    if (c->height < 1 || c->width < 1) return fail("camera image size must be at least 1x1");
    if (!isfinite(c->ox) || !isfinite(c->oy)) return fail("camera principal point has non-finite values");
    return 0;
}

/* SelectionConfig::validate (src/tracer.cpp:8-18). */
static int validate_cfg(const gvro_selection* s) {
    if (!(s->eta > 0.0 && s->eta < 1.0)) return fail("selection eta must be in (0, 1)");
    if (s->k_prime < 1) return fail("selection k_prime must be >= 1");
    if (s->coarse_downsample < 1) return fail("coarse downsample must be >= 1");
    return 0;
}

/* ------------------------------------------------------------------ geometry */

/* view_transform (src/scene.cpp:5-17): M' = R M + T, S' = R S R^T. */
static void view_transform(int K, const double* centers, const double* inv_cov, const gvro_camera* c,
                           double* cam_centers, double* cam_inv_cov) {
    double rt[9];
    transpose3(c->rotation, rt);
    for (int k = 0; k < K; ++k) {
        double m[3];
        mat_vec(c->rotation, centers + 3 * (long)k, m);
        for (int i = 0; i < 3; ++i) cam_centers[3 * (long)k + i] = m[i] + c->translation[i];
        double rs[9];
        mat_mul(c->rotation, inv_cov + 9 * (long)k, rs);
        mat_mul(rs, rt, cam_inv_cov + 9 * (long)k);
    }
}

/* pixel_ray (src/scene.cpp:19-22). */
static void pixel_ray(const gvro_camera* c, int row, int col, double* d) {
    d[0] = (row - c->oy) / c->focal;
    d[1] = (col - c->ox) / c->focal;
    d[2] = 1.0;
    const double n = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
    if (n > 0.0) {
        const double s = sqrt(n);
        d[0] /= s;
        d[1] /= s;
        d[2] /= s;
    }
}

typedef struct {
    int idx;
    double l, q, sigma;
} traced_t;

/* trace_kernel (src/tracer.cpp:20-35). */
static traced_t trace_kernel(const double* d, const double* m, const double* s, int idx) {
    double sd[3], sm[3], v[3], sv[3];
    mat_vec(s, d, sd);
    const double a = dot3(d, sd);
    mat_vec(s, m, sm);
    const double b = 0.5 * (dot3(m, sd) + dot3(d, sm));
    const double l = b / a;
    for (int i = 0; i < 3; ++i) v[i] = m[i] - l * d[i];
    mat_vec(s, v, sv);
    double q = -0.5 * dot3(v, sv);
    if (q > 0.0) q = 0.0; /* std::min(0.0, .) */
    traced_t t = {idx, l, q, 1.0 / sqrt(a)};
    return t;
}

/* ------------------------------------------------------------------ coarse select */

typedef struct {
    int grid_rows, grid_cols, ds;
    int* cell_start; /* CSR over cells, kernels ascending within a cell */
    int* cell_items;
    int dropped_behind;
} coarse_map_t;

/* coarse_select (src/tracer.cpp:37-113): per kernel in front, the pixel box of
 * the eta-level set (linearised projection widened by the projected camera-space
 * box, or full screen when that box straddles the near plane), pushed into every
 * ds x ds cell it overlaps. Produces per-kernel cell boxes (-1 when not pushed). */
static void coarse_boxes(int K, const double* cc, const double* cs, const gvro_camera* cam,
                         const gvro_selection* cfg, int* box, int* dropped) {
    const int ds = cfg->coarse_downsample;
    const double chi = 2.0 * log(1.0 / cfg->eta);
    const double f = cam->focal;
    *dropped = 0;
    for (int k = 0; k < K; ++k) {
        int* b = box + 4 * (long)k;
        b[0] = b[1] = b[2] = b[3] = -1;
        const double* m = cc + 3 * (long)k;
        const double z = m[2];
        if (z <= BEHIND_CAMERA_EPS) {
            ++*dropped;
            continue;
        }
        double cov[9];
        inverse3(cs + 9 * (long)k, cov);
        const double ci = cam->oy + f * m[0] / z;
        const double cj = cam->ox + f * m[1] / z;
        /* jac = [[f/z, 0, -f x/z^2], [0, f/z, -f y/z^2]]; cov2 = jac cov jac^T */
        const double jac[6] = {f / z, 0.0, -f * m[0] / (z * z), 0.0, f / z, -f * m[1] / (z * z)};
        double jc[6];
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 3; ++j) {
                double acc = 0.0;
                for (int t = 0; t < 3; ++t) acc += jac[3 * i + t] * cov[3 * t + j];
                jc[3 * i + j] = acc;
            }
        double cov2[4];
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) {
                double acc = 0.0;
                for (int t = 0; t < 3; ++t) acc += jc[3 * i + t] * jac[3 * j + t];
                cov2[2 * i + j] = acc;
            }
        const double rh = sqrt(fmax(0.0, chi * cov2[0]));
        const double rw = sqrt(fmax(0.0, chi * cov2[3]));
        double top = ci - rh, bottom = ci + rh, left = cj - rw, right = cj + rw;
        const double ext[3] = {sqrt(fmax(0.0, chi * cov[0])), sqrt(fmax(0.0, chi * cov[4])),
                               sqrt(fmax(0.0, chi * cov[8]))};
        if (m[2] - ext[2] <= BEHIND_CAMERA_EPS) {
            top = 0;
            bottom = cam->height - 1;
            left = 0;
            right = cam->width - 1;
        } else {
            for (int corner = 0; corner < 8; ++corner) {
                const double p[3] = {m[0] + ((corner & 1) ? ext[0] : -ext[0]),
                                     m[1] + ((corner & 2) ? ext[1] : -ext[1]),
                                     m[2] + ((corner & 4) ? ext[2] : -ext[2])};
                const double pi = cam->oy + f * p[0] / p[2];
                const double pj = cam->ox + f * p[1] / p[2];
                if (pi < top) top = pi;
                if (pi > bottom) bottom = pi;
                if (pj < left) left = pj;
                if (pj > right) right = pj;
            }
        }
        int row_lo = (int)floor(top - 1.0);
        if (row_lo < 0) row_lo = 0;
        int row_hi = (int)ceil(bottom + 1.0);
        if (row_hi > cam->height - 1) row_hi = cam->height - 1;
        int col_lo = (int)floor(left - 1.0);
        if (col_lo < 0) col_lo = 0;
        int col_hi = (int)ceil(right + 1.0);
        if (col_hi > cam->width - 1) col_hi = cam->width - 1;
        if (row_lo > row_hi || col_lo > col_hi) continue;
        b[0] = row_lo / ds;
        b[1] = row_hi / ds;
        b[2] = col_lo / ds;
        b[3] = col_hi / ds;
    }
}

static void coarse_select(int K, const double* cc, const double* cs, const gvro_camera* cam,
                          const gvro_selection* cfg, coarse_map_t* map) {
    const int ds = cfg->coarse_downsample;
    map->ds = ds;
    map->grid_rows = (cam->height + ds - 1) / ds;
    map->grid_cols = (cam->width + ds - 1) / ds;
    const long cells = (long)map->grid_rows * map->grid_cols;
    int* box = malloc(sizeof(int) * 4 * (size_t)(K > 0 ? K : 1));
    coarse_boxes(K, cc, cs, cam, cfg, box, &map->dropped_behind);
    map->cell_start = calloc((size_t)cells + 1, sizeof(int));
    for (int k = 0; k < K; ++k) {
        const int* b = box + 4 * (long)k;
        if (b[0] < 0) continue;
        for (int cr = b[0]; cr <= b[1]; ++cr)
            for (int c = b[2]; c <= b[3]; ++c) ++map->cell_start[(long)cr * map->grid_cols + c + 1];
    }
    for (long c = 0; c < cells; ++c) map->cell_start[c + 1] += map->cell_start[c];
    map->cell_items = malloc(sizeof(int) * (size_t)(map->cell_start[cells] > 0 ? map->cell_start[cells] : 1));
    int* fill = malloc(sizeof(int) * (size_t)cells);
    memcpy(fill, map->cell_start, sizeof(int) * (size_t)cells);
    for (int k = 0; k < K; ++k) { /* ascending k -> cells hold push_back order */
        const int* b = box + 4 * (long)k;
        if (b[0] < 0) continue;
        for (int cr = b[0]; cr <= b[1]; ++cr)
            for (int c = b[2]; c <= b[3]; ++c) map->cell_items[fill[(long)cr * map->grid_cols + c]++] = k;
    }
    free(fill);
    free(box);
}

/* ------------------------------------------------------------------ selection + blend */

static int traced_less(const traced_t* a, const traced_t* b) {
    if (a->l != b->l) return a->l < b->l;
    return a->idx < b->idx;
}

static int traced_cmp(const void* x, const void* y) {
    const traced_t* a = x;
    const traced_t* b = y;
    if (traced_less(a, b)) return -1;
    if (traced_less(b, a)) return 1;
    return 0;
}

/* normal_cdf (src/blender.cpp:13-15) */
static double normal_cdf(double x) { return 0.5 * erfc(-x * 0.7071067811865476); }
static double normal_pdf(double x) { return 0.3989422804014327 * exp(-0.5 * x * x); }

typedef struct {
    /* inputs */
    int K, D, Dc, H, W, kp;
    double tau;
    const double *attr, *cc, *cs;
    const gvro_camera* cam;
    const gvro_selection* cfg;
    const coarse_map_t* map;
    const int* all_front;
    int n_front;
    /* outputs */
    double *image, *alpha, *depth;
    traced_t* tape; /* [P*kp] */
    int* count;     /* [P] */
    double* weights; /* [P*kp] */
} render_job_t;

typedef struct {
    render_job_t* job;
    int row_begin, row_end;
} render_part_t;

static void* render_rows(void* arg) {
    render_part_t* part = arg;
    render_job_t* j = part->job;
    const double log_eta = log(j->cfg->eta);
    size_t cap = 64;
    traced_t* traced = malloc(sizeof(traced_t) * cap);
    double* peak = malloc(sizeof(double) * (size_t)j->kp);
    for (int i = part->row_begin; i < part->row_end; ++i) {
        for (int col = 0; col < j->W; ++col) {
            double d[3];
            pixel_ray(j->cam, i, col, d);
            const int* cand;
            int nc;
            if (j->cfg->coarse_enabled) {
                const long cell = (long)(i / j->map->ds) * j->map->grid_cols + col / j->map->ds;
                cand = j->map->cell_items + j->map->cell_start[cell];
                nc = j->map->cell_start[cell + 1] - j->map->cell_start[cell];
            } else {
                cand = j->all_front;
                nc = j->n_front;
            }
            /* trace every candidate (src/blender.cpp:107-110) */
            if ((size_t)nc > cap) {
                cap = (size_t)nc;
                traced = realloc(traced, sizeof(traced_t) * cap);
            }
            int n = 0;
            for (int t = 0; t < nc; ++t) {
                const int k = cand[t];
                if (j->cfg->coarse_enabled && j->cc[3 * (long)k + 2] <= BEHIND_CAMERA_EPS) continue;
                const traced_t tk = trace_kernel(d, j->cc + 3 * (long)k, j->cs + 9 * (long)k, k);
                /* fine_select (src/tracer.cpp:115-127): drop !(q > ln eta) */
                if (tk.q > log_eta) traced[n++] = tk;
            }
            qsort(traced, (size_t)n, sizeof(traced_t), traced_cmp);
            if (n > j->kp) n = j->kp;
            /* blend (src/blender.cpp:27-53) */
            double total_peak = 0.0;
            for (int k = 0; k < n; ++k) {
                peak[k] = exp(traced[k].q);
                total_peak += peak[k];
            }
            const size_t p = (size_t)i * j->W + col;
            double wsum = 0.0, wl = 0.0;
            for (int k = 0; k < n; ++k) {
                double acc = 0.0;
                for (int m = 0; m < n; ++m)
                    acc += peak[m] * normal_cdf((traced[k].l - traced[m].l) / traced[m].sigma);
                const double w = exp(-j->tau * acc) * peak[k];
                /* image += W attr, depth (src/blender.cpp:114-124) */
                for (int c = 0; c < j->D; ++c)
                    j->image[p * j->Dc + c] += w * j->attr[(size_t)j->D * traced[k].idx + c];
                wsum += w;
                wl += w * traced[k].l;
                j->weights[p * j->kp + k] = w;
                j->tape[p * j->kp + k] = traced[k];
            }
            j->alpha[p] = 1.0 - exp(-j->tau * total_peak);
            j->depth[p] = wsum > 1e-12 ? wl / wsum : 0.0;
            j->count[p] = n;
        }
    }
    free(peak);
    free(traced);
    return NULL;
}

/* resolve_threads (include/gvr/parallel.hpp:12-20) */
static int resolve_threads(int requested) {
    const char* env = getenv("GVR_THREADS");
    if (env) {
        const int n = atoi(env);
        if (n > 0) return n;
    }
    if (requested > 0) return requested;
    const long hw = sysconf(_SC_NPROCESSORS_ONLN);
    return hw > 0 ? (int)hw : 1;
}

/* parallel_for_partitions (include/gvr/parallel.hpp:25-43): contiguous row blocks. */
static void run_partitions(int count, int workers, void* (*fn)(void*), void* parts, size_t part_size,
                           void (*init)(void* part, int worker, int begin, int end, void* ctx), void* ctx) {
    if (workers > count) workers = count;
    if (workers < 1) workers = 1;
    if (count <= 0) return;
    pthread_t* th = malloc(sizeof(pthread_t) * (size_t)workers);
    const int base = count / workers, extra = count % workers;
    int begin = 0;
    for (int w = 0; w < workers; ++w) {
        const int len = base + (w < extra ? 1 : 0);
        void* part = (char*)parts + part_size * (size_t)w;
        init(part, w, begin, begin + len, ctx);
        begin += len;
        if (workers == 1)
            fn(part);
        else
            pthread_create(&th[w], NULL, fn, part);
    }
    if (workers > 1)
        for (int w = 0; w < workers; ++w) pthread_join(th[w], NULL);
    free(th);
}

static void init_render_part(void* part, int w, int b, int e, void* ctx) {
    (void)w;
    render_part_t* p = part;
    p->job = ctx;
    p->row_begin = b;
    p->row_end = e;
}

typedef struct {
    int H, W, kp, D, K;
    double* cc;
    double* cs;
    traced_t* tape;
    int* count;
    double* weights;
} forward_state_t;

static void free_state(forward_state_t* s) {
    free(s->cc);
    free(s->cs);
    free(s->tape);
    free(s->count);
    free(s->weights);
}

/* detail::render_core (src/blender.cpp:66-137). */
static int render_core(int K, int D, double tau, const double* centers, const double* inv_cov,
                       const double* attr, const gvro_camera* cam, const gvro_selection* cfg, int threads,
                       double* image, double* alpha, double* depth, forward_state_t* st) {
    memset(st, 0, sizeof *st);
    if (validate_scene(K, D, tau, centers, inv_cov, attr)) return 1;
    if (validate_camera(cam)) return 1;
    if (validate_cfg(cfg)) return 1;
    const int H = cam->height, W = cam->width, Dc = D > 1 ? D : 1;
    const size_t P = (size_t)H * W;
    st->H = H;
    st->W = W;
    st->kp = cfg->k_prime;
    st->D = D;
    st->K = K;
    st->cc = malloc(sizeof(double) * 3 * (size_t)(K > 0 ? K : 1));
    st->cs = malloc(sizeof(double) * 9 * (size_t)(K > 0 ? K : 1));
    view_transform(K, centers, inv_cov, cam, st->cc, st->cs);

    coarse_map_t map;
    memset(&map, 0, sizeof map);
    int* all_front = NULL;
    int n_front = 0;
    if (cfg->coarse_enabled) {
        coarse_select(K, st->cc, st->cs, cam, cfg, &map);
    } else {
        all_front = malloc(sizeof(int) * (size_t)(K > 0 ? K : 1));
        for (int k = 0; k < K; ++k)
            if (st->cc[3 * (long)k + 2] > BEHIND_CAMERA_EPS) all_front[n_front++] = k;
    }
    memset(image, 0, sizeof(double) * P * Dc);
    st->tape = calloc(P * (size_t)cfg->k_prime, sizeof(traced_t));
    st->count = calloc(P, sizeof(int));
    st->weights = calloc(P * (size_t)cfg->k_prime, sizeof(double));

    render_job_t job = {K, D, Dc, H, W, cfg->k_prime, tau, attr, st->cc, st->cs, cam, cfg, &map,
                        all_front, n_front, image, alpha, depth, st->tape, st->count, st->weights};
    const int workers = resolve_threads(threads);
    render_part_t* parts = calloc((size_t)(workers > 0 ? workers : 1), sizeof(render_part_t));
    run_partitions(H, workers, render_rows, parts, sizeof(render_part_t), init_render_part, &job);
    free(parts);
    free(all_front);
    free(map.cell_start);
    free(map.cell_items);

    /* validate_finite (src/blender.cpp:132-134) */
    if (!all_finite(image, (long)(P * Dc)) || !all_finite(alpha, (long)P) || !all_finite(depth, (long)P)) {
        free_state(st);
        return fail("image contains non-finite values");
    }
    return 0;
}

int gvro_render(int K, int D, double tau, const double* centers, const double* inv_cov,
                const double* attr, const gvro_camera* cam, const gvro_selection* cfg, int threads,
                double* image, double* alpha, double* depth, int* topk_idx, double* topk_w,
                double* topk_l, double* topk_q, double* topk_sigma) {
    forward_state_t st;
    const int rc = render_core(K, D, tau, centers, inv_cov, attr, cam, cfg, threads, image, alpha, depth, &st);
    if (rc) return rc;
    const size_t P = (size_t)st.H * st.W;
    for (size_t p = 0; p < P; ++p)
        for (int s = 0; s < st.kp; ++s) {
            const size_t o = p * st.kp + s;
            const int ok = s < st.count[p];
            if (topk_idx) topk_idx[o] = ok ? st.tape[o].idx : -1;
            if (topk_w) topk_w[o] = ok ? st.weights[o] : 0.0;
            if (topk_l) topk_l[o] = ok ? st.tape[o].l : 0.0;
            if (topk_q) topk_q[o] = ok ? st.tape[o].q : 0.0;
            if (topk_sigma) topk_sigma[o] = ok ? st.tape[o].sigma : 0.0;
        }
    free_state(&st);
    return 0;
}

/* ------------------------------------------------------------------ backward */

typedef struct {
    const forward_state_t* st;
    const gvro_camera* cam;
    const double *attr, *d_image, *d_alpha;
    double tau;
    int through_t, through_rho;
} bwd_job_t;

typedef struct {
    bwd_job_t* job;
    int row_begin, row_end;
    double* d_center;  /* [K*3] camera space */
    double* d_inv_cov; /* [K*9] camera space */
    double* d_attr;    /* [K*D] */
} bwd_part_t;

static void* backward_rows(void* arg) {
    bwd_part_t* part = arg;
    const bwd_job_t* j = part->job;
    const forward_state_t* st = j->st;
    const int kp = st->kp, D = st->D, W = st->W;
    const double tau = j->tau;
    double* peak = malloc(sizeof(double) * (size_t)kp * 6);
    double* trans = peak + kp;
    double* d_peak = trans + kp;
    double* d_l = d_peak + kp;
    double* d_q = d_l + kp;
    double* d_sigma = d_q + kp;
    for (int i = part->row_begin; i < part->row_end; ++i) {
        for (int col = 0; col < W; ++col) {
            const size_t p = (size_t)i * W + col;
            const traced_t* sel = st->tape + p * kp;
            const int n = st->count[p];
            if (n == 0) continue;
            /* src/grad.cpp:79-94 */
            double total_peak = 0.0;
            for (int k = 0; k < n; ++k) {
                peak[k] = exp(sel[k].q);
                total_peak += peak[k];
            }
            for (int k = 0; k < n; ++k) {
                double a = 0.0;
                for (int m = 0; m < n; ++m) a += peak[m] * normal_cdf((sel[k].l - sel[m].l) / sel[m].sigma);
                trans[k] = exp(-tau * a);
            }
            const double galpha = j->d_alpha[p];
            for (int k = 0; k < n; ++k) d_peak[k] = d_l[k] = d_q[k] = d_sigma[k] = 0.0;
            /* alpha path (src/grad.cpp:103-106) */
            if (j->through_t && galpha != 0.0) {
                const double d_total = galpha * tau * exp(-tau * total_peak);
                for (int m = 0; m < n; ++m) d_peak[m] += d_total;
            }
            /* src/grad.cpp:108-136 */
            for (int k = 0; k < n; ++k) {
                const double* at = j->attr + (size_t)D * sel[k].idx;
                double d_weight = 0.0;
                for (int c = 0; c < D; ++c) d_weight += j->d_image[p * D + c] * at[c];
                const double weight = trans[k] * peak[k];
                if (weight != 0.0 || d_weight != 0.0) {
                    double* da = part->d_attr + (size_t)D * sel[k].idx;
                    for (int c = 0; c < D; ++c) da[c] += weight * j->d_image[p * D + c];
                }
                if (d_weight == 0.0) continue;
                if (j->through_rho) d_peak[k] += d_weight * trans[k];
                if (j->through_t) {
                    const double d_acc = -tau * trans[k] * (d_weight * peak[k]);
                    if (d_acc != 0.0) {
                        for (int m = 0; m < n; ++m) {
                            const double u = sel[k].l - sel[m].l;
                            const double z = u / sel[m].sigma;
                            d_peak[m] += d_acc * normal_cdf(z);
                            const double d_cdf = d_acc * peak[m];
                            const double pdf = normal_pdf(z) / sel[m].sigma;
                            d_l[k] += d_cdf * pdf;
                            d_l[m] -= d_cdf * pdf;
                            d_sigma[m] -= d_cdf * pdf * z;
                        }
                    }
                }
            }
            for (int k = 0; k < n; ++k) d_q[k] += d_peak[k] * peak[k];
            /* chain to camera-space center / inv_cov (src/grad.cpp:141-173) */
            double d[3];
            pixel_ray(j->cam, i, col, d);
            for (int k = 0; k < n; ++k) {
                if (d_l[k] == 0.0 && d_q[k] == 0.0 && d_sigma[k] == 0.0) continue;
                const int idx = sel[k].idx;
                const double* m = st->cc + 3 * (size_t)idx;
                const double* s = st->cs + 9 * (size_t)idx;
                double sd[3], v[3], sv[3];
                mat_vec(s, d, sd);
                const double a = dot3(d, sd);
                for (int t = 0; t < 3; ++t) v[t] = m[t] - sel[k].l * d[t];
                mat_vec(s, v, sv);
                double dm[3] = {0, 0, 0}, ds[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
                if (d_l[k] != 0.0) {
                    const double scale = d_l[k] / a;
                    for (int r = 0; r < 3; ++r) dm[r] += scale * sd[r];
                    for (int r = 0; r < 3; ++r)
                        for (int c = 0; c < 3; ++c)
                            ds[3 * r + c] += scale * (0.5 * (m[r] * d[c] + d[r] * m[c]) - sel[k].l * (d[r] * d[c]));
                }
                if (d_q[k] != 0.0) {
                    for (int r = 0; r < 3; ++r) dm[r] -= d_q[k] * sv[r];
                    for (int r = 0; r < 3; ++r)
                        for (int c = 0; c < 3; ++c) ds[3 * r + c] -= 0.5 * d_q[k] * (v[r] * v[c]);
                }
                if (d_sigma[k] != 0.0) {
                    const double d_a = -0.5 * pow(sel[k].sigma, 3) * d_sigma[k];
                    for (int r = 0; r < 3; ++r)
                        for (int c = 0; c < 3; ++c) ds[3 * r + c] += d_a * (d[r] * d[c]);
                }
                for (int r = 0; r < 3; ++r) part->d_center[3 * (size_t)idx + r] += dm[r];
                for (int r = 0; r < 9; ++r) part->d_inv_cov[9 * (size_t)idx + r] += ds[r];
            }
        }
    }
    free(peak);
    return NULL;
}

static void init_bwd_part(void* part, int w, int b, int e, void* ctx) {
    (void)w;
    bwd_part_t* p = part;
    p->job = ctx;
    p->row_begin = b;
    p->row_end = e;
}

/* backward (src/grad.cpp:49-199) on a rendered state. */
static void backward_from_state(forward_state_t* st, int K, int D, const double* centers, const double* inv_cov,
                                const double* attr, double tau, const gvro_camera* cam, int threads,
                                const double* d_image, const double* d_alpha, int through_transmittance,
                                int through_density, double* d_center, double* d_inv_cov, double* d_attr,
                                double* d_rotation, double* d_translation) {
    bwd_job_t job = {st, cam, attr, d_image, d_alpha, tau, through_transmittance, through_density};
    const int workers_req = resolve_threads(threads);
    int workers = workers_req < st->H ? workers_req : st->H;
    if (workers < 1) workers = 1;
    bwd_part_t* parts = calloc((size_t)workers, sizeof(bwd_part_t));
    for (int w = 0; w < workers; ++w) {
        parts[w].d_center = calloc(3 * (size_t)(K > 0 ? K : 1), sizeof(double));
        parts[w].d_inv_cov = calloc(9 * (size_t)(K > 0 ? K : 1), sizeof(double));
        parts[w].d_attr = calloc((size_t)(D > 0 ? D : 1) * (size_t)(K > 0 ? K : 1), sizeof(double));
    }
    run_partitions(st->H, workers, backward_rows, parts, sizeof(bwd_part_t), init_bwd_part, &job);

    /* fixed worker-order reduction (src/grad.cpp:176-182) */
    double* tc = calloc(3 * (size_t)(K > 0 ? K : 1), sizeof(double));
    double* ts = calloc(9 * (size_t)(K > 0 ? K : 1), sizeof(double));
    double* ta = calloc((size_t)(D > 0 ? D : 1) * (size_t)(K > 0 ? K : 1), sizeof(double));
    for (int w = 0; w < workers; ++w) {
        for (size_t i = 0; i < 3 * (size_t)K; ++i) tc[i] += parts[w].d_center[i];
        for (size_t i = 0; i < 9 * (size_t)K; ++i) ts[i] += parts[w].d_inv_cov[i];
        for (size_t i = 0; i < (size_t)D * K; ++i) ta[i] += parts[w].d_attr[i];
        free(parts[w].d_center);
        free(parts[w].d_inv_cov);
        free(parts[w].d_attr);
    }
    free(parts);

    /* camera -> object space, once per kernel (src/grad.cpp:184-197) */
    const double* r = cam->rotation;
    double rt[9];
    transpose3(r, rt);
    double dR[9] = {0}, dT[3] = {0};
    for (int k = 0; k < K; ++k) {
        const double* dm = tc + 3 * (size_t)k;
        const double* dS = ts + 9 * (size_t)k;
        double oc[3], tmp[9], oS[9];
        mat_vec(rt, dm, oc);
        mat_mul(rt, dS, tmp);
        mat_mul(tmp, r, oS);
        if (d_center) memcpy(d_center + 3 * (size_t)k, oc, sizeof oc);
        if (d_inv_cov) memcpy(d_inv_cov + 9 * (size_t)k, oS, sizeof oS);
        if (d_attr) memcpy(d_attr + (size_t)D * k, ta + (size_t)D * k, sizeof(double) * (size_t)D);
        for (int t = 0; t < 3; ++t) dT[t] += dm[t];
        const double* mo = centers + 3 * (size_t)k;
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) dR[3 * a + b] += dm[a] * mo[b];
        double t2[9], t3[9];
        for (int t = 0; t < 9; ++t) t2[t] = 2.0 * dS[t];
        mat_mul(t2, r, t3);
        mat_mul(t3, inv_cov + 9 * (size_t)k, tmp);
        for (int t = 0; t < 9; ++t) dR[t] += tmp[t];
    }
    if (d_rotation) memcpy(d_rotation, dR, sizeof dR);
    if (d_translation) memcpy(d_translation, dT, sizeof dT);
    free(tc);
    free(ts);
    free(ta);
}

int gvro_backward(int K, int D, double tau, const double* centers, const double* inv_cov,
                  const double* attr, const gvro_camera* cam, const gvro_selection* cfg, int threads,
                  const double* d_image, const double* d_alpha, int through_transmittance,
                  int through_density, double* d_center, double* d_inv_cov, double* d_attr,
                  double* d_rotation, double* d_translation) {
    const int Dc = D > 1 ? D : 1;
    const size_t P = (size_t)cam->height * cam->width;
    double* image = malloc(sizeof(double) * P * Dc);
    double* alpha = malloc(sizeof(double) * P);
    double* depth = malloc(sizeof(double) * P);
    forward_state_t st;
    const int rc = render_core(K, D, tau, centers, inv_cov, attr, cam, cfg, threads, image, alpha, depth, &st);
    free(image);
    free(alpha);
    free(depth);
    if (rc) return rc;
    backward_from_state(&st, K, D, centers, inv_cov, attr, tau, cam, threads, d_image, d_alpha, through_transmittance,
                        through_density, d_center, d_inv_cov, d_attr, d_rotation, d_translation);
    free_state(&st);
    return 0;
}

/* One fwd+bwd step as the reference's loss loop runs it: render_with_tape ->
 * ScalarLoss::value (src/grad.cpp:201-216, w = 1) -> backward. D >= 1. */
int gvro_fwd_bwd_step(int K, int D, double tau, const double* centers, const double* inv_cov,
                      const double* attr, const gvro_camera* cam, const gvro_selection* cfg, int threads,
                      const double* target_image, const double* target_alpha, double* loss_out,
                      double* d_center, double* d_attr) {
    const size_t P = (size_t)cam->height * cam->width;
    double* image = malloc(sizeof(double) * P * (size_t)D);
    double* alpha = malloc(sizeof(double) * P);
    double* depth = malloc(sizeof(double) * P);
    forward_state_t st;
    const int rc = render_core(K, D, tau, centers, inv_cov, attr, cam, cfg, threads, image, alpha, depth, &st);
    if (rc) {
        free(image);
        free(alpha);
        free(depth);
        return rc;
    }
    double loss = 0.0;
    for (size_t i = 0; i < P * (size_t)D; ++i) {
        const double diff = image[i] - target_image[i];
        loss += 0.5 * diff * diff;
        image[i] = diff; /* d_image in place */
    }
    for (size_t i = 0; i < P; ++i) {
        const double diff = alpha[i] - target_alpha[i];
        loss += 0.5 * diff * diff;
        alpha[i] = diff;
    }
    if (loss_out) *loss_out = loss;
    backward_from_state(&st, K, D, centers, inv_cov, attr, tau, cam, threads, image, alpha, 1, 1, d_center, NULL,
                        d_attr, NULL, NULL);
    free_state(&st);
    free(image);
    free(alpha);
    free(depth);
    return 0;
}

int gvro_coarse_boxes(int K, int D, double tau, const double* centers, const double* inv_cov,
                      const double* attr, const gvro_camera* cam, const gvro_selection* cfg,
                      int* cell_box, int* dropped_behind) {
    if (validate_scene(K, D, tau, centers, inv_cov, attr)) return 1;
    if (validate_camera(cam)) return 1;
    if (validate_cfg(cfg)) return 1;
    double* cc = malloc(sizeof(double) * 3 * (size_t)(K > 0 ? K : 1));
    double* cs = malloc(sizeof(double) * 9 * (size_t)(K > 0 ? K : 1));
    view_transform(K, centers, inv_cov, cam, cc, cs);
    int dropped = 0;
    coarse_boxes(K, cc, cs, cam, cfg, cell_box, &dropped);
    if (dropped_behind) *dropped_behind = dropped;
    free(cc);
    free(cs);
    return 0;
}

/* ------------------------------------------------------------------ sampler + helpers */

/* sample_attributes (src/sampler.cpp:11-51): render, then per pixel in row-major
 * order scatter W (or W / max(sum W, kSupportEps) when normalized) into the
 * support and the weighted attribute sums; kernels with support < 1e-8
 * (include/gvr/sampler.hpp:18) are zeroed and masked. */
int gvro_sample_attributes(int K, int D, double tau, const double* centers, const double* inv_cov,
                           const double* attr, const gvro_camera* cam, const gvro_selection* cfg, int threads,
                           const double* observed, int obs_h, int obs_w, int channels, int normalized,
                           double* attrs, double* support, unsigned char* masked) {
    if (obs_h != cam->height || obs_w != cam->width) return fail("observed image size does not match the camera");
    const int Dc = D > 1 ? D : 1;
    const size_t P = (size_t)cam->height * cam->width;
    double* image = malloc(sizeof(double) * P * Dc);
    double* alpha = malloc(sizeof(double) * P);
    double* depth = malloc(sizeof(double) * P);
    forward_state_t st;
    const int rc = render_core(K, D, tau, centers, inv_cov, attr, cam, cfg, threads, image, alpha, depth, &st);
    free(image);
    free(alpha);
    free(depth);
    if (rc) return rc;
    memset(attrs, 0, sizeof(double) * (size_t)K * channels);
    memset(support, 0, sizeof(double) * (size_t)K);
    for (size_t p = 0; p < P; ++p) {
        const int n = st.count[p];
        double denom = 0.0;
        if (normalized) {
            for (int s = 0; s < n; ++s) denom += st.weights[p * st.kp + s];
            denom = denom > 1e-8 ? denom : 1e-8;
        }
        for (int s = 0; s < n; ++s) {
            const int k = st.tape[p * st.kp + s].idx;
            const double w = st.weights[p * st.kp + s];
            const double ww = normalized ? w / denom : w;
            support[k] += ww;
            for (int c = 0; c < channels; ++c) attrs[(size_t)channels * k + c] += ww * observed[p * channels + c];
        }
    }
    for (int k = 0; k < K; ++k) {
        if (support[k] < 1e-8) {
            for (int c = 0; c < channels; ++c) attrs[(size_t)channels * k + c] = 0.0;
            masked[k] = 1;
        } else {
            for (int c = 0; c < channels; ++c) attrs[(size_t)channels * k + c] /= support[k];
            masked[k] = 0;
        }
    }
    free_state(&st);
    return 0;
}

/* Per pixel: transmittance_at (src/blender.cpp:19-25) over the pixel's selected
 * traced kernels at depth t[p], and normalized_weights (src/blender.cpp:55-62)
 * of its weights (K'-padded with 0). Outputs nullable. */
int gvro_pixel_helpers(int K, int D, double tau, const double* centers, const double* inv_cov,
                       const double* attr, const gvro_camera* cam, const gvro_selection* cfg, int threads,
                       const double* t, double* trans_out, double eps, double* norm_w) {
    const int Dc = D > 1 ? D : 1;
    const size_t P = (size_t)cam->height * cam->width;
    double* image = malloc(sizeof(double) * P * Dc);
    double* alpha = malloc(sizeof(double) * P);
    double* depth = malloc(sizeof(double) * P);
    forward_state_t st;
    const int rc = render_core(K, D, tau, centers, inv_cov, attr, cam, cfg, threads, image, alpha, depth, &st);
    free(image);
    free(alpha);
    free(depth);
    if (rc) return rc;
    for (size_t p = 0; p < P; ++p) {
        const int n = st.count[p];
        if (trans_out) {
            double acc = 0.0;
            for (int s = 0; s < n; ++s) {
                const traced_t* k = &st.tape[p * st.kp + s];
                acc += exp(k->q) * normal_cdf((t[p] - k->l) / k->sigma);
            }
            trans_out[p] = exp(-tau * acc);
        }
        if (norm_w) {
            double total = 0.0;
            for (int s = 0; s < n; ++s) total += st.weights[p * st.kp + s];
            const double denom = total > eps ? total : eps;
            for (int s = 0; s < st.kp; ++s) norm_w[p * st.kp + s] = s < n ? st.weights[p * st.kp + s] / denom : 0.0;
        }
    }
    free_state(&st);
    return 0;
}

/* shade_lambert (src/blender.cpp:146-172); normals[H*W*3], alpha/depth[H*W], out[H*W*3]. */
int gvro_shade_lambert(const gvro_camera* cam, const double* normals, const double* alpha, const double* depth,
                       const double* light_pos, const double* light_color, double* out) {
    const int H = cam->height, W = cam->width;
    double rt[9];
    transpose3(cam->rotation, rt);
    memset(out, 0, sizeof(double) * (size_t)H * W * 3);
    for (int i = 0; i < H; ++i)
        for (int j = 0; j < W; ++j) {
            const size_t p = (size_t)i * W + j;
            if (alpha[p] <= 0.0) continue;
            double n[3] = {normals[3 * p], normals[3 * p + 1], normals[3 * p + 2]};
            const double len = sqrt(dot3(n, n));
            if (len < 1e-12) continue;
            for (int c = 0; c < 3; ++c) n[c] /= len;
            double d[3], pc[3], po[3], tl[3];
            pixel_ray(cam, i, j, d);
            for (int c = 0; c < 3; ++c) pc[c] = depth[p] * d[c] - cam->translation[c];
            mat_vec(rt, pc, po);
            for (int c = 0; c < 3; ++c) tl[c] = light_pos[c] - po[c];
            const double tn = sqrt(dot3(tl, tl));
            for (int c = 0; c < 3; ++c) tl[c] /= tn;
            double intensity = dot3(n, tl);
            if (intensity < 0.0) intensity = 0.0;
            for (int c = 0; c < 3; ++c) out[3 * p + c] = intensity * light_color[c];
        }
    return 0;
}
