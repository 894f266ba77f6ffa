/*
 * potr_oracle.c -- CPU restatement of the POTR hot paths.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path (paper_2601_14821_b200/csrc).  Only tests/, the smoke() entry of
 * __graft_entry__.py and the cpu_baseline / --impl reference legs of bench.py
 * may load it.  The product never links or calls it.
 *
 * It restates, in plain C99 float64 with no FMA contraction
 * (-ffp-contract=off), the algorithm of the reference package
 * (/root/reference/pkg/src/potr, cited as file:line below):
 *
 *   rasterizer.py:40-53    quat_to_rotmat
 *   rasterizer.py:56-97    project_splats
 *   rasterizer.py:100-110  splat_colors (sh.py:23-51 sh_basis)
 *   rasterizer.py:246-250  valid ids + stable argsort by view depth
 *   rasterizer.py:113-203  _composite (splat-major, records every contribution)
 *   rasterizer.py:226-230  camera_importance  (bincount(T*alpha)/P)
 *   rasterizer.py:232-243  prune_deltas       (forward form)
 *   rasterizer.py:322-352  forward_stats      (dSE, bincount, mse, camera-order sum)
 *   compaction.py:89-243   build_weighted_system .. compact_scene
 *
 * Accumulations follow the reference's order: bincount adds records in record
 * order (splat-major, row-major pixels); cameras are summed in index order;
 * numpy's pairwise summation is restated for np.mean.  Parity is pinned
 * against golden vectors produced by the reference itself
 * (tests/golden/, generator oracle/gen_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

/* Minimal pthread parallel-for (the reference maps cameras onto a thread pool,
 * rasterizer.py:304-308).  Work items are claimed in index order. */
typedef struct {
    void (*fn)(void *ctx, int64_t i, int worker);
    void *ctx;
    int64_t n;
    int64_t next;
    pthread_mutex_t mu;
    int nworkers;
} opool;

typedef struct {
    opool *pool;
    int worker;
} oworker;

static void *pool_main(void *arg) {
    oworker *w = (oworker *)arg;
    opool *p = w->pool;
    for (;;) {
        pthread_mutex_lock(&p->mu);
        int64_t i = p->next++;
        pthread_mutex_unlock(&p->mu);
        if (i >= p->n) break;
        p->fn(p->ctx, i, w->worker);
    }
    return NULL;
}

static void parallel_for(int64_t n, int threads, void (*fn)(void *, int64_t, int), void *ctx) {
    if (threads < 1) threads = 1;
    if (threads > n) threads = (int)(n > 0 ? n : 1);
    opool p;
    p.fn = fn;
    p.ctx = ctx;
    p.n = n;
    p.next = 0;
    p.nworkers = threads;
    pthread_mutex_init(&p.mu, NULL);
    pthread_t tid[256];
    oworker ws[256];
    if (threads > 256) threads = 256;
    for (int t = 1; t < threads; t++) {
        ws[t].pool = &p;
        ws[t].worker = t;
        pthread_create(&tid[t], NULL, pool_main, &ws[t]);
    }
    ws[0].pool = &p;
    ws[0].worker = 0;
    pool_main(&ws[0]);
    for (int t = 1; t < threads; t++) pthread_join(tid[t], NULL);
    pthread_mutex_destroy(&p.mu);
}

/* same layout as potr_camera in include/potr_b200.h */
typedef struct {
    double eye[3];
    double rot[9]; /* world-to-camera rows, row-major */
    double fx, fy, cx, cy;
    int32_t width, height;
} ocam;

/* rasterizer.py:22-26 */
#define ALPHA_FLOOR (1.0 / 255.0)
#define ALPHA_CAP 0.999
#define T_TERMINATE 1e-4
#define NEAR_CLIP 0.01
#define COV_DILATION 0.3

/* sh.py:11-18 */
#define SH_DC 0.28209479177387814
#define SH_C1 0.4886025119029199
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

/* sh.py:23-51 */
static void sh_basis16(double x, double y, double z, double *o) {
    double xx = x * x, yy = y * y, zz = z * z;
    double xy = x * y, yz = y * z, xz = x * z;
    o[0] = SH_DC;
    o[1] = -SH_C1 * y;
    o[2] = SH_C1 * z;
    o[3] = -SH_C1 * x;
    o[4] = SH_C2[0] * xy;
    o[5] = SH_C2[1] * yz;
    o[6] = SH_C2[2] * (2.0 * zz - xx - yy);
    o[7] = SH_C2[3] * xz;
    o[8] = SH_C2[4] * (xx - yy);
    o[9] = SH_C3[0] * y * (3.0 * xx - yy);
    o[10] = SH_C3[1] * xy * z;
    o[11] = SH_C3[2] * y * (4.0 * zz - xx - yy);
    o[12] = SH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    o[13] = SH_C3[4] * x * (4.0 * zz - xx - yy);
    o[14] = SH_C3[5] * z * (xx - yy);
    o[15] = SH_C3[6] * x * (xx - 3.0 * yy);
}

/* numpy pairwise summation of a contiguous float64 vector (the inner loop of
 * np.add.reduce, used by np.mean in rasterizer.py:335). */
static double pairwise_sum(const double *a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; i++) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
    }
}

/* ------------------------------------------------------------------------ */
/* Projection: rasterizer.py:56-97 (quat_to_rotmat :40-53)                   */

typedef struct {
    double mx, my, a, b, c, depth, radius;
    int valid;
} oproj;

static void project_one(const double *p, const double *s, const double *q, const ocam *cam,
                        oproj *out) {
    const double *W = cam->rot;
    double d0 = p[0] - cam->eye[0], d1 = p[1] - cam->eye[1], d2 = p[2] - cam->eye[2];
    /* (positions - eye) @ W.T runs through OpenBLAS dgemm, whose x86 kernels
     * accumulate the 3-term dot product with FMA in index order; restating
     * that reproduces the reference's depth key bit for bit. */
    double t0 = fma(d2, W[2], fma(d1, W[1], d0 * W[0]));
    double t1 = fma(d2, W[5], fma(d1, W[4], d0 * W[3]));
    double t2 = fma(d2, W[8], fma(d1, W[7], d0 * W[6]));
    int valid = t2 > NEAR_CLIP;
    double safe_z = valid ? t2 : 1.0;
    double inv_z = 1.0 / safe_z;
    double mx = cam->fx * t0 * inv_z + cam->cx;
    double my = cam->fy * t1 * inv_z + cam->cy;

    double w = q[0], x = q[1], y = q[2], z = q[3];
    double R[9];
    R[0] = 1 - 2 * (y * y + z * z);
    R[1] = 2 * (x * y - w * z);
    R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z);
    R[4] = 1 - 2 * (x * x + z * z);
    R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y);
    R[7] = 2 * (y * z + w * x);
    R[8] = 1 - 2 * (x * x + y * y);
    double s2[3] = {s[0] * s[0], s[1] * s[1], s[2] * s[2]};
    /* Sigma_ik = sum_j R_ij s2_j R_kj */
    double S[9];
    for (int i = 0; i < 3; i++)
        for (int k = 0; k < 3; k++) {
            double acc = 0.0;
            for (int j = 0; j < 3; j++) acc += R[i * 3 + j] * s2[j] * R[k * 3 + j];
            S[i * 3 + k] = acc;
        }
    /* Sigma_view_il = sum_j sum_k W_ij S_jk W_lk */
    double V[9];
    for (int i = 0; i < 3; i++)
        for (int l = 0; l < 3; l++) {
            double acc = 0.0;
            for (int j = 0; j < 3; j++)
                for (int k = 0; k < 3; k++) acc += W[i * 3 + j] * S[j * 3 + k] * W[l * 3 + k];
            V[i * 3 + l] = acc;
        }
    double J[6] = {cam->fx * inv_z, 0.0, -cam->fx * t0 * inv_z * inv_z,
                   0.0, cam->fy * inv_z, -cam->fy * t1 * inv_z * inv_z};
    double C[4];
    for (int i = 0; i < 2; i++)
        for (int l = 0; l < 2; l++) {
            double acc = 0.0;
            for (int j = 0; j < 3; j++)
                for (int k = 0; k < 3; k++) acc += J[i * 3 + j] * V[j * 3 + k] * J[l * 3 + k];
            C[i * 2 + l] = acc;
        }
    double a = C[0] + COV_DILATION;
    double b = C[1];
    double c = C[3] + COV_DILATION;
    double mid = 0.5 * (a + c);
    double det = a * c - b * b;
    double disc = mid * mid - det;
    double lam_max = mid + sqrt(disc > 0.0 ? disc : 0.0);
    double r = 3.0 * sqrt(lam_max);
    valid = valid && (mx >= -r) && (mx <= cam->width + r);
    valid = valid && (my >= -r) && (my <= cam->height + r);
    out->mx = mx;
    out->my = my;
    out->a = a;
    out->b = b;
    out->c = c;
    out->depth = t2;
    out->radius = r;
    out->valid = valid;
}

/* rasterizer.py:100-110 */
static void color_one(const double *p, const double *sh, const ocam *cam, double *rgb) {
    double d0 = p[0] - cam->eye[0], d1 = p[1] - cam->eye[1], d2 = p[2] - cam->eye[2];
    double norm = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
    if (norm == 0.0) norm = 1.0;
    double basis[16];
    sh_basis16(d0 / norm, d1 / norm, d2 / norm, basis);
    for (int ch = 0; ch < 3; ch++) {
        double acc = 0.0;
        for (int i = 0; i < 16; i++) acc += sh[ch * 16 + i] * basis[i];
        rgb[ch] = acc > 0.0 ? acc : 0.0;
    }
}

int oracle_project(int64_t n, const double *pos, const double *sh, const double *opac,
                   const double *scales, const double *rot, const ocam *cam, double *mean2d,
                   double *cov2d, double *depth, double *radius, uint8_t *valid, double *colors) {
    (void)opac;
    for (int64_t k = 0; k < n; k++) {
        oproj pr;
        project_one(pos + 3 * k, scales + 3 * k, rot + 4 * k, cam, &pr);
        mean2d[2 * k] = pr.mx;
        mean2d[2 * k + 1] = pr.my;
        cov2d[3 * k] = pr.a;
        cov2d[3 * k + 1] = pr.b;
        cov2d[3 * k + 2] = pr.c;
        depth[k] = pr.depth;
        radius[k] = pr.radius;
        valid[k] = (uint8_t)pr.valid;
        if (colors) color_one(pos + 3 * k, sh + 48 * k, cam, colors + 3 * k);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Depth order: rasterizer.py:248-250.  np.argsort(kind="stable") over the   */
/* valid ids == sort by (depth, id).                                          */

typedef struct {
    double depth;
    int64_t id;
} okey;

static int cmp_key(const void *x, const void *y) {
    const okey *a = (const okey *)x, *b = (const okey *)y;
    if (a->depth < b->depth) return -1;
    if (a->depth > b->depth) return 1;
    return (a->id > b->id) - (a->id < b->id);
}

/* Per-camera scratch: projection, order, records. */
typedef struct {
    int64_t n_valid;
    int64_t *order; /* valid ids in depth order */
    oproj *proj;
    double *colors; /* (n,3), zero for non-valid */
} oview;

static int view_prepare(int64_t n, const double *pos, const double *sh, const double *scales,
                        const double *rot, const ocam *cam, oview *v) {
    v->proj = (oproj *)malloc(sizeof(oproj) * (size_t)(n > 0 ? n : 1));
    v->colors = (double *)calloc((size_t)(3 * (n > 0 ? n : 1)), sizeof(double));
    okey *keys = (okey *)malloc(sizeof(okey) * (size_t)(n > 0 ? n : 1));
    v->order = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    if (!v->proj || !v->colors || !keys || !v->order) return -1;
    int64_t nv = 0;
    for (int64_t k = 0; k < n; k++) {
        project_one(pos + 3 * k, scales + 3 * k, rot + 4 * k, cam, &v->proj[k]);
        if (v->proj[k].valid) {
            keys[nv].depth = v->proj[k].depth;
            keys[nv].id = k;
            nv++;
            color_one(pos + 3 * k, sh + 48 * k, cam, v->colors + 3 * k);
        }
    }
    qsort(keys, (size_t)nv, sizeof(okey), cmp_key);
    for (int64_t i = 0; i < nv; i++) v->order[i] = keys[i].id;
    v->n_valid = nv;
    free(keys);
    return 0;
}

static void view_free(oview *v) {
    free(v->proj);
    free(v->colors);
    free(v->order);
}

int oracle_depth_order(int64_t n, const double *pos, const double *scales, const double *rot,
                       const ocam *cam, int64_t *order_out, int64_t *n_valid_out) {
    oview v;
    /* sh only needed for colors: pass a zero block */
    double *zsh = (double *)calloc((size_t)(48 * (n > 0 ? n : 1)), sizeof(double));
    if (!zsh) return -1;
    int rc = view_prepare(n, pos, zsh, scales, rot, cam, &v);
    free(zsh);
    if (rc) return rc;
    memcpy(order_out, v.order, sizeof(int64_t) * (size_t)v.n_valid);
    *n_valid_out = v.n_valid;
    view_free(&v);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Compositing: rasterizer.py:113-203.                                       */

typedef struct {
    int32_t splat; /* original id */
    int32_t pix;
    double alpha, t, p[3];
} orec;

typedef struct {
    orec *r;
    int64_t n, cap;
} orecs;

static int recs_push(orecs *R, const orec *x) {
    if (R->n == R->cap) {
        int64_t nc = R->cap ? R->cap * 2 : 16384;
        orec *nr = (orec *)realloc(R->r, sizeof(orec) * (size_t)nc);
        if (!nr) return -1;
        R->r = nr;
        R->cap = nc;
    }
    R->r[R->n++] = *x;
    return 0;
}

static int composite(const oview *v, const double *opac, const ocam *cam, double *image,
                     double *trans, orecs *R) {
    int W = cam->width, H = cam->height;
    for (int64_t i = 0; i < (int64_t)W * H; i++) {
        image[3 * i] = image[3 * i + 1] = image[3 * i + 2] = 0.0;
        trans[i] = 1.0;
    }
    for (int64_t oi = 0; oi < v->n_valid; oi++) {
        int64_t k = v->order[oi];
        const oproj *pr = &v->proj[k];
        double mx = pr->mx, my = pr->my, r = pr->radius;
        /* int(np.floor(.)) clipped; done in double to stay overflow-free */
        double x0 = floor(mx - r), x1 = ceil(mx + r), y0 = floor(my - r), y1 = ceil(my + r);
        if (x0 < 0) x0 = 0;
        if (y0 < 0) y0 = 0;
        if (x1 > W - 1) x1 = W - 1;
        if (y1 > H - 1) y1 = H - 1;
        if (x0 > x1 || y0 > y1) continue;
        double det = pr->a * pr->c - pr->b * pr->b;
        if (det <= 0.0) continue;
        double ia = pr->c / det, ib = -pr->b / det, ic = pr->a / det;
        double o = opac[k];
        const double *col = v->colors + 3 * k;
        for (int py = (int)y0; py <= (int)y1; py++) {
            double dy = (py + 0.5) - my;
            for (int px = (int)x0; px <= (int)x1; px++) {
                int64_t pix = (int64_t)py * W + px;
                double t_here = trans[pix];
                if (t_here < T_TERMINATE) continue;
                double dx = (px + 0.5) - mx;
                double power = -0.5 * (ia * dx * dx + ic * dy * dy) - ib * dx * dy;
                double alpha = o * exp(power);
                if (alpha > ALPHA_CAP) alpha = ALPHA_CAP;
                if (alpha < ALPHA_FLOOR) continue;
                if (R) {
                    orec x;
                    x.splat = (int32_t)k;
                    x.pix = (int32_t)pix;
                    x.alpha = alpha;
                    x.t = t_here;
                    x.p[0] = image[3 * pix];
                    x.p[1] = image[3 * pix + 1];
                    x.p[2] = image[3 * pix + 2];
                    if (recs_push(R, &x)) return -1;
                }
                double w = t_here * alpha;
                image[3 * pix] += w * col[0];
                image[3 * pix + 1] += w * col[1];
                image[3 * pix + 2] += w * col[2];
                trans[pix] = t_here * (1.0 - alpha);
            }
        }
    }
    return 0;
}

/* render_image (rasterizer.py:270-271) plus the records of render_with_records
 * (:246-267).  records_out may be NULL: then only the count is returned. */
int oracle_render(int64_t n, const double *pos, const double *sh, const double *opac,
                  const double *scales, const double *rot, const ocam *cam, double *image,
                  double *trans, int64_t *n_records, int32_t *rec_splat, int32_t *rec_pix,
                  double *rec_alpha, double *rec_t, double *rec_p, int64_t rec_cap) {
    oview v;
    if (view_prepare(n, pos, sh, scales, rot, cam, &v)) return -1;
    orecs R = {0, 0, 0};
    int rc = composite(&v, opac, cam, image, trans, &R);
    if (!rc) {
        *n_records = R.n;
        if (rec_splat && R.n <= rec_cap) {
            for (int64_t i = 0; i < R.n; i++) {
                rec_splat[i] = R.r[i].splat;
                rec_pix[i] = R.r[i].pix;
                rec_alpha[i] = R.r[i].alpha;
                rec_t[i] = R.r[i].t;
                rec_p[3 * i] = R.r[i].p[0];
                rec_p[3 * i + 1] = R.r[i].p[1];
                rec_p[3 * i + 2] = R.r[i].p[2];
            }
        }
    }
    free(R.r);
    view_free(&v);
    return rc;
}

/* One camera of forward_stats (rasterizer.py:322-336). */
static int one_camera(int64_t n, const double *pos, const double *sh, const double *opac,
                      const double *scales, const double *rot, const ocam *cam,
                      const double *target, double *imp, double *dmse, double *mse) {
    oview v;
    if (view_prepare(n, pos, sh, scales, rot, cam, &v)) return -1;
    int64_t P = (int64_t)cam->width * cam->height;
    double *image = (double *)malloc(sizeof(double) * (size_t)(3 * P));
    double *trans = (double *)malloc(sizeof(double) * (size_t)P);
    orecs R = {0, 0, 0};
    int rc = (!image || !trans) ? -1 : composite(&v, opac, cam, image, trans, &R);
    if (!rc) {
        /* camera_importance :226-230 -- bincount in record order, then / (W*H) */
        for (int64_t k = 0; k < n; k++) imp[k] = 0.0;
        for (int64_t i = 0; i < R.n; i++) imp[R.r[i].splat] += R.r[i].t * R.r[i].alpha;
        for (int64_t k = 0; k < n; k++) imp[k] = imp[k] / (double)P;
        if (target) {
            /* prune_deltas :240-243, dSE :333, dmse :334 */
            for (int64_t k = 0; k < n; k++) dmse[k] = 0.0;
            for (int64_t i = 0; i < R.n; i++) {
                const orec *x = &R.r[i];
                const double *pk = image + 3 * (int64_t)x->pix;
                const double *ct = target + 3 * (int64_t)x->pix;
                const double *cs = v.colors + 3 * (int64_t)x->splat;
                double a = x->alpha;
                double f = a / (1.0 - a);
                double dse = 0.0;
                for (int ch = 0; ch < 3; ch++) {
                    double pd = f * (pk[ch] - x->p[ch] - x->t * cs[ch]);
                    double term = pd * pd + 2.0 * pd * (pk[ch] - ct[ch]);
                    dse = ch == 0 ? term : dse + term;
                }
                dmse[x->splat] += dse;
            }
            for (int64_t k = 0; k < n; k++) dmse[k] = dmse[k] / ((double)P * 3.0);
            /* mse :335 */
            double *sq = (double *)malloc(sizeof(double) * (size_t)(3 * P));
            if (!sq) {
                rc = -1;
            } else {
                for (int64_t i = 0; i < 3 * P; i++) {
                    double d = image[i] - target[i];
                    sq[i] = d * d;
                }
                *mse = pairwise_sum(sq, 3 * P) / (double)(3 * P);
                free(sq);
            }
        }
    }
    free(R.r);
    free(image);
    free(trans);
    view_free(&v);
    return rc;
}

typedef struct {
    int64_t n;
    const double *pos, *sh, *opac, *scales, *rot;
    const ocam *cams;
    const double *const *targets;
    double *cam_imp, *dm, *ms;
    volatile int err;
} fs_ctx;

static void fs_item(void *vctx, int64_t s, int worker) {
    (void)worker;
    fs_ctx *c = (fs_ctx *)vctx;
    int rc = one_camera(c->n, c->pos, c->sh, c->opac, c->scales, c->rot, &c->cams[s],
                        c->targets ? c->targets[s] : NULL, c->cam_imp + s * c->n,
                        c->dm ? c->dm + s * c->n : NULL, c->ms ? &c->ms[s] : NULL);
    if (rc) c->err = 1;
}

/* forward_stats (rasterizer.py:311-352).  targets: ncam pointers or NULL.
 * camera_importance: (ncam, n) output.  Cameras may run on `threads` worker
 * threads; the per-camera results are reduced in camera index order, as the
 * reference does (:338-352), so the output does not depend on `threads`. */
int oracle_forward_stats(int64_t n, const double *pos, const double *sh, const double *opac,
                         const double *scales, const double *rot, int ncam, const ocam *cams,
                         const double *const *targets, int threads, double *importance,
                         double *camera_importance, double *delta_mse, double *mse_out) {
    double *dm = NULL, *ms = NULL;
    if (targets) {
        dm = (double *)malloc(sizeof(double) * (size_t)ncam * (size_t)(n > 0 ? n : 1));
        ms = (double *)malloc(sizeof(double) * (size_t)(ncam > 0 ? ncam : 1));
        if (!dm || !ms) return -1;
    }
    fs_ctx fc = {n, pos, sh, opac, scales, rot, cams, targets, camera_importance, dm, ms, 0};
    parallel_for(ncam, threads, fs_item, &fc);
    if (fc.err) {
        free(dm);
        free(ms);
        return -1;
    }
    /* importance = cam_imp.mean(axis=0): rows added in order, then / S */
    for (int64_t k = 0; k < n; k++) importance[k] = 0.0;
    for (int s = 0; s < ncam; s++)
        for (int64_t k = 0; k < n; k++) importance[k] += camera_importance[(int64_t)s * n + k];
    for (int64_t k = 0; k < n; k++) importance[k] = importance[k] / (double)ncam;
    if (targets) {
        double mse_total = 0.0;
        for (int64_t k = 0; k < n; k++) delta_mse[k] = 0.0;
        for (int s = 0; s < ncam; s++) {
            for (int64_t k = 0; k < n; k++) delta_mse[k] += dm[(int64_t)s * n + k];
            mse_total += ms[s];
        }
        for (int64_t k = 0; k < n; k++) delta_mse[k] = delta_mse[k] / (double)ncam;
        *mse_out = mse_total / (double)ncam;
    }
    free(dm);
    free(ms);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Tile binning restatement: the per-tile splat lists a */
/* tile rasterizer must walk, derived from the reference's clipped bbox       */
/* (rasterizer.py:135-151) and its stable depth order (:248-250).            */
/* tile_offsets: (ntiles+1); tile_splats: capacity cap.  Returns total count  */
/* in *total (even when cap is too small).                                    */

int oracle_tile_lists(int64_t n, const double *pos, const double *scales, const double *rot,
                      const ocam *cam, int tile_w, int tile_h, int64_t *tile_offsets,
                      int32_t *tile_splats, int64_t cap, int64_t *total) {
    oview v;
    double *zsh = (double *)calloc((size_t)(48 * (n > 0 ? n : 1)), sizeof(double));
    if (!zsh) return -1;
    int rc = view_prepare(n, pos, zsh, scales, rot, cam, &v);
    free(zsh);
    if (rc) return rc;
    int W = cam->width, H = cam->height;
    int tw = (W + tile_w - 1) / tile_w, th = (H + tile_h - 1) / tile_h;
    int64_t ntiles = (int64_t)tw * th;
    int64_t *cnt = (int64_t *)calloc((size_t)(ntiles + 1), sizeof(int64_t));
    int32_t *bb = (int32_t *)malloc(sizeof(int32_t) * 4 * (size_t)(v.n_valid > 0 ? v.n_valid : 1));
    if (!cnt || !bb) return -1;
    for (int pass = 0; pass < 2; pass++) {
        if (pass == 1) {
            int64_t acc = 0;
            for (int64_t t = 0; t < ntiles; t++) {
                int64_t c = cnt[t];
                tile_offsets[t] = acc;
                cnt[t] = acc;
                acc += c;
            }
            tile_offsets[ntiles] = acc;
            *total = acc;
            if (acc > cap) break;
        }
        for (int64_t oi = 0; oi < v.n_valid; oi++) {
            int64_t k = v.order[oi];
            const oproj *pr = &v.proj[k];
            int32_t *b = bb + 4 * oi;
            if (pass == 0) {
                double x0 = floor(pr->mx - pr->radius), x1 = ceil(pr->mx + pr->radius);
                double y0 = floor(pr->my - pr->radius), y1 = ceil(pr->my + pr->radius);
                if (x0 < 0) x0 = 0;
                if (y0 < 0) y0 = 0;
                if (x1 > W - 1) x1 = W - 1;
                if (y1 > H - 1) y1 = H - 1;
                double det = pr->a * pr->c - pr->b * pr->b;
                if (x0 > x1 || y0 > y1 || det <= 0.0) {
                    b[0] = -1;
                    continue;
                }
                b[0] = (int32_t)x0 / tile_w;
                b[1] = (int32_t)x1 / tile_w;
                b[2] = (int32_t)y0 / tile_h;
                b[3] = (int32_t)y1 / tile_h;
            }
            if (b[0] < 0) continue;
            for (int ty = b[2]; ty <= b[3]; ty++)
                for (int tx = b[0]; tx <= b[1]; tx++) {
                    int64_t t = (int64_t)ty * tw + tx;
                    if (pass == 0)
                        cnt[t]++;
                    else
                        tile_splats[cnt[t]++] = (int32_t)k;
                }
        }
    }
    free(cnt);
    free(bb);
    view_free(&v);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* SH recompute: compaction.py:89-243                                         */

static const double RGB_TO_YCOCG[9] = {0.25, 0.5, 0.25, 0.5, 0.0, -0.5, -0.25, 0.5, -0.25};
static const double YCOCG_TO_RGB[9] = {1.0, 1.0, -1.0, 1.0, 0.0, 1.0, 1.0, -1.0, -1.0};

/* (3,16) block conversion: compaction.py:80-86 (einsum "ij,...jc->...ic") */
static void coeffs_convert(const double *M, const double *in, double *out) {
    for (int i = 0; i < 3; i++)
        for (int c = 0; c < 16; c++) {
            double acc = 0.0;
            for (int j = 0; j < 3; j++) acc += M[i * 3 + j] * in[j * 16 + c];
            out[i * 16 + c] = acc;
        }
}

/* Upper Cholesky A = U^T U of an m x m matrix (row-major, stride 16), in place.
 * LAPACK dpotrf semantics: fails when a pivot is <= 0 or NaN. */
static int chol_upper(double *A, int m) {
    for (int j = 0; j < m; j++) {
        double ajj = A[j * 16 + j];
        for (int k = 0; k < j; k++) ajj -= A[k * 16 + j] * A[k * 16 + j];
        if (!(ajj > 0.0)) return j + 1;
        ajj = sqrt(ajj);
        A[j * 16 + j] = ajj;
        for (int c = j + 1; c < m; c++) {
            double v = A[j * 16 + c];
            for (int k = 0; k < j; k++) v -= A[k * 16 + j] * A[k * 16 + c];
            A[j * 16 + c] = v / ajj;
        }
    }
    return 0;
}

/* dpotrs: U^T y = b, U x = y */
static void chol_solve_upper(const double *U, int m, double *b) {
    for (int i = 0; i < m; i++) {
        double v = b[i];
        for (int k = 0; k < i; k++) v -= U[k * 16 + i] * b[k];
        b[i] = v / U[i * 16 + i];
    }
    for (int i = m - 1; i >= 0; i--) {
        double v = b[i];
        for (int k = i + 1; k < m; k++) v -= U[i * 16 + k] * b[k];
        b[i] = v / U[i * 16 + i];
    }
}

/* _solve_channel (compaction.py:127-148).  Y: (ns,16) weighted basis rows;
 * c: (ns) weighted channel values.  Returns 0 ok, 1 ok after jitter, -1 fail. */
static int solve_channel(const double *Y, const double *c, int ns, const int *mask, double lam,
                         double *out) {
    int cols[16], m = 0;
    for (int i = 0; i < 16; i++)
        if (mask[i]) cols[m++] = i;
    double A[256] = {0}, Asave[256], b[16];
    for (int i = 0; i < m; i++) {
        for (int j = 0; j < m; j++) {
            double acc = 0.0;
            for (int s = 0; s < ns; s++) acc = fma(Y[s * 16 + cols[i]], Y[s * 16 + cols[j]], acc);
            A[i * 16 + j] = acc;
        }
        double acc = 0.0;
        for (int s = 0; s < ns; s++) acc = fma(Y[s * 16 + cols[i]], c[s], acc);
        b[i] = acc;
    }
    for (int i = 0; i < m; i++) A[i * 16 + i] += (cols[i] == 0) ? 0.0 : lam;
    memcpy(Asave, A, sizeof(A));
    int status = 0;
    if (chol_upper(A, m)) {
        memcpy(A, Asave, sizeof(A));
        for (int i = 0; i < m; i++) A[i * 16 + i] += 1e-10;
        if (chol_upper(A, m)) return -1;
        status = 1;
    }
    chol_solve_upper(A, m, b);
    for (int i = 0; i < 16; i++) out[i] = 0.0;
    for (int i = 0; i < m; i++) out[cols[i]] = b[i];
    return status;
}

/* _PROBES (compaction.py:32-37) and _fallback_dc (:161-166) */
static void fallback_dc(const double *sh, double *rgb, double *ycocg) {
    double acc[3] = {0.0, 0.0, 0.0};
    for (int i = -1; i <= 1; i++)
        for (int j = -1; j <= 1; j++)
            for (int k = -1; k <= 1; k++) {
                if (i == 0 && j == 0 && k == 0) continue;
                double nrm = sqrt((double)(i * i) + (double)(j * j) + (double)(k * k));
                double basis[16];
                sh_basis16(i / nrm, j / nrm, k / nrm, basis);
                for (int ch = 0; ch < 3; ch++) {
                    double col = 0.0;
                    for (int q = 0; q < 16; q++) col += basis[q] * sh[ch * 16 + q];
                    acc[ch] += col;
                }
            }
    memset(rgb, 0, sizeof(double) * 48);
    for (int ch = 0; ch < 3; ch++) rgb[ch * 16] = acc[ch] / 26.0 / SH_DC;
    coeffs_convert(RGB_TO_YCOCG, rgb, ycocg);
}

/* compact_splat (compaction.py:169-192).  w: (S) per-camera importances of
 * this splat.  status: 0 ok, 1 jitter used, 2 failed (RidgeError), 3 DC
 * fallback (no camera sees it). */
static int compact_one(const double *p, const double *sh, int ncam, const ocam *cams,
                       const double *w, double lambda_y, double par_thr, double zero_thr,
                       double *rgb, double *ycocg, double *Ybuf, double *Cbuf) {
    int ns = 0;
    for (int s = 0; s < ncam; s++) {
        if (!(w[s] > 0.0)) continue;
        double d0 = p[0] - cams[s].eye[0], d1 = p[1] - cams[s].eye[1], d2 = p[2] - cams[s].eye[2];
        double nrm = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
        double basis[16];
        sh_basis16(d0 / nrm, d1 / nrm, d2 / nrm, basis);
        /* colors = basis @ sh^T (compaction.py:104, a BLAS product in the
         * reference): fused multiply-adds in two interleaved partial sums
         * (even / odd coefficients), the order the device uses */
        double col[3];
        for (int ch = 0; ch < 3; ch++) {
            double a0 = 0.0, a1 = 0.0;
            for (int i = 0; i < 16; i += 2) {
                a0 = fma(basis[i], sh[ch * 16 + i], a0);
                a1 = fma(basis[i + 1], sh[ch * 16 + i + 1], a1);
            }
            col[ch] = a0 + a1;
        }
        for (int i = 0; i < 16; i++) Ybuf[ns * 16 + i] = basis[i] * w[s];
        for (int ch = 0; ch < 3; ch++) {
            double y = col[0] * RGB_TO_YCOCG[ch * 3] + col[1] * RGB_TO_YCOCG[ch * 3 + 1] +
                       col[2] * RGB_TO_YCOCG[ch * 3 + 2];
            Cbuf[ch * ncam + ns] = y * w[s];
        }
        ns++;
    }
    if (ns == 0) {
        fallback_dc(sh, rgb, ycocg);
        return 3;
    }
    /* sparsify_parallel_columns :110-124 */
    double gram[256], norms[16];
    for (int i = 0; i < 16; i++)
        for (int j = 0; j < 16; j++) {
            double acc = 0.0;
            for (int s = 0; s < ns; s++) acc = fma(Ybuf[s * 16 + i], Ybuf[s * 16 + j], acc);
            gram[i * 16 + j] = acc;
        }
    for (int i = 0; i < 16; i++) norms[i] = sqrt(gram[i * 16 + i]);
    int mask[16] = {0};
    mask[0] = 1;
    for (int i = 1; i < 16; i++) {
        if (norms[i] == 0.0) continue;
        int par = 0;
        for (int j = 0; j < 16; j++) {
            if (!mask[j]) continue;
            double cs = fabs(gram[i * 16 + j]) / (norms[i] * norms[j]);
            if (cs > par_thr) par = 1;
        }
        if (!par) mask[i] = 1;
    }
    double lam[3] = {lambda_y, 3.0 * lambda_y, 3.0 * lambda_y};
    int status = 0;
    double yc[48];
    for (int ch = 0; ch < 3; ch++) {
        double first[16];
        int rc = solve_channel(Ybuf, Cbuf + ch * ncam, ns, mask, lam[ch], first);
        if (rc < 0) return 2;
        if (rc > 0) status = 1;
        int m2[16];
        for (int i = 0; i < 16; i++) m2[i] = mask[i] && !(i > 0 && fabs(first[i]) < zero_thr);
        rc = solve_channel(Ybuf, Cbuf + ch * ncam, ns, m2, lam[ch], yc + ch * 16);
        if (rc < 0) return 2;
        if (rc > 0) status = 1;
    }
    memcpy(ycocg, yc, sizeof(yc));
    coeffs_convert(YCOCG_TO_RGB, yc, rgb);
    return status;
}

/* compact_scene (compaction.py:195-243).  camera_importance: (ncam, n).
 * Outputs rgb/ycocg (n,3,16); failed splats keep their original coefficients
 * (rgb = sh, ycocg = RGB->YCoCg(sh)).  status per splat as compact_one. */
typedef struct {
    int64_t n;
    const double *pos, *sh;
    int ncam;
    const ocam *cams;
    const double *cam_imp;
    double lambda_y, par_thr, zero_thr;
    double *out_rgb, *out_ycocg;
    int8_t *status;
    int64_t chunk;
    volatile int err;
} cp_ctx;

static void cp_item(void *vctx, int64_t blk, int worker) {
    (void)worker;
    cp_ctx *c = (cp_ctx *)vctx;
    int ncam = c->ncam;
    double *Y = (double *)malloc(sizeof(double) * 16 * (size_t)(ncam > 0 ? ncam : 1));
    double *C = (double *)malloc(sizeof(double) * 3 * (size_t)(ncam > 0 ? ncam : 1));
    double *w = (double *)malloc(sizeof(double) * (size_t)(ncam > 0 ? ncam : 1));
    if (!Y || !C || !w) {
        c->err = 1;
    } else {
        int64_t lo = blk * c->chunk, hi = lo + c->chunk < c->n ? lo + c->chunk : c->n;
        for (int64_t k = lo; k < hi; k++) {
            for (int s = 0; s < ncam; s++) w[s] = c->cam_imp[(int64_t)s * c->n + k];
            double rgb[48], yc[48];
            int st = compact_one(c->pos + 3 * k, c->sh + 48 * k, ncam, c->cams, w, c->lambda_y,
                                 c->par_thr, c->zero_thr, rgb, yc, Y, C);
            c->status[k] = (int8_t)st;
            if (st == 2) {
                memcpy(rgb, c->sh + 48 * k, sizeof(rgb));
                coeffs_convert(RGB_TO_YCOCG, rgb, yc);
            }
            memcpy(c->out_rgb + 48 * k, rgb, sizeof(rgb));
            memcpy(c->out_ycocg + 48 * k, yc, sizeof(yc));
        }
    }
    free(Y);
    free(C);
    free(w);
}

/* compact_scene (compaction.py:195-243).  camera_importance: (ncam, n).
 * Outputs rgb/ycocg (n,3,16); failed splats keep their original coefficients
 * (rgb = sh, ycocg = RGB->YCoCg(sh)).  status per splat as compact_one. */
int oracle_compact(int64_t n, const double *pos, const double *sh, int ncam, const ocam *cams,
                   const double *camera_importance, double lambda_y, double par_thr,
                   double zero_thr, int threads, double *out_rgb, double *out_ycocg,
                   int8_t *status) {
    cp_ctx c = {n, pos, sh, ncam, cams, camera_importance, lambda_y, par_thr, zero_thr,
                out_rgb, out_ycocg, status, 256, 0};
    parallel_for((n + c.chunk - 1) / c.chunk, threads, cp_item, &c);
    return c.err ? -1 : 0;
}

int oracle_num_threads(void) {
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}
