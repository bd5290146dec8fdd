/*
 * ts_oracle_kernels.c — TEST INFRASTRUCTURE ONLY (the CPU checker, never the product).
 *
 * Plain-C restatement of the per-pixel loops of the TeT-Splatting reference kernels
 * (/root/reference/pkg/src/tetsplat/kernels/_core.pyx).  Only tests/, bench.py's
 * cpu_baseline leg and __graft_entry__.smoke() may load this library.
 *
 * Arithmetic is FP64 throughout, evaluated in the reference's operation order and
 * compiled with -ffp-contract=off (gcc on x86-64 without -march emits no FMA, so the
 * reference build has none either).  Every function cites the lines it restates.
 *
 * Differences from the reference that do not change results:
 *  - the forward pass does not materialise per-pixel (idx, alpha) lists; the
 *    backward pass re-walks the identical deterministic forward sequence per pixel
 *    to regenerate them (same records, same order as _core.pyx:206-209);
 *  - threading is OpenMP over tiles / rows instead of a ThreadPoolExecutor
 *    (raster.py:168-175); the backward keeps private per-thread buffers that are
 *    summed in thread order, like raster.py:217-247.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EPS_DET 2e-12 /* _core.pyx:12 */

static const int FACES[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}}; /* _core.pyx:14-18 */

/* _core.pyx:21-26 */
static inline double sigmoid_(double x) {
    if (x >= 0) return 1.0 / (1.0 + exp(-x));
    double e = exp(x);
    return e / (1.0 + e);
}
/* _core.pyx:29-32 */
static inline double softplus_(double x) { return x > 30.0 ? x : log1p(exp(x)); }
/* _core.pyx:35-36 */
static inline double alpha_unclipped_(double fp, double fn, double s) {
    return 1.0 - exp(softplus_(-s * fp) - softplus_(-s * fn));
}

typedef struct {
    const double *proj, *depths, *f, *normals, *md, *colors, *bbox;
} scene_t;

/* _core.pyx:39-64 */
static inline int face_hit_(const scene_t *S, int64_t k, int fi, double px, double py,
                            double *zp_out, double *f_out) {
    int ia = FACES[fi][0], ib = FACES[fi][1], ic = FACES[fi][2];
    const double *P = S->proj + k * 8;
    double ax = P[ia * 2], ay = P[ia * 2 + 1];
    double m00 = P[ib * 2] - ax, m10 = P[ib * 2 + 1] - ay;
    double m01 = P[ic * 2] - ax, m11 = P[ic * 2 + 1] - ay;
    double det = m00 * m11 - m01 * m10;
    if (fabs(det) < EPS_DET) return 0;
    double rx = px - ax, ry = py - ay;
    double u = (m11 * rx - m01 * ry) / det;
    double v = (-m10 * rx + m00 * ry) / det;
    if (u < 0.0 || v < 0.0 || u + v > 1.0) return 0;
    const double *Z = S->depths + k * 4, *F = S->f + k * 4;
    double za = Z[ia], zb = Z[ib], zc = Z[ic];
    double w0 = (1.0 - u - v) / za, w1 = u / zb, w2 = v / zc;
    double Ssum = w0 + w1 + w2;
    *f_out = (w0 * F[ia] + w1 * F[ib] + w2 * F[ic]) / Ssum;
    *zp_out = 1.0 / Ssum;
    return 1;
}

/* _core.pyx:67-95 */
static inline int splat_hits_(const scene_t *S, int64_t k, double px, double py, double *f_prev,
                              double *f_next, int *fi_prev, int *fi_next) {
    const double *B = S->bbox + k * 4;
    if (px < B[0] || px > B[2] || py < B[1] || py > B[3]) return 0;
    double z_lo = 0, z_hi = 0, f_lo = 0, f_hi = 0, zp, fh;
    int n = 0, lo_fi = -1, hi_fi = -1;
    for (int fi = 0; fi < 4; fi++) {
        if (!face_hit_(S, k, fi, px, py, &zp, &fh)) continue;
        if (n == 0) {
            z_lo = zp; z_hi = zp; f_lo = fh; f_hi = fh; lo_fi = fi; hi_fi = fi;
        } else {
            if (zp < z_lo) { z_lo = zp; f_lo = fh; lo_fi = fi; }
            if (zp > z_hi) { z_hi = zp; f_hi = fh; hi_fi = fi; }
        }
        n++;
    }
    if (n < 2) return 0;
    *f_prev = f_lo; *f_next = f_hi; *fi_prev = lo_fi; *fi_next = hi_fi;
    return 1;
}

/* One pixel of forward_tiles (_core.pyx:158-229): window pops, hit, blend, early stop.
 * rec_idx/rec_alpha (capacity L) receive the blended records when non-NULL. */
static int pixel_forward_(const scene_t *S, const int64_t *list, int64_t L, int n_w, double s,
                          double t_stop, double alpha_clip, double px, double py, int has_color,
                          double acc[8], int64_t *rec_idx, double *rec_alpha, int64_t *widx,
                          double *wz) {
    int wcount = 0, n_blend = 0;
    int64_t pos = 0;
    double T = 1.0;
    for (int c = 0; c < 8; c++) acc[c] = 0.0;
    for (;;) {
        while (wcount < n_w && pos < L) { /* _core.pyx:171-174 */
            widx[wcount] = list[pos];
            wz[wcount] = S->md[list[pos]];
            wcount++; pos++;
        }
        if (wcount == 0) break;
        int m = 0; /* strict-< argmin, first index wins: _core.pyx:177-180 */
        for (int i = 1; i < wcount; i++)
            if (wz[i] < wz[m]) m = i;
        int64_t k = widx[m];
        for (int i = m; i < wcount - 1; i++) { widx[i] = widx[i + 1]; wz[i] = wz[i + 1]; }
        wcount--;
        double fp, fn, a;
        int fip, fin;
        if (!splat_hits_(S, k, px, py, &fp, &fn, &fip, &fin)) continue;
        a = alpha_unclipped_(fp, fn, s);
        if (a <= 0.0) continue; /* _core.pyx:193 */
        if (a > alpha_clip) a = alpha_clip;
        acc[0] += T * a;
        acc[1] += T * a * S->md[k];
        acc[2] += T * a * S->normals[k * 3 + 0];
        acc[3] += T * a * S->normals[k * 3 + 1];
        acc[4] += T * a * S->normals[k * 3 + 2];
        if (has_color) {
            acc[5] += T * a * S->colors[k * 3 + 0];
            acc[6] += T * a * S->colors[k * 3 + 1];
            acc[7] += T * a * S->colors[k * 3 + 2];
        }
        if (rec_idx) { rec_idx[n_blend] = k; rec_alpha[n_blend] = a; }
        n_blend++;
        T *= 1.0 - a;
        if (T < t_stop) break; /* _core.pyx:211-213 */
    }
    return n_blend;
}

/* forward_tiles over every touched tile (_core.pyx:98-229, raster.py:149-177).
 * Maps are written for touched tiles only (caller zero-fills).  counts (H*W int32,
 * nullable) receives the per-pixel number of blended records (_core.pyx:227-228). */
int or_forward(const double *proj, const double *depths, const double *f, const double *normals,
               const double *md, const double *colors, const double *bbox, const int64_t *starts,
               const int64_t *items, int tile_size, int tiles_x, int tiles_y, int width,
               int height, int n_w, double s, double t_stop, double alpha_clip,
               double *normal_map, double *depth_map, double *opacity_map, double *color_map,
               int32_t *counts, int nthreads) {
    scene_t S = {proj, depths, f, normals, md, colors, bbox};
    int has_color = colors != NULL && color_map != NULL;
    int64_t T = (int64_t)tiles_x * tiles_y;
    if (n_w < 1) return -1;
#pragma omp parallel num_threads(nthreads > 0 ? nthreads : 1)
    {
        int64_t *widx = (int64_t *)malloc(sizeof(int64_t) * n_w);
        double *wz = (double *)malloc(sizeof(double) * n_w);
#pragma omp for schedule(dynamic, 1)
        for (int64_t tid = 0; tid < T; tid++) {
            int64_t lo = starts[tid], L = starts[tid + 1] - lo;
            if (L <= 0) continue;
            int x0 = (int)(tid % tiles_x) * tile_size, y0 = (int)(tid / tiles_x) * tile_size;
            for (int local = 0; local < tile_size * tile_size; local++) {
                int xi = x0 + local % tile_size, yi = y0 + local / tile_size;
                if (xi >= width || yi >= height) continue;
                double acc[8];
                int nb = pixel_forward_(&S, items + lo, L, n_w, s, t_stop, alpha_clip, xi + 0.5,
                                        yi + 0.5, has_color, acc, NULL, NULL, widx, wz);
                int64_t p = (int64_t)yi * width + xi;
                opacity_map[p] = acc[0];
                depth_map[p] = acc[1];
                normal_map[p * 3 + 0] = acc[2];
                normal_map[p * 3 + 1] = acc[3];
                normal_map[p * 3 + 2] = acc[4];
                if (has_color) {
                    color_map[p * 3 + 0] = acc[5];
                    color_map[p * 3 + 1] = acc[6];
                    color_map[p * 3 + 2] = acc[7];
                }
                if (counts) counts[p] = nb;
            }
        }
        free(widx);
        free(wz);
    }
    return 0;
}

/* reference_render (_core.pyx:232-292): exact mean-depth order (lexsort with the
 * splat index as tie-break, passed in as `order`), no tiles, no window, no early stop. */
int or_reference_render(const double *proj, const double *depths, const double *f,
                        const double *normals, const double *md, const double *colors,
                        const double *bbox, int64_t K, const int64_t *order, int width, int height,
                        double s, double alpha_clip, double *normal_map, double *depth_map,
                        double *opacity_map, double *color_map, int nthreads) {
    scene_t S = {proj, depths, f, normals, md, colors, bbox};
    int has_color = colors != NULL && color_map != NULL;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
    for (int yi = 0; yi < height; yi++) {
        double py = yi + 0.5;
        for (int xi = 0; xi < width; xi++) {
            double px = xi + 0.5, T = 1.0, acc[8] = {0};
            for (int64_t oi = 0; oi < K; oi++) {
                int64_t k = order[oi];
                double fp, fn, a;
                int fip, fin;
                if (!splat_hits_(&S, k, px, py, &fp, &fn, &fip, &fin)) continue;
                a = alpha_unclipped_(fp, fn, s);
                if (a <= 0.0) continue;
                if (a > alpha_clip) a = alpha_clip;
                acc[0] += T * a;
                acc[1] += T * a * md[k];
                acc[2] += T * a * normals[k * 3 + 0];
                acc[3] += T * a * normals[k * 3 + 1];
                acc[4] += T * a * normals[k * 3 + 2];
                if (has_color) {
                    acc[5] += T * a * colors[k * 3 + 0];
                    acc[6] += T * a * colors[k * 3 + 1];
                    acc[7] += T * a * colors[k * 3 + 2];
                }
                T *= 1.0 - a;
            }
            int64_t p = (int64_t)yi * width + xi;
            opacity_map[p] = acc[0];
            depth_map[p] = acc[1];
            for (int c = 0; c < 3; c++) normal_map[p * 3 + c] = acc[2 + c];
            if (has_color)
                for (int c = 0; c < 3; c++) color_map[p * 3 + c] = acc[5 + c];
        }
    }
    return 0;
}

typedef struct {
    double *d_f, *d_proj, *d_depths, *d_normals, *d_md, *d_colors;
} grads_t;

/* _core.pyx:295-341 */
static inline void face_hit_backward_(const scene_t *S, int64_t k, int fi, double px, double py,
                                      double g, grads_t *G) {
    int ia = FACES[fi][0], ib = FACES[fi][1], ic = FACES[fi][2];
    const double *P = S->proj + k * 8, *Z = S->depths + k * 4, *F = S->f + k * 4;
    double ax = P[ia * 2], ay = P[ia * 2 + 1];
    double m00 = P[ib * 2] - ax, m10 = P[ib * 2 + 1] - ay;
    double m01 = P[ic * 2] - ax, m11 = P[ic * 2 + 1] - ay;
    double det = m00 * m11 - m01 * m10;
    double rx = px - ax, ry = py - ay;
    double u = (m11 * rx - m01 * ry) / det;
    double v = (-m10 * rx + m00 * ry) / det;
    double za = Z[ia], zb = Z[ib], zc = Z[ic];
    double w0 = (1.0 - u - v) / za, w1 = u / zb, w2 = v / zc;
    double Ssum = w0 + w1 + w2;
    double f_hit = (w0 * F[ia] + w1 * F[ib] + w2 * F[ic]) / Ssum;
    double *df = G->d_f + k * 4, *dz = G->d_depths + k * 4, *dp = G->d_proj + k * 8;
    df[ia] += g * w0 / Ssum;
    df[ib] += g * w1 / Ssum;
    df[ic] += g * w2 / Ssum;
    double dw0 = g * (F[ia] - f_hit) / Ssum;
    double dw1 = g * (F[ib] - f_hit) / Ssum;
    double dw2 = g * (F[ic] - f_hit) / Ssum;
    dz[ia] += dw0 * (-w0 / za);
    dz[ib] += dw1 * (-w1 / zb);
    dz[ic] += dw2 * (-w2 / zc);
    double gu = -dw0 / za + dw1 / zb;
    double gv = -dw0 / za + dw2 / zc;
    double qx = (m11 * gu - m10 * gv) / det;
    double qy = (-m01 * gu + m00 * gv) / det;
    dp[ia * 2] += -qx * (1.0 - u - v);
    dp[ia * 2 + 1] += -qy * (1.0 - u - v);
    dp[ib * 2] += -qx * u;
    dp[ib * 2 + 1] += -qy * u;
    dp[ic * 2] += -qx * v;
    dp[ic * 2 + 1] += -qy * v;
}

/* backward_tiles (_core.pyx:344-471) + the ordered merge of raster.py:217-247.
 * Per pixel the forward walk is replayed to regenerate the saved (idx, alpha) records
 * (same values, same order as _core.pyx:206-209), then walked back to front.
 * Gradient outputs are ACCUMULATED (+=), caller zero-fills. */
int or_backward(const double *proj, const double *depths, const double *f, const double *normals,
                const double *md, const double *colors, const double *bbox, int64_t K,
                const int64_t *starts, const int64_t *items, int tile_size, int tiles_x,
                int tiles_y, int width, int height, int n_w, double s, double t_stop,
                double alpha_clip, const double *d_normal_map, const double *d_depth_map,
                const double *d_opacity_map, const double *d_color_map, double *d_f,
                double *d_proj, double *d_depths, double *d_normals, double *d_md,
                double *d_colors, int nthreads) {
    scene_t S = {proj, depths, f, normals, md, colors, bbox};
    int has_color = colors != NULL && d_color_map != NULL && d_colors != NULL;
    int64_t T = (int64_t)tiles_x * tiles_y;
    int64_t maxL = 0;
    for (int64_t t = 0; t < T; t++)
        if (starts[t + 1] - starts[t] > maxL) maxL = starts[t + 1] - starts[t];
    if (nthreads < 1) nthreads = 1;
    /* static contiguous tile chunks per thread, private buffers, ordered merge */
    grads_t *priv = (grads_t *)calloc(nthreads, sizeof(grads_t));
    for (int t = 0; t < nthreads; t++) {
        priv[t].d_f = (double *)calloc(K * 4 + 1, sizeof(double));
        priv[t].d_proj = (double *)calloc(K * 8 + 1, sizeof(double));
        priv[t].d_depths = (double *)calloc(K * 4 + 1, sizeof(double));
        priv[t].d_normals = (double *)calloc(K * 3 + 1, sizeof(double));
        priv[t].d_md = (double *)calloc(K + 1, sizeof(double));
        priv[t].d_colors = (double *)calloc(K * 3 + 1, sizeof(double));
    }
#pragma omp parallel num_threads(nthreads)
    {
        int me = 0;
#ifdef _OPENMP
        me = omp_get_thread_num();
#endif
        grads_t *G = &priv[me];
        int64_t *widx = (int64_t *)malloc(sizeof(int64_t) * n_w);
        double *wz = (double *)malloc(sizeof(double) * n_w);
        int64_t *ridx = (int64_t *)malloc(sizeof(int64_t) * (maxL + 1));
        double *ral = (double *)malloc(sizeof(double) * (maxL + 1));
        double *Ts = (double *)malloc(sizeof(double) * (maxL + 1));
        int64_t per = (T + nthreads - 1) / nthreads;
        int64_t t0 = me * per, t1 = t0 + per < T ? t0 + per : T;
        for (int64_t tid = t0; tid < t1; tid++) {
            int64_t lo = starts[tid], L = starts[tid + 1] - lo;
            if (L <= 0) continue;
            int x0 = (int)(tid % tiles_x) * tile_size, y0 = (int)(tid / tiles_x) * tile_size;
            for (int local = 0; local < tile_size * tile_size; local++) {
                int xi = x0 + local % tile_size, yi = y0 + local / tile_size;
                if (xi >= width || yi >= height) continue;
                double px = xi + 0.5, py = yi + 0.5, acc[8];
                int m = pixel_forward_(&S, items + lo, L, n_w, s, t_stop, alpha_clip, px, py,
                                       has_color, acc, ridx, ral, widx, wz);
                if (m == 0) continue;
                int64_t p = (int64_t)yi * width + xi;
                double g_o = d_opacity_map[p], g_d = d_depth_map[p];
                double gn0 = d_normal_map[p * 3], gn1 = d_normal_map[p * 3 + 1],
                       gn2 = d_normal_map[p * 3 + 2];
                double gc0 = 0, gc1 = 0, gc2 = 0;
                if (has_color) {
                    gc0 = d_color_map[p * 3]; gc1 = d_color_map[p * 3 + 1]; gc2 = d_color_map[p * 3 + 2];
                }
                double Tt = 1.0; /* _core.pyx:415-418 */
                for (int i = 0; i < m; i++) { Ts[i] = Tt; Tt *= 1.0 - ral[i]; }
                double suf_o = 0, suf_d = 0, sn0 = 0, sn1 = 0, sn2 = 0, sc0 = 0, sc1 = 0, sc2 = 0;
                for (int i = m - 1; i >= 0; i--) { /* _core.pyx:423-471 */
                    int64_t k = ridx[i];
                    double a = ral[i], Ti = Ts[i], w = Ti * a, one_m = 1.0 - a;
                    const double *N = normals + k * 3;
                    G->d_md[k] += g_d * w;
                    G->d_normals[k * 3 + 0] += gn0 * w;
                    G->d_normals[k * 3 + 1] += gn1 * w;
                    G->d_normals[k * 3 + 2] += gn2 * w;
                    if (has_color) {
                        G->d_colors[k * 3 + 0] += gc0 * w;
                        G->d_colors[k * 3 + 1] += gc1 * w;
                        G->d_colors[k * 3 + 2] += gc2 * w;
                    }
                    double d_alpha = (g_o * (Ti - suf_o / one_m) + g_d * (Ti * md[k] - suf_d / one_m));
                    d_alpha += gn0 * (Ti * N[0] - sn0 / one_m);
                    d_alpha += gn1 * (Ti * N[1] - sn1 / one_m);
                    d_alpha += gn2 * (Ti * N[2] - sn2 / one_m);
                    if (has_color) {
                        const double *C = colors + k * 3;
                        d_alpha += gc0 * (Ti * C[0] - sc0 / one_m);
                        d_alpha += gc1 * (Ti * C[1] - sc1 / one_m);
                        d_alpha += gc2 * (Ti * C[2] - sc2 / one_m);
                    }
                    suf_o += w;
                    suf_d += w * md[k];
                    sn0 += w * N[0];
                    sn1 += w * N[1];
                    sn2 += w * N[2];
                    if (has_color) {
                        const double *C = colors + k * 3;
                        sc0 += w * C[0]; sc1 += w * C[1]; sc2 += w * C[2];
                    }
                    double fp, fn_, a_un;
                    int fip, fin;
                    if (!splat_hits_(&S, k, px, py, &fp, &fn_, &fip, &fin)) continue;
                    a_un = alpha_unclipped_(fp, fn_, s);
                    if (a_un <= 0.0 || a_un > alpha_clip) continue;
                    double ratio = 1.0 - a_un;
                    double da_dfp = s * ratio * sigmoid_(-s * fp);
                    double da_dfn = -s * ratio * sigmoid_(-s * fn_);
                    face_hit_backward_(&S, k, fip, px, py, d_alpha * da_dfp, G);
                    face_hit_backward_(&S, k, fin, px, py, d_alpha * da_dfn, G);
                }
            }
        }
        free(widx); free(wz); free(ridx); free(ral); free(Ts);
    }
    for (int t = 0; t < nthreads; t++) {
        for (int64_t i = 0; i < K * 4; i++) { d_f[i] += priv[t].d_f[i]; d_depths[i] += priv[t].d_depths[i]; }
        for (int64_t i = 0; i < K * 8; i++) d_proj[i] += priv[t].d_proj[i];
        for (int64_t i = 0; i < K * 3; i++) d_normals[i] += priv[t].d_normals[i];
        for (int64_t i = 0; i < K; i++) d_md[i] += priv[t].d_md[i];
        if (has_color)
            for (int64_t i = 0; i < K * 3; i++) d_colors[i] += priv[t].d_colors[i];
        free(priv[t].d_f); free(priv[t].d_proj); free(priv[t].d_depths);
        free(priv[t].d_normals); free(priv[t].d_md); free(priv[t].d_colors);
    }
    free(priv);
    return 0;
}

/* _core.pyx:474-514 */
static inline double tet_gradient_(const double *pos, const double *sdf, const int64_t *tet,
                                   double g[3], double c1[3], double c2[3], double c3[3]) {
    int64_t v0 = tet[0], v1 = tet[1], v2 = tet[2], v3 = tet[3];
    double e1x = pos[v1 * 3] - pos[v0 * 3], e1y = pos[v1 * 3 + 1] - pos[v0 * 3 + 1],
           e1z = pos[v1 * 3 + 2] - pos[v0 * 3 + 2];
    double e2x = pos[v2 * 3] - pos[v0 * 3], e2y = pos[v2 * 3 + 1] - pos[v0 * 3 + 1],
           e2z = pos[v2 * 3 + 2] - pos[v0 * 3 + 2];
    double e3x = pos[v3 * 3] - pos[v0 * 3], e3y = pos[v3 * 3 + 1] - pos[v0 * 3 + 1],
           e3z = pos[v3 * 3 + 2] - pos[v0 * 3 + 2];
    c1[0] = e2y * e3z - e2z * e3y; c1[1] = e2z * e3x - e2x * e3z; c1[2] = e2x * e3y - e2y * e3x;
    c2[0] = e3y * e1z - e3z * e1y; c2[1] = e3z * e1x - e3x * e1z; c2[2] = e3x * e1y - e3y * e1x;
    c3[0] = e1y * e2z - e1z * e2y; c3[1] = e1z * e2x - e1x * e2z; c3[2] = e1x * e2y - e1y * e2x;
    double det = e1x * c1[0] + e1y * c1[1] + e1z * c1[2];
    g[0] = g[1] = g[2] = 0.0;
    if (det != 0.0) {
        double df1 = sdf[v1] - sdf[v0], df2 = sdf[v2] - sdf[v0], df3 = sdf[v3] - sdf[v0];
        for (int c = 0; c < 3; c++) g[c] = (df1 * c1[c] + df2 * c2[c] + df3 * c3[c]) / det;
    }
    return det;
}

/* _core.pyx:517-541 */
static inline void chain_dg_(const int64_t *tet, double det, const double g[3], const double c1[3],
                             const double c2[3], const double c3[3], const double d_g[3],
                             double *d_sdf, double *d_deform) {
    if (det == 0.0) return;
    double d1 = (c1[0] * d_g[0] + c1[1] * d_g[1] + c1[2] * d_g[2]) / det;
    double d2 = (c2[0] * d_g[0] + c2[1] * d_g[1] + c2[2] * d_g[2]) / det;
    double d3 = (c3[0] * d_g[0] + c3[1] * d_g[1] + c3[2] * d_g[2]) / det;
    double dfs[4] = {-(d1 + d2 + d3), d1, d2, d3};
    for (int c = 0; c < 4; c++) {
        int64_t v = tet[c];
        d_sdf[v] += dfs[c];
        d_deform[v * 3 + 0] -= dfs[c] * g[0];
        d_deform[v * 3 + 1] -= dfs[c] * g[1];
        d_deform[v * 3 + 2] -= dfs[c] * g[2];
    }
}

/* eikonal_kernel (_core.pyx:544-568) */
double or_eikonal(const double *pos, const double *sdf, const int64_t *tets, const int64_t *tet_set,
                  int64_t n_set, double eps_normal, double *d_sdf, double *d_deform) {
    double loss = 0.0, g[3], c1[3], c2[3], c3[3], d_g[3];
    for (int64_t i = 0; i < n_set; i++) {
        const int64_t *tet = tets + tet_set[i] * 4;
        double det = tet_gradient_(pos, sdf, tet, g, c1, c2, c3);
        double norm = pow(g[0] * g[0] + g[1] * g[1] + g[2] * g[2], 0.5);
        loss += (norm - 1.0) * (norm - 1.0);
        if (norm > eps_normal) {
            double w = 2.0 * (norm - 1.0) / norm;
            d_g[0] = w * g[0]; d_g[1] = w * g[1]; d_g[2] = w * g[2];
            chain_dg_(tet, det, g, c1, c2, c3, d_g, d_sdf, d_deform);
        }
    }
    return loss;
}

/* normal_consistency_kernel (_core.pyx:571-668) */
double or_normal_consistency(const double *pos, const double *sdf, int64_t N, const int64_t *tets,
                             int64_t K, const int64_t *edges, int64_t E, double eps_normal,
                             double *d_sdf, double *d_deform) {
    double *n_t = (double *)calloc(K * 3, sizeof(double));
    double *gnorm = (double *)calloc(K, sizeof(double));
    double *counts = (double *)calloc(N, sizeof(double));
    double *n_v = (double *)calloc(N * 3, sizeof(double));
    double *anorm = (double *)calloc(N, sizeof(double));
    double *d_nv = (double *)calloc(N * 3, sizeof(double));
    double loss = 0.0, g[3], c1[3], c2[3], c3[3], d_g[3], d_nt[3];
    for (int64_t k = 0; k < K; k++) { /* :603-617 */
        tet_gradient_(pos, sdf, tets + k * 4, g, c1, c2, c3);
        double norm = pow(g[0] * g[0] + g[1] * g[1] + g[2] * g[2], 0.5);
        gnorm[k] = norm;
        if (norm < eps_normal) continue;
        for (int c = 0; c < 3; c++) n_t[k * 3 + c] = g[c] / norm;
        for (int c = 0; c < 4; c++) {
            int64_t v = tets[k * 4 + c];
            counts[v] += 1.0;
            for (int d = 0; d < 3; d++) n_v[v * 3 + d] += n_t[k * 3 + d];
        }
    }
    for (int64_t v = 0; v < N; v++) { /* :618-629 */
        if (counts[v] == 0.0) continue;
        for (int d = 0; d < 3; d++) n_v[v * 3 + d] /= counts[v];
        double an = pow(pow(n_v[v * 3], 2) + pow(n_v[v * 3 + 1], 2) + pow(n_v[v * 3 + 2], 2), 0.5);
        if (an < eps_normal) continue;
        anorm[v] = an;
        for (int d = 0; d < 3; d++) n_v[v * 3 + d] /= an;
    }
    for (int64_t e = 0; e < E; e++) { /* :631-640 */
        int64_t a = edges[e * 2], b = edges[e * 2 + 1];
        if (anorm[a] == 0.0 || anorm[b] == 0.0) continue;
        loss += 1.0 - (n_v[a * 3] * n_v[b * 3] + n_v[a * 3 + 1] * n_v[b * 3 + 1] +
                       n_v[a * 3 + 2] * n_v[b * 3 + 2]);
        for (int c = 0; c < 3; c++) {
            d_nv[a * 3 + c] -= n_v[b * 3 + c];
            d_nv[b * 3 + c] -= n_v[a * 3 + c];
        }
    }
    for (int64_t v = 0; v < N; v++) { /* :642-649 */
        if (anorm[v] == 0.0) continue;
        double dot = n_v[v * 3] * d_nv[v * 3] + n_v[v * 3 + 1] * d_nv[v * 3 + 1] +
                     n_v[v * 3 + 2] * d_nv[v * 3 + 2];
        for (int c = 0; c < 3; c++) d_nv[v * 3 + c] = (d_nv[v * 3 + c] - n_v[v * 3 + c] * dot) / anorm[v];
    }
    for (int64_t k = 0; k < K; k++) { /* :651-667 */
        if (gnorm[k] < eps_normal) continue;
        d_nt[0] = d_nt[1] = d_nt[2] = 0.0;
        for (int c = 0; c < 4; c++) {
            int64_t v = tets[k * 4 + c];
            double inv = 1.0 / counts[v];
            for (int d = 0; d < 3; d++) d_nt[d] += d_nv[v * 3 + d] * inv;
        }
        const double *nt = n_t + k * 3;
        double dot = nt[0] * d_nt[0] + nt[1] * d_nt[1] + nt[2] * d_nt[2];
        for (int d = 0; d < 3; d++) d_g[d] = (d_nt[d] - nt[d] * dot) / gnorm[k];
        double det = tet_gradient_(pos, sdf, tets + k * 4, g, c1, c2, c3);
        chain_dg_(tets + k * 4, det, g, c1, c2, c3, d_g, d_sdf, d_deform);
    }
    free(n_t); free(gnorm); free(counts); free(n_v); free(anorm); free(d_nv);
    return loss;
}
