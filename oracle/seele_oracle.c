/*
 * seele_oracle.c -- CPU fp64 restatement of the Seele reference render hot
 * path.  TEST INFRASTRUCTURE ONLY: this file is the checker that the CUDA
 * path is compared against.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.  The product
 * path (paper_2503_05168_b200) never links or calls it.
 *
 * Parity pinning: tests/golden/ holds vectors produced by running the
 * reference Python package (/root/reference/pkg/src/seele) in the build
 * container (script: tests/golden/make_golden.py).  tests/test_oracle.py
 * checks this restatement against them (discrete outputs bit-exact, floats
 * to 1e-9).
 *
 * Every function cites the reference file:line it restates (paths relative
 * to /root/reference/pkg/src/seele/).  Arithmetic follows the reference's
 * operation order in fp64 and is compiled with -ffp-contract=off, so the
 * only differences from numpy are ulp-level (numpy small matmuls go through
 * OpenBLAS with FMA; np.exp is a SIMD exp).  Discrete outputs (reject
 * reasons, tile rects, sort order, ranges, contributor counts, cost
 * counters) are therefore reproduced with probability ~1.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OC_TILE 16
#define OC_WARP 32

typedef struct {
    double position[3];
    double orientation[4]; /* camera-to-world, (w,x,y,z), already normalised (model.py:150-155) */
    double fov_x, fov_y;
    double near_clip;
    int32_t width, height;
} oc_camera;

typedef struct {
    int32_t engine;   /* 0 = "ref", 1 = "cr"  (render.py:28) */
    int32_t group_w;  /* 1, 2 or 4            (render.py:48-49) */
    int32_t sh_degree;
    int32_t opacity_aware;
    double alpha_theta;
    double gamma_threshold;
    double background[3];
} oc_config;

/* model.py:24-41 */
static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

/* model.py:83-93 quaternion_to_matrix, (w,x,y,z) */
static void quat_to_mat(const double q[4], double r[3][3]) {
    double w = q[0], x = q[1], y = q[2], z = q[3];
    r[0][0] = 1 - 2 * (y * y + z * z);
    r[0][1] = 2 * (x * y - w * z);
    r[0][2] = 2 * (x * z + w * y);
    r[1][0] = 2 * (x * y + w * z);
    r[1][1] = 1 - 2 * (x * x + z * z);
    r[1][2] = 2 * (y * z - w * x);
    r[2][0] = 2 * (x * z - w * y);
    r[2][1] = 2 * (y * z + w * x);
    r[2][2] = 1 - 2 * (x * x + y * y);
}

/* model.py:264-305 sh_to_color (one channel) */
static double sh_channel(const double *s, double x, double y, double z, int degree) {
    double c = SH_C0 * s[0];
    if (degree >= 1) {
        c = c - SH_C1 * y * s[1] + SH_C1 * z * s[2] - SH_C1 * x * s[3];
    }
    if (degree >= 2) {
        double xx = x * x, yy = y * y, zz = z * z;
        double xy = x * y, yz = y * z, xz = x * z;
        c = c + SH_C2[0] * xy * s[4] + SH_C2[1] * yz * s[5] + SH_C2[2] * (2.0 * zz - xx - yy) * s[6] +
            SH_C2[3] * xz * s[7] + SH_C2[4] * (xx - yy) * s[8];
        if (degree >= 3) {
            c = c + SH_C3[0] * y * (3.0 * xx - yy) * s[9] + SH_C3[1] * xy * z * s[10] +
                SH_C3[2] * y * (4.0 * zz - xx - yy) * s[11] +
                SH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy) * s[12] +
                SH_C3[4] * x * (4.0 * zz - xx - yy) * s[13] + SH_C3[5] * z * (xx - yy) * s[14] +
                SH_C3[6] * x * (xx - 3.0 * yy) * s[15];
        }
    }
    c = c + 0.5;
    return c > 0.0 ? c : 0.0;
}

/* preprocess.py:149-156 _axis_range: inclusive tile interval [first, last]; first > last = empty */
static void axis_range(double lo, double hi, int n_tiles, int32_t *first_out, int32_t *last_out) {
    double first = floor(lo / OC_TILE);
    if (first * OC_TILE == lo) first -= 1.0;
    double last = floor(hi / OC_TILE);
    if (first < 0.0) first = 0.0;
    if (last > (double)(n_tiles - 1)) last = (double)(n_tiles - 1);
    if (first > last) {
        *first_out = 1;
        *last_out = 0;
    } else {
        *first_out = (int32_t)first;
        *last_out = (int32_t)last;
    }
}

/*
 * Per-Gaussian preprocessing: plan_frame's loop body (render.py:94-108) ->
 * Gaussian3D rotation normalisation (model.py:122, 76-80) -> project_detailed
 * (preprocess.py:89-146) -> bin_tiles rectangle (preprocess.py:159-189).
 * status: 0 ok, 1 near-culled, 2 degenerate.  rect = (tx0, tx1, ty0, ty1)
 * inclusive; tx0 > tx1 or ty0 > ty1 means no tiles.
 */
void oracle_preprocess(int64_t n, const double *pos, const double *log_scale, const double *rot,
                       const double *opac, const double *sh, const oc_camera *cam,
                       const oc_config *cfg, int8_t *status, double *mean2d, double *conic,
                       double *depth, double *color, double *r2_out, int32_t *rect) {
    double rc[3][3];
    quat_to_mat(cam->orientation, rc);
    /* world_to_view = rc^T (preprocess.py:99) */
    double w2v[3][3];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) w2v[i][j] = rc[j][i];
    /* model.py:178-184 */
    double fx = cam->width / (2.0 * tan(cam->fov_x / 2.0));
    double fy = cam->height / (2.0 * tan(cam->fov_y / 2.0));
    double cx = cam->width / 2.0, cy = cam->height / 2.0;
    int tiles_x = (cam->width + OC_TILE - 1) / OC_TILE;
    int tiles_y = (cam->height + OC_TILE - 1) / OC_TILE;

#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        const double *p = pos + 3 * i;
        double d[3] = {p[0] - cam->position[0], p[1] - cam->position[1], p[2] - cam->position[2]};
        double t[3];
        /* world_to_view @ (position - cam.position) (preprocess.py:100): numpy hands this 3x3 @ 3 product
         * to OpenBLAS dgemv, whose kernel on this container accumulates with fused multiply-adds left to
         * right -- t[r] = fma(w[r][2], d[2], fma(w[r][1], d[1], w[r][0] d[0])) matches numpy bit for bit
         * on every tested splat (tools/blas_order.py), the plain sum does not for ~25 % of them.  The depth
         * feeds the sort, where one ulp decides near-ties (fp32 container positions make them common). */
        for (int r = 0; r < 3; r++) t[r] = fma(w2v[r][2], d[2], fma(w2v[r][1], d[1], w2v[r][0] * d[0]));
        double z = t[2];
        rect[4 * i + 0] = 1;
        rect[4 * i + 1] = 0;
        rect[4 * i + 2] = 1;
        rect[4 * i + 3] = 0;
        if (z <= cam->near_clip) { /* preprocess.py:101-103 */
            status[i] = 1;
            continue;
        }
        double m0 = fx * t[0] / z + cx; /* preprocess.py:107 */
        double m1 = fy * t[1] / z + cy;
        double jac[2][3] = {{fx / z, 0.0, -fx * t[0] / (z * z)}, {0.0, fy / z, -fy * t[1] / (z * z)}};
        double jw[2][3];
        for (int r = 0; r < 2; r++)
            for (int c = 0; c < 3; c++)
                jw[r][c] = jac[r][0] * w2v[0][c] + jac[r][1] * w2v[1][c] + jac[r][2] * w2v[2][c];
        /* Gaussian3D normalises the rotation (model.py:122, 76-80) */
        const double *qr = rot + 4 * i;
        double qn = sqrt(qr[0] * qr[0] + qr[1] * qr[1] + qr[2] * qr[2] + qr[3] * qr[3]);
        double q[4] = {qr[0] / qn, qr[1] / qn, qr[2] / qn, qr[3] / qn};
        /* covariance3d (model.py:256-261) */
        double rg[3][3], m[3][3], cv[3][3], cov[3][3];
        quat_to_mat(q, rg);
        double es[3] = {exp(log_scale[3 * i]), exp(log_scale[3 * i + 1]), exp(log_scale[3 * i + 2])};
        for (int r = 0; r < 3; r++)
            for (int c = 0; c < 3; c++) m[r][c] = rg[r][c] * es[c];
        for (int r = 0; r < 3; r++)
            for (int c = 0; c < 3; c++) cv[r][c] = m[r][0] * m[c][0] + m[r][1] * m[c][1] + m[r][2] * m[c][2];
        for (int r = 0; r < 3; r++)
            for (int c = 0; c < 3; c++) cov[r][c] = 0.5 * (cv[r][c] + cv[c][r]);
        /* cov2d = jw cov jw^T + 0.3 I, symmetrised (preprocess.py:116-121) */
        double tmp[2][3], c2[2][2], s2[2][2];
        for (int r = 0; r < 2; r++)
            for (int c = 0; c < 3; c++)
                tmp[r][c] = jw[r][0] * cov[0][c] + jw[r][1] * cov[1][c] + jw[r][2] * cov[2][c];
        for (int r = 0; r < 2; r++)
            for (int c = 0; c < 2; c++)
                c2[r][c] = tmp[r][0] * jw[c][0] + tmp[r][1] * jw[c][1] + tmp[r][2] * jw[c][2];
        c2[0][0] += 0.3;
        c2[1][1] += 0.3;
        for (int r = 0; r < 2; r++)
            for (int c = 0; c < 2; c++) s2[r][c] = 0.5 * (c2[r][c] + c2[c][r]);
        double det = s2[0][0] * s2[1][1] - s2[0][1] * s2[1][0];
        if (!isfinite(det) || det <= 1e-12) { /* preprocess.py:122-124 */
            status[i] = 2;
            continue;
        }
        status[i] = 0;
        double ia = s2[1][1] / det, ib = -s2[0][1] / det, ic = s2[0][0] / det; /* 125-127 */
        mean2d[2 * i] = m0;
        mean2d[2 * i + 1] = m1;
        conic[3 * i] = ia;
        conic[3 * i + 1] = ib;
        conic[3 * i + 2] = ic;
        depth[i] = z;
        /* view direction in world space (preprocess.py:129-131) */
        double nrm = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        double vx = d[0] / nrm, vy = d[1] / nrm, vz = d[2] / nrm;
        for (int ch = 0; ch < 3; ch++)
            color[3 * i + ch] = sh_channel(sh + 48 * i + 16 * ch, vx, vy, vz, cfg->sh_degree);
        /* effective_radius_sq (preprocess.py:68-71, 133-135) */
        double r2;
        if (cfg->opacity_aware) {
            r2 = 2.0 * log(opac[i] / cfg->alpha_theta);
            if (r2 > 9.0) r2 = 9.0;
            if (r2 < 0.0) r2 = 0.0;
        } else {
            r2 = 9.0;
        }
        r2_out[i] = r2;
        /* bin_tiles extent box (preprocess.py:166-186) */
        if (r2 <= 0.0) continue;
        double detp = ia * ic - ib * ib;
        double cxx = ic / detp, cyy = ia / detp;
        double hx = sqrt(r2 * cxx), hy = sqrt(r2 * cyy);
        axis_range(m0 - hx, m0 + hx, tiles_x, &rect[4 * i + 0], &rect[4 * i + 1]);
        axis_range(m1 - hy, m1 + hy, tiles_y, &rect[4 * i + 2], &rect[4 * i + 3]);
    }
}

/* ------------------------------------------------------------------------- */
/* Sort (sorting.py:32-54): order pairs by (tile_id, depth, gaussian_ref).    */

typedef struct {
    int32_t tile;
    int32_t ref;
    double depth;
} oc_pair;

static int pair_cmp(const void *a, const void *b) {
    const oc_pair *x = (const oc_pair *)a, *y = (const oc_pair *)b;
    if (x->tile != y->tile) return x->tile < y->tile ? -1 : 1;
    if (x->depth != y->depth) return x->depth < y->depth ? -1 : 1;
    if (x->ref != y->ref) return x->ref < y->ref ? -1 : 1;
    return 0;
}

/*
 * Build the sorted intersection list for the projected splats.
 * refs are 0..P-1 in assembled order (render.py:108, 118); rect/depth are
 * indexed by ref.  Pairs are emitted ty-major, tx-minor (preprocess.py:179-189)
 * and then sorted.  Returns the number of pairs; when out arrays are NULL only
 * counts.  range_start/range_end are per tile (empty tiles: start == end == 0).
 */
int64_t oracle_sort_pairs(int64_t p, const int32_t *rect, const double *depth, int32_t tiles_x,
                          int32_t tiles_y, int32_t *pair_tile, int32_t *pair_ref,
                          int64_t *range_start, int64_t *range_end) {
    int64_t total = 0;
    for (int64_t r = 0; r < p; r++) {
        const int32_t *rc = rect + 4 * r;
        if (rc[0] > rc[1] || rc[2] > rc[3]) continue;
        total += (int64_t)(rc[1] - rc[0] + 1) * (rc[3] - rc[2] + 1);
    }
    if (!pair_tile) return total;
    /* np.lexsort((ref, depth, tile)) (sorting.py:43): the primary key partitions the pairs into tiles, so
     * each tile's pairs are gathered (emission order) and sorted by the full comparator independently --
     * the same order as one global sort, with the tiles sorted in parallel. */
    const int64_t n_tiles = (int64_t)tiles_x * tiles_y;
    int64_t *start = (int64_t *)calloc((size_t)n_tiles + 1, sizeof(int64_t));
    for (int64_t r = 0; r < p; r++) {
        const int32_t *rc = rect + 4 * r;
        if (rc[0] > rc[1] || rc[2] > rc[3]) continue;
        for (int32_t ty = rc[2]; ty <= rc[3]; ty++)
            for (int32_t tx = rc[0]; tx <= rc[1]; tx++) start[(int64_t)ty * tiles_x + tx + 1]++;
    }
    for (int64_t t = 0; t < n_tiles; t++) start[t + 1] += start[t];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_tiles ? n_tiles : 1));
    for (int64_t t = 0; t < n_tiles; t++) fill[t] = start[t];
    oc_pair *pairs = (oc_pair *)malloc(sizeof(oc_pair) * (total ? total : 1));
    for (int64_t r = 0; r < p; r++) {
        const int32_t *rc = rect + 4 * r;
        if (rc[0] > rc[1] || rc[2] > rc[3]) continue;
        for (int32_t ty = rc[2]; ty <= rc[3]; ty++)
            for (int32_t tx = rc[0]; tx <= rc[1]; tx++) {
                const int64_t t = (int64_t)ty * tiles_x + tx;
                oc_pair *q = pairs + fill[t]++;
                q->tile = (int32_t)t;
                q->ref = (int32_t)r;
                q->depth = depth[r];
            }
    }
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t t = 0; t < n_tiles; t++)
        if (start[t + 1] - start[t] > 1)
            qsort(pairs + start[t], (size_t)(start[t + 1] - start[t]), sizeof(oc_pair), pair_cmp);
    for (int64_t t = 0; t < n_tiles; t++) {
        range_start[t] = start[t] < start[t + 1] ? start[t] : 0;
        range_end[t] = start[t] < start[t + 1] ? start[t + 1] : 0;
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < total; i++) {
        pair_tile[i] = pairs[i].tile;
        pair_ref[i] = pairs[i].ref;
    }
    free(pairs);
    free(fill);
    free(start);
    return total;
}

/* ------------------------------------------------------------------------- */
/* Rasterization (rasterize.py).                                              */

/* rasterize.py:146-151 _alphas (one pixel) */
static inline double oc_alpha(double px, double py, const double *mean, const double *cn, double o) {
    double dx = px - mean[0];
    double dy = py - mean[1];
    double q = cn[0] * dx * dx + 2.0 * cn[1] * dx * dy + cn[2] * dy * dy;
    double a = o * exp(-0.5 * q);
    return a < 0.99 ? a : 0.99;
}

/* model-warp index of tile pixel (lx, ly) (rasterize.py:200, 267-271, 291-298) */
static inline int model_warp_of(int lx, int ly, int engine, int w) {
    if (engine == 0 || w <= 2) return ly >> 1;
    /* w = 4: 2 groups per model-warp, group-row-major */
    int g = (ly / 4) * 4 + (lx / 4);
    return g / 2;
}

/*
 * Rasterize one tile with either engine: rasterize_reference (rasterize.py:180-232)
 * or rasterize_contribution_aware (rasterize.py:249-322), including the lockstep
 * cost counters (208-223, 291-313) and the background composite (228-231).
 * Writes color/contrib for valid pixels and adds counters into cost[4]
 * = {alpha_eval, blend, leader_eval, warp_steps}.
 */
static void raster_tile(int tile_id, int tiles_x, int width, int height, const int32_t *refs,
                        int64_t count, const double *means, const double *conics,
                        const double *colors, const double *opac, const oc_config *cfg,
                        double *image, int32_t *contrib, int64_t cost[4]) {
    int ox = (tile_id % tiles_x) * OC_TILE, oy = (tile_id / tiles_x) * OC_TILE;
    double C[256][3], T[256];
    int done[256], cnt[256], valid[256];
    for (int p = 0; p < 256; p++) {
        int x = ox + (p & 15), y = oy + (p >> 4);
        valid[p] = (x < width) && (y < height);
        done[p] = !valid[p];
        T[p] = 1.0;
        C[p][0] = C[p][1] = C[p][2] = 0.0;
        cnt[p] = 0;
    }
    int cr = cfg->engine == 1;
    int w = cr ? cfg->group_w : 1;
    double th = cfg->alpha_theta, gm = cfg->gamma_threshold;
    int64_t c_alpha = 0, c_blend = 0, c_leader = 0, c_steps = 0;
    for (int64_t j = 0; j < count; j++) {
        int all_done = 1;
        for (int p = 0; p < 256; p++) all_done &= done[p];
        if (all_done) break;
        int r = refs[j];
        const double *mn = means + 2 * r, *cn = conics + 3 * r, *col = colors + 3 * r;
        double o = opac[r];
        double a[256];
        int blend[256];
        int warp_live[8] = {0}, warp_pass[8] = {0}, warp_blend[8] = {0};
        if (!cr) {
            for (int p = 0; p < 256; p++) {
                int lx = p & 15, ly = p >> 4;
                int live = !done[p];
                blend[p] = 0;
                if (!live) continue;
                a[p] = oc_alpha(ox + lx + 0.5, oy + ly + 0.5, mn, cn, o);
                blend[p] = a[p] >= th;
                int k = ly >> 1;
                warp_live[k] = 1;
                if (blend[p]) warp_blend[k] = 1;
            }
            for (int k = 0; k < 8; k++) {
                c_alpha += warp_live[k];
                c_blend += warp_blend[k];
                c_steps += warp_live[k] + warp_blend[k];
            }
        } else {
            int gs = OC_TILE / w;
            for (int p = 0; p < 256; p++) blend[p] = 0;
            for (int gy = 0; gy < gs; gy++)
                for (int gx = 0; gx < gs; gx++) {
                    int live_g = 0;
                    for (int dy = 0; dy < w; dy++)
                        for (int dx = 0; dx < w; dx++) live_g |= !done[(gy * w + dy) * 16 + gx * w + dx];
                    int k = model_warp_of(gx * w, gy * w, 1, w);
                    if (!live_g) continue;
                    warp_live[k] = 1;
                    /* leader = top-left member; its alpha counts even if it is done (rasterize.py:281) */
                    double la = oc_alpha(ox + gx * w + 0.5, oy + gy * w + 0.5, mn, cn, o);
                    if (!(la >= th)) continue;
                    warp_pass[k] = 1;
                    for (int dy = 0; dy < w; dy++)
                        for (int dx = 0; dx < w; dx++) {
                            int p = (gy * w + dy) * 16 + gx * w + dx;
                            if (done[p]) continue;
                            a[p] = (dx == 0 && dy == 0) ? la
                                                        : oc_alpha(ox + gx * w + dx + 0.5, oy + gy * w + dy + 0.5, mn, cn, o);
                            blend[p] = a[p] >= th;
                            if (blend[p]) warp_blend[k] = 1;
                        }
                }
            for (int k = 0; k < 8; k++) {
                c_leader += warp_live[k];
                c_alpha += warp_pass[k];
                c_blend += warp_blend[k];
                c_steps += warp_live[k] + warp_pass[k];
            }
        }
        /* _blend (rasterize.py:169-177): blend on mask, then done |= T < gamma */
        for (int p = 0; p < 256; p++) {
            if (!blend[p]) continue;
            double wgt = T[p] * a[p];
            C[p][0] += wgt * col[0];
            C[p][1] += wgt * col[1];
            C[p][2] += wgt * col[2];
            T[p] *= 1.0 - a[p];
            cnt[p] += 1;
            if (T[p] < gm) done[p] = 1;
        }
    }
    for (int p = 0; p < 256; p++) {
        if (!valid[p]) continue;
        int x = ox + (p & 15), y = oy + (p >> 4);
        int64_t pix = (int64_t)y * width + x;
        for (int ch = 0; ch < 3; ch++) image[3 * pix + ch] = C[p][ch] + T[p] * cfg->background[ch];
        if (contrib) contrib[pix] = cnt[p];
    }
    cost[0] += c_alpha;
    cost[1] += c_blend;
    cost[2] += c_leader;
    cost[3] += c_steps;
}

/*
 * render_frame's tile loop (render.py:194-225): every tile (empty tiles get
 * the background), deterministic merge, counters summed.  refs index the
 * per-projected arrays.  cost_out = {alpha_eval, blend, leader_eval, warp_steps}.
 */
void oracle_raster_frame(int32_t width, int32_t height, const int32_t *pair_ref,
                         const int64_t *range_start, const int64_t *range_end, const double *means,
                         const double *conics, const double *colors, const double *opac,
                         const oc_config *cfg, int32_t n_threads, double *image, int32_t *contrib,
                         int64_t *cost_out) {
    int tiles_x = (width + OC_TILE - 1) / OC_TILE;
    int tiles_y = (height + OC_TILE - 1) / OC_TILE;
    int n_tiles = tiles_x * tiles_y;
    int64_t c0 = 0, c1 = 0, c2 = 0, c3 = 0;
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#endif
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : c0, c1, c2, c3)
    for (int t = 0; t < n_tiles; t++) {
        int64_t cost[4] = {0, 0, 0, 0};
        int64_t s = range_start[t], e = range_end[t];
        raster_tile(t, tiles_x, width, height, pair_ref + s, e - s, means, conics, colors, opac, cfg,
                    image, contrib, cost);
        c0 += cost[0];
        c1 += cost[1];
        c2 += cost[2];
        c3 += cost[3];
    }
    cost_out[0] = c0;
    cost_out[1] = c1;
    cost_out[2] = c2;
    cost_out[3] = c3;
}

/*
 * select_clusters (residency.py:38-54) with pose_feature (compiler.py:113-121)
 * and CameraPose.forward (model.py:174-176): nearest 1+m centroids by squared
 * distance in the 6-D feature space, ties toward the smaller id.
 */
int oracle_select_clusters(const oc_camera *cam, const double *centroids, int32_t n, int32_t m,
                           double beta, const double *pos_mean, double pos_scale, int32_t *out) {
    if (m >= n || m < 0 || pos_scale <= 0.0) return -1;
    double rc[3][3];
    quat_to_mat(cam->orientation, rc);
    double f[6];
    for (int k = 0; k < 3; k++) f[k] = (cam->position[k] - pos_mean[k]) / pos_scale;
    for (int k = 0; k < 3; k++) f[3 + k] = beta * rc[k][2];
    double *d2 = (double *)malloc(sizeof(double) * n);
    int *used = (int *)calloc(n, sizeof(int));
    for (int c = 0; c < n; c++) {
        double s = 0.0;
        for (int k = 0; k < 6; k++) {
            double v = centroids[6 * c + k] - f[k];
            s += v * v;
        }
        d2[c] = s;
    }
    for (int s = 0; s <= m; s++) {
        int best = -1;
        for (int c = 0; c < n; c++) {
            if (used[c]) continue;
            if (best < 0 || d2[c] < d2[best]) best = c;
        }
        used[best] = 1;
        out[s] = best;
    }
    free(d2);
    free(used);
    return 0;
}
