// C-ABI of the B200 Seele render path (include/seele_b200.h): argument checks,
// per-frame camera constants, workspace carve-up and the stream-ordered
// launch sequence of one frame.  No allocation, no host synchronisation.
#include <math.h>
#include <stdarg.h>

#include <atomic>
#include <stdio.h>
#include <string.h>

#include "common.cuh"

namespace seele {

namespace {

thread_local char g_err[512] = "";
std::atomic<long long> g_launches{0};
thread_local bool g_prof = false;
thread_local cudaEvent_t g_ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};

inline void prof_mark(int i, cudaStream_t st) {
    if (g_prof) cudaEventRecord(g_ev[i], st);
}

// Small per-thread ring of events for cross-stream ordering (reuse is safe:
// cudaStreamWaitEvent captures the event's state when it is called).
cudaEvent_t next_event() {
    thread_local cudaEvent_t ring[16] = {};
    thread_local int at = 0;
    at = (at + 1) & 15;
    if (!ring[at] && cudaEventCreateWithFlags(&ring[at], cudaEventDisableTiming) != cudaSuccess) return nullptr;
    return ring[at];
}

int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int cuda_fail(cudaError_t e, const char *where) {
    snprintf(g_err, sizeof(g_err), "CUDA error in %s: %s", where, cudaGetErrorString(e));
    return SEELE_ERR_CUDA;
}

size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

struct Carver {
    char *base;
    size_t off = 0;
    template <typename T>
    T *take(long long count) {
        T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
        off += align_up(sizeof(T) * (size_t)(count > 0 ? count : 1));
        return p;
    }
};

int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = v > 0 ? v : 148;
    }
    return cached[dev];
}

// CameraPose.rotation_matrix / focal / principal_point (model.py:170-184) and
// world_to_view = R^T (preprocess.py:99), in host fp64 like the reference.
CamK make_cam(const seele_camera &c) {
    CamK k;
    const double w = c.orientation[0], x = c.orientation[1], y = c.orientation[2], z = c.orientation[3];
    const double r[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                         2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                         2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) k.w2v[3 * i + j] = r[3 * j + i];
    for (int i = 0; i < 3; i++) k.pos[i] = c.position[i];
    k.fx = c.width / (2.0 * tan(c.fov_x / 2.0));
    k.fy = c.height / (2.0 * tan(c.fov_y / 2.0));
    k.cx = c.width / 2.0;
    k.cy = c.height / 2.0;
    k.near_clip = c.near_clip;
    k.width = c.width;
    k.height = c.height;
    k.tiles_x = (c.width + kTile - 1) / kTile;
    k.tiles_y = (c.height + kTile - 1) / kTile;
    return k;
}

int check_camera(const seele_camera *c) {
    if (!c) return fail(SEELE_ERR_INVALID_ARGUMENT, "camera is null");
    if (c->width < kTile || c->height < kTile)
        return fail(SEELE_ERR_DATA, "width and height must be >= 16, got %d x %d", c->width, c->height);
    if (!(c->fov_x > 0.0 && c->fov_x < M_PI) || !(c->fov_y > 0.0 && c->fov_y < M_PI))
        return fail(SEELE_ERR_DATA, "fov must lie in (0, pi)");
    long long tiles_x = (c->width + kTile - 1) / kTile, tiles_y = (c->height + kTile - 1) / kTile;
    if (tiles_x > kMaxTileAxis || tiles_y > kMaxTileAxis)
        return fail(SEELE_ERR_INVALID_ARGUMENT, "image too large (at most 4096 pixels per axis)");
    return SEELE_OK;
}

int check_config(const seele_config *c) {
    if (!c) return fail(SEELE_ERR_INVALID_ARGUMENT, "config is null");
    if (c->engine != 0 && c->engine != 1) return fail(SEELE_ERR_INVALID_ARGUMENT, "unknown engine %d", c->engine);
    if (c->group_w != 1 && c->group_w != 2 && c->group_w != 4)
        return fail(SEELE_ERR_INVALID_ARGUMENT, "group width must be 1, 2 or 4, got %d", c->group_w);
    if (c->sh_degree < 0 || c->sh_degree > 3)
        return fail(SEELE_ERR_INVALID_ARGUMENT, "SH degree must lie in [0, 3], got %d", c->sh_degree);
    if (c->tile_size != kTile) return fail(SEELE_ERR_INVALID_ARGUMENT, "tile size must be 16, got %d", c->tile_size);
    const int prec = c->precision & ~SEELE_KEEP_UNBINNED;
    if (prec != SEELE_PRECISION_FAST && prec != SEELE_PRECISION_EXACT)
        return fail(SEELE_ERR_INVALID_ARGUMENT, "unknown precision %d", c->precision);
    if (!(c->alpha_theta > 0.0) || !(c->gamma_threshold > 0.0))
        return fail(SEELE_ERR_INVALID_ARGUMENT, "thresholds must be positive");
    return SEELE_OK;
}

}  // namespace

void note_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

Workspace carve_workspace(void *base, long long n_max, long long cap, int width, int height) {
    Carver c{static_cast<char *>(base)};
    Workspace w;
    w.stats_ptr = nullptr;
    const long long n = n_max > 0 ? n_max : 1;
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    const long long tiles = (long long)tiles_x * tiles_y;
    // never-cleared state first (epoch + look-back words; zero-filled once by the owner)
    w.epoch = c.take<uint32_t>(1);
    w.look = c.take<unsigned long long>(kDepthBuckets / kDepthScanItems);
    w.status = c.take<uint8_t>(n);
    w.srec = c.take<uint4>(n);
    w.xrec = c.take<ExactRec>(n);
    w.rec = c.take<RasterRec>(n);
    w.bhist = c.take<uint32_t>(kDepthBuckets + 1);
    w.brec[0] = c.take<uint4>(n);
    w.brec[1] = c.take<uint4>(n);
    w.gfirst = c.take<uint32_t>(n / kDepthGroup + 2);
    w.dval[0] = c.take<uint32_t>(n);
    w.dval[1] = c.take<uint32_t>(n);
    w.drect[0] = c.take<uint32_t>(n);
    w.drect[1] = c.take<uint32_t>(n);
    const BinGeom g = bin_geometry(n, width, height);
    w.cmat = c.take<uint32_t>((long long)g.n_chunks * g.n_st);
    w.st_cnt = c.take<uint32_t>(g.n_st);
    w.st_start = c.take<uint32_t>(g.n_st + 1);
    w.seg_first = c.take<uint32_t>(g.n_st + 1);
    w.seg_st = c.take<uint32_t>(cap / kSeg + g.n_st + 1);
    w.seg_look = c.take<unsigned long long>((cap / kSeg + g.n_st + 1) * 16);
    w.ent = c.take<uint2>(cap);
    w.head_cnt = c.take<uint32_t>(tiles);
    w.pfinal = c.take<uint32_t>(cap);
    w.ranges = c.take<uint2>(tiles);
    w.tile_order = c.take<uint32_t>(tiles);
    w.tile_diff = c.take<int32_t>((long long)(tiles_x + 1) * (tiles_y + 1));
    w.counters = c.take<uint32_t>(CNT_COUNT);
    w.pairs64 = c.take<unsigned long long>(1);
    w.bytes = c.off;
    return w;
}

namespace {

__global__ void k_export_splats(Workspace ws, long long n, int8_t *status, double *depth, int32_t *rect, double *mean,
                                double *conic, double *opacity, float *color) {
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
        if (status) status[p] = (int8_t)ws.status[p];
        const bool ok = ws.status[p] == 0;
        const uint4 sr = ws.srec[p];
        if (depth) depth[p] = ok ? __hiloint2double((int)sr.w, (int)sr.z) : 0.0;
        if (rect) {
            rect[4 * p] = (int32_t)(sr.x & 0xffu);
            rect[4 * p + 1] = (int32_t)((sr.x >> 8) & 0xffu);
            rect[4 * p + 2] = (int32_t)((sr.x >> 16) & 0xffu);
            rect[4 * p + 3] = (int32_t)(sr.x >> 24);
        }
        if (mean) {
            const double2 m = ok ? ws.xrec[p].m : make_double2(0, 0);
            mean[2 * p] = m.x;
            mean[2 * p + 1] = m.y;
        }
        const double4 co = ok ? ws.xrec[p].co : make_double4(0, 0, 0, 0);
        if (conic) {
            conic[3 * p] = co.x;
            conic[3 * p + 1] = co.y;
            conic[3 * p + 2] = co.z;
        }
        if (opacity) opacity[p] = co.w;
        if (color) {
            const RasterRec r = ok ? ws.rec[p] : RasterRec{};
            color[3 * p] = r.r;
            color[3 * p + 1] = r.g;
            color[3 * p + 2] = r.b;
        }
    }
}

__global__ void k_export_ranges(const uint2 *ranges, int n, int32_t *out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint2 r = ranges[t];
    out[2 * t] = r.x < r.y ? (int32_t)r.x : 0;  // empty tiles -> (0, 0)
    out[2 * t + 1] = r.x < r.y ? (int32_t)r.y : 0;
}

}  // namespace
}  // namespace seele

using namespace seele;

extern "C" {

int32_t seele_abi_version(void) { return 1; }

int64_t seele_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

const char *seele_last_error(void) { return g_err; }

size_t seele_workspace_bytes(int64_t n_max, int64_t pair_capacity, int32_t width, int32_t height) {
    return carve_workspace(nullptr, n_max, pair_capacity, width, height).bytes;
}

int seele_render_split(const seele_scene *scene, const int64_t *ranges_dev, int32_t n_ranges, const seele_camera *cam,
                       const seele_config *cfg, void *workspace, size_t workspace_bytes, int64_t n_max,
                       int64_t pair_capacity, float *image_dev, int32_t *contrib_dev, int64_t *stats_dev, void *stream,
                       void *raster_stream) {
    g_err[0] = 0;
    int rc;
    if ((rc = check_camera(cam)) != SEELE_OK) return rc;
    if ((rc = check_config(cfg)) != SEELE_OK) return rc;
    if (!scene || scene->n < 0) return fail(SEELE_ERR_INVALID_ARGUMENT, "scene is null");
    if (scene->layout == SEELE_LAYOUT_PLANES) {
        if (!scene->planes || scene->plane_stride < scene->n)
            return fail(SEELE_ERR_INVALID_ARGUMENT, "planes layout needs planes and plane_stride >= n");
    } else if (scene->layout == SEELE_LAYOUT_F64) {
        if (scene->n > 0 && (!scene->positions || !scene->log_scales || !scene->rotations || !scene->opacities || !scene->sh))
            return fail(SEELE_ERR_INVALID_ARGUMENT, "f64 layout needs all five arrays");
    } else {
        return fail(SEELE_ERR_INVALID_ARGUMENT, "unknown scene layout %d", scene->layout);
    }
    if (n_ranges < 1 || n_ranges > SEELE_MAX_RANGES || !ranges_dev)
        return fail(SEELE_ERR_INVALID_ARGUMENT, "need 1..64 working-set ranges, got %d", n_ranges);
    if (n_max < 1 || n_max >= (1ll << 30) || pair_capacity < 1 || pair_capacity >= (1ll << 30))
        return fail(SEELE_ERR_INVALID_ARGUMENT, "n_max / pair_capacity out of range");
    if (!workspace || !image_dev || !stats_dev) return fail(SEELE_ERR_INVALID_ARGUMENT, "null output or workspace");
    Workspace ws = carve_workspace(workspace, n_max, pair_capacity, cam->width, cam->height);
    if (ws.bytes > workspace_bytes)
        return fail(SEELE_ERR_INVALID_ARGUMENT, "workspace too small (need %lld bytes)", (long long)ws.bytes);
    ws.stats_ptr = stats_dev;

    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const CamK ck = make_cam(*cam);
    CfgK cf;
    cf.engine = cfg->engine;
    cf.group_w = cfg->group_w;
    cf.sh_degree = cfg->sh_degree;
    cf.opacity_aware = cfg->opacity_aware;
    cf.precision = cfg->precision & ~SEELE_KEEP_UNBINNED;
    cf.keep_unbinned = (cfg->precision & SEELE_KEEP_UNBINNED) != 0;
    cf.alpha_theta = cfg->alpha_theta;
    set_gamma(cf, cfg->gamma_threshold);
    for (int i = 0; i < 3; i++) cf.bg[i] = cfg->background[i];
    SceneK sk;
    sk.layout = scene->layout;
    sk.n = scene->n;
    sk.pos = scene->positions;
    sk.log_scale = scene->log_scales;
    sk.rot = scene->rotations;
    sk.opac = scene->opacities;
    sk.sh = scene->sh;
    sk.planes = reinterpret_cast<const float4 *>(scene->planes);
    sk.plane_stride = scene->plane_stride;

    cudaError_t e;
    const int sms = stream_sms(st);  // (the plan partition's SMs on a partition stream)
    long long pre_blocks = (n_max + 255) / 256;
#ifndef SEELE_PRE_GRID_PER_SM
#define SEELE_PRE_GRID_PER_SM 3  // persistent: the resident CTAs of k_preprocess (launch bounds 256, 3)
#endif
    const long long pre_cap = (long long)(SEELE_PRE_GRID_PER_SM * sms);
    const int pre_grid = (int)(pre_blocks < pre_cap ? (pre_blocks > 0 ? pre_blocks : 1) : pre_cap);
    launch_frame_begin(ws, ck, stats_dev, st);
    prof_mark(0, st);
    launch_preprocess(sk, ranges_dev, n_ranges, ck, cf, ws, stats_dev, pre_grid, st);
    prof_mark(1, st);
    launch_depth_sort(ws, ck, n_max, stats_dev, st);
    prof_mark(2, st);
    launch_binning(ws, n_max, pair_capacity, ck, stats_dev, st);
    prof_mark(3, st);
    cudaStream_t rst = raster_stream ? static_cast<cudaStream_t>(raster_stream) : st;
    if (rst != st) {  // raster on its own stream, after the plan
        cudaEvent_t ev = next_event();
        if (!ev) return fail(SEELE_ERR_CUDA, "could not create a CUDA event");
        if ((e = cudaEventRecord(ev, st)) != cudaSuccess) return cuda_fail(e, "seele_render_split event");
        if ((e = cudaStreamWaitEvent(rst, ev, 0)) != cudaSuccess) return cuda_fail(e, "seele_render_split wait");
        prof_mark(3, rst);
    }
    launch_raster(ws, ws.pfinal, ck, cf, image_dev, contrib_dev, stats_dev, rst);
    prof_mark(4, rst);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "seele_render launch");
    return SEELE_OK;
}

int seele_render(const seele_scene *scene, const int64_t *ranges_dev, int32_t n_ranges, const seele_camera *cam,
                 const seele_config *cfg, void *workspace, size_t workspace_bytes, int64_t n_max,
                 int64_t pair_capacity, float *image_dev, int32_t *contrib_dev, int64_t *stats_dev, void *stream) {
    return seele_render_split(scene, ranges_dev, n_ranges, cam, cfg, workspace, workspace_bytes, n_max, pair_capacity,
                              image_dev, contrib_dev, stats_dev, stream, nullptr);
}

int seele_profile_enable(int32_t on) {
    g_err[0] = 0;
    if (on && !g_ev[0]) {
        for (int i = 0; i < 5; i++) {
            cudaError_t e = cudaEventCreate(&g_ev[i]);
            if (e != cudaSuccess) return cuda_fail(e, "seele_profile_enable");
        }
    }
    g_prof = on != 0;
    return SEELE_OK;
}

int seele_profile_read(float *ms_out, int32_t n) {
    g_err[0] = 0;
    if (!g_ev[0] || !ms_out || n < 0 || n > 4) return fail(SEELE_ERR_INVALID_ARGUMENT, "profiling not enabled or bad n");
    cudaError_t e = cudaEventSynchronize(g_ev[4]);
    if (e != cudaSuccess) return cuda_fail(e, "seele_profile_read");
    for (int i = 0; i < n; i++) {
        e = cudaEventElapsedTime(&ms_out[i], g_ev[i], g_ev[i + 1]);
        if (e != cudaSuccess) return cuda_fail(e, "seele_profile_read");
    }
    return SEELE_OK;
}

int seele_select_clusters(const seele_camera *cam, const double *centroids_dev, int32_t n_clusters, int32_t m,
                          double beta, const double *pos_mean, double pos_scale, const int64_t *chunk_dev,
                          int32_t *out_ids_dev, int64_t *ranges_out_dev, void *stream) {
    g_err[0] = 0;
    if (!cam || !centroids_dev || !pos_mean || !chunk_dev || !out_ids_dev || !ranges_out_dev)
        return fail(SEELE_ERR_INVALID_ARGUMENT, "null argument");
    if (n_clusters < 1 || n_clusters > 1024) return fail(SEELE_ERR_INVALID_ARGUMENT, "need 1..1024 clusters, got %d", n_clusters);
    if (m < 0 || m >= n_clusters)
        return fail(SEELE_ERR_INVALID_ARGUMENT, "m must be < %d, got %d", n_clusters, m);  // residency.py:49-50
    if (m + 2 > SEELE_MAX_RANGES) return fail(SEELE_ERR_INVALID_ARGUMENT, "too many clusters selected");
    if (!(pos_scale > 0.0)) return fail(SEELE_ERR_INVALID_ARGUMENT, "normalization scale must be positive");
    const CamK ck = make_cam(*cam);
    // pos_mean is a host pointer (3 doubles), passed by value to the kernel
    launch_select(ck, centroids_dev, n_clusters, m, beta, pos_mean, pos_scale, chunk_dev, out_ids_dev,
                  ranges_out_dev, static_cast<cudaStream_t>(stream));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "seele_select_clusters");
    return SEELE_OK;
}

int seele_plan_export(void *workspace, int64_t n_max, int64_t pair_capacity, int32_t width, int32_t height,
                      int64_t n_ws, int64_t n_pairs, const seele_plan_view *out, void *stream) {
    g_err[0] = 0;
    if (!workspace || !out) return fail(SEELE_ERR_INVALID_ARGUMENT, "null argument");
    if (n_pairs > pair_capacity || n_ws > n_max) return fail(SEELE_ERR_INVALID_ARGUMENT, "sizes exceed the workspace");
    const Workspace ws = carve_workspace(workspace, n_max, pair_capacity, width, height);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long tiles = (long long)((width + kTile - 1) / kTile) * ((height + kTile - 1) / kTile);
    cudaError_t e = cudaSuccess;
    if (out->pair_pos && n_pairs > 0)
        e = cudaMemcpyAsync(out->pair_pos, ws.pfinal, sizeof(uint32_t) * n_pairs, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "seele_plan_export copy");
    if (out->pair_tile && n_pairs > 0) launch_fill_pair_tiles(ws.ranges, (int)tiles, out->pair_tile, st);
    if (out->ranges) {
        k_export_ranges<<<(int)((tiles + 255) / 256), 256, 0, st>>>(ws.ranges, (int)tiles, out->ranges);
        note_launches(1);
    }
    if (n_ws > 0)
        k_export_splats<<<(int)((n_ws + 255) / 256 < 4096 ? (n_ws + 255) / 256 : 4096), 256, 0, st>>>(
            ws, n_ws, out->status, out->depth, out->rect, out->mean, out->conic, out->opacity, out->color);
    if (n_ws > 0) note_launches(1);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "seele_plan_export");
    return SEELE_OK;
}

int seele_harvest_topk(void *workspace, int64_t n_max, int64_t pair_capacity, const seele_camera *cam,
                       const seele_config *cfg, const int64_t *ids_dev, int32_t k, uint8_t *flags_dev, void *stream) {
    g_err[0] = 0;
    int rc;
    if ((rc = check_camera(cam)) != SEELE_OK) return rc;
    if ((rc = check_config(cfg)) != SEELE_OK) return rc;
    if (!workspace || !ids_dev || !flags_dev) return fail(SEELE_ERR_INVALID_ARGUMENT, "null argument");
    if (k < 1 || k > 32) return fail(SEELE_ERR_INVALID_ARGUMENT, "k must lie in [1, 32], got %d", k);
    const Workspace ws = carve_workspace(workspace, n_max, pair_capacity, cam->width, cam->height);
    const CamK ck = make_cam(*cam);
    CfgK cf{};
    cf.engine = cfg->engine;
    cf.group_w = cfg->group_w;
    cf.alpha_theta = cfg->alpha_theta;
    set_gamma(cf, cfg->gamma_threshold);
    launch_harvest(cfg->engine == 0 ? 0 : cfg->group_w, ws, ws.pfinal, ck, cf, ids_dev, k, flags_dev,
                   static_cast<cudaStream_t>(stream));
    cudaError_t e;
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "seele_harvest_topk");
    return SEELE_OK;
}

int seele_contributions(void *workspace, int64_t n_max, int64_t pair_capacity, const seele_camera *cam,
                        const seele_config *cfg, int64_t n_ws, int32_t *row_of_pos_dev, double *out_dev, void *stream) {
    g_err[0] = 0;
    int rc;
    if ((rc = check_camera(cam)) != SEELE_OK) return rc;
    if ((rc = check_config(cfg)) != SEELE_OK) return rc;
    if (!workspace || !row_of_pos_dev || !out_dev) return fail(SEELE_ERR_INVALID_ARGUMENT, "null argument");
    if (n_ws < 0 || n_ws > n_max) return fail(SEELE_ERR_INVALID_ARGUMENT, "n_ws out of [0, n_max]");
    const Workspace ws = carve_workspace(workspace, n_max, pair_capacity, cam->width, cam->height);
    const CamK ck = make_cam(*cam);
    CfgK cf{};
    cf.engine = cfg->engine;
    cf.group_w = cfg->group_w;
    cf.alpha_theta = cfg->alpha_theta;
    set_gamma(cf, cfg->gamma_threshold);
    launch_contributions(cfg->engine == 0 ? 0 : cfg->group_w, ws, ws.pfinal, ck, cf, n_ws, row_of_pos_dev, out_dev,
                         static_cast<cudaStream_t>(stream));
    cudaError_t e;
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "seele_contributions");
    return SEELE_OK;
}

int seele_skip_bound(void *workspace, int64_t n_max, int64_t pair_capacity, const seele_camera *cam,
                     const seele_config *cfg, double *bound_dev, void *stream) {
    g_err[0] = 0;
    int rc;
    if ((rc = check_camera(cam)) != SEELE_OK) return rc;
    if ((rc = check_config(cfg)) != SEELE_OK) return rc;
    if (!workspace || !bound_dev) return fail(SEELE_ERR_INVALID_ARGUMENT, "null argument");
    const Workspace ws = carve_workspace(workspace, n_max, pair_capacity, cam->width, cam->height);
    const CamK ck = make_cam(*cam);
    CfgK cf{};
    cf.engine = cfg->engine;
    cf.group_w = cfg->group_w;
    cf.alpha_theta = cfg->alpha_theta;
    set_gamma(cf, cfg->gamma_threshold);
    launch_skip_bound(cfg->group_w, ws, ws.pfinal, ck, cf, bound_dev, static_cast<cudaStream_t>(stream));
    cudaError_t e;
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "seele_skip_bound");
    return SEELE_OK;
}

int seele_partition_create(int32_t plan_sms, int32_t n_streams, void **plan_streams, void **raster_streams,
                           int32_t *plan_sms_out, int32_t *raster_sms_out) {
    g_err[0] = 0;
    if (plan_sms < 1 || n_streams < 1 || n_streams > 64 || !plan_streams || !raster_streams || !plan_sms_out ||
        !raster_sms_out)
        return fail(SEELE_ERR_INVALID_ARGUMENT, "partition: bad arguments");
    int po = 0, ro = 0;
    const int rc = partition_create(plan_sms, n_streams, plan_streams, raster_streams, &po, &ro);
    if (rc != 0) return fail(SEELE_ERR_CUDA, "partition: green contexts unavailable or split refused (%d)", rc);
    *plan_sms_out = po;
    *raster_sms_out = ro;
    return SEELE_OK;
}

}  // extern "C"
