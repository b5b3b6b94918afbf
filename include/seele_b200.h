/*
 * seele_b200.h -- C-ABI of the B200 (sm_100a) Seele render hot path.
 *
 * The reference (pkg/src/seele, pure Python) has no FFI; its operator
 * boundary is the Python call render.render_frame(scene, cam, cfg)
 * (render.py:172-179), plan_frame (render.py:90) and
 * residency.select_clusters / ResidentRenderer.select/assemble
 * (residency.py:38-54, 214-220).  Each entry point below replaces one of
 * those; the Python shims in paper_2503_05168_b200/ bind them with ctypes
 * (see INTEGRATION.md).
 *
 * Conventions
 *  - Plain pointers and sizes only.  All "dev" pointers are CUDA device
 *    pointers owned by the caller (PyTorch); the library never allocates
 *    per frame and keeps no global device state.
 *  - Every call is asynchronous on the given cudaStream_t (passed as void*)
 *    unless documented otherwise.  Counters are written to device memory.
 *  - Return value: seele_status.  A message for the last failure on the
 *    calling thread is available from seele_last_error().
 */
#ifndef SEELE_B200_H
#define SEELE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error convention: maps onto pkg/src/seele/errors.py:5-30. */
typedef enum seele_status {
    SEELE_OK = 0,
    SEELE_ERR_INVALID_ARGUMENT = 1, /* InvalidArgumentError (render.py:45-51, residency.py:49-50) */
    SEELE_ERR_DATA = 2,             /* DataError (model.py validators) */
    SEELE_ERR_CONTRACT = 3,         /* ContractViolationError (rasterize.py:154-156) */
    SEELE_ERR_CUDA = 4,             /* CUDA runtime failure */
    SEELE_ERR_CAPACITY = 5          /* workspace too small; see stats[SEELE_STAT_TILE_PAIRS] */
} seele_status;

/* CameraPose (model.py:132-184).  orientation = camera-to-world (w,x,y,z),
 * already normalised by the caller exactly as CameraPose.__post_init__ does. */
typedef struct seele_camera {
    double position[3];
    double orientation[4];
    double fov_x;
    double fov_y;
    double near_clip;
    int32_t width;
    int32_t height;
} seele_camera;

/* EngineConfig (render.py:31-51) minus `threads` (tiles map to CTAs). */
typedef struct seele_config {
    int32_t engine;        /* 0 = "ref" (rasterize.py:180), 1 = "cr" (rasterize.py:249) */
    int32_t group_w;       /* 1, 2 or 4 */
    int32_t sh_degree;     /* 0..3 */
    int32_t opacity_aware; /* opacity_aware_filter */
    double alpha_theta;
    double gamma_threshold;
    double background[3];
    int32_t precision;     /* SEELE_PRECISION_* */
    int32_t tile_size;     /* must be 16 */
} seele_config;

enum {
    SEELE_PRECISION_FAST = 0,  /* fp32 blend + guard bands + fp64 re-decision (default) */
    SEELE_PRECISION_EXACT = 1, /* every alpha / transmittance in fp64 */
    /* flag OR-ed into precision: also keep the projected splats that bin to no tile (depth, mean, conic,
     * colour) for seele_plan_export; a frame's own stages never read them, so they are skipped by default */
    SEELE_KEEP_UNBINNED = 0x100
};

/* Scene in HBM.  Two layouts:
 *  SEELE_LAYOUT_F64:   SceneArrays as given (model.py:308-374): positions
 *                      [n,3], log_scales [n,3], rotations [n,4] (raw; the
 *                      kernel normalises as Gaussian3D does), opacities [n]
 *                      decoded, sh [n,3,16]; all float64.
 *  SEELE_LAYOUT_PLANES: the cluster-container record (io.py:22-25) transposed
 *                      into 15 float4 planes of `plane_stride` elements:
 *                      P0 = (x, y, z, opacity logit), P1 = (scale0..2, 0),
 *                      P2 = raw rotation (w,x,y,z), P3..P14 = sh[3][16]
 *                      channel-major.  Opacity is decoded with the container's
 *                      clip(sigmoid(logit)) (io.py:33-34) and the rotation is
 *                      normalised twice (io.py:226-229 then model.py:122).
 * ids [n] int64 global ids (only read by seele_plan_export). */
typedef struct seele_scene {
    int32_t layout;
    int32_t _pad;
    int64_t n;
    const double *positions;
    const double *log_scales;
    const double *rotations;
    const double *opacities;
    const double *sh;
    const float *planes;
    int64_t plane_stride;
    const int64_t *ids;
} seele_scene;

enum { SEELE_LAYOUT_F64 = 0, SEELE_LAYOUT_PLANES = 1 };

/* Working set = concatenation of ranges of the resident scene, in order
 * (ResidentRenderer.assemble, residency.py:217-220: shared chunk first, then
 * the selected clusters nearest-first).  Device array of int64 pairs
 * (start, count); count of ranges <= SEELE_MAX_RANGES. */
#define SEELE_MAX_RANGES 64

/* Device stats vector (int64), written by seele_render.  Indices: */
enum {
    SEELE_STAT_ALPHA_EVAL = 0, /* FrameStats fields, rasterize.py:51-62 */
    SEELE_STAT_BLEND = 1,
    SEELE_STAT_LEADER_EVAL = 2,
    SEELE_STAT_WARP_STEPS = 3,
    SEELE_STAT_TILE_PAIRS = 4,
    SEELE_STAT_CULLED_NEAR = 5,
    SEELE_STAT_DROPPED_DEGENERATE = 6,
    SEELE_STAT_PROJECTED = 7,   /* splats surviving cull (len(plan.ids)) */
    SEELE_STAT_BINNED = 8,      /* splats with >= 1 tile */
    SEELE_STAT_WORKING_SET = 9, /* assembled splat count */
    SEELE_STAT_OVERFLOW = 10,   /* 1 if tile pairs exceeded the workspace capacity */
    SEELE_STAT_SKIPPED_PIXEL_STEPS = 11, /* fast path: live (pixel, splat) steps skipped by the warp-region test */
    SEELE_STAT_ALPHA_REDECIDE = 12, /* fast path: lane alpha tests re-decided in fp64 */
    SEELE_STAT_T_AMBIGUOUS = 13,    /* fast path: pixel T < gamma tests decided by exact fp64 recomputation */
    SEELE_STAT_LIVE_PIXEL_STEPS = 14, /* fast path: (live pixel, iterated splat) pairs */
    SEELE_STAT_PIXEL_BLENDS = 15,     /* fast path: (pixel, splat) blends */
    SEELE_STAT_COUNT = 16
};

/* Bytes of workspace needed for up to n_max assembled splats, pair_capacity
 * tile pairs and a width x height image (n_max, pair_capacity < 2^30; at most
 * 65536 pixels per axis).  The caller zero-fills a workspace ONCE when it
 * allocates it: the radix passes' look-back words are epoch-tagged and never
 * cleared per frame. */
size_t seele_workspace_bytes(int64_t n_max, int64_t pair_capacity, int32_t width, int32_t height);

/* One frame: plan_frame (render.py:90-141) + every tile of render_frame
 * (render.py:194-225).  ranges_dev: working-set ranges (device, int64
 * [n_ranges][2]); n_ranges <= SEELE_MAX_RANGES; may be produced on device by
 * seele_select_clusters.  Outputs: image_dev float32 [H,W,3] (background
 * composited), contrib_dev int32 [H,W] per-pixel blend count (nullable),
 * stats_dev int64 [SEELE_STAT_COUNT].  If the frame needs more than
 * pair_capacity pairs, stats[SEELE_STAT_OVERFLOW] = 1, stats[TILE_PAIRS] holds
 * the need and the image is not written (the caller grows the workspace and
 * calls again). */
int seele_render(const seele_scene *scene, const int64_t *ranges_dev, int32_t n_ranges,
                 const seele_camera *cam, const seele_config *cfg, void *workspace,
                 size_t workspace_bytes, int64_t n_max, int64_t pair_capacity, float *image_dev,
                 int32_t *contrib_dev, int64_t *stats_dev, void *stream);

/* seele_render with the raster (the last stage) issued on raster_stream
 * after the plan stages on `stream` (ordered by an event).  Lets a caller
 * with several frames in flight give the latency-bound plan stages a
 * higher stream priority than the issue-bound raster of another frame.
 * raster_stream == NULL: same as seele_render. */
int seele_render_split(const seele_scene *scene, const int64_t *ranges_dev, int32_t n_ranges,
                       const seele_camera *cam, const seele_config *cfg, void *workspace,
                       size_t workspace_bytes, int64_t n_max, int64_t pair_capacity, float *image_dev,
                       int32_t *contrib_dev, int64_t *stats_dev, void *stream, void *raster_stream);

/* SM partition for pipelined trajectories (no reference counterpart: a
 * B200-side scheduling aid).  Splits the device's SMs into two green
 * contexts -- plan_sms SMs for the plan stages, the rest for the raster --
 * and creates n_streams non-blocking streams in each (cudaStream_t handles in
 * plan_streams[i] / raster_streams[i], valid for the process lifetime).
 * Passing a plan stream as `stream` and a raster stream as `raster_stream`
 * to seele_render_split runs one frame's plan beside another frame's raster;
 * persistent grids are sized by the partition's SM count.  The granted SM
 * counts (rounded to the hardware's granularity, 8 on sm_100) are returned.
 * SEELE_ERR_CUDA when the driver has no green contexts. */
int seele_partition_create(int32_t plan_sms, int32_t n_streams, void **plan_streams, void **raster_streams,
                           int32_t *plan_sms_out, int32_t *raster_sms_out);

/* Image metrics on the device (metrics.py:44-112) of two (H, W, 3) fp64
 * images a_dev, b_dev: PSNR in dB (+inf when equal) and mean SSIM over the
 * BT.601 luminance (11x11 Gaussian window, sigma 1.5, valid positions).  The
 * result is one double at out_dev; scratch_dev holds
 * seele_metrics_scratch_doubles(width, height) doubles.  Stream-ordered. */
int seele_psnr(const double *a_dev, const double *b_dev, int64_t n, double *scratch_dev, double *out_dev,
               void *stream);
int seele_ssim(const double *a_dev, const double *b_dev, int32_t width, int32_t height, double *scratch_dev,
               double *out_dev, void *stream);
int64_t seele_metrics_scratch_doubles(int32_t width, int32_t height);

/* Contribution harvest of one pose (compiler.py:196-231): for the frame LAST
 * RENDERED into this workspace with the same camera and config, flags[p] = 1
 * for every assembled position p whose splat is among some pixel's k
 * strongest blend weights T * alpha (weight > 0; ties toward the smaller id,
 * ids_dev[p] = gaussian id of position p).  1 <= k <= 32.  flags_dev is not
 * cleared (poses of a cluster accumulate).  Stream-ordered; no sync. */
int seele_harvest_topk(void *workspace, int64_t n_max, int64_t pair_capacity, const seele_camera *cam,
                       const seele_config *cfg, const int64_t *ids_dev, int32_t k, uint8_t *flags_dev, void *stream);

/* Dense contribution matrix of render_frame(..., record_contributions=True)
 * (render.py:172-193, 229-233; replaces the contrib_out rows of
 * rasterize.py:176-177): for the frame LAST RENDERED into this workspace
 * with the same camera and config (n_ws assembled splats), out_dev[r * W*H +
 * pixel] = T * alpha of every blend of plan ref r (the r-th accepted splat in
 * assembled order) at that pixel, in fp64 with the reference's schedule.
 * out_dev must hold P x W*H doubles, zero-filled by the caller (P = accepted
 * splats); row_of_pos_dev (n_ws int32) receives the plan ref of each assembled
 * position (-1: culled / degenerate).  Stream-ordered; no sync. */
int seele_contributions(void *workspace, int64_t n_max, int64_t pair_capacity, const seele_camera *cam,
                        const seele_config *cfg, int64_t n_ws, int32_t *row_of_pos_dev, double *out_dev, void *stream);

/* frame_skip_bound (render.py:236-256, rasterize.py:325-377): per-pixel
 * certified error bound of the group-gated engine (group width cfg->group_w)
 * for the frame LAST RENDERED into this workspace with the same camera and
 * config.  bound_dev: width * height doubles, row-major.  Stream-ordered after
 * that render; does not synchronise. */
int seele_skip_bound(void *workspace, int64_t n_max, int64_t pair_capacity, const seele_camera *cam,
                     const seele_config *cfg, double *bound_dev, void *stream);

/* select_clusters (residency.py:38-54) on device: nearest 1+m centroids
 * (fp64 squared distance in pose_feature space, compiler.py:113-121; ties
 * toward the smaller id) and the working-set range table for them:
 * ranges_out[0] = shared chunk, ranges_out[1+k] = chunk of selected cluster k.
* pos_mean: HOST pointer to 3 doubles.  centroids_dev: [n_clusters][6] fp64; chunk_dev: int64 [n_clusters+1][2]
 * (start, count), entry 0 = shared.  out_ids_dev: int32 [m+1]. */
int seele_select_clusters(const seele_camera *cam, const double *centroids_dev, int32_t n_clusters,
                          int32_t m, double beta, const double *pos_mean, double pos_scale,
                          const int64_t *chunk_dev, int32_t *out_ids_dev, int64_t *ranges_out_dev,
                          void *stream);

/* Parity / debug view of the last seele_render's plan in `workspace`
 * (FramePlan, render.py:54-79).  All outputs are device pointers (nullable):
 *   pair_pos   int32 [K]      assembled position of each sorted pair's splat
 *   pair_tile  int32 [K]      tile id of each sorted pair
 *   ranges     int32 [tiles][2] (start, end) per tile, empty tiles (0, 0)
 *   status     int8  [n_ws]   0 projected, 1 near-culled, 2 degenerate
 *   depth      f64   [n_ws]   view depth (valid where status == 0)
 *   rect       int32 [n_ws][4] tile rect (tx0, tx1, ty0, ty1), empty: tx0 > tx1
 *   mean       f64   [n_ws][2], conic f64 [n_ws][3] (a, b, c), opacity f64 [n_ws],
 *   color      f32   [n_ws][3]
 * K and n_ws are read from the stats of that frame by the caller. */
typedef struct seele_plan_view {
    int32_t *pair_pos;
    int32_t *pair_tile;
    int32_t *ranges;
    int8_t *status;
    double *depth;
    int32_t *rect;
    double *mean;
    double *conic;
    double *opacity;
    float *color;
} seele_plan_view;

int seele_plan_export(void *workspace, int64_t n_max, int64_t pair_capacity, int32_t width,
                      int32_t height, int64_t n_ws, int64_t n_pairs, const seele_plan_view *out,
                      void *stream);

/* Stage timing (development / bench instrumentation).  While enabled, every
 * seele_render on this thread records CUDA events at its stage boundaries:
 * [0] preprocess, [1] depth rank (compaction + sort), [2] pair emission +
 * tile sort + ranges, [3] raster (+ fp64 fix-up).  seele_profile_read
 * synchronises on the last event and writes the n <= 4 stage times (ms) of
 * the most recent frame. */
int seele_profile_enable(int32_t on);
int seele_profile_read(float *ms_out, int32_t n);

/* Message of the last failing call on this thread ("" if none). */
const char *seele_last_error(void);

/* ABI version (bumped on any signature change). */
int32_t seele_abi_version(void);

/* Number of CUDA kernels this library has launched in this process (all
 * threads); bench.py reads it around its timed region. */
int64_t seele_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* SEELE_B200_H */
