// Internal declarations shared by the sm_100a kernels of the Seele render path.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/seele_b200.h"

namespace seele {

constexpr int kTile = 16;            // TILE_SIZE (model.py:17)
constexpr int kTilePixels = 256;
constexpr int kWarp = 32;            // WARP_SIZE (rasterize.py:30)
constexpr double kAlphaClamp = 0.99; // ALPHA_CLAMP (rasterize.py:32)

// Per-frame camera constants, computed once on the host in fp64 exactly as
// CameraPose.focal / principal_point / rotation_matrix do (model.py:170-184).
struct CamK {
    double w2v[9];  // world_to_view = R_cw^T (preprocess.py:99), row-major
    double pos[3];
    double fx, fy, cx, cy, near_clip;
    int width, height, tiles_x, tiles_y;
};

struct CfgK {
    int engine, group_w, sh_degree, opacity_aware, precision;
    int keep_unbinned;  // SEELE_KEEP_UNBINNED: records of projected splats that bin to no tile (plan export)
    double alpha_theta, gamma;
    double bg[3];
    // gamma as floats rounded up / down (set_gamma): the FAST raster proves T >= gamma with gamma_up and
    // T < gamma with gamma_dn
    float gamma_up, gamma_dn;
};
inline void set_gamma(CfgK &c, double g) {
    c.gamma = g;
    float up = (float)g, dn = (float)g;
    if ((double)up < g) up = nextafterf(up, INFINITY);
    if ((double)dn > g) dn = nextafterf(dn, -INFINITY);
    c.gamma_up = up;
    c.gamma_dn = dn;
}

struct SceneK {
    int layout;
    long long n;
    const double *pos, *log_scale, *rot, *opac, *sh;
    const float4 *planes;
    long long plane_stride;
};

// Scalar counters living in the workspace (device), zeroed by every frame.
enum {
    CNT_WS = 0,           // assembled splats
    CNT_PAIRS = 2,        // tile pairs (0 on overflow; the u64 count is in stats)
    CNT_OVERFLOW = 3,
    CNT_SEGS = 5,         // super-tile list segments of the expand pass
    CNT_DONE_SCAN = 6,    // last-block ticket of the binning scan
    CNT_TICKET = 8,       // 16 per-pass tile tickets
    CNT_COUNT = 32
};

#ifndef SEELE_SORT_NT
#define SEELE_SORT_NT 512
#endif
#ifndef SEELE_SORT_IPT
#define SEELE_SORT_IPT 8
#endif
constexpr int kMaxTileAxis = 256;  // tiles per image axis (packed 8-bit tile rects)
constexpr int kLookBuckets = 3;    // look-back epoch tag of the depth bucket scan
constexpr int kLookSegs = 4;       // look-back epoch tag of the binning expand pass

// Binning (binning.cu): depth ranks cut into chunks of ~kBinChunkRanks (at least kBinChunksMin), super-tiles
// of 4 x 4 tiles.
#ifndef SEELE_BIN_CHUNK_RANKS
#define SEELE_BIN_CHUNK_RANKS 4096
#endif
constexpr long long kBinChunkRanks = SEELE_BIN_CHUNK_RANKS;
constexpr int kBinChunksMin = 64;
constexpr int kBinChunksMax = 4096;
constexpr int kSeg = 2048;  // entries per super-tile list segment (expand pass)
struct BinGeom {
    int tiles_x, tiles_y, stx, sty, n_st, n_chunks;
    int count_group;  // chunks per k_bin_count CTA
};
BinGeom bin_geometry(long long n_max, int width, int height);
// SMs of the device, and of the SM partition a stream belongs to (partition.cu; the device's when the
// stream is not a partition stream): persistent grids are sized by the latter
int stream_sms(cudaStream_t st);
int partition_create(int plan_sms, int n_streams, void **plan_streams, void **raster_streams, int *plan_out,
                     int *raster_out);

// Depth order (depth.cu): buckets of the order-preserving fp64 bit pattern of
// z above the near plane, 2^(52 - kDepthShift) = 65,536 per binade over 16
// binades (deeper splats share the last bucket); groups of ~kDepthGroup
// items are sorted exactly by (depth, position) by one CTA each.
constexpr int kDepthBuckets = 1 << 20;
constexpr int kDepthShift = 36;
constexpr int kDepthScanItems = 16384;  // buckets per CTA of the offset scan
constexpr int kDepthGroup = 1024;
constexpr int kDepthSmem = 2048;  // items a sort CTA holds in shared memory
constexpr int kDepthFinal = 0;    // dval / drect buffer holding the sorted order

__device__ __forceinline__ unsigned long long depth_order_key(double z) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(z);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);  // monotone in z over all finite doubles
}
__device__ __forceinline__ uint32_t depth_bucket_of_key(unsigned long long key, unsigned long long base) {
    const unsigned long long q = key > base ? (key - base) >> kDepthShift : 0ull;
    return q < (unsigned long long)(kDepthBuckets - 1) ? (uint32_t)q : (uint32_t)(kDepthBuckets - 1);
}

__device__ __forceinline__ uint32_t pack_rect(short4 r) {
    return (uint32_t)(r.x & 0xff) | ((uint32_t)(r.y & 0xff) << 8) | ((uint32_t)(r.z & 0xff) << 16) |
           ((uint32_t)(r.w & 0xff) << 24);
}

// FAST raster record of one splat (raster_fast.cu), written by preprocess.
// q' = q log2(e) / 2, so alpha = o 2^-q'; one 64-byte line, staged into
// shared memory by four 16-byte cp.async per splat.
struct __align__(16) RasterRec {
    // mean in pixel coordinates: hi floats, the lo parts (m - hi, ~2^-24 |m|) folded into the Cholesky
    // coordinates: u = l11 (x - mxh) + l21 (y - myh) - cu, w = l22 (y - myh) - cw
    float mxh, cu, myh, cw;
    float l11, l21, l22, o;    // Cholesky factor of the conic in q' units; opacity
    float q_lo, w_up, e0, e1;  // pass: q' < q_lo; in the bracket (re-decided): 0 <= q' - q_lo <= w_up, else
                               // fail; alpha relative error <= e0 + e1 q'
    float r, g, b;             // colour
    uint32_t p;                // assembled position (fp64 re-decisions)
};

// fp64 record of one binned splat for the exact paths (re-decisions, transmittance walks, the EXACT
// engine, plan export): everything a walk reads per splat in one 64-byte line (two 32-byte sectors)
// instead of three lines of three arrays.
struct __align__(64) ExactRec {
    double2 m;       // mean (pixel coordinates)
    double4 co;      // conic (a, b, c), opacity
    float q_lo, w_up;  // the FAST record's alpha bracket (RasterRec)
    uint32_t pad[2];
};

// Workspace carve-up; identical on every call for the same (n_max, cap, w, h).
struct Workspace {
    // per assembled splat (preprocess)
    uint8_t *status;
    // per assembled splat: tile rect packed in bytes (x0 | x1 << 8 | y0 << 16 | y1 << 24; x0 > x1: not binned),
    // its index in its depth bucket, the fp64 view depth (bits): one 16-byte record, what the depth scatter reads
    uint4 *srec;
    ExactRec *xrec;      // fp64 mean, conic + opacity, alpha bracket: the exact paths' record, one line
    RasterRec *rec;      // FAST raster records (also the colour of the exact engine)
    // depth order (depth.cu): bucket counts (K1) -> exclusive offsets, bhist[kDepthBuckets] = binned; each
    // binned splat's index inside its bucket (K1's atomic); bucket-order records (order key lo / hi, position,
    // packed tile rect x0 | x1 << 8 | y0 << 16 | y1 << 24) in brec[0] (brec[1]: merge buffer of large groups);
    // first bucket of each sort group; the sorted order in dval[0] / drect[0] (dval[1] / drect[1]: unused)
    uint32_t *bhist;     // [kDepthBuckets + 1]
    uint4 *brec[2];      // [n_max]
    uint32_t *gfirst;    // [n_max / kDepthGroup + 2]
    uint32_t *dval[2];
    uint32_t *drect[2];
    // binning (binning.cu): chunk x super-tile entry counts -> exclusive chunk bases; entries per super-tile,
    // list offsets, heavy-first order; entries (position, sub-rectangle) grouped by super-tile in depth order
    uint32_t *cmat;      // [n_chunks][n_st]
    uint32_t *st_cnt;    // [n_st]
    uint32_t *st_start;  // [n_st + 1]
    uint32_t *seg_first; // [n_st + 1] first list segment of each super-tile
    uint32_t *seg_st;    // [cap / kSeg + n_st + 1] super-tile of each segment
    unsigned long long *seg_look;  // [cap / kSeg + n_st + 1][16] epoch-tagged look-back words (never cleared)
    uint32_t *head_cnt;  // [tiles] pairs of the head ranks (chunk 0) per tile
    uint2 *ent;          // [cap]
    uint32_t *pfinal;    // sorted pair -> assembled position (sort_intersections order)
    uint2 *ranges;       // per tile [start, end)
    uint32_t *tile_order;  // raster launch order: tiles by descending pair count (heavy tiles first)
    // scratch
    unsigned long long *look;  // epoch-tagged look-back status words (depth bucket scan)
    int32_t *tile_diff;  // [(tiles_y + 1) x (tiles_x + 1)] 2D difference array of tile counts
    uint32_t *counters;  // CNT_COUNT
    uint32_t *epoch;     // frame epoch (never cleared)
    unsigned long long *pairs64;  // total tile pairs (u64)
    size_t bytes;

    int64_t *stats_ptr;  // the frame's stats vector (set by seele_render)
    __device__ __forceinline__ long long counters_binned() const { return stats_ptr[SEELE_STAT_BINNED]; }

    __device__ __forceinline__ unsigned long long *look_region(int) const { return look; }
};

Workspace carve_workspace(void *base, long long n_max, long long cap, int width, int height);

// ---- launch helpers (defined in the .cu files) -----------------------------
void launch_preprocess(const SceneK &s, const int64_t *ranges, int n_ranges, const CamK &cam,
                       const CfgK &cfg, const Workspace &ws, int64_t *stats, int grid,
                       cudaStream_t st);
void launch_select(const CamK &cam, const double *centroids, int n, int m, double beta,
                   const double *mean3, double scale, const int64_t *chunks, int32_t *out_ids,
                   int64_t *ranges_out, cudaStream_t st);
// frame start: counters, stats, epoch, range / histogram init (binning.cu)
void launch_frame_begin(const Workspace &ws, const CamK &cam, int64_t *stats, cudaStream_t st);
// exact (depth, position) order of the binned splats (depth.cu).
void launch_depth_sort(const Workspace &ws, const CamK &cam, long long n_max, int64_t *stats, cudaStream_t st);
// tile pairs in sort_intersections order: ranges, final pair -> position in ws.pfinal.
void launch_binning(const Workspace &ws, long long n_max, long long cap, const CamK &cam, int64_t *stats,
                    cudaStream_t st);
void launch_raster(const Workspace &ws, const uint32_t *pair_pos, const CamK &cam,
                   const CfgK &cfg, float *image, int32_t *contrib, int64_t *stats,
                   cudaStream_t st);
// FAST engine tile kernel (raster_fast.cu); W = 0 (ref) or CR group width.
void launch_harvest(int engine_w, const Workspace &ws, const uint32_t *pair_pos, const CamK &cam, const CfgK &cfg,
                    const int64_t *ids, int k, uint8_t *flags, cudaStream_t st);
void launch_contributions(int engine_w, const Workspace &ws, const uint32_t *pair_pos, const CamK &cam,
                          const CfgK &cfg, long long n_ws, int32_t *row_of_pos, double *out, cudaStream_t st);
void launch_skip_bound(int group_w, const Workspace &ws, const uint32_t *pair_pos, const CamK &cam, const CfgK &cfg,
                       double *bound, cudaStream_t st);
void launch_raster_fast(int W, const Workspace &ws, const uint32_t *pair_pos, const CamK &cam,
                        const CfgK &cfg, float *image, int32_t *contrib, int64_t *stats,
                        cudaStream_t st);


void launch_fill_pair_tiles(const uint2 *ranges, int n_tiles, int32_t *pair_tile, cudaStream_t st);

// Counts kernels this library has launched (seele_launch_count, api.cu).
void note_launches(int n);

}  // namespace seele
