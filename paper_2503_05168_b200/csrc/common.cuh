// Internal declarations shared by the sm_100a kernels of the Seele render path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/seele_b200.h"

namespace seele {

constexpr int kTile = 16;            // TILE_SIZE (model.py:17)
constexpr int kTilePixels = 256;
constexpr int kWarp = 32;            // WARP_SIZE (rasterize.py:30)
constexpr double kAlphaClamp = 0.99; // ALPHA_CLAMP (rasterize.py:32)
constexpr int kChunkBlocksMax = 2048;  // upper bound of the chunked scan / sort grid
constexpr int kSortBlock = 256;

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
    double alpha_theta, gamma;
    double bg[3];
};

struct SceneK {
    int layout;
    long long n;
    const double *pos, *log_scale, *rot, *opac, *sh;
    const float4 *planes;
    long long plane_stride;
};

// Scalar counters living in the workspace (device).
enum {
    CNT_WS = 0,      // assembled splats
    CNT_BINNED = 1,  // splats with >= 1 tile
    CNT_PAIRS = 2,   // tile pairs (0 on overflow; the u64 count is in stats)
    CNT_OVERFLOW = 3,
    CNT_COUNT = 8
};

// Workspace carve-up; identical on every call for the same (n_max, cap, w, h).
struct Workspace {
    // per assembled splat
    uint8_t *status;
    double *depth;
    uint32_t *tiles;
    short4 *rect;
    double2 *mean;
    double4 *conic_op;   // (a, b, c, opacity)
    float4 *color;       // (r, g, b, 0)
    float4 *fast;        // FAST raster: (q_lo, q_hi, opacity32, 0) alpha-test bracket in q
    // compaction + depth rank
    uint64_t *dkey[2];
    uint32_t *dval[2];
    // first pair of each depth-ranked splat (+ total); u64 to detect overflow
    unsigned long long *poff;
    uint32_t *tile_r0;   // first rank of each 2048-pair emission tile
    // pairs
    uint32_t *pkey[2];
    uint32_t *pval[2];
    uint2 *ranges;
    // scan / sort scratch
    unsigned long long *block_sums;  // kChunkBlocksMax + 1
    uint32_t *hist;                  // 256 * kChunkBlocksMax
    uint32_t *counters;              // CNT_COUNT
    unsigned long long *pairs64;     // total tile pairs (u64)
    size_t bytes;
};

Workspace carve_workspace(void *base, long long n_max, long long cap, int width, int height);

// ---- launch helpers (defined in the .cu files) -----------------------------
void launch_preprocess(const SceneK &s, const int64_t *ranges, int n_ranges, const CamK &cam,
                       const CfgK &cfg, const Workspace &ws, int64_t *stats, int grid,
                       cudaStream_t st);
void launch_select(const CamK &cam, const double *centroids, int n, int m, double beta,
                   const double *mean3, double scale, const int64_t *chunks, int32_t *out_ids,
                   int64_t *ranges_out, cudaStream_t st);
// compaction of binned splats in assembled order + stable depth sort.
// Returns pointers (inside ws) of the depth-sorted positions via *sorted_pos.
void launch_depth_rank(const Workspace &ws, long long n_max, int grid, int64_t *stats,
                       uint32_t **sorted_pos, cudaStream_t st);
void launch_binning(const Workspace &ws, const uint32_t *sorted_pos, long long n_max, long long cap,
                    const CamK &cam, int grid, int64_t *stats, uint32_t **pair_pos,
                    uint32_t **pair_tile, cudaStream_t st);
void launch_raster(const Workspace &ws, const uint32_t *pair_pos, const CamK &cam,
                   const CfgK &cfg, float *image, int32_t *contrib, int64_t *stats,
                   cudaStream_t st);
// FAST engine tile kernel (raster_fast.cu); W = 0 (ref) or CR group width.
void launch_raster_fast(int W, const Workspace &ws, const uint32_t *pair_pos, const CamK &cam,
                        const CfgK &cfg, float *image, int32_t *contrib, int64_t *stats,
                        cudaStream_t st);

// grid of the chunked scan / sort kernels (binning.cu)
int chunk_grid(int sms);
int pair_buffer(int n_tiles);      // ping-pong buffer holding the sorted pairs

// Counts kernels this library has launched (seele_launch_count, api.cu).
void note_launches(int n);

}  // namespace seele
