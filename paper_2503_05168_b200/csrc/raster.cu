// Tile rasterization on sm_100a: reference engine (rasterize.py:180-232) and
// contribution-aware engine (rasterize.py:249-322), with the reference's
// 32-lane lockstep cost counters (rasterize.py:208-223, 291-313).
//
// EXACT mapping: one CTA per 16x16 tile, one thread per pixel, and every
// hardware warp IS one of the reference's model-warps:
//   ref / cr w=1 / cr w=2 : warp k = tile pixel rows 2k, 2k+1
//   cr w=4                : warp k = 8x4 block (groups 2k, 2k+1 group-row-major)
// so the counters are __any_sync votes of the real warp, the CR leader test is
// broadcast with one ballot, and a model-warp's result depends only on its own
// 32 lanes and the tile's sorted list.  Splat batches are staged in shared
// memory 256 at a time; a tile stops when every pixel is done (rasterize.py:203).
//
// Two precisions give the same discrete result (contributor counts, done
// decisions, counters):
//  * EXACT: alpha and transmittance in fp64 in the reference's operation
//    order (libdevice exp).
//  * FAST (default, raster_fast.cu): 2x2 pixels per thread, fp64 q, fp32
//    alpha with certified error bounds; undecidable tests are re-decided
//    exactly in fp64 in place.
#include "raster_common.cuh"

namespace seele {

using namespace rast;

namespace {
// ---------------------------------------------------------------------------
// EXACT engine: fp64 throughout.
template <int W>
__global__ void __launch_bounds__(256) k_raster_exact(Workspace ws, const uint32_t *__restrict__ pair_pos, CamK cam,
                                                      CfgK cfg, float *image, int32_t *contrib, int64_t *stats) {
    __shared__ double s_mx[256], s_my[256], s_a[256], s_b[256], s_c[256], s_o[256];
    __shared__ float4 s_col[256];
    const int tile = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int lx, ly;
    pixel_of<W>(warp, lane, lx, ly);
    const int x = (tile % cam.tiles_x) * kTile + lx, y = (tile / cam.tiles_x) * kTile + ly;
    const bool valid = x < cam.width && y < cam.height;
    const double px = x + 0.5, py = y + 0.5;  // pixel centres (rasterize.py:122)
    int leader;
    unsigned gmask;
    group_of<W>(lane, leader, gmask);
    const bool is_leader = lane == leader;
    Px64 s{1.0, 0.0, 0.0, 0.0, 0, !valid};
    Counters k{0, 0, 0};
    const uint2 rg = ws.ranges[tile];
    for (uint32_t b0 = rg.x; b0 < rg.y; b0 += 256) {
        if (__syncthreads_count(!s.done) == 0) break;  // tile stops when every pixel is done
        const uint32_t i = b0 + tid;
        if (i < rg.y) {
            const uint32_t p = pair_pos[i];
            const double2 m = ws.mean[p];
            const double4 co = ws.conic_op[p];
            s_mx[tid] = m.x;
            s_my[tid] = m.y;
            s_a[tid] = co.x;
            s_b[tid] = co.y;
            s_c[tid] = co.z;
            s_o[tid] = co.w;
            const RasterRec &rr = ws.rec[p];
            s_col[tid] = make_float4(rr.r, rr.g, rr.b, 0.f);
        }
        __syncthreads();
        const int nb = min(256u, rg.y - b0);
        for (int j = 0; j < nb; j++) {
            const float4 col = s_col[j];
            if (!step64<W>(s, px, py, is_leader, leader, gmask, s_mx[j], s_my[j], s_a[j], s_b[j], s_c[j], s_o[j], col.x,
                           col.y, col.z, cfg.alpha_theta, cfg.gamma, k))
                break;
        }
    }
    if (valid) write_pixel(image, contrib, cam.width, x, y, s.C0, s.C1, s.C2, s.T, s.cnt, cfg);
    if (lane == 0) add_counters<W>(stats, k);
}

template <int W>
void launch_engine(const Workspace &ws, const uint32_t *pair_pos, const CamK &cam, const CfgK &cfg, float *image,
                   int32_t *contrib, int64_t *stats, cudaStream_t st) {
    const int n_tiles = cam.tiles_x * cam.tiles_y;
    if (cfg.precision == SEELE_PRECISION_EXACT) {
        k_raster_exact<W><<<n_tiles, 256, 0, st>>>(ws, pair_pos, cam, cfg, image, contrib, stats);
        note_launches(1);
    } else {
        launch_raster_fast(W, ws, pair_pos, cam, cfg, image, contrib, stats, st);
        note_launches(1);
    }
}

}  // namespace

void launch_raster(const Workspace &ws, const uint32_t *pair_pos, const CamK &cam, const CfgK &cfg, float *image,
                   int32_t *contrib, int64_t *stats, cudaStream_t st) {
    const int w = cfg.engine == 0 ? 0 : cfg.group_w;
    switch (w) {
        case 0: launch_engine<0>(ws, pair_pos, cam, cfg, image, contrib, stats, st); break;
        case 1: launch_engine<1>(ws, pair_pos, cam, cfg, image, contrib, stats, st); break;
        case 2: launch_engine<2>(ws, pair_pos, cam, cfg, image, contrib, stats, st); break;
        default: launch_engine<4>(ws, pair_pos, cam, cfg, image, contrib, stats, st); break;
    }
}

}  // namespace seele
