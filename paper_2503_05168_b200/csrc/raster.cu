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
            const double2 m = ws.xrec[p].m;
            const double4 co = ws.xrec[p].co;
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

// ---------------------------------------------------------------------------
// Certified per-pixel error bound of the group-gated engine
// (skipped_contribution_bound, rasterize.py:325-377): the contribution-aware
// schedule is replayed while tracking, per pixel, the transmittance the
// reference engine would have had; every splat that blends under the
// reference schedule but not under the group-gated one adds
// T_ref * alpha * max(rgb) to the pixel's bound.  fp64, reference operation
// order; one thread per pixel, the EXACT engine's pixel / group mapping.
template <int W>
__global__ void __launch_bounds__(256) k_skip_bound(Workspace ws, const uint32_t *__restrict__ pair_pos, CamK cam,
                                                    CfgK cfg, double *bound) {
    __shared__ double s_mx[256], s_my[256], s_a[256], s_b[256], s_c[256], s_o[256];
    __shared__ float s_cmax[256];
    const int tile = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int lx, ly;
    pixel_of<W>(warp, lane, lx, ly);
    const int x = (tile % cam.tiles_x) * kTile + lx, y = (tile / cam.tiles_x) * kTile + ly;
    const bool valid = x < cam.width && y < cam.height;
    const double px = x + 0.5, py = y + 0.5;
    int leader;
    unsigned gmask;
    group_of<W>(lane, leader, gmask);
    double t_cr = 1.0, t_ref = 1.0, b = 0.0;
    bool done_cr = !valid, done_ref = !valid;
    const double th = cfg.alpha_theta, gm = cfg.gamma;
    const uint2 rg = ws.ranges[tile];
    for (uint32_t b0 = rg.x; b0 < rg.y; b0 += 256) {
        if (__syncthreads_count(!(done_cr && done_ref)) == 0) break;  // rasterize.py:350-351
        const uint32_t i = b0 + tid;
        if (i < rg.y) {
            const uint32_t p = pair_pos[i];
            const double2 m = ws.xrec[p].m;
            const double4 co = ws.xrec[p].co;
            s_mx[tid] = m.x;
            s_my[tid] = m.y;
            s_a[tid] = co.x;
            s_b[tid] = co.y;
            s_c[tid] = co.z;
            s_o[tid] = co.w;
            const RasterRec &rr = ws.rec[p];
            s_cmax[tid] = fmaxf(fmaxf(rr.r, rr.g), rr.b);
        }
        __syncthreads();
        const int nb = min(256u, rg.y - b0);
        for (int j = 0; j < nb; j++) {  // (a done pixel's updates are no-ops: no per-splat early exit needed)
            const double a = alpha64(px, py, s_mx[j], s_my[j], s_a[j], s_b[j], s_c[j], s_o[j]);
            const bool live_cr = !done_cr;
            const bool live_g = (__ballot_sync(0xffffffffu, live_cr) & gmask) != 0u;
            const double leader_a = __shfl_sync(0xffffffffu, a, leader);  // alpha taken even if the leader is done
            const bool blend_cr = live_cr && live_g && leader_a >= th && a >= th;
            const bool blend_ref = !done_ref && a >= th;
            if (blend_ref && !blend_cr) b = __dadd_rn(b, __dmul_rn(__dmul_rn(t_ref, a), (double)s_cmax[j]));
            if (blend_cr) t_cr = __dmul_rn(t_cr, __dsub_rn(1.0, a));
            done_cr = done_cr || t_cr < gm;
            if (blend_ref) t_ref = __dmul_rn(t_ref, __dsub_rn(1.0, a));
            done_ref = done_ref || t_ref < gm;
        }
    }
    if (valid) bound[(long long)y * cam.width + x] = b;
}

// ---------------------------------------------------------------------------
// Contribution harvest (compiler.py:196-231, top_contributors_per_pixel): the
// EXACT engine's schedule (reference or contribution-aware, step64 semantics),
// keeping per pixel the k strongest blend weights T * alpha (ties toward the
// smaller gaussian id, like the reference's stable id-ascending sort) in
// shared memory; every splat in some pixel's top-k with weight > 0 is flagged
// by its assembled position.
constexpr int kHarvestMax = 32;

template <int W>
__global__ void __launch_bounds__(256) k_harvest(Workspace ws, const uint32_t *__restrict__ pair_pos, CamK cam, CfgK cfg,
                                                 const int64_t *__restrict__ ids, int k, uint8_t *flags) {
    extern __shared__ __align__(16) unsigned char smem[];
    double *s_w = reinterpret_cast<double *>(smem);                   // [kHarvestMax][256]
    uint32_t *s_p = reinterpret_cast<uint32_t *>(s_w + kHarvestMax * 256);  // [kHarvestMax][256] positions
    __shared__ double s_mx[256], s_my[256], s_a[256], s_b[256], s_c[256], s_o[256];
    __shared__ uint32_t s_pp[256];
    const int tile = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int lx, ly;
    pixel_of<W>(warp, lane, lx, ly);
    const int x = (tile % cam.tiles_x) * kTile + lx, y = (tile / cam.tiles_x) * kTile + ly;
    const bool valid = x < cam.width && y < cam.height;
    const double px = x + 0.5, py = y + 0.5;
    int leader;
    unsigned gmask;
    group_of<W>(lane, leader, gmask);
    const bool is_leader = lane == leader;
    double T = 1.0;
    bool done = !valid;
    int cnt = 0, mslot = 0;
    double mw = 0.0;
    int64_t mid = 0;
    const double th = cfg.alpha_theta, gm = cfg.gamma;
    const uint2 rg = ws.ranges[tile];
    for (uint32_t b0 = rg.x; b0 < rg.y; b0 += 256) {
        if (__syncthreads_count(!done) == 0) break;
        const uint32_t i = b0 + tid;
        if (i < rg.y) {
            const uint32_t p = pair_pos[i];
            const double2 m = ws.xrec[p].m;
            const double4 co = ws.xrec[p].co;
            s_mx[tid] = m.x;
            s_my[tid] = m.y;
            s_a[tid] = co.x;
            s_b[tid] = co.y;
            s_c[tid] = co.z;
            s_o[tid] = co.w;
            s_pp[tid] = p;
        }
        __syncthreads();
        const int nb = min(256u, rg.y - b0);
        for (int j = 0; j < nb; j++) {
            const bool live = !done;
            const unsigned lb = __ballot_sync(0xffffffffu, live);
            if (lb == 0u) break;  // (warp-uniform: the model-warp stops, rasterize.py:203 per warp is equivalent here)
            double al = 0.0;
            bool blend = false;
            if (W == 0) {
                if (live) {
                    al = alpha64(px, py, s_mx[j], s_my[j], s_a[j], s_b[j], s_c[j], s_o[j]);
                    blend = al >= th;
                }
            } else {  // step64's contribution-aware gate (rasterize.py:249-322)
                const bool glive = (lb & gmask) != 0u;
                double la = 0.0;
                bool lpass = false;
                if (is_leader && glive) {
                    la = alpha64(px, py, s_mx[j], s_my[j], s_a[j], s_b[j], s_c[j], s_o[j]);
                    lpass = la >= th;
                }
                const unsigned pb = __ballot_sync(0xffffffffu, lpass);
                if (live && ((pb >> leader) & 1u)) {
                    al = is_leader ? la : alpha64(px, py, s_mx[j], s_my[j], s_a[j], s_b[j], s_c[j], s_o[j]);
                    blend = al >= th;
                }
            }
            if (blend) {
                const double w = __dmul_rn(T, al);  // the contribution row (rasterize.py:176-177)
                const uint32_t p = s_pp[j];
                const int64_t id = ids[p];
                if (cnt < k) {
                    s_w[cnt * 256 + tid] = w;
                    s_p[cnt * 256 + tid] = p;
                    cnt++;
                    if (cnt == k) {  // full: locate the weakest entry
                        mslot = 0;
                        mw = s_w[tid];
                        mid = ids[s_p[tid]];
                        for (int q = 1; q < k; q++) {
                            const double wq = s_w[q * 256 + tid];
                            const int64_t iq = ids[s_p[q * 256 + tid]];
                            if (wq < mw || (wq == mw && iq > mid)) { mslot = q; mw = wq; mid = iq; }
                        }
                    }
                } else if (w > mw || (w == mw && id < mid)) {
                    s_w[mslot * 256 + tid] = w;
                    s_p[mslot * 256 + tid] = p;
                    mslot = 0;
                    mw = s_w[tid];
                    mid = ids[s_p[tid]];
                    for (int q = 1; q < k; q++) {
                        const double wq = s_w[q * 256 + tid];
                        const int64_t iq = ids[s_p[q * 256 + tid]];
                        if (wq < mw || (wq == mw && iq > mid)) { mslot = q; mw = wq; mid = iq; }
                    }
                }
                T = __dmul_rn(T, __dsub_rn(1.0, al));
                if (T < gm) done = true;
            }
        }
    }
    for (int q = 0; q < cnt; q++)
        if (s_w[q * 256 + tid] > 0.0) flags[s_p[q * 256 + tid]] = 1u;
}

// ---------------------------------------------------------------------------
// Dense contribution matrix (render.py:172-193 with record_contributions):
// the EXACT engine's schedule, every blend writes its weight T * alpha
// (rasterize.py:176-177) to out[row_of_pos[p] * n_pix + pixel], row = the
// splat's plan ref.  The caller zero-fills out (P x H*W fp64).
template <int W>
__global__ void __launch_bounds__(256) k_contrib(Workspace ws, const uint32_t *__restrict__ pair_pos, CamK cam,
                                                 CfgK cfg, const int32_t *__restrict__ row_of_pos, double *out) {
    __shared__ double s_mx[256], s_my[256], s_a[256], s_b[256], s_c[256], s_o[256];
    __shared__ uint32_t s_p[256];
    const int tile = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int lx, ly;
    pixel_of<W>(warp, lane, lx, ly);
    const int x = (tile % cam.tiles_x) * kTile + lx, y = (tile / cam.tiles_x) * kTile + ly;
    const bool valid = x < cam.width && y < cam.height;
    const double px = x + 0.5, py = y + 0.5;
    const long long n_pix = (long long)cam.width * cam.height, pix = (long long)y * cam.width + x;
    int leader;
    unsigned gmask;
    group_of<W>(lane, leader, gmask);
    const bool is_leader = lane == leader;
    Px64 s{1.0, 0.0, 0.0, 0.0, 0, !valid};
    Counters k{0, 0, 0};
    const uint2 rg = ws.ranges[tile];
    for (uint32_t b0 = rg.x; b0 < rg.y; b0 += 256) {
        if (__syncthreads_count(!s.done) == 0) break;
        const uint32_t i = b0 + tid;
        if (i < rg.y) {
            const uint32_t p = pair_pos[i];
            const double2 m = ws.xrec[p].m;
            const double4 co = ws.xrec[p].co;
            s_mx[tid] = m.x;
            s_my[tid] = m.y;
            s_a[tid] = co.x;
            s_b[tid] = co.y;
            s_c[tid] = co.z;
            s_o[tid] = co.w;
            s_p[tid] = p;
        }
        __syncthreads();
        const int nb = min(256u, rg.y - b0);
        for (int j = 0; j < nb; j++) {
            const int cnt0 = s.cnt;
            double w = 0.0;
            if (!step64<W>(s, px, py, is_leader, leader, gmask, s_mx[j], s_my[j], s_a[j], s_b[j], s_c[j], s_o[j], 0.f,
                           0.f, 0.f, cfg.alpha_theta, cfg.gamma, k, &w))
                break;
            if (s.cnt != cnt0 && valid) out[(long long)row_of_pos[s_p[j]] * n_pix + pix] = w;
        }
    }
}

// Plan ref of every assembled position (exclusive scan of status == 0; -1
// for rejected splats), one CTA.
__global__ void __launch_bounds__(1024) k_row_of_pos(Workspace ws, long long n_ws, int32_t *row_of_pos) {
    __shared__ int32_t s_w[32];
    __shared__ int32_t s_base;
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (long long b = 0; b < n_ws; b += 1024) {
        const long long p = b + threadIdx.x;
        const bool ok = p < n_ws && ws.status[p] == 0;
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        if (lane == 0) s_w[warp] = __popc(bal);
        __syncthreads();
        int before = s_base;
        for (int w = 0; w < warp; w++) before += s_w[w];
        before += __popc(bal & ((1u << lane) - 1u));
        if (p < n_ws) row_of_pos[p] = ok ? before : -1;
        __syncthreads();
        if (threadIdx.x == 0) {
            int t = 0;
            for (int w = 0; w < 32; w++) t += s_w[w];
            s_base += t;
        }
        __syncthreads();
    }
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

void launch_skip_bound(int group_w, const Workspace &ws, const uint32_t *pair_pos, const CamK &cam, const CfgK &cfg,
                       double *bound, cudaStream_t st) {
    const int n_tiles = cam.tiles_x * cam.tiles_y;
    switch (group_w) {
        case 1: k_skip_bound<1><<<n_tiles, 256, 0, st>>>(ws, pair_pos, cam, cfg, bound); break;
        case 2: k_skip_bound<2><<<n_tiles, 256, 0, st>>>(ws, pair_pos, cam, cfg, bound); break;
        default: k_skip_bound<4><<<n_tiles, 256, 0, st>>>(ws, pair_pos, cam, cfg, bound); break;
    }
    note_launches(1);
}

void launch_harvest(int engine_w, const Workspace &ws, const uint32_t *pair_pos, const CamK &cam, const CfgK &cfg,
                    const int64_t *ids, int k, uint8_t *flags, cudaStream_t st) {
    const int n_tiles = cam.tiles_x * cam.tiles_y;
    const size_t smem = (size_t)kHarvestMax * 256 * (sizeof(double) + sizeof(uint32_t));
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_harvest<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_harvest<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_harvest<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_harvest<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    switch (engine_w) {
        case 0: k_harvest<0><<<n_tiles, 256, smem, st>>>(ws, pair_pos, cam, cfg, ids, k, flags); break;
        case 1: k_harvest<1><<<n_tiles, 256, smem, st>>>(ws, pair_pos, cam, cfg, ids, k, flags); break;
        case 2: k_harvest<2><<<n_tiles, 256, smem, st>>>(ws, pair_pos, cam, cfg, ids, k, flags); break;
        default: k_harvest<4><<<n_tiles, 256, smem, st>>>(ws, pair_pos, cam, cfg, ids, k, flags); break;
    }
    note_launches(1);
}

void launch_contributions(int engine_w, const Workspace &ws, const uint32_t *pair_pos, const CamK &cam,
                          const CfgK &cfg, long long n_ws, int32_t *row_of_pos, double *out, cudaStream_t st) {
    const int n_tiles = cam.tiles_x * cam.tiles_y;
    k_row_of_pos<<<1, 1024, 0, st>>>(ws, n_ws, row_of_pos);
    switch (engine_w) {
        case 0: k_contrib<0><<<n_tiles, 256, 0, st>>>(ws, pair_pos, cam, cfg, row_of_pos, out); break;
        case 1: k_contrib<1><<<n_tiles, 256, 0, st>>>(ws, pair_pos, cam, cfg, row_of_pos, out); break;
        case 2: k_contrib<2><<<n_tiles, 256, 0, st>>>(ws, pair_pos, cam, cfg, row_of_pos, out); break;
        default: k_contrib<4><<<n_tiles, 256, 0, st>>>(ws, pair_pos, cam, cfg, row_of_pos, out); break;
    }
    note_launches(2);
}

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
