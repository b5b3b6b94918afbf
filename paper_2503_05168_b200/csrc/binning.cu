// Tile binning and the tile sort on sm_100a, over the binned splats in exact
// (depth, position) order (depth.cu).  The output is sort_intersections'
// order (sorting.py:32-54): pairs grouped by tile id, inside a tile by depth
// rank.  Depth order -> tile order is a transpose; it is done in two stable
// partitions, each counted up front so no pass has a look-back chain:
//
//   count   k_bin_count: the depth ranks are cut into C equal chunks; every
//           chunk counts its entries per super-tile (4 x 4 tiles, 64 x 64
//           pixels) -- a splat makes one entry per super-tile its tile rect
//           (bin_tiles, preprocess.py:159-189) touches -- into row c of a
//           C x S count matrix, and adds its rect to the 2D difference array
//           of per-tile pair counts (both by 2D difference arrays: four
//           shared-memory atomics per splat, whatever its size).
//   scan    k_bin_scan: exclusive scan of every super-tile column of the
//           count matrix over the chunks (in place: chunk c's first entry
//           slot inside super-tile s's list); the last CTA scans the
//           super-tile totals into list offsets and cuts every list into
//           segments of kSeg entries, turns the difference array into
//           per-tile counts and the tile ranges (sorting.py:46-53), and
//           orders the tiles heavy-first for the raster.
//   split   k_bin_split: each chunk re-reads its ranks and writes every entry
//           (position, the rect's 2-bit sub-rectangle inside the super-tile)
//           to its slot: chunk base + earlier warps of the chunk (per-warp
//           counts, scanned across warps) + earlier ranks of the warp round
//           (lane masks per super-tile, popc below the lane).
//   head    k_bin_head: chunk 0 -- the nearest, largest splats -- is not put
//           in the lists; one warp per tile pulls its pairs (they precede
//           every later rank in the tile).
//   expand  k_bin_expand takes the lists in segments of kSeg entries: every
//           entry covers a subset of the super-tile's 16 tiles, one ballot
//           per tile ranks it among the segment's warps, a decoupled look-back
//           along the super-tile's segments adds the pairs of earlier
//           segments, and the pairs are written with one coalesced store per
//           tile into ranges[tile].x + head pairs + earlier segments' pairs +
//           running count.
//
// Every size is read from device memory: a frame needs no host round trip.
#include <algorithm>

#include "onesweep.cuh"

namespace seele {

namespace {

constexpr int kSt = 4;  // super-tile edge in tiles
constexpr int kCountThreads = 256;
constexpr int kScanThreads = sweep::NT;  // 512 (block_scan)
#ifndef SEELE_EXPAND_THREADS
#define SEELE_EXPAND_THREADS 256
#endif
constexpr int kExpandThreads = SEELE_EXPAND_THREADS;  // 8 batches of 8 warps / 4 of 16 / 2 of 32 per segment
#ifndef SEELE_EXPAND_MINB
#define SEELE_EXPAND_MINB (1024 / SEELE_EXPAND_THREADS)
#endif
#ifndef SEELE_SPLIT_NW
#define SEELE_SPLIT_NW 16
#endif

// ---- frame start ---------------------------------------------------------------

__global__ void k_frame_begin(Workspace ws, int64_t *stats, int n_diff) {
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    if (tid == 0) {
        *ws.epoch += 1u;
        *ws.pairs64 = 0ull;
    }
    if (tid < SEELE_STAT_COUNT) stats[tid] = 0;
    if (tid < CNT_COUNT) ws.counters[tid] = 0u;
    for (int i = tid; i < kDepthBuckets / 4; i += stride) reinterpret_cast<uint4 *>(ws.bhist)[i] = make_uint4(0, 0, 0, 0);
    for (int i = tid; i < n_diff; i += stride) ws.tile_diff[i] = 0;
}

struct Rect {
    uint32_t x0, x1, y0, y1;
};
__device__ __forceinline__ Rect unpack_rect(uint32_t v) {
    return Rect{v & 0xffu, (v >> 8) & 0xffu, (v >> 16) & 0xffu, v >> 24};
}

// chunk c of the depth ranks: [c * K, min(n, (c + 1) * K)), K = ceil(n / C)
__device__ __forceinline__ void chunk_range(uint32_t n, uint32_t C, uint32_t c, uint32_t &r0, uint32_t &r1) {
    const uint32_t K = (n + C - 1) / C;
    r0 = min(n, c * K);
    r1 = min(n, r0 + K);
}

// ---- count -----------------------------------------------------------------------

// super-tile rect of a tile rect
struct StRect {
    uint32_t x0, x1, y0, y1;
};
__device__ __forceinline__ StRect st_rect(const Rect &rc) {
    return StRect{rc.x0 / kSt, rc.x1 / kSt, rc.y0 / kSt, rc.y1 / kSt};
}

// 2D inclusive prefix in place over rows [0, ny) x columns [0, nx) of a
// row-major array with row stride `stride`, by one warp (rows lane-parallel,
// then columns).
template <typename T>
__device__ __forceinline__ void warp_prefix2d(T *a, int nx, int ny, int stride) {
    const int lane = threadIdx.x & 31;
    const int per = (nx + 31) / 32;
    for (int y = 0; y < ny; y++) {
        T *row = a + y * stride;
        T run = 0;
        for (int j = 0; j < per; j++) {
            const int x = lane * per + j;
            if (x < nx) run += row[x];
        }
        T incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        T acc = incl - run;
        for (int j = 0; j < per; j++) {
            const int x = lane * per + j;
            if (x < nx) {
                acc += row[x];
                row[x] = acc;
            }
        }
    }
    __syncwarp();
    for (int x = lane; x < nx; x += 32) {
        T acc = 0;
        for (int y = 0; y < ny; y++) {
            acc += a[y * stride + x];
            a[y * stride + x] = acc;
        }
    }
    __syncwarp();
}

// One CTA per g.count_group (<= kCountMaxGroup) consecutive chunks, one warp per chunk for the prefix.
// Shared memory: per chunk a 2D difference array over the super-tile grid (-> entries per super-tile),
// then (if it fits) the CTA's one over the tile grid, flushed into the frame's by atomics on its nonzero
// cells.  Four shared-memory atomics per splat each, whatever its size.  Chunk 0 is the head
// (k_bin_head): no super-tile entries.
constexpr int kCountMaxGroup = kCountThreads / 32;
constexpr int kCountUnroll = 4;  // rects in flight per thread
__global__ void __launch_bounds__(kCountThreads) k_bin_count(Workspace ws, BinGeom g, int diff_in_smem) {
    extern __shared__ int32_t s_cnt[];  // [group][(sty + 1) * (stx + 1)] then [(tiles_y + 1) * (tiles_x + 1)]
    const int G = g.count_group;
    const int sx1 = g.stx + 1, n_sd = sx1 * (g.sty + 1);
    int32_t *s_diff = s_cnt + G * n_sd;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int tx1 = g.tiles_x + 1, n_diff = tx1 * (g.tiles_y + 1);
    for (int i = tid; i < G * n_sd; i += kCountThreads) s_cnt[i] = 0;
    if (diff_in_smem)
        for (int i = tid; i < n_diff; i += kCountThreads) s_diff[i] = 0;
    __syncthreads();
    int32_t *diff = diff_in_smem ? s_diff : ws.tile_diff;
    const uint32_t n = (uint32_t)ws.stats_ptr[SEELE_STAT_BINNED];
    const uint32_t C = (uint32_t)g.n_chunks, K = (n + C - 1) / C;
    const uint32_t c0 = blockIdx.x * (uint32_t)G;
    const uint32_t r0 = min(n, c0 * K), r1 = min(n, r0 + (uint32_t)G * K);
    const uint32_t *srect = ws.drect[kDepthFinal];
    unsigned long long pairs = 0ull;
    for (uint32_t rb = r0 + tid; rb < r1; rb += kCountUnroll * kCountThreads) {
        uint32_t v[kCountUnroll];
#pragma unroll
        for (int u = 0; u < kCountUnroll; u++) {
            const uint32_t r = rb + u * kCountThreads;
            v[u] = r < r1 ? srect[r] : 0u;
        }
#pragma unroll
        for (int u = 0; u < kCountUnroll; u++) {
            const uint32_t r = rb + u * kCountThreads;
            if (r >= r1) break;
            const Rect rc = unpack_rect(v[u]);
            pairs += (unsigned long long)((rc.x1 - rc.x0 + 1) * (rc.y1 - rc.y0 + 1));
            atomicAdd(&diff[rc.y0 * tx1 + rc.x0], 1);
            atomicAdd(&diff[rc.y0 * tx1 + rc.x1 + 1], -1);
            atomicAdd(&diff[(rc.y1 + 1) * tx1 + rc.x0], -1);
            atomicAdd(&diff[(rc.y1 + 1) * tx1 + rc.x1 + 1], 1);
            const uint32_t c = r / K;
            if (c == 0) continue;  // the head: emitted per tile (k_bin_head), not in the lists
            int32_t *sd = s_cnt + (c - c0) * n_sd;
            const StRect sr = st_rect(rc);
            atomicAdd(&sd[sr.y0 * sx1 + sr.x0], 1);
            atomicAdd(&sd[sr.y0 * sx1 + sr.x1 + 1], -1);
            atomicAdd(&sd[(sr.y1 + 1) * sx1 + sr.x0], -1);
            atomicAdd(&sd[(sr.y1 + 1) * sx1 + sr.x1 + 1], 1);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pairs += __shfl_xor_sync(0xffffffffu, pairs, o);
    if ((tid & 31) == 0 && pairs) atomicAdd(ws.pairs64, pairs);
    __syncthreads();
    const uint32_t c = c0 + warp;
    if (warp < G && c < C) {
        int32_t *sd = s_cnt + warp * n_sd;
        warp_prefix2d(sd, g.stx, g.sty, sx1);
        uint32_t *row = ws.cmat + (size_t)c * g.n_st;
        for (int i = tid & 31; i < g.n_st; i += 32) row[i] = (uint32_t)sd[(i / g.stx) * sx1 + i % g.stx];
    }
    if (diff_in_smem)
        for (int i = tid; i < n_diff; i += kCountThreads)
            if (s_diff[i]) atomicAdd(&ws.tile_diff[i], s_diff[i]);
}

// ---- scan ------------------------------------------------------------------------

// raster launch order bucket of a tile with c pairs: 32 - bits(c), heavy tiles first
__device__ __forceinline__ int heavy_bucket(uint32_t c) { return __clz(c); }

// CTA b scans super-tiles [32 b, 32 b + 32) (lane = super-tile, coalesced rows of
// the count matrix); its 16 warps take consecutive segments of the chunks.
// The last CTA to finish does the frame-wide scans.
__global__ void __launch_bounds__(kScanThreads) k_bin_scan(Workspace ws, BinGeom g, long long cap, int diff_in_smem) {
    extern __shared__ int32_t s_diff[];  // [(tiles_y + 1) * (tiles_x + 1)] if diff_in_smem
    __shared__ uint32_t s_seg[kScanThreads / 32][32];
    __shared__ bool s_last;
    __shared__ uint32_t s_bucket[33];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kScanThreads / 32;
    {
        const int s = blockIdx.x * 32 + lane;
        const bool ok = s < g.n_st;
        const int C = g.n_chunks, per = (C + NW - 1) / NW;
        const int c0 = min(C, warp * per), c1 = min(C, c0 + per);
        uint32_t *col = ws.cmat + (ok ? s : 0);
        uint32_t sum = 0;
        {
            int c = c0;
            for (; c + 16 <= c1; c += 16) {
                uint32_t v[16];
#pragma unroll
                for (int u = 0; u < 16; u++) v[u] = ok ? col[(size_t)(c + u) * g.n_st] : 0u;
#pragma unroll
                for (int u = 0; u < 16; u++) sum += v[u];
            }
            for (; c < c1; c++) sum += ok ? col[(size_t)c * g.n_st] : 0u;
        }
        s_seg[warp][lane] = sum;
        __syncthreads();
        if (warp == 0) {
            uint32_t run = 0;
            for (int w = 0; w < NW; w++) {
                const uint32_t v = s_seg[w][lane];
                s_seg[w][lane] = run;
                run += v;
            }
            if (ok) ws.st_cnt[s] = run;
        }
        __syncthreads();
        if (ok) {
            uint32_t run = s_seg[warp][lane];
            int c = c0;
            for (; c + 16 <= c1; c += 16) {
                uint32_t v[16];
#pragma unroll
                for (int u = 0; u < 16; u++) v[u] = col[(size_t)(c + u) * g.n_st];
#pragma unroll
                for (int u = 0; u < 16; u++) {
                    col[(size_t)(c + u) * g.n_st] = run;
                    run += v[u];
                }
            }
            for (; c < c1; c++) {
                const uint32_t v = col[(size_t)c * g.n_st];
                col[(size_t)c * g.n_st] = run;
                run += v;
            }
        }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&ws.counters[CNT_DONE_SCAN], 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // ---- last CTA: super-tile list offsets and segments; tile counts -> ranges; launch order
    const unsigned long long total = *(volatile unsigned long long *)ws.pairs64;
    const bool over = total > (unsigned long long)cap;
    {
        const int per = (g.n_st + kScanThreads - 1) / kScanThreads;
        const int a0 = min(g.n_st, tid * per), a1 = min(g.n_st, a0 + per);
        uint32_t part = 0, pseg = 0;
        for (int i = a0; i < a1; i++) {
            const uint32_t c = __ldcg(&ws.st_cnt[i]);
            part += c;
            pseg += (c + kSeg - 1) / kSeg;
        }
        uint32_t all, all_seg;
        uint32_t acc = sweep::block_scan<uint32_t>(part, all);
        uint32_t sacc = sweep::block_scan<uint32_t>(pseg, all_seg);
        for (int i = a0; i < a1; i++) {
            const uint32_t c = __ldcg(&ws.st_cnt[i]);
            ws.st_start[i] = acc;
            ws.seg_first[i] = sacc;
            if (!over)  // (on overflow the lists are not built and may exceed the segment table)
                for (uint32_t k = 0; k * kSeg < c; k++) ws.seg_st[sacc + k] = (uint32_t)i;
            acc += c;
            sacc += (c + kSeg - 1) / kSeg;
        }
        if (tid == 0) {
            ws.st_start[g.n_st] = all;
            ws.seg_first[g.n_st] = all_seg;
            ws.counters[CNT_SEGS] = over ? 0u : all_seg;
        }
    }
    const int tx1 = g.tiles_x + 1;
    const int ndiff = tx1 * (g.tiles_y + 1);
    int32_t *d = diff_in_smem ? s_diff : ws.tile_diff;  // in shared memory when it fits
    if (diff_in_smem)
        for (int i = tid; i < ndiff; i += kScanThreads) s_diff[i] = __ldcg(&ws.tile_diff[i]);  // (L2: other CTAs' atomics)
    __syncthreads();
    // 2D prefix sum in place: rows (one warp per row, lane-parallel scan), then columns
    {
        const int per = (g.tiles_x + 31) / 32;
        for (int y = warp; y < g.tiles_y; y += NW) {
            int32_t *row = d + y * tx1;
            int32_t run = 0;
            for (int j = 0; j < per; j++) {
                const int x = lane * per + j;
                if (x < g.tiles_x) run += row[x];
            }
            int32_t incl = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            int32_t acc = incl - run;
            for (int j = 0; j < per; j++) {
                const int x = lane * per + j;
                if (x < g.tiles_x) {
                    acc += row[x];
                    row[x] = acc;
                }
            }
        }
    }
    __syncthreads();
    for (int x = tid; x < g.tiles_x; x += kScanThreads) {
        int32_t acc = 0;
        for (int y = 0; y < g.tiles_y; y++) {
            acc += d[y * tx1 + x];
            d[y * tx1 + x] = acc;
        }
    }
    __syncthreads();
    // exclusive scan of the per-tile counts in linear tile order -> ranges; heavy-first raster order
    const int n_tiles = g.tiles_x * g.tiles_y;
    const int per = (n_tiles + kScanThreads - 1) / kScanThreads;
    const int a0 = min(n_tiles, tid * per), a1 = min(n_tiles, a0 + per);
    uint32_t part = 0;
    for (int i = a0; i < a1; i++) part += (uint32_t)d[(i / g.tiles_x) * tx1 + i % g.tiles_x];
    uint32_t all;
    uint32_t acc = sweep::block_scan<uint32_t>(part, all);
    if (tid < 33) s_bucket[tid] = 0u;
    __syncthreads();
    for (int i = a0; i < a1; i++) {
        const uint32_t c = (uint32_t)d[(i / g.tiles_x) * tx1 + i % g.tiles_x];
        ws.ranges[i] = over ? make_uint2(0u, 0u) : make_uint2(acc, acc + c);
        acc += c;
        atomicAdd(&s_bucket[heavy_bucket(c)], 1u);
    }
    __syncthreads();
    if (tid == 0) {  // exclusive scan over the 33 buckets
        uint32_t run = 0;
        for (int b = 0; b < 33; b++) {
            const uint32_t v = s_bucket[b];
            s_bucket[b] = run;
            run += v;
        }
    }
    __syncthreads();
    for (int i = a0; i < a1; i++) {  // raster launch order (within a bucket arbitrary; results do not depend on it)
        const uint32_t c = (uint32_t)d[(i / g.tiles_x) * tx1 + i % g.tiles_x];
        ws.tile_order[atomicAdd(&s_bucket[heavy_bucket(c)], 1u)] = (uint32_t)i;
    }
    if (tid == 0) {
        ws.stats_ptr[SEELE_STAT_TILE_PAIRS] = (int64_t)total;
        ws.stats_ptr[SEELE_STAT_OVERFLOW] = over ? 1 : 0;
        ws.counters[CNT_OVERFLOW] = over ? 1u : 0u;
        ws.counters[CNT_PAIRS] = over ? 0u : (uint32_t)total;
    }
}

// ---- split -------------------------------------------------------------------------

// sub-rectangle of a tile rect inside super-tile (sx, sy): x0 | x1 << 2 | y0 << 4 | y1 << 6, in tiles
// relative to the super-tile
__device__ __forceinline__ uint32_t sub_rect(const Rect &rc, uint32_t sx, uint32_t sy) {
    const uint32_t bx = sx * kSt, by = sy * kSt;
    const uint32_t lx0 = max(rc.x0, bx) - bx, lx1 = min(rc.x1, bx + kSt - 1) - bx;
    const uint32_t ly0 = max(rc.y0, by) - by, ly1 = min(rc.y1, by + kSt - 1) - by;
    return lx0 | (lx1 << 2) | (ly0 << 4) | (ly1 << 6);
}

// One CTA per chunk, NW warps; warp w takes ranks [r0 + w Kw, r0 + (w + 1) Kw) of the chunk.
// Shared memory, per warp, indexed like the super-tile difference array (row stride stx + 1): the entry
// counts -> running entry slot of every super-tile, and the lane masks of the current item block.
// A round of 32 ranks makes one work item per (rank, super-tile it touches), owner-major; items are
// taken 32 at a time, so big splats cost work in proportion to their super-tiles.  Inside an item
// block, an item's rank among the block's items of its super-tile is popc(mask & owners below);
// blocks are consecutive in owner order, so the order is (rank, super-tile) stable.
template <int NW>
__global__ void __launch_bounds__(NW * 32) k_bin_split(Workspace ws, BinGeom g) {
    extern __shared__ uint32_t s_sp[];  // cnt[NW][n_sd], mask[NW][n_sd]
    if (ws.counters[CNT_OVERFLOW] || blockIdx.x == 0) return;  // (chunk 0: the head, k_bin_head)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sx1 = g.stx + 1, n_sd = sx1 * (g.sty + 1);
    uint32_t *cnt = s_sp + (size_t)warp * n_sd, *mask = s_sp + (size_t)(NW + warp) * n_sd;
    for (int i = tid; i < 2 * NW * n_sd; i += NW * 32) s_sp[i] = 0u;
    __syncthreads();
    const uint32_t n = (uint32_t)ws.stats_ptr[SEELE_STAT_BINNED];
    uint32_t r0, r1;
    chunk_range(n, (uint32_t)g.n_chunks, blockIdx.x, r0, r1);
    const uint32_t Kw = (r1 - r0 + NW - 1) / NW;
    const uint32_t w0 = min(r1, r0 + warp * Kw), w1 = min(r1, w0 + Kw);
    const uint32_t *srect = ws.drect[kDepthFinal];
    const uint32_t *spos = ws.dval[kDepthFinal];
    // per-warp entry counts per super-tile: difference array (four updates per rank) + 2D prefix
    {
        int32_t *dw = reinterpret_cast<int32_t *>(cnt);
        for (uint32_t r = w0 + lane; r < w1; r += 32) {
            const StRect sr = st_rect(unpack_rect(srect[r]));
            atomicAdd(&dw[sr.y0 * sx1 + sr.x0], 1);
            atomicAdd(&dw[sr.y0 * sx1 + sr.x1 + 1], -1);
            atomicAdd(&dw[(sr.y1 + 1) * sx1 + sr.x0], -1);
            atomicAdd(&dw[(sr.y1 + 1) * sx1 + sr.x1 + 1], 1);
        }
        __syncwarp();
        warp_prefix2d(dw, g.stx, g.sty, sx1);
    }
    __syncthreads();
    // -> each warp's first slot per super-tile: list start + chunk base + earlier warps
    const uint32_t *cbase = ws.cmat + (size_t)blockIdx.x * g.n_st;
    for (int s = tid; s < g.n_st; s += NW * 32) {
        const int sd = (s / g.stx) * sx1 + s % g.stx;
        uint32_t run = ws.st_start[s] + cbase[s];
#pragma unroll
        for (int w = 0; w < NW; w++) {
            const uint32_t c = s_sp[(size_t)w * n_sd + sd];
            s_sp[(size_t)w * n_sd + sd] = run;
            run += c;
        }
    }
    __syncthreads();
    uint2 *ent = ws.ent;
    uint32_t rc_next = w0 + lane < w1 ? srect[w0 + lane] : 0u, p_next = w0 + lane < w1 ? spos[w0 + lane] : 0u;
    for (uint32_t b = w0; b < w1; b += 32) {
        const uint32_t r = b + lane;
        const bool valid = r < w1;
        const uint32_t rcw = rc_next, p = p_next;
        if (r + 32 < w1) {  // next round in flight
            rc_next = srect[r + 32];
            p_next = spos[r + 32];
        }
        const StRect sr = st_rect(unpack_rect(rcw));
        const uint32_t sw = sr.x1 - sr.x0 + 1;
        const uint32_t nst = valid ? sw * (sr.y1 - sr.y0 + 1) : 0u;
        uint32_t incl = nst;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const uint32_t excl = incl - nst;
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        for (uint32_t ib = 0; ib < total; ib += 32) {
            const uint32_t item = ib + lane;
            // owner: the lane whose [excl, incl) holds the item.  Lanes own consecutive item ranges
            // (every valid rank touches >= 1 super-tile; the invalid lanes are the last ones), so the owner
            // of item ib is the number of lanes ending at or before ib, and each later item of the block
            // advances it by the lanes starting in between.
            const uint32_t owner0 = __popc(__ballot_sync(0xffffffffu, incl <= ib));
            const uint32_t starts =
                __reduce_or_sync(0xffffffffu, (excl > ib && excl < ib + 32u && nst) ? 1u << (excl - ib) : 0u);
            const int owner = (int)min(31u, owner0 + __popc(starts & ((2u << lane) - 1u)));
            const uint32_t o_excl = __shfl_sync(0xffffffffu, excl, owner);
            const uint32_t o_rect = __shfl_sync(0xffffffffu, rcw, owner);
            const uint32_t o_pos = __shfl_sync(0xffffffffu, p, owner);
            const bool live = item < total;
            const Rect orc = unpack_rect(o_rect);
            const StRect osr = st_rect(orc);
            const uint32_t osw = osr.x1 - osr.x0 + 1;
            const uint32_t k = item - o_excl;
            // k / osw: exact in float (k < 2^16, osw <= 64: a few ulp of error stay far below the 0.5 / osw margin)
            const uint32_t ky = (uint32_t)__fdividef((float)k + 0.5f, (float)osw);
            const uint32_t sx = osr.x0 + (k - ky * osw), sy = osr.y0 + ky;
            const uint32_t sd = sy * sx1 + sx;
            const uint32_t obit = 1u << owner;
            if (live) atomicOr(&mask[sd], obit);
            __syncwarp();
            uint32_t m = 0u;
            if (live) {
                m = mask[sd];
                ent[cnt[sd] + __popc(m & (obit - 1u))] = make_uint2(o_pos, sub_rect(orc, sx, sy));
            }
            __syncwarp();  // every item has read the mask and slot of its super-tile
            if (live && (m >> owner) == 1u) {  // the highest owner advances the super-tile
                cnt[sd] += __popc(m);
                mask[sd] = 0u;
            }
            __syncwarp();
        }
    }
}

// ---- expand ------------------------------------------------------------------------

// tiles of a sub-rectangle as a 16-bit mask (bit 4 ly + lx)
__device__ __forceinline__ uint32_t sub_mask(uint32_t sub) {
    const uint32_t lx0 = sub & 3u, lx1 = (sub >> 2) & 3u, ly0 = (sub >> 4) & 3u, ly1 = sub >> 6;
    const uint32_t cols = (0xfu >> (3u - lx1 + lx0)) << lx0;  // bits lx0..lx1
    const uint32_t rows = (0xfu >> (3u - ly1 + ly0)) << ly0;  // rows ly0..ly1
    uint32_t m = 0u;
#pragma unroll
    for (int y = 0; y < kSt; y++)
        if ((rows >> y) & 1u) m |= cols << (4 * y);
    return m;
}

// entries [q0, q1) of super-tile s's list, segment `seg`
__device__ __forceinline__ void seg_span(const Workspace &ws, uint32_t seg, uint32_t &s, uint32_t &e0, uint32_t &e1) {
    s = ws.seg_st[seg];
    const uint32_t q0 = (seg - ws.seg_first[s]) * (uint32_t)kSeg;
    e0 = ws.st_start[s] + q0;
    e1 = min(ws.st_start[s + 1], e0 + (uint32_t)kSeg);
}

// A segment is kSeg = kExpandThreads * kSegBatches entries; thread tid holds entries tid + b * kExpandThreads
// (b < kSegBatches), all loaded up front.
constexpr int kSegBatches = kSeg / kExpandThreads;
static_assert(kSegBatches * kExpandThreads == kSeg, "segment tiling");

__device__ __forceinline__ void load_segment(const Workspace &ws, uint32_t e0, uint32_t e1, uint32_t (&m)[kSegBatches],
                                             uint32_t (&p)[kSegBatches]) {
    uint2 e[kSegBatches];
#pragma unroll
    for (int b = 0; b < kSegBatches; b++) {
        const uint32_t i = e0 + threadIdx.x + b * kExpandThreads;
        e[b] = i < e1 ? ws.ent[i] : make_uint2(0u, 0u);
    }
#pragma unroll
    for (int b = 0; b < kSegBatches; b++) {
        const uint32_t i = e0 + threadIdx.x + b * kExpandThreads;
        m[b] = i < e1 ? sub_mask(e[b].y) : 0u;
        p[b] = e[b].x;
    }
}

// a ballot the compiler may not merge with an identical earlier one (keeping 128 ballots live across the
// barriers of k_bin_expand would spill)
__device__ __forceinline__ uint32_t ballot_again(uint32_t pred) {
    uint32_t r;
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\tvote.sync.ballot.b32 %0, p, 0xffffffff;\n\t}"
                 : "=r"(r)
                 : "r"(pred));
    return r;
}

// Per list segment (taken by ticket, so every lower segment is running or done): tile j's first slot =
// ranges[tile j].x + its head pairs + its pairs in the super-tile's earlier segments, the last by a
// decoupled look-back (16 columns, one per tile) along the super-tile's segments -- its first segment
// starts the chain.  The segment's entries are ordered (batch, warp, lane); per (batch, warp) tile counts
// from one ballot each are scanned per tile, then every (batch, warp, tile) writes its pairs as one
// coalesced run.
__global__ void __launch_bounds__(kExpandThreads, SEELE_EXPAND_MINB) k_bin_expand(Workspace ws, BinGeom g) {
    constexpr int NW = kExpandThreads / 32;
    constexpr int NBW = kSegBatches * NW;  // (batch, warp) units of a segment
    static_assert(NBW == 64, "the per-tile scan takes two units per lane");
    __shared__ uint32_t s_cnt[16][NBW];  // [tile][batch * NW + warp]: pair count -> offset in the segment
    __shared__ uint32_t s_tot[16];
    __shared__ uint32_t s_base[16];
    __shared__ uint32_t s_seg;
    const uint32_t n_seg = ws.counters[CNT_SEGS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t epoch = *ws.epoch * 16u + kLookSegs;
    while (true) {
        if (tid == 0) s_seg = atomicAdd(&ws.counters[CNT_TICKET], 1u);
        __syncthreads();
        const uint32_t seg = s_seg;
        if (seg >= n_seg) break;
        uint32_t s, e0, e1;
        seg_span(ws, seg, s, e0, e1);
        uint32_t m[kSegBatches], p[kSegBatches];
        load_segment(ws, e0, e1, m, p);
        // per (batch, warp) pair counts of the 16 tiles: the entries' tile bits spread into bytes (four tiles
        // per word; a count <= 32 fits a byte) and summed over the warp by four hardware reductions
#pragma unroll
        for (int b = 0; b < kSegBatches; b++) {
            uint32_t c[4];
#pragma unroll
            for (int k = 0; k < 4; k++)
                c[k] = __reduce_add_sync(0xffffffffu, (((m[b] >> (4 * k)) & 0xfu) * 0x00204081u) & 0x01010101u);
            if (lane < 16) {
                const uint32_t w = (lane & 8) ? ((lane & 4) ? c[3] : c[2]) : ((lane & 4) ? c[1] : c[0]);
                s_cnt[lane][b * NW + warp] = (w >> (8 * (lane & 3))) & 0xffu;
            }
        }
        __syncthreads();
        // exclusive scan of every tile's 64 unit counts (warp w: tiles 2w, 2w + 1; lane: units 2l, 2l + 1)
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int j = 2 * warp + h;
            if (j >= 16) break;  // (more than 8 warps: the 16 tiles are taken by the first 8)
            const uint32_t a0 = s_cnt[j][2 * lane], a1 = s_cnt[j][2 * lane + 1];
            uint32_t incl = a0 + a1;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const uint32_t ex = incl - a0 - a1;
            s_cnt[j][2 * lane] = ex;
            s_cnt[j][2 * lane + 1] = ex + a0;
            if (lane == 31) s_tot[j] = incl;
        }
        __syncthreads();
        if (tid < 16) {
            const uint32_t prev = sweep::lookback(ws.seg_look + tid, 16, seg, epoch, s_tot[tid], seg == ws.seg_first[s]);
            const uint32_t tx = (s % g.stx) * kSt + (tid & 3), ty = (s / g.stx) * kSt + (tid >> 2);
            const bool in = tx < (uint32_t)g.tiles_x && ty < (uint32_t)g.tiles_y;
            const uint32_t t_id = ty * g.tiles_x + tx;
            s_base[tid] = in ? ws.ranges[t_id].x + ws.head_cnt[t_id] + prev : 0u;
        }
        __syncthreads();
#pragma unroll
        for (int h = 0; h < 2; h++) {  // unit offsets -> absolute slots
            const int j = 2 * warp + h;
            if (j >= 16) break;
            s_cnt[j][2 * lane] += s_base[j];
            s_cnt[j][2 * lane + 1] += s_base[j];
        }
        __syncthreads();
#pragma unroll
        for (int b = 0; b < kSegBatches; b++)
#pragma unroll
            for (int j = 0; j < 16; j++) {
                const uint32_t bb = ballot_again((m[b] >> j) & 1u);
                if ((m[b] >> j) & 1u) ws.pfinal[s_cnt[j][b * NW + warp] + __popc(bb & lt)] = p[b];
            }
        __syncthreads();  // s_cnt / s_base / s_seg are rewritten by the next segment
    }
}

// ---- head --------------------------------------------------------------------------

// The nearest ranks (chunk 0) hold the scene's largest splats: on C3 its ~3.3K ranks carry 12 % of the
// frame's pairs and 22x the average chunk's super-tile entries.  They precede every later rank in every
// tile, so they are emitted per tile, not through the super-tile lists: one warp per tile walks the head
// ranks in order (32 per ballot) and writes the ones covering its tile to ranges[tile].x + running count,
// after its CTA (one per super-tile) compacted the head ranks touching the super-tile into shared memory.
constexpr int kHeadThreads = 512;   // one CTA per super-tile, one warp per tile
constexpr int kHeadWindow = 4096;   // head ranks compacted per window
__global__ void __launch_bounds__(kHeadThreads) k_bin_head(Workspace ws, BinGeom g) {
    __shared__ uint32_t s_rect[kHeadWindow];  // the window's ranks touching this super-tile, in rank order
    __shared__ uint32_t s_idx[kHeadWindow];
    __shared__ uint32_t s_wn[kHeadThreads / 32];
    __shared__ uint32_t s_n;
    constexpr int NW = kHeadThreads / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t sx = blockIdx.x % (uint32_t)g.stx, sy = blockIdx.x / (uint32_t)g.stx;
    const uint32_t bx0 = sx * kSt, by0 = sy * kSt, bx1 = bx0 + kSt - 1, by1 = by0 + kSt - 1;
    const uint32_t tx = bx0 + (warp & 3), ty = by0 + (warp >> 2);  // this warp's tile
    const bool tile_ok = tx < (uint32_t)g.tiles_x && ty < (uint32_t)g.tiles_y;
    const uint32_t t = ty * g.tiles_x + tx;
    const bool over = ws.counters[CNT_OVERFLOW] != 0u;
    const uint32_t n = (uint32_t)ws.stats_ptr[SEELE_STAT_BINNED];
    uint32_t h0, h1;
    chunk_range(n, (uint32_t)g.n_chunks, 0u, h0, h1);
    const uint32_t *srect = ws.drect[kDepthFinal];
    const uint32_t *spos = ws.dval[kDepthFinal];
    const uint32_t base = tile_ok ? ws.ranges[t].x : 0u;
    const unsigned lt = (1u << lane) - 1u;
    uint32_t run = 0;
    for (uint32_t w0 = h0; w0 < h1; w0 += kHeadWindow) {
        const uint32_t w1 = min(h1, w0 + kHeadWindow);
        // compact the window's ranks touching the super-tile (rank order: rounds of NW x 32 ranks)
        uint32_t cnt = 0;
        for (uint32_t r0 = w0; r0 < w1; r0 += kHeadThreads) {
            const uint32_t r = r0 + tid;
            uint32_t v = 0u;
            bool hit = false;
            if (r < w1) {
                v = srect[r];
                const Rect rc = unpack_rect(v);
                hit = rc.x0 <= bx1 && rc.x1 >= bx0 && rc.y0 <= by1 && rc.y1 >= by0;
            }
            const unsigned bb = __ballot_sync(0xffffffffu, hit);
            if (lane == 0) s_wn[warp] = __popc(bb);
            __syncthreads();
            uint32_t before = 0, all = 0;
#pragma unroll
            for (int w = 0; w < NW; w++) {
                const uint32_t c = s_wn[w];
                before += w < warp ? c : 0u;
                all += c;
            }
            if (hit) {
                const uint32_t k = cnt + before + __popc(bb & lt);
                s_rect[k] = v;
                s_idx[k] = r;
            }
            cnt += all;
            __syncthreads();
        }
        // every tile walks the compacted list
        if (tile_ok) {
            for (uint32_t i0 = 0; i0 < cnt; i0 += 32) {
                const uint32_t i = i0 + lane;
                bool cov = false;
                if (i < cnt) {
                    const Rect rc = unpack_rect(s_rect[i]);
                    cov = tx >= rc.x0 && tx <= rc.x1 && ty >= rc.y0 && ty <= rc.y1;
                }
                const unsigned bb = __ballot_sync(0xffffffffu, cov);
                if (cov && !over) ws.pfinal[base + run + __popc(bb & lt)] = spos[s_idx[i]];
                run += __popc(bb);
            }
        }
        __syncthreads();  // the lists are rewritten by the next window
    }
    if (tile_ok && lane == 0) ws.head_cnt[t] = run;
}

__global__ void k_fill_pair_tiles(const uint2 *ranges, int n_tiles, int32_t *pair_tile) {
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const uint2 r = ranges[t];
        for (uint32_t i = r.x + threadIdx.x; i < r.y; i += blockDim.x) pair_tile[i] = t;
    }
}

long long ceil_div(long long a, long long b) { return (a + b - 1) / b; }

template <typename K>
void set_smem(K kernel, size_t bytes) {
    if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace

BinGeom bin_geometry(long long n_max, int width, int height) {
    BinGeom g;
    g.tiles_x = (width + kTile - 1) / kTile;
    g.tiles_y = (height + kTile - 1) / kTile;
    g.stx = (g.tiles_x + kSt - 1) / kSt;
    g.sty = (g.tiles_y + kSt - 1) / kSt;
    g.n_st = g.stx * g.sty;
    // chunks of ~2K ranks (fixed by n_max, not by the device, so the workspace size is too)
    long long c = (n_max + kBinChunkRanks - 1) / kBinChunkRanks;
    g.n_chunks = (int)(c < kBinChunksMin ? kBinChunksMin : (c > kBinChunksMax ? kBinChunksMax : c));
    g.count_group = 1;
    return g;
}

void launch_frame_begin(const Workspace &ws, const CamK &cam, int64_t *stats, cudaStream_t st) {
    const int n_diff = (cam.tiles_x + 1) * (cam.tiles_y + 1);
    const int grid = 256;  // (the depth histogram alone is 4 MB)
    k_frame_begin<<<grid, 256, 0, st>>>(ws, stats, n_diff);
    note_launches(1);
}

void launch_binning(const Workspace &ws, long long n_max, long long cap, const CamK &cam, int64_t *stats,
                    cudaStream_t st) {
    (void)stats;
    const BinGeom g = bin_geometry(n_max, cam.width, cam.height);
    const int sms = stream_sms(st);
    const size_t n_sd = (size_t)(g.stx + 1) * (g.sty + 1);
    const size_t diff_bytes = sizeof(int32_t) * (g.tiles_x + 1) * (g.tiles_y + 1);
    const size_t sd_bytes = sizeof(int32_t) * n_sd;
    BinGeom gc = g;  // count: groups of chunks per CTA, ~2 CTAs per SM (fewer flushes of the tile difference array)
    gc.count_group = (int)std::max<long long>(1, std::min<long long>(kCountMaxGroup, ceil_div(g.n_chunks, 2 * sms)));
    const int count_diff_smem = gc.count_group * sd_bytes + diff_bytes <= 160 * 1024;
    const size_t count_smem = gc.count_group * sd_bytes + (count_diff_smem ? diff_bytes : 0);
    set_smem(k_bin_count, count_smem);
    k_bin_count<<<(int)ceil_div(g.n_chunks, gc.count_group), kCountThreads, count_smem, st>>>(ws, gc, count_diff_smem);
    const int scan_diff_smem = diff_bytes <= 160 * 1024;
    const size_t scan_smem = scan_diff_smem ? diff_bytes : 0;
    set_smem(k_bin_scan, scan_smem);
    k_bin_scan<<<(g.n_st + 31) / 32, kScanThreads, scan_smem, st>>>(ws, g, cap, scan_diff_smem);
    // split: the widest CTA (16, 8 or 4 warps of the chunk) whose per-warp super-tile arrays fit 128 KB
    // (1080p: 16 warps; 16 vs 8 measured 0.197 vs 0.205 ms binning, C3)
    constexpr int NWS = SEELE_SPLIT_NW;
    const size_t split_w = 2 * NWS * sd_bytes, split8 = 2 * 8 * sd_bytes;
    if (split_w <= 128 * 1024) {
        set_smem(k_bin_split<NWS>, split_w);
        k_bin_split<NWS><<<g.n_chunks, NWS * 32, split_w, st>>>(ws, g);
    } else if (split8 <= 128 * 1024) {
        set_smem(k_bin_split<8>, split8);
        k_bin_split<8><<<g.n_chunks, 8 * 32, split8, st>>>(ws, g);
    } else {
        const size_t split4 = 2 * 4 * sd_bytes;
        set_smem(k_bin_split<4>, split4);
        k_bin_split<4><<<g.n_chunks, 4 * 32, split4, st>>>(ws, g);
    }
#ifndef SEELE_EXPAND_PER_SM
#define SEELE_EXPAND_PER_SM 4
#endif
    const long long max_seg = cap / kSeg + g.n_st + 1;
    const int xgrid = (int)std::min<long long>(max_seg, (long long)SEELE_EXPAND_PER_SM * sms);
    k_bin_head<<<g.n_st, kHeadThreads, 0, st>>>(ws, g);
    k_bin_expand<<<xgrid, kExpandThreads, 0, st>>>(ws, g);
    note_launches(5);
}

void launch_fill_pair_tiles(const uint2 *ranges, int n_tiles, int32_t *pair_tile, cudaStream_t st) {
    k_fill_pair_tiles<<<n_tiles < 4096 ? n_tiles : 4096, 256, 0, st>>>(ranges, n_tiles, pair_tile);
    note_launches(1);
}

}  // namespace seele
