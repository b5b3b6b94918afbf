// Tile binning and the tile sort on sm_100a, over the binned splats in exact
// (depth, position) order (depth.cu).  Every size is read from device
// memory, so a frame needs no host round trip:
//
//   pair scan    k_pair_scan: exclusive scan of each splat's row-entry count
//                in depth order (decoupled look-back), first rank of every
//                4096-entry row-pass tile, and the 2D / 1D difference arrays
//                of per-tile pair counts and per-row entry counts; the last
//                CTA turns them into the tile ranges (sorting.py:46-53), the
//                raster launch order, the row bases and the column-pass chunks.
//   row pass     k_row_pass: bin_tiles (preprocess.py:159-189) of each splat
//                as row entries (one per covered tile row, split into <= 3
//                columns), stably grouped by tile row: one onesweep pass whose
//                digit is the row.
//   column pass  k_col_pass: every row chunk expands its entries into pairs,
//                each written straight to its final slot (sorting.py:32-54
//                order) = tile range start + pairs of that column in earlier
//                chunks (look-back along the row) + earlier entries of the
//                chunk covering the column.
#include "onesweep.cuh"

namespace seele {

using namespace sweep;

#ifdef SEELE_SORT_TRACE
__device__ unsigned long long g_trace[8][4096][6];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define TRACE(pass, t, k) \
    if (threadIdx.x == 0 && (t) < 4096) g_trace[pass][t][k] = gtime();
#else
#define TRACE(pass, t, k)
#endif

namespace {

// ---- frame start ---------------------------------------------------------------

__global__ void k_frame_begin(Workspace ws, int64_t *stats, int n_diff, int tiles_y) {
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    if (tid == 0) {
        *ws.epoch += 1u;
        *ws.pairs64 = 0ull;
    }
    if (tid < SEELE_STAT_COUNT) stats[tid] = 0;
    if (tid < CNT_COUNT) ws.counters[tid] = 0u;
    for (int i = tid; i < kDepthBuckets / 4; i += stride) reinterpret_cast<uint4 *>(ws.bhist)[i] = make_uint4(0, 0, 0, 0);
    for (int i = tid; i < n_diff; i += stride) ws.tile_diff[i] = 0;
    for (int i = tid; i <= tiles_y; i += stride) ws.row_diff[i] = 0;
}

__device__ __forceinline__ short4 unpack_rect(uint32_t v) {
    return make_short4((short)(v & 0xff), (short)((v >> 8) & 0xff), (short)((v >> 16) & 0xff), (short)(v >> 24));
}

// ---- row entries: offsets, tile counts, ranges -------------------------------------

// Row entries cover at most kSegW columns (wider ones are split; pieces of one
// splat cover disjoint columns, so the per-column order is unaffected): the
// column pass's per-entry loops stay short.
#ifndef SEELE_SEGW
#define SEELE_SEGW 3
#endif
constexpr uint32_t kSegW = SEELE_SEGW;

// bin_tiles (preprocess.py:159-189) of splat rank r covers rect [x0,x1] x [y0,y1]
// -> ceil(w / kSegW) row entries per covered tile row y and w * h pairs.
// This persistent kernel scans the entry counts h in depth-rank order
// (decoupled look-back over 4096-rank tiles) into poff, marks the first rank
// of every 4096-entry tile of the row pass, counts pairs, and accumulates the
// 2D difference array of per-tile pair counts and the 1D one of per-row entry
// counts.  The last CTA turns those into the tile ranges (sorting.py:46-53),
// the row bases of the row pass and the chunk table of the column pass.
// raster launch order bucket of a tile with c pairs: 32 - bits(c), heavy tiles first
#ifndef SEELE_LIGHT_FIRST
__device__ __forceinline__ int tile_bucket(uint32_t c) { return __clz(c); }
#else
__device__ __forceinline__ int tile_bucket(uint32_t c) { return 32 - __clz(c); }
#endif

__global__ void __launch_bounds__(NT) k_pair_scan(Workspace ws, int tiles_x, int tiles_y, long long cap, int use_smem,
                                                  int64_t *stats) {
    extern __shared__ int32_t s_diff[];  // [(tiles_y + 1) * (tiles_x + 1)] if use_smem
    __shared__ int32_t s_row[kMaxTileAxis + 1];
    __shared__ bool s_last;
    __shared__ uint32_t s_prev;
    __shared__ unsigned long long s_pairs;
    const int tid = threadIdx.x;
    const int tx1 = tiles_x + 1;
    const int ndiff = tx1 * (tiles_y + 1);
    if (use_smem)
        for (int i = tid; i < ndiff; i += NT) s_diff[i] = 0;
    for (int i = tid; i <= tiles_y; i += NT) s_row[i] = 0;
    if (tid == 0) s_pairs = 0ull;
    int32_t *diff = use_smem ? s_diff : ws.tile_diff;
    const uint32_t n = (uint32_t)stats[SEELE_STAT_BINNED];
    const uint32_t *srect = ws.drect[kDepthFinal];
    const uint32_t n_etiles = (uint32_t)(cap / TILE) + 1u;  // tile_r0 entries kept (capacity)
    unsigned long long my_pairs = 0ull;
    while (true) {
        const uint32_t t = take_ticket(&ws.counters[CNT_TICKET + kLookScan]);
        if (t * TILE >= n) break;
        const uint32_t r0 = t * TILE + tid * IPT;
        uint32_t h[IPT], rr[IPT];
        uint32_t sum = 0;
#pragma unroll
        for (int k = 0; k < IPT; k++) rr[k] = srect[min(r0 + k, n - 1)];  // coalesced: rects in rank order
#pragma unroll
        for (int k = 0; k < IPT; k++) {
            h[k] = 0u;
            const uint32_t r = r0 + k;
            if (r < n) {
                const short4 rc = unpack_rect(rr[k]);
                const int w = rc.y - rc.x + 1, hh = rc.w - rc.z + 1;
                const int nseg = (w + kSegW - 1) / kSegW;  // row entries are split into <= kSegW columns
                h[k] = (uint32_t)(hh * nseg);
                my_pairs += (unsigned long long)(w * hh);
                atomicAdd(&diff[rc.z * tx1 + rc.x], 1);
                atomicAdd(&diff[rc.z * tx1 + rc.y + 1], -1);
                atomicAdd(&diff[(rc.w + 1) * tx1 + rc.x], -1);
                atomicAdd(&diff[(rc.w + 1) * tx1 + rc.y + 1], 1);
                atomicAdd(&s_row[rc.z], nseg);
                atomicAdd(&s_row[rc.w + 1], -nseg);
            }
            sum += h[k];
        }
        uint32_t agg;
        const uint32_t ex = block_scan<uint32_t>(sum, agg);
        if (tid < 32) {  // one warp: 32 predecessors per round trip
            const uint32_t pv = lookback_warp(ws.look_region(kLookScan), t, *ws.epoch * 16u + kLookScan, agg, t == 0);
            if (tid == 0) s_prev = pv;
        }
        __syncthreads();
        uint32_t run = s_prev + ex;
#pragma unroll
        for (int k = 0; k < IPT; k++) {
            const uint32_t r = r0 + k;
            if (r >= n) break;
            ws.poff[r] = run;
            const uint32_t end = run + h[k];
            for (uint32_t e = (run + TILE - 1) / TILE; e * TILE < end && e < n_etiles; e++) ws.tile_r0[e] = r;
            if (r == n - 1) ws.poff[n] = end;
            run = end;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_pairs += __shfl_xor_sync(0xffffffffu, my_pairs, o);
    if ((tid & 31) == 0 && my_pairs) atomicAdd(&s_pairs, my_pairs);
    __syncthreads();
    if (tid == 0 && s_pairs) atomicAdd(ws.pairs64, s_pairs);
    if (use_smem)
        for (int i = tid; i < ndiff; i += NT)
            if (s_diff[i]) atomicAdd(&ws.tile_diff[i], s_diff[i]);
    for (int i = tid; i <= tiles_y; i += NT)
        if (s_row[i]) atomicAdd(&ws.row_diff[i], s_row[i]);
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&ws.counters[CNT_DONE_SCAN], 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // ---- last CTA: per-tile counts -> ranges; row bases; chunk table
    const unsigned long long total = *(volatile unsigned long long *)ws.pairs64;
    const bool over = total > (unsigned long long)cap;
    int32_t *g = use_smem ? s_diff : ws.tile_diff;  // in shared memory when it fits
    if (use_smem)
        for (int i = tid; i < ndiff; i += NT) s_diff[i] = *(volatile int32_t *)&ws.tile_diff[i];
    __syncthreads();
    // 2D prefix sum in place: rows (one warp per row, lane-parallel scan), then columns
    {
        const int lane = tid & 31, warp = tid >> 5;
        const int per = (tiles_x + 31) / 32;
        for (int y = warp; y < tiles_y; y += NT / 32) {
            int32_t *row = g + y * tx1;
            int32_t run = 0;
            for (int j = 0; j < per; j++) {
                const int x = lane * per + j;
                if (x < tiles_x) run += row[x];
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
                if (x < tiles_x) {
                    acc += row[x];
                    row[x] = acc;
                }
            }
        }
    }
    __syncthreads();
    for (int x = tid; x < tiles_x; x += NT) {
        int32_t acc = 0;
        for (int y = 0; y < tiles_y; y++) {
            acc += g[y * tx1 + x];
            g[y * tx1 + x] = acc;
        }
    }
    __syncthreads();
    // exclusive scan of the per-tile counts in linear tile order -> ranges
    const int n_tiles = tiles_x * tiles_y;
    const int per = (n_tiles + NT - 1) / NT;
    const int a0 = tid * per, a1 = min(a0 + per, n_tiles);
    uint32_t part = 0;
    for (int i = a0; i < a1; i++) part += (uint32_t)g[(i / tiles_x) * tx1 + i % tiles_x];
    uint32_t all;
    uint32_t acc = block_scan<uint32_t>(part, all);
    __shared__ uint32_t s_bucket[33];
    if (tid < 33) s_bucket[tid] = 0u;
    __syncthreads();
    for (int i = a0; i < a1; i++) {
        const uint32_t c = (uint32_t)g[(i / tiles_x) * tx1 + i % tiles_x];
        ws.ranges[i] = over ? make_uint2(0u, 0u) : make_uint2(acc, acc + c);
        acc += c;
        atomicAdd(&s_bucket[tile_bucket(c)], 1u);
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
        const uint32_t c = (uint32_t)g[(i / tiles_x) * tx1 + i % tiles_x];
        ws.tile_order[atomicAdd(&s_bucket[tile_bucket(c)], 1u)] = (uint32_t)i;
    }
    // entries per row -> row bases (row pass digit bases) and column-pass chunks
    for (int i = tid; i <= tiles_y; i += NT) s_row[i] = *(volatile int32_t *)&ws.row_diff[i];
    __syncthreads();
    if (tid == 0) {
        int32_t rc = 0;
        uint32_t e = 0, c = 0;
        for (int y = 0; y < tiles_y; y++) {
            rc += s_row[y];
            ws.row_start[y] = e;
            ws.chunk_first[y] = c;
            e += (uint32_t)rc;
            c += ((uint32_t)rc + TILE - 1) / TILE;
        }
        ws.row_start[tiles_y] = e;
        ws.chunk_first[tiles_y] = c;
        stats[SEELE_STAT_TILE_PAIRS] = (int64_t)total;
        stats[SEELE_STAT_OVERFLOW] = over ? 1 : 0;
        ws.counters[CNT_OVERFLOW] = over ? 1u : 0u;
        ws.counters[CNT_PAIRS] = over ? 0u : (uint32_t)total;
        ws.counters[CNT_ENTRIES] = over ? 0u : e;
        ws.counters[CNT_CHUNKS] = over ? 0u : c;
    }
}

// ---- row pass ----------------------------------------------------------------------

struct RowSmem {
    RankSmem rs;
    uint32_t s_base[RADIX];
    union {
        struct {  // the ranks overlapping this tile
            uint32_t off[TILE + 3];
            uint32_t pos[TILE + 2];
            uint32_t rect[TILE + 2];  // x0 | x1 << 8 | y0 << 16
        } e;
        struct {  // the row-sorted tile
            uint32_t x[TILE];
            uint32_t p[TILE];
        } g;
    } u;
    uint32_t gx[TILE];  // generated entries in emission order
    uint32_t gp[TILE];
};

// Emits the row entries of 4096 consecutive entry slots in depth-rank order
// (ty-major inside a splat, like bin_tiles) and scatters them stably by row:
// one onesweep pass whose digit is the tile row.
// One ticket of the row pass; false once the tickets run past the entries.
__device__ __forceinline__ bool row_tile(const Workspace &ws, int64_t *stats, RowSmem &S, uint32_t t) {
    const uint32_t E = ws.counters[CNT_ENTRIES];
    const uint32_t base = t * TILE;
    if (base >= E) return false;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t n = (uint32_t)stats[SEELE_STAT_BINNED];
    const uint32_t *sorted = ws.dval[kDepthFinal];
    const uint32_t end = min(base + (uint32_t)TILE, E);
    const uint32_t r0 = ws.tile_r0[t];
    const uint32_t r1 = end < E ? ws.tile_r0[t + 1] : n - 1;  // last rank overlapping
    const int nr = (int)(r1 - r0 + 1);
    for (int k = tid; k <= nr; k += NT) {
        S.u.e.off[k] = ws.poff[r0 + k];
        if (k < nr) {
            S.u.e.pos[k] = sorted[r0 + k];
            S.u.e.rect[k] = ws.drect[kDepthFinal][r0 + k] & 0xffffffu;  // x0 | x1 << 8 | y0 << 16
        }
    }
    __syncthreads();
    const uint32_t i0 = base + (uint32_t)tid * IPT;
    if (i0 < end) {
        int lo = 0, hi = nr - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (S.u.e.off[mid] <= i0) lo = mid; else hi = mid - 1;
        }
        uint32_t rc = S.u.e.rect[lo];
        uint32_t xa = rc & 0xffu, xb = (rc >> 8) & 0xffu;
        uint32_t nseg = (xb - xa + kSegW) / kSegW;
        const uint32_t local = i0 - S.u.e.off[lo];
        uint32_t y = (rc >> 16) + local / nseg, seg = local % nseg;
        uint32_t next = S.u.e.off[lo + 1];
        uint32_t p = S.u.e.pos[lo];
        const uint32_t stop = min(i0 + (uint32_t)IPT, end);
        for (uint32_t i = i0; i < stop; i++) {
            if (i == next) {
                lo++;
                rc = S.u.e.rect[lo];
                xa = rc & 0xffu;
                xb = (rc >> 8) & 0xffu;
                nseg = (xb - xa + kSegW) / kSegW;
                y = rc >> 16;
                seg = 0;
                next = S.u.e.off[lo + 1];
                p = S.u.e.pos[lo];
            }
            const uint32_t s0 = xa + seg * kSegW, s1 = min(xb, s0 + kSegW - 1);
            S.gx[i - base] = s0 | (s1 << 8) | (y << 16);
            S.gp[i - base] = p;
            if (++seg == nseg) {
                seg = 0;
                y++;
            }
        }
    }
    __syncthreads();
    const int nv = (int)(end - base);
    uint32_t xk[IPT], pv[IPT], dig[IPT], pos[IPT];
#pragma unroll
    for (int r = 0; r < IPT; r++) {
        const int i = warp * 32 * IPT + r * 32 + lane;
        dig[r] = NO_DIGIT;
        if (i < nv) {
            xk[r] = S.gx[i];
            pv[r] = S.gp[i];
            dig[r] = xk[r] >> 16;
        }
    }
    uint32_t count;
#ifndef SEELE_ROW_BALLOT
#define SEELE_ROW_BALLOT 1
#endif
    block_rank<SEELE_ROW_BALLOT>(dig, pos, S.rs, count);
    if (tid < RADIX) {
        const uint32_t ex =
            lookback(ws.look_region(kLookRows) + tid, RADIX, t, *ws.epoch * 16u + kLookRows, count, t == 0);
        S.s_base[tid] = ws.row_start[min(tid, kMaxTileAxis)] + ex - S.rs.start[tid];
    }
#pragma unroll
    for (int r = 0; r < IPT; r++) {
        if (dig[r] == NO_DIGIT) continue;
        S.u.g.x[pos[r]] = xk[r];
        S.u.g.p[pos[r]] = pv[r];
    }
    __syncthreads();
    for (int i = tid; i < nv; i += NT) {
        const uint32_t x = S.u.g.x[i];
        const uint32_t dst = S.s_base[x >> 16] + (uint32_t)i;
        ws.ent_x[dst] = x;
        ws.ent_p[dst] = S.u.g.p[i];
    }
    return true;
}

// Persistent: each CTA takes tickets (in order over the grid) until none is left,
// so the grid is sized to the machine, not to the pair capacity.
#ifndef SEELE_ROW_MINB
#define SEELE_ROW_MINB 2
#endif
__global__ void __launch_bounds__(NT, SEELE_ROW_MINB) k_row_pass(Workspace ws, int64_t *stats) {
    extern __shared__ __align__(16) unsigned char smem[];
    RowSmem &S = *reinterpret_cast<RowSmem *>(smem);
    ticket_loop(&ws.counters[CNT_TICKET + kLookRows], [&](uint32_t t) { return row_tile(ws, stats, S, t); });

}

// ---- column pass ---------------------------------------------------------------------

constexpr int kColW = kMaxTileAxis + 1;
constexpr int kColStage = 12288;  // pairs staged per column group (48 KB + 12 KB)

struct ColSmem {
    int32_t cnt[NT / 32][kColW];      // per-warp counts -> per-warp staging offsets
    uint32_t mask[NT / 32][kColW];    // per-round lanes covering each column
    uint32_t cstart[kColW + 1];       // chunk-local first slot of each column
    uint32_t gbase[kColW];            // global slot of the chunk's first pair of each column
    uint32_t stage[kColStage];
    uint8_t stx[kColStage];
    uint32_t gfirst[kColW + 1];       // column groups that fit the staging buffer
    uint32_t chunk_first[kColW + 1];
    int n_groups;
    uint32_t row;
};

// One chunk (<= 4096 entries) of one tile row: expands every entry into its
// pairs and writes them to their final slots.  Inside the row, the pairs of
// tile (ty, tx) come from the entries covering tx in entry (= depth-rank)
// order, so slot = ranges[tile].x + (pairs of tx in earlier chunks of the
// row: look-back along the row's chunks) + (entries covering tx earlier in
// this chunk).  The last term: per-warp counts + exclusive scan over warps,
// and inside a warp round (32 entries) every lane ORs its bit into the lane
// mask of each column it covers, so its rank at column v is
// popc(mask_v & lanes_below) -- work proportional to the entry's width.
// Pairs are staged by column in shared memory and copied out as contiguous
// runs.
// One ticket (row chunk) of the column pass; false once the tickets run past the chunks.
__device__ __forceinline__ bool col_tile(const Workspace &ws, int tiles_x, int tiles_y, ColSmem &S, uint32_t t) {
    const uint32_t C = ws.counters[CNT_CHUNKS];
    if (t >= C) return false;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int y = tid; y < tiles_y; y += NT) S.chunk_first[y] = ws.chunk_first[y];
    __syncthreads();
    if (tid == 0) {  // row of chunk t: last y with chunk_first[y] <= t
        int lo = 0, hi = tiles_y - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (S.chunk_first[mid] <= t) lo = mid; else hi = mid - 1;
        }
        S.row = (uint32_t)lo;
    }
    for (int i = lane; i < kColW; i += 32) {
        S.cnt[warp][i] = 0;
        S.mask[warp][i] = 0u;
    }
    __syncthreads();
    const int ty = (int)S.row;
    const uint32_t k = t - ws.chunk_first[ty];
    const uint32_t s = ws.row_start[ty] + k * TILE, e = min(s + (uint32_t)TILE, ws.row_start[ty + 1]);
    uint32_t x0[IPT], x1[IPT], pv[IPT];
    const uint32_t wb = s + (uint32_t)(warp * 32 * IPT) + lane;
#pragma unroll
    for (int r = 0; r < IPT; r++) {
        const uint32_t i = min(wb + r * 32, e - 1);
        const uint32_t x = ws.ent_x[i];
        pv[r] = ws.ent_p[i];
        const bool valid = wb + r * 32 < e;
        x0[r] = valid ? (x & 0xffu) : 1u;  // absent: empty interval [1, 0]
        x1[r] = valid ? ((x >> 8) & 0xffu) : 0u;
    }
#pragma unroll
    for (int r = 0; r < IPT; r++) {
        if (x0[r] > x1[r]) continue;
        atomicAdd(&S.cnt[warp][x0[r]], 1);
        atomicAdd(&S.cnt[warp][x1[r] + 1], -1);
    }
    __syncwarp();
    constexpr int PER = (kColW + 31) / 32;  // columns per lane in warp-wide scans
    {
        int32_t v[PER], run = 0;
#pragma unroll
        for (int j = 0; j < PER; j++) {
            const int c = lane * PER + j;
            v[j] = c < kColW ? S.cnt[warp][c] : 0;
            run += v[j];
        }
        int32_t incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        int32_t acc = incl - run;
#pragma unroll
        for (int j = 0; j < PER; j++) {
            const int c = lane * PER + j;
            acc += v[j];
            if (c < kColW) S.cnt[warp][c] = acc;
        }
    }
    __syncthreads();
    uint32_t tot = 0;
    if (tid < kColW) {
#pragma unroll
        for (int w = 0; w < NT / 32; w++) {
            const int32_t c = S.cnt[w][tid];
            S.cnt[w][tid] = (int32_t)tot;
            tot += (uint32_t)c;
        }
    }
    uint32_t chunk_total;
    const uint32_t cs = block_scan<uint32_t>(tid < tiles_x ? tot : 0u, chunk_total);
    if (tid < tiles_x) {
        S.cstart[tid] = cs;
        const uint32_t ex = lookback(ws.look_region(kLookCols) + tid, RADIX, t, *ws.epoch * 16u + kLookCols, tot,
                                     k == 0);
        S.gbase[tid] = ws.ranges[ty * tiles_x + tid].x + ex;
#pragma unroll
        for (int w = 0; w < NT / 32; w++) S.cnt[w][tid] += (int32_t)cs;  // chunk-local staging offsets
    }
    if (tid == 0) S.cstart[tiles_x] = chunk_total;
    __syncthreads();
    if (tid == 0) {
        int g = 0;
        S.gfirst[0] = 0;
        if (chunk_total > (uint32_t)kColStage) {  // rare: greedy column groups that fit the staging buffer
            uint32_t gs = 0;
            for (int c = 0; c < tiles_x; c++) {
                if (S.cstart[c + 1] - gs > (uint32_t)kColStage) {
                    S.gfirst[++g] = (uint32_t)c;
                    gs = S.cstart[c];
                }
            }
        }
        S.gfirst[++g] = (uint32_t)tiles_x;
        S.n_groups = g;
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    for (int grp = 0; grp < S.n_groups; grp++) {
        const uint32_t ca = S.gfirst[grp], cb = S.gfirst[grp + 1];
        const uint32_t sbase = S.cstart[ca];
#pragma unroll 1
        for (int r = 0; r < IPT; r++) {
            // columns of this entry inside the current group
            const uint32_t a = max(x0[r], ca), b = min(x1[r] + 1u, cb);  // [a, b), at most kSegW columns
            // (fixed-trip predicated loops: entries cover <= kSegW columns)
#pragma unroll
            for (uint32_t c = 0; c < kSegW; c++)
                if (a + c < b) atomicOr(&S.mask[warp][a + c], 1u << lane);
            __syncwarp();
            uint32_t adv = 0u;  // per covered column: this lane is the highest covering lane (advances it)
            uint32_t n_cov[kSegW];
#pragma unroll
            for (uint32_t c = 0; c < kSegW; c++) {
                n_cov[c] = 0u;
                if (a + c >= b) continue;
                const uint32_t v = a + c;
                const uint32_t m = S.mask[warp][v];
                const uint32_t slot = (uint32_t)S.cnt[warp][v] + __popc(m & lt) - sbase;
                S.stage[slot] = pv[r];
                S.stx[slot] = (uint8_t)v;
                if ((m >> lane) == 1u) {
                    adv |= 1u << c;
                    n_cov[c] = __popc(m);
                }
            }
            __syncwarp();  // every lane has read the masks and counters of its columns
#pragma unroll
            for (uint32_t c = 0; c < kSegW; c++) {
                if (!((adv >> c) & 1u)) continue;
                S.cnt[warp][a + c] += n_cov[c];
                S.mask[warp][a + c] = 0u;
            }
            __syncwarp();
        }
        __syncthreads();
        const uint32_t n_stage = S.cstart[cb] - sbase;
        for (uint32_t i = tid; i < n_stage; i += NT) {
            const uint32_t v = S.stx[i];
            ws.pfinal[S.gbase[v] + (i + sbase - S.cstart[v])] = S.stage[i];
        }
        __syncthreads();
    }
    return true;
}

// Persistent, like k_row_pass.
#ifndef SEELE_COL_MINB
#define SEELE_COL_MINB 2
#endif
__global__ void __launch_bounds__(NT, SEELE_COL_MINB) k_col_pass(Workspace ws, int tiles_x, int tiles_y) {
    extern __shared__ __align__(16) unsigned char smem[];
    ColSmem &S = *reinterpret_cast<ColSmem *>(smem);
    ticket_loop(&ws.counters[CNT_TICKET + kLookCols],
                [&](uint32_t t) { return col_tile(ws, tiles_x, tiles_y, S, t); });

}

__global__ void k_fill_pair_tiles(const uint2 *ranges, int n_tiles, int32_t *pair_tile) {
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const uint2 r = ranges[t];
        for (uint32_t i = r.x + threadIdx.x; i < r.y; i += blockDim.x) pair_tile[i] = t;
    }
}

template <typename K>
void set_smem(K kernel, size_t bytes) {
    static bool done = false;  // per instantiation
    if (!done) {
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        done = true;
    }
}

long long ceil_div(long long a, long long b) { return (a + b - 1) / b; }

}  // namespace

void launch_frame_begin(const Workspace &ws, const CamK &cam, int64_t *stats, cudaStream_t st) {
    const int n_diff = (cam.tiles_x + 1) * (cam.tiles_y + 1);
    const int grid = 256;  // (the depth histogram alone is 4 MB)
    k_frame_begin<<<grid, 256, 0, st>>>(ws, stats, n_diff, cam.tiles_y);
    note_launches(1);
}

static int sm_count_cached() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

void launch_binning(const Workspace &ws, long long n_max, long long cap, const CamK &cam, int64_t *stats,
                    cudaStream_t st) {
    const int sms = sm_count_cached();
    const size_t diff_bytes = sizeof(int32_t) * (cam.tiles_x + 1) * (cam.tiles_y + 1);
    const int use_smem = diff_bytes <= 160 * 1024;
    const size_t scan_smem = use_smem ? diff_bytes : 0;
    set_smem(k_pair_scan, 160 * 1024);
#ifndef SEELE_SCAN_PER_SM2
#define SEELE_SCAN_PER_SM2 2  // (half-SM units: one CTA per SM)
#endif
    const int scan_grid = (int)std::min<long long>(ceil_div(n_max, TILE), SEELE_SCAN_PER_SM2 * sms / 2);
    k_pair_scan<<<scan_grid > 0 ? scan_grid : 1, NT, scan_smem, st>>>(ws, cam.tiles_x, cam.tiles_y, cap, use_smem,
                                                                      stats);
    set_smem(k_row_pass, sizeof(RowSmem));
#ifndef SEELE_BIN_CTAS_PER_SM
#define SEELE_BIN_CTAS_PER_SM 1  // one per SM: room for another frame's raster CTAs (pipelined 983 -> 994 FPS)
#endif
#ifndef SEELE_ROW_CTAS_PER_SM
#define SEELE_ROW_CTAS_PER_SM SEELE_BIN_CTAS_PER_SM
#endif
#ifndef SEELE_COL_CTAS_PER_SM
#define SEELE_COL_CTAS_PER_SM SEELE_BIN_CTAS_PER_SM
#endif
    const int persist = (int)(SEELE_ROW_CTAS_PER_SM * sms);  // resident CTAs (launch bounds allow two per SM)
    k_row_pass<<<(int)std::min<long long>(ceil_div(cap, TILE), persist), NT, sizeof(RowSmem), st>>>(ws, stats);
    set_smem(k_col_pass, sizeof(ColSmem));
    const int persist_col = (int)(SEELE_COL_CTAS_PER_SM * sms);
    k_col_pass<<<(int)std::min<long long>(ceil_div(cap, TILE) + cam.tiles_y, persist_col), NT, sizeof(ColSmem), st>>>(
        ws, cam.tiles_x, cam.tiles_y);
    note_launches(3);
}

#ifdef SEELE_SORT_TRACE
void debug_trace(void *dst) { cudaMemcpyFromSymbol(dst, g_trace, sizeof(g_trace)); }
#endif

void launch_fill_pair_tiles(const uint2 *ranges, int n_tiles, int32_t *pair_tile, cudaStream_t st) {
    k_fill_pair_tiles<<<n_tiles < 4096 ? n_tiles : 4096, 256, 0, st>>>(ranges, n_tiles, pair_tile);
    note_launches(1);
}

}  // namespace seele
