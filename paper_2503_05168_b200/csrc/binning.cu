// Tile binning and sort on sm_100a.  Every size is read from device memory,
// so a frame needs no host round trip:
//   1. ordered compaction of the binned splats (assembled order)        [scan]
//   2. stable LSD radix sort of their fp64 depth bits                    [depth rank]
//      -> order by (depth, assembled position), the reference's
//         (depth, gaussian_ref) tie-break (sorting.py:43, render.py:108)
//   3. exclusive scan of tile counts in depth-rank order, then pair emission
//      load-balanced by pairs (key = tile id, value = assembled position)
//                                                                        [bin_tiles,
//      preprocess.py:159-189]
//   4. stable LSD radix sort on the tile id (ceil(log2 tiles) bits): stability
//      keeps depth-rank order inside a tile -> (tile_id, depth, ref) order of
//      sort_intersections (sorting.py:32-54)
//   5. per-tile [start, end) ranges                                     [sorting.py:46-53]
//
// Radix passes: per-block digit histograms, one scan block per digit, and a
// scatter that ranks IPT x 256 items per iteration stably (warp
// __match_any_sync + per-(sub-round, warp) digit prefixes), stages them in
// shared memory in digit order and writes digit runs coalesced.
#include "common.cuh"

namespace seele {

namespace {

__device__ __forceinline__ long long chunk_size(long long n, int G) {
    long long c = (n + G - 1) / G;
    return (c + 1023) / 1024 * 1024;
}

// 256-thread block exclusive scan of one value per thread.
template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T &total) {
    __shared__ T s_warp[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        T w = lane < 8 ? s_warp[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            T y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < 8) s_warp[lane] = w;  // inclusive
    }
    __syncthreads();
    T warp_off = warp ? s_warp[warp - 1] : T(0);
    total = s_warp[7];
    __syncthreads();
    return warp_off + x - v;
}

// ---- 1. ordered compaction of binned splats ----------------------------------

__global__ void __launch_bounds__(256) k_compact_reduce(Workspace ws) {
    const long long n = ws.counters[CNT_WS];
    const long long c = chunk_size(n, gridDim.x);
    const long long b0 = (long long)blockIdx.x * c, b1 = min(b0 + c, n);
    unsigned long long acc = 0;
    for (long long i = b0 + threadIdx.x; i < b1; i += blockDim.x) acc += ws.tiles[i] > 0 ? 1ull : 0ull;
    unsigned long long tot;
    block_exclusive_scan<unsigned long long>(acc, tot);
    if (threadIdx.x == 0) ws.block_sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_compact_sums(Workspace ws, int G) {
    __shared__ unsigned long long s[kChunkBlocksMax];
    for (int i = threadIdx.x; i < G; i += blockDim.x) s[i] = ws.block_sums[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long run = 0;
        for (int i = 0; i < G; i++) {
            const unsigned long long v = s[i];
            s[i] = run;
            run += v;
        }
        ws.counters[CNT_BINNED] = (uint32_t)run;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < G; i += blockDim.x) ws.block_sums[i] = s[i];
}

__global__ void __launch_bounds__(256) k_compact_write(Workspace ws) {
    const long long n = ws.counters[CNT_WS];
    const long long c = chunk_size(n, gridDim.x);
    const long long b0 = (long long)blockIdx.x * c, b1 = min(b0 + c, n);
    unsigned long long run = ws.block_sums[blockIdx.x];
    for (long long t0 = b0; t0 < b1; t0 += blockDim.x) {
        const long long i = t0 + threadIdx.x;
        const unsigned v = (i < b1 && ws.tiles[i] > 0) ? 1u : 0u;
        unsigned long long tot;
        const unsigned long long ex = block_exclusive_scan<unsigned long long>(v, tot) + run;
        if (v) {
            ws.dkey[0][ex] = (uint64_t)__double_as_longlong(ws.depth[i]);
            ws.dval[0][ex] = (uint32_t)i;
        }
        run += tot;
    }
}

// ---- stable LSD radix sort passes ---------------------------------------------

template <typename K>
__global__ void __launch_bounds__(256) k_radix_hist(const K *__restrict__ keys, const uint32_t *n_ptr, int shift,
                                                    int bits, uint32_t *hist) {
    __shared__ uint32_t h[256];
    const int nd = 1 << bits;
    h[threadIdx.x] = 0;
    __syncthreads();
    const long long n = *n_ptr;
    const long long c = chunk_size(n, gridDim.x);
    const long long b0 = (long long)blockIdx.x * c, b1 = min(b0 + c, n);
    const K mask = (K)(nd - 1);
    for (long long i = b0 + threadIdx.x; i < b1; i += blockDim.x)
        atomicAdd(&h[(uint32_t)((keys[i] >> shift) & mask)], 1u);
    __syncthreads();
    if (threadIdx.x < nd) hist[(long long)threadIdx.x * gridDim.x + blockIdx.x] = h[threadIdx.x];
}

// Per digit d (one block each): exclusive scan over the G block counts of that
// digit, in place, and the digit total into tot[d].
__global__ void __launch_bounds__(256) k_radix_scan(uint32_t *hist, uint32_t *tot, int G) {
    uint32_t *row = hist + (long long)blockIdx.x * G;
    const int per = (G + 255) / 256;
    const int a = threadIdx.x * per, b = min(a + per, G);
    uint32_t sum = 0;
    for (int i = a; i < b; i++) sum += row[i];
    uint32_t total;
    uint32_t run = block_exclusive_scan<uint32_t>(sum, total);
    for (int i = a; i < b; i++) {
        const uint32_t v = row[i];
        row[i] = run;
        run += v;
    }
    if (threadIdx.x == 0) tot[blockIdx.x] = total;
}

template <typename K, int IPT>
__global__ void __launch_bounds__(256) k_radix_scatter(const K *__restrict__ kin, const uint32_t *__restrict__ vin,
                                                       K *__restrict__ kout, uint32_t *__restrict__ vout,
                                                       const uint32_t *n_ptr, int shift, int bits,
                                                       const uint32_t *__restrict__ hist,
                                                       const uint32_t *__restrict__ tot) {
    constexpr int TILE = 256 * IPT;
    __shared__ uint32_t s_base[256];            // global destination of the next item of each digit
    __shared__ uint32_t s_loc[256];             // digit offsets inside the staged tile
    __shared__ uint16_t s_wh[IPT][8][256];      // per (sub-round, warp, digit) counts -> prefixes
    __shared__ K s_key[TILE];
    __shared__ uint32_t s_val[TILE];
    const int nd = 1 << bits;
    const int G = gridDim.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t digit_total;
    const uint32_t digit_base = block_exclusive_scan<uint32_t>(tid < nd ? tot[tid] : 0u, digit_total);
    s_base[tid] = tid < nd ? digit_base + hist[(long long)tid * G + blockIdx.x] : 0u;
#pragma unroll
    for (int r = 0; r < IPT; r++)
        for (int w = 0; w < 8; w++) s_wh[r][w][tid] = 0;
    __syncthreads();
    const long long n = *n_ptr;
    const long long c = chunk_size(n, G);
    const long long b0 = (long long)blockIdx.x * c, b1 = min(b0 + c, n);
    const K mask = (K)(nd - 1);
    const unsigned lt = (1u << lane) - 1u;
    for (long long t0 = b0; t0 < b1; t0 += TILE) {
        const int n_tile = (int)min((long long)TILE, b1 - t0);
        K key[IPT];
        uint32_t val[IPT], dig[IPT], rank[IPT];
#pragma unroll
        for (int r = 0; r < IPT; r++) {  // striped: item t0 + r*256 + tid keeps the input order
            const int li = r * 256 + tid;
            const bool valid = li < n_tile;
            dig[r] = 0xffffffffu;
            if (valid) {
                key[r] = kin[t0 + li];
                val[r] = vin[t0 + li];
                dig[r] = (uint32_t)((key[r] >> shift) & mask);
            }
            const unsigned peers = __match_any_sync(0xffffffffu, dig[r]);
            rank[r] = __popc(peers & lt);
            if (valid && rank[r] == 0) s_wh[r][warp][dig[r]] = (uint16_t)__popc(peers);
        }
        __syncthreads();
        uint32_t cnt = 0;
        if (tid < nd) {
#pragma unroll
            for (int r = 0; r < IPT; r++)
#pragma unroll
                for (int w = 0; w < 8; w++) {
                    const uint32_t v = s_wh[r][w][tid];
                    s_wh[r][w][tid] = (uint16_t)cnt;
                    cnt += v;
                }
        }
        uint32_t tile_total;
        const uint32_t loc = block_exclusive_scan<uint32_t>(cnt, tile_total);
        if (tid < nd) s_loc[tid] = loc;
        __syncthreads();
#pragma unroll
        for (int r = 0; r < IPT; r++) {
            if (dig[r] == 0xffffffffu) continue;
            const uint32_t li = s_loc[dig[r]] + s_wh[r][warp][dig[r]] + rank[r];
            s_key[li] = key[r];
            s_val[li] = val[r];
        }
        __syncthreads();
        for (int li = tid; li < n_tile; li += 256) {  // digit runs land on consecutive addresses
            const K k = s_key[li];
            const uint32_t d = (uint32_t)((k >> shift) & mask);
            const uint32_t dst = s_base[d] + (uint32_t)li - s_loc[d];
            kout[dst] = k;
            vout[dst] = s_val[li];
        }
        __syncthreads();
        if (tid < nd) {
            s_base[tid] += cnt;
#pragma unroll
            for (int r = 0; r < IPT; r++)
                for (int w = 0; w < 8; w++) s_wh[r][w][tid] = 0;
        }
        __syncthreads();
    }
}

template <typename K>
int radix_sort(K *keys[2], uint32_t *vals[2], const uint32_t *n_ptr, int begin_bit, int end_bit, uint32_t *hist,
               uint32_t *tot, int G, cudaStream_t st) {
    int cur = 0;
    for (int shift = begin_bit; shift < end_bit; shift += 8) {
        const int bits = min(8, end_bit - shift);
        k_radix_hist<K><<<G, 256, 0, st>>>(keys[cur], n_ptr, shift, bits, hist);
        k_radix_scan<<<1 << bits, 256, 0, st>>>(hist, tot, G);
        k_radix_scatter<K, 4><<<G, 256, 0, st>>>(keys[cur], vals[cur], keys[cur ^ 1], vals[cur ^ 1], n_ptr, shift,
                                                 bits, hist, tot);
        cur ^= 1;
        note_launches(3);
    }
    return cur;
}

// ---- 3. pair emission, load-balanced by pairs ----------------------------------

// Exclusive scan of the tile counts in depth-rank order -> first pair of each rank.
__global__ void __launch_bounds__(256) k_pairs_reduce(Workspace ws, const uint32_t *__restrict__ sorted_pos) {
    const long long n = ws.counters[CNT_BINNED];
    const long long c = chunk_size(n, gridDim.x);
    const long long b0 = (long long)blockIdx.x * c, b1 = min(b0 + c, n);
    unsigned long long acc = 0;
    for (long long r = b0 + threadIdx.x; r < b1; r += blockDim.x) acc += ws.tiles[sorted_pos[r]];
    unsigned long long tot;
    block_exclusive_scan<unsigned long long>(acc, tot);
    if (threadIdx.x == 0) ws.block_sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_pairs_sums(Workspace ws, int G, long long cap, int64_t *stats) {
    __shared__ unsigned long long s[kChunkBlocksMax];
    for (int i = threadIdx.x; i < G; i += blockDim.x) s[i] = ws.block_sums[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long run = 0;
        for (int i = 0; i < G; i++) {
            const unsigned long long v = s[i];
            s[i] = run;
            run += v;
        }
        stats[SEELE_STAT_TILE_PAIRS] = (int64_t)run;
        const bool over = run > (unsigned long long)cap;
        ws.counters[CNT_OVERFLOW] = over ? 1u : 0u;
        ws.counters[CNT_PAIRS] = over ? 0u : (uint32_t)run;
        stats[SEELE_STAT_OVERFLOW] = over ? 1 : 0;
        ws.poff[ws.counters[CNT_BINNED]] = run;  // sentinel for the emission search
    }
    __syncthreads();
    for (int i = threadIdx.x; i < G; i += blockDim.x) ws.block_sums[i] = s[i];
}

__global__ void __launch_bounds__(256) k_pairs_scan(Workspace ws, const uint32_t *__restrict__ sorted_pos) {
    const long long n = ws.counters[CNT_BINNED];
    const long long c = chunk_size(n, gridDim.x);
    const long long b0 = (long long)blockIdx.x * c, b1 = min(b0 + c, n);
    unsigned long long run = ws.block_sums[blockIdx.x];
    for (long long t0 = b0; t0 < b1; t0 += blockDim.x) {
        const long long r = t0 + threadIdx.x;
        const unsigned long long v = r < b1 ? (unsigned long long)ws.tiles[sorted_pos[r]] : 0ull;
        unsigned long long tot;
        const unsigned long long ex = block_exclusive_scan<unsigned long long>(v, tot) + run;
        if (r < b1) ws.poff[r] = ex;
        run += tot;
    }
}

// bin_tiles emission (preprocess.py:179-189) in depth-rank order, balanced by
// pairs: pair tile t = [t * kEmitTile, (t + 1) * kEmitTile) starts inside rank
// tile_r0[t] (found per rank by k_emit_starts, no search).  A block stages
// the ranks overlapping its tile, and each thread expands 8 consecutive pairs
// (ty-major, tx-minor inside a splat) with one search and a walk.
constexpr int kEmitTile = 2048;
constexpr int kEmitPerThread = kEmitTile / 256;

__global__ void __launch_bounds__(256) k_emit_starts(Workspace ws) {
    const long long n = ws.counters[CNT_BINNED];
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
        const unsigned long long a = ws.poff[r], b = ws.poff[r + 1];
        for (unsigned long long t = (a + kEmitTile - 1) / kEmitTile; t * kEmitTile < b; t++) ws.tile_r0[t] = (uint32_t)r;
    }
}

__global__ void __launch_bounds__(256) k_emit(Workspace ws, const uint32_t *__restrict__ sorted_pos, int tiles_x,
                                              uint32_t *__restrict__ pkey, uint32_t *__restrict__ pval) {
    __shared__ unsigned long long s_off[kEmitTile + 2];
    __shared__ uint32_t s_pos[kEmitTile + 1];
    __shared__ short4 s_rc[kEmitTile + 1];
    if (ws.counters[CNT_OVERFLOW]) return;
    const long long n = ws.counters[CNT_BINNED];
    const unsigned long long k_total = ws.counters[CNT_PAIRS];
    const unsigned long long n_tiles = (k_total + kEmitTile - 1) / kEmitTile;
    for (unsigned long long t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const unsigned long long base = t * kEmitTile, end = min(base + kEmitTile, k_total);
        const long long r0 = ws.tile_r0[t];
        const long long r1 = t + 1 < n_tiles ? (long long)ws.tile_r0[t + 1] : n - 1;  // last rank overlapping
        const int nr = (int)(r1 - r0 + 1);
        for (int k = threadIdx.x; k <= nr; k += blockDim.x) {
            s_off[k] = ws.poff[r0 + k];
            if (k < nr) {
                const uint32_t p = sorted_pos[r0 + k];
                s_pos[k] = p;
                s_rc[k] = ws.rect[p];
            }
        }
        __syncthreads();
        const unsigned long long i0 = base + (unsigned long long)threadIdx.x * kEmitPerThread;
        if (i0 < end) {
            int lo = 0, hi = nr - 1;  // rank holding pair i0
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (s_off[mid] <= i0) lo = mid; else hi = mid - 1;
            }
            short4 rc = s_rc[lo];
            int w = rc.y - rc.x + 1;
            const int local = (int)(i0 - s_off[lo]);
            int ty = rc.z + local / w;
            int tx = rc.x + local % w;
            unsigned long long next = s_off[lo + 1];
            uint32_t p = s_pos[lo];
            const unsigned long long stop = min(i0 + kEmitPerThread, end);
            for (unsigned long long i = i0; i < stop; i++) {
                if (i == next) {  // next splat
                    lo++;
                    rc = s_rc[lo];
                    w = rc.y - rc.x + 1;
                    ty = rc.z;
                    tx = rc.x;
                    next = s_off[lo + 1];
                    p = s_pos[lo];
                }
                pkey[i] = (uint32_t)(ty * tiles_x + tx);
                pval[i] = p;
                if (++tx > rc.y) {
                    tx = rc.x;
                    ty++;
                }
            }
        }
        __syncthreads();
    }
}

// ---- 5. ranges --------------------------------------------------------------------

__global__ void k_clear_ranges(uint2 *ranges, int n_tiles) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_tiles; t += gridDim.x * blockDim.x)
        ranges[t] = make_uint2(0u, 0u);
}

__global__ void __launch_bounds__(256) k_ranges(Workspace ws, const uint32_t *__restrict__ pkey) {
    const long long k = ws.counters[CNT_PAIRS];
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (long long)gridDim.x * blockDim.x) {
        const uint32_t t = pkey[i];
        if (i == 0 || pkey[i - 1] != t) ws.ranges[t].x = (uint32_t)i;
        if (i == k - 1 || pkey[i + 1] != t) ws.ranges[t].y = (uint32_t)(i + 1);
    }
}

}  // namespace

int chunk_grid(int sms) {
    int g = 4 * sms;
    return g > kChunkBlocksMax ? kChunkBlocksMax : g;
}

int key_bits(int n) {
    int b = 1;
    while ((1 << b) < n) b++;
    return b;
}

// Which ping-pong buffer holds the sorted pairs (seele_plan_export).
int pair_buffer(int n_tiles) { return ((key_bits(n_tiles) + 7) / 8) & 1; }

void launch_depth_rank(const Workspace &ws, long long n_max, int grid, int64_t *stats, uint32_t **sorted_pos,
                       cudaStream_t st) {
    (void)stats;
    const int G = grid;
    k_compact_reduce<<<G, 256, 0, st>>>(ws);
    k_compact_sums<<<1, 1024, 0, st>>>(ws, G);
    k_compact_write<<<G, 256, 0, st>>>(ws);
    note_launches(3);
    uint64_t *k[2] = {ws.dkey[0], ws.dkey[1]};
    uint32_t *v[2] = {ws.dval[0], ws.dval[1]};
    // positive doubles order like their bit patterns; bit 63 (sign) is always 0
    (void)n_max;
    const int Gd = G;
    const int cur = radix_sort<uint64_t>(k, v, ws.counters + CNT_BINNED, 0, 63, ws.hist, ws.hist + 256LL * kChunkBlocksMax,
                                         Gd, st);
    *sorted_pos = v[cur];
}

void launch_binning(const Workspace &ws, const uint32_t *sorted_pos, long long n_max, long long cap, const CamK &cam,
                    int grid, int64_t *stats, uint32_t **pair_pos, uint32_t **pair_tile, cudaStream_t st) {
    (void)n_max;
    const int G = grid;
    k_pairs_reduce<<<G, 256, 0, st>>>(ws, sorted_pos);
    k_pairs_sums<<<1, 1024, 0, st>>>(ws, G, cap, stats);
    k_pairs_scan<<<G, 256, 0, st>>>(ws, sorted_pos);
    k_emit_starts<<<G, 256, 0, st>>>(ws);
    k_emit<<<G, 256, 0, st>>>(ws, sorted_pos, cam.tiles_x, ws.pkey[0], ws.pval[0]);
    note_launches(5);
    const int n_tiles = cam.tiles_x * cam.tiles_y;
    uint32_t *k[2] = {ws.pkey[0], ws.pkey[1]};
    uint32_t *v[2] = {ws.pval[0], ws.pval[1]};
    const int cur = radix_sort<uint32_t>(k, v, ws.counters + CNT_PAIRS, 0, key_bits(n_tiles), ws.hist,
                                         ws.hist + 256LL * kChunkBlocksMax, G, st);
    k_clear_ranges<<<(n_tiles + 255) / 256, 256, 0, st>>>(ws.ranges, n_tiles);
    k_ranges<<<G, 256, 0, st>>>(ws, k[cur]);
    note_launches(2);
    *pair_pos = v[cur];
    *pair_tile = k[cur];
}

}  // namespace seele
