// Tile binning and sort on sm_100a, all sizes read from device memory (no
// host round trip inside a frame):
//   1. ordered compaction of binned splats (assembled order)      [scan]
//   2. stable LSD radix sort of their fp64 depth bits             [depth rank]
//      -> order by (depth, assembled position) = the reference's
//         (depth, gaussian_ref) tie-break (sorting.py:43, render.py:108)
//   3. exclusive scan of tile counts in depth-rank order          [pair offsets]
//   4. pair emission: key = tile id, value = assembled position   [bin_tiles,
//      preprocess.py:179-189]; emitted in depth-rank order
//   5. stable LSD radix sort by tile id (ceil(log2 tiles) bits)   [sort_intersections,
//      sorting.py:32-54]: stability keeps depth-rank order inside a tile
//   6. per-tile [start, end) ranges                               [sorting.py:46-53]
//
// The radix sort ranks stably inside a CTA with __match_any_sync over the
// digit (warp-level multisplit) and a per-tile warp-prefix in shared memory.
#include "common.cuh"

namespace seele {

namespace {

__device__ __forceinline__ long long chunk_size(long long n, int G) {
    long long c = (n + G - 1) / G;
    return (c + 255) / 256 * 256;
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

// ---- chunked exclusive scan with a device-resident item count --------------

// mode 0: flag = tiles[p] > 0 over p < counters[CNT_WS]          (compaction)
// mode 1: value = tiles[sorted_pos[r]] over r < counters[CNT_BINNED] (pair offsets)
template <int MODE>
__device__ __forceinline__ unsigned long long scan_value(const Workspace &ws, const uint32_t *sorted_pos,
                                                         long long i) {
    if (MODE == 0) return ws.tiles[i] > 0 ? 1ull : 0ull;
    return (unsigned long long)ws.tiles[sorted_pos[i]];
}

template <int MODE>
__device__ __forceinline__ long long scan_count(const Workspace &ws) {
    return MODE == 0 ? (long long)ws.counters[CNT_WS] : (long long)ws.counters[CNT_BINNED];
}

template <int MODE>
__global__ void __launch_bounds__(256) k_chunk_reduce(Workspace ws, const uint32_t *sorted_pos) {
    const long long n = scan_count<MODE>(ws);
    const int G = gridDim.x;
    const long long c = chunk_size(n, G);
    const long long b0 = (long long)blockIdx.x * c;
    const long long b1 = min(b0 + c, n);
    unsigned long long acc = 0;
    for (long long i = b0 + threadIdx.x; i < b1; i += blockDim.x) acc += scan_value<MODE>(ws, sorted_pos, i);
    unsigned long long tot;
    block_exclusive_scan<unsigned long long>(acc, tot);
    if (threadIdx.x == 0) ws.block_sums[blockIdx.x] = tot;
}

// Single block: exclusive scan of G block sums; publishes the total.
template <int MODE>
__global__ void __launch_bounds__(1024) k_scan_sums(Workspace ws, int G, long long cap, int64_t *stats) {
    __shared__ unsigned long long s[kChunkBlocksMax];
    for (int i = threadIdx.x; i < G; i += blockDim.x) s[i] = ws.block_sums[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long run = 0;
        for (int i = 0; i < G; i++) {
            unsigned long long v = s[i];
            s[i] = run;
            run += v;
        }
        ws.block_sums[G] = run;
        if (MODE == 0) {
            ws.counters[CNT_BINNED] = (uint32_t)run;
        } else {
            ws.pairs64[0] = run;
            stats[SEELE_STAT_TILE_PAIRS] = (int64_t)run;
            const bool over = run > (unsigned long long)cap;
            ws.counters[CNT_OVERFLOW] = over ? 1u : 0u;
            ws.counters[CNT_PAIRS] = over ? 0u : (uint32_t)run;
            stats[SEELE_STAT_OVERFLOW] = over ? 1 : 0;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < G; i += blockDim.x) ws.block_sums[i] = s[i];
}

template <int MODE>
__global__ void __launch_bounds__(256) k_chunk_scan(Workspace ws, const uint32_t *sorted_pos) {
    const long long n = scan_count<MODE>(ws);
    const int G = gridDim.x;
    const long long c = chunk_size(n, G);
    const long long b0 = (long long)blockIdx.x * c;
    const long long b1 = min(b0 + c, n);
    unsigned long long run = ws.block_sums[blockIdx.x];
    for (long long t0 = b0; t0 < b1; t0 += blockDim.x) {
        const long long i = t0 + threadIdx.x;
        const unsigned long long v = i < b1 ? scan_value<MODE>(ws, sorted_pos, i) : 0ull;
        unsigned long long tot;
        const unsigned long long ex = block_exclusive_scan<unsigned long long>(v, tot) + run;
        if (i < b1) {
            if (MODE == 0) {
                if (v) {
                    ws.dkey[0][ex] = (uint64_t)__double_as_longlong(ws.depth[i]);
                    ws.dval[0][ex] = (uint32_t)i;
                }
            } else {
                ws.poff[i] = ex;
            }
        }
        run += tot;
    }
}

// ---- stable LSD radix sort, device-resident count --------------------------

template <typename K>
__global__ void __launch_bounds__(256) k_radix_hist(const K *__restrict__ keys, const uint32_t *n_ptr, int shift,
                                                    int bits, uint32_t *hist) {
    __shared__ uint32_t h[256];
    const int nd = 1 << bits;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const long long n = *n_ptr;
    const int G = gridDim.x;
    const long long c = chunk_size(n, G);
    const long long b0 = (long long)blockIdx.x * c;
    const long long b1 = min(b0 + c, n);
    const K mask = (K)(nd - 1);
    for (long long i = b0 + threadIdx.x; i < b1; i += blockDim.x) atomicAdd(&h[(uint32_t)((keys[i] >> shift) & mask)], 1u);
    __syncthreads();
    for (int d = threadIdx.x; d < nd; d += blockDim.x) hist[(long long)d * G + blockIdx.x] = h[d];
}

// Per digit d (one block each): exclusive scan over the G block counts of
// that digit, in place, and the digit total into tot[d].
__global__ void __launch_bounds__(256) k_radix_scan(uint32_t *hist, uint32_t *tot, int G) {
    const int d = blockIdx.x;
    uint32_t *row = hist + (long long)d * G;
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
    if (threadIdx.x == 0) tot[d] = total;
}

template <typename K>
__global__ void __launch_bounds__(256) k_radix_scatter(const K *__restrict__ kin, const uint32_t *__restrict__ vin,
                                                       K *__restrict__ kout, uint32_t *__restrict__ vout,
                                                       const uint32_t *n_ptr, int shift, int bits,
                                                       const uint32_t *__restrict__ hist,
                                                       const uint32_t *__restrict__ tot) {
    __shared__ uint32_t base[256];
    __shared__ uint32_t wh[2][8][256];
    const int nd = 1 << bits;
    const int G = gridDim.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // global base of digit d = (all keys with a smaller digit) + (digit d in earlier blocks)
    uint32_t digit_total;
    const uint32_t digit_base = block_exclusive_scan<uint32_t>(tid < nd ? tot[tid] : 0u, digit_total);
    base[tid] = tid < nd ? digit_base + hist[(long long)tid * G + blockIdx.x] : 0u;
    for (int w = 0; w < 8; w++) wh[0][w][tid] = wh[1][w][tid] = 0u;
    __syncthreads();
    const long long n = *n_ptr;
    const long long c = chunk_size(n, G);
    const long long b0 = (long long)blockIdx.x * c;
    const long long b1 = min(b0 + c, n);
    const K mask = (K)(nd - 1);
    const unsigned lt = (1u << lane) - 1u;
    int buf = 0;
    for (long long t0 = b0; t0 < b1; t0 += 256) {
        const long long i = t0 + tid;
        const bool valid = i < b1;
        K key = 0;
        uint32_t val = 0, d = 0xffffffffu;
        if (valid) {
            key = kin[i];
            val = vin[i];
            d = (uint32_t)((key >> shift) & mask);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const uint32_t rank = __popc(peers & lt);
        if (valid && rank == 0) wh[buf][warp][d] = __popc(peers);
        __syncthreads();
        uint32_t tot = 0;
        if (tid < nd) {
#pragma unroll
            for (int w = 0; w < 8; w++) {
                const uint32_t cnt = wh[buf][w][tid];
                wh[buf][w][tid] = tot;
                tot += cnt;
            }
        }
        __syncthreads();
        if (valid) {
            const uint32_t pos = base[d] + wh[buf][warp][d] + rank;
            kout[pos] = key;
            vout[pos] = val;
        }
        __syncthreads();
        if (tid < nd) {
            base[tid] += tot;
#pragma unroll
            for (int w = 0; w < 8; w++) wh[buf][w][tid] = 0u;
        }
        buf ^= 1;
    }
}

template <typename K>
int radix_sort(K *keys[2], uint32_t *vals[2], const uint32_t *n_ptr, int begin_bit, int end_bit, uint32_t *hist,
               int G, cudaStream_t st) {
    int cur = 0;
    uint32_t *tot = hist + 256LL * kChunkBlocksMax;
    for (int shift = begin_bit; shift < end_bit; shift += 8) {
        const int bits = min(8, end_bit - shift);
        k_radix_hist<K><<<G, 256, 0, st>>>(keys[cur], n_ptr, shift, bits, hist);
        k_radix_scan<<<1 << bits, 256, 0, st>>>(hist, tot, G);
        k_radix_scatter<K><<<G, 256, 0, st>>>(keys[cur], vals[cur], keys[cur ^ 1], vals[cur ^ 1], n_ptr, shift, bits,
                                              hist, tot);
        cur ^= 1;
        note_launches(3);
    }
    return cur;
}

// ---- pair emission and ranges -----------------------------------------------

// bin_tiles emission (preprocess.py:179-189), warp-cooperative: each warp
// takes 32 depth-ranked splats and writes their tile pairs one splat at a
// time with all 32 lanes (coalesced stores, no per-thread serial loops over
// the few splats that cover thousands of tiles).
__global__ void __launch_bounds__(256) k_emit(Workspace ws, const uint32_t *__restrict__ sorted_pos, int tiles_x,
                                              uint32_t *__restrict__ pkey, uint32_t *__restrict__ pval) {
    if (ws.counters[CNT_OVERFLOW]) return;
    const long long n = ws.counters[CNT_BINNED];
    const int lane = threadIdx.x & 31;
    const long long warp0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long n_warps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long base = warp0 * 32; base < n; base += n_warps * 32) {
        const long long r = base + lane;
        uint32_t p = 0, lo = 0, hi = 0;
        unsigned long long off = 0;
        if (r < n) {
            p = sorted_pos[r];
            const short4 rc = ws.rect[p];
            lo = (uint32_t)(uint16_t)rc.x | ((uint32_t)(uint16_t)rc.y << 16);
            hi = (uint32_t)(uint16_t)rc.z | ((uint32_t)(uint16_t)rc.w << 16);
            off = ws.poff[r];
        }
        const int m = (int)min(32LL, n - base);
        for (int g = 0; g < m; g++) {
            const uint32_t gp = __shfl_sync(0xffffffffu, p, g);
            const uint32_t glo = __shfl_sync(0xffffffffu, lo, g);
            const uint32_t ghi = __shfl_sync(0xffffffffu, hi, g);
            const unsigned long long goff = __shfl_sync(0xffffffffu, off, g);
            const int tx0 = (int)(glo & 0xffff), tx1 = (int)(glo >> 16);
            const int ty0 = (int)(ghi & 0xffff), ty1 = (int)(ghi >> 16);
            const int w = tx1 - tx0 + 1;
            const int cnt = w * (ty1 - ty0 + 1);
            for (int k = lane; k < cnt; k += 32) {
                const int ty = k / w;
                const int tx = k - ty * w;
                pkey[goff + k] = (uint32_t)((ty0 + ty) * tiles_x + tx0 + tx);
                pval[goff + k] = gp;
            }
        }
    }
}

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

void launch_depth_rank(const Workspace &ws, long long n_max, int grid, int64_t *stats, uint32_t **sorted_pos,
                       cudaStream_t st) {
    (void)n_max;
    const int G = grid;
    k_chunk_reduce<0><<<G, 256, 0, st>>>(ws, nullptr);
    k_scan_sums<0><<<1, 1024, 0, st>>>(ws, G, 0, stats);
    k_chunk_scan<0><<<G, 256, 0, st>>>(ws, nullptr);
    note_launches(3);
    uint64_t *k[2] = {ws.dkey[0], ws.dkey[1]};
    uint32_t *v[2] = {ws.dval[0], ws.dval[1]};
    // positive doubles order like their bit patterns; bit 63 (sign) is always 0
    const int cur = radix_sort<uint64_t>(k, v, ws.counters + CNT_BINNED, 0, 63, ws.hist, G, st);
    *sorted_pos = v[cur];
}

void launch_binning(const Workspace &ws, const uint32_t *sorted_pos, long long n_max, long long cap, const CamK &cam,
                    int grid, int64_t *stats, uint32_t **pair_pos, uint32_t **pair_tile, cudaStream_t st) {
    (void)n_max;
    const int G = grid;
    k_chunk_reduce<1><<<G, 256, 0, st>>>(ws, sorted_pos);
    k_scan_sums<1><<<1, 1024, 0, st>>>(ws, G, cap, stats);
    k_chunk_scan<1><<<G, 256, 0, st>>>(ws, sorted_pos);
    k_emit<<<G, 256, 0, st>>>(ws, sorted_pos, cam.tiles_x, ws.pkey[0], ws.pval[0]);
    note_launches(4);
    const int n_tiles = cam.tiles_x * cam.tiles_y;
    int bits = 1;
    while ((1 << bits) < n_tiles) bits++;
    uint32_t *k[2] = {ws.pkey[0], ws.pkey[1]};
    uint32_t *v[2] = {ws.pval[0], ws.pval[1]};
    const int cur = radix_sort<uint32_t>(k, v, ws.counters + CNT_PAIRS, 0, bits, ws.hist, G, st);
    k_clear_ranges<<<(n_tiles + 255) / 256, 256, 0, st>>>(ws.ranges, n_tiles);
    k_ranges<<<G, 256, 0, st>>>(ws, k[cur]);
    note_launches(2);
    *pair_pos = v[cur];
    *pair_tile = k[cur];
}

}  // namespace seele
