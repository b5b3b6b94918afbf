// Depth order of the binned splats on sm_100a: an exact (fp64 depth,
// assembled position) sort -- the order of np.lexsort((ref, depth, tile))
// inside every tile (sorting.py:32-54), refs being assigned in assembled
// order (render.py:108, 118) -- without quantised keys, tie fix-ups or a
// min / max round trip:
//
//   K1 (preprocess.cu)  every binned splat counts itself in the histogram of
//                       its depth bucket -- the top bits of the
//                       order-preserving fp64 bit pattern of z above the near
//                       plane (65,536 buckets per binade, 16 binades; deeper
//                       splats share the last bucket) -- and keeps the
//                       atomic's return value, its index inside the bucket.
//                       The bucket is a monotone function of z, so bucket
//                       order is depth order.
//   k_bucket_scan       exclusive offsets of the 2^20 buckets (16K per CTA,
//                       decoupled look-back) and the first bucket of every
//                       2048-item sort group.
//   k_bucket_scatter    each binned splat writes one 16-byte record (order
//                       key, position, packed tile rect) to offset + index:
//                       bucket order, arbitrary order inside a bucket.
//   k_bucket_sort       one CTA per group of whole buckets (~2048 items):
//                       every item's slot inside its bucket = the number of
//                       bucket members before it in (depth, position) order
//                       (buckets of <= 64 items, ~10 on C3), else a
//                       shared-memory bitonic sort of the group (<= 4096
//                       items), else -- thousands of splats within 1.5e-5
//                       relative depth, a wall facing the camera -- a merge
//                       sort in global memory by that CTA.
//
// Comparisons use the exact fp64 depth and the position, so equal depths
// order by position like the reference; the result is independent of the
// order of K1's atomics.
#include <algorithm>

#include "onesweep.cuh"

namespace seele {

namespace {

constexpr int kScanThreads = 1024;
constexpr int kPerThread = kDepthScanItems / kScanThreads;  // 16 buckets per thread
static_assert(kPerThread % 4 == 0 && kDepthBuckets % kDepthScanItems == 0, "scan tiling");
constexpr int kSortThreads = 256;
constexpr int kRankMaxBucket = 128;  // buckets up to this size are ranked by counting


// (depth, position) strictly before
__device__ __forceinline__ bool before(unsigned long long ka, uint32_t pa, unsigned long long kb, uint32_t pb) {
    return ka < kb || (ka == kb && pa < pb);
}
__device__ __forceinline__ unsigned long long rec_key(const uint4 &r) {
    return ((unsigned long long)r.y << 32) | r.x;
}
__device__ __forceinline__ bool rec_before(const uint4 &a, const uint4 &b) {
    return before(rec_key(a), a.z, rec_key(b), b.z);
}

// Exclusive bucket offsets: CTA t scans buckets [t K, (t + 1) K), K = kDepthScanItems, and resolves its prefix
// by look-back over the lower CTAs.  Bucket c with items [lo, hi) starts every sort group g with
// lo < g G <= hi at bucket c + 1 (gfirst[g] = c + 1 = the first bucket whose offset is >= g G).
__global__ void __launch_bounds__(kScanThreads) k_bucket_scan(Workspace ws, const int64_t *stats) {
    using namespace sweep;
    __shared__ uint32_t s_warp[kScanThreads / 32];
    __shared__ uint32_t s_prev;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t t = blockIdx.x;
    const uint32_t n = (uint32_t)stats[SEELE_STAT_BINNED];
    uint4 *seg = reinterpret_cast<uint4 *>(ws.bhist + (size_t)t * kDepthScanItems) + tid * (kPerThread / 4);
    uint4 c[kPerThread / 4];
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < kPerThread / 4; k++) {
        c[k] = seg[k];
        sum += c[k].x + c[k].y + c[k].z + c[k].w;
    }
    uint32_t x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = s_warp[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        s_warp[lane] = w;
        const uint32_t prev = lookback_warp(ws.look_region(kLookBuckets), t, *ws.epoch * 16u + kLookBuckets,
                                            __shfl_sync(0xffffffffu, w, 31), t == 0);
        if (lane == 0) s_prev = prev;
    }
    __syncthreads();
    uint32_t run = s_prev + (warp ? s_warp[warp - 1] : 0u) + x - sum;  // offset of this thread's first bucket
    const uint32_t b_first = t * kDepthScanItems + tid * kPerThread;
#pragma unroll
    for (int k = 0; k < kPerThread / 4; k++) {
        const uint32_t cnt[4] = {c[k].x, c[k].y, c[k].z, c[k].w};
        uint32_t o[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            o[u] = run;
            const uint32_t hi = run + cnt[u];
            // groups starting at the next bucket (rare: one per ~2048 items)
            for (uint32_t g = run / kDepthGroup + 1; g * (uint32_t)kDepthGroup <= hi && g * (uint32_t)kDepthGroup < n;
                 g++)
                ws.gfirst[g] = b_first + 4 * k + u + 1;
            run = hi;
        }
        seg[k] = make_uint4(o[0], o[1], o[2], o[3]);
    }
    if (t == 0 && tid == 0) {
        ws.gfirst[0] = 0u;
        ws.bhist[kDepthBuckets] = n;
    }
}

#ifndef SEELE_SCATTER_THREADS
#define SEELE_SCATTER_THREADS 256
#endif
// One assembled splat per thread (the grid covers them all): every load of a warp is in flight together.
__global__ void __launch_bounds__(SEELE_SCATTER_THREADS) k_bucket_scatter(Workspace ws, CamK cam) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= ws.counters[CNT_WS]) return;
    const uint4 sr = ws.srec[p];  // (packed rect, bucket index, depth): one load, then the bucket offset
    if ((sr.x & 0xffu) > ((sr.x >> 8) & 0xffu)) return;  // not binned
    const unsigned long long key = depth_order_key(__hiloint2double((int)sr.w, (int)sr.z));
    const uint32_t slot = ws.bhist[depth_bucket_of_key(key, depth_order_key(cam.near_clip))] + sr.y;
    ws.brec[0][slot] = make_uint4((uint32_t)key, (uint32_t)(key >> 32), p, sr.x);
}

union SortSmem {
    struct {
        unsigned long long pk[kDepthSmem];  // in-bucket order key: low 36 bits of (key - base) << 28 | position
        uint2 pr[kDepthSmem];               // (position, packed rect)
        uint16_t b0[kDepthSmem], b1[kDepthSmem];  // the item's bucket as a group-local [begin, end)
    } r;
    uint4 rec[kDepthSmem];  // full records: bitonic / merge paths
};

// Bitonic sort of the n (<= kDepthSmem) records in shared memory by (key, pos);
// slots n.. are padded with +inf.
__device__ void smem_bitonic(SortSmem &S, int n) {
    int p2 = 1;
    while (p2 < n) p2 <<= 1;
    for (int i = n + threadIdx.x; i < p2; i += blockDim.x) S.rec[i] = make_uint4(~0u, ~0u, ~0u, 0u);
    __syncthreads();
    for (int k = 2; k <= p2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int t = threadIdx.x; t < p2 / 2; t += blockDim.x) {
                const int i = 2 * t - (t & (j - 1));  // lower index of the pair (bit j clear)
                const int l = i + j;
                const bool up = (i & k) == 0;
                const uint4 a = S.rec[i], b = S.rec[l];
                if (rec_before(b, a) == up) {
                    S.rec[i] = b;
                    S.rec[l] = a;
                }
            }
            __syncthreads();
        }
    }
}

// Merge sort of a large group [s, e) by one CTA in global memory: chunks of
// kDepthSmem sorted in shared memory, then rounds of pairwise merges (merge
// path: every thread finds its output span's split by binary search) between
// brec[0] and brec[1]; positions and rects end in dval[0] / drect[0].
__device__ void global_merge_sort(const Workspace &ws, SortSmem &S, uint32_t s, uint32_t e) {
    const uint32_t m = e - s;
    uint4 *x = ws.brec[1] + s, *y = ws.brec[0] + s;
    for (uint32_t c0 = 0; c0 < m; c0 += kDepthSmem) {  // chunks: y -> x
        const int cn = (int)min((uint32_t)kDepthSmem, m - c0);
        for (int i = threadIdx.x; i < cn; i += blockDim.x) S.rec[i] = y[c0 + i];
        __syncthreads();
        smem_bitonic(S, cn);
        for (int i = threadIdx.x; i < cn; i += blockDim.x) x[c0 + i] = S.rec[i];
        __syncthreads();
    }
    bool in_x = true;
    for (uint32_t w = kDepthSmem; w < m; w <<= 1) {
        const uint4 *a = in_x ? x : y;
        uint4 *b = in_x ? y : x;
        for (uint32_t a0 = 0; a0 < m; a0 += 2 * w) {
            const uint32_t a1 = min(a0 + w, m), b1 = min(a0 + 2 * w, m);
            const uint32_t la = a1 - a0, lb = b1 - a1, len = la + lb;
            const uint32_t per = (len + blockDim.x - 1) / blockDim.x;
            const uint32_t o0 = min(threadIdx.x * per, len), o1 = min(o0 + per, len);
            // merge path split of diagonal o0: i items from A, o0 - i from B
            uint32_t lo = o0 > lb ? o0 - lb : 0u, hi = min(o0, la);
            while (lo < hi) {
                const uint32_t i = (lo + hi) >> 1;
                if (rec_before(a[a1 + (o0 - i - 1)], a[a0 + i])) hi = i; else lo = i + 1;
            }
            uint32_t i = lo, j = o0 - lo;
            for (uint32_t o = o0; o < o1; o++) {
                const bool take_a = j >= lb || (i < la && !rec_before(a[a1 + j], a[a0 + i]));
                b[a0 + o] = take_a ? a[a0 + i] : a[a1 + j];
                if (take_a) i++; else j++;
            }
        }
        __syncthreads();
        in_x = !in_x;
    }
    const uint4 *res = in_x ? x : y;
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        const uint4 r = res[i];
        ws.dval[0][s + i] = r.z;
        ws.drect[0][s + i] = r.w;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kSortThreads) k_bucket_sort(Workspace ws, CamK cam, const int64_t *stats) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SortSmem &S = *reinterpret_cast<SortSmem *>(smem_raw);
    const uint32_t n = (uint32_t)stats[SEELE_STAT_BINNED];
    const uint32_t ng = (n + kDepthGroup - 1) / kDepthGroup;
    const uint32_t n_ws = ws.counters[CNT_WS];
    const unsigned long long base = depth_order_key(cam.near_clip);
    const uint4 *in = ws.brec[0];
    uint32_t *pout = ws.dval[0], *rout = ws.drect[0];
    for (uint32_t g = blockIdx.x; g < ng; g += gridDim.x) {
        const uint32_t s = ws.bhist[ws.gfirst[g]];
        const uint32_t e = (g + 1) * (uint32_t)kDepthGroup >= n ? n : ws.bhist[ws.gfirst[g + 1]];
        if (e <= s) continue;
        const uint32_t m = e - s;
        if (m > (uint32_t)kDepthSmem) {
            global_merge_sort(ws, S, s, e);
            continue;
        }
        constexpr int U = kDepthSmem / kSortThreads;
        uint32_t bk[U];  // each item's depth bucket
        {
            uint4 r[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint32_t i = threadIdx.x + u * kSortThreads;
                if (i < m) r[u] = in[s + i];
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint32_t i = threadIdx.x + u * kSortThreads;
                bk[u] = i < m ? depth_bucket_of_key(rec_key(r[u]), base) : 0u;
                if (i < m) {
                    // inside one bucket (< the clamped last one) the keys share every bit above bit 36 of
                    // key - base, so (low 36 bits, position) orders them; positions < 2^28
                    const unsigned long long rel = rec_key(r[u]) - base;
                    S.r.pk[i] = ((rel & ((1ull << kDepthShift) - 1ull)) << 28) | r[u].z;
                    S.r.pr[i] = make_uint2(r[u].z, r[u].w);
                }
            }
        }
        __syncthreads();
        // bucket bounds: the scanned bucket offsets (bhist, exclusive, bhist[kDepthBuckets] = n) give every
        // item its bucket's [begin, end) inside the group directly
        bool small = n_ws < (1u << 28);  // (positions fit the packed key)
        {
            uint32_t lo[U], hi[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint32_t i = threadIdx.x + u * kSortThreads;
                lo[u] = i < m ? ws.bhist[bk[u]] : s;
                hi[u] = i < m ? ws.bhist[bk[u] + 1] : s;
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint32_t i = threadIdx.x + u * kSortThreads;
                if (i < m) {
                    S.r.b0[i] = (uint16_t)(lo[u] - s);
                    S.r.b1[i] = (uint16_t)(hi[u] - s);
                    small &= hi[u] - lo[u] <= (uint32_t)kRankMaxBucket && bk[u] != (uint32_t)(kDepthBuckets - 1);
                }
            }
        }
        if (__syncthreads_and(small)) {
            // slot inside the bucket = members before it in (depth, position) order
            for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
                const unsigned long long k = S.r.pk[i];
                const uint32_t lo = S.r.b0[i], hi = S.r.b1[i];
                uint32_t rank = 0;
                for (uint32_t j = lo; j < hi; j++) rank += S.r.pk[j] < k;
                const uint2 pr = S.r.pr[i];
                pout[s + lo + rank] = pr.x;
                rout[s + lo + rank] = pr.y;
            }
        } else {
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) S.rec[i] = in[s + i];
            __syncthreads();
            smem_bitonic(S, (int)m);
            for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
                pout[s + i] = S.rec[i].z;
                rout[s + i] = S.rec[i].w;
            }
        }
        __syncthreads();  // the staging array is reused by the next group
    }
}

}  // namespace

void launch_depth_sort(const Workspace &ws, const CamK &cam, long long n_max, int64_t *stats, cudaStream_t st) {
    const int sms = stream_sms(st);
    k_bucket_scan<<<kDepthBuckets / kDepthScanItems, kScanThreads, 0, st>>>(ws, stats);
#ifndef SEELE_SCATTER_PER_SM
#define SEELE_SCATTER_PER_SM 4
#endif
    const long long sc_blocks = (n_max + SEELE_SCATTER_THREADS - 1) / SEELE_SCATTER_THREADS;
    k_bucket_scatter<<<(int)std::max<long long>(sc_blocks, 1), SEELE_SCATTER_THREADS, 0, st>>>(ws, cam);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_bucket_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SortSmem));
        attr = true;
    }
#ifndef SEELE_BSORT_PER_SM
#define SEELE_BSORT_PER_SM 8  // (vs 5: depth 0.076 -> 0.072 ms serial, C3)
#endif
    const long long groups = n_max / kDepthGroup + 1;
    const int so_grid = (int)std::min<long long>(groups, SEELE_BSORT_PER_SM * sms);
    k_bucket_sort<<<so_grid, kSortThreads, sizeof(SortSmem), st>>>(ws, cam, stats);
    note_launches(3);
}

}  // namespace seele
