// Single-pass ("onesweep") building blocks of the stable LSD radix passes and
// the prefix scans of the binning stage, sm_100a.
//
// A pass is ONE kernel: every CTA takes a ticket (dynamic tile id, so every
// lower tile is already resident when it looks back), ranks its NT * IPT items by
// digit inside the CTA (per-bit warp ballots + per-warp digit counters in
// shared memory, stable in input order), publishes its per-digit counts and
// resolves their exclusive prefix over the lower tiles by decoupled look-back,
// then scatters the digit-sorted tile with coalesced runs.  Loads are issued
// unconditionally (clamped index) so all IPT of them are in flight at once.  The per-digit
// global bases come from an up-front histogram.
//
// Status words are tagged with a per-pass epoch (frame counter * 16 + pass id),
// so the look-back arrays are never cleared: a word from an older pass simply
// does not match.  The workspace must be zero-filled once when allocated.
#pragma once
#include "common.cuh"

namespace seele {
namespace sweep {

constexpr int NT = SEELE_SORT_NT;    // threads per CTA
constexpr int IPT = SEELE_SORT_IPT;  // items per thread
constexpr int TILE = NT * IPT;   // items per CTA tile
constexpr int RADIX = 256;       // max digit values per pass (status stride)
constexpr uint32_t FLAG_AGG = 1u << 30;
constexpr uint32_t FLAG_INC = 2u << 30;
constexpr uint32_t VAL_MASK = (1u << 30) - 1u;
constexpr uint32_t NO_DIGIT = 0xffffffffu;

__device__ __forceinline__ void publish(unsigned long long *w, uint32_t epoch, uint32_t flag, uint32_t v) {
    const unsigned long long x = ((unsigned long long)epoch << 32) | flag | (v < VAL_MASK ? v : VAL_MASK);
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(w), "l"(x) : "memory");
}

__device__ __forceinline__ unsigned long long peek(const unsigned long long *w) {
    unsigned long long x;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(w) : "memory");
    return x;
}

// Decoupled look-back for one column (digit) of a status matrix laid out
// [tile][stride]: publishes this tile's aggregate, walks back to the nearest
// inclusive prefix, publishes its own inclusive prefix and returns the
// exclusive one.  Values saturate at VAL_MASK (only reachable on overflow).
//
// The walk reads its predecessor first (in steady state it already holds an
// inclusive prefix: one round trip); otherwise it reads windows of kWindow
// predecessors with independent loads, so a wave of CTAs that start together
// resolves kWindow tiles per L2 round trip instead of one.  Measured best at
// 4 (16: depth sort 168 us / binning 289 us; 4: 155 / 263 us): wider windows
// cost more registers and issue than the round trips they save.
#ifndef SEELE_LOOK_WINDOW
#define SEELE_LOOK_WINDOW 4
#endif
constexpr int kWindow = SEELE_LOOK_WINDOW;

// `start` marks the first tile of a chain (tile 0, or the first chunk of a
// segment whose chain restarts).
__device__ __forceinline__ uint32_t lookback(unsigned long long *col, int stride, uint32_t tile, uint32_t epoch,
                                             uint32_t mine, bool start) {
    if (start) {
        publish(col + (size_t)tile * stride, epoch, FLAG_INC, mine);
        return 0u;
    }
    publish(col + (size_t)tile * stride, epoch, FLAG_AGG, mine);
    uint32_t sum = 0;
    long long j = (long long)tile - 1;  // nearest predecessor not yet consumed
    {
        const unsigned long long x = peek(col + (size_t)j * stride);
        if ((uint32_t)(x >> 32) == epoch) {
            sum = (uint32_t)x & VAL_MASK;
            if ((uint32_t)x & FLAG_INC) {
                publish(col + (size_t)tile * stride, epoch, FLAG_INC, sum + mine);
                return sum;
            }
            j--;
        }
    }
    while (true) {
        unsigned long long x[kWindow];
#pragma unroll
        for (int w = 0; w < kWindow; w++) x[w] = j - w >= 0 ? peek(col + (size_t)(j - w) * stride) : 0ull;
        bool done = false;
        int used = 0;
#pragma unroll
        for (int w = 0; w < kWindow; w++) {
            if (done || used < w) continue;  // consume in order up to the first gap / inclusive
            if (j - w < 0 || (uint32_t)(x[w] >> 32) != epoch) continue;
            const uint32_t lo = (uint32_t)x[w];
            sum += lo & VAL_MASK;
            if (sum > VAL_MASK) sum = VAL_MASK;
            used = w + 1;
            done = (lo & FLAG_INC) != 0u;
        }
        if (done) break;
        j -= used;
        if (used == 0) __nanosleep(32);  // predecessor still ranking
    }
    publish(col + (size_t)tile * stride, epoch, FLAG_INC, sum + mine);
    return sum;
}

// Look-back of a single column (stride 1) by one whole warp: the 32 lanes
// read 32 predecessors per round trip (coalesced), the warp consumes them in
// order up to the first one not yet published or the first inclusive prefix.
// Returns the exclusive prefix in every lane.
__device__ __forceinline__ uint32_t lookback_warp(unsigned long long *col, uint32_t tile, uint32_t epoch,
                                                  uint32_t mine, bool start) {
    const int lane = threadIdx.x & 31;
    if (start) {
        if (lane == 0) publish(col + tile, epoch, FLAG_INC, mine);
        return 0u;
    }
    if (lane == 0) publish(col + tile, epoch, FLAG_AGG, mine);
    uint32_t sum = 0;
    long long j = (long long)tile - 1;
    while (true) {
        const long long jj = j - lane;
        const unsigned long long x = jj >= 0 ? peek(col + jj) : 0ull;
        const bool valid = jj >= 0 && (uint32_t)(x >> 32) == epoch;
        const unsigned vb = __ballot_sync(0xffffffffu, valid);
        const unsigned ib = __ballot_sync(0xffffffffu, valid && ((uint32_t)x & FLAG_INC) != 0u);
        const int gap = ~vb ? __ffs(~vb) - 1 : 32;
        const int inc = ib ? __ffs(ib) - 1 : 32;
        const bool done = inc < gap;
        const int take = done ? inc + 1 : gap;
        sum += __reduce_add_sync(0xffffffffu, lane < take ? ((uint32_t)x & VAL_MASK) : 0u);
        if (sum > VAL_MASK) sum = VAL_MASK;
        if (done) break;
        j -= take;
        if (take == 0) __nanosleep(32);  // predecessor still counting
    }
    if (lane == 0) publish(col + tile, epoch, FLAG_INC, sum + mine);
    return sum;
}

// 256-thread block exclusive scan of one value per thread (uses its own smem).
template <typename T>
__device__ __forceinline__ T block_scan(T v, T &total) {
    __shared__ T s_warp[NT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        T w = lane < NT / 32 ? s_warp[lane] : T(0);
#pragma unroll
        for (int o = 1; o < NT / 32; o <<= 1) {
            const T y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < NT / 32) s_warp[lane] = w;
    }
    __syncthreads();
    const T off = warp ? s_warp[warp - 1] : T(0);
    total = s_warp[NT / 32 - 1];
    __syncthreads();
    return off + x - v;
}

// Per-CTA scratch of block_rank.
struct __align__(16) RankSmem {
    uint32_t cnt[NT / 32][RADIX];  // per-warp digit counters -> per-warp exclusive offsets
    uint32_t start[RADIX];         // first slot of each digit in the sorted tile
    uint32_t total;                // ranked items in the tile
};

// Stable in-tile ranking; kBallot: peers by per-bit ballots instead of
// __match_any_sync (faster on sm_100: depth sort 186 -> 165 us).  Item (warp w, round r, lane l) is tile item
// w * 32 * IPT + r * 32 + l; dig[r] = NO_DIGIT marks an absent item.  On
// return pos[r] is the item's slot in the digit-sorted tile, sm.start[d] the
// first slot of digit d, and thread d (< RADIX) holds the tile's count of
// digit d in `count`.
template <bool kBallot, int IPT_ = IPT>
__device__ __forceinline__ void block_rank(const uint32_t (&dig)[IPT_], uint32_t (&pos)[IPT_], RankSmem &sm,
                                           uint32_t &count) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int d = lane; d < RADIX; d += 32) sm.cnt[warp][d] = 0u;
    __syncwarp();
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < IPT_; r++) {
        const uint32_t d = dig[r];
        unsigned peers;
        if (kBallot) {
            // lanes with the same 8-bit digit: one ballot per bit (absent items excluded)
            peers = __ballot_sync(0xffffffffu, d != NO_DIGIT);
#pragma unroll
            for (int b = 0; b < 8; b++) {
                const uint32_t bit = (d >> b) & 1u;
                const unsigned bb = __ballot_sync(0xffffffffu, bit);
                peers &= bb ^ (bit - 1u);  // bit set: lanes with the bit; clear: lanes without
            }
        } else {
            peers = __match_any_sync(0xffffffffu, d);
        }
        const uint32_t base = d != NO_DIGIT ? sm.cnt[warp][d] : 0u;
        const uint32_t rk = __popc(peers & lt);
        __syncwarp();
        if (d != NO_DIGIT && rk == 0u) sm.cnt[warp][d] = base + __popc(peers);
        __syncwarp();
        pos[r] = base + rk;
    }
    __syncthreads();
    uint32_t total = 0;
    if (tid < RADIX) {
#pragma unroll
        for (int w = 0; w < NT / 32; w++) {
            const uint32_t c = sm.cnt[w][tid];
            sm.cnt[w][tid] = total;
            total += c;
        }
    }
    uint32_t all;
    const uint32_t st = block_scan<uint32_t>(tid < RADIX ? total : 0u, all);
    if (tid < RADIX) sm.start[tid] = st;
    if (tid == 0) sm.total = all;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < IPT_; r++)
        if (dig[r] != NO_DIGIT) pos[r] += sm.start[dig[r]] + sm.cnt[warp][dig[r]];
    count = total;
}

// Persistent ticket loop (one ticket at a time: prefetching the next ticket
// made the look-back chains wait on CTAs still busy with their current one).
template <typename F>
__device__ __forceinline__ void ticket_loop(uint32_t *counter, F &&body) {
    __shared__ uint32_t s_t;
    while (true) {
        if (threadIdx.x == 0) s_t = atomicAdd(counter, 1u);
        __syncthreads();
        const uint32_t t = s_t;
        if (!body(t)) break;
        __syncthreads();
    }
}

__device__ __forceinline__ uint32_t take_ticket(uint32_t *counter) {
    __shared__ uint32_t s_t;
    if (threadIdx.x == 0) s_t = atomicAdd(counter, 1u);
    __syncthreads();
    return s_t;
}

}  // namespace sweep
}  // namespace seele
