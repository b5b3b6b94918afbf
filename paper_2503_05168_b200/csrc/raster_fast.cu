// FAST tile rasterizer (default precision) on sm_100a.
//
// One CTA of 64 threads per 16x16 tile; each thread owns a 2x2 pixel quad, so
// the per-splat work that does not depend on the pixel (shared-memory loads,
// votes, loop control, a' dx, c' dy^2) is paid once per four pixels.  Each of
// the reference's model-warps (rasterize.py:200, 267-271, 291-298) is exactly
// 8 consecutive threads, i.e. one byte of a warp ballot:
//   ref / cr w=1 / cr w=2 : model-warp k = quad row k (pixel rows 2k, 2k+1)
//   cr w=4                : model-warp k = 4x2 quads (groups 2k, 2k+1)
// so the lockstep counters are per-byte "any" tests of the real ballots.
// A hardware warp covers a 16x8 pixel region (tile rows 0-7 / 8-15).
//
// Contribution-aware engine (rasterize.py:249-322): for w = 2 the group IS
// the thread's quad, so the leader verdict is the sign of the quad's first
// pixel's d; for w = 4 the group is 4 threads and the leader thread's verdict
// is broadcast by ballot.  The members' alphas are evaluated together with
// the leader's (packed fp32x2) and masked by the verdict: a warp-step in
// which no leader of the warp passes is rare once the warp-region cull below
// has run (5 % of C3's relevant warp-steps, SEELE_RASTER_PROFILE), so a
// leader-first branch would not pay for itself.
//
// Work skipping (exact): each lane tests one staged splat -- the minimum of
// q' over the warp's 16x8 pixel-centre rectangle (closed form in Cholesky
// coordinates, rect_reaches) against the top of its alpha bracket with the
// evaluation margins.  A warp whose region it misses cannot blend or pass a
// leader test with that splat, so it skips it; the reference still charges one lockstep step to
// every live model-warp (alpha_eval for ref, leader_eval for cr), which the
// warp adds per skipped splat from its (unchanged) live mask.
//
// Exactness (same discrete result as the fp64 reference), everything in fp32:
//  * alpha test: q' = log2(e) q / 2 evaluated in fp32 (Cholesky form, folded
//    mean) has |q'32 - q'| <= e0q + e1q q' (derivation at
//    write_raster_record), giving the bracket [q_lo, q_up): q'32 < q_lo
//    passes, q'32 >= q_up fails, in between the pixel is re-decided with the
//    reference's fp64 formula (alpha64).  The decisions are sign bits of
//    q'32 - q_lo and q'32 - q_up (exact for float subtraction).
//  * transmittance: alpha32 = min(o 2^-q'32, 0.99) has relative error
//    <= e0 + e1 q'; 1 - alpha32 is exact for alpha >= 0.5 and within 2^-25
//    otherwise.  Each pixel carries T in fp32 and a bound D >= |T32 - T|,
//    D' = D (1 - alpha) + T alpha (e0 + e1 q') + 1e-7 T, products rounded
//    upward (the 1e-7 T term on every live step, blending or not).  A clear
//    sign of T32 - (D + gamma) (rounded up) proves T >= gamma; otherwise
//    T + D < gamma proves the pixel done, and in between
//    its transmittance is recomputed exactly in fp64 over the tile list so
//    far (exact_transmittance, warp-cooperative) and the decision is the
//    reference's.
//
// Data flow per warp: batches of 32 records (64 B each) are staged in shared
// memory by cp.async one batch ahead; a batch's relevance to the warp's
// region is one ballot; the blend of a step is branch-free packed math with
// 0 / 1 factors (sign-bit masks & liveness & the group leader's verdict).
#include "raster_common.cuh"

namespace seele {

using namespace rast;

namespace {

constexpr int kBatch = 32;  // splats staged per warp batch
constexpr double kQ = 0.72134752044448170368;  // log2(e) / 2: q' = kQ q

using Staged = RasterRec;

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ uint32_t fbits(float x) { return __float_as_uint(x); }
// c += (ballot & mask) != 0, as one predicated add
__device__ __forceinline__ void count_any(uint32_t &c, unsigned ballot, unsigned mask) {
    asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\tand.b32 t, %1, %2;\n\tsetp.ne.u32 p, t, 0;\n\t@p add.u32 %0, %0, 1;\n\t}"
        : "+r"(c)
        : "r"(ballot), "r"(mask));
}
// sqrt within a few ulp (MUFU), for bounds that are widened anyway
__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// The two pixels of a quad row are one float2 (.x = left, .y = right) so the
// per-pixel math runs as packed fp32x2 instructions (FFMA2 / FMUL2 / FADD2,
// per-element rounding: bit-identical to scalar fmaf).
__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
__device__ __forceinline__ float lane_of(const float2 &v, int c) { return c ? v.y : v.x; }

// q' of the four quad pixels (fp32 Cholesky form, error model at
// preprocess.cu write_raster_record), pixel centres and mean in absolute
// pixel coordinates: q[r] = (q of (x0, y0 + r), q of (x0 + 1, y0 + r)).
__device__ __forceinline__ void quad_q(const Staged &sg, float2 lxp, float2 lyp, float2 q[2]) {
    const float2 dx = __fadd2_rn(lxp, f2(-sg.mxh));
    const float2 dy = __fadd2_rn(lyp, f2(-sg.myh));
    const float2 t = __ffma2_rn(f2(sg.l21), dy, f2(-sg.cu));  // (the mean's lo parts, write_raster_record)
    const float2 w = __ffma2_rn(f2(sg.l22), dy, f2(-sg.cw));
    const float2 ww = __fmul2_rn(w, w);
    const float2 u0 = __ffma2_rn(f2(sg.l11), dx, f2(t.x)), u1 = __ffma2_rn(f2(sg.l11), dx, f2(t.y));
    q[0] = __ffma2_rn(u0, u0, f2(ww.x));
    q[1] = __ffma2_rn(u1, u1, f2(ww.y));
}

// Conservative test whether some point of the pixel-centre rectangle
// [x0, x1] x [y0, y1] (tile-relative) can have q' <= qmax: the minimum of q'
// over the rectangle is 0 if the mean lies inside, else it lies on an edge,
// where it is a 1D quadratic minimised in closed form (Cholesky coordinates).
// The minimiser may be computed approximately (fast division): q' is evaluated
// exactly at the point taken, and at an interior minimum an error e in its
// position changes q' only by O(e^2), far inside the margin.
__device__ __forceinline__ bool rect_reaches(float mx, float my, float l11, float l21, float l22, float qmax, float x0,
                                             float x1, float y0, float y1) {
    if (mx >= x0 && mx <= x1 && my >= y0 && my <= y1) return true;
    const float cyy = fmaf(l21, l21, l22 * l22);  // q' = (l11 dx + l21 dy)^2 + l22^2 dy^2
    float qmin = INFINITY;
#pragma unroll
    for (int e = 0; e < 2; e++) {  // horizontal edges y = y0, y1: minimiser dx = -l21 dy / l11
        const float dy = (e ? y1 : y0) - my;
        const float dx = fminf(fmaxf(__fdividef(-l21 * dy, l11), x0 - mx), x1 - mx);
        const float u1 = fmaf(l11, dx, l21 * dy), u2 = l22 * dy;
        qmin = fminf(qmin, fmaf(u1, u1, u2 * u2));
    }
#pragma unroll
    for (int e = 0; e < 2; e++) {  // vertical edges x = x0, x1: minimiser dy = -l11 l21 dx / (l21^2 + l22^2)
        const float dx = (e ? x1 : x0) - mx;
        const float dy = fminf(fmaxf(__fdividef(-l11 * l21 * dx, cyy), y0 - my), y1 - my);
        const float u1 = fmaf(l11, dx, l21 * dy), u2 = l22 * dy;
        qmin = fminf(qmin, fmaf(u1, u1, u2 * u2));
    }
    return qmin <= qmax;
}

// Exact fp64 transmittance of pixel (px, py) after the tile's splats k0..k1
// (reference semantics, rasterize.py:146-177), for a pixel live throughout:
// it blends splat k iff alpha_k >= theta and, for CR, its group leader's
// alpha_k >= theta (a live pixel keeps its group live).  alpha >= theta is
// decided from fp64 q against the fp32 bracket (valid a fortiori), with the
// reference formula inside it.
// (NeedAlpha = false: only the verdict, e.g. of a CR group leader; alpha is not computed when the bracket decides)
template <bool NeedAlpha>
__device__ __forceinline__ bool exact_test(double px, double py, const double2 &m, const double4 &co, float q_lo,
                                           float w_up, double th, double &a) {
    const double dx = px - m.x, dy = py - m.y;
    const double q = fma(co.x * dx, dx, fma(2.0 * co.y * dx, dy, (co.z * dy) * dy));
    const double qp = kQ * q;
    if (qp > (double)q_lo + (double)w_up) return false;  // (an empty bracket: q_lo = -inf, w_up = 0)
    if (qp < (double)q_lo) {
        if (NeedAlpha) a = fmin(co.w * exp(-0.5 * q), kAlphaClamp);
        return true;
    }
    a = alpha64(px, py, m.x, m.y, co.x, co.y, co.z, co.w);
    return a >= th;
}

// Warp-cooperative: all 32 lanes take every 32nd splat of k0..k1, the fp64
// factors are multiplied in a shuffle tree (a different association than the
// reference's running product: relative difference ~1e-15, far inside any
// decision margin that reaches this path).
template <int W>
__device__ __forceinline__ double exact_transmittance(const Workspace &ws, const uint32_t *__restrict__ pair_pos,
                                                   uint32_t k0, uint32_t k1, int px, int py, int lx, int ly,
                                                   double th) {
    const int lane = threadIdx.x & 31;
    double T = 1.0;
    // kWalkU splats per lane and round, their loads issued before any is used: a long walk (C4: ~1-2K
    // splats per event) pays the dependent-load latency (position, then record) once per round
#ifndef SEELE_WALK_U
#define SEELE_WALK_U 1
#endif
    constexpr int kU = SEELE_WALK_U;
    uint32_t k = k0 + lane;
    for (; k + 32 * (kU - 1) <= k1; k += 32 * kU) {
        uint32_t p[kU];
#pragma unroll
        for (int u = 0; u < kU; u++) p[u] = pair_pos[k + 32 * u];
        double2 m[kU];
        double4 co[kU];
        float2 f[kU];
#pragma unroll
        for (int u = 0; u < kU; u++) {
            m[u] = ws.xrec[p[u]].m;
            co[u] = ws.xrec[p[u]].co;
            f[u] = *reinterpret_cast<const float2 *>(&ws.xrec[p[u]].q_lo);  // (q_lo, w_up)
        }
#pragma unroll
        for (int u = 0; u < kU; u++) {
            double a;
            if (W >= 2 && !exact_test<false>(lx + 0.5, ly + 0.5, m[u], co[u], f[u].x, f[u].y, th, a)) continue;
            if (!exact_test<true>(px + 0.5, py + 0.5, m[u], co[u], f[u].x, f[u].y, th, a)) continue;
            T = __dmul_rn(T, __dsub_rn(1.0, a));
        }
    }
    for (; k <= k1; k += 32) {
        const uint32_t p = pair_pos[k];
        const double2 m = ws.xrec[p].m;
        const double4 co = ws.xrec[p].co;
        const float2 f = *reinterpret_cast<const float2 *>(&ws.xrec[p].q_lo);  // (q_lo, w_up)
        double a;
        if (W >= 2 && !exact_test<false>(lx + 0.5, ly + 0.5, m, co, f.x, f.y, th, a)) continue;
        if (!exact_test<true>(px + 0.5, py + 0.5, m, co, f.x, f.y, th, a)) continue;
        T = __dmul_rn(T, __dsub_rn(1.0, a));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) T = __dmul_rn(T, __shfl_xor_sync(0xffffffffu, T, o));
    return T;
}

// fp64 re-decision of the quad pixels in `need` (alpha inside its bracket): the reference's alpha and
// its verdict alpha >= theta.  Inlined (96 registers, no spills): an out-of-line call made the allocator move a
// loop counter around the call's link register every step (C3 raster 0.447 -> 0.441 ms).
struct Redecided {
    float al[4];
    bool pass[4];
};
__device__ __forceinline__ Redecided redecide(const Workspace &ws, uint32_t p, int x0, int y0, uint32_t need, double th) {
    Redecided r;
    const double2 m = ws.xrec[p].m;
    const double4 co = ws.xrec[p].co;
#pragma unroll
    for (int s = 0; s < 4; s++) {
        r.al[s] = 0.0f;
        r.pass[s] = false;
        if (!((need >> s) & 1u)) continue;
        const double a64 =
            alpha64((double)(x0 + (s & 1)) + 0.5, (double)(y0 + (s >> 1)) + 0.5, m.x, m.y, co.x, co.y, co.z, co.w);
        r.al[s] = (float)a64;
        r.pass[s] = a64 >= th;
    }
    return r;
}

// Pixel slot s of a quad array (s = 2 * row + column).
__device__ __forceinline__ float &slot(float2 (&v)[2], int s) { return (s & 1) ? v[s >> 1].y : v[s >> 1].x; }

// SEELE_RASTER_WARPS = 1: one warp (half tile) per CTA, so a warp that finishes early frees its slot
// instead of waiting for the other half of its tile; 2: one CTA of two warps per tile
#ifndef SEELE_RASTER_WARPS
#define SEELE_RASTER_WARPS 2
#endif
constexpr int kRWarps = SEELE_RASTER_WARPS;
#ifndef SEELE_RASTER_MINB
#define SEELE_RASTER_MINB (18 / kRWarps)  // (nine two-warp CTAs: ~95 registers, no spills; C3 0.524 -> 0.515 ms vs 7, 8 and 10 measured)
#endif
template <int W>
__global__ void __launch_bounds__(32 * kRWarps, SEELE_RASTER_MINB) k_raster_quad(Workspace ws, const uint32_t *__restrict__ pair_pos, CamK cam,
                                                        CfgK cfg, float *image, int32_t *contrib, int64_t *stats) {
    // per warp, double-buffered: each warp stages and walks the list on its own; batch b + 1 is in flight
    // (cp.async) while batch b is rasterized
    // records staged field-chunk major ([chunk][lane], 16 B each): a warp's cp.async writes and the cull's
    // per-lane reads are conflict-free (a 64-byte lane stride put 16 lanes on one bank group)
    __shared__ float4 s_stage[kRWarps][2][4][kBatch];
    // per pixel: tile splats it was live for (written at its death)
    __shared__ uint32_t s_di[32 * kRWarps][4];
    __shared__ float s_T[32 * kRWarps][4];  // per pixel: transmittance at its death
    // heavy tiles first (binning.cu k_bin_scan); with one warp per CTA, CTAs 2t and 2t + 1 are the halves of tile t
    const int tile = (int)ws.tile_order[kRWarps == 2 ? blockIdx.x : blockIdx.x >> 1];
    const int lid = threadIdx.x;  // thread within the CTA (shared-memory slot)
    const int wslot = lid >> 5;   // warp within the CTA (shared-memory slot)
    const int tid = kRWarps == 2 ? lid : (int)((blockIdx.x & 1u) << 5) + lid;  // thread within the tile
    const int lane = tid & 31, warp = tid >> 5;
    const int mw = tid >> 3, i = tid & 7;
    // this model-warp's byte of a warp ballot (through an opaque move: the compiler would otherwise
    // rematerialise it from %tid inside the step loop, an S2R whose latency lands on every step)
    unsigned bm;
    asm volatile("mov.b32 %0, %1;" : "=r"(bm) : "r"(0xffu << (lane & 24)));
    int bx, by;
    if (W == 4) {
        bx = 4 * (mw & 1) + (i & 3);
        by = 2 * (mw >> 1) + (i >> 2);
    } else {
        bx = i;
        by = mw;
    }
    const int ox = (tile % cam.tiles_x) * kTile, oy = (tile / cam.tiles_x) * kTile;
    const int x0 = ox + 2 * bx, y0 = oy + 2 * by;
    // Liveness as 0 / 1 float factors (1.0f = 0x3f800000): a pixel's blend factor is its pass sign mask & live
    // & its group leader's verdict, one LOP3 per pixel.  Out-of-image pixels start dead.
    float2 Lf[2];
    uint32_t *di = s_di[lid];
#pragma unroll
    for (int s = 0; s < 4; s++) {
        const bool v = x0 + (s & 1) < cam.width && y0 + (s >> 1) < cam.height;
        slot(Lf, s) = v ? 1.0f : 0.0f;
        di[s] = v ? 0xffffffffu : 0u;
    }
    int nlive = (Lf[0].x != 0.f) + (Lf[0].y != 0.f) + (Lf[1].x != 0.f) + (Lf[1].y != 0.f);
    bool qlive = nlive != 0;
    unsigned lb = __ballot_sync(0xffffffffu, qlive);
    const float lx0 = (float)x0 + 0.5f, ly0 = (float)y0 + 0.5f;  // centre of pixel 0 (exact in fp32)
    float2 lxp = make_float2(lx0, lx0 + 1.0f), lyp = make_float2(ly0, ly0 + 1.0f);
    // the pixel-centre pairs through an opaque move: the compiler otherwise rebuilds the pair registers
    // (lx0 + 1) every step for the packed subtractions
    asm volatile("mov.b64 %0, %0;" : "+l"(*reinterpret_cast<unsigned long long *>(&lxp)));
    asm volatile("mov.b64 %0, %0;" : "+l"(*reinterpret_cast<unsigned long long *>(&lyp)));
    // w = 4: the group is the 2x2 of quads whose top-left quad holds the leader pixel
    const int g_off = (i & 2);
    const int leader_lane = (lane & ~7) + g_off;
    const unsigned gmask = 0x33u << ((lane & ~7) + g_off);
    const bool leader_thread = W != 4 || (i == g_off);
    const double th64 = cfg.alpha_theta;
    float2 T[2], L[2], C[2][3], cnt[2];  // L = T32 - D: a lower bound of the exact transmittance
#pragma unroll
    for (int r = 0; r < 2; r++) {
        T[r] = f2(1.0f);
        L[r] = f2(1.0f);
        C[r][0] = C[r][1] = C[r][2] = f2(0.0f);
        cnt[r] = f2(0.0f);
    }
    // CR group leader pixel (rasterize.py:235-246): top-left pixel of the w x w group
    // (the rare paths and the epilogue take the quad origin back from the pixel centres, so the loop keeps the
    // centres, not the integer origin, in registers)
    auto qx0 = [&]() { return (int)lxp.x; };
    auto qy0 = [&]() { return (int)lyp.x; };
    const int lead_xo = W == 4 ? 4 * (bx >> 1) - 2 * bx : 0, lead_yo = W == 4 ? 4 * (by >> 1) - 2 * by : 0;
    uint32_t c_alpha = 0, c_blend = 0, n_skip = 0;
    // rare-path counters (alpha re-decisions, exact transmittance walks) in shared memory, off the registers
    __shared__ uint32_t s_rare[32 * kRWarps][2];
    s_rare[lid][0] = 0u;
    s_rare[lid][1] = 0u;
#ifdef SEELE_RASTER_PROFILE
    uint32_t pr_rel = 0, pr_nolead = 0, pr_noblend = 0, pr_amb = 0, pr_death = 0;
#endif
    const uint2 rg = ws.ranges[tile];

    const float ry0 = warp ? 8.5f : 0.5f, ry1 = ry0 + 7.0f;  // this warp's pixel-centre rows (tile-relative)
    // cp.async of one splat's record + box into buffer `buf` (idx past the list: nothing)
    auto stage = [&](uint32_t idx, uint32_t p, int buf) {
        if (idx < rg.y) {
            const float4 *src = reinterpret_cast<const float4 *>(ws.rec + p);
#pragma unroll
            for (int k = 0; k < 4; k++) cp_async16(&s_stage[wslot][buf][k][lane], src + k);
        }
        cp_async_commit();
    };
    uint32_t p_next = rg.x + lane < rg.y ? pair_pos[rg.x + lane] : 0u;
    stage(rg.x + lane, p_next, 0);
    p_next = rg.x + kBatch + lane < rg.y ? pair_pos[rg.x + kBatch + lane] : 0u;
    int buf = 0;
    for (uint32_t b0 = rg.x; b0 < rg.y && lb != 0u; b0 += kBatch, buf ^= 1) {
        __syncwarp();  // every lane is done with buffer buf ^ 1 (batch b - 1)
        stage(b0 + kBatch + lane, p_next, buf ^ 1);
        const uint32_t i2 = b0 + 2 * kBatch + lane;
        p_next = i2 < rg.y ? pair_pos[i2] : 0u;
        cp_async_wait<1>();  // this lane's part of batch b has landed
        __syncwarp();
        const float4(*s_g)[kBatch] = s_stage[wslot][buf];
        // record of staged splat i (chunks read as 16-byte vectors)
        auto staged = [&](int i) {
            Staged r;
            float4 *d = reinterpret_cast<float4 *>(&r);
#pragma unroll
            for (int k = 0; k < 4; k++) d[k] = s_g[k][i];
            return r;
        };
        bool rel = false;
        if (b0 + lane < rg.y) {  // (the box test of round 1 dropped: the exact refinement alone is cheaper)
            const Staged sv = staged(lane);
            {
                // exact refinement in tile-relative floats; the margin covers the fp32 evaluation (twice the
                // bracket width) and the float mean, |error| <= ep = 2^-23 (|d| + 32) px, times
                // |grad q'| <= 2 P sqrt(q')
                const float mx = sv.mxh - (float)ox, my = sv.myh - (float)oy;
                // (margin terms only need upper bounds: approximate square roots, widened by 1e-4)
                const float P = 1.0001f * sqrt_approx(fmaf(sv.l11, sv.l11, fmaf(sv.l21, sv.l21, sv.l22 * sv.l22)));
                // (the hi mean alone: its lo part, <= 2^-24 |m|, joins the tile-relative rounding)
                const float ep = 1.2e-7f * (fabsf(mx) + fabsf(my) + fabsf(sv.mxh) + fabsf(sv.myh) + 32.0f);
                const float qh = __fadd_ru(sv.q_lo, sv.w_up), pe = P * ep;  // top of the alpha bracket
                const float qm = qh + 2.0f * (qh - sv.q_lo) + 1e-6f * qh + 2.2f * pe * (1.0001f * sqrt_approx(fmaxf(qh, 0.f))) +
                                 1.1f * pe * pe + 1e-6f;
                // (an empty bracket, o < theta: w_up = 0, nothing can pass)
                rel = sv.w_up > 0.0f && rect_reaches(mx, my, sv.l11, sv.l21, sv.l22, qm, 0.5f, 15.5f, ry0, ry1);
            }
        }
        uint32_t mlo = __ballot_sync(0xffffffffu, rel);
        __syncwarp();
        const int nb = (int)min((uint32_t)kBatch, rg.y - b0);
        // skipped splats of the batch (charged to the live pixels via the death steps); a pixel that dies in
        // the batch takes back the skipped splats after its death
        const uint32_t skipped = ~mlo & (nb == kBatch ? ~0u : (1u << nb) - 1u);
        n_skip += (uint32_t)__popc(skipped) * (uint32_t)nlive;
        while (mlo) {
            const int j = __ffs(mlo) - 1;  // next relevant splat
            mlo &= mlo - 1u;
            const Staged sg = staged(j);
#ifdef SEELE_RASTER_PROFILE
            pr_rel++;
#endif
            const float4 rc3 = make_float4(sg.r, sg.g, sg.b, 0.0f);
            float2 q[2], al[2], d[2], E[2];
            quad_q(sg, lxp, lyp, q);
            const uint32_t wb = fbits(sg.w_up);
            bool amb = false;  // some pixel with 0 <= q' - q_lo <= w_up (bit patterns: a negative d is huge)
#pragma unroll
            for (int r = 0; r < 2; r++) {
                al[r] = __fmul2_rn(f2(sg.o), make_float2(ex2_approx(-q[r].x), ex2_approx(-q[r].y)));
                d[r] = __fadd2_rn(q[r], f2(-sg.q_lo));  // sign set <=> q' < q_lo: surely passes
                E[r] = __ffma2_rn(f2(sg.e1), q[r], f2(sg.e0));
                amb |= fbits(d[r].x) <= wb;
                amb |= fbits(d[r].y) <= wb;
            }
            // pass masks: all ones <=> q' < q_lo (surely passes), from the sign of d
            uint32_t sgn[4];
#pragma unroll
            for (int s = 0; s < 4; s++) sgn[s] = (uint32_t)((int)fbits(slot(d, s)) >> 31);
            // group leader verdicts, blend factors (pass mask & liveness (1.0f / 0) & the leader's verdict,
            // one LOP3 per pixel) and the warp's blend ballot, from the pass masks
            const bool glive = W == 4 ? (lb & gmask) != 0u : qlive;
            unsigned pb = 0u, bb;
            float2 m[2];
            auto verdicts = [&]() {
                uint32_t my = ~0u;  // all-ones if this thread's group leader passed (ref / w = 1: no leader test)
                if (W == 2 || W == 4) {
                    // the leader's alpha counts even if the leader pixel is done (rasterize.py:281)
                    pb = __ballot_sync(0xffffffffu, leader_thread && glive && sgn[0] != 0u);
                    // w = 2: the group is the thread's own quad, its leader verdict is its own pass mask
                    my = W == 2 ? (glive ? sgn[0] : 0u) : 0u - ((pb >> leader_lane) & 1u);
                }
#pragma unroll
                for (int r = 0; r < 2; r++)
                    m[r] = make_float2(__uint_as_float(sgn[2 * r] & fbits(Lf[r].x) & my),
                                       __uint_as_float(sgn[2 * r + 1] & fbits(Lf[r].y) & my));
                bb = __ballot_sync(0xffffffffu,
                                   (fbits(m[0].x) | fbits(m[0].y) | fbits(m[1].x) | fbits(m[1].y)) != 0u);
            };
            // alpha = min(o 2^-q', 0.99): the clamp can only bind for o > 0.99 (the error model covers
            // 0.99f vs 0.99 and a clamp of the exact value); such splats (warp-uniform) take the rare path
            const bool hi_o = sg.o > 0.99f;
            const bool rare = __any_sync(0xffffffffu, amb || hi_o);
            // the verdicts are formed before the rare branch resolves (its vote's latency overlaps them) and
            // formed again on the rare path
            verdicts();
#ifdef SEELE_RASTER_PROFILE
            pr_amb += __any_sync(0xffffffffu, amb);
#endif
            if (rare) {
                if (hi_o) {
#pragma unroll
                    for (int r = 0; r < 2; r++) al[r] = make_float2(fminf(al[r].x, 0.99f), fminf(al[r].y, 0.99f));
                }
                // inside the bracket: decide with the reference formula in fp64 (rare); needed for live pixels
                // and for the group leader pixel while its group is live
                uint32_t need = 0;
#pragma unroll
                for (int s = 0; s < 4; s++) {
                    const bool nd = slot(Lf, s) != 0.0f || (W >= 2 && s == 0 && leader_thread && glive);
                    if (nd && fbits(slot(d, s)) <= wb) need |= 1u << s;
                }
                if (__any_sync(0xffffffffu, need != 0u)) {
                    if (need) {
                        const Redecided rd = redecide(ws, sg.p, qx0(), qy0(), need, th64);
#pragma unroll
                        for (int s = 0; s < 4; s++) {
                            if (!((need >> s) & 1u)) continue;
                            slot(al, s) = rd.al[s];
                            sgn[s] = rd.pass[s] ? ~0u : 0u;
                            slot(E, s) = 6.2e-8f;  // rounding of a64 to float
                        }
                        s_rare[lid][0] += __popc(need);
                    }
                    verdicts();
                }
            }
            if (W == 2 || W == 4) count_any(c_alpha, pb, bm);
#ifdef SEELE_RASTER_PROFILE
            pr_nolead += pb == 0u;
            pr_noblend += bb == 0u;
#endif
            if (bb == 0u) continue;  // (no pixel of the warp blends: 5 % of C3's steps)
            count_any(c_blend, bb, bm);
            if (W == 1) count_any(c_alpha, bb, bm);  // each pixel is its own leader
            float2 y[2];
#pragma unroll
            for (int r = 0; r < 2; r++) {  // _blend (rasterize.py:169-177) on a pixel pair, masked by 0/1 factors
                const float2 am = __fmul2_rn(al[r], m[r]);
                const float2 t0 = T[r];
                const float2 wgt = __fmul2_rn(t0, am);  // T alpha, or 0
                C[r][0] = __ffma2_rn(wgt, f2(rc3.x), C[r][0]);
                C[r][1] = __ffma2_rn(wgt, f2(rc3.y), C[r][1]);
                C[r][2] = __ffma2_rn(wgt, f2(rc3.z), C[r][2]);
                const float2 nam = make_float2(-am.x, -am.y);  // (a negated operand, no instruction)
                const float2 omm = __fadd2_rn(f2(1.0f), nam);  // 1 - alpha, or 1
                // |omm - (1 - alpha_ref)| <= alpha (e0 + e1 q'); the new T = T - T alpha has one rounding of
                // the exact T (1 - alpha32) after the rounding of T alpha, together <= 2^-24 T: the 1e-7 T term,
                // charged on every live step (a step that does not blend only loosens D by it: two
                // instructions fewer than masking it)
                const float2 c7 = __fmul2_ru(t0, f2(1.0e-7f));
                const float2 t1 = __fadd2_rn(t0, make_float2(-wgt.x, -wgt.y));
                // the bound kept as L = T32 - D: L' = L omm - te rounded down, te = T alpha E + 1e-7 T rounded
                // up (the 2^-10 widening of e0, e1 covers the rounding of T alpha in wgt), is T32' - D' for
                // the D recurrence D' = D omm + te, so T32' - (T32' - L') bounds T from below and
                // T32' + (T32' - L') from above
                const float2 te = __ffma2_ru(wgt, E[r], c7);
                const float2 l1 = __ffma2_rd(L[r], omm, make_float2(-te.x, -te.y));
                T[r] = t1;
                L[r] = l1;
                // sign set <=> L < gamma_up (a clear sign proves T >= gamma); done pixels carry T = L = 1e30
                // (their transmittance is parked in s_T) and never test positive
                y[r] = __fadd2_rn(l1, f2(-cfg.gamma_up));
                cnt[r] = __fadd2_rn(cnt[r], m[r]);
            }
            if (__any_sync(0xffffffffu, (int)(fbits(y[0].x) | fbits(y[0].y) | fbits(y[1].x) | fbits(y[1].y)) < 0)) {
#ifdef SEELE_RASTER_PROFILE
                pr_death++;
#endif
                uint32_t ambT = 0;
#pragma unroll
                for (int s = 0; s < 4; s++) {
                    if ((int)fbits(slot(y, s)) >= 0) continue;
                    if (__fmaf_ru(slot(T, s), 2.0f, -slot(L, s)) < cfg.gamma_dn) {  // T32 + D < gamma: done
                        slot(Lf, s) = 0.0f;
                        s_T[lid][s] = slot(T, s);
                        slot(T, s) = 1e30f;
                        slot(L, s) = 1e30f;
                        di[s] = b0 + (uint32_t)j - rg.x + 1u;  // its death step: tile splats processed
                        nlive--;
                        n_skip -= (uint32_t)__popc(skipped >> j >> 1);
                    } else {
                        ambT |= 1u << s;
#ifdef SEELE_AMB_PROFILE
                        {  // (debug build: histogram of the relative bound D / T at T-ambiguous events)
                            const float rel = (slot(T, s) - slot(L, s)) / fmaxf(slot(T, s), 1e-30f);
                            const int bk = rel < 1e-5f ? 0 : rel < 1e-4f ? 1 : rel < 1e-3f ? 2 : rel < 1e-2f ? 3 : 4;
                            atomicAdd((unsigned long long *)stats + 11 + bk, 1ull);
                        }
#endif
                    }
                }
                unsigned ambw = __ballot_sync(0xffffffffu, ambT != 0u);
                while (ambw) {
                    // T < gamma undecidable in fp32: recompute that pixel's transmittance exactly (fp64,
                    // reference formula) over every splat of the tile up to this one, all 32 lanes together,
                    // then decide.  A live pixel's blends depend only on its own alphas (and its group
                    // leader's for CR).
                    const int src = __ffs(ambw) - 1;
                    const uint32_t am = __shfl_sync(0xffffffffu, ambT, src);
                    const int s = __ffs(am) - 1;
                    const int sx0 = __shfl_sync(0xffffffffu, qx0(), src), sy0 = __shfl_sync(0xffffffffu, qy0(), src);
                    const int px = sx0 + (s & 1), py = sy0 + (s >> 1);
                    const int gx = sx0 + __shfl_sync(0xffffffffu, lead_xo, src);
                    const int gy = sy0 + __shfl_sync(0xffffffffu, lead_yo, src);
                    const double Tx = exact_transmittance<W>(ws, pair_pos, rg.x, b0 + (uint32_t)j, px, py, gx, gy, th64);
                    if (lane == src) {
                        s_rare[lid][1]++;
#pragma unroll
                        for (int ss = 0; ss < 4; ss++) {
                            if (ss != s) continue;
                            slot(T, ss) = (float)Tx;
                            slot(L, ss) = __fmul_rd(slot(T, ss), 0.99999994f);  // D = 2^-24 T: the rounding of Tx
                            if (Tx < cfg.gamma) {
                                slot(Lf, ss) = 0.0f;
                                s_T[lid][ss] = slot(T, ss);
                                slot(T, ss) = 1e30f;
                                slot(L, ss) = 1e30f;
                                di[ss] = b0 + (uint32_t)j - rg.x + 1u;
                                nlive--;
                                n_skip -= (uint32_t)__popc(skipped >> j >> 1);
                            }
                        }
                        ambT &= ~(1u << s);
                    }
                    ambw = __ballot_sync(0xffffffffu, ambT != 0u);
                }
                qlive = nlive != 0;
                lb = __ballot_sync(0xffffffffu, qlive);
                if (lb == 0u) break;
            }
        }
    }
    cp_async_wait<0>();  // no copy outlives the kernel
    // pixels still live at the end took every splat of the list
    uint32_t n_live = 0, n_blend = 0, mw_steps = 0;
#pragma unroll
    for (int s = 0; s < 4; s++) {
        if (di[s] == 0xffffffffu) di[s] = rg.y > rg.x ? rg.y - rg.x : 0u;
        n_live += di[s];
        n_blend += (uint32_t)slot(cnt, s);
        mw_steps = max(mw_steps, di[s]);
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) mw_steps = max(mw_steps, __shfl_xor_sync(0xffffffffu, mw_steps, o));
    uint32_t c_leader = 0;
    if (W == 0) c_alpha = mw_steps; else c_leader = mw_steps;
    const uint32_t w_red = __reduce_add_sync(0xffffffffu, s_rare[lid][0]);
    const uint32_t w_tamb = __reduce_add_sync(0xffffffffu, s_rare[lid][1]);
    const uint32_t w_live = __reduce_add_sync(0xffffffffu, n_live);
    const uint32_t w_blend = __reduce_add_sync(0xffffffffu, n_blend);
    const uint32_t w_skip = __reduce_add_sync(0xffffffffu, n_skip);
#ifdef SEELE_RASTER_PROFILE
    if (lane == 0) {  // (profile build: warp-step phase counts replace the fast-path counters 11..15)
        unsigned long long *sp = (unsigned long long *)stats;
        atomicAdd(sp + 11, (unsigned long long)pr_rel);
        atomicAdd(sp + 12, (unsigned long long)pr_nolead);
        atomicAdd(sp + 13, (unsigned long long)pr_noblend);
        atomicAdd(sp + 14, (unsigned long long)pr_amb);
        atomicAdd(sp + 15, (unsigned long long)pr_death);
    }
    if (false) {
#elif defined(SEELE_AMB_PROFILE)
    if (false) {  // (debug build: counters 11..15 hold the D / T histogram of T-ambiguous events)
#else
    if (lane == 0) {
#endif
        unsigned long long *sp = (unsigned long long *)stats;
        if (w_red) atomicAdd(sp + SEELE_STAT_ALPHA_REDECIDE, (unsigned long long)w_red);
        if (w_tamb) atomicAdd(sp + SEELE_STAT_T_AMBIGUOUS, (unsigned long long)w_tamb);
        if (w_live) atomicAdd(sp + SEELE_STAT_LIVE_PIXEL_STEPS, (unsigned long long)w_live);
        if (w_blend) atomicAdd(sp + SEELE_STAT_PIXEL_BLENDS, (unsigned long long)w_blend);
        if (w_skip) atomicAdd(sp + SEELE_STAT_SKIPPED_PIXEL_STEPS, (unsigned long long)w_skip);
    }
#pragma unroll
    for (int s = 0; s < 4; s++) {
        const int ex0 = qx0(), ey0 = qy0();
        if (ex0 + (s & 1) >= cam.width || ey0 + (s >> 1) >= cam.height) continue;
        const long long pix = (long long)(ey0 + (s >> 1)) * cam.width + ex0 + (s & 1);
        const int r = s >> 1, c = s & 1;
        const float Ts = slot(Lf, s) != 0.0f ? slot(T, s) : s_T[lid][s];
        image[3 * pix + 0] = fmaf(Ts, (float)cfg.bg[0], lane_of(C[r][0], c));  // background (rasterize.py:228-231)
        image[3 * pix + 1] = fmaf(Ts, (float)cfg.bg[1], lane_of(C[r][1], c));
        image[3 * pix + 2] = fmaf(Ts, (float)cfg.bg[2], lane_of(C[r][2], c));
        if (contrib) contrib[pix] = (int32_t)slot(cnt, s);
    }
    // the four model-warps' counters summed in the warp: one set of atomics per warp (the stats words are
    // shared by every CTA)
    const uint32_t ca = i == 0 ? c_alpha : 0u, cb = i == 0 ? c_blend : 0u, cl = i == 0 ? c_leader : 0u;
    Counters k{__reduce_add_sync(0xffffffffu, ca), __reduce_add_sync(0xffffffffu, cb),
               __reduce_add_sync(0xffffffffu, cl)};
    if (lane == 0) add_counters<W>(stats, k);
}
}  // namespace

void launch_raster_fast(int W, const Workspace &ws, const uint32_t *pair_pos, const CamK &cam, const CfgK &cfg,
                        float *image, int32_t *contrib, int64_t *stats, cudaStream_t st) {
    const int n_cta = cam.tiles_x * cam.tiles_y * (2 / kRWarps), nt = 32 * kRWarps;
    switch (W) {
        case 0: k_raster_quad<0><<<n_cta, nt, 0, st>>>(ws, pair_pos, cam, cfg, image, contrib, stats); break;
        case 1: k_raster_quad<1><<<n_cta, nt, 0, st>>>(ws, pair_pos, cam, cfg, image, contrib, stats); break;
        case 2: k_raster_quad<2><<<n_cta, nt, 0, st>>>(ws, pair_pos, cam, cfg, image, contrib, stats); break;
        default: k_raster_quad<4><<<n_cta, nt, 0, st>>>(ws, pair_pos, cam, cfg, image, contrib, stats); break;
    }
}

}  // namespace seele
