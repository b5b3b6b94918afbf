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
// the thread's quad, so the leader test is one alpha per thread and the
// member alphas run only if some leader of the warp passed; for w = 4 the
// group is 4 threads and the leader thread's verdict is broadcast by ballot.
//
// Work skipping (exact): every staged splat carries the box of pixel centres
// that can pass its alpha test (preprocess write_raster_record).  A warp
// whose region misses the box cannot blend or pass a leader test with that
// splat, so it skips it; the reference still charges one lockstep step to
// every live model-warp (alpha_eval for ref, leader_eval for cr), which the
// warp adds per skipped splat from its (unchanged) live mask.
//
// Exactness (same discrete result as the fp64 reference), everything in fp32:
//  * alpha test: q' = log2(e) q / 2 evaluated in fp32 (Cholesky form, hi/lo
//    tile-relative mean) has |q'32 - q'| <= e0q + e1q q' (derivation at
//    write_raster_record); q'32 < q_lo' passes,
//    q'32 > q_hi' fails, in between the pixel is re-decided with the
//    reference's fp64 formula (alpha64).
//  * transmittance: alpha32 = min(o 2^-q'32, 0.99) with relative error
//    <= e0 + e1 q'; 1 - alpha for alpha > 0.5 is rebuilt as (1 - o) +
//    o (1 - 2^-q') so it keeps ~5e-7 relative accuracy.  Each pixel carries T
//    in fp32 and an absolute bound D >= |T32 - T|, D' = D (1 - alpha) +
//    T (ef + 2^-24).  T < gamma is decided in fp32 unless T lies within D of
//    gamma; then the pixel's transmittance is recomputed exactly in fp64 over
//    the tile list so far (exact_transmittance) and the decision is the
//    reference's.
#include "raster_common.cuh"

namespace seele {

using namespace rast;

namespace {

constexpr int kBatch = 32;  // splats staged per warp batch
constexpr double kQ = 0.72134752044448170368;  // log2(e) / 2: q' = kQ q

struct __align__(16) Staged {
    float mxh, mxl, myh, myl;  // tile-relative mean as hi + lo floats
    float l11, l21, l22, o;    // Cholesky factor of the conic in q' units; opacity
    float q_lo, q_hi, e0, e1;  // alpha-test bracket in q'; alpha relative error model e0 + e1 q'
    float r, g, b, om_o;       // colour; 1 - opacity
    uint32_t p, pad[3];        // assembled position (fp64 re-decisions)
};

__device__ __forceinline__ uint32_t slice_any(unsigned ballot, int shift) { return ((ballot >> shift) & 0xffu) != 0u; }

// Quad state: four pixels, slot s = (x0 + (s & 1), y0 + (s >> 1)); the two
// pixels of a quad row r = s >> 1 are one float2 (.x = left, .y = right) so
// the per-pixel math runs as packed fp32x2 instructions (FFMA2 / FMUL2 /
// FADD2, per-element round-to-nearest: bit-identical to scalar fmaf).
struct Quad {
    float2 T[2], D[2], C[2][3];
    float2 cnt[2];  // blends per pixel (exact in fp32 below 2^24)
};

__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
__device__ __forceinline__ float lane_of(const float2 &v, int c) { return c ? v.y : v.x; }

// q' of the four quad pixels (fp32 Cholesky form, error model at
// preprocess.cu write_raster_record): q[r] = (q of (x0, y0 + r), q of (x0 + 1, y0 + r)).
__device__ __forceinline__ void quad_q(const Staged &sg, float2 lxp, float2 lyp, float2 q[2]) {
    const float2 dx = __fadd2_rn(__fadd2_rn(lxp, f2(-sg.mxh)), f2(-sg.mxl));
    const float2 dy = __fadd2_rn(__fadd2_rn(lyp, f2(-sg.myh)), f2(-sg.myl));
    const float2 t = __fmul2_rn(f2(sg.l21), dy);
    const float2 w = __fmul2_rn(f2(sg.l22), dy);
    const float2 ww = __fmul2_rn(w, w);
    const float2 u0 = __ffma2_rn(f2(sg.l11), dx, f2(t.x)), u1 = __ffma2_rn(f2(sg.l11), dx, f2(t.y));
    q[0] = __ffma2_rn(u0, u0, f2(ww.x));
    q[1] = __ffma2_rn(u1, u1, f2(ww.y));
}

// Conservative test whether some point of the pixel-centre rectangle
// [x0, x1] x [y0, y1] (tile-relative) can have q' <= qmax: the minimum of q'
// over the rectangle is 0 if the mean lies inside, else it lies on an edge,
// where it is a 1D quadratic minimised in closed form (Cholesky coordinates).
__device__ __forceinline__ bool rect_reaches(float mx, float my, float l11, float l21, float l22, float qmax, float x0,
                                             float x1, float y0, float y1) {
    if (mx >= x0 && mx <= x1 && my >= y0 && my <= y1) return true;
    const float cyy = fmaf(l21, l21, l22 * l22);  // q' = (l11 dx + l21 dy)^2 + l22^2 dy^2
    float qmin = INFINITY;
#pragma unroll
    for (int e = 0; e < 2; e++) {  // horizontal edges y = y0, y1: minimiser dx = -l21 dy / l11
        const float dy = (e ? y1 : y0) - my;
        const float dx = fminf(fmaxf(-l21 * dy / l11, x0 - mx), x1 - mx);
        const float u1 = fmaf(l11, dx, l21 * dy), u2 = l22 * dy;
        qmin = fminf(qmin, fmaf(u1, u1, u2 * u2));
    }
#pragma unroll
    for (int e = 0; e < 2; e++) {  // vertical edges x = x0, x1: minimiser dy = -l11 l21 dx / (l21^2 + l22^2)
        const float dx = (e ? x1 : x0) - mx;
        const float dy = fminf(fmaxf(-l11 * l21 * dx / cyy, y0 - my), y1 - my);
        const float u1 = fmaf(l11, dx, l21 * dy), u2 = l22 * dy;
        qmin = fminf(qmin, fmaf(u1, u1, u2 * u2));
    }
    return qmin <= qmax;
}

// alpha >= theta of the quad pixels in `need` (bit s); fills al / om / ef for
// them: om = 1 - alpha, ef = bound on |om - (1 - alpha_ref)|.  Pixels inside
// the bracket are re-decided with the reference formula in fp64 (rare).
__device__ __forceinline__ uint32_t quad_alphas(const Staged &sg, const float2 q[2], int x0, int y0, uint32_t need,
                                                const Workspace &ws, double th64, float2 al[2], float2 om[2],
                                                float2 ef[2], uint32_t &n_redecide) {
    uint32_t pass = 0, amb = 0, hi = 0;
#pragma unroll
    for (int r = 0; r < 2; r++) {
        const float2 e = __fmul2_rn(f2(sg.o), make_float2(ex2_approx(-q[r].x), ex2_approx(-q[r].y)));
        al[r] = make_float2(fminf(e.x, (float)kAlphaClamp), fminf(e.y, (float)kAlphaClamp));
        om[r] = __ffma2_rn(al[r], f2(-1.0f), f2(1.0f));
        ef[r] = __ffma2_rn(al[r], __ffma2_rn(f2(sg.e1), q[r], f2(sg.e0)), f2(6.0e-8f));
#pragma unroll
        for (int c = 0; c < 2; c++) {
            const int s = 2 * r + c;
            const float qs = lane_of(q[r], c);
            hi |= (lane_of(e, c) > 0.5f ? 1u : 0u) << s;
            pass |= (qs < sg.q_lo ? 1u : 0u) << s;
            amb |= (qs >= sg.q_lo && qs <= sg.q_hi ? 1u : 0u) << s;
        }
    }
    hi &= need;
    if (__any_sync(0xffffffffu, hi != 0u)) {
        // high alpha: 1 - alpha = (1 - o) + o (1 - 2^-q') keeps ~5e-7 relative accuracy (1 - alpha32
        // would lose it by a factor alpha / (1 - alpha)); a surely clamped alpha is exactly 0.99
#pragma unroll
        for (int s = 0; s < 4; s++) {
            if (!((hi >> s) & 1u)) continue;
            const int r = s >> 1, c = s & 1;
            const float qs = lane_of(q[r], c), als = lane_of(al[r], c);
            const float e = sg.o * ex2_approx(-qs);
            float oms = lane_of(om[r], c), efs = lane_of(ef[r], c);
            if (e >= 0.99f * (1.0f + 4.0f * fmaf(sg.e1, qs, sg.e0))) {
                oms = (float)(1.0 - kAlphaClamp);
                efs = 1.0e-9f;
            } else if (als < (float)kAlphaClamp) {
                const float x = 0.69314718f * qs;  // 1 - e^-x, x < ln 2
                float em = fmaf(-x, 1.0f / 362880.0f, 1.0f / 40320.0f);
                em = fmaf(-x, em, 1.0f / 5040.0f);
                em = fmaf(-x, em, 1.0f / 720.0f);
                em = fmaf(-x, em, 1.0f / 120.0f);
                em = fmaf(-x, em, 1.0f / 24.0f);
                em = fmaf(-x, em, 1.0f / 6.0f);
                em = fmaf(-x, em, 0.5f);
                em = fmaf(-x, em, 1.0f);
                em *= x;
                oms = fmaf(sg.o, em, sg.om_o);
                efs = fmaf(6.2e-7f, oms, als * fmaf(sg.e1, qs, sg.e0));
            }
            if (c) { om[r].y = oms; ef[r].y = efs; } else { om[r].x = oms; ef[r].x = efs; }
        }
    }
    amb &= need;
    if (amb) {  // inside the bracket: decide with the reference formula in fp64
        const double2 m = ws.mean[sg.p];
        const double4 co = ws.conic_op[sg.p];
#pragma unroll
        for (int s = 0; s < 4; s++) {
            if (!((amb >> s) & 1u)) continue;
            const int r = s >> 1, c = s & 1;
            const double a64 = alpha64((double)(x0 + c) + 0.5, (double)(y0 + r) + 0.5, m.x, m.y, co.x, co.y, co.z,
                                       co.w);
            const float a32 = (float)a64, o32 = (float)(1.0 - a64);
            if (c) { al[r].y = a32; om[r].y = o32; ef[r].y = 1.0e-9f; } else { al[r].x = a32; om[r].x = o32; ef[r].x = 1.0e-9f; }
            pass |= (a64 >= th64 ? 1u : 0u) << s;
            n_redecide++;
        }
    }
    return pass & need;
}

// alpha >= theta of one pixel (the CR group leader, slot 0 of its quad),
// same arithmetic as quad_alphas.
__device__ __forceinline__ bool pixel_alpha(const Staged &sg, float q, int px, int py, const Workspace &ws,
                                            double th64, float &al, float &om, float &ef, uint32_t &n_redecide) {
    const float e = sg.o * ex2_approx(-q);
    al = fminf(e, (float)kAlphaClamp);
    om = 1.0f - al;
    ef = fmaf(al, fmaf(sg.e1, q, sg.e0), 6.0e-8f);
    bool pass = q < sg.q_lo;
    if (e > 0.5f) {
        if (e >= 0.99f * (1.0f + 4.0f * fmaf(sg.e1, q, sg.e0))) {
            om = (float)(1.0 - kAlphaClamp);
            ef = 1.0e-9f;
        } else if (al < (float)kAlphaClamp) {
            const float x = 0.69314718f * q;
            float em = fmaf(-x, 1.0f / 362880.0f, 1.0f / 40320.0f);
            em = fmaf(-x, em, 1.0f / 5040.0f);
            em = fmaf(-x, em, 1.0f / 720.0f);
            em = fmaf(-x, em, 1.0f / 120.0f);
            em = fmaf(-x, em, 1.0f / 24.0f);
            em = fmaf(-x, em, 1.0f / 6.0f);
            em = fmaf(-x, em, 0.5f);
            em = fmaf(-x, em, 1.0f);
            em *= x;
            om = fmaf(sg.o, em, sg.om_o);
            ef = fmaf(6.2e-7f, om, al * fmaf(sg.e1, q, sg.e0));
        }
    }
    if (!pass && q <= sg.q_hi) {
        const double2 m = ws.mean[sg.p];
        const double4 co = ws.conic_op[sg.p];
        const double a64 = alpha64((double)px + 0.5, (double)py + 0.5, m.x, m.y, co.x, co.y, co.z, co.w);
        al = (float)a64;
        om = (float)(1.0 - a64);
        ef = 1.0e-9f;
        pass = a64 >= th64;
        n_redecide++;
    }
    return pass;
}

// Exact fp64 transmittance of pixel (px, py) after the tile's splats k0..k1
// (reference semantics, rasterize.py:146-177), for a pixel live throughout:
// it blends splat k iff alpha_k >= theta and, for CR, its group leader's
// alpha_k >= theta (a live pixel keeps its group live).  alpha >= theta is
// decided from fp64 q against the fp32 bracket (valid a fortiori), with the
// reference formula inside it.
__device__ __forceinline__ bool exact_test(double px, double py, const double2 &m, const double4 &co, float q_lo,
                                           float q_hi, double th, double &a) {
    const double dx = px - m.x, dy = py - m.y;
    const double q = fma(co.x * dx, dx, fma(2.0 * co.y * dx, dy, (co.z * dy) * dy));
    const double qp = kQ * q;
    if (qp > (double)q_hi) return false;
    if (qp < (double)q_lo) {
        a = fmin(co.w * exp(-0.5 * q), kAlphaClamp);
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
__device__ __noinline__ double exact_transmittance(const Workspace &ws, const uint32_t *__restrict__ pair_pos,
                                                   uint32_t k0, uint32_t k1, int px, int py, int lx, int ly,
                                                   double th) {
    const int lane = threadIdx.x & 31;
    double T = 1.0;
    for (uint32_t k = k0 + lane; k <= k1; k += 32) {
        const uint32_t p = pair_pos[k];
        const double2 m = ws.mean[p];
        const double4 co = ws.conic_op[p];
        const float4 f = ws.rq[p];
        double a;
        if (W >= 2 && !exact_test(lx + 0.5, ly + 0.5, m, co, f.x, f.y, th, a)) continue;
        if (!exact_test(px + 0.5, py + 0.5, m, co, f.x, f.y, th, a)) continue;
        T = __dmul_rn(T, __dsub_rn(1.0, a));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) T = __dmul_rn(T, __shfl_xor_sync(0xffffffffu, T, o));
    return T;
}

template <int W>
__global__ void __launch_bounds__(64, 10) k_raster_quad(Workspace ws, const uint32_t *__restrict__ pair_pos, CamK cam,
                                                        CfgK cfg, float *image, int32_t *contrib, int64_t *stats) {
    __shared__ Staged s_stage[2][kBatch];  // per warp: each warp stages and walks the list on its own
    const int tile = (int)ws.tile_order[blockIdx.x];  // heavy tiles first (binning.cu k_pair_scan)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int mw = tid >> 3, i = tid & 7;
    const int shift = lane & 24;  // byte of this model-warp in a warp ballot
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
    uint32_t valid = 0;
#pragma unroll
    for (int s = 0; s < 4; s++)
        if (x0 + (s & 1) < cam.width && y0 + (s >> 1) < cam.height) valid |= 1u << s;
    uint32_t live = valid;  // bit s: pixel s not done (out-of-image pixels start done)
    const float lx0 = 2 * bx + 0.5f, ly0 = 2 * by + 0.5f;  // tile-relative centre of pixel 0
    const float2 lxp = make_float2(lx0, lx0 + 1.0f), lyp = make_float2(ly0, ly0 + 1.0f);
    // w = 4: the group is the 2x2 of quads whose top-left quad holds the leader pixel
    const int g_off = (i & 2);
    const int leader_lane = (lane & ~7) + g_off;
    const unsigned gmask = 0x33u << ((lane & ~7) + g_off);
    const bool leader_thread = W != 4 || (i == g_off);
    const double th64 = cfg.alpha_theta;
    const float gm = (float)cfg.gamma;
    Quad st;
#pragma unroll
    for (int r = 0; r < 2; r++) {
        st.T[r] = f2(1.0f);
        st.D[r] = f2(0.0f);
        st.C[r][0] = st.C[r][1] = st.C[r][2] = f2(0.0f);
    }
    st.cnt[0] = st.cnt[1] = f2(0.0f);
    // CR group leader pixel (rasterize.py:235-246): top-left pixel of the w x w group
    const int lead_x = W == 4 ? ox + 4 * (bx >> 1) : x0, lead_y = W == 4 ? oy + 4 * (by >> 1) : y0;
    // Per pixel: number of tile splats it was live for (its death step); out-of-image pixels 0.
    // The reference charges a model-warp's alpha_eval (ref) / leader_eval (cr) once per splat while
    // any of its pixels is live, i.e. the max death step over its pixels.
    __shared__ uint32_t s_di[64][4];  // per pixel: tile splats it was live for (written at its death)
    uint32_t *di = s_di[tid];
#pragma unroll
    for (int s = 0; s < 4; s++) di[s] = ((valid >> s) & 1u) ? 0xffffffffu : 0u;
    uint32_t c_alpha = 0, c_blend = 0, n_redecide = 0, n_tamb = 0, n_skip = 0;
#ifdef SEELE_RASTER_PROFILE
    uint32_t pr_steps = 0, pr_member = 0, pr_blend = 0, pr_near = 0, pr_hi = 0;
#endif
    const uint2 rg = ws.ranges[tile];

    Staged *s_g = s_stage[warp];
    const float ry0 = warp ? 8.5f : 0.5f, ry1 = ry0 + 7.0f;  // this warp's pixel-centre rows (tile-relative)
    for (uint32_t b0 = rg.x; b0 < rg.y; b0 += kBatch) {
        if (!__any_sync(0xffffffffu, live != 0u)) break;  // this warp's pixels are all done
        const uint32_t idx = b0 + lane;
        bool rel = false;
        __syncwarp();
        if (idx < rg.y) {
            const uint32_t p = pair_pos[idx];
            const double2 m = ws.mean[p];
            const float4 rc = ws.rc[p];
            const float4 rq = ws.rq[p];
            const float4 col = ws.color[p];
            const float4 bb = ws.bbox[p];
            Staged sv;
            const double mxr = m.x - (double)ox, myr = m.y - (double)oy;
            sv.mxh = (float)mxr;
            sv.mxl = (float)(mxr - (double)sv.mxh);
            sv.myh = (float)myr;
            sv.myl = (float)(myr - (double)sv.myh);
            sv.l11 = rc.x;
            sv.l21 = rc.y;
            sv.l22 = rc.z;
            sv.o = rc.w;
            sv.q_lo = rq.x;
            sv.q_hi = rq.y;
            sv.r = col.x;
            sv.g = col.y;
            sv.b = col.z;
            sv.om_o = col.w;
            sv.e0 = rq.z;
            sv.e1 = rq.w;
            sv.p = p;
            s_g[lane] = sv;
            rel = bb.y >= ox + 0.5f && bb.x <= ox + 15.5f && bb.w >= oy + ry0 && bb.z <= oy + ry1;
            if (rel) {
                // exact refinement; the margin covers the fp32 evaluation (twice the bracket width) and the
                // plain-float mean (|error| <= 2^-24 (|d| + 23) px, times |grad q'| <= 2 P sqrt(q'))
                const float P = sqrtf(fmaf(rc.x, rc.x, fmaf(rc.y, rc.y, rc.z * rc.z)));
                const float qm = rq.y + 2.0f * (rq.y - rq.x) + 1e-6f * rq.y + 1e-5f * P * sqrtf(fmaxf(rq.y, 0.f)) +
                                 1e-6f;
                rel = rect_reaches((float)mxr, (float)myr, rc.x, rc.y, rc.z, qm, 0.5f, 15.5f, ry0, ry1);
            }
        }
        uint32_t mlo = __ballot_sync(0xffffffffu, rel);
        __syncwarp();
        const int nb = (int)min((uint32_t)kBatch, rg.y - b0);
        int jprev = -1;
        unsigned lb = __ballot_sync(0xffffffffu, live != 0u);
        while (lb != 0u) {
            int j;
            if (mlo) {
                j = __ffs(mlo) - 1;
                mlo &= mlo - 1u;
            } else {
                j = nb;  // no more relevant splats: charge the rest of the batch
            }
            const uint32_t gap = (uint32_t)(j - jprev - 1);  // skipped splats (charged via the death steps)
            if (gap) n_skip += gap * __popc(live);
            if (j >= nb) break;
            jprev = j;
            const uint32_t step = b0 + (uint32_t)j - rg.x + 1u;  // tile splats processed including this one
            const Staged &sg = s_g[j];
#ifdef SEELE_RASTER_PROFILE
            pr_steps++;
#endif
            float2 q[2], al[2], om[2], ef[2];
            quad_q(sg, lxp, lyp, q);
            uint32_t blend;
            if (W == 0 || W == 1) {
                blend = quad_alphas(sg, q, x0, y0, live, ws, th64, al, om, ef, n_redecide);
                if (W == 1) {  // every pixel is its own group and leader
                    const unsigned pb = __ballot_sync(0xffffffffu, blend != 0u);
                    c_alpha += slice_any(pb, shift);
                }
            } else {
                // One alpha evaluation of all four pixels serves both phases (the member phase runs on ~95 % of
                // steps): the leader pixel's alpha counts even if that pixel is done (rasterize.py:281), the
                // members blend if live, their group's leader passed and their own alpha passes.
                const bool glive = W == 2 ? live != 0u : (lb & gmask) != 0u;
                const uint32_t lbit = (leader_thread && glive) ? 1u : 0u;
                const uint32_t pass = quad_alphas(sg, q, x0, y0, live | lbit, ws, th64, al, om, ef, n_redecide);
                const bool lpass = (pass & lbit) != 0u;
                const unsigned pb = __ballot_sync(0xffffffffu, lpass);
                c_alpha += slice_any(pb, shift);
                const bool my_pass = (pb >> (W == 2 ? lane : leader_lane)) & 1u;
                blend = my_pass ? (pass & live) : 0u;
            }
            const unsigned bb = __ballot_sync(0xffffffffu, blend != 0u);
            if (bb == 0u) continue;
#ifdef SEELE_RASTER_PROFILE
            pr_blend++;
            pr_hi += __any_sync(0xffffffffu, (al[0].x > 0.5f) | (al[0].y > 0.5f) | (al[1].x > 0.5f) | (al[1].y > 0.5f)) ? 1 : 0;
#endif
            c_blend += slice_any(bb, shift);
            uint32_t near = 0;
            float2 m01[2];
#pragma unroll
            for (int r = 0; r < 2; r++) {  // _blend (rasterize.py:169-177) on a pixel pair, masked by 0/1 factors
                // 0/1 factors from the blend bits: (bit << 29) lands on the exponent of 1.0f (0x3f800000)
                const uint32_t bl = blend >> (2 * r);
                const float2 m = make_float2(__uint_as_float(0x3f800000u & (0u - (bl & 1u))),
                                             __uint_as_float(0x3f800000u & (0u - ((bl >> 1) & 1u))));
                const float2 nm = __ffma2_rn(m, f2(-1.0f), f2(1.0f));
                m01[r] = m;
                const float2 t0 = st.T[r];
                const float2 wgt = __fmul2_rn(t0, __fmul2_rn(al[r], m));  // T alpha, or 0
                st.C[r][0] = __ffma2_rn(wgt, f2(sg.r), st.C[r][0]);
                st.C[r][1] = __ffma2_rn(wgt, f2(sg.g), st.C[r][1]);
                st.C[r][2] = __ffma2_rn(wgt, f2(sg.b), st.C[r][2]);
                const float2 omm = __ffma2_rn(om[r], m, nm);  // 1 - alpha (exactly), or 1
                const float2 t1 = __fmul2_rn(t0, omm);
                const float2 d1 = __ffma2_rn(st.D[r], omm, __fmul2_rn(t0, __fmul2_rn(ef[r], m)));
                st.T[r] = t1;
                st.D[r] = d1;
                const float2 lo = __fadd2_rn(t1, make_float2(-d1.x, -d1.y));
                near |= ((lo.x < gm ? 1u : 0u) | (lo.y < gm ? 2u : 0u)) << (2 * r);
            }
#pragma unroll
            st.cnt[0] = __fadd2_rn(st.cnt[0], m01[0]);
            st.cnt[1] = __fadd2_rn(st.cnt[1], m01[1]);
            near &= blend;  // T may be below gamma: decide below
            if (__any_sync(0xffffffffu, near != 0u)) {
#ifdef SEELE_RASTER_PROFILE
                pr_near++;
#endif
                uint32_t amb = 0;
#pragma unroll
                for (int s = 0; s < 4; s++) {
                    if (!((near >> s) & 1u)) continue;
                    if (lane_of(st.T[s >> 1], s & 1) + lane_of(st.D[s >> 1], s & 1) < gm) {  // surely below: done
                        live &= ~(1u << s);
                        di[s] = step;
                    } else {
                        amb |= 1u << s;
                    }
                }
                unsigned ambw = __ballot_sync(0xffffffffu, amb != 0u);
                while (ambw) {
                    // T < gamma undecidable in fp32: recompute that pixel's transmittance exactly (fp64,
                    // reference formula) over every splat of the tile up to this one, all 32 lanes together,
                    // then decide.  A live pixel's blends depend only on its own alphas (and its group
                    // leader's for CR).
                    const int src = __ffs(ambw) - 1;
                    const uint32_t am = __shfl_sync(0xffffffffu, amb, src);
                    const int s = __ffs(am) - 1;
                    const int px = __shfl_sync(0xffffffffu, x0, src) + (s & 1);
                    const int py = __shfl_sync(0xffffffffu, y0, src) + (s >> 1);
                    const int gx = __shfl_sync(0xffffffffu, lead_x, src), gy = __shfl_sync(0xffffffffu, lead_y, src);
                    const double T = exact_transmittance<W>(ws, pair_pos, rg.x, b0 + (uint32_t)j, px, py, gx, gy, th64);
                    if (lane == src) {
                        n_tamb++;
#pragma unroll
                        for (int ss = 0; ss < 4; ss++) {
                            if (ss != s) continue;
                            if (ss & 1) {
                                st.T[ss >> 1].y = (float)T;
                                st.D[ss >> 1].y = 6.0e-8f * (float)T;
                            } else {
                                st.T[ss >> 1].x = (float)T;
                                st.D[ss >> 1].x = 6.0e-8f * (float)T;
                            }
                            if (T < cfg.gamma) {
                                live &= ~(1u << ss);
                                di[ss] = step;
                            }
                        }
                        amb &= ~(1u << s);
                    }
                    ambw = __ballot_sync(0xffffffffu, amb != 0u);
                }
            }
            lb = __ballot_sync(0xffffffffu, live != 0u);
        }
    }
    // pixels still live at the end took every splat of the list
    uint32_t n_live = 0, n_blend = 0, mw_steps = 0;
#pragma unroll
    for (int s = 0; s < 4; s++) {
        if (di[s] == 0xffffffffu) di[s] = rg.y > rg.x ? rg.y - rg.x : 0u;
        n_live += di[s];
        n_blend += (uint32_t)lane_of(st.cnt[s >> 1], s & 1);
        mw_steps = max(mw_steps, di[s]);
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) mw_steps = max(mw_steps, __shfl_xor_sync(0xffffffffu, mw_steps, o));
    uint32_t c_leader = 0;
    if (W == 0) c_alpha = mw_steps; else c_leader = mw_steps;
    const uint32_t w_red = __reduce_add_sync(0xffffffffu, n_redecide);
    const uint32_t w_tamb = __reduce_add_sync(0xffffffffu, n_tamb);
    const uint32_t w_live = __reduce_add_sync(0xffffffffu, n_live);
    const uint32_t w_blend = __reduce_add_sync(0xffffffffu, n_blend);
    const uint32_t w_skip = __reduce_add_sync(0xffffffffu, n_skip);
#ifdef SEELE_RASTER_PROFILE
    if (lane == 0) {  // debug build: warp-step counters in stats slots 11..15
        unsigned long long *sp = (unsigned long long *)stats;
        atomicAdd(sp + 11, (unsigned long long)pr_steps);
        atomicAdd(sp + 12, (unsigned long long)pr_member);
        atomicAdd(sp + 13, (unsigned long long)pr_blend);
        atomicAdd(sp + 14, (unsigned long long)pr_near);
        atomicAdd(sp + 15, (unsigned long long)pr_hi);
    }
    return;
#endif
    if (lane == 0) {
        unsigned long long *sp = (unsigned long long *)stats;
        if (w_red) atomicAdd(sp + SEELE_STAT_ALPHA_REDECIDE, (unsigned long long)w_red);
        if (w_tamb) atomicAdd(sp + SEELE_STAT_T_AMBIGUOUS, (unsigned long long)w_tamb);
        if (w_live) atomicAdd(sp + SEELE_STAT_LIVE_PIXEL_STEPS, (unsigned long long)w_live);
        if (w_blend) atomicAdd(sp + SEELE_STAT_PIXEL_BLENDS, (unsigned long long)w_blend);
        if (w_skip) atomicAdd(sp + SEELE_STAT_SKIPPED_PIXEL_STEPS, (unsigned long long)w_skip);
    }
#pragma unroll
    for (int s = 0; s < 4; s++) {
        if (!((valid >> s) & 1u)) continue;
        const long long pix = (long long)(y0 + (s >> 1)) * cam.width + x0 + (s & 1);
        const int r = s >> 1, c = s & 1;
        const float T = lane_of(st.T[r], c);
        image[3 * pix + 0] = fmaf(T, (float)cfg.bg[0], lane_of(st.C[r][0], c));  // background (rasterize.py:228-231)
        image[3 * pix + 1] = fmaf(T, (float)cfg.bg[1], lane_of(st.C[r][1], c));
        image[3 * pix + 2] = fmaf(T, (float)cfg.bg[2], lane_of(st.C[r][2], c));
        if (contrib) contrib[pix] = (int32_t)lane_of(st.cnt[r], c);
    }
    if (i == 0) {
        Counters k{c_alpha, c_blend, c_leader};
        add_counters<W>(stats, k);
    }
}

}  // namespace

void launch_raster_fast(int W, const Workspace &ws, const uint32_t *pair_pos, const CamK &cam, const CfgK &cfg,
                        float *image, int32_t *contrib, int64_t *stats, cudaStream_t st) {
    const int n_tiles = cam.tiles_x * cam.tiles_y;
    switch (W) {
        case 0: k_raster_quad<0><<<n_tiles, 64, 0, st>>>(ws, pair_pos, cam, cfg, image, contrib, stats); break;
        case 1: k_raster_quad<1><<<n_tiles, 64, 0, st>>>(ws, pair_pos, cam, cfg, image, contrib, stats); break;
        case 2: k_raster_quad<2><<<n_tiles, 64, 0, st>>>(ws, pair_pos, cam, cfg, image, contrib, stats); break;
        default: k_raster_quad<4><<<n_tiles, 64, 0, st>>>(ws, pair_pos, cam, cfg, image, contrib, stats); break;
    }
}

}  // namespace seele
