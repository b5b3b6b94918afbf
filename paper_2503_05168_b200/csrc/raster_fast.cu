// FAST tile rasterizer (default precision) on sm_100a.
//
// One CTA of 64 threads per 16x16 tile; each thread owns a 2x2 pixel quad, so
// the per-splat work that does not depend on the pixel (shared-memory loads,
// votes, loop control, the fp64 products a dx, 2b dx, c dy^2) is paid once
// per four pixels, and the four pixels' math is branch-free so the scheduler
// can interleave their dependency chains.  Each of the reference's
// model-warps (rasterize.py:200, 267-271, 291-298) is exactly 8 consecutive
// threads, i.e. one byte of a warp ballot:
//   ref / cr w=1 / cr w=2 : model-warp k = quad row k (pixel rows 2k, 2k+1)
//   cr w=4                : model-warp k = 4x2 quads (groups 2k, 2k+1)
// so the lockstep counters are per-byte "any" tests of the real ballots.
//
// Contribution-aware engine (rasterize.py:249-322): for w = 2 the group IS the
// thread's quad, so the leader test is one alpha per thread and the member
// phase runs only if some leader of the warp passed -- when none does the
// three member alphas are skipped (the reduced-cost path).  For w = 4 the
// group is 4 threads; the leader thread's verdict is broadcast via the ballot.
//
// Exactness (same discrete result as the fp64 reference):
//  * alpha test: q = a dx^2 + 2b dx dy + c dy^2 in fp64 from tile-relative
//    means (error vs numpy <= 1e-15 kappa q), rounded once to fp32; preprocess
//    widened q_th = 2 ln(o / theta) by both errors into [q_lo, q_hi].  q32 <
//    q_lo blends, q32 > q_hi skips, in between the pixel is re-decided with the
//    reference's own fp64 formula (alpha64).
//  * transmittance: alpha32 = min(o32 ex2.approx(-q32 log2(e)/2), 0.99) has
//    |alpha32 - alpha| <= alpha (3.8e-7 + 6e-8 q); for alpha > 0.5 the factor
//    1 - alpha is rebuilt as (1 - o) + o (1 - e^{-q/2}) (polynomial, ~5e-7
//    relative) instead of losing a factor alpha / (1 - alpha).  Each pixel
//    carries T as the fp64 product of its factors (no rounding drift) and an
//    absolute bound D >= |T64 - T|:  D' = D (1 - alpha) + T ef, ef = the bound
//    on |(1 - alpha32) - (1 - alpha)|.  T < gamma
//    is decided in fp32 unless T lies within D of gamma; then that pixel's
//    transmittance is recomputed exactly in fp64 over the tile list so far
//    (exact_transmittance) and the decision is the reference's.
#include "raster_common.cuh"

namespace seele {

using namespace rast;

namespace {

constexpr float kNegHalfLog2e = -0.72134752044448170f;
constexpr int kBatch = 64;

struct __align__(16) Staged {
    double mx, my;    // mean relative to the tile origin (fp64)
    double a, b2, c;  // conic (a, 2b, c)
    float q_lo, q_hi, o;
    uint32_t p;       // assembled position (for the fp64 re-decision)
    float r, g, b, om_o;  // colour; 1 - opacity (rounded once from fp64)
};

__device__ __forceinline__ uint32_t slice_any(unsigned ballot, int shift) { return ((ballot >> shift) & 0xffu) != 0u; }

// Quad state: four pixels, slot s = (x0 + (s & 1), y0 + (s >> 1)).
struct Quad {
    double T64[4];  // transmittance, exact product of the fp32-accurate factors
    float T[4], D[4], C[4][3];
    int cnt[4];
};

// fp32 alphas of the quad pixels selected by `need` from their fp64 q; sets
// bit s of the returned mask when alpha_s >= theta.  Also returns, per pixel,
// the transmittance factor om = 1 - alpha and ef, the bound on the relative
// error of om times om (so a blend adds T * ef to the absolute bound on T).
// Pixels inside the bracket are re-decided with the reference formula (rare).
__device__ __forceinline__ uint32_t quad_alphas(const Staged &sg, double lx0, double ly0, int x0, int y0,
                                                uint32_t need, const Workspace &ws, double th64, float al[4],
                                                double om[4], float ef[4], uint32_t &n_redecide) {
    const double dx0 = lx0 - sg.mx, dx1 = (lx0 + 1.0) - sg.mx;
    const double dy0 = ly0 - sg.my, dy1 = (ly0 + 1.0) - sg.my;
    const double ax0 = sg.a * dx0, ax1 = sg.a * dx1, bx0 = sg.b2 * dx0, bx1 = sg.b2 * dx1;
    const double cy0 = (sg.c * dy0) * dy0, cy1 = (sg.c * dy1) * dy1;
    const double q[4] = {fma(ax0, dx0, fma(bx0, dy0, cy0)), fma(ax1, dx1, fma(bx1, dy0, cy0)),
                         fma(ax0, dx0, fma(bx0, dy1, cy1)), fma(ax1, dx1, fma(bx1, dy1, cy1))};
    uint32_t pass = 0, amb = 0, hi = 0;
    float q32[4];
#pragma unroll
    for (int s = 0; s < 4; s++) {
        q32[s] = (float)q[s];
        const float e = sg.o * ex2_approx(kNegHalfLog2e * q32[s]);
        al[s] = fminf(e, (float)kAlphaClamp);
        om[s] = 1.0 - (double)al[s];  // exact
        // |alpha32 - alpha| <= alpha (3.8e-7 + 6e-8 q): ex2.approx, exponent and opacity roundings
        ef[s] = al[s] * fmaf(6.0e-8f, q32[s], 3.8e-7f);
        hi |= (e > 0.5f ? 1u : 0u) << s;
        pass |= (q32[s] < sg.q_lo ? 1u : 0u) << s;
        amb |= (q32[s] >= sg.q_lo && q32[s] <= sg.q_hi ? 1u : 0u) << s;
    }
    hi &= need;
    if (__any_sync(0xffffffffu, hi != 0u)) {
        // high alpha: 1 - alpha = (1 - o) + o (1 - e^{-q/2}) keeps ~5e-7 relative accuracy
        // (1 - alpha32 would lose it by a factor alpha / (1 - alpha)); clamped alpha is exactly 0.99
#pragma unroll
        for (int s = 0; s < 4; s++) {
            if (!((hi >> s) & 1u)) continue;
            if (al[s] >= (float)kAlphaClamp && sg.o * ex2_approx(kNegHalfLog2e * q32[s]) >= 0.99000105f) {
                om[s] = 1.0 - (double)kAlphaClamp;
                ef[s] = 0.0f;
            } else if (al[s] < (float)kAlphaClamp) {
                const float x = 0.5f * q32[s];
                float em = fmaf(-x, 1.0f / 362880.0f, 1.0f / 40320.0f);
                em = fmaf(-x, em, 1.0f / 5040.0f);
                em = fmaf(-x, em, 1.0f / 720.0f);
                em = fmaf(-x, em, 1.0f / 120.0f);
                em = fmaf(-x, em, 1.0f / 24.0f);
                em = fmaf(-x, em, 1.0f / 6.0f);
                em = fmaf(-x, em, 0.5f);
                em = fmaf(-x, em, 1.0f);
                em *= x;  // 1 - e^{-x}, x < ln 2
                const float omf = fmaf(sg.o, em, sg.om_o);
                om[s] = (double)omf;
                ef[s] = 6.2e-7f * omf;
            }
        }
    }
    amb &= need;
    if (amb) {  // inside the bracket: decide with the reference formula in fp64
        const double2 m = ws.mean[sg.p];
        const double4 co = ws.conic_op[sg.p];
#pragma unroll
        for (int s = 0; s < 4; s++) {
            if (!((amb >> s) & 1u)) continue;
            const double a64 = alpha64((double)(x0 + (s & 1)) + 0.5, (double)(y0 + (s >> 1)) + 0.5, m.x, m.y, co.x,
                                       co.y, co.z, co.w);
            al[s] = (float)a64;
            om[s] = 1.0 - a64;
            ef[s] = 0.0f;
            pass |= (a64 >= th64 ? 1u : 0u) << s;
            n_redecide++;
        }
    }
    return pass & need;
}

// Exact fp64 transmittance of pixel (px, py) after the tile's splats k0..k1
// (reference semantics, rasterize.py:146-177), for a pixel live throughout:
// it blends splat k iff alpha_k >= theta and, for CR, its group leader's
// alpha_k >= theta (a live pixel keeps its group live).
// alpha >= theta decided like the fast path (fp64 q against the certified
// bracket, reference formula inside it); returns alpha64 when it passes.
__device__ __forceinline__ bool exact_test(double px, double py, const double2 &m, const double4 &co, float q_lo,
                                           float q_hi, double th, double &a) {
    const double dx = px - m.x, dy = py - m.y;
    const double q = fma(co.x * dx, dx, fma(2.0 * co.y * dx, dy, (co.z * dy) * dy));
    const float q32 = (float)q;
    if (q32 > q_hi) return false;
    if (q32 < q_lo) {
        a = fmin(co.w * exp(-0.5 * q), kAlphaClamp);
        return true;
    }
    a = alpha64(px, py, m.x, m.y, co.x, co.y, co.z, co.w);
    return a >= th;
}

template <int W>
__device__ __forceinline__ double exact_transmittance(const Workspace &ws, const uint32_t *__restrict__ pair_pos,
                                                   uint32_t k0, uint32_t k1, int px, int py, int lx, int ly,
                                                   double th) {
    constexpr int U = 2;  // independent record loads in flight
    double T = 1.0;
    for (uint32_t k = k0; k <= k1; k += U) {
        double2 m[U];
        double4 co[U];
        float4 f[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            if (k + u > k1) break;
            const uint32_t p = pair_pos[k + u];
            m[u] = ws.mean[p];
            co[u] = ws.conic_op[p];
            f[u] = ws.fast[p];
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            if (k + u > k1) break;
            double a;
            if (W >= 2 && !exact_test(lx + 0.5, ly + 0.5, m[u], co[u], f[u].x, f[u].y, th, a)) continue;
            if (!exact_test(px + 0.5, py + 0.5, m[u], co[u], f[u].x, f[u].y, th, a)) continue;
            T = __dmul_rn(T, __dsub_rn(1.0, a));
        }
    }
    return T;
}

template <int W>
__global__ void __launch_bounds__(64, 8) k_raster_quad(Workspace ws, const uint32_t *__restrict__ pair_pos, CamK cam,
                                                       CfgK cfg, float *image, int32_t *contrib, int64_t *stats) {
    __shared__ Staged s_g[kBatch];
    const int tile = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31;
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
    const double lx0 = 2 * bx + 0.5, ly0 = 2 * by + 0.5;  // tile-relative centre of pixel 0
    // w = 4: the group is the 2x2 of quads whose top-left quad holds the leader pixel
    const int g_off = (i & 2);
    const int leader_lane = (lane & ~7) + g_off;
    const unsigned gmask = 0x33u << ((lane & ~7) + g_off);
    const bool leader_thread = W != 4 || (i == g_off);
    const double th64 = cfg.alpha_theta;
    const float gm_lo = (float)cfg.gamma * (1.0f - 2.0e-7f), gm_hi = (float)cfg.gamma * (1.0f + 2.0e-7f);
    Quad st;
#pragma unroll
    for (int s = 0; s < 4; s++) {
        st.T64[s] = 1.0;
        st.T[s] = 1.0f;
        st.D[s] = 0.0f;
        st.C[s][0] = st.C[s][1] = st.C[s][2] = 0.0f;
        st.cnt[s] = 0;
    }
    // CR group leader pixel (rasterize.py:235-246): top-left pixel of the w x w group
    const int lead_x = W == 4 ? ox + 4 * (bx >> 1) : x0, lead_y = W == 4 ? oy + 4 * (by >> 1) : y0;
    uint32_t c_alpha = 0, c_blend = 0, c_leader = 0, n_redecide = 0, n_tamb = 0;
    uint32_t n_live = 0, n_blend = 0;  // pixel-level work (roofline model in bench.py)
    const uint2 rg = ws.ranges[tile];

    for (uint32_t b0 = rg.x; b0 < rg.y; b0 += kBatch) {
        if (__syncthreads_count(live != 0u) == 0) break;  // tile stops when every pixel is done
        const uint32_t idx = b0 + tid;
        if (idx < rg.y) {
            const uint32_t p = pair_pos[idx];
            const double2 m = ws.mean[p];
            const double4 co = ws.conic_op[p];
            const float4 f = ws.fast[p];
            const float4 col = ws.color[p];
            Staged sv;
            sv.mx = m.x - (double)ox;
            sv.my = m.y - (double)oy;
            sv.a = co.x;
            sv.b2 = 2.0 * co.y;
            sv.c = co.z;
            sv.q_lo = f.x;
            sv.q_hi = f.y;
            sv.o = f.z;
            sv.p = p;
            sv.r = col.x;
            sv.g = col.y;
            sv.b = col.z;
            sv.om_o = f.w;
            s_g[tid] = sv;
        }
        __syncthreads();
        const int nb = (int)min((uint32_t)kBatch, rg.y - b0);
        for (int j = 0; j < nb; j++) {
            const unsigned lb = __ballot_sync(0xffffffffu, live != 0u);
            if (lb == 0u) break;  // all four model-warps of this warp are done
            const Staged &sg = s_g[j];
            const uint32_t mw_live = slice_any(lb, shift);
            n_live += __popc(live);
            float al[4], ef[4];
            double om[4];
            uint32_t blend;
            if (W == 0 || W == 1) {
                blend = quad_alphas(sg, lx0, ly0, x0, y0, live, ws, th64, al, om, ef, n_redecide);
                if (W == 0) {
                    c_alpha += mw_live;
                } else {  // w = 1: every pixel is its own group and leader
                    const unsigned pb = __ballot_sync(0xffffffffu, blend != 0u);
                    c_leader += mw_live;
                    c_alpha += slice_any(pb, shift);
                }
            } else {
                // leader phase: the leader pixel's alpha counts even if that pixel is done (rasterize.py:281)
                const bool glive = W == 2 ? live != 0u : (lb & gmask) != 0u;
                const uint32_t lneed = (leader_thread && glive) ? 1u : 0u;
                const uint32_t lpass = quad_alphas(sg, lx0, ly0, x0, y0, lneed, ws, th64, al, om, ef, n_redecide);
                const unsigned pb = __ballot_sync(0xffffffffu, lpass != 0u);
                c_leader += mw_live;
                c_alpha += slice_any(pb, shift);
                blend = 0u;
                if (pb != 0u) {  // member phase (rasterize.py:283-289), skipped when no leader of the warp passed
                    const bool my_pass = (pb >> (W == 2 ? lane : leader_lane)) & 1u;
                    const uint32_t mneed = my_pass ? live : 0u;
                    blend = quad_alphas(sg, lx0, ly0, x0, y0, mneed, ws, th64, al, om, ef, n_redecide);
                }
            }
            const unsigned bb = __ballot_sync(0xffffffffu, blend != 0u);
            if (bb == 0u) continue;
            c_blend += slice_any(bb, shift);
            n_blend += __popc(blend);
            uint32_t amb = 0;
#pragma unroll
            for (int s = 0; s < 4; s++) {  // _blend (rasterize.py:169-177), predicated per pixel
                const bool on = (blend >> s) & 1u;
                const float a = on ? al[s] : 0.0f;
                const float t0 = st.T[s];
                const float wgt = t0 * a;
                st.C[s][0] = fmaf(wgt, sg.r, st.C[s][0]);
                st.C[s][1] = fmaf(wgt, sg.g, st.C[s][1]);
                st.C[s][2] = fmaf(wgt, sg.b, st.C[s][2]);
                st.T64[s] *= on ? om[s] : 1.0;
                const float t1 = (float)st.T64[s];
                st.T[s] = t1;
                const float d1 = fmaf(st.D[s], (float)(on ? om[s] : 1.0), t0 * ef[s]);
                st.D[s] = on ? d1 : st.D[s];
                st.cnt[s] += on ? 1 : 0;
                const bool done = on && (t1 + d1 < gm_lo);
                const bool unsure = on && !done && (t1 - d1 < gm_hi);
                live &= ~((done ? 1u : 0u) << s);
                amb |= (unsure ? 1u : 0u) << s;
            }
            if (amb != 0u) {
                // T < gamma undecidable in fp32: recompute this pixel's transmittance exactly (fp64,
                // reference formula) over every splat up to this one, then decide.  A live pixel's
                // blends depend only on its own alphas (and its group leader's for CR), so this is
                // self-contained; rare, and the other warps of the SM keep running meanwhile.
                n_tamb += __popc(amb);
                const uint32_t k_end = b0 + (uint32_t)j;
#pragma unroll
                for (int s = 0; s < 4; s++) {
                    if (!((amb >> s) & 1u)) continue;
                    const double T = exact_transmittance<W>(ws, pair_pos, rg.x, k_end, x0 + (s & 1), y0 + (s >> 1),
                                                            lead_x, lead_y, th64);
                    st.T64[s] = T;
                    st.T[s] = (float)T;
                    st.D[s] = 0.0f;
                    if (T < cfg.gamma) live &= ~(1u << s);
                }
            }
        }
    }
    const uint32_t w_red = __reduce_add_sync(0xffffffffu, n_redecide);
    const uint32_t w_tamb = __reduce_add_sync(0xffffffffu, n_tamb);
    const uint32_t w_live = __reduce_add_sync(0xffffffffu, n_live);
    const uint32_t w_blend = __reduce_add_sync(0xffffffffu, n_blend);
    if (lane == 0) {
        unsigned long long *st = (unsigned long long *)stats;
        if (w_red) atomicAdd(st + SEELE_STAT_ALPHA_REDECIDE, (unsigned long long)w_red);
        if (w_tamb) atomicAdd(st + SEELE_STAT_T_AMBIGUOUS, (unsigned long long)w_tamb);
        if (w_live) atomicAdd(st + SEELE_STAT_LIVE_PIXEL_STEPS, (unsigned long long)w_live);
        if (w_blend) atomicAdd(st + SEELE_STAT_PIXEL_BLENDS, (unsigned long long)w_blend);
    }
#pragma unroll
    for (int s = 0; s < 4; s++) {
        if (!((valid >> s) & 1u)) continue;
        const long long pix = (long long)(y0 + (s >> 1)) * cam.width + x0 + (s & 1);
        image[3 * pix + 0] = fmaf(st.T[s], (float)cfg.bg[0], st.C[s][0]);  // background (rasterize.py:228-231)
        image[3 * pix + 1] = fmaf(st.T[s], (float)cfg.bg[1], st.C[s][1]);
        image[3 * pix + 2] = fmaf(st.T[s], (float)cfg.bg[2], st.C[s][2]);
        if (contrib) contrib[pix] = st.cnt[s];
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
