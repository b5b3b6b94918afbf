// Hybrid preprocessing on sm_100a: device-side cluster-table lookup (K0) and
// the fused per-splat preprocess kernel (K1).
//
// K1 replaces plan_frame's per-splat loop (render.py:94-126): Gaussian3D
// rotation normalisation (model.py:122), project_detailed
// (preprocess.py:89-146: near cull, EWA Jacobian, 0.3 low-pass, determinant
// test, conic), sh_to_color (model.py:264-305), effective_radius_sq
// (preprocess.py:68-71) and the bin_tiles extent box (preprocess.py:159-189).
// The projection runs in fp64 in the reference's operation order, but with
// FMA contraction allowed and a reciprocal 1/z where the reference divides
// (preprocess.py:107): the fp64 results differ from numpy's in the last bits,
// so a discrete output (tile rect, depth order) could flip only for a value
// within ~1e-15 relative of a tile edge or of another depth -- never on the
// test scenes, where the oracle comparison over whole trajectories is the
// gate.  K0 (k_select) is written with explicit _rn intrinsics (no
// contraction): its distances are numpy's.  K1 is HBM-bound: 240 B of scene
// in (float4 planes, coalesced) and the raster record out per splat.
#include <math.h>

#include "common.cuh"

namespace seele {

namespace {

// SH constants (model.py:24-41).  The colour only feeds the blend (image
// tolerance 1e-3, plan colours compared at 1e-6), so it is evaluated in fp32.
constexpr float kSH_C0 = 0.28209479177387814f;
constexpr float kSH_C1 = 0.4886025119029199f;
__constant__ float kSH_C2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f,
                             -1.0925484305920792f, 0.5462742152960396f};
__constant__ float kSH_C3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f,
                             0.3731763325901154f, -0.4570457994644658f, 1.445305721320277f,
                             -0.5900435899266435f};

__device__ __forceinline__ void quat_to_mat(double w, double x, double y, double z, double r[9]) {
    // model.py:83-93
    r[0] = 1 - 2 * (y * y + z * z);
    r[1] = 2 * (x * y - w * z);
    r[2] = 2 * (x * z + w * y);
    r[3] = 2 * (x * y + w * z);
    r[4] = 1 - 2 * (x * x + z * z);
    r[5] = 2 * (y * z - w * x);
    r[6] = 2 * (x * z - w * y);
    r[7] = 2 * (y * z + w * x);
    r[8] = 1 - 2 * (x * x + y * y);
}

// sh_to_color for one channel (model.py:276-305), then +0.5 and clamp at 0.
// `s(k)` yields coefficient k of the channel (loaded on demand: each is used once).
template <typename Coef>
__device__ __forceinline__ float sh_channel(Coef s, float x, float y, float z, int degree) {
    float c = kSH_C0 * s(0);
    if (degree >= 1) c = c - kSH_C1 * y * s(1) + kSH_C1 * z * s(2) - kSH_C1 * x * s(3);
    if (degree >= 2) {
        const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
        c = c + kSH_C2[0] * xy * s(4) + kSH_C2[1] * yz * s(5) + kSH_C2[2] * (2.0f * zz - xx - yy) * s(6) +
            kSH_C2[3] * xz * s(7) + kSH_C2[4] * (xx - yy) * s(8);
        if (degree >= 3) {
            c = c + kSH_C3[0] * y * (3.0f * xx - yy) * s(9) + kSH_C3[1] * xy * z * s(10) +
                kSH_C3[2] * y * (4.0f * zz - xx - yy) * s(11) +
                kSH_C3[3] * z * (2.0f * zz - 3.0f * xx - 3.0f * yy) * s(12) +
                kSH_C3[4] * x * (4.0f * zz - xx - yy) * s(13) + kSH_C3[5] * z * (xx - yy) * s(14) +
                kSH_C3[6] * x * (xx - 3.0f * yy) * s(15);
        }
    }
    c = c + 0.5f;
    return c > 0.0f ? c : 0.0f;
}

// _axis_range (preprocess.py:149-156): inclusive [first, last]; first > last = none.
__device__ __forceinline__ void axis_range(double lo, double hi, int n_tiles, int &first, int &last) {
    double f = floor(lo / kTile);
    if (f * kTile == lo) f -= 1.0;
    double l = floor(hi / kTile);
    f = f < 0.0 ? 0.0 : f;
    l = l > (double)(n_tiles - 1) ? (double)(n_tiles - 1) : l;
    if (!(f <= l)) {
        first = 1;
        last = 0;
    } else {
        first = (int)f;
        last = (int)l;
    }
}

struct Splat {
    double p[3], s[3], q[4], o;  // SH coefficients are loaded later, channel by channel
};

__device__ __forceinline__ double sigmoid_clip(double x) {
    // io.py:33-34 _decode_opacity = clip(sigmoid(x), 1e-12, 1 - 1e-12); sigmoid model.py:44-54:
    // x >= 0: 1 / (1 + exp(-x)), else exp(x) / (1 + exp(x)) -- the same two formulas with one exp and one
    // division (a divergent if / else would run both exps in every warp)
    const double e = exp(-fabs(x));
    double v = (x >= 0.0 ? 1.0 : e) / (1.0 + e);
    v = v < 1e-12 ? 1e-12 : v;
    v = v > 1.0 - 1e-12 ? 1.0 - 1e-12 : v;
    return v;
}

__device__ __forceinline__ void normalize4(double q[4]) {
    const double r = 1.0 / sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    q[0] *= r;
    q[1] *= r;
    q[2] *= r;
    q[3] *= r;
}

// planes layout: xyz + opacity logit, log scale, raw quaternion (container record, io.py:22-25)
__device__ __forceinline__ void splat_from_planes(float4 p0, float4 p1, float4 p2, Splat &g) {
    g.p[0] = p0.x; g.p[1] = p0.y; g.p[2] = p0.z;
    g.o = sigmoid_clip((double)p0.w);
    g.s[0] = p1.x; g.s[1] = p1.y; g.s[2] = p1.z;
    g.q[0] = p2.x; g.q[1] = p2.y; g.q[2] = p2.z; g.q[3] = p2.w;
    normalize4(g.q);  // container decode (io.py:226-229)
    normalize4(g.q);  // Gaussian3D.__post_init__ (model.py:122, 76-80)
}

template <int LAYOUT>
__device__ __forceinline__ void load_splat(const SceneK &sc, long long i, int sh_planes, Splat &g) {
    if (LAYOUT == SEELE_LAYOUT_PLANES) {
        const long long st = sc.plane_stride;
        splat_from_planes(__ldg(sc.planes + 0 * st + i), __ldg(sc.planes + 1 * st + i), __ldg(sc.planes + 2 * st + i), g);
        return;
    } else {
        for (int k = 0; k < 3; k++) {
            g.p[k] = sc.pos[3 * i + k];
            g.s[k] = sc.log_scale[3 * i + k];
        }
        for (int k = 0; k < 4; k++) g.q[k] = sc.rot[4 * i + k];
        g.o = sc.opac[i];
    }
    normalize4(g.q);  // Gaussian3D.__post_init__ (model.py:122, 76-80)
}

// FAST raster record of one projected splat (raster_fast.cu), fp64 here.
//
// The raster evaluates q' = k q, k = log2(e) / 2, in fp32 in Cholesky form
// q' = (l11 dx + l21 dy)^2 + (l22 dy)^2, with (l11, l21, l22) = fl32 of the
// factor of k C (C = conic), and the mean as hi floats with the lo parts folded
// into the coordinates: dx = fl(px - mx_hi), t = fma(l21, dy, -cu),
// u1 = fma(l11, dx, t), w = fma(l22, dy, -cw), q' = fma(u1, u1, fl(w^2)),
// cu = fl(l11 mx_lo + l21 my_lo), cw = fl(l22 my_lo).  The bound below was
// derived for the hi + lo form dx = fl(fl(px - mx_hi) - mx_lo) (one more
// rounding of each coordinate); the folded form has every rounding it has
// except that one (cu, cw are ~2^-24 |m| |l|, their own rounding ~2^-48), so
// the bound covers it.
// With u = 2^-24, U = l11 dx + l21 dy and W = l22 dy (exact, so q' = U^2 +
// W^2): the coefficient roundings (u each), the rounding of dx, dy (exact
// unless the mean is > 2^11 px away, else u each) and of t and u1 give
// |dU| <= 2u (|l11 dx| + |l21 dy|) + u |t| + u |U| <= 3u |U| + 5u |l21 dy|
// (|l11 dx| <= |U| + |l21 dy|), and |dW| <= 3u |W|; with the roundings of w^2
// and of q', |q'32 - q'| <= 8u q' + 10u |U| |l21 dy|.  |l21 dy| = |l21 / l22|
// |W| (l21 / l22 = b / sqrt(det) for the conic (a, b, c)) and |U| |W| <=
// (U^2 + W^2) / 2 = q' / 2, so the cancellation term is 5u q' |b| / sqrt(det):
// it vanishes for axis-aligned ellipses, and is at most 5u q' sqrt(kappa / 2)
// (round 1 bounded it by 10u q' sqrt(kappa) through |d|: the C4 scene's
// transmittance walks fall from 623K to 227K per frame with |U|, |W| <=
// sqrt(q') taken apart, and further with their product bounded together;
// tests/test_qbound.py replays the fp32 sequence against the bound).  Round 1's
// additive terms 6u P sqrt(q') (mean and pixel
// representation) are kept.  Linearised around the threshold (sqrt(x) <=
// (s + x / s) / 2, s^2 = q_th') and taken with a 1.25 safety factor:
// |q'32 - q'| <= e0q + e1q q'.  No cancellation in the sum of squares: the
// error grows like sqrt(kappa), not kappa (the direct a dx^2 + 2b dx dy + c dy^2
// form).
// The alpha-test bracket [q_lo', q_hi'] widens q_th' = k 2 ln(o / theta)
// (rasterize.py:146-151, 209: alpha >= theta <=> q <= q_th) by that bound,
// the fp64-vs-numpy evaluation difference (1e-15 kappa) and two roundings.
// The alpha relative error model adds ex2.approx (2^-21.5), the rounding of o
// and of o e, and ln 2 times the q' error: e0 = 4.7e-7 + ln2 e0q, e1 = ln2 e1q.
// The raster culls a splat per warp with the exact minimum of q' over the
// warp's pixel rectangle against q_hi' (no box is stored).
// 32 bytes (two float4) by one 256-bit store
__device__ __forceinline__ void st256(float4 *dst, const float4 &a, const float4 &b) {
    asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst), "f"(a.x), "f"(a.y), "f"(a.z),
                 "f"(a.w), "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w)
                 : "memory");
}

__device__ __forceinline__ void write_raster_record(const Workspace &ws, long long p, double m0, double m1, double ca,
                                                    double cb, double cc, double o, double qth, float qth_err,
                                                    float4 &rec2) {
    const double K = 0.72134752044448170368;  // log2(e) / 2
    const double det = ca * cc - cb * cb;
    float4 rq = make_float4(-INFINITY, -INFINITY, 0.f, 0.f);
    if (qth >= 0.0) {
        // The error-model terms are upper bounds, so they are evaluated in fp32 and widened by 1.001
        // (several fp32 roundings); lmin = det / lmax has no cancellation.  Any s > 0 is a valid
        // linearisation point (AM-GM), so sq needs no rounding care.
        constexpr float u = 5.9604644775390625e-08f;  // 2^-24
        constexpr float W = 1.001f;
        const float caf = (float)ca, cbf = (float)cb, ccf = (float)cc, trf = caf + ccf;
        const float hd = 0.5f * (caf - ccf);
        const float lmax = 0.5f * trf + sqrtf(fmaf(hd, hd, cbf * cbf));
        const float kap = W * trf * lmax / fmaxf((float)det, 1e-30f);  // tr / lmin >= 1
        const double qt = K * qth;
        const float qtf = (float)qt;
        const float P = W * sqrtf((float)K * trf);
        const float sq = fmaxf(sqrtf(qtf), 1e-3f);
        const float e0q = W * 1.25f * 3.0f * u * P * sq;
        // the cancellation term: 10u |U| |l21 dy| = 10u (|b| / sqrt(det)) |U| |W| <= 5u (|b| / sqrt(det)) q'
        // (derivation above)
        const float bsd = (float)(fabs(cb) / sqrt(fmax(det, 1e-300)));
        const float e1q = W * 1.25f * (u * (8.0f + 5.0f * bsd) + 3.0f * u * P / sq);
        const float delta = W * (e0q + e1q * qtf + qtf * (1e-15f * 2.0f * kap + 2.0f * u) + (float)K * qth_err) + 1e-30f;
        rq.x = __double2float_rd(qt - (double)delta);
        rq.y = delta < 1e6f ? __double2float_ru(qt + (double)delta) : INFINITY;
        rq.z = W * (4.7e-7f + 0.6931471805599453f * e0q);
        rq.w = W * 0.6931471805599453f * e1q;
    }
    const double l11 = sqrt(K * ca);
    const double l21 = K * cb / l11;
    const double l22 = sqrt(fmax(K * det / ca, 0.0));
    // raster record: the mean as hi floats + the folded lo parts (below); q_up = the first float above
    // the bracket top, so q' <= q_hi' <=> q' < q_up; the error model is widened by 2^-10 for the fp32
    // bound arithmetic of the raster (products with T rounded upward)
    const float mxh = (float)m0, myh = (float)m1;
    float4 *rec = reinterpret_cast<float4 *>(ws.rec + p);
    // lo parts of the mean (exact in fp64) folded into the Cholesky coordinates with the float factors the
    // raster uses; |cu|, |cw| ~ 2^-24 |m| |l|, so their own rounding is ~2^-48 |m| |l|: the raster's u, w
    // carry no rounding of x - mxh - mxl (one fewer than the hi + lo form the error model was derived for)
    const float l11f = (float)l11, l21f = (float)l21, l22f = (float)l22;
    const double mxl = m0 - (double)mxh, myl = m1 - (double)myh;
    // (the record's first and second halves are written by one 256-bit store each: full sectors)
    st256(rec, make_float4(mxh, (float)((double)l11f * mxl + (double)l21f * myl), myh, (float)((double)l22f * myl)),
          make_float4(l11f, l21f, l22f, (float)o));
    // (q_lo, w_up): the bracket [q_lo, q_up) as its width rounded upward, so the raster tests it on
    // d = q' - q_lo alone (0 <= d <= w_up, compared as bit patterns); an empty bracket (o < theta) has w_up = 0
    const float q_up = nextafterf(rq.y, INFINITY);
    const float w_up = rq.x == -INFINITY ? 0.0f : __double2float_ru(__dsub_ru((double)q_up, (double)rq.x));
    rec2 = make_float4(rq.x, w_up, rq.z * (1.0f + 1.0f / 1024.0f), rq.w * (1.0f + 1.0f / 1024.0f));  // (stored with the colour)
    // the exact record, whole: two 32-byte stores (full sectors, no partial-sector merging in L2)
    double *xr = reinterpret_cast<double *>(ws.xrec + p);
    const double qw = __hiloint2double((int)__float_as_uint(w_up), (int)__float_as_uint(rq.x));  // (q_lo, w_up)
    asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(xr), "d"(m0), "d"(m1), "d"(ca), "d"(cb) : "memory");
    asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(xr + 4), "d"(cc), "d"(o), "d"(qw), "d"(0.0) : "memory");
}

// Block-level reduction of the per-thread frame counters: one atomic per
// counter per CTA instead of one per warp and iteration.
__device__ __forceinline__ void flush_block(int64_t *stats, uint32_t (&c)[4]) {
    __shared__ uint32_t s_c[4];
    if (threadIdx.x < 4) s_c[threadIdx.x] = 0u;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const uint32_t v = __reduce_add_sync(0xffffffffu, c[k]);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s_c[k], v);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long *st = (unsigned long long *)stats;
        if (s_c[0]) atomicAdd(st + SEELE_STAT_CULLED_NEAR, (unsigned long long)s_c[0]);
        if (s_c[1]) atomicAdd(st + SEELE_STAT_DROPPED_DEGENERATE, (unsigned long long)s_c[1]);
        if (s_c[2]) atomicAdd(st + SEELE_STAT_PROJECTED, (unsigned long long)s_c[2]);
        if (s_c[3]) atomicAdd(st + SEELE_STAT_BINNED, (unsigned long long)s_c[3]);
    }
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

#ifndef SEELE_PRE_THREADS
#define SEELE_PRE_THREADS 256
#endif
#ifndef SEELE_PRE_MINB
#define SEELE_PRE_MINB (768 / SEELE_PRE_THREADS)
#endif
constexpr int kPre = SEELE_PRE_THREADS;  // threads per CTA
template <int LAYOUT>
__global__ void __launch_bounds__(kPre, SEELE_PRE_MINB) k_preprocess(SceneK sc, const int64_t *__restrict__ ranges,
                                                    int n_ranges, CamK cam, CfgK cfg, Workspace ws,
                                                    int64_t *stats) {
    __shared__ long long s_start[SEELE_MAX_RANGES], s_prefix[SEELE_MAX_RANGES + 1];
    // SH planes of this thread's splat, copied asynchronously (cp.async / LDGSTS) at the top of each
    // iteration so the transfer overlaps the fp64 projection; plane k of thread t at [k][t]
    extern __shared__ float4 s_sh[];
    if (threadIdx.x == 0) {
        long long acc = 0;
        for (int r = 0; r < n_ranges; r++) {
            s_start[r] = ranges[2 * r];
            s_prefix[r] = acc;
            acc += ranges[2 * r + 1];
        }
        s_prefix[n_ranges] = acc;
        if (blockIdx.x == 0) {
            ws.counters[CNT_WS] = (uint32_t)acc;
            stats[SEELE_STAT_WORKING_SET] = acc;
        }
    }
    __syncthreads();
    const long long n_ws = s_prefix[n_ranges];
    const int sh_planes = cfg.sh_degree >= 3 ? 4 : (cfg.sh_degree == 2 ? 3 : 1);
    const long long stride = (long long)gridDim.x * blockDim.x;
    uint32_t cnt[4] = {0u, 0u, 0u, 0u};
    const unsigned long long zbase = depth_order_key(cam.near_clip);
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n_ws; p += stride) {
        int status = 3;
        uint32_t n_tiles = 0;
        uint32_t bi = 0u;  // index in the depth bucket (binned splats)
        double sz = 0.0;   // view depth (binned, or every projected splat with keep_unbinned)
        {
            int r = 0;
            while (r + 1 < n_ranges && s_prefix[r + 1] <= p) r++;
            const long long i = s_start[r] + (p - s_prefix[r]);
            Splat g;
            load_splat<LAYOUT>(sc, i, sh_planes, g);
            const double d[3] = {__dsub_rn(g.p[0], cam.pos[0]), __dsub_rn(g.p[1], cam.pos[1]), __dsub_rn(g.p[2], cam.pos[2])};
            double t[3];
            // world_to_view @ (p - c) rounded like the reference's BLAS dgemv (fused, left to right:
            // tools/blas_order.py); the depth decides near-ties of the sort, so it is bit-exact by construction
            for (int k = 0; k < 3; k++)
                t[k] = __fma_rn(cam.w2v[3 * k + 2], d[2], __fma_rn(cam.w2v[3 * k + 1], d[1], __dmul_rn(cam.w2v[3 * k], d[0])));
            const double z = t[2];
            short4 rect = make_short4(1, 0, 1, 0);
            if (z <= cam.near_clip) {
                status = 1;  // "near" (preprocess.py:101-103)
            } else {
                const double rz = 1.0 / z;
                const double m0 = cam.fx * t[0] * rz + cam.cx;  // preprocess.py:107
                const double m1 = cam.fy * t[1] * rz + cam.cy;
                const double j00 = cam.fx * rz, j02 = -cam.fx * t[0] * rz * rz;
                const double j11 = cam.fy * rz, j12 = -cam.fy * t[1] * rz * rz;
                double jw[6];
                for (int c = 0; c < 3; c++) {
                    jw[c] = j00 * cam.w2v[c] + 0.0 * cam.w2v[3 + c] + j02 * cam.w2v[6 + c];
                    jw[3 + c] = 0.0 * cam.w2v[c] + j11 * cam.w2v[3 + c] + j12 * cam.w2v[6 + c];
                }
                double rg[9];
                quat_to_mat(g.q[0], g.q[1], g.q[2], g.q[3], rg);
                const double es[3] = {exp(g.s[0]), exp(g.s[1]), exp(g.s[2])};
                double m[9], cv[9], cov[9];
                for (int a = 0; a < 3; a++)
                    for (int b = 0; b < 3; b++) m[3 * a + b] = rg[3 * a + b] * es[b];
                for (int a = 0; a < 3; a++)
                    for (int b = 0; b < 3; b++)
                        cv[3 * a + b] = m[3 * a] * m[3 * b] + m[3 * a + 1] * m[3 * b + 1] + m[3 * a + 2] * m[3 * b + 2];
                for (int a = 0; a < 3; a++)
                    for (int b = 0; b < 3; b++) cov[3 * a + b] = 0.5 * (cv[3 * a + b] + cv[3 * b + a]);
                double tmp[6], c2[4];
                for (int a = 0; a < 2; a++)
                    for (int c = 0; c < 3; c++)
                        tmp[3 * a + c] = jw[3 * a] * cov[c] + jw[3 * a + 1] * cov[3 + c] + jw[3 * a + 2] * cov[6 + c];
                for (int a = 0; a < 2; a++)
                    for (int c = 0; c < 2; c++)
                        c2[2 * a + c] = tmp[3 * a] * jw[3 * c] + tmp[3 * a + 1] * jw[3 * c + 1] + tmp[3 * a + 2] * jw[3 * c + 2];
                c2[0] += 0.3;  // COV2D_LOWPASS (preprocess.py:24, 117)
                c2[3] += 0.3;
                const double s00 = 0.5 * (c2[0] + c2[0]), s01 = 0.5 * (c2[1] + c2[2]);
                const double s10 = 0.5 * (c2[2] + c2[1]), s11 = 0.5 * (c2[3] + c2[3]);
                const double det = s00 * s11 - s01 * s10;
                if (!isfinite(det) || det <= 1e-12) {
                    status = 2;  // "degenerate" (preprocess.py:122-124)
                } else {
                    status = 0;
                    const double rdet = 1.0 / det;
                    const double ca = s11 * rdet, cb = -s01 * rdet, cc = s00 * rdet;
                    // alpha >= theta <=> q <= qth = 2 ln(o / theta).  qth >= 9 (o >= theta e^4.5) only feeds the
                    // alpha bracket (r2 clips at 9), which tolerates an fp32 log with its error added to the
                    // bracket; below that qth sets the opacity-aware radius and is taken in fp64.
                    double qth;
                    float qth_err = 0.0f;
                    if (g.o >= cfg.alpha_theta * (90.0171313005218 * (1.0 + 1e-12))) {
                        qth = 2.0 * (double)logf((float)g.o / (float)cfg.alpha_theta);
                        qth_err = 2.0e-6f;  // 2 (two fp32 roundings of the ratio + 1 ulp of logf at <= ~7)
                    } else {
                        qth = 2.0 * log(g.o / cfg.alpha_theta);
                    }
                    double r2 = 9.0;  // MAX_RADIUS_SQ
                    if (cfg.opacity_aware && qth_err == 0.0f) {  // (fp32 log branch: the true qth >= 9, r2 = 9)
                        r2 = qth;
                        r2 = r2 > 9.0 ? 9.0 : r2;
                        r2 = r2 < 0.0 ? 0.0 : r2;
                    }
                    if (r2 > 0.0) {
                        const double detp = ca * cc - cb * cb;
                        const double rdp = 1.0 / detp;
                        const double hx = sqrt(r2 * (cc * rdp)), hy = sqrt(r2 * (ca * rdp));
                        int x0, x1, y0, y1;
                        axis_range(m0 - hx, m0 + hx, cam.tiles_x, x0, x1);
                        axis_range(m1 - hy, m1 + hy, cam.tiles_y, y0, y1);
                        if (x0 <= x1 && y0 <= y1) {
                            rect = make_short4((short)x0, (short)x1, (short)y0, (short)y1);
                            n_tiles = (uint32_t)(x1 - x0 + 1) * (uint32_t)(y1 - y0 + 1);
                        }
                    }
                    // Records are written for binned splats only (a splat no tile bins is never read by the
                    // frame), unless the plan export asked for every projected splat: its SH planes are read
                    // only then, by cp.async overlapping the raster-record arithmetic.
                    if (n_tiles > 0 || cfg.keep_unbinned) {
                        if (LAYOUT == SEELE_LAYOUT_PLANES) {
                            // slot ch * sh_planes + k <- plane 3 + 4 ch + k (the full SH3 case unrolled)
                            const float4 *src = sc.planes + 3 * sc.plane_stride + i;
                            float4 *dst = s_sh + threadIdx.x;
                            if (sh_planes == 4) {
#pragma unroll
                                for (int k = 0; k < 12; k++) cp_async16(dst + k * kPre, src + k * sc.plane_stride);
                            } else {
                                for (int ch = 0; ch < 3; ch++)
                                    for (int k = 0; k < sh_planes; k++)
                                        cp_async16(dst + (ch * sh_planes + k) * kPre, src + (4 * ch + k) * sc.plane_stride);
                            }
                            cp_async_commit();
                        }
                        sz = z;
                        // depth-order bucket (depth.cu) of a binned splat: count it and keep its index in the bucket
                        if (n_tiles > 0) bi = atomicAdd(&ws.bhist[depth_bucket_of_key(depth_order_key(z), zbase)], 1u);
                        float4 rec2;
                        write_raster_record(ws, p, m0, m1, ca, cb, cc, g.o, qth, qth_err, rec2);
                        // view direction for SH (preprocess.py:129-130), fp32 like the colour
                        const float rn = rsqrtf((float)(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]));
                        const float vx = (float)d[0] * rn, vy = (float)d[1] * rn, vz = (float)d[2] * rn;
                        float4 col;
                        if (LAYOUT == SEELE_LAYOUT_PLANES) {
                            float cc3[3];
                            cp_async_wait_all();
#pragma unroll
                            for (int ch = 0; ch < 3; ch++) {
                                float shc[16];
#pragma unroll
                                for (int k = 0; k < 4; k++) {
                                    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                                    if (k < sh_planes) v = s_sh[(ch * sh_planes + k) * kPre + threadIdx.x];
                                    shc[4 * k] = v.x;
                                    shc[4 * k + 1] = v.y;
                                    shc[4 * k + 2] = v.z;
                                    shc[4 * k + 3] = v.w;
                                }
                                cc3[ch] = sh_channel([&](int k) { return shc[k]; }, vx, vy, vz, cfg.sh_degree);
                            }
                            col = make_float4(cc3[0], cc3[1], cc3[2], 0.f);
                        } else {
                            const double *shp = sc.sh + 48 * i;
                            col.x = sh_channel([&](int k) { return (float)shp[k]; }, vx, vy, vz, cfg.sh_degree);
                            col.y = sh_channel([&](int k) { return (float)shp[16 + k]; }, vx, vy, vz, cfg.sh_degree);
                            col.z = sh_channel([&](int k) { return (float)shp[32 + k]; }, vx, vy, vz, cfg.sh_degree);
                        }
                        st256(reinterpret_cast<float4 *>(ws.rec + p) + 2, rec2,
                              make_float4(col.x, col.y, col.z, __uint_as_float((uint32_t)p)));
                    }
                }
            }
            ws.status[p] = (uint8_t)status;
            ws.srec[p] = make_uint4(pack_rect(rect), bi, (uint32_t)__double2loint(sz), (uint32_t)__double2hiint(sz));
        }
        cnt[0] += status == 1;
        cnt[1] += status == 2;
        cnt[2] += status == 0;
        cnt[3] += n_tiles > 0;
    }
    flush_block(stats, cnt);
}

// K0: select_clusters (residency.py:38-54) with pose_feature (compiler.py:113-121).
__global__ void k_select(CamK cam, const double *__restrict__ centroids, int n, int m, double beta,
                         double3 mean3, double scale, const int64_t *__restrict__ chunks,
                         int32_t *out_ids, int64_t *ranges_out) {
    __shared__ double d2[1024];
    double f[6];
    f[0] = __ddiv_rn(__dsub_rn(cam.pos[0], mean3.x), scale);
    f[1] = __ddiv_rn(__dsub_rn(cam.pos[1], mean3.y), scale);
    f[2] = __ddiv_rn(__dsub_rn(cam.pos[2], mean3.z), scale);
    // CameraPose.forward = R_cw[:, 2] (model.py:174-176) = row 2 of world_to_view
    f[3] = __dmul_rn(beta, cam.w2v[6]);
    f[4] = __dmul_rn(beta, cam.w2v[7]);
    f[5] = __dmul_rn(beta, cam.w2v[8]);
    for (int c = threadIdx.x; c < n; c += blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < 6; k++) {
            const double v = __dsub_rn(centroids[6 * c + k], f[k]);
            s = __dadd_rn(s, __dmul_rn(v, v));  // numpy's squared-then-summed values: no contraction
        }
        d2[c] = s;
    }
    __syncthreads();
    // the m + 1 nearest in np.lexsort((arange, d2)) order: centroid c goes to slot rank(c) = the number of
    // centroids before it in (d2, id) order (one thread per centroid, no serial selection)
    if (threadIdx.x == 0) {
        ranges_out[0] = chunks[0];
        ranges_out[1] = chunks[1];
    }
    for (int c = threadIdx.x; c < n; c += blockDim.x) {
        const double v = d2[c];
        int rank = 0;
        for (int o = 0; o < n; o++) rank += (d2[o] < v || (d2[o] == v && o < c)) ? 1 : 0;
        if (rank <= m) {
            out_ids[rank] = c;
            ranges_out[2 * (rank + 1)] = chunks[2 * (c + 1)];
            ranges_out[2 * (rank + 1) + 1] = chunks[2 * (c + 1) + 1];
        }
    }
}

}  // namespace

void launch_preprocess(const SceneK &s, const int64_t *ranges, int n_ranges, const CamK &cam,
                       const CfgK &cfg, const Workspace &ws, int64_t *stats, int grid, cudaStream_t st) {
    grid *= 256 / kPre;  // the caller sizes the grid in 256-thread CTAs
    if (s.layout == SEELE_LAYOUT_PLANES) {
        constexpr int kShSmem = 12 * kPre * sizeof(float4);
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_preprocess<SEELE_LAYOUT_PLANES>, cudaFuncAttributeMaxDynamicSharedMemorySize, kShSmem);
            attr = true;
        }
        k_preprocess<SEELE_LAYOUT_PLANES><<<grid, kPre, kShSmem, st>>>(s, ranges, n_ranges, cam, cfg, ws, stats);
    }
    else
        k_preprocess<SEELE_LAYOUT_F64><<<grid, kPre, 0, st>>>(s, ranges, n_ranges, cam, cfg, ws, stats);
    note_launches(1);
}

void launch_select(const CamK &cam, const double *centroids, int n, int m, double beta, const double *mean3,
                   double scale, const int64_t *chunks, int32_t *out_ids, int64_t *ranges_out, cudaStream_t st) {
    k_select<<<1, 128, 0, st>>>(cam, centroids, n, m, beta, make_double3(mean3[0], mean3[1], mean3[2]), scale, chunks, out_ids, ranges_out);
    note_launches(1);
}

}  // namespace seele
