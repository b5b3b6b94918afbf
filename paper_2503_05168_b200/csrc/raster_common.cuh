// Shared device helpers of the two raster engines (raster.cu, raster_fast.cu):
// the reference's alpha in fp64 (rasterize.py:146-151), the model-warp pixel
// and CR-group geometry, the lockstep counters and one exact fp64 step.
#pragma once
#include "common.cuh"

namespace seele {
namespace rast {

// rasterize.py:146-151 in fp64, reference operation order, no contraction.
__device__ __forceinline__ double alpha64(double px, double py, double mx, double my, double a, double b, double c,
                                          double o) {
    const double dx = __dsub_rn(px, mx), dy = __dsub_rn(py, my);
    const double q = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(a, dx), dx), __dmul_rn(__dmul_rn(__dmul_rn(2.0, b), dx), dy)),
                               __dmul_rn(__dmul_rn(c, dy), dy));
    const double al = __dmul_rn(o, exp(__dmul_rn(-0.5, q)));
    return al < kAlphaClamp ? al : kAlphaClamp;
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Pixel owned by (warp, lane) for engine width W (0 = ref).
template <int W>
__device__ __forceinline__ void pixel_of(int warp, int lane, int &lx, int &ly) {
    if (W == 4) {
        lx = 8 * (warp & 1) + (lane & 7);
        ly = 4 * (warp >> 1) + (lane >> 3);
    } else {
        lx = lane & 15;
        ly = 2 * warp + (lane >> 4);
    }
}

// CR group geometry inside the warp: leader lane and member mask.
template <int W>
__device__ __forceinline__ void group_of(int lane, int &leader, unsigned &mask) {
    if (W == 4) {
        const int g = (lane & 7) >> 2;
        leader = 4 * g;
        mask = 0x0F0F0F0Fu << (4 * g);
    } else if (W == 2) {
        const int g = (lane & 15) >> 1;
        leader = 2 * g;
        mask = (3u << (2 * g)) | (3u << (16 + 2 * g));
    } else {
        leader = lane;
        mask = 1u << lane;
    }
}

// Per-warp lockstep counters (warp-uniform).  warp_steps is derived at the
// end: ref = alpha_eval + blend, cr = leader_eval + alpha_eval.
struct Counters {
    uint32_t alpha, blend, leader;
};

template <int W>
__device__ __forceinline__ void add_counters(int64_t *stats, const Counters &k) {
    unsigned long long *st = (unsigned long long *)stats;
    const unsigned long long steps = W == 0 ? (unsigned long long)k.alpha + k.blend
                                            : (unsigned long long)k.leader + k.alpha;
    if (k.alpha) atomicAdd(st + SEELE_STAT_ALPHA_EVAL, (unsigned long long)k.alpha);
    if (k.blend) atomicAdd(st + SEELE_STAT_BLEND, (unsigned long long)k.blend);
    if (k.leader) atomicAdd(st + SEELE_STAT_LEADER_EVAL, (unsigned long long)k.leader);
    if (steps) atomicAdd(st + SEELE_STAT_WARP_STEPS, steps);
}

// fp64 state of one pixel.
struct Px64 {
    double T, C0, C1, C2;
    int cnt;
    bool done;
};

// One splat against one model-warp, fp64, reference semantics.  Returns false
// when every lane of the warp is done before this splat (nothing charged).
template <int W>
__device__ __forceinline__ bool step64(Px64 &s, double px, double py, bool is_leader, int leader, unsigned gmask,
                                       double mx, double my, double a, double b, double c, double o, float r, float g,
                                       float bl, double th, double gm, Counters &k, double *w_out = nullptr) {
    const bool live = !s.done;
    const unsigned lb = __ballot_sync(0xffffffffu, live);
    if (lb == 0u) return false;
    double al = 0.0;
    bool blend = false;
    if (W == 0) {
        if (live) {
            al = alpha64(px, py, mx, my, a, b, c, o);
            blend = al >= th;
        }
        k.alpha += 1;
    } else {
        const bool glive = (lb & gmask) != 0u;
        double la = 0.0;
        bool lpass = false;
        if (is_leader && glive) {  // leader alpha counts even if the leader itself is done (rasterize.py:281)
            la = alpha64(px, py, mx, my, a, b, c, o);
            lpass = la >= th;
        }
        const unsigned pb = __ballot_sync(0xffffffffu, lpass);
        const bool my_pass = (pb >> leader) & 1u;
        if (live && my_pass) {
            al = is_leader ? la : alpha64(px, py, mx, my, a, b, c, o);
            blend = al >= th;
        }
        k.leader += 1;
        k.alpha += pb != 0u;
    }
    k.blend += __any_sync(0xffffffffu, blend);
    if (blend) {  // _blend (rasterize.py:169-177)
        const double wgt = __dmul_rn(s.T, al);
        if (w_out) *w_out = wgt;  // the contribution row entry (rasterize.py:176-177)
        s.C0 = __dadd_rn(s.C0, __dmul_rn(wgt, (double)r));
        s.C1 = __dadd_rn(s.C1, __dmul_rn(wgt, (double)g));
        s.C2 = __dadd_rn(s.C2, __dmul_rn(wgt, (double)bl));
        s.T = __dmul_rn(s.T, __dsub_rn(1.0, al));
        s.cnt += 1;
        if (s.T < gm) s.done = true;
    }
    return true;
}

__device__ __forceinline__ void write_pixel(float *image, int32_t *contrib, int width, int x, int y, double C0,
                                            double C1, double C2, double T, int cnt, const CfgK &cfg) {
    const long long pix = (long long)y * width + x;  // background composite (rasterize.py:228-231)
    image[3 * pix + 0] = (float)__dadd_rn(C0, __dmul_rn(T, cfg.bg[0]));
    image[3 * pix + 1] = (float)__dadd_rn(C1, __dmul_rn(T, cfg.bg[1]));
    image[3 * pix + 2] = (float)__dadd_rn(C2, __dmul_rn(T, cfg.bg[2]));
    if (contrib) contrib[pix] = cnt;
}

}  // namespace rast
}  // namespace seele
