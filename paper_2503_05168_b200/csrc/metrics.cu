// Image quality metrics on the device (metrics.py:44-112): PSNR and SSIM of
// two (H, W, 3) fp64 images, so a trajectory can be scored without host
// readback.  fp64 throughout; deterministic block sums, then one final sum.
//
//  * psnr: 10 log10(1 / mean((a - b)^2)) over every channel, +inf if equal.
//  * ssim: BT.601 luminance, 11x11 Gaussian window (sigma 1.5, normalised),
//    "valid" positions only (scipy convolve2d mode="valid" of the symmetric
//    kernel), K1 = 0.01, K2 = 0.03, mean over the valid positions.
#include <math.h>

#include "common.cuh"

namespace seele {
namespace {

constexpr int kWin = 11;
constexpr int kThreads = 256;

__constant__ double c_ssim_kernel[kWin * kWin];

// Block sum of one double per thread into out[blockIdx.x] (fixed order: deterministic).
__device__ __forceinline__ void block_sum(double v, double *out) {
    __shared__ double s[kThreads / 32];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kThreads / 32; w++) t += s[w];
        out[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(kThreads) k_sq_diff(const double *a, const double *b, long long n, double *part) {
    double acc = 0.0;
    for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n; i += (long long)gridDim.x * kThreads) {
        const double d = a[i] - b[i];
        acc = fma(d, d, acc);
    }
    block_sum(acc, part);
}

__global__ void k_luma(const double *img, long long n_px, double *out) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n_px) return;
    const double *p = img + 3 * i;
    out[i] = p[0] * 0.299 + p[1] * 0.587 + p[2] * 0.114;  // img @ _LUMA (metrics.py:65-69)
}

// One valid window position per thread.
__global__ void __launch_bounds__(kThreads) k_ssim(const double *la, const double *lb, int w, int h, double *part) {
    const int vw = w - kWin + 1, vh = h - kWin + 1;
    const long long n = (long long)vw * vh;
    constexpr double c1 = 0.01 * 0.01, c2 = 0.03 * 0.03;
    double acc = 0.0;
    for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n; i += (long long)gridDim.x * kThreads) {
        const int x = (int)(i % vw), y = (int)(i / vw);
        double ma = 0.0, mb = 0.0, saa = 0.0, sbb = 0.0, sab = 0.0;
        for (int dy = 0; dy < kWin; dy++) {
            const double *ra = la + (long long)(y + dy) * w + x, *rb = lb + (long long)(y + dy) * w + x;
#pragma unroll
            for (int dx = 0; dx < kWin; dx++) {
                const double k = c_ssim_kernel[dy * kWin + dx], va = ra[dx], vb = rb[dx];
                ma = fma(k, va, ma);
                mb = fma(k, vb, mb);
                saa = fma(k, va * va, saa);
                sbb = fma(k, vb * vb, sbb);
                sab = fma(k, va * vb, sab);
            }
        }
        const double var_a = saa - ma * ma, var_b = sbb - mb * mb, cov = sab - ma * mb;
        acc += ((2.0 * ma * mb + c1) * (2.0 * cov + c2)) / ((ma * ma + mb * mb + c1) * (var_a + var_b + c2));
    }
    block_sum(acc, part);
}

__global__ void k_final(const double *part, int n, double scale, int mode, double *out) {
    if (threadIdx.x != 0) return;
    double t = 0.0;
    for (int i = 0; i < n; i++) t += part[i];
    const double mean = t * scale;
    out[0] = mode == 0 ? (mean == 0.0 ? INFINITY : 10.0 * log10(1.0 / mean)) : mean;
}

constexpr int kParts = 592;  // 4 x 148

}  // namespace
}  // namespace seele

using namespace seele;

extern "C" {

int seele_psnr(const double *a_dev, const double *b_dev, int64_t n, double *scratch_dev, double *out_dev,
               void *stream) {
    if (!a_dev || !b_dev || !scratch_dev || !out_dev || n < 1) return SEELE_ERR_INVALID_ARGUMENT;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    k_sq_diff<<<kParts, kThreads, 0, st>>>(a_dev, b_dev, n, scratch_dev);
    k_final<<<1, 32, 0, st>>>(scratch_dev, kParts, 1.0 / (double)n, 0, out_dev);
    return cudaGetLastError() == cudaSuccess ? SEELE_OK : SEELE_ERR_CUDA;
}

int seele_ssim(const double *a_dev, const double *b_dev, int32_t width, int32_t height, double *scratch_dev,
               double *out_dev, void *stream) {
    if (!a_dev || !b_dev || !scratch_dev || !out_dev) return SEELE_ERR_INVALID_ARGUMENT;
    if (width < kWin || height < kWin) return SEELE_ERR_INVALID_ARGUMENT;
    static bool init = false;
    if (!init) {  // normalised 11x11 Gaussian, sigma 1.5 (metrics.py:57-62)
        double k1[kWin], s = 0.0, k2[kWin * kWin];
        for (int i = 0; i < kWin; i++) k1[i] = exp(-0.5 * ((i - 5.0) / 1.5) * ((i - 5.0) / 1.5));
        for (int i = 0; i < kWin; i++)
            for (int j = 0; j < kWin; j++) s += (k2[i * kWin + j] = k1[i] * k1[j]);
        for (double &v : k2) v /= s;
        if (cudaMemcpyToSymbol(c_ssim_kernel, k2, sizeof(k2)) != cudaSuccess) return SEELE_ERR_CUDA;
        init = true;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long n_px = (long long)width * height;
    double *la = scratch_dev + kParts, *lb = la + n_px;
    k_luma<<<(int)((n_px + 255) / 256), 256, 0, st>>>(a_dev, n_px, la);
    k_luma<<<(int)((n_px + 255) / 256), 256, 0, st>>>(b_dev, n_px, lb);
    k_ssim<<<kParts, kThreads, 0, st>>>(la, lb, width, height, scratch_dev);
    const long long valid = (long long)(width - kWin + 1) * (height - kWin + 1);
    k_final<<<1, 32, 0, st>>>(scratch_dev, kParts, 1.0 / (double)valid, 1, out_dev);
    return cudaGetLastError() == cudaSuccess ? SEELE_OK : SEELE_ERR_CUDA;
}

int64_t seele_metrics_scratch_doubles(int32_t width, int32_t height) {
    return (int64_t)kParts + 2LL * width * height;
}

}  // extern "C"
