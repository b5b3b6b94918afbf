// SM partitions for the frame pipeline (green contexts, CUDA driver API >= 12.4, resolved at run time
// through cudaGetDriverEntryPoint so the library has no link dependency on libcuda).
//
// The plan stages of a frame (preprocess, depth order, binning: HBM- and latency-bound, small grids) and
// the raster of another frame (issue-bound, every SM) compete for the same SMs when frames are merely
// put on different streams: the raster's CTAs fill the machine and the plan kernels wait for them to
// drain.  Two green contexts split the SMs: plan streams run on `plan_sms` SMs, raster streams on the
// rest, so one frame's plan runs beside another frame's raster.  Kernels launched (runtime API) into a
// partition's streams run on its SMs only; device memory and events are shared with the primary context.
#include <cuda.h>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace seele {

namespace {

struct DrvApi {
    CUresult (*getDevResource)(CUdevice, CUdevResource *, CUdevResourceType) = nullptr;
    CUresult (*split)(CUdevResource *, unsigned int *, const CUdevResource *, CUdevResource *, unsigned int,
                      unsigned int) = nullptr;
    CUresult (*genDesc)(CUdevResourceDesc *, CUdevResource *, unsigned int) = nullptr;
    CUresult (*create)(CUgreenCtx *, CUdevResourceDesc, CUdevice, unsigned int) = nullptr;
    CUresult (*streamCreate)(CUstream *, CUgreenCtx, unsigned int, int) = nullptr;
    CUresult (*deviceGet)(CUdevice *, int) = nullptr;
    bool ok = false;
};

template <typename F>
bool entry(const char *name, F &fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess || !p)
        return false;
    fn = reinterpret_cast<F>(p);
    return true;
}

DrvApi &drv() {
    static DrvApi d;
    static std::once_flag once;
    std::call_once(once, [] {
        d.ok = entry("cuDeviceGetDevResource", d.getDevResource) && entry("cuDevSmResourceSplitByCount", d.split) &&
               entry("cuDevResourceGenerateDesc", d.genDesc) && entry("cuGreenCtxCreate", d.create) &&
               entry("cuGreenCtxStreamCreate", d.streamCreate) && entry("cuDeviceGet", d.deviceGet);
    });
    return d;
}

struct PartStream {
    cudaStream_t s;
    int sms;
};
std::mutex g_mu;
std::vector<PartStream> g_streams;  // every partition stream created, with its partition's SM count

}  // namespace

int stream_sms(cudaStream_t st) {
    if (st) {
        std::lock_guard<std::mutex> lk(g_mu);
        for (const PartStream &p : g_streams)
            if (p.s == st) return p.sms;
    }
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
}

int partition_create(int plan_sms, int n_streams, void **plan_streams, void **raster_streams, int *plan_out,
                     int *raster_out) {
    DrvApi &d = drv();
    if (!d.ok) return -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaFree(0) != cudaSuccess) return -2;  // primary context active
    CUdevice cd;
    if (d.deviceGet(&cd, dev) != CUDA_SUCCESS) return -2;
    CUdevResource all, grp, rem;
    if (d.getDevResource(cd, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return -3;
    unsigned int ng = 1;
    if (d.split(&grp, &ng, &all, &rem, 0, (unsigned)plan_sms) != CUDA_SUCCESS || ng != 1 || rem.sm.smCount == 0)
        return -4;
    CUdevResourceDesc dp, dr;
    CUgreenCtx gp, gr;
    if (d.genDesc(&dp, &grp, 1) != CUDA_SUCCESS || d.genDesc(&dr, &rem, 1) != CUDA_SUCCESS) return -5;
    if (d.create(&gp, dp, cd, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
        d.create(&gr, dr, cd, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS)
        return -6;
    std::lock_guard<std::mutex> lk(g_mu);
    for (int i = 0; i < n_streams; i++) {
        CUstream a, b;
        if (d.streamCreate(&a, gp, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS ||
            d.streamCreate(&b, gr, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS)
            return -7;
        plan_streams[i] = a;
        raster_streams[i] = b;
        g_streams.push_back({reinterpret_cast<cudaStream_t>(a), (int)grp.sm.smCount});
        g_streams.push_back({reinterpret_cast<cudaStream_t>(b), (int)rem.sm.smCount});
    }
    *plan_out = (int)grp.sm.smCount;
    *raster_out = (int)rem.sm.smCount;
    return 0;
}

}  // namespace seele
