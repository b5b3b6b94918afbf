// Probe: SM partitions by green contexts (driver API) with runtime launches into their streams.
// Prints the SMs each partition's kernel ran on and whether two partitions' kernels overlap in time.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <set>
#include <vector>
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char *s; cuGetErrorString(r, &s); printf("%s -> %s\n", #x, s); return 1; } } while (0)
#define RK(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("%s -> %s\n", #x, cudaGetErrorString(r)); return 1; } } while (0)
__global__ void k_smid(unsigned *out, long long spin) {
    unsigned s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    long long t0 = clock64(); while (clock64() - t0 < spin) {}
    if (threadIdx.x == 0) out[blockIdx.x] = s;
}
int main(int argc, char **argv) {
    int nA = argc > 1 ? atoi(argv[1]) : 112;
    RK(cudaSetDevice(0)); RK(cudaFree(0));
    CUdevice dev; CK(cuDeviceGet(&dev, 0));
    CUdevResource all; CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    printf("device SMs %u\n", all.sm.smCount);
    CUdevResource grp, rem; unsigned ng = 1;
    CK(cuDevSmResourceSplitByCount(&grp, &ng, &all, &rem, 0, nA));
    printf("split: %u group(s) of %u SMs, remainder %u SMs\n", ng, grp.sm.smCount, rem.sm.smCount);
    CUdevResourceDesc dA, dB; CK(cuDevResourceGenerateDesc(&dA, &grp, 1)); CK(cuDevResourceGenerateDesc(&dB, &rem, 1));
    CUgreenCtx gA, gB; CK(cuGreenCtxCreate(&gA, dA, dev, CU_GREEN_CTX_DEFAULT_STREAM)); CK(cuGreenCtxCreate(&gB, dB, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream sA, sB; CK(cuGreenCtxStreamCreate(&sA, gA, CU_STREAM_NON_BLOCKING, 0)); CK(cuGreenCtxStreamCreate(&sB, gB, CU_STREAM_NON_BLOCKING, 0));
    unsigned *buf; RK(cudaMalloc(&buf, 2 * 4096 * sizeof(unsigned)));  // primary-context allocation
    cudaEvent_t e[4]; for (auto &x : e) RK(cudaEventCreate(&x));
    const long long spin = 2000000;  // ~1 ms per block
    RK(cudaEventRecord(e[0], (cudaStream_t)sA));
    k_smid<<<4096, 64, 0, (cudaStream_t)sA>>>(buf, spin);
    RK(cudaGetLastError());
    RK(cudaEventRecord(e[1], (cudaStream_t)sA));
    RK(cudaEventRecord(e[2], (cudaStream_t)sB));
    k_smid<<<1024, 64, 0, (cudaStream_t)sB>>>(buf + 4096, spin);
    RK(cudaGetLastError());
    RK(cudaEventRecord(e[3], (cudaStream_t)sB));
    RK(cudaDeviceSynchronize());
    std::vector<unsigned> h(2 * 4096); RK(cudaMemcpy(h.data(), buf, h.size() * 4, cudaMemcpyDeviceToHost));
    std::set<unsigned> a(h.begin(), h.begin() + 4096), b(h.begin() + 4096, h.begin() + 4096 + 1024);
    int both = 0; for (unsigned s : a) both += b.count(s);
    float ta, tb, tab; RK(cudaEventElapsedTime(&ta, e[0], e[1])); RK(cudaEventElapsedTime(&tb, e[2], e[3])); RK(cudaEventElapsedTime(&tab, e[0], e[3]));
    printf("A: %zu distinct SMs, B: %zu distinct SMs, shared %d; A %.2f ms, B %.2f ms, A start -> B end %.2f ms\n",
           a.size(), b.size(), both, ta, tb, tab);
    return 0;
}
