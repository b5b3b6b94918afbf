// Development microbenchmark of the depth sort and the tile binning/sort
// (binning.cu) on synthetic C3-like data, linked against the library objects.
//   make -C tools sortbench && ./tools/sortbench [n] [reps]
// Checks the depth order and the pair order against a CPU reference.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../paper_2503_05168_b200/csrc/common.cuh"

using namespace seele;
namespace seele { void debug_trace(void *dst); }

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

int main(int argc, char **argv) {
    const long long n = argc > 1 ? atoll(argv[1]) : 2350000;
    const int reps = argc > 2 ? atoi(argv[2]) : 20;
    const int W = 1920, H = 1080;
    CamK cam{};
    cam.width = W;
    cam.height = H;
    cam.tiles_x = (W + 15) / 16;
    cam.tiles_y = (H + 15) / 16;
    std::mt19937_64 rng(1);
    std::uniform_real_distribution<double> ud(0.2, 20.0);
    std::vector<double> depth(n);
    std::vector<uint32_t> tiles(n);
    std::vector<short4> rect(n);
    unsigned long long lo = ~0ull, hi = 0;
    long long binned = 0, pairs = 0;
    for (long long i = 0; i < n; i++) {
        depth[i] = ud(rng);
        if (i % 97 == 0) depth[i] = depth[i / 2];  // exact ties
        if (i % 89 == 0) depth[i] = depth[i / 3] * (1.0 + 1e-13 * (double)(rng() % 7));  // within one key step
        if (i >= 1000 && i < 1100) depth[i] = 7.0 + 1e-14 * (double)(1100 - i);  // one long run, reversed
        const bool b = (rng() % 100) < 81;
        if (b) {
            const int w = 1 + (int)(rng() % 5), h = 1 + (int)(rng() % 4);
            const int x0 = (int)(rng() % (cam.tiles_x - w + 1)), y0 = (int)(rng() % (cam.tiles_y - h + 1));
            rect[i] = make_short4(x0, x0 + w - 1, y0, y0 + h - 1);
            tiles[i] = w * h;
            const unsigned long long kb = *(unsigned long long *)&depth[i];
            lo = std::min(lo, kb);
            hi = std::max(hi, kb);
            binned++;
            pairs += w * h;
        } else {
            rect[i] = make_short4(1, 0, 1, 0);
            tiles[i] = 0;
        }
    }
    const long long cap = pairs + 4096;
    printf("n=%lld binned=%lld pairs=%lld\n", n, binned, pairs);
    const size_t bytes = carve_workspace(nullptr, n, cap, W, H).bytes;
    void *base;
    CK(cudaMalloc(&base, bytes));
    CK(cudaMemset(base, 0, bytes));
    Workspace ws = carve_workspace(base, n, cap, W, H);
    int64_t *stats;
    CK(cudaMalloc(&stats, sizeof(int64_t) * SEELE_STAT_COUNT));
    ws.stats_ptr = stats;
    CK(cudaMemcpy(ws.depth, depth.data(), 8 * n, cudaMemcpyHostToDevice));

    CK(cudaMemcpy(ws.rect, rect.data(), 8 * n, cudaMemcpyHostToDevice));
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    cudaEvent_t e[4];
    for (auto &x : e) CK(cudaEventCreate(&x));
    float t_sort = 0, t_bin = 0;
    const uint32_t n32 = (uint32_t)n;
    const unsigned long long mm[2] = {lo, hi};
    for (int r = 0; r < reps + 2; r++) {
        launch_frame_begin(ws, cam, stats, st);
        CK(cudaMemcpyAsync(ws.counters + CNT_WS, &n32, 4, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(ws.minmax, mm, 16, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(stats + SEELE_STAT_BINNED, &binned, 8, cudaMemcpyHostToDevice, st));
        CK(cudaEventRecord(e[0], st));
        launch_depth_sort(ws, n, stats, st);
        CK(cudaEventRecord(e[1], st));
        launch_binning(ws, n, cap, cam, stats, st);
        CK(cudaEventRecord(e[2], st));
        CK(cudaStreamSynchronize(st));
        float a, b;
        CK(cudaEventElapsedTime(&a, e[0], e[1]));
        CK(cudaEventElapsedTime(&b, e[1], e[2]));
        if (r >= 2) {
            t_sort += a / reps;
            t_bin += b / reps;
        }
    }
    CK(cudaGetLastError());
    printf("depth sort %.1f us   binning %.1f us\n", 1e3 * t_sort, 1e3 * t_bin);
#ifdef SEELE_SORT_TRACE
    {
        static unsigned long long tr[8][4096][6];
        debug_trace(tr);
        const int ntile = (int)((n + kSortTile - 1) / kSortTile);
        for (int p = 0; p < kDepthPasses; p++) {
            unsigned long long t0 = ~0ull, t1 = 0;
            double ph[4] = {0, 0, 0, 0};
            for (int t = 0; t < ntile && t < 4096; t++) {
                t0 = std::min(t0, tr[p][t][0]);
                t1 = std::max(t1, tr[p][t][4]);
                for (int k = 0; k < 4; k++) ph[k] += (double)(tr[p][t][k + 1] - tr[p][t][k]) / ntile;
            }
            printf("pass %d: span %.1f us; per tile load %.2f rank %.2f lookback %.2f scatter %.2f us\n", p,
                   (t1 - t0) / 1e3, ph[0] / 1e3, ph[1] / 1e3, ph[2] / 1e3, ph[3] / 1e3);
        }
        // start-time spread of the first pass
        for (int t = 0; t < ntile; t += ntile / 8) printf("  tile %d start +%.1f us end +%.1f us\n", t,
            (tr[1][t][0] - tr[1][0][0]) / 1e3, (tr[1][t][4] - tr[1][0][0]) / 1e3);
    }
#endif
    // verify depth order
    uint32_t np;
    CK(cudaMemcpy(&np, ws.counters + CNT_LONG_RUNS, 4, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> order(n);
    CK(cudaMemcpy(order.data(), ws.dval[kDepthFinal], 4 * n, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> want;
    for (long long i = 0; i < n; i++)
        if (tiles[i]) want.push_back((uint32_t)i);
    std::stable_sort(want.begin(), want.end(), [&](uint32_t a, uint32_t b) { return depth[a] < depth[b]; });
    long long bad = 0;
    for (long long i = 0; i < binned; i++) bad += order[i] != want[i];
    printf("long runs %u, order mismatches %lld\n", np, bad);
    // verify pairs: (tile, rank) order
    std::vector<uint32_t> pf(pairs);
    std::vector<uint2> rg(cam.tiles_x * cam.tiles_y);
    CK(cudaMemcpy(pf.data(), ws.pfinal, 4 * pairs, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(rg.data(), ws.ranges, 8 * rg.size(), cudaMemcpyDeviceToHost));
    std::vector<std::vector<uint32_t>> per(rg.size());
    for (long long k = 0; k < binned; k++) {
        const short4 rc = rect[want[k]];
        for (int y = rc.z; y <= rc.w; y++)
            for (int x = rc.x; x <= rc.y; x++) per[y * cam.tiles_x + x].push_back(want[k]);
    }
    long long pbad = 0, off = 0;
    for (size_t t = 0; t < rg.size(); t++) {
        const uint2 r = rg[t];
        const long long len = r.x < r.y ? r.y - r.x : 0;
        if (len != (long long)per[t].size() || (len && r.x != off)) pbad++;
        for (long long j = 0; j < len && j < (long long)per[t].size(); j++) pbad += pf[r.x + j] != per[t][j];
        off += per[t].size();
    }
    printf("pair mismatches %lld\n", pbad);
    return (bad || pbad) ? 1 : 0;
}
