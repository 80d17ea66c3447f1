// Standalone timing of launch_radix_sort (sort.cu) for several sizes and key
// distributions.  Build: make -C tools sortbench (links ../paper_2406_12080_b200/csrc/_obj/sort.o)
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include "../paper_2406_12080_b200/csrc/hs_kernels.h"
#include <cub/device/device_radix_sort.cuh>

namespace hs { std::atomic<unsigned long long> g_kernel_launches{0}; }
#ifdef SORT_PROF
extern __device__ unsigned long long g_sort_prof[4096][8];
static void dump_prof(uint64_t n) {
    static unsigned long long h[4096][8];
    cudaMemcpyFromSymbol(h, g_sort_prof, sizeof(h));
    const uint64_t tiles = (n + 4095) / 4096;
    unsigned long long t0 = ~0ull;
    for (uint64_t t = 0; t < tiles && t < 4096; ++t) t0 = std::min(t0, h[t][0]);
    double acc[8] = {0};
    for (uint64_t t = 0; t < tiles && t < 4096; ++t)
        for (int k = 1; k < 7; ++k) acc[k] += (double)(h[t][k] - h[t][k - 1]);
    printf("  n=%llu tiles=%llu mean phase us: acquire %.2f rank %.2f scan %.2f reorder+lookback %.2f scatter %.2f\n",
           (unsigned long long)n, (unsigned long long)tiles, acc[1] / tiles / 1e3, acc[2] / tiles / 1e3, acc[3] / tiles / 1e3, acc[5] / tiles / 1e3, acc[6] / tiles / 1e3);
    for (uint64_t t = 0; t < tiles && t < 4096; t += tiles / 8 + 1)
        printf("  tile %5llu start %.2f end %.2f us\n", (unsigned long long)t, (h[t][0] - t0) / 1e3, (h[t][6] - t0) / 1e3);
}
#endif

int main() {
    const uint64_t sizes[] = {1u << 20, 2300000, 4600000, 9200000, 36000000, 140000000};
    for (int dist = 0; dist < 2; ++dist)
    for (uint64_t n : sizes) {
        std::vector<uint32_t> hk(n), hv(n);
        std::mt19937 rng(1);
        for (uint64_t i = 0; i < n; ++i) {
            hk[i] = dist == 0 ? rng() : (uint32_t)(((uint64_t)i * 8160 / n) << 8 | (rng() & 0xff));  // 1: tile-sorted-ish
            hv[i] = (uint32_t)i;
        }
        if (dist == 1) { for (uint64_t i = 0; i < n; ++i) { uint64_t j = rng() % n; std::swap(hk[i], hk[j]); } }
        uint32_t *k[2], *v[2], *scratch; uint64_t* dn;
        for (int b = 0; b < 2; ++b) { cudaMalloc(&k[b], n * 4); cudaMalloc(&v[b], n * 4); }
        const int passes = dist == 0 ? 4 : 2, begin = dist == 0 ? 0 : 8;
        cudaMalloc(&scratch, hs::sort_scratch_words(n, passes) * 4);
        cudaMalloc(&dn, 8);
        cudaMemcpy(dn, &n, 8, cudaMemcpyHostToDevice);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        float best = 1e9;
        for (int rep = 0; rep < 10; ++rep) {
            cudaMemcpy(k[0], hk.data(), n * 4, cudaMemcpyHostToDevice);
            cudaMemcpy(v[0], hv.data(), n * 4, cudaMemcpyHostToDevice);
            cudaEventRecord(e0);
            hs::launch_radix_sort(k, v, dn, n, begin, passes, dist == 0 ? 32 : 13, scratch, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
        }
#ifdef SORT_PROF
        dump_prof(n);
#endif
        std::vector<uint32_t> ok(n), ov(n);
        cudaMemcpy(ok.data(), k[passes & 1], n * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(ov.data(), v[passes & 1], n * 4, cudaMemcpyDeviceToHost);
        bool good = true;
        const uint32_t mask = dist == 0 ? 0xffffffffu : 0xffffff00u;
        for (uint64_t i = 1; i < n && good; ++i) {
            const uint32_t a = ok[i - 1] & mask, b = ok[i] & mask;
            if (a > b || (a == b && ov[i - 1] > ov[i] && dist == 0)) good = false;
        }
        printf("dist=%d n=%9llu passes=%d: %8.1f us (%.1f us/pass) %s err=%s\n", dist, (unsigned long long)n, passes,
               best * 1e3, best * 1e3 / passes, good ? "sorted" : "NOT SORTED", cudaGetErrorString(cudaGetLastError()));
        {   // calibration only: CUB's onesweep on the same keys and bit range (not used by the library)
            size_t tmp_bytes = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k[0], k[1], v[0], v[1], (int)n, begin, begin + 8 * passes);
            void* tmp; cudaMalloc(&tmp, tmp_bytes);
            float cbest = 1e9;
            for (int rep = 0; rep < 10; ++rep) {
                cudaMemcpy(k[0], hk.data(), n * 4, cudaMemcpyHostToDevice);
                cudaMemcpy(v[0], hv.data(), n * 4, cudaMemcpyHostToDevice);
                cudaEventRecord(e0);
                cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k[0], k[1], v[0], v[1], (int)n, begin, begin + 8 * passes);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1); cbest = std::min(cbest, ms);
            }
            printf("   cub SortPairs same bits: %8.1f us\n", cbest * 1e3);
            cudaFree(tmp);
        }
        for (int b = 0; b < 2; ++b) { cudaFree(k[b]); cudaFree(v[b]); }
        cudaFree(scratch); cudaFree(dn);
    }
}
