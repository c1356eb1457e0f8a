// Shared-memory update throughput on one B200, measured in-repo: the ceiling of
// the collision count (k_count_frag), whose inner step is four red.shared.add.u32
// per lane to byte counters at pseudo-random ids of a 64K-id block.
// Same launch shape as the count: 512 threads, two CTAs per SM, 72 KB of shared
// memory each.  Variants (lane-updates per SM cycle = the figure of merit):
//   red_random   red.shared.add.u32, random word per lane        (the count's pattern)
//   red_distinct red.shared.add.u32, lane l -> bank l            (no bank conflicts)
//   red_dummy25  as red_random with 25% of the lanes on a per-lane dummy word
//   rmw_random   ld.shared + add + st.shared (not atomic; a bucketed design's floor)
// Prints one JSON line.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e_ = (x);                                                   \
        if (e_ != cudaSuccess) {                                                \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            return 1;                                                           \
        }                                                                       \
    } while (0)

constexpr int THREADS = 512, WORDS = 16384;  // 64K byte counters

__device__ __forceinline__ uint32_t xs32(uint32_t &s) {
    s ^= s << 13;
    s ^= s >> 17;
    s ^= s << 5;
    return s;
}

template <int MODE>
__global__ void __launch_bounds__(THREADS, 2) k_upd(int iters, uint32_t *sink) {
    extern __shared__ __align__(16) uint32_t cw[];
    for (int i = threadIdx.x; i < WORDS + 32; i += THREADS) cw[i] = 0u;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(cw);
    const uint32_t dummy = base + 4u * (WORDS + lane);
    uint32_t s = 0x9e3779b9u * (blockIdx.x * THREADS + threadIdx.x + 1);
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const uint32_t x = xs32(s);
            const uint32_t v = 1u << ((x & 3u) * 8u);
            uint32_t a;
            if (MODE == 1) a = base + 4u * ((((x >> 2) & (WORDS / 32 - 1)) << 5) | (uint32_t)lane);
            else a = base + 4u * ((x >> 2) & (WORDS - 1));
            if (MODE == 2 && (x >> 30) == 0u) a = dummy;
            if (MODE == 3) {
                uint32_t o;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(o) : "r"(a));
                asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(o + v));
            } else {
                asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v));
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) sink[blockIdx.x] = cw[blockIdx.x & (WORDS - 1)];
}

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    CK(cudaSetDevice(dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
    const int smem = 72 * 1024, grid = sms * 2 * 8, iters = 4096;
    uint32_t *sink;
    CK(cudaMalloc(&sink, grid * 4));
    void (*ks[4])(int, uint32_t *) = {k_upd<0>, k_upd<1>, k_upd<2>, k_upd<3>};
    const char *names[4] = {"red_random", "red_distinct", "red_dummy25", "rmw_random"};
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    printf("{\"what\": \"shared-memory update throughput (tools/peaks/smem_red_peak.cu): %d CTAs x %d threads, 2 per SM, 72 KB smem, 4 updates per lane per iteration\", \"sms\": %d, \"clock_rate_mhz_attr\": %d",
           grid, THREADS, sms, clk_khz / 1000);
    for (int m = 0; m < 4; m++) {
        CK(cudaFuncSetAttribute(ks[m], cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        ks[m]<<<grid, THREADS, smem>>>(64, sink);  // warm-up
        CK(cudaDeviceSynchronize());
        float best = 1e30f;
        for (int r = 0; r < 5; r++) {
            CK(cudaEventRecord(a));
            ks[m]<<<grid, THREADS, smem>>>(iters, sink);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            if (ms < best) best = ms;
        }
        const double lanes = (double)grid * THREADS * iters * 4;
        printf(", \"%s\": {\"ms\": %.4f, \"lane_updates_per_s\": %.4e}", names[m], best, lanes / (best * 1e-3));
    }
    printf("}\n");
    return 0;
}
