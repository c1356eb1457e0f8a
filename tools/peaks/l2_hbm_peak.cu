// In-repo B200 bandwidth probe (tools/measure_peaks.py): read-only streams of a
// buffer that fits in L2 (re-read many times: L2 -> SM bandwidth) and of one far
// larger than L2 (HBM read bandwidth), float4 loads, grid = 148 SMs x resident
// CTAs, CUDA-event timing after warm-up.  Prints one JSON line.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

__global__ void __launch_bounds__(512) k_read(const float4 *__restrict__ p, long long n4, int reps, float *out) {
    float acc = 0.f;
    for (int r = 0; r < reps; r++)
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
            const float4 v = __ldcg(p + i);  // L2 only: the L1 must not serve the re-reads
            acc += v.x + v.y + v.z + v.w;
        }
    if (acc == 12345.678f) out[0] = acc;  // keeps the loads
}

static double run(long long bytes, int reps, int iters) {
    float4 *p;
    float *o;
    cudaMalloc(&p, bytes);
    cudaMalloc(&o, 4);
    cudaMemset(p, 0, bytes);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = sms * 4;
    const long long n4 = bytes / 16;
    for (int i = 0; i < 3; i++) k_read<<<grid, 512>>>(p, n4, reps, o);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double best = 0;
    for (int i = 0; i < iters; i++) {
        cudaEventRecord(a);
        k_read<<<grid, 512>>>(p, n4, reps, o);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double gbs = (double)bytes * reps / (ms * 1e-3) / 1e9;
        if (gbs > best) best = gbs;
    }
    cudaFree(p);
    cudaFree(o);
    return best;
}

int main() {
    const double l2 = run(48ll << 20, 200, 10);   // 48 MiB: resident in the 126 MB L2 (both halves)
    const double l2s = run(24ll << 20, 400, 10);  // 24 MiB
    const double hbm = run(4ll << 30, 1, 10);     // 4 GiB: streamed from HBM
    printf("{\"l2_read_gbs_48MiB\": %.1f, \"l2_read_gbs_24MiB\": %.1f, \"hbm_read_gbs_4GiB\": %.1f}\n", l2, l2s, hbm);
    return 0;
}
