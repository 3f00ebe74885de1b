// Shared-memory data-pipe peak of this B200 (the denominator of K5's roofline):
// every warp of a full-occupancy grid issues back-to-back conflict-free LDS.128 (each quarter-warp
// reads 128 contiguous bytes: one wavefront) from a 16 KB shared buffer; bytes = 16 x lanes x loads.
// The loaded values are folded into a register that is written out, so no load is dead.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_peak smem_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kThreads = 512, kIters = 4096, kUnroll = 16;

__global__ void __launch_bounds__(kThreads) lds_peak(float *out, int salt)
{
    __shared__ __align__(16) float4 buf[1024];
    for (int i = threadIdx.x; i < 1024; i += kThreads) buf[i] = make_float4(i, i + 1, i + 2, i + salt);
    __syncthreads();
    const unsigned base = (unsigned)__cvta_generic_to_shared(buf);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned a = base + (unsigned)((warp * 32 + lane) & 1023) * 16u;   // lane-contiguous: conflict-free
    float acc = 0.f;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            float4 v;
            const unsigned addr = base + ((a - base + (unsigned)u * 512u) & 16383u);
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
            acc += (v.x + v.y) + (v.z + v.w);
        }
        a += 16u * 32u;
    }
    if (acc == -1.f) out[threadIdx.x] = acc;   // never true for these values; keeps the loads live
}

int main()
{
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);     // kHz (max)
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lds_peak, kThreads, 0);
    float *out;
    cudaMalloc(&out, kThreads * sizeof(float));
    const int grid = sms * per_sm * 4;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) lds_peak<<<grid, kThreads>>>(out, w);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int r = 0; r < reps; ++r) lds_peak<<<grid, kThreads>>>(out, r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)reps * grid * kThreads * (double)kIters * kUnroll * 16.0;
    const double gbs = bytes / (ms * 1e-3) / 1e9;
    std::printf("{\"smem_lds128_gbs\": %.1f, \"sms\": %d, \"blocks_per_sm\": %d, \"sm_clock_max_mhz\": %.1f, "
                "\"bytes_per_clk_per_sm_at_max\": %.2f, \"ms\": %.3f, \"err\": \"%s\"}\n",
                gbs, sms, per_sm, clk / 1e3, gbs * 1e9 / (sms * clk * 1e3), ms, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
