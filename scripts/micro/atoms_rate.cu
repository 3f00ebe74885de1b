// Shared-memory atomic add throughput: conflict-free ATOMS.ADD (lane L -> bank L) vs LDS/STS, one SM's
// view of the LSU wavefront cost (ncu l1tex__data_pipe_lsu_wavefronts_mem_shared per instruction).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atoms_rate atoms_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_atoms(int *out, int iters, int stride) {
    __shared__ int sm[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned a = (unsigned)__cvta_generic_to_shared(sm + (warp * 32 + lane * stride) % 8192);
    for (int i = 0; i < iters; ++i) {
        asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a), "r"(i) : "memory");
        asm volatile("red.shared.add.s32 [%0+4096], %1;" ::"r"(a), "r"(i) : "memory");
    }
    __syncthreads();
    out[blockIdx.x * blockDim.x + threadIdx.x] = sm[threadIdx.x];
}
__global__ void k_lds(int *out, int iters) {
    __shared__ int sm[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned a = (unsigned)__cvta_generic_to_shared(sm + warp * 32 + lane);
    int acc = 0;
    for (int i = 0; i < iters; ++i) {
        int v, w;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
        asm volatile("ld.shared.u32 %0, [%1+4096];" : "=r"(w) : "r"(a));
        acc += v ^ w;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    int *d; cudaMalloc(&d, 148 * 4 * 1024 * sizeof(int));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 4096, blocks = 148 * 4, threads = 1024;
    for (int rep = 0; rep < 2; ++rep) {
        for (int stride : {1, 2, 32}) {
            cudaEventRecord(a); k_atoms<<<blocks, threads>>>(d, iters, stride); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double ops = 2.0 * iters * blocks * (threads / 32);   // warp instructions
            printf("ATOMS stride %2d: %.3f ms, %.3f warp-instr/clk/SM (1.965 GHz)\n", stride, ms, ops / (ms * 1e-3) / 148 / 1.965e9);
        }
        cudaEventRecord(a); k_lds<<<blocks, threads>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double ops = 2.0 * iters * blocks * (threads / 32);
        printf("LDS.32        : %.3f ms, %.3f warp-instr/clk/SM\n", ms, ops / (ms * 1e-3) / 148 / 1.965e9);
    }
    return 0;
}
