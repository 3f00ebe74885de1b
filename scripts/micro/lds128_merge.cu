// How many shared-memory wavefronts does one warp's LDS.128 cost for a given address pattern?
// (ncu: l1tex__data_pipe_lsu_wavefronts_mem_shared / smsp__inst_executed_op_shared_ld)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds128_merge lds128_merge.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float4 lds128(unsigned a)
{
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
template <int PAT>
__global__ void k(float *out, int iters)
{
    __shared__ float4 sm[2560];
    for (int i = threadIdx.x; i < 2560; i += blockDim.x) sm[i] = make_float4(i, i, i, i);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    int q;
    const int qw = lane >> 3, ql = lane & 7;              // quarter-warp, lane in quarter
    if (PAT == 0) q = lane;                               // 8 distinct per quarter (32 total)
    else if (PAT == 1) q = 8 * qw + (ql >> 2);            // 2 distinct per quarter, adjacent lanes
    else if (PAT == 2) q = 8 * qw + (ql * 3) / 8;         // 3 distinct per quarter
    else if (PAT == 3) q = 8 * qw + (ql >> 1);            // 4 distinct per quarter (pairs)
    else if (PAT == 4) q = 8 * qw + (ql * 5) / 8;         // 5 distinct per quarter
    else if (PAT == 5) q = 8 * qw + (ql & 1);             // 2 distinct per quarter, alternating lanes
    else if (PAT == 6) q = 8 * qw + 4 * (ql >> 2);        // 2 distinct per quarter, 4 quads (64 B) apart
    else q = 40 * qw + 17 * (ql >> 2);                    // 2 distinct per quarter, different 128-B lines
    const unsigned a = (unsigned)__cvta_generic_to_shared(sm + q + 64 * (threadIdx.x >> 5));
    float acc = 0.f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {                      // 8 copies 256 quads apart (same banks)
            const float4 v = lds128(a + 4096u * (unsigned)c + 16u * (unsigned)(__float_as_int(acc) & 0));
            acc += v.x + v.y + v.z + v.w;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main()
{
    float *d; cudaMalloc(&d, 148 * 256 * sizeof(float));
    k<0><<<148, 256>>>(d, 100); k<1><<<148, 256>>>(d, 100); k<2><<<148, 256>>>(d, 100); k<3><<<148, 256>>>(d, 100);
    k<4><<<148, 256>>>(d, 100); k<5><<<148, 256>>>(d, 100); k<6><<<148, 256>>>(d, 100); k<7><<<148, 256>>>(d, 100);
    cudaDeviceSynchronize();
    printf("done\n");
    return 0;
}
