// reduce_probe.cu -- which element types the sm_100a TMA bulk reduce-add accepts
// (not part of libcpa): a 32 x 8 box of 64-bit values added into a [64][16]
// global tile by cp.reduce.async.bulk.tensor (2D, 64B swizzle) with the tensor
// map typed UINT64 / INT64, and by the 1-D cp.reduce.async.bulk .add.u64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/reduce_probe tools/reduce_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "ptx_tools.cuh"

using namespace cpa;

__global__ void k_tensor(const __grid_constant__ CUtensorMap m, int x, int y)
{
    __shared__ __align__(1024) unsigned long long box[32 * 8];
    const int r = threadIdx.x;  // 32 threads: row r, 8 values (64B-swizzled chunks)
    for (int k = 0; k < 4; k++) {
        const int c = k ^ ((r >> 1) & 3);
        box[r * 8 + 2 * c] = (unsigned long long)(1000 * r + 2 * k) - 5;  // some negative-looking wrap below
        box[r * 8 + 2 * c + 1] = (unsigned long long)(1000 * r + 2 * k + 1);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (r == 0) {
        tma_reduce_add_2d(&m, x, y, smem_u32(box));
        bulk_commit();
        bulk_wait<0>();
    }
}

__global__ void k_tensor_f64(const __grid_constant__ CUtensorMap m, int x, int y)
{
    __shared__ __align__(1024) double box[32 * 8];
    const int r = threadIdx.x;
    for (int k = 0; k < 4; k++) {
        const int c = k ^ ((r >> 1) & 3);
        box[r * 8 + 2 * c] = 0.5 * r + 2 * k;
        box[r * 8 + 2 * c + 1] = 0.5 * r + 2 * k + 1;
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (r == 0) {
        tma_reduce_add_2d(&m, x, y, smem_u32(box));
        bulk_commit();
        bulk_wait<0>();
    }
}

__global__ void k_linear(unsigned long long *g)
{
    __shared__ __align__(128) unsigned long long row[32][8];
    for (int k = 0; k < 8; k++) row[threadIdx.x][k] = 7 + k;
    fence_proxy_async_smem();
    __syncwarp();
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u64 [%0], [%1], 64;" ::"l"(g + threadIdx.x * 16),
                 "r"(smem_u32(&row[threadIdx.x][0]))
                 : "memory");
    bulk_commit();
    bulk_wait<0>();
}

int main()
{
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    unsigned long long *g;
    cudaMalloc(&g, 64 * 16 * 8);
    for (int t = 0; t < 1; t++) {   // t = 1 (INT64) traps: rejected at run time
        cudaMemset(g, 0, 64 * 16 * 8);
        CUtensorMap m;
        cuuint64_t dims[2] = {16, 64}, str[1] = {16 * 8};
        cuuint32_t box[2] = {8, 32}, es[2] = {1, 1};
        CUresult r = enc(&m, t ? CU_TENSOR_MAP_DATA_TYPE_INT64 : CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, g, dims, str, box,
                         es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        k_tensor<<<1, 32>>>(m, 8, 16);
        k_tensor<<<1, 32>>>(m, 8, 16);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[64 * 16];
        cudaMemcpy(h, g, sizeof h, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int rr = 0; rr < 32; rr++)
            for (int j = 0; j < 8; j++)
                bad += h[(16 + rr) * 16 + 8 + j] != 2 * ((unsigned long long)(1000 * rr + j) - (j % 2 ? 0 : 5));
        printf("tensor reduce-add %s: encode=%d launch=%s mismatches=%d\n", t ? "INT64" : "UINT64", (int)r,
               cudaGetErrorString(e), bad);
        if (e != cudaSuccess) return 1;
    }
    {   // FLOAT64 tensor reduce-add (the float path's fp64 sum_hw)
        cudaMemset(g, 0, 64 * 16 * 8);
        CUtensorMap m;
        cuuint64_t dims[2] = {16, 64}, str[1] = {16 * 8};
        cuuint32_t box[2] = {8, 32}, es[2] = {1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        k_tensor_f64<<<1, 32>>>(m, 8, 16);
        k_tensor_f64<<<1, 32>>>(m, 8, 16);
        cudaError_t e = cudaDeviceSynchronize();
        double h[64 * 16];
        cudaMemcpy(h, g, sizeof h, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int rr = 0; rr < 32; rr++)
            for (int j = 0; j < 8; j++) bad += h[(16 + rr) * 16 + 8 + j] != 2.0 * (0.5 * rr + j);
        printf("tensor reduce-add FLOAT64: encode=%d launch=%s mismatches=%d\n", (int)r, cudaGetErrorString(e), bad);
        if (e != cudaSuccess) return 1;
    }
    cudaMemset(g, 0, 64 * 16 * 8);
    k_linear<<<1, 32>>>(g);
    k_linear<<<1, 32>>>(g);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[64 * 16];
    cudaMemcpy(h, g, sizeof h, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int rr = 0; rr < 32; rr++)
        for (int k = 0; k < 8; k++) bad += h[rr * 16 + k] != 2ull * (7 + k);
    printf("1-D bulk reduce-add u64: %s mismatches=%d\n", cudaGetErrorString(e), bad);
    return 0;
}
