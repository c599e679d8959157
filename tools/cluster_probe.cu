// probe: shared-address encodings in a 2-CTA cluster (debug aid)
#include <cstdio>
#include <cstdint>
#include "ptx_tools.cuh"
using namespace cpa;
__global__ void __cluster_dims__(2, 1, 1) k(unsigned *out)
{
    __shared__ uint64_t bar;
    uint32_t a = smem_u32(&bar);
    uint32_t r = cluster_ctarank();
    if (threadIdx.x == 0) {
        out[r * 4 + 0] = a;
        out[r * 4 + 1] = mapa_shared(a, 0);
        out[r * 4 + 2] = mapa_shared(a, 1);
        out[r * 4 + 3] = a & 0xFEFFFFFFu;
    }
}
int main()
{
    unsigned *d, h[8];
    cudaMalloc(&d, 32);
    k<<<2, 32>>>(d);
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    for (int r = 0; r < 2; r++) printf("rank %d: cta=%08x mapa0=%08x mapa1=%08x masked=%08x\n", r, h[4*r], h[4*r+1], h[4*r+2], h[4*r+3]);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
