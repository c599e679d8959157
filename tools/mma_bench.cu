// mma_bench.cu -- calibration microbenchmark (not part of libcpa): raw
// tcgen05.mma issue rate from static smem tiles, one CTA per SM, one thread
// issuing. Measures the achievable MAC/clk/SM of kind::i8 M=128 x N=256 x K=32
// for each operand-major combination (and kind::f16 as a reference), so the
// cross-term kernel's roofline can be stated against what the hardware does.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "ptx_tools.cuh"

using namespace cpa;

// commit_every: issue tcgen05.commit to an mbarrier after every C MMAs (0 = never);
// wait_every: additionally wait (try_wait) on a pre-completed barrier per commit.
__global__ void __launch_bounds__(128, 1) k_mma_commit(int iters, uint32_t idesc, int commit_every, int do_wait,
                                                     unsigned long long *cycles)
{
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar[8], done;
    __shared__ uint32_t tslot;
    const uint32_t sb = smem_u32(smem);
    for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x) ((uint32_t *)smem)[i] = 0x01010101u * (i & 3);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; i++) mbar_init(smem_u32(&bar[i]), 1);
        mbar_init(smem_u32(&done), 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) tmem_alloc<512>(smem_u32(&tslot));
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = tslot;
    if (threadIdx.x == 0) {
        const uint32_t a = sb, b = sb + 16384;
        long long t0 = clock64();
        int n = 0, c = 0;
        for (int it = 0; it < iters; it++) {
#pragma unroll
            for (int k = 0; k < 4; k++) {
                uint64_t ad = smem_desc_sw128(a + k * 4096, 8192, 1024);
                uint64_t bd = smem_desc_sw128(b + k * 4096, 16384, 1024);
                mma_i8(tm + (it & 1) * 256, ad, bd, idesc, 1);
                if (commit_every && ++n == commit_every) {
                    n = 0;
                    if (do_wait && c >= 8) {  // barrier committed 8 commits ago: wait for it
                        mbar_wait(smem_u32(&bar[c & 7]), ((c >> 3) - 1) & 1);
                        tc_fence_after();
                    }
                    mma_commit(smem_u32(&bar[c & 7]));
                    c++;
                }
            }
        }
        mma_commit(smem_u32(&done));
        mbar_wait(smem_u32(&done), 0);
        long long t1 = clock64();
        cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
    }
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc<512>(tm);
}

template <int KIND>  // 0 = i8, 1 = f16(bf16)
__global__ void __launch_bounds__(128, 1) k_mma(int iters, uint32_t idesc, unsigned long long *cycles)
{
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const uint32_t sb = smem_u32(smem);
    for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x) ((uint32_t *)smem)[i] = 0x01010101u * (i & 3);
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) tmem_alloc<512>(smem_u32(&tslot));
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = tslot;
    if (threadIdx.x == 0) {
        const uint32_t a = sb, b = sb + 16384;
        long long t0 = clock64();
        for (int it = 0; it < iters; it++) {
#pragma unroll
            for (int k = 0; k < 4; k++) {
                uint64_t ad = smem_desc_sw128(a + k * 4096, 8192, 1024);
                uint64_t bd = smem_desc_sw128(b + k * 4096, 16384, 1024);
                if (KIND == 0) mma_i8(tm + (it & 1) * 256, ad, bd, idesc, 1);
                else mma_bf16(tm + (it & 1) * 256, ad, bd, idesc, 1);
            }
        }
        mma_commit(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), 0);
        long long t1 = clock64();
        cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
    }
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc<512>(tm);
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *d;
    cudaMalloc(&d, sizeof(unsigned long long) * sms);
    const int iters = 20000;
    cudaFuncSetAttribute(k_mma<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(k_mma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    struct V { const char *name; int kind; uint32_t idesc; double macs; };
    const uint32_t base_i8 = (2u << 4) | (0u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
    const uint32_t base_f16 = (1u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
    V vs[] = {
        {"i8  A=MN B=MN", 0, base_i8 | (1u << 15) | (1u << 16), 128.0 * 256 * 32},
        {"i8  A=K  B=MN", 0, base_i8 | (1u << 16), 128.0 * 256 * 32},
        {"i8  A=MN B=K ", 0, base_i8 | (1u << 15), 128.0 * 256 * 32},
        {"i8  A=K  B=K ", 0, base_i8, 128.0 * 256 * 32},
        {"bf16 A=K B=K ", 1, base_f16, 128.0 * 256 * 16},
    };
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    for (auto &v : vs) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(e0);
            if (v.kind == 0) k_mma<0><<<sms, 128, 65536>>>(iters, v.idesc, d);
            else k_mma<1><<<sms, 128, 65536>>>(iters, v.idesc, d);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long h[256];
        cudaMemcpy(h, d, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
        double cyc = 0;
        for (int i = 0; i < sms; i++) cyc += h[i];
        cyc /= sms;
        const double n = 4.0 * iters;
        const double macs_per_clk = v.macs * n / cyc;
        const double tops = 2.0 * v.macs * n * sms / (ms * 1e-3) / 1e12;
        printf("%s : %.1f clk/MMA  %.0f MAC/clk/SM  %.0f TOPS (event)  err=%s\n", v.name, cyc / n, macs_per_clk,
               tops, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFuncSetAttribute(k_mma_commit, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    for (int ce : {0, 1, 2, 4, 8}) {
        for (int w = 0; w < 2; w++) {
            if (ce == 0 && w) continue;
            k_mma_commit<<<sms, 128, 65536>>>(iters, vs[0].idesc, ce, w, d);
            cudaDeviceSynchronize();
            unsigned long long h[256];
            cudaMemcpy(h, d, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
            double cyc = 0;
            for (int i = 0; i < sms; i++) cyc += h[i];
            cyc /= sms;
            printf("i8 commit every %d MMAs, wait(8 back)=%d : %.1f clk/MMA  err=%s\n", ce, w, cyc / (4.0 * iters),
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
