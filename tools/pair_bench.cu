// pair_bench.cu -- calibration microbenchmark (not part of libcpa): issue rate
// of tcgen05.mma.cta_group::2 kind::i8 (M=256 across a CTA pair) from static
// shared-memory tiles laid out exactly like the cross-term kernel's stages
// (both operands MN-major, 128-byte swizzle, 3-stage ring, one multicast
// commit per stage, the issuer waiting on the commit STAGES stages back).
// No producers: this is the tensor-pipe ceiling the cross-term kernel's
// pipeline can approach.  Variants: accumulators per stage (NT), N per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/pair_bench tools/pair_bench.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "ptx_tools.cuh"

using namespace cpa;

constexpr int STAGES = 3;
constexpr int STAGE_BYTES = 49152;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
k_pair(int stages_total, int nt, int n_mma, int kk_per_stage, int mode, uint32_t idesc, unsigned long long *cycles)
{
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar[STAGES];
    __shared__ uint32_t tslot;
    const uint32_t sb = smem_u32(smem);
    const uint32_t rank = cluster_ctarank();
    for (int i = threadIdx.x; i < STAGES * STAGE_BYTES / 4; i += blockDim.x) ((uint32_t *)smem)[i] = 0x01010101u * (i & 3);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) mbar_init(smem_u32(&bar[s]), 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) tmem_alloc_pair<512>(smem_u32(&tslot));
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tm = tslot;
    if (threadIdx.x == 0 && rank == 0) {
        long long t0 = clock64();
        for (int it = 0; it < stages_total; it++) {
            const int s = mode == 3 ? 0 : mode == 4 ? (it & 1) : it % STAGES;
            if (mode == 6 && it >= STAGES) {
                mbar_wait(smem_u32(&bar[s]), ((it / STAGES) - 1) & 1);
                tc_fence_after();
            }
            if (mode == 0 && it >= STAGES) {
                mbar_wait_cluster(smem_u32(&bar[s]), ((it / STAGES) - 1) & 1);
                tc_fence_after();
            }
            const uint32_t a = sb + s * STAGE_BYTES, b = a + 16384;
            if (mode >= 5) {
                // precomputed descriptors: one 64-bit add per MMA (start address in 16-byte units)
                const uint64_t a0 = smem_desc_sw128(sb, 16384, 1024) + (uint64_t)((s * STAGE_BYTES) >> 4);
                const uint64_t b0 = a0 + (16384 >> 4);
                for (int k = 0; k < kk_per_stage; k++) {
                    mma_i8_pair(tm, a0 + k * 256, b0 + k * 256, idesc, 1);
                    mma_i8_pair(tm + 256, a0 + k * 256, b0 + 1024 + k * 256, idesc, 1);
                }
                if (mode == 6) mma_commit_pair(smem_u32(&bar[s]), 0x3);
                continue;
            }
            for (int k = 0; k < kk_per_stage; k++) {
                const uint64_t ad = smem_desc_sw128(a + (k & 3) * 4096, 16384, 1024);
                for (int n = 0; n < nt; n++) {
                    const uint64_t bd = smem_desc_sw128(b + (n & 1) * 16384 + (k & 3) * 4096, 16384, 1024);
                    mma_i8_pair(tm + n * n_mma, ad, bd, idesc, 1);  // n*n_mma <= 512
                }
            }
            if (mode < 2) mma_commit_pair(smem_u32(&bar[s]), 0x3);
        }
        if (mode >= 2 && mode != 6) mma_commit_pair(smem_u32(&bar[0]), 0x3);
        // drain: wait for the last commit of every slot
        if (mode == 0 || mode == 6) {
            for (int it = stages_total; it < stages_total + STAGES; it++) {
                const int s = it % STAGES;
                mbar_wait_cluster(smem_u32(&bar[s]), ((it / STAGES) - 1) & 1);
            }
        } else {
            // mode 1: every slot got stages_total/STAGES commits; mode 2: bar[0] one
            const int last = mode >= 2 ? 0 : (stages_total - 1) / STAGES;
            mbar_wait_cluster(smem_u32(&bar[mode >= 2 ? 0 : (stages_total - 1) % STAGES]), last & 1);
        }
        long long t1 = clock64();
        cycles[blockIdx.x / 2] = (unsigned long long)(t1 - t0);
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc_pair<512>(tm);
    }
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *d;
    cudaMalloc(&d, sizeof(unsigned long long) * sms);
    cudaFuncSetAttribute(k_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, STAGES * STAGE_BYTES);
    struct V { int nt, n, kk, mode; };
    // mode 0: 3-stage ring, wait on the commit STAGES back; 1: commit per stage,
    // never wait; 2: no commits until the end
    // 3: no commits, one stage buffer; 4: no commits, two stage buffers
    // 5: precomputed descriptors, no commits; 6: precomputed + commit/wait ring (CTA-scope wait)
    V vs[] = {{2, 256, 4, 6}, {2, 256, 2, 6}, {2, 256, 1, 6}, {2, 256, 4, 6}, {2, 256, 2, 6}};
    const int stages_total = 20000;
    for (auto &v : vs) {
        const uint32_t idesc = idesc_i8(256, v.n, true);
        float ms = 0;
        for (int rep = 0; rep < 2; rep++) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k_pair<<<sms / 2 * 2, 128, STAGES * STAGE_BYTES>>>(stages_total, v.nt, v.n, v.kk, v.mode, idesc, d);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        cudaError_t e = cudaGetLastError();
        unsigned long long h[128];
        cudaMemcpy(h, d, sizeof(unsigned long long) * (sms / 2), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < sms / 2; i++) avg += (double)h[i];
        avg /= sms / 2;
        const double macs_per_sm = (double)stages_total * v.kk * v.nt * 128.0 * v.n * 32;
        const double ops = 2.0 * macs_per_sm * (sms / 2 * 2);
        printf("mode=%d NT=%d N=%d K-steps/stage=%d: %.1f MAC/clk/SM, %.0f TOPS (%s), %.3f ms\n", v.mode, v.nt, v.n, v.kk,
               macs_per_sm / avg, ops / (ms * 1e-3) / 1e12, cudaGetErrorString(e), ms);
    }
    return 0;
}
