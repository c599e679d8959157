// synth_dev.cu -- device side of the synthetic CPA workload generator.
// Bit-identical to sy_traces() (synth.c): both evaluate synth_core.h.
// Input generation only; not part of the CPA product path.
#include <cuda_runtime.h>

#include "synth.h"
#include "synth_core.h"

namespace {

struct DevParams {
    sy_params p;
};

__global__ void k_columns(DevParams dp, int64_t *mu, uint16_t *leakmask)
{
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= dp.p.m) return;
    mu[j] = sy_mu_q32(&dp.p, j);
    uint16_t m = 0;
    for (int b = 0; b < 16; b++)
        if (dp.p.leak[b] == j) m |= (uint16_t)(1u << b);
    leakmask[j] = m;
}

template <int DT>
__global__ void k_traces(DevParams dp, const int32_t *__restrict__ gauss,
                         const uint8_t *__restrict__ leakv, const int64_t *__restrict__ mu,
                         const uint16_t *__restrict__ leakmask, int64_t i0, int64_t n,
                         void *out, int64_t ld)
{
    const int groups = (dp.p.m + 15) / 16;
    int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = n * groups;
    for (; gid < total; gid += (int64_t)gridDim.x * blockDim.x) {
        int64_t t = gid / groups;
        int g = (int)(gid % groups);
        uint64_t tkey = sy_trace_key(dp.p.seed, i0 + t);
        const uint8_t *lv = leakv + 16 * t;
        int j0 = g * 16;
        int cnt = min(16, dp.p.m - j0);
        int64_t vals[16];
#pragma unroll
        for (int q = 0; q < 16; q++) {
            int j = j0 + q;
            int64_t v = 0;
            if (q < cnt) {
                v = mu[j];
                uint16_t lm = leakmask[j];
                for (int b = 0; lm; b++, lm >>= 1)
                    if (lm & 1) v += dp.p.a_q32 * (int64_t)lv[b];
                v += (int64_t)gauss[sy_noise_u16(tkey, j)] * dp.p.sigma_q16;
            }
            vals[q] = v;
        }
        if (DT == SY_S8 || DT == SY_U8) {
            uint8_t *row = (uint8_t *)out + t * ld + j0;
            uint8_t bytes[16];
#pragma unroll
            for (int q = 0; q < 16; q++)
                bytes[q] = DT == SY_S8 ? (uint8_t)sy_to_s8(vals[q]) : sy_to_u8(vals[q]);
            if (cnt == 16 && ((uintptr_t)row & 15) == 0) {
                *(uint4 *)row = *(const uint4 *)bytes;
            } else {
                for (int q = 0; q < cnt; q++) row[q] = bytes[q];
            }
        } else {
            float *row = (float *)out + t * ld + j0;
            for (int q = 0; q < cnt; q++) row[q] = sy_to_f32(vals[q]);
        }
    }
}

}  // namespace

extern "C" int sy_dev_traces(const sy_params *p, int dtype, const int32_t *d_gauss,
                             const uint8_t *d_leakv, int64_t i0, int64_t n, void *d_out,
                             int64_t ld, void *stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    DevParams dp{*p};
    int64_t *mu = nullptr;
    uint16_t *lm = nullptr;
    if (cudaMallocAsync(&mu, sizeof(int64_t) * p->m, s) != cudaSuccess) return 1;
    if (cudaMallocAsync(&lm, sizeof(uint16_t) * p->m, s) != cudaSuccess) return 1;
    k_columns<<<(p->m + 255) / 256, 256, 0, s>>>(dp, mu, lm);
    int blocks = 148 * 16;
    if (dtype == SY_S8)
        k_traces<SY_S8><<<blocks, 256, 0, s>>>(dp, d_gauss, d_leakv, mu, lm, i0, n, d_out, ld);
    else if (dtype == SY_U8)
        k_traces<SY_U8><<<blocks, 256, 0, s>>>(dp, d_gauss, d_leakv, mu, lm, i0, n, d_out, ld);
    else
        k_traces<SY_F32><<<blocks, 256, 0, s>>>(dp, d_gauss, d_leakv, mu, lm, i0, n, d_out, ld);
    cudaFreeAsync(mu, s);
    cudaFreeAsync(lm, s);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
