// classsum.cu -- class-sum ("partition") accumulation of the cross term for the
// single-byte selection models HW_LAST / HW_FIRST.
//
// For these models the hypothesis of trace i, byte b, sub-key k depends on one
// text byte only: H = f(t_b(i) ^ k) with f(x) = HW(InvS[x]) (HW_LAST) or HW(S[x])
// (HW_FIRST).  Grouping the traces by x = t_b(i) gives, exactly,
//     sum_i H * W_ij = sum_x f(x ^ k) * S_b[x][j],   S_b[x][j] = sum_{i: t_b(i)=x} W_ij,
// so the 4096 MACs per (trace, sample) of the contraction become 16 adds (one
// per byte) plus a small 16 x 256 x 256 x M contraction.  The adds are done
// without atomics: the traces are counting-sorted by t_b per byte (k_cs_hist,
// k_cs_scan, k_cs_scatter), then one warp owns each (byte, class, 128-sample
// column tile) and sums that class's rows in registers (k_cs_sum).  All integer
// arithmetic is exact, so the result equals the tensor-core path bit for bit
// whatever the order of the sorted rows.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace cpa {
namespace {

// per-byte class counts: smem histogram per block, then one global add per bin
__global__ void __launch_bounds__(256) k_cs_hist(const uint8_t *__restrict__ tx, int64_t n, int32_t *__restrict__ cnt)
{
    __shared__ int32_t h[16 * 256];
    for (int i = threadIdx.x; i < 16 * 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int b = 0; b < 16; b++) atomicAdd(&h[b * 256 + tx[i * 16 + b]], 1);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 16 * 256; i += blockDim.x)
        if (h[i]) atomicAdd(&cnt[i], h[i]);
}

// exclusive scan of each byte's 256 counts: off[b][0..256], cursor[b][x] = off[b][x]
__global__ void __launch_bounds__(256) k_cs_scan(const int32_t *__restrict__ cnt, int32_t *__restrict__ off,
                                                 int32_t *__restrict__ cur)
{
    __shared__ int32_t s[256];
    const int b = blockIdx.x, x = threadIdx.x;
    s[x] = cnt[b * 256 + x];
    __syncthreads();
    for (int d = 1; d < 256; d <<= 1) {  // Hillis-Steele inclusive scan
        const int v = x >= d ? s[x - d] : 0;
        __syncthreads();
        s[x] += v;
        __syncthreads();
    }
    const int excl = s[x] - cnt[b * 256 + x];
    off[b * 257 + x] = excl;
    cur[b * 256 + x] = excl;
    if (x == 255) off[b * 257 + 256] = s[255];
}

// perm[b * pstride + pos] = trace index, rows of class x at [off[b][x], off[b][x+1])
__global__ void __launch_bounds__(256) k_cs_scatter(const uint8_t *__restrict__ tx, int64_t n, int64_t pstride,
                                                    int32_t *__restrict__ cur, int32_t *__restrict__ perm)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int b = 0; b < 16; b++) {
            const int pos = atomicAdd(&cur[b * 256 + tx[i * 16 + b]], 1);
            perm[(int64_t)b * pstride + pos] = (int32_t)i;
        }
    }
}

#ifndef CS_MLP
#define CS_MLP 8
#endif

#ifndef CS_LD
#define CS_LD 1
#endif
__device__ __forceinline__ uint4 ld_nc_v4(const void *p)
{
    uint4 v;
#if CS_LD == 1
    asm volatile("ld.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
#elif CS_LD == 2
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
#else
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
#endif
    return v;
}

// S_b[x][j] += class sums of nch chunks of traces for columns [jc0, jc0 + mc)
// (S row bx = 256 b + x, stride mc, int32: |S| <= 2^23 * 128).  One warp per
// (128-sample column tile, chunk, byte, class), in that order, so the warps in
// flight share one chunk x 128-byte column slice of W (~4 MB, whole 128-byte
// lines) and one 2 MB tile of S in L2, and the rows they gather span few 2 MB
// pages (TLB).  Chunk ch's rows are W + (ch * clen + perm) * ld, its sorted
// order perm + ch * 16 * clen + b * clen, its class offsets off + ch * 16 * 257.
// Lane (r = lane / 8, c = lane % 8) reads 16 samples of rows p0 + r, p0 + r + 4,
// ... of the class;
// bytes are biased to u8 (s8 ^ 0x80) and summed as packed 16-bit pairs (<= 256
// rows of 255 per window), flushed to int32.
__global__ void __launch_bounds__(256) k_cs_sum(const uint8_t *__restrict__ W, int64_t ld, int32_t jc0, int32_t mc,
                                                int32_t sgn, const int32_t *__restrict__ perm, int32_t nch,
                                                int64_t clen, const int32_t *__restrict__ off,
                                                int32_t *__restrict__ S)
{
    const int lane = threadIdx.x & 31;
    const int r = lane >> 3, c = lane & 7;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int ntile = (mc + 127) / 128;
    const uint32_t bias = sgn ? 0x80808080u : 0u;
    for (int64_t item = gw; item < (int64_t)ntile * nch * 4096; item += nw) {
        const int tile = (int)(item / ((int64_t)nch * 4096));
        const int ch = (int)((item >> 12) % nch), bx = (int)(item & 4095), b = bx >> 8;
        const int jl = tile * 128 + c * 16;
        const bool live = jl < mc;  // this lane's 16 columns exist (16-aligned: reads stay inside ld)
        const int32_t *of = off + ch * 16 * 257 + b * 257 + (bx & 255);
        const int p0 = of[0], p1 = of[1];
        const int32_t *pb = perm + ((int64_t)ch * 16 + b) * clen;
        const uint8_t *wc = W + (int64_t)ch * clen * ld + jc0 + jl;
        int32_t full[16];
#pragma unroll
        for (int e = 0; e < 16; e++) full[e] = 0;
        uint32_t lo[4] = {0, 0, 0, 0}, hi[4] = {0, 0, 0, 0};
        int cnt = 0, win = 0;
        auto flush = [&]() {
#pragma unroll
            for (int q = 0; q < 4; q++) {
                full[4 * q + 0] += (int32_t)(lo[q] & 0xffffu);
                full[4 * q + 2] += (int32_t)(lo[q] >> 16);
                full[4 * q + 1] += (int32_t)(hi[q] & 0xffffu);
                full[4 * q + 3] += (int32_t)(hi[q] >> 16);
                lo[q] = hi[q] = 0;
            }
        };
        if (live) {
            // CS_MLP rows per lane in flight: their indices first, then all the
            // row loads, then the adds (the loop is latency-bound otherwise)
            for (int p = p0 + r; p < p1; p += 4 * CS_MLP) {
                int64_t idx[CS_MLP];
#pragma unroll
                for (int u = 0; u < CS_MLP; u++) idx[u] = (p + 4 * u < p1) ? pb[p + 4 * u] : -1;
                uint4 wv[CS_MLP];
#pragma unroll
                for (int u = 0; u < CS_MLP; u++)
                    wv[u] = idx[u] >= 0 ? ld_nc_v4(wc + idx[u] * ld) : make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int u = 0; u < CS_MLP; u++) {
                    const uint32_t ws[4] = {wv[u].x ^ bias, wv[u].y ^ bias, wv[u].z ^ bias, wv[u].w ^ bias};
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        lo[q] += ws[q] & 0x00ff00ffu;          // bytes 0, 2
                        hi[q] += (ws[q] >> 8) & 0x00ff00ffu;   // bytes 1, 3
                    }
                }
                cnt += CS_MLP;  // a padded (zero) row adds 128 per byte biased (s8), 0 after the correction
                win += CS_MLP;
                if (win >= 256 - CS_MLP) {
                    flush();
                    win = 0;
                }
            }
            flush();
        }
        if (sgn) {
#pragma unroll
            for (int e = 0; e < 16; e++) full[e] -= 128 * cnt;
        }
#pragma unroll
        for (int e = 0; e < 16; e++) {
            full[e] += __shfl_xor_sync(0xffffffffu, full[e], 8);
            full[e] += __shfl_xor_sync(0xffffffffu, full[e], 16);
        }
        if (r == 0 && live) {
            int32_t *dst = S + (int64_t)bx * mc + jl;
#pragma unroll
            for (int e = 0; e < 16; e++)  // the chunks' warps of one (tile, class) run concurrently
                if (jl + e < mc) atomicAdd(dst + e, full[e]);
        }
    }
}

// sum_hw[256 b + k][jc0 + j] += sum_x f(x ^ k) * S_b[x][j]: block = (32-column
// tile, byte b), thread = sub-key k, exact int64 (IMAD.WIDE).
__global__ void __launch_bounds__(256) k_cs_contract(const int32_t *__restrict__ S, int32_t mc, int32_t jc0,
                                                     int32_t M, const uint8_t *__restrict__ f,
                                                     int64_t *__restrict__ hw)
{
    __shared__ __align__(16) int32_t s[256][32];
    __shared__ int32_t fs[256];
    const int b = blockIdx.y, j0 = blockIdx.x * 32, k = threadIdx.x;
    fs[k] = f[k];
    for (int t = threadIdx.x; t < 256 * 32; t += blockDim.x) {
        const int x = t >> 5, e = t & 31;
        s[x][e] = (j0 + e < mc) ? S[(int64_t)(b * 256 + x) * mc + j0 + e] : 0;
    }
    __syncthreads();
    int64_t acc[32];
#pragma unroll
    for (int e = 0; e < 32; e++) acc[e] = 0;
#pragma unroll 2
    for (int x = 0; x < 256; x++) {
        const int fv = fs[x ^ k];
        const int4 *row = (const int4 *)s[x];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int4 v = row[q];
            acc[4 * q + 0] += (int64_t)v.x * fv;
            acc[4 * q + 1] += (int64_t)v.y * fv;
            acc[4 * q + 2] += (int64_t)v.z * fv;
            acc[4 * q + 3] += (int64_t)v.w * fv;
        }
    }
    int64_t *dst = hw + (int64_t)(b * 256 + k) * M + jc0 + j0;
#pragma unroll
    for (int e = 0; e < 32; e++)
        if (j0 + e < mc) dst[e] += acc[e];
}

}  // namespace

int64_t cs_perm_words(int64_t n) { return 16 * n; }

cudaError_t launch_cs_sort(const uint8_t *d_texts, int64_t n, int64_t pstride, int32_t *d_cnt, int32_t *d_off,
                           int32_t *d_cur, int32_t *d_perm, int num_sms, cudaStream_t s, int *launches)
{
    cudaError_t e = cudaMemsetAsync(d_cnt, 0, sizeof(int32_t) * 4096, s);
    if (e != cudaSuccess) return e;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 4 * num_sms) blocks = 4 * num_sms;
    if (blocks < 1) blocks = 1;
    k_cs_hist<<<(int)blocks, 256, 0, s>>>(d_texts, n, d_cnt);
    k_cs_scan<<<16, 256, 0, s>>>(d_cnt, d_off, d_cur);
    int64_t sb = (n + 255) / 256;
    if (sb > 16 * num_sms) sb = 16 * num_sms;
    if (sb < 1) sb = 1;
    k_cs_scatter<<<(int)sb, 256, 0, s>>>(d_texts, n, pstride, d_cur, d_perm);
    if (launches) *launches += 3;
    return cudaGetLastError();
}

cudaError_t launch_cs_sum(const uint8_t *d_w, int64_t ld, int32_t nch, int64_t clen, int32_t jc0, int32_t mc,
                          bool w_signed, const int32_t *d_perm, const int32_t *d_off, int32_t *d_S, int num_sms,
                          cudaStream_t s, int *launches)
{
    const int64_t items = (int64_t)((mc + 127) / 128) * nch * 4096;
    int64_t blocks = (items + 7) / 8;  // 8 warps per block
    if (blocks > 8 * num_sms) blocks = 8 * num_sms;
    k_cs_sum<<<(int)blocks, 256, 0, s>>>(d_w, ld, jc0, mc, w_signed ? 1 : 0, d_perm, nch, clen, d_off, d_S);
    if (launches) *launches += 1;
    return cudaGetLastError();
}

cudaError_t launch_cs_contract(const int32_t *d_S, int32_t M, int32_t jc0, int32_t mc, const uint8_t *d_f,
                               int64_t *d_hw, cudaStream_t s, int *launches)
{
    dim3 g((mc + 31) / 32, 16);
    k_cs_contract<<<g, 256, 0, s>>>(d_S, mc, jc0, M, d_f, d_hw);
    if (launches) *launches += 1;
    return cudaGetLastError();
}

}  // namespace cpa
