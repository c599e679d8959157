// kernels.cu -- the HBM/latency-bound steps of the path:
//   a3 model sums      sum_i H_i, sum_i H_i^2 per (b, k)            [P:75]
//   a4 trace moments   sum_i W_ij, sum_i W_ij^2 per sample j        [P:79]
//   a8 finalize        Eq. (1) [P:69] in fp64 + max |rho| per (b,k) [P:83]
//   a9 phase 4         per-byte ranking / best sub-key              [P:87]
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "kernels.h"

namespace cpa {
namespace {

__device__ __forceinline__ int shiftrows_src(int b) { return (b & 3) + 4 * (((b >> 2) + (b & 3)) & 3); }

// ---------------------------------------------------------------------------
// a3: one block = 16 warps (warp = key byte b), lane owns keys lane + 32 q.
// H = V[c_s][c_b ^ k]; per-thread int32 partials, one int64 atomic per (b,k).
// ---------------------------------------------------------------------------
constexpr int MS_THREADS = 512;
constexpr int MS_CHUNK = 2048;  // max traces per block (int32-exact: 64 * 2048)
constexpr int MS_MIN_BLOCKS = 296;  // 2 per SM: spread small N over the GPU
constexpr int MS_STAGE = 256;   // traces staged in smem at a time

template <typename Acc>
__global__ void __launch_bounds__(MS_THREADS)
k_modelsums(const uint8_t *__restrict__ texts, int64_t n, int chunk, const uint8_t *__restrict__ vtab,
            Acc *sum_h, Acc *sum_h2, Acc *count)
{
    extern __shared__ uint8_t sm[];
    uint8_t *vs = sm;              // 64 KB
    uint8_t *ts = sm + 65536;      // MS_STAGE x 16
    for (int i = threadIdx.x; i < 4096; i += MS_THREADS) ((uint4 *)vs)[i] = ((const uint4 *)vtab)[i];
    const int b = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sb = shiftrows_src(b);
    int32_t s1[8], s2[8];
#pragma unroll
    for (int q = 0; q < 8; q++) s1[q] = s2[q] = 0;
    const int64_t i0 = (int64_t)blockIdx.x * chunk;
    const int64_t i1 = min(n, i0 + chunk);
    for (int64_t base = i0; base < i1; base += MS_STAGE) {
        __syncthreads();
        const int cnt = (int)min((int64_t)MS_STAGE, i1 - base);
        for (int t = threadIdx.x; t < cnt; t += MS_THREADS)
            ((uint4 *)ts)[t] = ((const uint4 *)texts)[base + t];
        __syncthreads();
        for (int t = 0; t < cnt; t++) {
            const uint32_t cb = ts[t * 16 + b], cs = ts[t * 16 + sb];
            const uint8_t *vrow = vs + cs * 256;
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const int32_t h = vrow[cb ^ (uint32_t)(lane + 32 * q)];
                s1[q] += h;
                s2[q] += h * h;
            }
        }
    }
#pragma unroll
    for (int q = 0; q < 8; q++) {
        const int hidx = b * 256 + lane + 32 * q;
        if constexpr (std::is_integral<Acc>::value) {
            atomicAdd((unsigned long long *)&sum_h[hidx], (unsigned long long)(long long)s1[q]);
            atomicAdd((unsigned long long *)&sum_h2[hidx], (unsigned long long)(long long)s2[q]);
        } else {
            atomicAdd(&sum_h[hidx], (Acc)s1[q]);
            atomicAdd(&sum_h2[hidx], (Acc)s2[q]);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if constexpr (std::is_integral<Acc>::value)
            atomicAdd((unsigned long long *)count, (unsigned long long)n);
        else
            atomicAdd(count, (Acc)n);
    }
}

// ---------------------------------------------------------------------------
// a4: HBM-bound single pass.  Work item = (16-sample column group, `rows`-row
// chunk), flattened so no thread idles on the ragged column edge.  Samples are
// biased to u = w + 128 (s8) so sum u accumulates in packed 16-bit lanes (two
// bytes per IADD, flushed every 256 rows) and sum u^2 in uint32 (exact:
// 65025 * rows < 2^32 for rows <= 2^16); sum w = sum u - 128 n, sum w^2 = sum u^2 - 256 sum u
// + 16384 n, all in exact integers.
// ---------------------------------------------------------------------------
constexpr int MO_THREADS = 256;
constexpr int MO_MAX_ROWS = 1 << 16;  // uint32 exactness of sum u^2
constexpr int MO_UNROLL = 8;

__device__ __forceinline__ uint4 ld_stream16(const void *p)
{
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

template <bool SIGNED>
__global__ void __launch_bounds__(MO_THREADS)
k_moments_i8(const uint8_t *__restrict__ w, int64_t ld, int64_t n, int32_t M, int64_t items, int64_t rows,
             unsigned long long *sum_w, unsigned long long *sum_w2)
{
    const int groups = (M + 15) >> 4;
    const int64_t item = (int64_t)blockIdx.x * MO_THREADS + threadIdx.x;
    if (item >= items) return;
    const int g = (int)(item % groups);
    const int64_t r0 = (item / groups) * rows;
    const int64_t r1 = min(n, r0 + rows);
    const int j0 = g * 16;
    uint32_t p1[8];   // packed 16-bit partial sums of u, lanes = (byte 0,2) / (1,3) of each word
    uint32_t s1[16];  // flushed sums of u
    uint32_t s2[16];  // sums of u^2
#pragma unroll
    for (int q = 0; q < 16; q++) s1[q] = s2[q] = 0;
#pragma unroll
    for (int q = 0; q < 8; q++) p1[q] = 0;
    const uint8_t *col = w + j0;
    const uint32_t bias = SIGNED ? 0x80808080u : 0u;
    int64_t r = r0;
    int since_flush = 0;
    auto consume = [&](uint4 v) {
        const uint32_t ws[4] = {v.x ^ bias, v.y ^ bias, v.z ^ bias, v.w ^ bias};
#pragma unroll
        for (int k = 0; k < 4; k++) {
            p1[2 * k] += ws[k] & 0x00FF00FFu;
            p1[2 * k + 1] += (ws[k] >> 8) & 0x00FF00FFu;
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const uint32_t u = (ws[k] >> (8 * e)) & 0xFF;
                s2[4 * k + e] += u * u;
            }
        }
    };
    auto flush = [&]() {
#pragma unroll
        for (int k = 0; k < 4; k++) {
            s1[4 * k + 0] += p1[2 * k] & 0xFFFF;
            s1[4 * k + 2] += p1[2 * k] >> 16;
            s1[4 * k + 1] += p1[2 * k + 1] & 0xFFFF;
            s1[4 * k + 3] += p1[2 * k + 1] >> 16;
            p1[2 * k] = p1[2 * k + 1] = 0;
        }
    };
    for (; r + MO_UNROLL <= r1; r += MO_UNROLL) {
        uint4 v[MO_UNROLL];
#pragma unroll
        for (int u = 0; u < MO_UNROLL; u++) v[u] = ld_stream16(col + (r + u) * ld);
#pragma unroll
        for (int u = 0; u < MO_UNROLL; u++) consume(v[u]);
        since_flush += MO_UNROLL;
        if (since_flush >= 256) {  // 16-bit lanes hold <= 257 * 255
            flush();
            since_flush = 0;
        }
    }
    flush();
    for (; r < r1; r++) consume(ld_stream16(col + r * ld));  // < MO_UNROLL rows
    flush();
    const int64_t nrows = r1 - r0;
#pragma unroll
    for (int q = 0; q < 16; q++) {
        if (j0 + q < M) {
            long long sw = (long long)s1[q], sw2 = (long long)s2[q];
            if (SIGNED) {
                sw2 = sw2 - 256LL * sw + 16384LL * nrows;  // sum (u-128)^2
                sw = sw - 128LL * nrows;                   // sum (u-128)
            }
            atomicAdd(&sum_w[j0 + q], (unsigned long long)sw);
            atomicAdd(&sum_w2[j0 + q], (unsigned long long)sw2);
        }
    }
}

// ---------------------------------------------------------------------------
// a8: Eq. (1) with the fixed, FMA-free fp64 sequence of DESIGN.md:
//   num = N*S_hw - S_h*S_w ; dw = N*S_w2 - S_w^2 ; dh = N*S_h2 - S_h^2 (int64)
//   rho = (double)num / (sqrt((double)dw) * sqrt((double)dh)), 0 if dw or dh
//   is 0, clamped to [-1, 1].  Host guarantees N <= 2^23 so all fit int64.
// ---------------------------------------------------------------------------
__global__ void k_sqrt_dw_i8(const int64_t *__restrict__ sw, const int64_t *__restrict__ sw2,
                             const int64_t *__restrict__ count, int32_t M, double *out)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= M) return;
    const int64_t n = *count;
    const int64_t dw = n * sw2[j] - sw[j] * sw[j];
    const double d = __dsqrt_rn(__ll2double_rn(dw));
    out[j] = d;
    out[M + j] = d != 0.0 ? __drcp_rn(d) : 0.0;  // for the no-rho filter of k_finalize_rows
}

struct Best {
    double v;   // |rho|
    double r;   // signed rho
    int j;
};
__device__ __forceinline__ bool better(const Best &a, const Best &b)
{
    return a.v > b.v || (a.v == b.v && a.j < b.j);
}
__device__ __forceinline__ Best warp_best(Best x)
{
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        Best y;
        y.v = __shfl_xor_sync(0xffffffffu, x.v, off);
        y.r = __shfl_xor_sync(0xffffffffu, x.r, off);
        y.j = __shfl_xor_sync(0xffffffffu, x.j, off);
        if (better(y, x)) x = y;
    }
    return x;
}

constexpr int FIN_THREADS = 256;

__device__ __forceinline__ void block_best_store(Best best, int h, const FinalizeOut &o)
{
    __shared__ Best red[FIN_THREADS / 32];
    best = warp_best(best);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x < 32) {
        Best x = threadIdx.x < FIN_THREADS / 32 ? red[threadIdx.x] : Best{-1.0, 0.0, 0x7fffffff};
        x = warp_best(x);
        if (threadIdx.x == 0) {
            o.maxabs[h] = x.v;
            o.argmax[h] = x.j + o.col0;
            o.peak[h] = x.r;
        }
    }
}

// ---------------------------------------------------------------------------
// a8: one block = R hypothesis rows x all M samples (R = 1 by default, see
// launch_fin).  Per column pair a thread loads the per-sample terms (sqrt(dw),
// sum W: L2-resident, shared by all 4096 rows) once for its R rows; U column
// pairs of 16-byte sum_hw loads are in flight per thread.  Every cell is the
// fixed, FMA-free Eq. (1) sequence of DESIGN.md (fin_cell), so rho equals the
// oracle's rho_B bit for bit.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double fin_cell(int64_t v, int64_t n, int64_t s_h, int64_t s_w, double den_w, double den_h)
{
    double r = 0.0;
    if (den_w != 0.0 && den_h != 0.0) {
        const int64_t num = n * v - s_h * s_w;
        r = __ddiv_rn(__ll2double_rn(num), __dmul_rn(den_w, den_h));
        r = fmin(1.0, fmax(-1.0, r));
    }
    return r;
}
__device__ __forceinline__ double fin_cell(double v, double n, double s_h, double s_w, double den_w, double den_h)
{
    double r = 0.0;
    if (den_w != 0.0 && den_h != 0.0) {
        const double num = __dsub_rn(__dmul_rn(n, v), __dmul_rn(s_h, s_w));
        r = __ddiv_rn(num, __dmul_rn(den_w, den_h));
        r = fmin(1.0, fmax(-1.0, r));
    }
    return r;
}
__device__ __forceinline__ double fin_den_h(int64_t n, int64_t s_h, int64_t s_h2)
{
    return __dsqrt_rn(__ll2double_rn(n * s_h2 - s_h * s_h));
}
__device__ __forceinline__ double fin_den_h(double n, double s_h, double s_h2)
{
    const double dh = __dsub_rn(__dmul_rn(n, s_h2), __dmul_rn(s_h, s_h));
    return dh > 0.0 ? __dsqrt_rn(dh) : 0.0;
}
template <typename T> struct Pair2;
template <> struct Pair2<int64_t> { using type = longlong2; };
template <> struct Pair2<int32_t> { using type = int2; };
// VV consecutive sum_hw elements loaded with ONE evict-first vector load (8 or 16 bytes)
template <int BYTES> struct LdT;
template <> struct LdT<8> { using type = int2; };
template <> struct LdT<16> { using type = int4; };
template <typename TH, int VV> struct alignas(VV * sizeof(TH)) RowV { TH e[VV]; };
template <typename TH, int VV>
__device__ __forceinline__ RowV<TH, VV> ldcs_row(const TH *p)
{
    using L = typename LdT<VV * sizeof(TH)>::type;
    const L q = __ldcs((const L *)p);
    RowV<TH, VV> r;
    memcpy(&r, &q, sizeof(q));
    return r;
}
template <> struct Pair2<double> { using type = double2; };

// Without rho output (streamed checkpoints, sharded maxima) only max|rho| and
// its argmax are needed, so most cells skip the fp64 division (the kernel is
// fp64-issue-bound, not HBM-bound, when it writes nothing): with
// a_j = |num_j| * fl(1/den_w_j) (one DMUL; den_h is the same for the whole row)
// and the exact value rho_j = fl(num_j / fl(den_w_j den_h)), rho_j den_h / a_j
// lies in [1 - 4.01u, 1 + 4.01u] (u = 2^-53: two roundings on each side), so a
// cell with a_j < a_best (1 - 2^-48) has |rho_j| < |rho_best| strictly (and the
// clamp to 1 keeps <=); such a cell, at a larger j than the thread's best, can
// neither beat nor tie-break it.  Every other cell is computed exactly as above,
// so max|rho|, argmax and the signed peak are bit-identical to the full kernel.
constexpr double kFinSkip = 1.0 - 3.552713678800501e-15;  // 1 - 2^-48

// TH: element type of the sum_hw rows (T, or int32 for narrow sums, widened on load)
#ifndef FIN_MAXIMA_MINB
#define FIN_MAXIMA_MINB 5  // 5 resident blocks with 2 row loads in flight (tools/gpu_ab_w.sh)
#endif
template <int U, typename T, typename TH = T, int MINB = FIN_MAXIMA_MINB>
__global__ void __launch_bounds__(FIN_THREADS, MINB)
k_finalize_maxima(const TH *__restrict__ hw, const T *__restrict__ sw, const T *__restrict__ sh,
                  const T *__restrict__ sh2, const T *__restrict__ count, const double *__restrict__ sqrt_dw,
                  int32_t M, FinalizeOut o)
{
    const int h = o.h0 + blockIdx.x;
    const T n = *count;
    const T s_h = sh[h];
    const double den_h = fin_den_h(n, s_h, sh2[h]);
    const TH *row = hw + (int64_t)h * M;
    const double *rcp_w = sqrt_dw + M;
    // Skip threshold shared by the block (= the row): the largest a_best (1 - 2^-48)
    // any thread has seen.  A cell below it is strictly below THAT thread's best
    // cell, so it can be neither the row's maximum nor tie with it, whichever
    // thread and sample it belongs to.  (A per-thread threshold let each lane's
    // first few, still-rising maxima through: nearly every warp step ran some
    // lane's fp64 division, and the kernel was issue-bound, ~3 TB/s.)  Positive
    // doubles order as their bit patterns: the maximum is an integer atomicMax.
    __shared__ unsigned long long s_thr;
    if (threadIdx.x == 0) s_thr = 0ull;
    __syncthreads();
    Best best{-1.0, 0.0, 0x7fffffff};
    double thr = 0.0;  // this thread's copy of the block threshold (refreshed per group)
    // sqrt(dw_j) is only needed by the (now rare) cells that pass the filter:
    // loaded there (hoisting the group's per-sample loads ahead of its cells
    // measured slower: 88 registers, half the resident blocks)
    auto visit = [&](T v, int j, double rw, T s_w) {
        double num;
        if constexpr (std::is_integral<T>::value) num = __ll2double_rn(n * v - s_h * s_w);
        else num = __dsub_rn(__dmul_rn(n, v), __dmul_rn(s_h, s_w));
        const double a = __dmul_rn(fabs(num), rw);
        if (a < thr) return;  // strictly below some thread's best: skip the division
        const double x = fin_cell(v, n, s_h, s_w, sqrt_dw[j], den_h);
        const double ax = fabs(x);
        if (ax > best.v) {
            best = Best{ax, x, j};
            const double t = __dmul_rn(a, kFinSkip);
            if (t > thr) {
                thr = t;
                atomicMax(&s_thr, (unsigned long long)__double_as_longlong(t));
            }
        }
    };
    auto refresh = [&] {
        const double t = __longlong_as_double((long long)*(volatile unsigned long long *)&s_thr);
        if (t > thr) thr = t;
    };
    int j = 0;
    // VV samples per row load: 16 bytes (2 int64 / fp64, 4 int32), else 8 bytes
    // (int32 rows with M % 4 == 2); the ragged last group is predicated, not a
    // loop of single samples: each of its iterations would wait out a full load
    // latency (per block: ~6 us at any M, 25% of the kernel at M = 20000)
    auto vec_path = [&](auto vc) {
        constexpr int VV = decltype(vc)::value;
        using T2 = typename Pair2<T>::type;
        const int MV = M / VV;
        for (int p0 = threadIdx.x; p0 < MV; p0 += U * FIN_THREADS) {
            RowV<TH, VV> v[U];
#pragma unroll
            for (int u = 0; u < U; u++)
                if (p0 + u * FIN_THREADS < MV) v[u] = ldcs_row<TH, VV>(row + (int64_t)(p0 + u * FIN_THREADS) * VV);
            refresh();
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int p = p0 + u * FIN_THREADS;
                if (p >= MV) break;
#pragma unroll
                for (int e = 0; e < VV; e += 2) {
                    const int jj = VV * p + e;
                    const double2 rw = *(const double2 *)(rcp_w + jj);
                    const T2 swp = *(const T2 *)(sw + jj);
                    visit((T)v[u].e[e], jj, rw.x, swp.x);
                    visit((T)v[u].e[e + 1], jj + 1, rw.y, swp.y);
                }
            }
        }
        j = M;
    };
    constexpr int V16 = 16 / (int)sizeof(TH);
    if (M % V16 == 0) vec_path(std::integral_constant<int, V16>{});
    else if (V16 > 2 && (M & 1) == 0) vec_path(std::integral_constant<int, 2>{});
    for (j += threadIdx.x; j < M; j += FIN_THREADS) visit((T)row[j], j, rcp_w[j], sw[j]);
    block_best_store(best, h, o);
}

template <int R, int U, typename T, typename TH = T>
__global__ void __launch_bounds__(FIN_THREADS)
k_finalize_rows(const TH *__restrict__ hw, const T *__restrict__ sw, const T *__restrict__ sh,
                const T *__restrict__ sh2, const T *__restrict__ count, const double *__restrict__ sqrt_dw, int32_t M,
                FinalizeOut o)
{
    using T2 = typename Pair2<T>::type;
    const int hb = o.h0 + blockIdx.x * R;
    const int nr = min(R, o.h1 - hb);
    const T n = *count;
    T s_h[R];
    double den_h[R];
    Best best[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
        const int h = hb + (r < nr ? r : 0);
        s_h[r] = sh[h];
        den_h[r] = fin_den_h(n, s_h[r], sh2[h]);
        best[r] = Best{-1.0, 0.0, 0x7fffffff};
    }
    const TH *row0 = hw + (int64_t)hb * M;
    double *rrow0 = o.rho ? o.rho + (int64_t)(hb - o.h0) * M : nullptr;
    auto keep = [&](int r, double x, int j) {
        const double a = fabs(x);
        if (a > best[r].v) best[r] = Best{a, x, j};  // j ascending per thread: lowest-j ties
    };
    int j = 0;
    // VV samples per row load, as in k_finalize_maxima; rho rows 16-byte aligned
    auto vec_path = [&](auto vc) {
        constexpr int VV = decltype(vc)::value;
        const int MV = M / VV;
        for (int p0 = threadIdx.x; p0 < MV; p0 += U * FIN_THREADS) {  // ragged last group predicated
            RowV<TH, VV> v[U][R];
#pragma unroll
            for (int u = 0; u < U; u++)
#pragma unroll
                for (int r = 0; r < R; r++)
                    if (r < nr && p0 + u * FIN_THREADS < MV)
                        v[u][r] = ldcs_row<TH, VV>(row0 + (int64_t)r * M + (int64_t)(p0 + u * FIN_THREADS) * VV);
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int p = p0 + u * FIN_THREADS;
                if (p >= MV) break;
#pragma unroll
                for (int e = 0; e < VV; e += 2) {
                    const int jj = VV * p + e;
                    const double2 dw = *(const double2 *)(sqrt_dw + jj);
                    const T2 swp = *(const T2 *)(sw + jj);
#pragma unroll
                    for (int r = 0; r < R; r++) {
                        if (r >= nr) break;
                        double2 x;
                        x.x = fin_cell((T)v[u][r].e[e], n, s_h[r], swp.x, dw.x, den_h[r]);
                        x.y = fin_cell((T)v[u][r].e[e + 1], n, s_h[r], swp.y, dw.y, den_h[r]);
                        keep(r, x.x, jj);
                        keep(r, x.y, jj + 1);
                        if (rrow0) __stcs((double2 *)(rrow0 + (int64_t)r * M + jj), x);
                    }
                }
            }
        }
        j = M;
    };
    if (((uintptr_t)o.rho & 15) == 0) {
        constexpr int V16 = 16 / (int)sizeof(TH);
        if (M % V16 == 0) vec_path(std::integral_constant<int, V16>{});
        else if (V16 > 2 && (M & 1) == 0) vec_path(std::integral_constant<int, 2>{});
    }
    for (j += threadIdx.x; j < M; j += FIN_THREADS) {
#pragma unroll
        for (int r = 0; r < R; r++) {
            if (r >= nr) break;
            const double x = fin_cell((T)row0[(int64_t)r * M + j], n, s_h[r], sw[j], sqrt_dw[j], den_h[r]);
            keep(r, x, j);
            if (rrow0) rrow0[(int64_t)r * M + j] = x;
        }
    }
    // per-row block reductions (the shared staging array is reused: barrier between rows)
    __shared__ Best red[R][FIN_THREADS / 32];
#pragma unroll
    for (int r = 0; r < R; r++) {
        const Best b = warp_best(best[r]);
        if ((threadIdx.x & 31) == 0) red[r][threadIdx.x >> 5] = b;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int r = warp; r < nr; r += FIN_THREADS / 32) {
        Best x = lane < FIN_THREADS / 32 ? red[r][lane] : Best{-1.0, 0.0, 0x7fffffff};
        x = warp_best(x);
        if (lane == 0) {
            o.maxabs[hb + r] = x.v;
            o.argmax[hb + r] = x.j + o.col0;
            o.peak[hb + r] = x.r;
        }
    }
}

// float path: all sums fp64 (same shape as the int accumulator)
// The float sums are of the centred samples c = w - o_j (cpa_set_offsets).  dw
// is offset-invariant, but SPEC's degenerate-column rule [S:293] compares it
// with the RAW second moment: dw <= 1e-12 * N * sum w^2 -> rho = 0 (marked by a
// 0 here), with sum w^2 = sum c^2 + 2 o_j sum c + N o_j^2 rebuilt from the
// centred sums (the same decision as the oracle's raw-sum test, or_rho_eq1_f64_grid)
__global__ void k_sqrt_dw_f64(const double *__restrict__ sw, const double *__restrict__ sw2,
                              const double *__restrict__ count, const float *__restrict__ offset, int32_t M,
                              double *out)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= M) return;
    const double n = *count;
    const double dw = __dsub_rn(__dmul_rn(n, sw2[j]), __dmul_rn(sw[j], sw[j]));
    const double o = offset ? (double)offset[j] : 0.0;
    const double raw2 = sw2[j] + o * (2.0 * sw[j] + n * o);
    const double d = (dw > 1e-12 * n * raw2) ? __dsqrt_rn(dw) : 0.0;
    out[j] = d;
    out[M + j] = d != 0.0 ? __drcp_rn(d) : 0.0;  // for the no-rho filter of k_finalize_rows
}

// ---------------------------------------------------------------------------
// a9: per byte b (block), thread k: rank = 1 + #{k' better than k}
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_phase4(FinalizeOut o)
{
    __shared__ double m[256];
    const int b = blockIdx.x, k = threadIdx.x;
    m[k] = o.maxabs[b * 256 + k];
    __syncthreads();
    const double mk = m[k];
    int r = 1;
    for (int k2 = 0; k2 < 256; k2++) {
        const double a = m[k2];
        r += (a > mk || (a == mk && k2 < k)) ? 1 : 0;
    }
    o.rank[b * 256 + k] = r;
    if (r == 1) {
        o.best[b] = k;
        o.best[16 + b] = o.argmax[b * 256 + k];
        o.best_rho[b] = o.peak[b * 256 + k];
    }
}

// ---------------------------------------------------------------------------
// Phase-3 merge over sample-axis shards: per hypothesis h, the shard with the
// largest max|rho| wins, ties to the lowest global sample index [S:298] (the
// shards' argmax already carry their column base).  In place into shard 0.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_merge_shards(int32_t G, double *maxabs, int32_t *argmax, double *peak)
{
    const int h = blockIdx.x * blockDim.x + threadIdx.x;
    if (h >= 4096) return;
    double v = maxabs[h], r = peak[h];
    int32_t j = argmax[h];
    for (int g = 1; g < G; g++) {
        const double v2 = maxabs[(int64_t)g * 4096 + h];
        const int32_t j2 = argmax[(int64_t)g * 4096 + h];
        if (v2 > v || (v2 == v && j2 < j)) {
            v = v2;
            j = j2;
            r = peak[(int64_t)g * 4096 + h];
        }
    }
    maxabs[h] = v;
    argmax[h] = j;
    peak[h] = r;
}

// ---------------------------------------------------------------------------
// a3 for large N: H(b,k) depends on a trace only through the byte pair
// (c_b, c_s) = (c[b], c[SR(b)]), so
//   sum_i H = sum_{x,y} cnt_b[x][y] * V[y][x ^ k],  sum_i H^2 likewise with V^2,
// with cnt_b the (exact, integer) histogram of the pairs: 16 N atomics plus a
// fixed 16 x 256 x 65536 contraction instead of 4096 N table lookups.
// ---------------------------------------------------------------------------
__global__ void k_texthist(const uint8_t *__restrict__ texts, int64_t n, uint32_t *hist)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint4 t4 = __ldg((const uint4 *)texts + i);
        const uint32_t w[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
        for (int b = 0; b < 16; b++) {
            const int sb = shiftrows_src(b);
            const uint32_t cb = (w[b >> 2] >> (8 * (b & 3))) & 0xFF;
            const uint32_t cs = (w[sb >> 2] >> (8 * (sb & 3))) & 0xFF;
            atomicAdd(&hist[(b << 16) | (cb << 8) | cs], 1u);
        }
    }
}

constexpr int HC_X = 8;  // histogram rows (x = c_b) per block (4 and 16 measured the same)
// Thread z owns column z of V (one byte of V[y][z] per y, reused for the HC_X
// rows of the block) and accumulates, for each row x, the key k = x ^ z; the
// counts are staged transposed, [y][x], so one 16-byte broadcast load gives 4
// rows' counts.  3 shared loads per 2 x HC_X multiply-adds (the per-(x, k)
// layout needed 2 per 2: the contraction was shared-load-bound).  For a fixed
// row x, z -> x ^ z is a bijection, so the per-key sums go through shared
// memory without atomics (one row at a time), then one int64 atomic per key.
template <typename Acc>
__global__ void __launch_bounds__(256)
k_hist_contract(const uint32_t *__restrict__ hist, const uint8_t *__restrict__ vtab, Acc *sum_h, Acc *sum_h2,
                Acc *count, int64_t n)
{
    extern __shared__ __align__(16) uint8_t sm[];
    uint8_t *vs = sm;                                // 64 KB: V[y][z]
    uint32_t *ct = (uint32_t *)(sm + 65536);         // 256 x HC_X counts, [y][x]
    __shared__ uint32_t sk1[256], sk2[256];
    const int b = blockIdx.y, x0 = blockIdx.x * HC_X, z = threadIdx.x;
    for (int i = threadIdx.x; i < 4096; i += 256) ((uint4 *)vs)[i] = ((const uint4 *)vtab)[i];
    for (int i = threadIdx.x; i < HC_X * 256; i += 256) {
        const int xx = i >> 8, y = i & 255;  // coalesced read of row x0 + xx
        ct[y * HC_X + xx] = hist[(b << 16) | ((x0 + xx) << 8) | y];
    }
    sk1[z] = 0;
    sk2[z] = 0;
    __syncthreads();
    uint32_t a1[HC_X], a2[HC_X];  // exact: <= 8 N and 64 N for N <= 2^23
#pragma unroll
    for (int xx = 0; xx < HC_X; xx++) a1[xx] = a2[xx] = 0;
#pragma unroll 2
    for (int y = 0; y < 256; y++) {
        const uint32_t v = vs[y * 256 + z], v2 = v * v;
        const uint4 *c4 = (const uint4 *)(ct + y * HC_X);
#pragma unroll
        for (int q = 0; q < HC_X / 4; q++) {
            const uint4 c = c4[q];
            a1[4 * q] += c.x * v;
            a2[4 * q] += c.x * v2;
            a1[4 * q + 1] += c.y * v;
            a2[4 * q + 1] += c.y * v2;
            a1[4 * q + 2] += c.z * v;
            a2[4 * q + 2] += c.z * v2;
            a1[4 * q + 3] += c.w * v;
            a2[4 * q + 3] += c.w * v2;
        }
    }
#pragma unroll
    for (int xx = 0; xx < HC_X; xx++) {
        const int k = (x0 + xx) ^ z;  // distinct over the block's threads for this row
        sk1[k] += a1[xx];
        sk2[k] += a2[xx];
        __syncthreads();
    }
    const int h = b * 256 + z;
    if constexpr (std::is_integral<Acc>::value) {
        atomicAdd((unsigned long long *)&sum_h[h], (unsigned long long)sk1[z]);
        atomicAdd((unsigned long long *)&sum_h2[h], (unsigned long long)sk2[z]);
        if (blockIdx.x == 0 && blockIdx.y == 0 && z == 0) atomicAdd((unsigned long long *)count, (unsigned long long)n);
    } else {
        atomicAdd(&sum_h[h], (Acc)sk1[z]);
        atomicAdd(&sum_h2[h], (Acc)sk2[z]);
        if (blockIdx.x == 0 && blockIdx.y == 0 && z == 0) atomicAdd(count, (Acc)n);
    }
}

template <typename Acc>
cudaError_t hist_contract(const uint32_t *d_hist, int64_t n, const uint8_t *d_vtab, Acc *d_sum_h, Acc *d_sum_h2,
                          Acc *d_count, cudaStream_t s, int *launches)
{
    static std::atomic<unsigned long long> attr{0};
    cudaError_t e = smem_attr_once((const void *)k_hist_contract<Acc>, 65536 + HC_X * 256 * 4, attr);
    if (e != cudaSuccess) return e;
    k_hist_contract<Acc><<<dim3(256 / HC_X, 16), 256, 65536 + HC_X * 256 * 4, s>>>(d_hist, d_vtab, d_sum_h, d_sum_h2,
                                                                                   d_count, n);
    if (launches) (*launches)++;
    return cudaGetLastError();
}

template <typename Acc>
cudaError_t modelsums(const uint8_t *d_texts, int64_t n, const uint8_t *d_vtab, uint32_t *d_hist, Acc *d_sum_h,
                      Acc *d_sum_h2, Acc *d_count, cudaStream_t s, int *launches)
{
    static std::atomic<unsigned long long> attr_ms{0}, attr_hc{0};
    cudaError_t e0 = smem_attr_once((const void *)k_modelsums<Acc>, 65536 + MS_STAGE * 16, attr_ms);
    if (e0 == cudaSuccess) e0 = smem_attr_once((const void *)k_hist_contract<Acc>, 65536 + HC_X * 256 * 4, attr_hc);
    if (e0 != cudaSuccess) return e0;
    if (d_hist && n >= kHistMinTraces) {
        cudaError_t e = cudaMemsetAsync(d_hist, 0, sizeof(uint32_t) * 16 * 65536, s);
        if (e != cudaSuccess) return e;
        k_texthist<<<1184, 256, 0, s>>>(d_texts, n, d_hist);
        k_hist_contract<Acc><<<dim3(256 / HC_X, 16), 256, 65536 + HC_X * 256 * 4, s>>>(d_hist, d_vtab, d_sum_h,
                                                                                       d_sum_h2, d_count, n);
        if (launches) (*launches) += 2;
        return cudaGetLastError();
    }
    int64_t chunk = (n + MS_MIN_BLOCKS - 1) / MS_MIN_BLOCKS;
    chunk = chunk < 16 ? 16 : (chunk > MS_CHUNK ? MS_CHUNK : chunk);
    const int blocks = (int)((n + chunk - 1) / chunk);
    k_modelsums<Acc><<<blocks, MS_THREADS, 65536 + MS_STAGE * 16, s>>>(d_texts, n, (int)chunk, d_vtab, d_sum_h,
                                                                         d_sum_h2, d_count);
    if (launches) (*launches)++;
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_modelsums(const uint8_t *d_texts, int64_t n, const uint8_t *d_vtab, uint32_t *d_hist,
                             int64_t *d_sum_h, int64_t *d_sum_h2, int64_t *d_count, cudaStream_t s, int *launches)
{
    return modelsums<int64_t>(d_texts, n, d_vtab, d_hist, d_sum_h, d_sum_h2, d_count, s, launches);
}

cudaError_t launch_modelsums_f64(const uint8_t *d_texts, int64_t n, const uint8_t *d_vtab, uint32_t *d_hist,
                                 double *d_sum_h, double *d_sum_h2, double *d_count, cudaStream_t s, int *launches)
{
    return modelsums<double>(d_texts, n, d_vtab, d_hist, d_sum_h, d_sum_h2, d_count, s, launches);
}

cudaError_t launch_hist_clear(uint32_t *d_hist, cudaStream_t s)
{
    return cudaMemsetAsync(d_hist, 0, sizeof(uint32_t) * 16 * 65536, s);
}

cudaError_t launch_hist_contract(const uint32_t *d_hist, int64_t n, const uint8_t *d_vtab, int64_t *d_sum_h,
                                 int64_t *d_sum_h2, int64_t *d_count, cudaStream_t s, int *launches)
{
    return hist_contract<int64_t>(d_hist, n, d_vtab, d_sum_h, d_sum_h2, d_count, s, launches);
}

cudaError_t launch_hist_contract_f64(const uint32_t *d_hist, int64_t n, const uint8_t *d_vtab, double *d_sum_h,
                                     double *d_sum_h2, double *d_count, cudaStream_t s, int *launches)
{
    return hist_contract<double>(d_hist, n, d_vtab, d_sum_h, d_sum_h2, d_count, s, launches);
}

cudaError_t launch_moments_i8(const void *d_w, int64_t ld, int64_t n, int32_t M, bool w_signed,
                              int64_t *d_sum_w, int64_t *d_sum_w2, int blocks_per_sm, cudaStream_t s,
                              int *launches)
{
    // one resident wave: rows per item so that (groups x chunks) fills the
    // GPU's resident threads exactly once (no wave-quantisation tail);
    // blocks_per_sm > 0 caps the wave (room for a concurrent cross term)
    int dev = 0, sms = 0, per_sm = 0;  // per device: a process may drive several GPUs
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_moments_i8<true>, MO_THREADS, 0);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    const int bps = (blocks_per_sm > 0 && blocks_per_sm < per_sm) ? blocks_per_sm : per_sm;
    const int64_t resident = (int64_t)sms * bps * MO_THREADS;
    const int64_t groups = (M + 15) / 16;
    int64_t chunks = resident / groups;
    if (chunks < 1) chunks = 1;
    int64_t rows = (n + chunks - 1) / chunks;
    rows = (rows + MO_UNROLL - 1) / MO_UNROLL * MO_UNROLL;
    if (rows < 64) rows = 64;
    if (rows > MO_MAX_ROWS) rows = MO_MAX_ROWS;
    const int64_t items = groups * ((n + rows - 1) / rows);
    const unsigned grid = (unsigned)((items + MO_THREADS - 1) / MO_THREADS);
    if (w_signed)
        k_moments_i8<true><<<grid, MO_THREADS, 0, s>>>((const uint8_t *)d_w, ld, n, M, items, rows,
                                                        (unsigned long long *)d_sum_w,
                                                        (unsigned long long *)d_sum_w2);
    else
        k_moments_i8<false><<<grid, MO_THREADS, 0, s>>>((const uint8_t *)d_w, ld, n, M, items, rows,
                                                         (unsigned long long *)d_sum_w,
                                                         (unsigned long long *)d_sum_w2);
    if (launches) (*launches)++;
    return cudaGetLastError();
}

// a8 launch: with rho, one row per block and 4 column pairs in flight per
// thread (tools/fin_bench.py: 4.0 / 5.0 / 5.5 TB/s at M = 5000 / 20000 / 48000,
// +9% over a plain one-row loop; R = 2..8 rows per block sharing the per-sample
// loads were slower: more registers, fewer resident blocks); without rho, the
// filtered maxima kernel from M = 8192 on (-13% / -23% at M = 20000 / 48000)
constexpr int kFinFilterMinM = 8192;
#ifndef FIN_MAXIMA_U
#define FIN_MAXIMA_U 2  // 16-byte row loads in flight per thread (maxima kernel; 4 with 4 blocks: slower)
#endif
// int32 rows: 2 16-byte loads (8 samples) in flight per thread, 5 resident blocks
// (tools/fin_bench.py, M = 20000: 0.133 ms vs 0.156 for 4 loads / 4 blocks; 3
// loads 0.147; C5 checkpoint maxima 3.89 vs 4.45 ms per step)
#ifndef FIN_NARROW_MAXIMA_U
#define FIN_NARROW_MAXIMA_U 2
#endif
#ifndef FIN_NARROW_ROWS_U
#define FIN_NARROW_ROWS_U 4  // rho-writing kernel, int32 rows: 16-byte row loads in flight per thread
#endif
#ifndef FIN_NARROW_MAXIMA_MINB
#define FIN_NARROW_MAXIMA_MINB 5
#endif
// narrow (int32) sum_hw rows: FIN_NARROW_UX times the row loads in flight per
// thread (each load is 16 bytes either way; 1 measured best)
#ifndef FIN_NARROW_UX
#define FIN_NARROW_UX 1
#endif
template <typename T, typename TH = T>
static cudaError_t launch_fin(const TH *hw, const T *sw, const T *sh, const T *sh2, const T *cnt,
                              const double *sqrt_dw, int32_t M, const FinalizeOut &o, cudaStream_t s)
{
    constexpr int X = sizeof(TH) < sizeof(T) ? FIN_NARROW_UX : 1;
    const int rows = o.h1 - o.h0;
    if (o.rho == nullptr && M >= kFinFilterMinM)
        k_finalize_maxima<(X > 1 || sizeof(TH) == sizeof(T)) ? FIN_MAXIMA_U * X : FIN_NARROW_MAXIMA_U, T, TH,
                          sizeof(TH) == sizeof(T) ? FIN_MAXIMA_MINB : FIN_NARROW_MAXIMA_MINB>
            <<<rows, FIN_THREADS, 0, s>>>(hw, sw, sh, sh2, cnt, sqrt_dw, M, o);
    else
        k_finalize_rows<1, (sizeof(TH) == sizeof(T) || X > 1) ? 4 * X : FIN_NARROW_ROWS_U, T, TH>
            <<<rows, FIN_THREADS, 0, s>>>(hw, sw, sh, sh2, cnt, sqrt_dw, M, o);
    return cudaGetLastError();
}

cudaError_t launch_finalize_i8(const int64_t *d_accum, int32_t M, double *d_sqrt_dw, const FinalizeOut &o,
                               cudaStream_t s, int *launches, const int32_t *d_hw32)
{
    const int64_t *hw = d_accum;
    const int64_t *sw = d_accum + 4096LL * M;
    const int64_t *sw2 = sw + M;
    const int64_t *sh = sw2 + M;
    const int64_t *sh2 = sh + 4096;
    const int64_t *cnt = sh2 + 4096;
    k_sqrt_dw_i8<<<(M + 255) / 256, 256, 0, s>>>(sw, sw2, cnt, M, d_sqrt_dw);
    cudaError_t e = d_hw32 ? launch_fin<int64_t, int32_t>(d_hw32, sw, sh, sh2, cnt, d_sqrt_dw, M, o, s)
                           : launch_fin<int64_t>(hw, sw, sh, sh2, cnt, d_sqrt_dw, M, o, s);
    if (e != cudaSuccess) return e;
    if (launches) (*launches) += 2;
    return cudaGetLastError();
}

// CPA_OPT_NARROW flush: sum_hw (int64) += hw32 (int32), n elements, then the
// shadow is dead (the caller drops it)
__global__ void k_widen_hw(const int4 *__restrict__ src, longlong2 *__restrict__ dst, int64_t n4)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const int4 v = __ldcs(src + i);
        longlong2 a = dst[2 * i], b = dst[2 * i + 1];
        a.x += v.x;
        a.y += v.y;
        b.x += v.z;
        b.y += v.w;
        dst[2 * i] = a;
        dst[2 * i + 1] = b;
    }
}
cudaError_t launch_widen_hw(const int32_t *d_hw32, int64_t *d_hw, int64_t n, int num_sms, cudaStream_t s,
                            int *launches)
{
    if (n % 4 != 0) return cudaErrorInvalidValue;  // 4096 M: always a multiple of 4
    k_widen_hw<<<num_sms * 8, 256, 0, s>>>((const int4 *)d_hw32, (longlong2 *)d_hw, n / 4);
    if (launches) (*launches)++;
    return cudaGetLastError();
}

cudaError_t launch_finalize_f64(const double *d_accum, int32_t M, const float *d_offset, double *d_sqrt_dw,
                                const FinalizeOut &o, cudaStream_t s, int *launches)
{
    const double *hw = d_accum;
    const double *sw = d_accum + 4096LL * M;
    const double *sw2 = sw + M;
    const double *sh = sw2 + M;
    const double *sh2 = sh + 4096;
    const double *cnt = sh2 + 4096;
    k_sqrt_dw_f64<<<(M + 255) / 256, 256, 0, s>>>(sw, sw2, cnt, d_offset, M, d_sqrt_dw);
    cudaError_t e = launch_fin<double>(hw, sw, sh, sh2, cnt, d_sqrt_dw, M, o, s);
    if (e != cudaSuccess) return e;
    if (launches) (*launches) += 2;
    return cudaGetLastError();
}

cudaError_t launch_merge_shards(int32_t G, double *maxabs, int32_t *argmax, double *peak, cudaStream_t s,
                                int *launches)
{
    k_merge_shards<<<16, 256, 0, s>>>(G, maxabs, argmax, peak);
    if (launches) (*launches)++;
    return cudaGetLastError();
}

cudaError_t launch_phase4(const FinalizeOut &o, cudaStream_t s, int *launches)
{
    k_phase4<<<16, 256, 0, s>>>(o);
    if (launches) (*launches)++;
    return cudaGetLastError();
}

}  // namespace cpa

// ---------------------------------------------------------------------------
// a6 pre-pass: float traces -> centred, per-sample scaled fp16 hi plane + e4m3
// lo plane, and fp64 moments.  With c = w - o_j and s_j = 2^e_j (exact):
//     hi = fp16(c s_j),  lo = e4m3_satfinite(c s_j - hi)
// so that c s_j ~= hi + lo.  The cross term multiplies both by H 2^-16 -- as
// fp16 (kind::f16; its bit pattern is H << 8) for hi and as e5m2 (kind::f8f6f4;
// its code is the byte H itself) for lo -- into ONE fp32 accumulator, so the
// generator needs no conversion arithmetic; the spill multiplies column j by
// 2^16 / s_j (exact).  |lo| is at most half an fp16 ulp of c s_j (<= 2^-11
// |c s_j|) and e4m3 keeps 4 significant bits of it down to 2^-6 (steps of 2^-9
// below), so the per-element error is at most 2^-15 |c s_j| + 2^-10 against a
// spread of 2^7..2^8 (k_scale_f32): the same relative budget as fp16 + 4 bits.
// fp16 holds 2^15 (the range-repair threshold), 128x that spread; beyond it the
// column's scale is lowered and its planes rewritten (k_fix_scale, k_resplit_f32).
// Thread = 4 consecutive samples (one float4 per row) over SP_ROWS rows.
// ---------------------------------------------------------------------------
namespace cpa {
namespace {
constexpr int SP_THREADS = 256;
#ifndef SP_ROWS_N
#define SP_ROWS_N 128  // C3: 3920 blocks, 6.6 waves (512: 1.66 waves, the second one two-thirds empty)
#endif
constexpr int SP_ROWS = SP_ROWS_N;  // rows per block of the split pre-pass
#ifndef SP_U_ROWS
#define SP_U_ROWS 4
#endif
constexpr int SP_U = SP_U_ROWS;
#ifndef SP_STORE_CS
#define SP_STORE_CS 1  // evict-first plane stores: C3 split 0.773-0.788 -> 0.752-0.756 ms
#endif
// |c s_j| from which the fp16 hi plane is not trusted (fp16 max 65504): the
// column's scale is lowered and its planes rewritten (k_fix_scale, k_resplit_f32)
constexpr float kF16Safe = 32768.0f;

__device__ __forceinline__ uint16_t f16_bits(float x)
{
    return __half_as_ushort(__float2half_rn(x));
}
__device__ __forceinline__ float f16_val(uint16_t b)
{
    return __half2float(__ushort_as_half(b));
}
// two fp32 -> two e4m3 bytes (round to nearest even, saturating): x in the low byte
__device__ __forceinline__ uint32_t e4m3x2(float x, float y)
{
    uint16_t d;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(d) : "f"(y), "f"(x));
    return d;
}

__global__ void __launch_bounds__(SP_THREADS)
k_split_f32(const float *__restrict__ w, int64_t ld, int64_t n, int32_t M, const float *__restrict__ offset,
            const float *__restrict__ scale, uint16_t *__restrict__ hi, uint8_t *__restrict__ lo, int64_t ldh,
            int64_t ldl, double *sum_w, double *sum_w2, int *nonfinite, uint32_t *cmax, int *range)
{
    const int g = blockIdx.x * SP_THREADS + threadIdx.x;
    const int j0 = g * 4;
    if (j0 >= M) return;
    const int cnt = min(4, M - j0);
    float o[4], sc[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
        o[q] = (q < cnt && offset) ? offset[j0 + q] : 0.0f;
        sc[q] = q < cnt ? scale[j0 + q] : 1.0f;
    }
    double s1[4] = {0, 0, 0, 0}, s2[4] = {0, 0, 0, 0};
    float amax[4] = {0, 0, 0, 0};  // max |c| of this thread's rows (range repair)
    bool bad = false;
    const int64_t r0 = (int64_t)blockIdx.y * SP_ROWS;
    const int64_t r1 = min(n, r0 + SP_ROWS);
    // SP_U rows' loads in flight per thread before any use (HBM-bound: one row
    // at a time left too few bytes in flight for the latency)
    for (int64_t rb = r0; rb < r1; rb += SP_U) {
    float xs[SP_U][4];
#pragma unroll
    for (int u = 0; u < SP_U; u++) {
        const int64_t r = rb + u;
        if (r < r1 && cnt == 4) {
            const float4 v = __ldcs((const float4 *)(w + r * ld + j0));
            xs[u][0] = v.x; xs[u][1] = v.y; xs[u][2] = v.z; xs[u][3] = v.w;
        } else {
#pragma unroll
            for (int q = 0; q < 4; q++) xs[u][q] = (r < r1 && q < cnt) ? w[r * ld + j0 + q] : 0.0f;
        }
    }
#pragma unroll
    for (int u = 0; u < SP_U; u++) {
        const int64_t r = rb + u;
        if (r >= r1) break;
        const float *x = xs[u];
        uint16_t h[4];
        float l[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            bad |= !isfinite(x[q]);
            const float c = __fsub_rn(x[q], o[q]);
            const float cs = __fmul_rn(c, sc[q]);  // exact: power of two
            amax[q] = fmaxf(amax[q], fabsf(c));      // (NaN is reported as non-finite)
            h[q] = f16_bits(cs);
            l[q] = __fsub_rn(cs, f16_val(h[q]));  // exact
            s1[q] += (double)c;
            s2[q] += (double)c * (double)c;
        }
        uint16_t *hp = hi + r * ldh + j0;
        uint8_t *lp = lo + r * ldl + j0;
        const uint32_t l8 = e4m3x2(l[0], l[1]) | (e4m3x2(l[2], l[3]) << 16);
        if (cnt == 4) {
            if (SP_STORE_CS) {  // planes (1.5 GB at C3) are read back once, by TMA: evict-first
                __stcs((uint2 *)hp, make_uint2(h[0] | ((uint32_t)h[1] << 16), h[2] | ((uint32_t)h[3] << 16)));
                __stcs((unsigned int *)lp, l8);
            } else {
                *(uint2 *)hp = make_uint2(h[0] | ((uint32_t)h[1] << 16), h[2] | ((uint32_t)h[3] << 16));
                *(uint32_t *)lp = l8;
            }
        } else {
            for (int q = 0; q < cnt; q++) {
                hp[q] = h[q];
                lp[q] = (uint8_t)(l8 >> (8 * q));
            }
        }
    }
    }
    for (int q = 0; q < cnt; q++) {
        atomicAdd(&sum_w[j0 + q], s1[q]);
        atomicAdd(&sum_w2[j0 + q], s2[q]);
    }
    bool over = false;
    for (int q = 0; q < cnt; q++) {
        atomicMax(&cmax[j0 + q], __float_as_uint(amax[q]));  // non-negative floats order as their bits
        over |= amax[q] * sc[q] >= kF16Safe;
    }
    if (bad) atomicOr(nonfinite, 1);
    if (over) atomicOr(range, 1);
}

// Range repair (rare; both kernels exit at once unless *range is set): a column
// whose |c s_j| reached kF16Safe in this chunk (an outlier far beyond the spread
// the scale was chosen from) gets a smaller scale, from this chunk's max |c|, and
// its hi/lo planes are rewritten before the cross term reads them.  The spill
// uses the scale in force for the chunk, so later chunks keep the new one.
__global__ void k_fix_scale(const int *range, const uint32_t *cmax, int32_t M, float *scale, float *inv_scale,
                            uint8_t *colflag)
{
    if (*range == 0) return;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= M) return;
    const float r = __uint_as_float(cmax[j]);
    uint8_t f = 0;
    if (isfinite(r) && r * scale[j] >= kF16Safe) {
        int E;
        frexpf(r, &E);
        const int e = min(64, max(-64, 8 - E));
        scale[j] = ldexpf(1.0f, e);
        inv_scale[j] = ldexpf(1.0f, 16 - e);  // also undoes the 2^-16 of the A operands
        f = 1;
    }
    colflag[j] = f;
}

__global__ void __launch_bounds__(SP_THREADS)
k_resplit_f32(const int *range, const uint8_t *colflag, const float *__restrict__ w, int64_t ld, int64_t n, int32_t M,
              const float *__restrict__ offset, const float *__restrict__ scale, uint16_t *__restrict__ hi,
              uint8_t *__restrict__ lo, int64_t ldh, int64_t ldl)
{
    if (*range == 0) return;
    const int j = blockIdx.x * SP_THREADS + threadIdx.x;
    if (j >= M || !colflag[j]) return;
    const float o = offset ? offset[j] : 0.0f, sc = scale[j];
    const int64_t r0 = (int64_t)blockIdx.y * SP_ROWS, r1 = min(n, r0 + SP_ROWS);
    for (int64_t r = r0; r < r1; r++) {
        const float cs = __fmul_rn(__fsub_rn(w[r * ld + j], o), sc);
        const uint16_t h = f16_bits(cs);
        hi[r * ldh + j] = h;
        lo[r * ldl + j] = (uint8_t)e4m3x2(__fsub_rn(cs, f16_val(h)), 0.0f);
    }
}

// Default per-sample offsets: the mean of the first n (<= 1024) traces, in fp64
// rounded to fp32.  Centring on (an estimate of) the mean rather than on one
// trace keeps the cross term's fp32 TMEM partial sums small: with o_j off the
// mean by ~sigma, sum_i H_i c_ij grows like 4 K sigma over a K-trace unit; with
// the mean of n traces, like 4 K sigma / sqrt(n) + sqrt(K) sigma.  Block = 32
// columns x 8 row groups; each thread sums every 8th row of its column (8 loads
// in flight), then a shared-memory reduction over the row groups.
constexpr int MR_COLS = 32, MR_GROUPS = 8;
__global__ void __launch_bounds__(MR_COLS * MR_GROUPS)
k_mean_rows(const float *__restrict__ w, int64_t ld, int64_t n, int32_t M, float *out)
{
    __shared__ double part[MR_GROUPS][MR_COLS];
    const int tc = threadIdx.x % MR_COLS, g = threadIdx.x / MR_COLS;
    const int j = blockIdx.x * MR_COLS + tc;
    double s = 0.0;
    if (j < M) {
        int64_t i = g;
        for (; i + 7 * MR_GROUPS < n; i += 8 * MR_GROUPS) {
            float v[8];
#pragma unroll
            for (int u = 0; u < 8; u++) v[u] = w[(i + u * MR_GROUPS) * ld + j];
#pragma unroll
            for (int u = 0; u < 8; u++) s += (double)v[u];
        }
        for (; i < n; i += MR_GROUPS) s += (double)w[i * ld + j];
    }
    part[g][tc] = s;
    __syncthreads();
    if (g == 0 && j < M) {
        double t = 0.0;
        for (int k = 0; k < MR_GROUPS; k++) t += part[k][tc];
        out[j] = n > 0 ? (float)(t / (double)n) : 0.0f;
    }
}

// Per-sample scale s_j = 2^e_j for the split: the largest |w - o_j| over the
// first n rows, r, is brought into [2^7, 2^8) (e_j clamped to [-64, 64]; 1 when
// r is 0 or not finite).  inv_scale = 2^16 / s_j (exact; the 2^16 undoes the
// H 2^-16 of the cross term's A operands).
__global__ void k_scale_f32(const float *__restrict__ w, int64_t ld, int64_t n, int32_t M,
                            const float *__restrict__ offset, float *scale, float *inv_scale)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= M) return;
    const float o = offset ? offset[j] : 0.0f;
    float r = 0.0f;
    for (int64_t i = 0; i < n; i++) r = fmaxf(r, fabsf(__fsub_rn(w[i * ld + j], o)));
    int e = 0;
    if (r > 0.0f && isfinite(r)) {
        int E;
        frexpf(r, &E);  // r in [2^(E-1), 2^E)
        e = min(64, max(-64, 8 - E));
    }
    scale[j] = ldexpf(1.0f, e);
    inv_scale[j] = ldexpf(1.0f, 16 - e);
}
}  // namespace

// ---------------------------------------------------------------------------
// Staging repack: n packed rows of rb bytes (as copied 1D from the host) ->
// rows of pitch `pitch` bytes (a multiple of 16, as TMA requires).  Thread =
// one 16-byte output chunk, built from five aligned 32-bit source words and
// funnel shifts.  The source buffer carries >= 20 bytes of readable slack.
// ---------------------------------------------------------------------------
namespace {
constexpr int RP_THREADS = 256;
__global__ void __launch_bounds__(RP_THREADS)
k_repack(const uint8_t *__restrict__ src, int64_t rb, uint8_t *__restrict__ dst, int64_t pitch, int64_t n)
{
    const int64_t q = (int64_t)blockIdx.x * RP_THREADS + threadIdx.x;
    if (q * 16 >= rb) return;
    for (int64_t r = blockIdx.y; r < n; r += gridDim.y) {
        const int64_t s = r * rb + q * 16;
        const uint32_t *a = (const uint32_t *)(src + (s & ~(int64_t)3));
        const uint32_t sh = (uint32_t)(s & 3) * 8;
        uint32_t w[5];
#pragma unroll
        for (int i = 0; i < 5; i++) w[i] = __ldg(a + i);
        uint4 o;
        o.x = __funnelshift_r(w[0], w[1], sh);
        o.y = __funnelshift_r(w[1], w[2], sh);
        o.z = __funnelshift_r(w[2], w[3], sh);
        o.w = __funnelshift_r(w[3], w[4], sh);
        *(uint4 *)(dst + r * pitch + q * 16) = o;
    }
}
}  // namespace

cudaError_t launch_repack(const uint8_t *d_src, int64_t rb, uint8_t *d_dst, int64_t pitch, int64_t n,
                          cudaStream_t s, int *launches)
{
    if (n <= 0) return cudaSuccess;
    const int64_t nq = (rb + 15) / 16;
    dim3 grid((unsigned)((nq + RP_THREADS - 1) / RP_THREADS), (unsigned)(n < 4096 ? n : 4096));
    k_repack<<<grid, RP_THREADS, 0, s>>>(d_src, rb, d_dst, pitch, n);
    if (launches) (*launches)++;
    return cudaGetLastError();
}

cudaError_t launch_split_f32(const float *d_w, int64_t ld, int64_t n, int32_t M, const float *d_offset,
                             const float *d_scale, uint16_t *d_hi, uint8_t *d_lo, int64_t ldh, int64_t ldl,
                             double *d_sum_w, double *d_sum_w2, int *d_nonfinite, uint8_t *d_scratch, cudaStream_t s,
                             int *launches)
{
    const int groups = (M + 3) / 4;
    dim3 grid((groups + SP_THREADS - 1) / SP_THREADS, (unsigned)((n + SP_ROWS - 1) / SP_ROWS));
    // per chunk: column maxima and the range flag start at zero
    uint32_t *cmax = reinterpret_cast<uint32_t *>(d_scratch);
    int *range = reinterpret_cast<int *>(d_scratch + 4 * (size_t)M);
    uint8_t *colflag = d_scratch + 4 * (size_t)M + 16;
    cudaError_t e = cudaMemsetAsync(d_scratch, 0, 4 * (size_t)M + 16, s);
    if (e != cudaSuccess) return e;
    float *scale = const_cast<float *>(d_scale);
    k_split_f32<<<grid, SP_THREADS, 0, s>>>(d_w, ld, n, M, d_offset, d_scale, d_hi, d_lo, ldh, ldl, d_sum_w, d_sum_w2,
                                            d_nonfinite, cmax, range);
    k_fix_scale<<<(M + 127) / 128, 128, 0, s>>>(range, cmax, M, scale, scale + M, colflag);
    dim3 grid1((M + SP_THREADS - 1) / SP_THREADS, grid.y);
    k_resplit_f32<<<grid1, SP_THREADS, 0, s>>>(range, colflag, d_w, ld, n, M, d_offset, d_scale, d_hi, d_lo, ldh, ldl);
    if (launches) (*launches) += 3;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Partial-sum spill, second half: the cross term stored each work unit's raw
// 32-bit accumulators into its trace chunk's slice part[kc][4096][part_ld]; add
// the slices into sum_hw.  Thread = 4 consecutive samples of one row (16-byte
// loads of every slice, all in flight before the adds).
// ---------------------------------------------------------------------------
namespace {
constexpr int PR_THREADS = 256;
constexpr int PR_MAXKC = 8;  // slices loaded ahead per batch
template <bool F32>
__global__ void __launch_bounds__(PR_THREADS)
k_part_reduce(const uint32_t *__restrict__ part, int32_t kc_count, int64_t part_ld, int32_t M,
              const float *__restrict__ inv_scale, void *hw)
{
    const int64_t q4 = part_ld / 4;
    const int64_t slice = 4096 * part_ld;
    for (int64_t g = (int64_t)blockIdx.x * PR_THREADS + threadIdx.x; g < 4096 * q4; g += (int64_t)gridDim.x * PR_THREADS) {
        const int64_t h = g / q4;
        const int j0 = (int)(g - h * q4) * 4;
        if (j0 >= M) continue;
        const uint4 *src = (const uint4 *)(part + h * part_ld + j0);
        if constexpr (F32) {
            double a[4] = {0.0, 0.0, 0.0, 0.0};
            for (int k0 = 0; k0 < kc_count; k0 += PR_MAXKC) {
                uint4 v[PR_MAXKC];
#pragma unroll
                for (int k = 0; k < PR_MAXKC; k++)
                    if (k0 + k < kc_count) v[k] = __ldcs(src + (k0 + k) * (slice / 4));
#pragma unroll
                for (int k = 0; k < PR_MAXKC; k++)
                    if (k0 + k < kc_count) {
                        a[0] += (double)__uint_as_float(v[k].x);
                        a[1] += (double)__uint_as_float(v[k].y);
                        a[2] += (double)__uint_as_float(v[k].z);
                        a[3] += (double)__uint_as_float(v[k].w);
                    }
            }
            double *row = (double *)hw + h * M;
#pragma unroll
            for (int e = 0; e < 4; e++)
                if (j0 + e < M) row[j0 + e] += a[e] * (double)inv_scale[j0 + e];  // power of two: exact
        } else {
            int64_t a[4] = {0, 0, 0, 0};
            for (int k0 = 0; k0 < kc_count; k0 += PR_MAXKC) {
                uint4 v[PR_MAXKC];
#pragma unroll
                for (int k = 0; k < PR_MAXKC; k++)
                    if (k0 + k < kc_count) v[k] = __ldcs(src + (k0 + k) * (slice / 4));
#pragma unroll
                for (int k = 0; k < PR_MAXKC; k++)
                    if (k0 + k < kc_count) {
                        a[0] += (int32_t)v[k].x;
                        a[1] += (int32_t)v[k].y;
                        a[2] += (int32_t)v[k].z;
                        a[3] += (int32_t)v[k].w;
                    }
            }
            int64_t *row = (int64_t *)hw + h * M;
#pragma unroll
            for (int e = 0; e < 4; e++)
                if (j0 + e < M) row[j0 + e] += a[e];
        }
    }
}
int part_reduce_grid(int64_t part_ld)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t need = (4096 * (part_ld / 4) + PR_THREADS - 1) / PR_THREADS;
    const int64_t cap = (int64_t)sms * 8;  // 8 resident blocks per SM, grid-stride beyond
    return (int)(need < cap ? need : cap);
}
}  // namespace

cudaError_t launch_part_reduce_i32(const uint32_t *d_part, int32_t kc_count, int64_t part_ld, int32_t M,
                                   int64_t *d_hw, cudaStream_t s, int *launches)
{
    k_part_reduce<false><<<part_reduce_grid(part_ld), PR_THREADS, 0, s>>>(d_part, kc_count, part_ld, M, nullptr, d_hw);
    if (launches) (*launches)++;
    return cudaGetLastError();
}

cudaError_t launch_part_reduce_f32(const uint32_t *d_part, int32_t kc_count, int64_t part_ld, int32_t M,
                                   const float *d_inv_scale, double *d_hw, cudaStream_t s, int *launches)
{
    k_part_reduce<true><<<part_reduce_grid(part_ld), PR_THREADS, 0, s>>>(d_part, kc_count, part_ld, M, d_inv_scale,
                                                                         d_hw);
    if (launches) (*launches)++;
    return cudaGetLastError();
}

cudaError_t launch_mean_rows(const float *d_w, int64_t ld, int64_t n, int32_t M, float *d_out, cudaStream_t s,
                             int *launches)
{
    k_mean_rows<<<(M + MR_COLS - 1) / MR_COLS, MR_COLS * MR_GROUPS, 0, s>>>(d_w, ld, n, M, d_out);
    if (launches) (*launches)++;
    return cudaGetLastError();
}

cudaError_t launch_scale_f32(const float *d_w, int64_t ld, int64_t n, int32_t M, const float *d_offset,
                             float *d_scale, float *d_inv_scale, cudaStream_t s, int *launches)
{
    k_scale_f32<<<(M + 127) / 128, 128, 0, s>>>(d_w, ld, n, M, d_offset, d_scale, d_inv_scale);
    if (launches) (*launches)++;
    return cudaGetLastError();
}
}  // namespace cpa
