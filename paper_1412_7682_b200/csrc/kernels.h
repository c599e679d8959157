// kernels.h -- internal launchers of libcpa (not part of the C ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

namespace cpa {

// Opt-in dynamic shared memory beyond 48 KB is a per-device-context attribute of
// a kernel: remember it per device ordinal (bit d of `done`), so that a process
// driving several GPUs sets it on each; setting it twice is harmless, so a race
// between host threads costs nothing but a repeated call.
inline cudaError_t smem_attr_once(const void *fn, int bytes, std::atomic<unsigned long long> &done)
{
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = dev < 64 ? 1ull << dev : 0ull;
    if (bit && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess && bit) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

// a3: Phase 1 model sums [P:75]; also adds n to the trace count word.  With a
// 16 x 65536 uint32 scratch (d_hist) and n >= kHistMinTraces the byte-pair
// histogram path is used (exact integer counts, then a fixed contraction).
constexpr int64_t kHistMinTraces = 65536;
cudaError_t launch_modelsums(const uint8_t *d_texts, int64_t n, const uint8_t *d_vtab, uint32_t *d_hist,
                             int64_t *d_sum_h, int64_t *d_sum_h2, int64_t *d_count,
                             cudaStream_t s, int *launches);
cudaError_t launch_modelsums_f64(const uint8_t *d_texts, int64_t n, const uint8_t *d_vtab, uint32_t *d_hist,
                                 double *d_sum_h, double *d_sum_h2, double *d_count,
                                 cudaStream_t s, int *launches);

// a3 with the histogram filled by the cross-term kernel (d_hist passed to
// launch_xterm_*, cleared first): only the contraction (+ n to the count)
cudaError_t launch_hist_clear(uint32_t *d_hist, cudaStream_t s);
cudaError_t launch_hist_contract(const uint32_t *d_hist, int64_t n, const uint8_t *d_vtab, int64_t *d_sum_h,
                                 int64_t *d_sum_h2, int64_t *d_count, cudaStream_t s, int *launches);
cudaError_t launch_hist_contract_f64(const uint32_t *d_hist, int64_t n, const uint8_t *d_vtab, double *d_sum_h,
                                     double *d_sum_h2, double *d_count, cudaStream_t s, int *launches);

// a4: Phase 2 trace moments sum W, sum W^2 [P:79] (int8 traces, exact int64)
cudaError_t launch_moments_i8(const void *d_w, int64_t ld, int64_t n, int32_t M, bool w_signed,
                              int64_t *d_sum_w, int64_t *d_sum_w2, int blocks_per_sm, cudaStream_t s,
                              int *launches);

// a5: cross term (tcgen05 kind::i8, CTA pairs).  With d_sum_w / d_sum_w2 set,
// the kernel also adds a4's sum W, sum W^2 (fused moments).
int xterm_smem_bytes();
int xterm_f32_bk(bool nt2);  // traces per stage of the float cross term variant (the TMA box height of its planes)
int64_t xterm_i8_auto_kchunk(int32_t M, int64_t N, int num_sms, bool remote_epilogue = false);
// Variant choice: NT = 2 sample tiles per unit (A tile reused twice, a4 fused,
// epilogue serialised with the unit's MMAs) or NT = 1 with double-buffered TMEM
// accumulators (the epilogue overlaps the next unit; a4 as a separate pass) --
// the latter was meant for short units (wide / few traces) but measured slower
// (xterm.cu), so force: 0 or 1 = NT = 2, 2 = NT = 1 overlapped.
struct XtermI8Plan {
    bool overlapped = false;
    int64_t kc_len = 0;
};
XtermI8Plan xterm_i8_plan(int32_t M, int64_t N, int num_sms, bool remote_epilogue, int force);
// tmap_hw (may be null: red.add.u64 spill): sum_hw as int64 [4096][M], box 8 x 32,
// 64-byte swizzle -- the epilogue spills by bulk tensor reduce-add (M even).
// hw_zero: sum_hw is all zero before the launch (the library zeroed it and
// nothing was added since); with one trace chunk per unit the spill then stores.
cudaError_t launch_xterm_i8(const CUtensorMap &tmap_w, const CUtensorMap *tmap_hw, const uint8_t *d_texts,
                            const uint8_t *d_vtab, int64_t *d_hw, int *d_counter, int32_t M, int64_t N, int64_t kc_len,
                            bool w_signed, int num_sms, cudaStream_t stream, int *launches, int64_t *d_sum_w = nullptr,
                            int64_t *d_sum_w2 = nullptr, uint32_t *d_hist = nullptr,
                            int64_t *const *owners = nullptr, unsigned long long *d_clk = nullptr,
                            bool overlapped = false, bool hw_zero = false, uint32_t *d_part = nullptr,
                            int64_t part_ld = 0, int32_t *d_hw32 = nullptr);
// d_hw32 non-null (CPA_OPT_NARROW): the cross term goes to that int32 [4096][M]
// array instead of d_hw (the caller guarantees N max|H| max|W| < 2^31); not with
// tmap_hw, d_part or owners
// Partial-sum spill (d_part non-null, part_ld >= M a multiple of 8): every work
// unit stores its raw 32-bit accumulators into part[kc][4096][part_ld] (kc = its
// trace chunk) instead of adding them into sum_hw; then launch_part_reduce adds
//   I8:  sum_hw[h][j] += sum_kc (int64) part[kc][h][j]                (exact)
//   F32: sum_hw[h][j] += (sum_kc (double) part[kc][h][j]) * inv_scale[j]
// (inv_scale a power of two: the product is exact, as in the atomic spill).
cudaError_t launch_part_reduce_i32(const uint32_t *d_part, int32_t kc_count, int64_t part_ld, int32_t M,
                                   int64_t *d_hw, cudaStream_t s, int *launches);
cudaError_t launch_part_reduce_f32(const uint32_t *d_part, int32_t kc_count, int64_t part_ld, int32_t M,
                                   const float *d_inv_scale, double *d_hw, cudaStream_t s, int *launches);

// a6: float traces.  Split pre-pass: c = w - offset[j], hi = fp16(c s_j),
// lo = e4m3(c s_j - hi) into [n][ldh] fp16 / [n][ldl] byte planes (s_j =
// scale[j], a power of two from launch_scale_f32 over the first traces); fp64
// sum c, sum c^2; sets *nonfinite on NaN/Inf [S:140].  Cross term: kind::f16 on
// hi and kind::f8f6f4 on lo into one fp32 TMEM accumulator per <= 4096-trace
// unit (A operands H 2^-16), spilled to fp64 times inv_scale[j] = 2^16 / s_j.  d_scale = [M] scale | [M] inv_scale;
// a column whose |c s_j| reaches 2^15 in a chunk gets a smaller scale and its
// planes rewritten before the cross term (d_scratch: 5 M + 16 bytes).
// default float offsets: mean of the first n rows (the caller passes n <= 1024)
cudaError_t launch_mean_rows(const float *d_w, int64_t ld, int64_t n, int32_t M, float *d_out, cudaStream_t s,
                             int *launches);
cudaError_t launch_scale_f32(const float *d_w, int64_t ld, int64_t n, int32_t M, const float *d_offset,
                             float *d_scale, float *d_inv_scale, cudaStream_t s, int *launches);
cudaError_t launch_split_f32(const float *d_w, int64_t ld, int64_t n, int32_t M, const float *d_offset,
                             const float *d_scale, uint16_t *d_hi, uint8_t *d_lo, int64_t ldh, int64_t ldl,
                             double *d_sum_w, double *d_sum_w2, int *d_nonfinite, uint8_t *d_scratch, cudaStream_t s,
                             int *launches);
// nt2: the V_F32N variant (one H tile feeds two sample tiles, single-buffered
// accumulators, units <= 24576 traces); else NT = 1 (double-buffered, <= 4096)
int64_t xterm_f32_auto_kchunk(int32_t M, int64_t N, int num_sms, bool nt2);
// tmap_hw (may be null: fp64 atomics): sum_hw as fp64 [4096][M], box 8 x 32, 64B
// swizzle -- the spill by bulk tensor reduce-add (M even)
cudaError_t launch_xterm_f32(const CUtensorMap &tmap_hi, const CUtensorMap &tmap_lo, const CUtensorMap *tmap_hw,
                             const uint8_t *d_texts,
                             const uint8_t *d_vtab, double *d_hw, const float *d_inv_scale, int *d_counter, int32_t M,
                             int64_t N, int64_t kc_len, int num_sms, cudaStream_t stream, int *launches,
                             uint32_t *d_hist = nullptr, unsigned long long *d_clk = nullptr, bool nt2 = false,
                             uint32_t *d_part = nullptr, int64_t part_ld = 0);

// a5 for the single-byte models (HW_LAST / HW_FIRST), class sums (classsum.cu):
// counting sort of n traces by text byte per byte (perm: 16 x n int32, off: 16 x
// 257), per chunk of clen traces; then
// per block of mc samples from jc0 (jc0 % 16 == 0, 16-byte rows): S [4096][mc]
// int32 class sums += (launch_cs_sum, per trace chunk) and then sum_hw[256 b + k]
// [jc0 + j] += sum_x f(x ^ k) S_b[x][j] (launch_cs_contract), f = row 0 of d_vtab.
cudaError_t launch_cs_sort(const uint8_t *d_texts, int64_t n, int64_t pstride, int32_t *d_cnt, int32_t *d_off,
                           int32_t *d_cur, int32_t *d_perm, int num_sms, cudaStream_t s, int *launches);
cudaError_t launch_cs_sum(const uint8_t *d_w, int64_t ld, int32_t nch, int64_t clen, int32_t jc0, int32_t mc,
                          bool w_signed, const int32_t *d_perm, const int32_t *d_off, int32_t *d_S, int num_sms,
                          cudaStream_t s, int *launches);
cudaError_t launch_cs_contract(const int32_t *d_S, int32_t M, int32_t jc0, int32_t mc, const uint8_t *d_f,
                               int64_t *d_hw, cudaStream_t s, int *launches);

// a1 staging: n rows of rb contiguous bytes -> rows of `pitch` bytes (multiple
// of 16).  d_src needs >= 20 bytes of readable slack past n*rb.
cudaError_t launch_repack(const uint8_t *d_src, int64_t rb, uint8_t *d_dst, int64_t pitch, int64_t n,
                          cudaStream_t s, int *launches);

// a8/a9: Phase 3 + 4 [P:81-87]
struct FinalizeOut {
    double *rho;       // optional [h1-h0][M]: row h at (h - h0) * M
    int32_t h0 = 0;    // hypothesis rows [h0, h1) of this launch
    int32_t h1 = 4096;
    int32_t col0 = 0;  // global index of sample 0 (sample-axis sharding); added to argmax
    double *maxabs;    // [4096]
    int32_t *argmax;   // [4096]
    double *peak;      // [4096] signed rho at argmax
    int32_t *rank;     // [4096]
    int32_t *best;     // [16] best k, [16] peak sample (packed: best[0..15], best[16..31])
    double *best_rho;  // [16]
};
cudaError_t launch_finalize_i8(const int64_t *d_accum, int32_t M, double *d_sqrt_dw,
                               const FinalizeOut &o, cudaStream_t s, int *launches,
                               const int32_t *d_hw32 = nullptr);  // non-null: sum_hw rows from this int32 shadow
// CPA_OPT_NARROW flush: d_hw[i] += d_hw32[i], i < n (n a multiple of 4)
cudaError_t launch_widen_hw(const int32_t *d_hw32, int64_t *d_hw, int64_t n, int num_sms, cudaStream_t s,
                            int *launches);
// float path: d_offset = the context's per-sample offsets (the sums are centred
// on them; the degenerate-column rule needs the raw second moment)
cudaError_t launch_finalize_f64(const double *d_accum, int32_t M, const float *d_offset, double *d_sqrt_dw,
                                const FinalizeOut &o, cudaStream_t s, int *launches);
cudaError_t launch_phase4(const FinalizeOut &o, cudaStream_t s, int *launches);
// Phase-3 merge of G shards' per-hypothesis maxima (stacked [G][4096]) into
// shard 0's slots: max |rho|, ties to the lowest (global) sample index
cudaError_t launch_merge_shards(int32_t G, double *maxabs, int32_t *argmax, double *peak, cudaStream_t s,
                                int *launches);

}  // namespace cpa
