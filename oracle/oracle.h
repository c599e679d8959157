/*
 * oracle.h -- plain, slow, single-threaded CPU oracle for the CPA hot path of
 * Gamaarachchi, Ragel & Jayasinghe, "Accelerating Correlation Power Analysis
 * Using GPUs" (arXiv:1412.7682).  PAPER.md line numbers are cited as [P:n],
 * SPEC.md lines as [S:n].
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_1412_7682_b200/) and neither includes the other.
 *
 * Conventions:
 *   hypothesis index h = 256*b + k  (b = key byte 0..15, k = sub-key guess)
 *   traces W are row-major N x ld (trace i = row i, sample j contiguous) [P:65]
 *   texts are N x 16 bytes, byte b = AES state byte b (column-major) [S:107]
 *   sums run over i = 0..N-1 (Eq. (1)'s "sum_{i=0}^{N}" read as N terms) [P:69, S:299]
 */
#ifndef CPA_ORACLE_H
#define CPA_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* selection-function models [P:63; S:85] */
enum { OR_HD_LAST = 0, OR_HW_LAST = 1, OR_HW_FIRST = 2 };

/* ---- AES-128 (FIPS-197), needed by the selection function ------------- */
void or_aes_tables(uint8_t sbox[256], uint8_t inv_sbox[256]);
void or_shiftrows_src(uint8_t sr[16]);
void or_expand_key(const uint8_t key[16], uint8_t rk[11][16]);
void or_invert_key_schedule(const uint8_t rk[16], int round, uint8_t key[16]);
void or_encrypt_with_states(const uint8_t pt[16], const uint8_t key[16],
                            uint8_t ct[16], uint8_t round10_in[16]);

/* ---- Phase 1 input: selection value H [P:67; S:85] -------------- */
int or_selection(int model, const uint8_t text[16], int b, int k);

/* ---- Phase 1: model sums  sum_h[h], sum_h2[h]  (exact int64) [P:75] ---- */
void or_model_sums(int model, const uint8_t *texts, int64_t n,
                   int64_t *sum_h, int64_t *sum_h2);

/* ---- Phase 2: trace sums over the listed sample columns [P:79] ---------
 * w_signed: 1 = int8 traces, 0 = uint8 traces.
 * sum_hw is [4096][ncols]; sum_w, sum_w2 are [ncols].                       */
void or_trace_sums_i8(const void *W, int w_signed, int64_t n, int64_t ld,
                      const int32_t *cols, int ncols,
                      int64_t *sum_w, int64_t *sum_w2);
void or_cross_sums_i8(int model, const uint8_t *texts, const void *W,
                      int w_signed, int64_t n, int64_t ld,
                      const int32_t *cols, int ncols, int64_t *sum_hw);

/* Same sums restricted to a list of hypotheses h (rows of sum_hw follow
 * `hyps`): used to check full-size GPU runs on sampled outputs.             */
void or_model_sums_hyps(int model, const uint8_t *texts, int64_t n, const int32_t *hyps,
                        int nhyps, int64_t *sum_h, int64_t *sum_h2);
void or_cross_sums_hyps_i8(int model, const uint8_t *texts, const void *W, int w_signed,
                           int64_t n, int64_t ld, const int32_t *cols, int ncols,
                           const int32_t *hyps, int nhyps, int64_t *sum_hw);

/* ---- Eq. (1) from the exact integer sums (reference B) [P:69] ----------
 * Returns 0 on success, -1 if an intermediate does not fit int64.          */
int or_rho_eq1(int64_t n, int64_t s_hw, int64_t s_h, int64_t s_h2,
               int64_t s_w, int64_t s_w2, double *rho);
/* rho[h][c] for every hypothesis and listed column, from the sums above.   */
int or_rho_eq1_grid(int64_t n, const int64_t *sum_hw, const int64_t *sum_h,
                    const int64_t *sum_h2, const int64_t *sum_w,
                    const int64_t *sum_w2, int ncols, double *rho);

/* ---- textbook two-pass Pearson (reference A) [S:274-280] ---------------- */
void or_rho_two_pass_i8(int model, const uint8_t *texts, const void *W,
                        int w_signed, int64_t n, int64_t ld,
                        const int32_t *cols, int ncols, const int32_t *hyps,
                        int nhyps, double *rho);
void or_rho_two_pass_f32(int model, const uint8_t *texts, const float *W,
                         int64_t n, int64_t ld, const int32_t *cols, int ncols,
                         const int32_t *hyps, int nhyps, double *rho);

/* ---- float-trace variant sums, fp64 accumulation [S:297] --------------- */
void or_sums_f32(int model, const uint8_t *texts, const float *W, int64_t n,
                 int64_t ld, const int32_t *cols, int ncols,
                 double *sum_hw, double *sum_w, double *sum_w2);
/* Eq. (1) in fp64 from fp64 sums (float path) */
void or_rho_eq1_f64_grid(int64_t n, const double *sum_hw, const int64_t *sum_h,
                         const int64_t *sum_h2, const double *sum_w,
                         const double *sum_w2, int ncols, double *rho);

/* ---- Phase 3: max |rho| over the columns, lowest column on ties [P:83] -- */
void or_phase3(const double *rho, int ncols, const int32_t *cols,
               double *maxabs, int32_t *argmax, double *peak);

/* ---- Phase 4: per byte rank keys by maxabs, ties to lower k [P:87] ------ */
void or_phase4(const double *maxabs, uint8_t best[16], int32_t *rank);

#ifdef __cplusplus
}
#endif
#endif
