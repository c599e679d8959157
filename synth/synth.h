/*
 * synth.h -- seeded synthetic CPA workload generator (inputs only).
 *
 * Produces what the paper's SASEBO captures provided [P:168]: N plaintexts /
 * ciphertexts of an unprotected AES-128 with a known key, and N x M power
 * traces that leak, at one sample per key byte, the last-round register
 * Hamming distance (or a Hamming weight) plus Gaussian noise [S:327].
 *
 * This module holds none of the CPA method's arithmetic (no hypotheses over
 * key guesses, no sums, no correlation).  It has its own AES implementation
 * and shares no code with oracle/ or with the product path; both of those
 * consume its output.  Host (synth.c) and device (synth_dev.cu) generators
 * produce bit-identical values: every value is a function of (seed, i, j)
 * through a counter-based integer hash, fixed-point (Q32) integer arithmetic,
 * and a caller-supplied inverse-normal-CDF table.
 */
#ifndef CPA_SYNTH_H
#define CPA_SYNTH_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { SY_LEAK_HD_LAST = 0, SY_LEAK_HW_LAST = 1, SY_LEAK_HW_FIRST = 2 };
enum { SY_S8 = 0, SY_U8 = 1, SY_F32 = 2 };

typedef struct {
    uint64_t seed;
    int32_t m;            /* samples per trace */
    int32_t leak[16];     /* leak sample position of key byte b */
    int64_t mu_lo_q32;    /* per-sample baseline mu_j ~ U[mu_lo, mu_hi] (Q32) */
    int64_t mu_hi_q32;
    int64_t a_q32;        /* leak amplitude a (Q32) */
    int64_t sigma_q16;    /* noise sigma (Q16) */
} sy_params;

/* 65536-entry inverse normal CDF, Phi^-1((u + 0.5) / 65536), in Q16. */
void sy_gauss_table(int32_t table[65536]);

/* Texts and per-byte leakage values for traces [i0, i0+n):
 *   texts: n x 16 (ciphertexts for *_LAST models, plaintexts for HW_FIRST)
 *   leakv: n x 16 (value planted at leak[b]; 0..8)                           */
void sy_texts(const sy_params *p, const uint8_t key[16], int leak_model,
              int64_t i0, int64_t n, uint8_t *texts, uint8_t *leakv);

/* Trace samples for traces [i0, i0+n) and the listed columns (ncols, or all
 * M columns if cols == NULL) into out (row stride ld elements).              */
void sy_traces(const sy_params *p, int dtype, const int32_t *gauss,
               const uint8_t *leakv, int64_t i0, int64_t n,
               const int32_t *cols, int ncols, void *out, int64_t ld);

/* Device generator (synth_dev.cu): all M columns of traces [i0, i0+n);
 * d_leakv (n x 16) and d_gauss (65536) are device pointers.                  */
int sy_dev_traces(const sy_params *p, int dtype, const int32_t *d_gauss,
                  const uint8_t *d_leakv, int64_t i0, int64_t n, void *d_out,
                  int64_t ld, void *stream);

#ifdef __cplusplus
}
#endif
#endif
