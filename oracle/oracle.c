/*
 * oracle.c -- plain single-threaded CPU oracle for the CPA hot path of
 * arXiv:1412.7682 ("Accelerating Correlation Power Analysis Using GPUs").
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Everything here is written as the
 * plain definition, in the paper's order and notation: no blocking, no fusion,
 * no reordering beyond a loop order.  Shares nothing with the CUDA path.
 *
 * Pins (tests/test_oracle_*.py, run with -m "not gpu"):
 *   AES tables / schedule / encryption  -> FIPS-197 App. A.1, B, C.1 values
 *   selection function                  -> FIPS-197 App. B round-10 states
 *   sums                                -> brute force, numpy int64 matmul,
 *                                          closed forms (sum_k H = 1024 ...)
 *   rho (Eq. (1) and two-pass)          -> W = +-H gives +-1, numpy.corrcoef,
 *                                          exact rationals via fractions
 *   phase 3 / 4                         -> constructed surfaces [S:263-264]
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* AES-128 per FIPS-197.  Tables are built from the field definition          */
/* (GF(2^8) modulo x^8+x^4+x^3+x+1, FIPS-197 Sec. 4.2) and the affine map     */
/* of Sec. 5.1.1 -- not typed in -- so the FIPS vectors in the tests pin them. */
/* ------------------------------------------------------------------------ */

static uint8_t g_sbox[256], g_inv[256], g_sr[16];
static int g_ready = 0;

static uint8_t gf_mul(uint8_t a, uint8_t b) /* FIPS-197 Sec. 4.2 */
{
    uint8_t p = 0;
    for (int i = 0; i < 8; i++) {
        if (b & 1) p ^= a;
        uint8_t hi = a & 0x80;
        a <<= 1;
        if (hi) a ^= 0x1b;
        b >>= 1;
    }
    return p;
}

static void init_tables(void)
{
    if (g_ready) return;
    for (int x = 0; x < 256; x++) {
        /* multiplicative inverse, {00} -> {00} (FIPS-197 Sec. 5.1.1 step 1) */
        uint8_t inv = 0;
        for (int y = 1; y < 256; y++)
            if (gf_mul((uint8_t)x, (uint8_t)y) == 1) { inv = (uint8_t)y; break; }
        /* affine transformation, c = {63} (FIPS-197 eq. 5.1) */
        uint8_t s = 0;
        for (int i = 0; i < 8; i++) {
            int bit = ((inv >> i) & 1) ^ ((inv >> ((i + 4) % 8)) & 1) ^
                      ((inv >> ((i + 5) % 8)) & 1) ^ ((inv >> ((i + 6) % 8)) & 1) ^
                      ((inv >> ((i + 7) % 8)) & 1) ^ ((0x63 >> i) & 1);
            s |= (uint8_t)(bit << i);
        }
        g_sbox[x] = s;
    }
    for (int x = 0; x < 256; x++) g_inv[g_sbox[x]] = (uint8_t)x;
    /* ShiftRows source map by brute force: shift row r left by r (Sec. 5.1.2),
     * state byte index = r + 4c (column-major, [S:64, S:107]).               */
    for (int r = 0; r < 4; r++)
        for (int c = 0; c < 4; c++)
            g_sr[r + 4 * c] = (uint8_t)(r + 4 * ((c + r) % 4));
    g_ready = 1;
}

void or_aes_tables(uint8_t sbox[256], uint8_t inv_sbox[256])
{
    init_tables();
    memcpy(sbox, g_sbox, 256);
    memcpy(inv_sbox, g_inv, 256);
}

void or_shiftrows_src(uint8_t sr[16])
{
    init_tables();
    memcpy(sr, g_sr, 16);
}

void or_expand_key(const uint8_t key[16], uint8_t rk[11][16]) /* FIPS-197 Sec. 5.2 */
{
    init_tables();
    uint8_t w[44][4];
    uint8_t rcon = 1;
    for (int i = 0; i < 4; i++)
        for (int j = 0; j < 4; j++) w[i][j] = key[4 * i + j];
    for (int i = 4; i < 44; i++) {
        uint8_t t[4] = {w[i - 1][0], w[i - 1][1], w[i - 1][2], w[i - 1][3]};
        if (i % 4 == 0) {
            uint8_t t0 = t[0];               /* RotWord */
            t[0] = t[1]; t[1] = t[2]; t[2] = t[3]; t[3] = t0;
            for (int j = 0; j < 4; j++) t[j] = g_sbox[t[j]]; /* SubWord */
            t[0] ^= rcon;
            rcon = gf_mul(rcon, 2);
        }
        for (int j = 0; j < 4; j++) w[i][j] = w[i - 4][j] ^ t[j];
    }
    for (int r = 0; r < 11; r++)
        for (int i = 0; i < 4; i++)
            for (int j = 0; j < 4; j++) rk[r][4 * i + j] = w[4 * r + i][j];
}

/* Run the schedule of Sec. 5.2 backwards from round `round` to round 0
 * ("using the round key, the actual key can be derived" [P:63]).            */
void or_invert_key_schedule(const uint8_t rk[16], int round, uint8_t key[16])
{
    init_tables();
    uint8_t w[44][4];
    uint8_t rcons[10];
    rcons[0] = 1;
    for (int i = 1; i < 10; i++) rcons[i] = gf_mul(rcons[i - 1], 2);
    for (int i = 0; i < 4; i++)
        for (int j = 0; j < 4; j++) w[4 * round + i][j] = rk[4 * i + j];
    for (int i = 4 * round + 3; i >= 4; i--) {
        /* w[i] = w[i-4] ^ t(w[i-1])  =>  w[i-4] = w[i] ^ t(w[i-1]) */
        uint8_t t[4] = {w[i - 1][0], w[i - 1][1], w[i - 1][2], w[i - 1][3]};
        if (i % 4 == 0) {
            uint8_t t0 = t[0];
            t[0] = t[1]; t[1] = t[2]; t[2] = t[3]; t[3] = t0;
            for (int j = 0; j < 4; j++) t[j] = g_sbox[t[j]];
            t[0] ^= rcons[i / 4 - 1];
        }
        for (int j = 0; j < 4; j++) w[i - 4][j] = w[i][j] ^ t[j];
    }
    for (int i = 0; i < 4; i++)
        for (int j = 0; j < 4; j++) key[4 * i + j] = w[i][j];
}

static void mix_columns(uint8_t s[16]) /* FIPS-197 Sec. 5.1.3 */
{
    for (int c = 0; c < 4; c++) {
        uint8_t a0 = s[4 * c], a1 = s[4 * c + 1], a2 = s[4 * c + 2], a3 = s[4 * c + 3];
        s[4 * c + 0] = gf_mul(a0, 2) ^ gf_mul(a1, 3) ^ a2 ^ a3;
        s[4 * c + 1] = a0 ^ gf_mul(a1, 2) ^ gf_mul(a2, 3) ^ a3;
        s[4 * c + 2] = a0 ^ a1 ^ gf_mul(a2, 2) ^ gf_mul(a3, 3);
        s[4 * c + 3] = gf_mul(a0, 3) ^ a1 ^ a2 ^ gf_mul(a3, 2);
    }
}

/* FIPS-197 Sec. 5.1 Cipher(); also returns the state at the start of round 10
 * (the "round-9 output" register value [S:42]).                             */
void or_encrypt_with_states(const uint8_t pt[16], const uint8_t key[16],
                            uint8_t ct[16], uint8_t round10_in[16])
{
    init_tables();
    uint8_t rk[11][16], s[16], t[16];
    or_expand_key(key, rk);
    for (int i = 0; i < 16; i++) s[i] = pt[i] ^ rk[0][i];
    for (int r = 1; r <= 10; r++) {
        if (r == 10) memcpy(round10_in, s, 16);
        for (int i = 0; i < 16; i++) s[i] = g_sbox[s[i]];        /* SubBytes */
        for (int i = 0; i < 16; i++) t[i] = s[g_sr[i]];          /* ShiftRows */
        memcpy(s, t, 16);
        if (r != 10) mix_columns(s);                             /* MixColumns */
        for (int i = 0; i < 16; i++) s[i] ^= rk[r][i];           /* AddRoundKey */
    }
    memcpy(ct, s, 16);
}

/* ------------------------------------------------------------------------ */
/* Selection function H_i for (byte position b, sub-key guess k) [P:67]       */
/* ------------------------------------------------------------------------ */

static int hamming_weight(unsigned v) /* count set bits, one by one */
{
    int c = 0;
    for (int i = 0; i < 8; i++) c += (v >> i) & 1;
    return c;
}

int or_selection(int model, const uint8_t text[16], int b, int k)
{
    init_tables();
    switch (model) {
    case OR_HD_LAST: /* HW(InvS(c[b] ^ k) ^ c[SR(b)])  [S:85] */
        return hamming_weight(g_inv[text[b] ^ k] ^ text[g_sr[b]]);
    case OR_HW_LAST: /* HW(InvS(c[b] ^ k)) */
        return hamming_weight(g_inv[text[b] ^ k]);
    case OR_HW_FIRST: /* HW(S(p[b] ^ k)), first-round variant [P:63] */
        return hamming_weight(g_sbox[text[b] ^ k]);
    default:
        abort();
    }
}

/* ------------------------------------------------------------------------ */
/* Phase 1: sum_i H_i and sum_i H_i^2 per (sub-key, byte) [P:75]              */
/* ------------------------------------------------------------------------ */
void or_model_sums(int model, const uint8_t *texts, int64_t n,
                   int64_t *sum_h, int64_t *sum_h2)
{
    for (int h = 0; h < 4096; h++) {
        int b = h / 256, k = h % 256;
        int64_t s1 = 0, s2 = 0;
        for (int64_t i = 0; i < n; i++) {
            int64_t H = or_selection(model, texts + 16 * i, b, k);
            s1 += H;
            s2 += H * H;
        }
        sum_h[h] = s1;
        sum_h2[h] = s2;
    }
}

/* ------------------------------------------------------------------------ */
/* Phase 2: sum_i W_ij, sum_i W_ij^2 and sum_i W_ij H_i [P:79]                */
/* ------------------------------------------------------------------------ */
static inline int64_t wval(const void *W, int w_signed, int64_t ld, int64_t i, int64_t j)
{
    return w_signed ? (int64_t)((const int8_t *)W)[i * ld + j]
                    : (int64_t)((const uint8_t *)W)[i * ld + j];
}

void or_trace_sums_i8(const void *W, int w_signed, int64_t n, int64_t ld,
                      const int32_t *cols, int ncols, int64_t *sum_w, int64_t *sum_w2)
{
    for (int c = 0; c < ncols; c++) {
        int64_t s1 = 0, s2 = 0;
        for (int64_t i = 0; i < n; i++) {
            int64_t w = wval(W, w_signed, ld, i, cols[c]);
            s1 += w;
            s2 += w * w;
        }
        sum_w[c] = s1;
        sum_w2[c] = s2;
    }
}

void or_cross_sums_i8(int model, const uint8_t *texts, const void *W, int w_signed,
                      int64_t n, int64_t ld, const int32_t *cols, int ncols,
                      int64_t *sum_hw)
{
    int64_t *acc = sum_hw;
    memset(acc, 0, sizeof(int64_t) * 4096 * (size_t)ncols);
    for (int h = 0; h < 4096; h++) {
        int b = h / 256, k = h % 256;
        int64_t *row = acc + (size_t)h * ncols;
        for (int64_t i = 0; i < n; i++) {
            int64_t H = or_selection(model, texts + 16 * i, b, k);
            if (w_signed) {
                const int8_t *wi = (const int8_t *)W + i * ld;
                for (int c = 0; c < ncols; c++) row[c] += H * (int64_t)wi[cols[c]];
            } else {
                const uint8_t *wi = (const uint8_t *)W + i * ld;
                for (int c = 0; c < ncols; c++) row[c] += H * (int64_t)wi[cols[c]];
            }
        }
    }
}

void or_model_sums_hyps(int model, const uint8_t *texts, int64_t n, const int32_t *hyps,
                        int nhyps, int64_t *sum_h, int64_t *sum_h2)
{
    for (int a = 0; a < nhyps; a++) {
        int b = hyps[a] / 256, k = hyps[a] % 256;
        int64_t s1 = 0, s2 = 0;
        for (int64_t i = 0; i < n; i++) {
            int64_t H = or_selection(model, texts + 16 * i, b, k);
            s1 += H;
            s2 += H * H;
        }
        sum_h[a] = s1;
        sum_h2[a] = s2;
    }
}

void or_cross_sums_hyps_i8(int model, const uint8_t *texts, const void *W, int w_signed,
                           int64_t n, int64_t ld, const int32_t *cols, int ncols,
                           const int32_t *hyps, int nhyps, int64_t *sum_hw)
{
    memset(sum_hw, 0, sizeof(int64_t) * (size_t)nhyps * (size_t)ncols);
    for (int a = 0; a < nhyps; a++) {
        int b = hyps[a] / 256, k = hyps[a] % 256;
        int64_t *row = sum_hw + (size_t)a * ncols;
        for (int64_t i = 0; i < n; i++) {
            int64_t H = or_selection(model, texts + 16 * i, b, k);
            for (int c = 0; c < ncols; c++) row[c] += H * wval(W, w_signed, ld, i, cols[c]);
        }
    }
}

/* ------------------------------------------------------------------------ */
/* Eq. (1) [P:69] from the exact integer sums ("reference B"):                */
/*   num = N*S_hw - S_h*S_w ; dw = N*S_w2 - S_w^2 ; dh = N*S_h2 - S_h^2       */
/*   rho = (double)num / (sqrt((double)dw) * sqrt((double)dh))               */
/* Products in __int128; each of num, dw, dh must fit int64 and is converted  */
/* from int64 (round to nearest).  dw == 0 or dh == 0 -> 0 [S:293]; clamp to  */
/* [-1, 1] [S:246].  No a*b+c pattern, so no FMA contraction can apply.       */
/* ------------------------------------------------------------------------ */
static int fits64(__int128 v)
{
    return v >= (__int128)INT64_MIN && v <= (__int128)INT64_MAX;
}

int or_rho_eq1(int64_t n, int64_t s_hw, int64_t s_h, int64_t s_h2,
               int64_t s_w, int64_t s_w2, double *rho)
{
    __int128 num = (__int128)n * s_hw - (__int128)s_h * s_w;
    __int128 dw = (__int128)n * s_w2 - (__int128)s_w * s_w;
    __int128 dh = (__int128)n * s_h2 - (__int128)s_h * s_h;
    if (!fits64(num) || !fits64(dw) || !fits64(dh)) return -1;
    if (dw == 0 || dh == 0) { *rho = 0.0; return 0; }
    double den_w = sqrt((double)(int64_t)dw);
    double den_h = sqrt((double)(int64_t)dh);
    double den = den_w * den_h;
    double r = (double)(int64_t)num / den;
    if (r > 1.0) r = 1.0;
    if (r < -1.0) r = -1.0;
    *rho = r;
    return 0;
}

int or_rho_eq1_grid(int64_t n, const int64_t *sum_hw, const int64_t *sum_h,
                    const int64_t *sum_h2, const int64_t *sum_w,
                    const int64_t *sum_w2, int ncols, double *rho)
{
    for (int h = 0; h < 4096; h++)
        for (int c = 0; c < ncols; c++)
            if (or_rho_eq1(n, sum_hw[(size_t)h * ncols + c], sum_h[h], sum_h2[h],
                           sum_w[c], sum_w2[c], &rho[(size_t)h * ncols + c]))
                return -1;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Textbook two-pass Pearson ("reference A") [S:274-280]: means first, then   */
/* centred cross/auto products, each summed with Neumaier compensation.       */
/* ------------------------------------------------------------------------ */
typedef struct { double s, c; } ksum;
static void kadd(ksum *a, double x) /* Neumaier's improved Kahan summation */
{
    double t = a->s + x;
    if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x;
    else a->c += (x - t) + a->s;
    a->s = t;
}
static double kval(const ksum *a) { return a->s + a->c; }

static double pearson_two_pass(const double *x, const double *y, int64_t n, double eps_rel)
{
    ksum sx = {0, 0}, sy = {0, 0};
    for (int64_t i = 0; i < n; i++) { kadd(&sx, x[i]); kadd(&sy, y[i]); }
    double mx = kval(&sx) / (double)n, my = kval(&sy) / (double)n;
    ksum cxy = {0, 0}, cxx = {0, 0}, cyy = {0, 0}, syy = {0, 0};
    for (int64_t i = 0; i < n; i++) {
        double dx = x[i] - mx, dy = y[i] - my;
        kadd(&cxy, dx * dy);
        kadd(&cxx, dx * dx);
        kadd(&cyy, dy * dy);
        kadd(&syy, y[i] * y[i]);
    }
    double vxx = kval(&cxx), vyy = kval(&cyy);
    /* degenerate variance -> 0 [S:293]: exact zero for integer data,
     * relative eps for float data                                            */
    if (vxx <= 0.0 || vyy <= 0.0) return 0.0;
    if (eps_rel > 0.0 && vyy <= eps_rel * kval(&syy)) return 0.0;
    double r = kval(&cxy) / sqrt(vxx * vyy);
    if (r > 1.0) r = 1.0;
    if (r < -1.0) r = -1.0;
    return r;
}

void or_rho_two_pass_i8(int model, const uint8_t *texts, const void *W, int w_signed,
                        int64_t n, int64_t ld, const int32_t *cols, int ncols,
                        const int32_t *hyps, int nhyps, double *rho)
{
    double *x = (double *)malloc(sizeof(double) * (size_t)n);
    double *y = (double *)malloc(sizeof(double) * (size_t)n);
    for (int a = 0; a < nhyps; a++) {
        int h = hyps[a];
        for (int64_t i = 0; i < n; i++)
            x[i] = (double)or_selection(model, texts + 16 * i, h / 256, h % 256);
        for (int c = 0; c < ncols; c++) {
            for (int64_t i = 0; i < n; i++) y[i] = (double)wval(W, w_signed, ld, i, cols[c]);
            rho[(size_t)a * ncols + c] = pearson_two_pass(x, y, n, 0.0);
        }
    }
    free(x);
    free(y);
}

void or_rho_two_pass_f32(int model, const uint8_t *texts, const float *W, int64_t n,
                         int64_t ld, const int32_t *cols, int ncols,
                         const int32_t *hyps, int nhyps, double *rho)
{
    double *x = (double *)malloc(sizeof(double) * (size_t)n);
    double *y = (double *)malloc(sizeof(double) * (size_t)n);
    for (int a = 0; a < nhyps; a++) {
        int h = hyps[a];
        for (int64_t i = 0; i < n; i++)
            x[i] = (double)or_selection(model, texts + 16 * i, h / 256, h % 256);
        for (int c = 0; c < ncols; c++) {
            for (int64_t i = 0; i < n; i++) y[i] = (double)W[i * ld + cols[c]];
            rho[(size_t)a * ncols + c] = pearson_two_pass(x, y, n, 1e-12);
        }
    }
    free(x);
    free(y);
}

/* float-trace sums, accumulated in double [S:239, S:297] */
void or_sums_f32(int model, const uint8_t *texts, const float *W, int64_t n,
                 int64_t ld, const int32_t *cols, int ncols,
                 double *sum_hw, double *sum_w, double *sum_w2)
{
    for (int c = 0; c < ncols; c++) {
        double s1 = 0, s2 = 0;
        for (int64_t i = 0; i < n; i++) {
            double w = (double)W[i * ld + cols[c]];
            s1 += w;
            s2 += w * w;
        }
        sum_w[c] = s1;
        sum_w2[c] = s2;
    }
    memset(sum_hw, 0, sizeof(double) * 4096 * (size_t)ncols);
    for (int h = 0; h < 4096; h++) {
        double *row = sum_hw + (size_t)h * ncols;
        for (int64_t i = 0; i < n; i++) {
            double H = (double)or_selection(model, texts + 16 * i, h / 256, h % 256);
            for (int c = 0; c < ncols; c++) row[c] += H * (double)W[i * ld + cols[c]];
        }
    }
}

void or_rho_eq1_f64_grid(int64_t n, const double *sum_hw, const int64_t *sum_h,
                         const int64_t *sum_h2, const double *sum_w,
                         const double *sum_w2, int ncols, double *rho)
{
    double N = (double)n;
    for (int h = 0; h < 4096; h++) {
        double dh = N * (double)sum_h2[h] - (double)sum_h[h] * (double)sum_h[h];
        for (int c = 0; c < ncols; c++) {
            double num = N * sum_hw[(size_t)h * ncols + c] - (double)sum_h[h] * sum_w[c];
            double dw = N * sum_w2[c] - sum_w[c] * sum_w[c];
            double r = 0.0;
            if (dh > 0.0 && dw > 1e-12 * N * sum_w2[c]) r = num / (sqrt(dw) * sqrt(dh));
            if (r > 1.0) r = 1.0;
            if (r < -1.0) r = -1.0;
            rho[(size_t)h * ncols + c] = r;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* Phase 3 [P:83]: for each (sub-key, byte) the maximum |rho| over the sample */
/* points [S:292]; ties -> lowest sample index [S:298].  `cols` ascending.     */
/* ------------------------------------------------------------------------ */
void or_phase3(const double *rho, int ncols, const int32_t *cols,
               double *maxabs, int32_t *argmax, double *peak)
{
    for (int h = 0; h < 4096; h++) {
        double best = -1.0, pk = 0.0;
        int32_t arg = -1;
        for (int c = 0; c < ncols; c++) {
            double r = rho[(size_t)h * ncols + c];
            if (fabs(r) > best) { best = fabs(r); arg = cols[c]; pk = r; }
        }
        maxabs[h] = best;
        argmax[h] = arg;
        peak[h] = pk;
    }
}

/* ------------------------------------------------------------------------ */
/* Phase 4 [P:87]: "sub keys that have maximum correlation" per byte; rank is */
/* 1 + number of keys strictly better (higher maxabs, or equal and lower k).  */
/* ------------------------------------------------------------------------ */
void or_phase4(const double *maxabs, uint8_t best[16], int32_t *rank)
{
    for (int b = 0; b < 16; b++) {
        for (int k = 0; k < 256; k++) {
            int r = 1;
            for (int k2 = 0; k2 < 256; k2++) {
                double a = maxabs[256 * b + k2], m = maxabs[256 * b + k];
                if (a > m || (a == m && k2 < k)) r++;
            }
            rank[256 * b + k] = r;
            if (r == 1) best[b] = (uint8_t)k;
        }
    }
}
