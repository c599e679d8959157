/*
 * synth.c -- host side of the synthetic CPA workload generator (see synth.h).
 * Its AES-128 is written independently of oracle/ (S-box from log/antilog
 * tables over generator 3, state held as [row][column]).
 */
#include "synth.h"
#include "synth_core.h"

#include <math.h>
#include <string.h>

/* ---- AES-128 (FIPS-197), independent implementation ------------------- */
static uint8_t S[256];
static int s_ready = 0;

static uint8_t xt(uint8_t a) { return (uint8_t)((a << 1) ^ ((a & 0x80) ? 0x1b : 0)); }

static void sy_init_sbox(void)
{
    if (s_ready) return;
    uint8_t lg[256] = {0}, ex[256] = {0};
    uint8_t x = 1;
    for (int i = 0; i < 255; i++) { /* powers of the generator {03} */
        ex[i] = x;
        lg[x] = (uint8_t)i;
        x = (uint8_t)(x ^ xt(x));
    }
    for (int v = 0; v < 256; v++) {
        uint8_t inv = v ? ex[(255 - lg[v]) % 255] : 0;
        uint8_t r = inv;
        uint8_t s = inv;
        for (int k = 0; k < 4; k++) { /* affine map as x ^ rotl1..rotl4(x) ^ 0x63 */
            s = (uint8_t)((s << 1) | (s >> 7));
            r ^= s;
        }
        S[v] = r ^ 0x63;
    }
    s_ready = 1;
}

static void aes_encrypt(const uint8_t pt[16], const uint8_t key[16], uint8_t ct[16],
                        uint8_t r10in[16], uint8_t r1sb[16])
{
    uint8_t st[4][4], k[4][4], tmp[4];
    uint8_t rc = 1;
    for (int c = 0; c < 4; c++)
        for (int r = 0; r < 4; r++) { st[r][c] = pt[4 * c + r] ^ key[4 * c + r]; k[r][c] = key[4 * c + r]; }
    for (int round = 1; round <= 10; round++) {
        if (round == 10)
            for (int c = 0; c < 4; c++)
                for (int r = 0; r < 4; r++) r10in[4 * c + r] = st[r][c];
        for (int r = 0; r < 4; r++)
            for (int c = 0; c < 4; c++) st[r][c] = S[st[r][c]];
        if (round == 1)
            for (int c = 0; c < 4; c++)
                for (int r = 0; r < 4; r++) r1sb[4 * c + r] = st[r][c];
        for (int r = 1; r < 4; r++) { /* rotate row r left by r */
            for (int c = 0; c < 4; c++) tmp[c] = st[r][(c + r) & 3];
            for (int c = 0; c < 4; c++) st[r][c] = tmp[c];
        }
        if (round != 10)
            for (int c = 0; c < 4; c++) {
                uint8_t a0 = st[0][c], a1 = st[1][c], a2 = st[2][c], a3 = st[3][c];
                uint8_t all = a0 ^ a1 ^ a2 ^ a3;
                st[0][c] ^= all ^ xt(a0 ^ a1);
                st[1][c] ^= all ^ xt(a1 ^ a2);
                st[2][c] ^= all ^ xt(a2 ^ a3);
                st[3][c] ^= all ^ xt(a3 ^ a0);
            }
        /* next round key, column by column */
        uint8_t t0 = S[k[1][3]] ^ rc, t1 = S[k[2][3]], t2 = S[k[3][3]], t3 = S[k[0][3]];
        rc = xt(rc);
        k[0][0] ^= t0; k[1][0] ^= t1; k[2][0] ^= t2; k[3][0] ^= t3;
        for (int c = 1; c < 4; c++)
            for (int r = 0; r < 4; r++) k[r][c] ^= k[r][c - 1];
        for (int r = 0; r < 4; r++)
            for (int c = 0; c < 4; c++) st[r][c] ^= k[r][c];
    }
    for (int c = 0; c < 4; c++)
        for (int r = 0; r < 4; r++) ct[4 * c + r] = st[r][c];
}

static int popcnt8(uint8_t v)
{
    int c = 0;
    while (v) { c += v & 1; v >>= 1; }
    return c;
}

/* ---- noise table -------------------------------------------------------- */
static double phi(double x) { return 0.5 * erfc(-x / sqrt(2.0)); }

void sy_gauss_table(int32_t table[65536])
{
    for (int u = 0; u < 65536; u++) {
        double target = ((double)u + 0.5) / 65536.0;
        double lo = -10.0, hi = 10.0;
        for (int it = 0; it < 80; it++) {
            double mid = 0.5 * (lo + hi);
            if (phi(mid) < target) lo = mid; else hi = mid;
        }
        table[u] = (int32_t)llround(0.5 * (lo + hi) * 65536.0);
    }
}

/* ---- texts and planted leakage ----------------------------------------- */
void sy_texts(const sy_params *p, const uint8_t key[16], int leak_model,
              int64_t i0, int64_t n, uint8_t *texts, uint8_t *leakv)
{
    sy_init_sbox();
    for (int64_t t = 0; t < n; t++) {
        int64_t i = i0 + t;
        uint64_t h0 = sy_mix64(p->seed ^ 0xA4093822299F31D0ULL ^ ((uint64_t)i * 0x9E3779B97F4A7C15ULL));
        uint64_t h1 = sy_mix64(h0 ^ 0x082EFA98EC4E6C89ULL);
        uint8_t pt[16], ct[16], r10[16], r1sb[16];
        for (int b = 0; b < 8; b++) { pt[b] = (uint8_t)(h0 >> (8 * b)); pt[8 + b] = (uint8_t)(h1 >> (8 * b)); }
        aes_encrypt(pt, key, ct, r10, r1sb);
        for (int b = 0; b < 16; b++) {
            /* register position feeding ciphertext byte b after ShiftRows */
            int r = b & 3, c = b >> 2, src = r + 4 * ((c + r) & 3);
            uint8_t v;
            if (leak_model == SY_LEAK_HD_LAST) v = (uint8_t)popcnt8(r10[src] ^ ct[src]);
            else if (leak_model == SY_LEAK_HW_LAST) v = (uint8_t)popcnt8(r10[src]);
            else v = (uint8_t)popcnt8(r1sb[b]);
            leakv[16 * t + b] = v;
            texts[16 * t + b] = (leak_model == SY_LEAK_HW_FIRST) ? pt[b] : ct[b];
        }
    }
}

/* ---- traces --------------------------------------------------------------- */
void sy_traces(const sy_params *p, int dtype, const int32_t *gauss,
               const uint8_t *leakv, int64_t i0, int64_t n,
               const int32_t *cols, int ncols, void *out, int64_t ld)
{
    int nc = cols ? ncols : p->m;
    for (int64_t t = 0; t < n; t++) {
        uint64_t tkey = sy_trace_key(p->seed, i0 + t);
        for (int c = 0; c < nc; c++) {
            int32_t j = cols ? cols[c] : c;
            int64_t v = sy_value_q32(p, gauss, tkey, leakv + 16 * t, j, sy_mu_q32(p, j));
            if (dtype == SY_S8) ((int8_t *)out)[t * ld + c] = sy_to_s8(v);
            else if (dtype == SY_U8) ((uint8_t *)out)[t * ld + c] = sy_to_u8(v);
            else ((float *)out)[t * ld + c] = sy_to_f32(v);
        }
    }
}
