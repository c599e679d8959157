// aes_host.cpp -- host-side AES-128 pieces the engine needs (FIPS-197):
// S-box / inverse for the selection tables, and the key schedule + its
// inversion for Phase 4's "round key -> actual key" step [P:63].
// (Independent of oracle/ and synth/: inverse by exponentiation x^254.)
#include <cstdint>
#include <cstring>

#include "tables.h"

namespace cpa {

static uint8_t gmul(uint8_t a, uint8_t b)
{
    uint8_t r = 0;
    while (b) {
        if (b & 1) r ^= a;
        a = (uint8_t)((a << 1) ^ ((a & 0x80) ? 0x1b : 0));
        b >>= 1;
    }
    return r;
}

static uint8_t gpow(uint8_t a, int e)
{
    uint8_t r = 1;
    while (e) {
        if (e & 1) r = gmul(r, a);
        a = gmul(a, a);
        e >>= 1;
    }
    return r;
}

void aes_sboxes(uint8_t sbox[256], uint8_t inv[256])
{
    for (int x = 0; x < 256; x++) {
        uint8_t y = x ? gpow((uint8_t)x, 254) : 0;  // multiplicative inverse in GF(2^8)
        static const int offs[5] = {0, 4, 5, 6, 7};
        uint8_t s = 0x63;
        for (int i = 0; i < 8; i++) {  // affine map, FIPS-197 eq. (5.1)
            uint8_t bit = 0;
            for (int k = 0; k < 5; k++) bit ^= (y >> ((i + offs[k]) & 7)) & 1;
            s ^= (uint8_t)(bit << i);
        }
        sbox[x] = s;
    }
    for (int x = 0; x < 256; x++) inv[sbox[x]] = (uint8_t)x;
}

// V[y][x]: selection value as a function of the ciphertext byte pair, so that
// H(b, k) = V[c[SR(b)]][c[b] ^ k] for every model (HW models ignore y).
void build_vtable(int model, uint8_t *v /* 65536 */)
{
    uint8_t s[256], inv[256];
    aes_sboxes(s, inv);
    for (int y = 0; y < 256; y++)
        for (int x = 0; x < 256; x++) {
            uint8_t val;
            if (model == 0) val = (uint8_t)__builtin_popcount(inv[x] ^ y);  // HD last round [S:85]
            else if (model == 1) val = (uint8_t)__builtin_popcount(inv[x]);  // HW last round
            else val = (uint8_t)__builtin_popcount(s[x]);                    // HW first round
            v[y * 256 + x] = val;
        }
}

void aes_expand_key(const uint8_t key[16], uint8_t rk[11][16])
{
    uint8_t s[256], inv[256];
    aes_sboxes(s, inv);
    std::memcpy(rk[0], key, 16);
    uint8_t rc = 1;
    for (int r = 1; r <= 10; r++) {
        const uint8_t *p = rk[r - 1];
        uint8_t t[4] = {(uint8_t)(s[p[13]] ^ rc), s[p[14]], s[p[15]], s[p[12]]};
        for (int c = 0; c < 4; c++)
            for (int i = 0; i < 4; i++) {
                uint8_t prev = c ? rk[r][4 * (c - 1) + i] : t[i];
                rk[r][4 * c + i] = p[4 * c + i] ^ prev;
            }
        rc = gmul(rc, 2);
    }
}

void aes_invert_key_schedule(const uint8_t rk_in[16], int round, uint8_t key[16])
{
    uint8_t s[256], inv[256];
    aes_sboxes(s, inv);
    uint8_t rcon[11];
    rcon[1] = 1;
    for (int i = 2; i <= 10; i++) rcon[i] = gmul(rcon[i - 1], 2);
    uint8_t cur[16];
    std::memcpy(cur, rk_in, 16);
    for (int r = round; r >= 1; r--) {
        uint8_t prev[16];
        for (int c = 3; c >= 1; c--)
            for (int i = 0; i < 4; i++) prev[4 * c + i] = cur[4 * c + i] ^ cur[4 * (c - 1) + i];
        uint8_t t[4] = {(uint8_t)(s[prev[13]] ^ rcon[r]), s[prev[14]], s[prev[15]], s[prev[12]]};
        for (int i = 0; i < 4; i++) prev[i] = cur[i] ^ t[i];
        std::memcpy(cur, prev, 16);
    }
    std::memcpy(key, cur, 16);
}

}  // namespace cpa
