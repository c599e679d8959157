// tables.h -- host-side AES helpers of libcpa (internal).
#pragma once
#include <cstdint>

namespace cpa {
void aes_sboxes(uint8_t sbox[256], uint8_t inv[256]);
void build_vtable(int model, uint8_t *v /* 256 x 256 */);
void aes_expand_key(const uint8_t key[16], uint8_t rk[11][16]);
void aes_invert_key_schedule(const uint8_t rk[16], int round, uint8_t key[16]);
}  // namespace cpa
