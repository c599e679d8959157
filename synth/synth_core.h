/*
 * synth_core.h -- the per-sample value function shared by the host and device
 * synthetic generators (synth.c / synth_dev.cu).  Integer-only, so both sides
 * produce identical bits.
 */
#ifndef CPA_SYNTH_CORE_H
#define CPA_SYNTH_CORE_H
#include <stdint.h>
#include "synth.h"

#ifdef __CUDACC__
#define SY_FN static __host__ __device__ __forceinline__
#else
#define SY_FN static inline
#endif

/* splitmix64 finaliser (Steele, Lea, Flood 2014) */
SY_FN uint64_t sy_mix64(uint64_t x)
{
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

SY_FN uint64_t sy_trace_key(uint64_t seed, int64_t i)
{
    return sy_mix64(seed * 0x9E3779B97F4A7C15ULL ^ (uint64_t)i ^ 0x243F6A8885A308D3ULL);
}

/* 16-bit uniform for noise of sample (i, j) given the trace key */
SY_FN uint32_t sy_noise_u16(uint64_t tkey, int32_t j)
{
    return (uint32_t)(sy_mix64(tkey ^ ((uint64_t)(uint32_t)j * 0xD1B54A32D192ED03ULL)) >> 48);
}

SY_FN int64_t sy_mu_q32(const sy_params *p, int32_t j)
{
    uint64_t span = (uint64_t)(p->mu_hi_q32 - p->mu_lo_q32) + 1ULL;
    uint64_t r = sy_mix64(p->seed ^ 0x13198A2E03707344ULL ^ ((uint64_t)(uint32_t)j << 20));
    return p->mu_lo_q32 + (int64_t)(r % span);
}

/* value (Q32) of sample j of a trace: mu_j + a * leak (if j is a leak sample)
 * + sigma * z.  leakv: the trace's 16 planted values.                        */
SY_FN int64_t sy_value_q32(const sy_params *p, const int32_t *gauss, uint64_t tkey,
                           const uint8_t *leakv, int32_t j, int64_t mu)
{
    int64_t v = mu;
    for (int b = 0; b < 16; b++)
        if (p->leak[b] == j) v += p->a_q32 * (int64_t)leakv[b];
    v += (int64_t)gauss[sy_noise_u16(tkey, j)] * p->sigma_q16;
    return v;
}

SY_FN int8_t sy_to_s8(int64_t v)
{
    int64_t r = (v + (1LL << 31)) >> 32; /* round half up, arithmetic shift */
    if (r < -128) r = -128;
    if (r > 127) r = 127;
    return (int8_t)r;
}

SY_FN uint8_t sy_to_u8(int64_t v)
{
    int64_t r = (v + (1LL << 31)) >> 32;
    if (r < 0) r = 0;
    if (r > 255) r = 255;
    return (uint8_t)r;
}

SY_FN float sy_to_f32(int64_t v)
{
    return (float)((double)v * 2.3283064365386963e-10); /* exact: v < 2^53, x 2^-32 */
}

#endif
