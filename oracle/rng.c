/*
 * rng.c -- oracle (TEST INFRASTRUCTURE ONLY): the counter-based random-number
 * contract R1/R2 that every sampling step of the method draws from.
 *
 * The paper does not fix an RNG (walks P:67-69, EdgeSample P:74,
 * NegativeSample P:76 are unspecified); reading R1 fixes
 * Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11) so that the CPU oracle and
 * the GPU path can draw identical numbers from independent implementations.
 */
#include "ne_oracle.h"

/* Philox4x32 constants, as published by Salmon et al. (SC'11, Table 2 / the
 * Random123 reference implementation). */
#define OR_PHILOX_M0 0xD2511F53u
#define OR_PHILOX_M1 0xCD9E8D57u
#define OR_PHILOX_W0 0x9E3779B9u
#define OR_PHILOX_W1 0xBB67AE85u

/* One Philox4x32 round: two 32x32->64 multiplies, then the S-box/P-box
 * permutation (hi1^c1^k0, lo1, hi0^c3^k1, lo0). */
static void philox_round(uint32_t c[4], const uint32_t k[2])
{
    uint64_t p0 = (uint64_t)OR_PHILOX_M0 * (uint64_t)c[0];
    uint64_t p1 = (uint64_t)OR_PHILOX_M1 * (uint64_t)c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k[0];
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c[3] ^ k[1];
    uint32_t n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
}

/* R1: Philox4x32-10.  Round r (r = 0..9) uses key + r*(W0, W1). */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c[4] = { ctr[0], ctr[1], ctr[2], ctr[3] };
    uint32_t k[2] = { key[0], key[1] };
    int r;
    for (r = 0; r < 10; ++r) {
        if (r > 0) { k[0] += OR_PHILOX_W0; k[1] += OR_PHILOX_W1; }
        philox_round(c, k);
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

/* R2: uniform index in [0, n) from a 64-bit draw: floor(r64 * n / 2^64).
 * (Bias <= n / 2^64; a 32-bit multiply-high would be biased by up to n/2^32.) */
uint64_t or_uniform_index(uint64_t r64, uint64_t n)
{
    unsigned __int128 prod = (unsigned __int128)r64 * (unsigned __int128)n;
    return (uint64_t)(prod >> 64);
}
