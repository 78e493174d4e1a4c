/*
 * oracle/rng.c -- the counter-based randomness of DESIGN.md C5.
 * TEST INFRASTRUCTURE ONLY (see orc.h).
 *
 * ChaCha20 block function exactly as RFC 8439 section 2.3 (pinned by the
 * RFC's test vector in tests/golden/chacha20_rfc8439.txt).
 * stream(seed, tag, sub, idx) is the idx-th little-endian 64-bit word of the
 * keystream with key = (lo32(seed), hi32(seed), tag, lo32(sub), hi32(sub),
 * 0, 0, 0), nonce = (0, 0, 0), block counter = idx >> 3.
 */
#include "orc.h"

static uint32_t rotl(uint32_t x, int n) { return (x << n) | (x >> (32 - n)); }
#define QR(a, b, c, d)                    \
    a += b; d ^= a; d = rotl(d, 16);      \
    c += d; b ^= c; b = rotl(b, 12);      \
    a += b; d ^= a; d = rotl(d, 8);       \
    c += d; b ^= c; b = rotl(b, 7);

void orc_chacha20_block(const uint32_t key[8], uint32_t counter, const uint32_t nonce[3], uint32_t out[16])
{
    uint32_t s[16] = {0x61707865, 0x3320646e, 0x79622d32, 0x6b206574,
                      key[0], key[1], key[2], key[3], key[4], key[5], key[6], key[7],
                      counter, nonce[0], nonce[1], nonce[2]};
    uint32_t x[16];
    for (int i = 0; i < 16; i++) x[i] = s[i];
    for (int r = 0; r < 10; r++) {
        QR(x[0], x[4], x[8], x[12]);
        QR(x[1], x[5], x[9], x[13]);
        QR(x[2], x[6], x[10], x[14]);
        QR(x[3], x[7], x[11], x[15]);
        QR(x[0], x[5], x[10], x[15]);
        QR(x[1], x[6], x[11], x[12]);
        QR(x[2], x[7], x[8], x[13]);
        QR(x[3], x[4], x[9], x[14]);
    }
    for (int i = 0; i < 16; i++) out[i] = x[i] + s[i];
}

u64 orc_stream(u64 seed, uint32_t tag, u64 sub, u64 idx)
{
    uint32_t key[8] = {(uint32_t)seed, (uint32_t)(seed >> 32), tag, (uint32_t)sub,
                       (uint32_t)(sub >> 32), 0, 0, 0};
    uint32_t nonce[3] = {0, 0, 0}, out[16];
    orc_chacha20_block(key, (uint32_t)(idx >> 3), nonce, out);
    int w = (int)(idx & 7);
    return (u64)out[2 * w] | ((u64)out[2 * w + 1] << 32);
}

/* Uniform mod q from two stream words (2*idx2, 2*idx2+1): (w1*2^64 + w0) mod q.
 * The bias is at most q/2^128. */
u64 orc_uniform_mod(u64 seed, uint32_t tag, u64 sub, u64 idx2, u64 q)
{
    u64 w0 = orc_stream(seed, tag, sub, 2 * idx2);
    u64 w1 = orc_stream(seed, tag, sub, 2 * idx2 + 1);
    return (u64)((((u128)w1 << 64) | w0) % q);
}

/* Centred binomial with parameter eta <= 32 from one 64-bit word:
 * popcount(low eta bits) - popcount(next eta bits). */
int orc_cbd(u64 w, int eta)
{
    u64 m = (eta == 64) ? ~0ull : ((1ull << eta) - 1);
    return __builtin_popcountll(w & m) - __builtin_popcountll((w >> eta) & m);
}
