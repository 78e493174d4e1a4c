/*
 * oracle/arith.c -- 64-bit modular arithmetic, primality, prime search (C1)
 * and primitive roots (C2).  TEST INFRASTRUCTURE ONLY (see orc.h).
 *
 * Everything is computed the obvious way: products in unsigned __int128 and
 * reduced with the C '%' operator.
 */
#include "orc.h"
#include <math.h>

long orc_ledger[LG_COUNT];
long orc_ks_level[ORC_MAXP];

u64 orc_mul(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
u64 orc_add(u64 a, u64 b, u64 q) { return (u64)(((u128)a + b) % q); }
u64 orc_sub(u64 a, u64 b, u64 q) { return (u64)(((u128)a + q - b) % q); }

u64 orc_pow(u64 a, u64 e, u64 q)
{
    u64 r = 1 % q;
    a %= q;
    while (e) {
        if (e & 1) r = orc_mul(r, a, q);
        a = orc_mul(a, a, q);
        e >>= 1;
    }
    return r;
}

/* q prime: Fermat inverse a^(q-2). */
u64 orc_inv(u64 a, u64 q) { return orc_pow(a, q - 2, q); }

/* Deterministic Miller-Rabin with the first 12 prime bases: exact for all
 * 64-bit integers (C1). */
int orc_is_prime(u64 n)
{
    static const u64 bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return 0;
    for (int i = 0; i < 12; i++) {
        if (n == bases[i]) return 1;
        if (n % bases[i] == 0) return 0;
    }
    u64 d = n - 1;
    int s = 0;
    while ((d & 1) == 0) { d >>= 1; s++; }
    for (int i = 0; i < 12; i++) {
        u64 x = orc_pow(bases[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int comp = 1;
        for (int r = 1; r < s; r++) {
            x = orc_mul(x, x, n);
            if (x == n - 1) { comp = 0; break; }
        }
        if (comp) return 0;
    }
    return 1;
}

unsigned orc_brv(unsigned x, int bits)
{
    unsigned r = 0;
    for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

/* Residue mod q of the integer nearest to x (round-half-even, the default
 * IEEE rounding of rint).  Used for every scalar constant (C4: "scalar
 * constants c are bit-pinned as llrint(c*scale) mod q_i").  Works for any
 * finite double: |x| >= 2^52 is already an integer m*2^e with m < 2^53. */
u64 orc_residue_of_double(double x, u64 q)
{
    double r = rint(x);
    int neg = r < 0;
    if (neg) r = -r;
    u64 res;
    if (r < 9.0e18) {
        res = ((u64)r) % q;
    } else {
        int e;
        double m = frexp(r, &e);           /* r = m * 2^e, m in [0.5,1) */
        u64 mi = (u64)ldexp(m, 53);        /* exact 53-bit integer      */
        e -= 53;                           /* r = mi * 2^e, e > 0       */
        res = orc_mul(mi % q, orc_pow(2, (u64)e, q), q);
    }
    return neg ? (res == 0 ? 0 : q - res) : res;
}
