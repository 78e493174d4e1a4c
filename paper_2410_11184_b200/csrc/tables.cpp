// tables.cpp -- host-side RNS tables of the product (independent of oracle/).
//
// DESIGN.md C1 (prime selection), C2 (psi), C3 (twiddle layout), C12
// (canonical scales).  PAPER.md gives none of these (it calls HEaaN's FGb
// preset, PAPER.md 386-411); they are our readings, shared with the oracle
// only as written conventions.
#include <math.h>

#include <algorithm>
#include <cstring>

#include "hs_internal.h"

u64 hs_mulmod(u64 a, u64 b, u64 q) { return (u64)((u128)a * b % q); }

u64 hs_powmod(u64 a, u64 e, u64 q)
{
    u64 acc = 1 % q, base = a % q;
    for (; e; e >>= 1, base = hs_mulmod(base, base, q))
        if (e & 1) acc = hs_mulmod(acc, base, q);
    return acc;
}

u64 hs_invmod(u64 a, u64 q) { return hs_powmod(a, q - 2, q); }

u64 hs_shoup_const(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }

// Miller-Rabin, bases = first 12 primes: deterministic below 3.3e24 > 2^64.
static bool probable_prime(u64 n)
{
    const u64 B[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return false;
    for (u64 b : B)
        if (n % b == 0) return n == b;
    u64 d = n - 1;
    int r = 0;
    while (!(d & 1)) d >>= 1, r++;
    for (u64 b : B) {
        u64 x = hs_powmod(b, d, n);
        if (x == 1 || x == n - 1) continue;
        bool witness = true;
        for (int i = 1; i < r && witness; i++) {
            x = hs_mulmod(x, x, n);
            if (x == n - 1) witness = false;
        }
        if (witness) return false;
    }
    return true;
}

static bool taken(const std::vector<u64> &v, u64 q) { return std::find(v.begin(), v.end(), q) != v.end(); }

// C1 sized: 2^b - t 2N + 1, t = 1, 2, ...
static u64 sized_prime(int bits, u64 two_n, const std::vector<u64> &used)
{
    for (u64 q = (1ull << bits) - two_n + 1;; q -= two_n)
        if (probable_prime(q) && !taken(used, q)) return q;
}

// C1 derived: the prime 2N t + 1 nearest to D (ties to the smaller), not used.
static u64 nearest_prime(u64 D, u64 two_n, const std::vector<u64> &used)
{
    u64 below = (D - 1) / two_n * two_n + 1, above = below + two_n;
    while (true) {
        u64 c;
        if (D - below <= above - D) {
            c = below;
            below -= two_n;
        } else {
            c = above;
            above += two_n;
        }
        if (probable_prime(c) && !taken(used, c)) return c;
    }
}

// C2: psi = x^((q-1)/2N), x = 2, 3, ... the first with psi^N = -1.
static u64 root_2n(u64 q, u64 n)
{
    for (u64 x = 2;; x++) {
        u64 g = hs_powmod(x, (q - 1) / (2 * n), q);
        if (hs_powmod(g, n, q) == q - 1) return g;
    }
}

static unsigned bitrev(unsigned v, int bits)
{
    unsigned r = 0;
    for (int i = 0; i < bits; i++, v >>= 1) r = (r << 1) | (v & 1);
    return r;
}

u64 hs_residue_of_double(double x, u64 q)
{
    double r = rint(x);  // round-half-even
    bool neg = std::signbit(r);
    r = fabs(r);
    u64 m;
    if (r < 9.0e18) {
        m = (u64)r % q;
    } else {
        int e;
        double f = frexp(r, &e);
        u64 mant = (u64)ldexp(f, 53);
        m = hs_mulmod(mant % q, hs_powmod(2, (u64)(e - 53), q), q);
    }
    return (neg && m) ? q - m : m;
}

int hs_galois_elt(const hs_params *P, int r)
{
    int n0 = P->n / 2;
    r = ((r % n0) + n0) % n0;
    return (int)hs_powmod(5, (u64)r, 2ull * P->n);
}

void hs_build_params(const hs_params_desc *d, hs_params *P)
{
    if (!d || d->log_n < 3 || d->log_n > 17 || d->n_q < 1 || d->n_p < 1 || d->alpha < 1 ||
        d->n_q + d->n_p > HS_MAXP || !d->q_bits || !d->p_bits || !d->log2_anchor || d->log2_anchor[d->n_q - 1] == 0)
        throw HsError(HS_EINVAL, "hs_ckks_params: inconsistent descriptor");
    for (int i = 0; i < d->n_q; i++)
        if (d->q_bits[i] < 20 || d->q_bits[i] > 60) throw HsError(HS_EINVAL, "Q prime bits must be in [20, 60]");
    for (int i = 0; i < d->n_p; i++)
        if (d->p_bits[i] < 20 || d->p_bits[i] > 61) throw HsError(HS_EINVAL, "P prime bits must be in [20, 61]");
    // key-switch limits: the ModUp / inner-product argument blocks
    // hold HS_MAXDIG digit offsets; BConv folds at most 9 sources; every
    // digit block is alpha primes wide and the extended basis has n_p special
    // primes, which the kernels take to be the same count.
    const int dnum = (d->n_q + d->alpha - 1) / d->alpha;
    if (d->n_p != d->alpha) throw HsError(HS_EINVAL, "hs_ckks_params: n_p must equal alpha");
    if (d->alpha > 9) throw HsError(HS_EINVAL, "hs_ckks_params: alpha > 9 (BConv source limit)");
    if (dnum > HS_MAXDIG) throw HsError(HS_EINVAL, "hs_ckks_params: more than 16 key-switch digits");
    P->log_n = d->log_n;
    P->n = 1 << d->log_n;
    P->n_q = d->n_q;
    P->n_p = d->n_p;
    P->L = d->n_q - 1;
    P->alpha = d->alpha;
    P->dnum = (d->n_q + d->alpha - 1) / d->alpha;
    const u64 two_n = 2ull * P->n;
    const int np = d->n_q + d->n_p;
    P->prime.assign(np, 0);
    P->scale.assign(d->n_q, 0.0);
    std::vector<u64> used;
    auto is_derived = [&](int l) { return l >= 1 && d->log2_anchor[l - 1] == 0; };
    for (int l = 0; l < d->n_q; l++)
        if (!is_derived(l)) used.push_back(P->prime[l] = sized_prime(d->q_bits[l], two_n, used));
    for (int k = 0; k < d->n_p; k++) used.push_back(P->prime[d->n_q + k] = sized_prime(d->p_bits[k], two_n, used));
    for (int l = P->L; l >= 0; l--) {
        P->scale[l] = d->log2_anchor[l] ? ldexp(1.0, d->log2_anchor[l])
                                        : (P->scale[l + 1] * P->scale[l + 1]) / (double)P->prime[l + 1];
        if (is_derived(l)) used.push_back(P->prime[l] = nearest_prime((u64)rint(P->scale[l]), two_n, used));
    }
    // per-prime constants and twiddles
    const int N = P->n;
    P->psi.resize(np);
    P->pk.resize(np);
    P->tw.resize(np);
    P->n_inv.resize(np);
    P->n_inv_sh.resize(np);
    for (int i = 0; i < np; i++) {
        u64 q = P->prime[i];
        u64 g = root_2n(q, N), gi = hs_invmod(g, q);
        P->psi[i] = g;
        u64 qinv = 1;  // q^{-1} mod 2^64 by Newton
        for (int it = 0; it < 6; it++) qinv *= 2 - q * qinv;
        u64 r64 = (u64)(((u128)1 << 64) % q);
        P->pk[i] = PrimeK{q, (u64)(0 - qinv), r64, hs_shoup_const(r64, q)};
        std::vector<u64> &t = P->tw[i];
        t.assign((size_t)4 * N, 0);
        // powers psi^e for e < N, then index by bit reversal
        std::vector<u64> pw(N), ipw(N);
        pw[0] = ipw[0] = 1;
        for (int e = 1; e < N; e++) {
            pw[e] = hs_mulmod(pw[e - 1], g, q);
            ipw[e] = hs_mulmod(ipw[e - 1], gi, q);
        }
        for (int k = 0; k < N; k++) {
            unsigned e = bitrev((unsigned)k, d->log_n);
            t[k] = pw[e];
            t[N + k] = hs_shoup_const(pw[e], q);
            t[2 * N + k] = ipw[e];
            t[3 * N + k] = hs_shoup_const(ipw[e], q);
        }
        P->n_inv[i] = hs_invmod((u64)N % q, q);
        P->n_inv_sh[i] = hs_shoup_const(P->n_inv[i], q);
    }
    // lazy 128-bit accumulation of the evk inner product: dnum products plus
    // the fused P*d term (C8), each <= (q-1)^2, reduced by d_reduce128, whose
    // REDC step needs the high word below 2^64 - q (kernels.cu)
    for (int i = 0; i < np; i++) {
        const u64 q = P->prime[i];
        const u128 worst = (u128)(dnum + 1) * (u128)(q - 1) * (u128)(q - 1);
        if (worst >= ((u128)(~0ull - q) << 64))
            throw HsError(HS_EINVAL, "hs_ckks_params: dnum too large for the 128-bit inner-product accumulator");
    }
    P->p_mod_q.resize(d->n_q);
    P->p_inv_mod_q.resize(d->n_q);
    for (int l = 0; l < d->n_q; l++) {
        u64 q = P->prime[l], prod = 1;
        for (int k = 0; k < d->n_p; k++) prod = hs_mulmod(prod, P->prime[d->n_q + k] % q, q);
        P->p_mod_q[l] = prod;
        P->p_inv_mod_q[l] = hs_invmod(prod, q);
    }
}
