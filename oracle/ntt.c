/*
 * oracle/ntt.c -- RNS parameter set (C1, C2, C12) and the negacyclic NTT (C3).
 * TEST INFRASTRUCTURE ONLY (see orc.h).
 *
 * The NTT definition (C3):
 *     ntt(a)_i = sum_j a_j * psi^((2*brv(i)+1)*j)  mod q
 * i.e. evaluation of a(X) at the odd powers of psi, in bit-reversed order.
 * orc_ntt_naive is that definition written out (O(N^2)); orc_ntt_fwd is the
 * textbook iterative Cooley-Tukey network with bit-reversed psi powers,
 * checked against the naive one in tests/test_oracle_ring.py.
 */
#include "orc.h"
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* C1 "sized" primes: for bit size b, q = 2^b - t*2N + 1 for t = 1, 2, ...:
 * the first prime not already taken. */
static u64 next_prime(int bits, int log_n, const u64 *taken, int n_taken)
{
    u64 two_n = 2ull << log_n;
    for (u64 t = 1;; t++) {
        u64 q = (1ull << bits) - t * two_n + 1;
        if (!orc_is_prime(q)) continue;
        int dup = 0;
        for (int i = 0; i < n_taken; i++) if (taken[i] == q) dup = 1;
        if (!dup) return q;
    }
}

/* C1 "derived" primes: the prime p = 2N t + 1 nearest to D (ties: smaller p),
 * not already taken. */
static u64 nearest_prime(u64 D, int log_n, const u64 *taken, int n_taken)
{
    u64 two_n = 2ull << log_n;
    u64 lo = ((D - 1) / two_n) * two_n + 1;   /* largest 2Nt+1 <= D */
    u64 hi = lo + two_n;                       /* smallest 2Nt+1 > D */
    for (;;) {
        u64 cand;
        if (D - lo <= hi - D) { cand = lo; lo -= two_n; }
        else { cand = hi; hi += two_n; }
        if (!orc_is_prime(cand)) continue;
        int dup = 0;
        for (int i = 0; i < n_taken; i++) if (taken[i] == cand) dup = 1;
        if (!dup) return cand;
    }
}

/* C2: psi = x^((q-1)/2N) for the smallest x >= 2 with psi^N = -1 mod q. */
static u64 find_psi(u64 q, int log_n)
{
    u64 n = 1ull << log_n;
    for (u64 x = 2;; x++) {
        u64 psi = orc_pow(x, (q - 1) / (2 * n), q);
        if (orc_pow(psi, n, q) == q - 1) return psi;
    }
}

orc_params *orc_params_new(int log_n, int n_q, const int *q_bits, int n_p, const int *p_bits,
                           int alpha, const int *log2_anchor)
{
    if (n_q + n_p > ORC_MAXP || n_q < 1 || n_p < 1 || alpha < 1 || log2_anchor[n_q - 1] == 0) return NULL;
    orc_params *P = calloc(1, sizeof(*P));
    P->log_n = log_n;
    P->n = 1 << log_n;
    P->n_q = n_q;
    P->n_p = n_p;
    P->L = n_q - 1;
    P->alpha = alpha;
    P->dnum = (n_q + alpha - 1) / alpha;
    /* C1: q_l is "derived" when level l-1 is not anchored (its canonical scale
     * is Delta_l^2 / q_l); q_0, the other q_l and the p_k are "sized".
     * Sized primes first (q in level order, then p), then derived primes from
     * the top level down, each the NTT prime nearest to rint(Delta_l). */
    int np = n_q + n_p;
    u64 taken[ORC_MAXP];
    int nt = 0;
    for (int i = 0; i < n_q; i++) {
        int derived = i >= 1 && log2_anchor[i - 1] == 0;
        if (!derived) { P->prime[i] = next_prime(q_bits[i], log_n, taken, nt); taken[nt++] = P->prime[i]; }
    }
    for (int k = 0; k < n_p; k++) {
        P->prime[n_q + k] = next_prime(p_bits[k], log_n, taken, nt);
        taken[nt++] = P->prime[n_q + k];
    }
    /* C12 canonical scales: Delta_l = 2^anchor[l] where anchor[l] != 0 (the top
     * level must be anchored); otherwise Delta_l = (Delta_{l+1} * Delta_{l+1}) / q_{l+1},
     * the scale of a product of two level-(l+1) ciphertexts after rescaling. */
    for (int l = P->L; l >= 0; l--) {
        if (log2_anchor[l] != 0) P->scale[l] = ldexp(1.0, log2_anchor[l]);
        else P->scale[l] = (P->scale[l + 1] * P->scale[l + 1]) / (double)P->prime[l + 1];
        if (l >= 1 && log2_anchor[l - 1] == 0) {
            P->prime[l] = nearest_prime((u64)rint(P->scale[l]), log_n, taken, nt);
            taken[nt++] = P->prime[l];
        }
    }
    int N = P->n;
    for (int i = 0; i < np; i++) {
        u64 q = P->prime[i];
        P->psi[i] = find_psi(q, log_n);
        u64 ipsi = orc_inv(P->psi[i], q);
        P->psi_rev[i] = malloc(sizeof(u64) * N);
        P->ipsi_rev[i] = malloc(sizeof(u64) * N);
        for (int k = 0; k < N; k++) {
            unsigned e = orc_brv((unsigned)k, log_n);
            P->psi_rev[i][k] = orc_pow(P->psi[i], e, q);
            P->ipsi_rev[i][k] = orc_pow(ipsi, e, q);
        }
        P->n_inv[i] = orc_inv((u64)N % q, q);
    }
    for (int i = 0; i < n_q; i++) {
        u64 q = P->prime[i], pm = 1;
        for (int k = 0; k < n_p; k++) pm = orc_mul(pm, P->prime[n_q + k] % q, q);
        P->p_mod_q[i] = pm;
        P->p_inv_mod_q[i] = orc_inv(pm, q);
    }
    return P;
}

void orc_params_free(orc_params *P)
{
    if (!P) return;
    for (int i = 0; i < P->n_q + P->n_p; i++) { free(P->psi_rev[i]); free(P->ipsi_rev[i]); }
    free(P);
}

/* Forward negacyclic NTT, Cooley-Tukey, natural order in, bit-reversed out. */
void orc_ntt_fwd(const orc_params *P, int pi, u64 *a)
{
    const u64 q = P->prime[pi];
    const u64 *w = P->psi_rev[pi];
    int N = P->n, t = N;
    for (int m = 1; m < N; m <<= 1) {
        t >>= 1;
        for (int i = 0; i < m; i++) {
            u64 S = w[m + i];
            for (int j = 2 * i * t; j < 2 * i * t + t; j++) {
                u64 U = a[j], V = orc_mul(a[j + t], S, q);
                a[j] = orc_add(U, V, q);
                a[j + t] = orc_sub(U, V, q);
            }
        }
    }
    #pragma omp atomic
    orc_ledger[LG_NTT]++;
}

/* Inverse: Gentleman-Sande, bit-reversed in, natural out, times N^{-1}. */
void orc_ntt_inv(const orc_params *P, int pi, u64 *a)
{
    const u64 q = P->prime[pi];
    const u64 *w = P->ipsi_rev[pi];
    int N = P->n, t = 1;
    for (int m = N; m > 1; m >>= 1) {
        int h = m >> 1, j1 = 0;
        for (int i = 0; i < h; i++) {
            u64 S = w[h + i];
            for (int j = j1; j < j1 + t; j++) {
                u64 U = a[j], V = a[j + t];
                a[j] = orc_add(U, V, q);
                a[j + t] = orc_mul(orc_sub(U, V, q), S, q);
            }
            j1 += 2 * t;
        }
        t <<= 1;
    }
    for (int j = 0; j < N; j++) a[j] = orc_mul(a[j], P->n_inv[pi], q);
    #pragma omp atomic
    orc_ledger[LG_NTT]++;
}

/* The C3 definition, O(N^2): used only to pin orc_ntt_fwd on small N. */
void orc_ntt_naive(const orc_params *P, int pi, u64 *a)
{
    const u64 q = P->prime[pi];
    int N = P->n;
    u64 *out = calloc(N, sizeof(u64));
    for (int i = 0; i < N; i++) {
        u64 e = 2 * (u64)orc_brv((unsigned)i, P->log_n) + 1;
        u64 root = orc_pow(P->psi[pi], e, q), pw = 1, acc = 0;
        for (int j = 0; j < N; j++) {
            acc = orc_add(acc, orc_mul(a[j], pw, q), q);
            pw = orc_mul(pw, root, q);
        }
        out[i] = acc;
    }
    memcpy(a, out, sizeof(u64) * N);
    free(out);
}

/* C10: sigma_k in the NTT domain.  Slot i holds a(psi^{e_i}), e_i = 2 brv(i)+1;
 * sigma_k(a)(psi^{e_i}) = a(psi^{e_i k}), so out[i] = in[perm[i]] with
 * perm[i] = brv(((e_i * k mod 2N) - 1) / 2). */
void orc_galois_perm(const orc_params *P, int k, unsigned *perm)
{
    u64 two_n = 2ull * P->n;
    for (int i = 0; i < P->n; i++) {
        u64 e = 2 * (u64)orc_brv((unsigned)i, P->log_n) + 1;
        u64 ek = (e * (u64)k) % two_n;
        perm[i] = orc_brv((unsigned)((ek - 1) / 2), P->log_n);
    }
}
