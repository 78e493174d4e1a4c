/*
 * oracle/encode.c -- CKKS canonical-embedding encode/decode in quad precision
 * (C4).  TEST INFRASTRUCTURE ONLY (see orc.h).
 *
 * Slot j <-> evaluation at zeta^(g_j), zeta = exp(i*pi/N), g_j = 5^j mod 2N,
 * j < N0 = N/2 (section 2.2: messages are C^{N/2}).
 * Encode: m_t = rint( Delta * (2/N) * Re( sum_j z_j zeta^(-g_j t) ) ), t < N.
 * With w[e] = z_j at e = g_j (zero elsewhere) the sum is the length-2N DFT
 * X[t] = sum_e w[e] exp(-2 pi i e t / 2N); it is computed by a plain radix-2
 * FFT in __float128 (pinned against the naive DFT in tests).  Computing in
 * quad makes the rounding decision agree with any other >= 100-bit-accurate
 * evaluation except on a set of inputs of measure ~2^-45 per coefficient.
 */
#include "orc.h"
#include <quadmath.h>
#include <stdlib.h>
#include <string.h>

typedef struct { __float128 re, im; } qc;

static int tw_logn = -1;
static qc *tw = NULL; /* exp(-2 pi i k / 2N), k < N */

static void ensure_twiddles(int log_n)
{
    if (tw_logn == log_n) return;
    free(tw);
    int n2 = 2 << log_n;
    tw = malloc(sizeof(qc) * (n2 / 2));
    for (int k = 0; k < n2 / 2; k++) {
        __float128 ang = -2 * M_PIq * (__float128)k / (__float128)n2;
        tw[k].re = cosq(ang);
        tw[k].im = sinq(ang);
    }
    tw_logn = log_n;
}

/* In-place iterative radix-2 DFT of length n2 = 2N, sign = -1 (forward, the
 * twiddle table) or +1 (conjugate twiddles). */
static void fft(qc *a, int log_n2, int sign)
{
    int n2 = 1 << log_n2;
    for (int i = 0; i < n2; i++) {
        int j = (int)orc_brv((unsigned)i, log_n2);
        if (j > i) { qc t = a[i]; a[i] = a[j]; a[j] = t; }
    }
    for (int len = 2; len <= n2; len <<= 1) {
        int step = n2 / len;
        for (int s = 0; s < n2; s += len) {
            for (int k = 0; k < len / 2; k++) {
                qc w = tw[k * step];
                if (sign > 0) w.im = -w.im;
                qc u = a[s + k], v = a[s + k + len / 2];
                qc vw = {v.re * w.re - v.im * w.im, v.re * w.im + v.im * w.re};
                a[s + k].re = u.re + vw.re;
                a[s + k].im = u.im + vw.im;
                a[s + k + len / 2].re = u.re - vw.re;
                a[s + k + len / 2].im = u.im - vw.im;
            }
        }
    }
}

static void encode_finish(const orc_params *P, qc *w, double scale, int level, int with_p, u64 *out);

/* out: (level+1) limbs of N residues, coefficient domain. */
void orc_encode_coeffs(const orc_params *P, const double *re, const double *im, double scale, int level, u64 *out)
{
    int N = P->n, N0 = N / 2, n2 = 2 * N;
    ensure_twiddles(P->log_n);
    qc *w = calloc(n2, sizeof(qc));
    u64 g = 1;
    for (int j = 0; j < N0; j++) {
        w[g].re = re[j];
        w[g].im = im ? im[j] : 0;
        g = (g * 5) % (u64)n2;
    }
    encode_finish(P, w, scale, level, 0, out);
}

/* the same from quad-precision slot values (bootstrapping diagonals, G11) */
void orc_encode_coeffs_q(const orc_params *P, const __float128 *re, const __float128 *im, double scale, int level,
                         u64 *out)
{
    int N = P->n, N0 = N / 2, n2 = 2 * N;
    ensure_twiddles(P->log_n);
    qc *w = calloc(n2, sizeof(qc));
    u64 g = 1;
    for (int j = 0; j < N0; j++) {
        w[g].re = re[j];
        w[g].im = im[j];
        g = (g * 5) % (u64)n2;
    }
    encode_finish(P, w, scale, level, 0, out);
}

/* ... and in the extended basis Q_level u P: limbs q_0..q_level then p_0..p_{np-1}
 * of the same integer coefficients (C17 double-hoisted BSGS plaintexts) */
void orc_encode_coeffs_q_pq(const orc_params *P, const __float128 *re, const __float128 *im, double scale, int level,
                            u64 *out)
{
    int N = P->n, N0 = N / 2, n2 = 2 * N;
    ensure_twiddles(P->log_n);
    qc *w = calloc(n2, sizeof(qc));
    u64 g = 1;
    for (int j = 0; j < N0; j++) {
        w[g].re = re[j];
        w[g].im = im[j];
        g = (g * 5) % (u64)n2;
    }
    encode_finish(P, w, scale, level, 1, out);
}

static void encode_finish(const orc_params *P, qc *w, double scale, int level, int with_p, u64 *out)
{
    int N = P->n;
    fft(w, P->log_n + 1, -1);
    __float128 f = (__float128)scale * 2 / (__float128)N;
    for (int t = 0; t < N; t++) {
        __float128 v = rintq(w[t].re * f);
        i128 m = (i128)v;
        for (int i = 0; i <= level; i++) {
            i128 q = (i128)P->prime[i];
            i128 r = m % q;
            if (r < 0) r += q;
            out[(size_t)i * N + t] = (u64)r;
        }
        for (int k = 0; with_p && k < P->n_p; k++) {
            i128 q = (i128)P->prime[P->n_q + k];
            i128 r = m % q;
            if (r < 0) r += q;
            out[(size_t)(level + 1 + k) * N + t] = (u64)r;
        }
    }
    free(w);
}

/* coeff: N signed integer coefficients; z_j = (1/scale) sum_t m_t zeta^(g_j t). */
void orc_decode_coeffs(const orc_params *P, const i128 *coeff, double scale, double *re, double *im)
{
    int N = P->n, N0 = N / 2, n2 = 2 * N;
    ensure_twiddles(P->log_n);
    qc *w = calloc(n2, sizeof(qc));
    for (int t = 0; t < N; t++) w[t].re = (__float128)coeff[t];
    fft(w, P->log_n + 1, +1);
    u64 g = 1;
    for (int j = 0; j < N0; j++) {
        re[j] = (double)(w[g].re / (__float128)scale);
        if (im) im[j] = (double)(w[g].im / (__float128)scale);
        g = (g * 5) % (u64)n2;
    }
    free(w);
}

/* Naive O(N*N0) encode value (before rounding), for the FFT pin in tests:
 * returns Delta*(2/N)*Re(sum_j z_j zeta^(-g_j t)) as a double. */
double orc_encode_naive_coeff(const orc_params *P, const double *re, const double *im, double scale, int t)
{
    int N = P->n, N0 = N / 2;
    __float128 acc = 0;
    u64 g = 1;
    for (int j = 0; j < N0; j++) {
        __float128 ang = -M_PIq * (__float128)((g * (u64)t) % (2ull * N)) / (__float128)N;
        acc += (__float128)re[j] * cosq(ang) - (__float128)(im ? im[j] : 0) * sinq(ang);
        g = (g * 5) % (2ull * N);
    }
    return (double)(acc * (__float128)scale * 2 / (__float128)N);
}
