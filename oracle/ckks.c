/*
 * oracle/ckks.c -- RNS-CKKS scheme operations of the oracle.
 * TEST INFRASTRUCTURE ONLY (see orc.h).
 *
 * PAPER.md section 2.2.1 (lines 262-271) lists the functionalities: KeyGen,
 * Enc, Dec, Add, Mult, Rot.  The paper delegates all of them to HEaaN
 * (line 386), so each convention below is a DESIGN.md reading:
 *   C5 randomness, C6 pk/Enc, C7 hybrid key switching, C8 HMult,
 *   C9 rescale, C10 rotation, C11 operand levels, C12 canonical scales.
 * Ciphertexts are kept in the NTT domain, limb-major.
 */
#include "orc.h"
#include <stdlib.h>
#include <string.h>
#include <math.h>

enum { TAG_SK = 1, TAG_PK_A = 2, TAG_PK_E = 3, TAG_KSK_A = 4, TAG_KSK_E = 5,
       TAG_ENC_V = 6, TAG_ENC_E0 = 7, TAG_ENC_E1 = 8, TAG_ENC_A = 9 };
#define ETA_ERR 21
#define ETA_V 1

orc_ct *orc_ct_alloc(const orc_params *P, int level, int ncomp)
{
    orc_ct *c = malloc(sizeof(*c));
    c->level = level;
    c->ncomp = ncomp;
    c->a = calloc((size_t)ncomp * (level + 1) * P->n, sizeof(u64));
    return c;
}

orc_ct *orc_ct_copy(const orc_params *P, const orc_ct *s)
{
    orc_ct *c = orc_ct_alloc(P, s->level, s->ncomp);
    memcpy(c->a, s->a, sizeof(u64) * (size_t)s->ncomp * (s->level + 1) * P->n);
    return c;
}

void orc_ct_release(orc_ct *c)
{
    if (!c) return;
    free(c->a);
    free(c);
}

/* keep limbs 0..level (exact: the value mod Q_level is unchanged) */
static orc_ct *drop_limbs(const orc_params *P, const orc_ct *s, int level)
{
    orc_ct *c = orc_ct_alloc(P, level, s->ncomp);
    for (int k = 0; k < s->ncomp; k++)
        for (int i = 0; i <= level; i++)
            memcpy(LIMB(P, c, k, i), LIMB(P, s, k, i), sizeof(u64) * P->n);
    return c;
}

/* ---------------------------------------------------------------- keys (C5, C6, C7) */

/* integer coefficient vector -> NTT-domain residues for prime index pi */
static void int_to_ntt(const orc_params *P, const int64_t *v, int pi, u64 *out)
{
    u64 q = P->prime[pi];
    for (int t = 0; t < P->n; t++) {
        int64_t x = v[t] % (int64_t)q;
        out[t] = (u64)(x < 0 ? x + (int64_t)q : x);
    }
    orc_ntt_fwd(P, pi, out);
}

static void sample_cbd_vec(const orc_params *P, u64 seed, uint32_t tag, u64 sub, int eta, int64_t *out)
{
    for (int t = 0; t < P->n; t++) out[t] = orc_cbd(orc_stream(seed, tag, sub, (u64)t), eta);
}

/* sparse ternary secret with exactly h non-zeros: partial Fisher-Yates over
 * positions, word 2i picks j = i + w mod (N-i), bit 0 of word 2i+1 the sign. */
static void sample_secret(const orc_params *P, u64 seed, int h, int64_t *s)
{
    int N = P->n;
    int *perm = malloc(sizeof(int) * N);
    for (int i = 0; i < N; i++) perm[i] = i;
    memset(s, 0, sizeof(int64_t) * N);
    for (int i = 0; i < h; i++) {
        u64 w = orc_stream(seed, TAG_SK, 0, 2 * (u64)i);
        int j = i + (int)(w % (u64)(N - i));
        int t = perm[i]; perm[i] = perm[j]; perm[j] = t;
        u64 sg = orc_stream(seed, TAG_SK, 0, 2 * (u64)i + 1);
        s[perm[i]] = (sg & 1) ? -1 : 1;
    }
    free(perm);
}

/* C7: evk_j = (-a_j s + e_j + [i in D_j] (P mod q_i) s', a_j) over Q_L u P. */
static void make_swk(const orc_params *P, const orc_keys *K, u64 seed, int key_id, const u64 *sprime, orc_swk *out)
{
    int N = P->n, nt = P->n_q + P->n_p;
    out->galois = key_id;
    out->dnum = P->dnum;
    out->k = malloc(sizeof(u64) * (size_t)P->dnum * 2 * nt * N);
    int64_t *e = malloc(sizeof(int64_t) * N);
    for (int j = 0; j < P->dnum; j++) {
        u64 sub = (u64)key_id * 256 + (u64)j;
        sample_cbd_vec(P, seed, TAG_KSK_E, sub, ETA_ERR, e);
        #pragma omp parallel for
        for (int i = 0; i < nt; i++) {
            u64 q = P->prime[i];
            u64 *k0 = out->k + (((size_t)j * 2 + 0) * nt + i) * N;
            u64 *k1 = out->k + (((size_t)j * 2 + 1) * nt + i) * N;
            int_to_ntt(P, e, i, k0);  /* k0 = e_j (NTT) */
            const u64 *s = K->s_ntt + (size_t)i * N;
            int in_digit = (i < P->n_q) && (i / P->alpha == j);
            for (int t = 0; t < N; t++) {
                u64 a = orc_uniform_mod(seed, TAG_KSK_A, sub, (u64)i * N + t, q);
                k1[t] = a;
                u64 v = orc_sub(k0[t], orc_mul(a, s[t], q), q);
                if (in_digit) v = orc_add(v, orc_mul(P->p_mod_q[i], sprime[(size_t)i * N + t], q), q);
                k0[t] = v;
            }
        }
    }
    free(e);
}

int orc_galois_of_rot(const orc_params *P, int r)
{
    int N0 = P->n / 2;
    r %= N0;
    if (r < 0) r += N0;
    return (int)orc_pow(5, (u64)r, 2ull * P->n);
}

orc_keys *orc_keygen(const orc_params *P, u64 seed, int h, const int *galois, int n_galois, int relin)
{
    int N = P->n, nt = P->n_q + P->n_p;
    orc_keys *K = calloc(1, sizeof(*K));
    K->s_coeff = malloc(sizeof(int64_t) * N);
    sample_secret(P, seed, h, K->s_coeff);
    K->s_ntt = malloc(sizeof(u64) * (size_t)nt * N);
    #pragma omp parallel for
    for (int i = 0; i < nt; i++) int_to_ntt(P, K->s_coeff, i, K->s_ntt + (size_t)i * N);
    /* pk over Q_L */
    K->pk = malloc(sizeof(u64) * 2 * (size_t)P->n_q * N);
    int64_t *e = malloc(sizeof(int64_t) * N);
    sample_cbd_vec(P, seed, TAG_PK_E, 0, ETA_ERR, e);
    #pragma omp parallel for
    for (int i = 0; i < P->n_q; i++) {
        u64 q = P->prime[i];
        u64 *b = K->pk + (size_t)i * N, *a = K->pk + ((size_t)P->n_q + i) * N;
        int_to_ntt(P, e, i, b);
        for (int t = 0; t < N; t++) {
            a[t] = orc_uniform_mod(seed, TAG_PK_A, 0, (u64)i * N + t, q);
            b[t] = orc_sub(b[t], orc_mul(a[t], K->s_ntt[(size_t)i * N + t], q), q);
        }
    }
    free(e);
    K->n_swk = n_galois + (relin ? 1 : 0);
    K->swk = calloc(K->n_swk, sizeof(orc_swk));
    u64 *sp = malloc(sizeof(u64) * (size_t)nt * N);
    unsigned *perm = malloc(sizeof(unsigned) * N);
    int w = 0;
    if (relin) {
        for (size_t x = 0; x < (size_t)nt * N; x++) {
            u64 q = P->prime[x / N];
            sp[x] = orc_mul(K->s_ntt[x], K->s_ntt[x], q);
        }
        make_swk(P, K, seed, 0, sp, &K->swk[w++]);
    }
    for (int g = 0; g < n_galois; g++) {
        orc_galois_perm(P, galois[g], perm);
        for (int i = 0; i < nt; i++)
            for (int t = 0; t < N; t++) sp[(size_t)i * N + t] = K->s_ntt[(size_t)i * N + perm[t]];
        make_swk(P, K, seed, galois[g], sp, &K->swk[w++]);
    }
    free(sp);
    free(perm);
    return K;
}

void orc_keys_free(orc_keys *K)
{
    if (!K) return;
    for (int i = 0; i < K->n_swk; i++) free(K->swk[i].k);
    free(K->swk);
    free(K->s_coeff);
    free(K->s_ntt);
    free(K->pk);
    free(K);
}

const orc_swk *orc_find_key(const orc_keys *K, int galois)
{
    for (int i = 0; i < K->n_swk; i++)
        if (K->swk[i].galois == galois) return &K->swk[i];
    return NULL;
}

/* ---------------------------------------------------------------- Enc / Dec (C6) */

/* pt: (level+1) limbs of coefficient-domain residues. */
orc_ct *orc_encrypt_pk(const orc_params *P, const orc_keys *K, const u64 *pt, int level, u64 seed, u64 ct_index)
{
    int N = P->n;
    orc_ct *c = orc_ct_alloc(P, level, 2);
    int64_t *v = malloc(sizeof(int64_t) * N), *e0 = malloc(sizeof(int64_t) * N), *e1 = malloc(sizeof(int64_t) * N);
    sample_cbd_vec(P, seed, TAG_ENC_V, ct_index, ETA_V, v);
    sample_cbd_vec(P, seed, TAG_ENC_E0, ct_index, ETA_ERR, e0);
    sample_cbd_vec(P, seed, TAG_ENC_E1, ct_index, ETA_ERR, e1);
    #pragma omp parallel for
    for (int i = 0; i <= level; i++) {
        u64 q = P->prime[i];
        u64 *vn = malloc(sizeof(u64) * N), *m = malloc(sizeof(u64) * N);
        int_to_ntt(P, v, i, vn);
        memcpy(m, pt + (size_t)i * N, sizeof(u64) * N);
        orc_ntt_fwd(P, i, m);
        u64 *c0 = LIMB(P, c, 0, i), *c1 = LIMB(P, c, 1, i);
        int_to_ntt(P, e0, i, c0);
        int_to_ntt(P, e1, i, c1);
        const u64 *b = K->pk + (size_t)i * N, *a = K->pk + ((size_t)P->n_q + i) * N;
        for (int t = 0; t < N; t++) {
            c0[t] = orc_add(orc_add(c0[t], orc_mul(vn[t], b[t], q), q), m[t], q);
            c1[t] = orc_add(c1[t], orc_mul(vn[t], a[t], q), q);
        }
        free(vn);
        free(m);
    }
    free(v); free(e0); free(e1);
    return c;
}

orc_ct *orc_encrypt_sk(const orc_params *P, const orc_keys *K, const u64 *pt, int level, u64 seed, u64 ct_index)
{
    int N = P->n;
    orc_ct *c = orc_ct_alloc(P, level, 2);
    int64_t *e = malloc(sizeof(int64_t) * N);
    sample_cbd_vec(P, seed, TAG_ENC_E0, ct_index, ETA_ERR, e);
    #pragma omp parallel for
    for (int i = 0; i <= level; i++) {
        u64 q = P->prime[i];
        u64 *m = malloc(sizeof(u64) * N);
        memcpy(m, pt + (size_t)i * N, sizeof(u64) * N);
        orc_ntt_fwd(P, i, m);
        u64 *c0 = LIMB(P, c, 0, i), *c1 = LIMB(P, c, 1, i);
        int_to_ntt(P, e, i, c0);
        for (int t = 0; t < N; t++) {
            u64 a = orc_uniform_mod(seed, TAG_ENC_A, ct_index, (u64)i * N + t, q);
            c1[t] = a;
            c0[t] = orc_add(orc_sub(c0[t], orc_mul(a, K->s_ntt[(size_t)i * N + t], q), q), m[t], q);
        }
        free(m);
    }
    free(e);
    return c;
}

/* m = c0 + c1 s mod Q_l, returned as coefficient-domain residues (l+1 limbs). */
void orc_decrypt(const orc_params *P, const orc_keys *K, const orc_ct *c, u64 *out)
{
    int N = P->n;
    #pragma omp parallel for
    for (int i = 0; i <= c->level; i++) {
        u64 q = P->prime[i];
        const u64 *c0 = LIMB(P, c, 0, i), *c1 = LIMB(P, c, 1, i);
        u64 *o = out + (size_t)i * N;
        for (int t = 0; t < N; t++) o[t] = orc_add(c0[t], orc_mul(c1[t], K->s_ntt[(size_t)i * N + t], q), q);
        orc_ntt_inv(P, i, o);
    }
}

/* ---------------------------------------------------------------- arithmetic */

orc_ct *orc_op_level_down(const orc_params *P, const orc_ct *a, int target)
{
    if (a->level == target) return orc_ct_copy(P, a);
    orc_ledger[LG_LEVELDOWN]++;
    return orc_op_mult_const(P, a, 1.0, target);
}

static void match_levels(const orc_params *P, const orc_ct *a, const orc_ct *b, orc_ct **a2, orc_ct **b2)
{
    int l = a->level < b->level ? a->level : b->level;
    *a2 = orc_op_level_down(P, a, l);
    *b2 = orc_op_level_down(P, b, l);
}

static orc_ct *addsub(const orc_params *P, const orc_ct *a0, const orc_ct *b0, int sub)
{
    orc_ct *a, *b;
    match_levels(P, a0, b0, &a, &b);
    int nc = a->ncomp > b->ncomp ? a->ncomp : b->ncomp;
    orc_ct *c = orc_ct_alloc(P, a->level, nc);
    for (int k = 0; k < nc; k++)
        for (int i = 0; i <= a->level; i++) {
            u64 q = P->prime[i];
            u64 *o = LIMB(P, c, k, i);
            for (int t = 0; t < P->n; t++) {
                u64 x = k < a->ncomp ? LIMB(P, a, k, i)[t] : 0;
                u64 y = k < b->ncomp ? LIMB(P, b, k, i)[t] : 0;
                o[t] = sub ? orc_sub(x, y, q) : orc_add(x, y, q);
            }
        }
    orc_ct_release(a);
    orc_ct_release(b);
    return c;
}

orc_ct *orc_op_add(const orc_params *P, const orc_ct *a, const orc_ct *b) { return addsub(P, a, b, 0); }
orc_ct *orc_op_sub(const orc_params *P, const orc_ct *a, const orc_ct *b) { return addsub(P, a, b, 1); }

orc_ct *orc_op_mult_int(const orc_params *P, const orc_ct *a, int64_t c)
{
    orc_ct *r = orc_ct_copy(P, a);
    for (int k = 0; k < a->ncomp; k++)
        for (int i = 0; i <= a->level; i++) {
            u64 q = P->prime[i];
            int64_t cm = c % (int64_t)q;
            u64 cu = (u64)(cm < 0 ? cm + (int64_t)q : cm);
            u64 *o = LIMB(P, r, k, i);
            for (int t = 0; t < P->n; t++) o[t] = orc_mul(o[t], cu, q);
        }
    return r;
}

/* c0 += rint(c * Delta_l) (a constant polynomial is constant in the NTT domain) */
orc_ct *orc_op_add_const(const orc_params *P, const orc_ct *a, double c)
{
    orc_ct *r = orc_ct_copy(P, a);
    double v = c * P->scale[a->level];
    for (int i = 0; i <= a->level; i++) {
        u64 q = P->prime[i], C = orc_residue_of_double(v, q);
        u64 *o = LIMB(P, r, 0, i);
        for (int t = 0; t < P->n; t++) o[t] = orc_add(o[t], C, q);
    }
    return r;
}

/* C9: a'_i = (a_i - [a_l]_centred) * q_l^{-1} mod q_i */
orc_ct *orc_op_rescale(const orc_params *P, const orc_ct *a)
{
    int l = a->level, N = P->n;
    orc_ct *r = orc_ct_alloc(P, l - 1, a->ncomp);
    u64 ql = P->prime[l];
    u64 *last = malloc(sizeof(u64) * N);
    for (int k = 0; k < a->ncomp; k++) {
        memcpy(last, LIMB(P, a, k, l), sizeof(u64) * N);
        orc_ntt_inv(P, l, last);
        #pragma omp parallel for
        for (int i = 0; i < l; i++) {
            u64 q = P->prime[i], qinv = orc_inv(ql % q, q);
            u64 *v = malloc(sizeof(u64) * N);
            for (int t = 0; t < N; t++) {
                u64 x = last[t];
                if (x <= (ql - 1) / 2) v[t] = x % q;             /* centred rep >= 0 */
                else v[t] = orc_sub(0, (ql - x) % q, q);         /* centred rep < 0  */
            }
            orc_ntt_fwd(P, i, v);
            const u64 *ai = LIMB(P, a, k, i);
            u64 *o = LIMB(P, r, k, i);
            for (int t = 0; t < N; t++) o[t] = orc_mul(orc_sub(ai[t], v[t], q), qinv, q);
            free(v);
        }
    }
    free(last);
    orc_ledger[LG_RESCALE]++;
    return r;
}

/* C12: multiply by a real constant and land at level `target` < level with the
 * canonical scale: drop to target+1, multiply by rint(c*sc) with
 * sc = (Delta_target * q_{target+1}) / Delta_level, rescale by q_{target+1}. */
orc_ct *orc_op_mult_const(const orc_params *P, const orc_ct *a, double c, int target)
{
    orc_ct *d = drop_limbs(P, a, target + 1);
    double sc = (P->scale[target] * (double)P->prime[target + 1]) / P->scale[a->level];
    double v = c * sc;
    for (int i = 0; i <= target + 1; i++) {
        u64 q = P->prime[i], C = orc_residue_of_double(v, q);
        for (int k = 0; k < d->ncomp; k++) {
            u64 *o = LIMB(P, d, k, i);
            for (int t = 0; t < P->n; t++) o[t] = orc_mul(o[t], C, q);
        }
    }
    orc_ct *r = orc_op_rescale(P, d);
    orc_ct_release(d);
    orc_ledger[LG_CMULT]++;
    return r;
}

/* Plaintext (slot vector) multiply, landing like mult_const (same sc). */
orc_ct *orc_op_mult_pt(const orc_params *P, const orc_ct *a, const double *re, const double *im, int target)
{
    int N = P->n;
    orc_ct *d = drop_limbs(P, a, target + 1);
    double sc = (P->scale[target] * (double)P->prime[target + 1]) / P->scale[a->level];
    u64 *pt = malloc(sizeof(u64) * (size_t)(target + 2) * N);
    orc_encode_coeffs(P, re, im, sc, target + 1, pt);
    #pragma omp parallel for
    for (int i = 0; i <= target + 1; i++) {
        u64 q = P->prime[i];
        u64 *m = pt + (size_t)i * N;
        orc_ntt_fwd(P, i, m);
        for (int k = 0; k < d->ncomp; k++) {
            u64 *o = LIMB(P, d, k, i);
            for (int t = 0; t < N; t++) o[t] = orc_mul(o[t], m[t], q);
        }
    }
    free(pt);
    orc_ct *r = orc_op_rescale(P, d);
    orc_ct_release(d);
    orc_ledger[LG_PMULT]++;
    return r;
}

/* tensor: (a0 b0, a0 b1 + a1 b0, a1 b1) at the common level (C8) */
orc_ct *orc_op_tensor(const orc_params *P, const orc_ct *a0, const orc_ct *b0)
{
    orc_ct *a, *b;
    match_levels(P, a0, b0, &a, &b);
    orc_ct *c = orc_ct_alloc(P, a->level, 3);
    for (int i = 0; i <= a->level; i++) {
        u64 q = P->prime[i];
        const u64 *x0 = LIMB(P, a, 0, i), *x1 = LIMB(P, a, 1, i), *y0 = LIMB(P, b, 0, i), *y1 = LIMB(P, b, 1, i);
        u64 *d0 = LIMB(P, c, 0, i), *d1 = LIMB(P, c, 1, i), *d2 = LIMB(P, c, 2, i);
        for (int t = 0; t < P->n; t++) {
            d0[t] = orc_mul(x0[t], y0[t], q);
            d1[t] = orc_add(orc_mul(x0[t], y1[t], q), orc_mul(x1[t], y0[t], q), q);
            d2[t] = orc_mul(x1[t], y1[t], q);
        }
    }
    orc_ct_release(a);
    orc_ct_release(b);
    orc_ledger[LG_TENSOR]++;
    return c;
}

/* ---------------------------------------------------------------- key switching (C7) */

/* C7 exact centred basis conversion: the integer X = sum_k y_k (S/s_k) lies in
 * [0, ns S); v = round(X / S) = round(sum_k y_k / s_k) makes X - v S the
 * centred representative of X mod S.  v in binary64: each quotient (double)y_k
 * / (double)s_k correctly rounded, summed in k order from 0.0, v = floor(f +
 * 0.5) (C7). */
static u64 bconv_round(const u64 *z, size_t stride, size_t t, const u64 *s, int ns)
{
    double f = 0.0;
    for (int k = 0; k < ns; k++) f += (double)z[(size_t)k * stride + t] / (double)s[k];
    return (u64)floor(f + 0.5);
}

/* ModUp (C7 first half): digit j = primes [j alpha, min((j+1) alpha, nl)) of d
 * (NTT domain, nl limbs) extended to every target prime q_0..q_level,
 * p_0..p_{np-1}.  Returns ext[j][g][N], NTT domain; the digit's own limbs are
 * d's limbs unchanged. */
u64 *orc_ks_modup(const orc_params *P, int level, const u64 *d)
{
    int N = P->n, nq = P->n_q, np = P->n_p, alpha = P->alpha;
    int nl = level + 1, beta = (nl + alpha - 1) / alpha, ntg = nl + np;
    u64 *ext = malloc(sizeof(u64) * (size_t)beta * ntg * N);
    u64 *x = malloc(sizeof(u64) * (size_t)nl * N);
    /* coefficient form of d */
    memcpy(x, d, sizeof(u64) * (size_t)nl * N);
    #pragma omp parallel for
    for (int i = 0; i < nl; i++) orc_ntt_inv(P, i, x + (size_t)i * N);
    for (int j = 0; j < beta; j++) {
        int lo = j * alpha, hi = (j + 1) * alpha < nl ? (j + 1) * alpha : nl; /* digit primes [lo,hi) */
        /* y_i = x_i * qhat_i^{-1} mod q_i */
        int dn = hi - lo;
        u64 *y = malloc(sizeof(u64) * (size_t)dn * N);
        for (int a = 0; a < dn; a++) {
            int i = lo + a;
            u64 q = P->prime[i], qh = 1;
            for (int b = lo; b < hi; b++) if (b != i) qh = orc_mul(qh, P->prime[b] % q, q);
            u64 qhi = orc_inv(qh, q);
            for (int t = 0; t < N; t++) y[(size_t)a * N + t] = orc_mul(x[(size_t)i * N + t], qhi, q);
        }
        #pragma omp parallel for
        for (int g = 0; g < ntg; g++) {
            int pi = g < nl ? g : nq + (g - nl);
            u64 p = P->prime[pi];
            u64 *e = ext + ((size_t)j * ntg + g) * N;
            if (pi >= lo && pi < hi) {
                memcpy(e, d + (size_t)pi * N, sizeof(u64) * N);   /* own limb: unchanged */
            } else {
                u64 *qhp = malloc(sizeof(u64) * dn);
                for (int a = 0; a < dn; a++) {
                    u64 v = 1;
                    for (int b = lo; b < hi; b++) if (b != lo + a) v = orc_mul(v, P->prime[b] % p, p);
                    qhp[a] = v;
                }
                for (int t = 0; t < N; t++) {
                    u64 s = 0;
                    for (int a = 0; a < dn; a++) s = orc_add(s, orc_mul(y[(size_t)a * N + t] % p, qhp[a], p), p);
                    e[t] = s;
                }
                free(qhp);
                orc_ntt_fwd(P, pi, e);
            }
        }
        free(y);
    }
    free(x);
    return ext;
}

/* inner product with the evaluation key: acc[c][g] = sum_j sigma(ext_j)[g] key_j[c][g]
 * where sigma(v)[t] = v[perm[t]] (perm NULL = identity).  acc[2][ntg][N]. */
void orc_ks_inner(const orc_params *P, const orc_swk *key, int level, const u64 *ext, const unsigned *perm,
                     u64 *acc)
{
    int N = P->n, nq = P->n_q, np = P->n_p, nt = nq + np, alpha = P->alpha;
    int nl = level + 1, beta = (nl + alpha - 1) / alpha, ntg = nl + np;
    memset(acc, 0, sizeof(u64) * (size_t)2 * ntg * N);
    #pragma omp parallel for
    for (int g = 0; g < ntg; g++) {
        int pi = g < nl ? g : nq + (g - nl);
        u64 p = P->prime[pi];
        u64 *a0 = acc + (size_t)g * N, *a1 = acc + ((size_t)ntg + g) * N;
        for (int j = 0; j < beta; j++) {
            const u64 *e = ext + ((size_t)j * ntg + g) * N;
            const u64 *k0 = key->k + (((size_t)j * 2 + 0) * nt + pi) * N;
            const u64 *k1 = key->k + (((size_t)j * 2 + 1) * nt + pi) * N;
            for (int t = 0; t < N; t++) {
                u64 v = e[perm ? perm[t] : (unsigned)t];
                a0[t] = orc_add(a0[t], orc_mul(v, k0[t], p), p);
                a1[t] = orc_add(a1[t], orc_mul(v, k1[t], p), p);
            }
        }
    }
}

/* SURVEY 8(f) rank 1 (digit-parallel key switch): the inner product over the
 * digits [j0, j1) only.  The accumulator of C7 is a sum over the digits mod q;
 * the partial sums of any partition of the digits, added mod q, are that sum
 * (modular addition is exact and order-free). */
void orc_ks_inner_digits(const orc_params *P, const orc_swk *key, int level, const u64 *ext, int j0, int j1,
                         u64 *acc)
{
    int N = P->n, nq = P->n_q, np = P->n_p, nt = nq + np;
    int nl = level + 1, ntg = nl + np;
    memset(acc, 0, sizeof(u64) * (size_t)2 * ntg * N);
    #pragma omp parallel for
    for (int g = 0; g < ntg; g++) {
        int pi = g < nl ? g : nq + (g - nl);
        u64 p = P->prime[pi];
        u64 *a0 = acc + (size_t)g * N, *a1 = acc + ((size_t)ntg + g) * N;
        for (int j = j0; j < j1; j++) {
            const u64 *e = ext + ((size_t)j * ntg + g) * N;
            const u64 *k0 = key->k + (((size_t)j * 2 + 0) * nt + pi) * N;
            const u64 *k1 = key->k + (((size_t)j * 2 + 1) * nt + pi) * N;
            for (int t = 0; t < N; t++) {
                a0[t] = orc_add(a0[t], orc_mul(e[t], k0[t], p), p);
                a1[t] = orc_add(a1[t], orc_mul(e[t], k1[t], p), p);
            }
        }
    }
}

/* ModDown (C7 second half): out_c = (acc_Q - BConv_{P->Q}(acc_P)) * P^{-1} */
/* ModDown of ONE component A [ntg][N] (basis Q_level u P) -> out [nl][N] */
void orc_ks_moddown1(const orc_params *P, int level, const u64 *A, u64 *out)
{
    int N = P->n, nq = P->n_q, np = P->n_p;
    int nl = level + 1;
    {
        u64 *z = malloc(sizeof(u64) * (size_t)np * N);
        for (int k = 0; k < np; k++) {
            int pi = nq + k;
            u64 p = P->prime[pi], ph = 1;
            for (int b = 0; b < np; b++) if (b != k) ph = orc_mul(ph, P->prime[nq + b] % p, p);
            u64 phi = orc_inv(ph, p);
            memcpy(z + (size_t)k * N, A + (size_t)(nl + k) * N, sizeof(u64) * N);
            orc_ntt_inv(P, pi, z + (size_t)k * N);
            for (int t = 0; t < N; t++) z[(size_t)k * N + t] = orc_mul(z[(size_t)k * N + t], phi, p);
        }
        #pragma omp parallel for
        for (int i = 0; i < nl; i++) {
            u64 q = P->prime[i];
            u64 *php = malloc(sizeof(u64) * np);
            for (int k = 0; k < np; k++) {
                u64 v = 1;
                for (int b = 0; b < np; b++) if (b != k) v = orc_mul(v, P->prime[nq + b] % q, q);
                php[k] = v;
            }
            u64 *conv = malloc(sizeof(u64) * N);
            /* exact centred conversion (C7): subtract v P, v = round(sum_k y_k / p_k) */
            for (int t = 0; t < N; t++) {
                u64 s = 0;
                for (int k = 0; k < np; k++) {
                    u64 y = z[(size_t)k * N + t];
                    s = orc_add(s, orc_mul(y % q, php[k], q), q);
                }
                u64 v = bconv_round(z, N, t, P->prime + nq, np);
                conv[t] = orc_sub(s, orc_mul(v, P->p_mod_q[i], q), q);
            }
            orc_ntt_fwd(P, i, conv);
            for (int t = 0; t < N; t++)
                out[(size_t)i * N + t] = orc_mul(orc_sub(A[(size_t)i * N + t], conv[t], q), P->p_inv_mod_q[i], q);
            free(conv);
            free(php);
        }
        free(z);
    }
}

static void ks_moddown(const orc_params *P, int level, const u64 *acc, u64 *out0, u64 *out1)
{
    size_t ntg = (size_t)level + 1 + P->n_p;
    orc_ks_moddown1(P, level, acc, out0);
    orc_ks_moddown1(P, level, acc + ntg * P->n, out1);
}

/* C8 fused ModDown + rescale: divide the extended accumulator (basis
 * Q_level u P) by S = P q_level in one centred basis conversion from the
 * source set {p_0..p_{np-1}, q_level} to q_0..q_{level-1}:
 *   z_k = iNTT(acc_{s_k}) * (S/s_k)^{-1} mod s_k,
 *   conv_i = sum_k z_k (S/s_k mod q_i) - #{k: z_k > (s_k-1)/2} (S mod q_i),
 *   out_i = (acc_i - NTT(conv_i)) S^{-1} mod q_i,  i < level.
 * acc: [2][level+1+np][N]; out0/out1: level limbs each. */
void orc_ks_moddown_rescale(const orc_params *P, int level, const u64 *acc, u64 *out0, u64 *out1)
{
    int N = P->n, nq = P->n_q, np = P->n_p;
    int nl = level + 1, ntg = nl + np, ns = np + 1;
    int *src = malloc(sizeof(int) * ns), *slot = malloc(sizeof(int) * ns);
    u64 *sprime = malloc(sizeof(u64) * ns);
    for (int k = 0; k < np; k++) {
        src[k] = nq + k;      /* prime index   */
        slot[k] = nl + k;     /* acc limb      */
    }
    src[np] = level;
    slot[np] = level;
    for (int k = 0; k < ns; k++) sprime[k] = P->prime[src[k]];
    for (int c = 0; c < 2; c++) {
        const u64 *A = acc + (size_t)c * ntg * N;
        u64 *out = c == 0 ? out0 : out1;
        u64 *z = malloc(sizeof(u64) * (size_t)ns * N);
        for (int k = 0; k < ns; k++) {
            u64 s = P->prime[src[k]], sh = 1;
            for (int b = 0; b < ns; b++) if (b != k) sh = orc_mul(sh, P->prime[src[b]] % s, s);
            u64 shi = orc_inv(sh, s);
            memcpy(z + (size_t)k * N, A + (size_t)slot[k] * N, sizeof(u64) * N);
            orc_ntt_inv(P, src[k], z + (size_t)k * N);
            for (int t = 0; t < N; t++) z[(size_t)k * N + t] = orc_mul(z[(size_t)k * N + t], shi, s);
        }
        #pragma omp parallel for
        for (int i = 0; i < level; i++) {
            u64 q = P->prime[i];
            u64 *shq = malloc(sizeof(u64) * ns);
            u64 smq = 1;
            for (int k = 0; k < ns; k++) {
                u64 v = 1;
                for (int b = 0; b < ns; b++) if (b != k) v = orc_mul(v, P->prime[src[b]] % q, q);
                shq[k] = v;
                smq = orc_mul(smq, P->prime[src[k]] % q, q);
            }
            u64 sinv = orc_inv(smq, q);
            u64 *conv = malloc(sizeof(u64) * N);
            for (int t = 0; t < N; t++) {
                u64 s = 0;
                for (int k = 0; k < ns; k++) {
                    u64 y = z[(size_t)k * N + t];
                    s = orc_add(s, orc_mul(y % q, shq[k], q), q);
                }
                u64 v = bconv_round(z, N, t, sprime, ns);
                conv[t] = orc_sub(s, orc_mul(v, smq, q), q);
            }
            orc_ntt_fwd(P, i, conv);
            for (int t = 0; t < N; t++)
                out[(size_t)i * N + t] = orc_mul(orc_sub(A[(size_t)i * N + t], conv[t], q), sinv, q);
            free(conv);
            free(shq);
        }
        free(z);
    }
    free(src);
    free(slot);
    free(sprime);
}

/* d: (level+1) limbs NTT domain.  out0/out1: (level+1) limbs NTT domain. */
void orc_keyswitch(const orc_params *P, const orc_swk *key, int level, const u64 *d, u64 *out0, u64 *out1)
{
    int ntg = level + 1 + P->n_p;
    u64 *ext = orc_ks_modup(P, level, d);
    u64 *acc = malloc(sizeof(u64) * (size_t)2 * ntg * P->n);
    orc_ks_inner(P, key, level, ext, NULL, acc);
    ks_moddown(P, level, acc, out0, out1);
    free(acc);
    free(ext);
    ORC_COUNT_KS(level);
}

/* the two halves of a key switch around its accumulator (digit-parallel
 * path): the partial accumulator of digits [j0, j1), and the ModDown of a
 * (summed) accumulator [2][level+1+n_p][N] */
void orc_ks_partial(const orc_params *P, const orc_swk *key, int level, const u64 *d, int j0, int j1, u64 *acc)
{
    u64 *ext = orc_ks_modup(P, level, d);
    orc_ks_inner_digits(P, key, level, ext, j0, j1, acc);
    free(ext);
}
void orc_ks_finish(const orc_params *P, int level, const u64 *acc, u64 *out0, u64 *out1)
{
    ks_moddown(P, level, acc, out0, out1);
}

/* relinearise a degree-2 ciphertext (no rescale) */
orc_ct *orc_op_relin(const orc_params *P, const orc_keys *K, const orc_ct *d)
{
    const orc_swk *rk = orc_find_key(K, 0);
    int l = d->level;
    size_t sz = (size_t)(l + 1) * P->n;
    u64 *k0 = malloc(sizeof(u64) * sz), *k1 = malloc(sizeof(u64) * sz);
    orc_keyswitch(P, rk, l, LIMB(P, d, 2, 0), k0, k1);
    orc_ct *c = orc_ct_alloc(P, l, 2);
    for (int i = 0; i <= l; i++) {
        u64 q = P->prime[i];
        for (int t = 0; t < P->n; t++) {
            LIMB(P, c, 0, i)[t] = orc_add(LIMB(P, d, 0, i)[t], k0[(size_t)i * P->n + t], q);
            LIMB(P, c, 1, i)[t] = orc_add(LIMB(P, d, 1, i)[t], k1[(size_t)i * P->n + t], q);
        }
    }
    free(k0);
    free(k1);
    return c;
}

/* C8 relinearise + rescale in one division: acc = sum_j ModUp(d2)_j evk_j
 * (basis Q_l u P), plus P (d0, d1) on the Q limbs, divided by P q_l
 * (ks_moddown_rescale).  Output at level l - 1, canonical scale as a rescale. */
orc_ct *orc_op_relin_rescale(const orc_params *P, const orc_keys *K, const orc_ct *d)
{
    const orc_swk *rk = orc_find_key(K, 0);
    int l = d->level, N = P->n, nl = l + 1, ntg = nl + P->n_p;
    u64 *ext = orc_ks_modup(P, l, LIMB(P, d, 2, 0));
    u64 *acc = malloc(sizeof(u64) * (size_t)2 * ntg * N);
    orc_ks_inner(P, rk, l, ext, NULL, acc);
    for (int c = 0; c < 2; c++)
        for (int i = 0; i < nl; i++) {
            u64 q = P->prime[i];
            const u64 *x = LIMB(P, d, c, i);
            u64 *a = acc + ((size_t)c * ntg + i) * N;
            for (int t = 0; t < N; t++) a[t] = orc_add(a[t], orc_mul(x[t], P->p_mod_q[i], q), q);
        }
    orc_ct *r = orc_ct_alloc(P, l - 1, 2);
    orc_ks_moddown_rescale(P, l, acc, LIMB(P, r, 0, 0), LIMB(P, r, 1, 0));
    free(acc);
    free(ext);
    ORC_COUNT_KS(l);
    orc_ledger[LG_RESCALE]++;
    return r;
}

/* C8: HMult = tensor -> relinearise + rescale (one division by P q_l) */
orc_ct *orc_op_mult(const orc_params *P, const orc_keys *K, const orc_ct *a, const orc_ct *b)
{
    orc_ct *d = orc_op_tensor(P, a, b);
    orc_ct *r = orc_op_relin_rescale(P, K, d);
    orc_ct_release(d);
    orc_ledger[LG_HMULT]++;
    return r;
}

/* C10: sigma_k on both components then KS(sigma_k(c1)) from sigma_k(s) to s */
orc_ct *orc_op_galois(const orc_params *P, const orc_keys *K, const orc_ct *a, int k)
{
    int N = P->n, l = a->level;
    const orc_swk *key = orc_find_key(K, k);
    if (!key) return NULL;
    unsigned *perm = malloc(sizeof(unsigned) * N);
    orc_galois_perm(P, k, perm);
    orc_ct *s = orc_ct_alloc(P, l, 2);
    for (int c = 0; c < 2; c++)
        for (int i = 0; i <= l; i++)
            for (int t = 0; t < N; t++) LIMB(P, s, c, i)[t] = LIMB(P, a, c, i)[perm[t]];
    size_t sz = (size_t)(l + 1) * N;
    u64 *k0 = malloc(sizeof(u64) * sz), *k1 = malloc(sizeof(u64) * sz);
    orc_keyswitch(P, key, l, LIMB(P, s, 1, 0), k0, k1);
    orc_ct *r = orc_ct_alloc(P, l, 2);
    for (int i = 0; i <= l; i++) {
        u64 q = P->prime[i];
        for (int t = 0; t < N; t++) {
            LIMB(P, r, 0, i)[t] = orc_add(LIMB(P, s, 0, i)[t], k0[(size_t)i * N + t], q);
            LIMB(P, r, 1, i)[t] = k1[(size_t)i * N + t];
        }
    }
    free(k0);
    free(k1);
    free(perm);
    orc_ct_release(s);
    orc_ledger[LG_ROT]++;
    return r;
}

/* left rotation by r (G1): out_j = in_{j+r} */
orc_ct *orc_op_rotate(const orc_params *P, const orc_keys *K, const orc_ct *a, int r)
{
    return orc_op_galois(P, K, a, orc_galois_of_rot(P, r));
}

/* C16 hoisted rotations (Halevi-Shoup 2018 hoisting): ModUp(c1) ONCE, then
 * for each r: out = (sigma(c0) + ks0, ks1) with (ks0, ks1) =
 * ModDown(sum_j sigma(ext_j) key_j), sigma = the Galois map of rotation r
 * applied to the extended NTT-domain digits.  Decrypts like orc_op_rotate;
 * the words differ (BConv does not commute with sigma's sign flips exactly).
 * Returns 0, or -1 if a key is missing (out[] then partially filled). */
int orc_op_rotate_hoisted(const orc_params *P, const orc_keys *K, const orc_ct *a, const int *rots, int n,
                          orc_ct **out)
{
    int N = P->n, l = a->level, ntg = l + 1 + P->n_p;
    u64 *ext = orc_ks_modup(P, l, LIMB(P, a, 1, 0));
    u64 *acc = malloc(sizeof(u64) * (size_t)2 * ntg * N);
    unsigned *perm = malloc(sizeof(unsigned) * N);
    int rc = 0;
    for (int i = 0; i < n; i++) out[i] = NULL;
    for (int i = 0; i < n && rc == 0; i++) {
        int k = orc_galois_of_rot(P, rots[i]);
        const orc_swk *key = orc_find_key(K, k);
        if (!key) {
            rc = -1;
            break;
        }
        orc_galois_perm(P, k, perm);
        orc_ks_inner(P, key, l, ext, perm, acc);
        orc_ct *r = orc_ct_alloc(P, l, 2);
        ks_moddown(P, l, acc, LIMB(P, r, 0, 0), LIMB(P, r, 1, 0));
        for (int j = 0; j <= l; j++) {
            u64 q = P->prime[j];
            u64 *o = LIMB(P, r, 0, j);
            const u64 *c0 = LIMB(P, a, 0, j);
            for (int t = 0; t < N; t++) o[t] = orc_add(c0[perm[t]], o[t], q);
        }
        out[i] = r;
        ORC_COUNT_KS(l);
        orc_ledger[LG_ROT]++;
    }
    free(perm);
    free(acc);
    free(ext);
    return rc;
}

orc_ct *orc_op_conjugate(const orc_params *P, const orc_keys *K, const orc_ct *a)
{
    return orc_op_galois(P, K, a, 2 * P->n - 1);
}
