/*
 * oracle/api.c -- flat C entry points of liborc.so for the Python test
 * harness (oracle/oracle.py, via ctypes).  TEST INFRASTRUCTURE ONLY.
 */
#include "orc.h"
#include <omp.h>
#include <stdlib.h>
#include <string.h>

orc_params *orc_params_new(int, int, const int *, int, const int *, int, const int *);
void orc_params_free(orc_params *);
orc_keys *orc_keygen(const orc_params *, u64, int, const int *, int, int);
void orc_keys_free(orc_keys *);
orc_ct *orc_encrypt_pk(const orc_params *, const orc_keys *, const u64 *, int, u64, u64);
orc_ct *orc_encrypt_sk(const orc_params *, const orc_keys *, const u64 *, int, u64, u64);
void orc_decrypt(const orc_params *, const orc_keys *, const orc_ct *, u64 *);
double orc_encode_naive_coeff(const orc_params *, const double *, const double *, double, int);


orc_params *orc_api_params(int log_n, int n_q, const int *q_bits, int n_p, const int *p_bits, int alpha,
                           const int *log2_anchor)
{
    return orc_params_new(log_n, n_q, q_bits, n_p, p_bits, alpha, log2_anchor);
}
void orc_api_params_free(orc_params *P) { orc_params_free(P); }
void orc_api_primes(const orc_params *P, u64 *out) { memcpy(out, P->prime, sizeof(u64) * (P->n_q + P->n_p)); }
u64 orc_api_psi(const orc_params *P, int i) { return P->psi[i]; }
double orc_api_scale(const orc_params *P, int l) { return P->scale[l]; }

void orc_api_ntt(const orc_params *P, int pi, u64 *a, int inverse)
{
    if (inverse) orc_ntt_inv(P, pi, a);
    else orc_ntt_fwd(P, pi, a);
}
void orc_api_ntt_naive(const orc_params *P, int pi, u64 *a) { orc_ntt_naive(P, pi, a); }
void orc_api_galois_perm(const orc_params *P, int k, unsigned *perm) { orc_galois_perm(P, k, perm); }
void orc_api_chacha20(const uint32_t *key, uint32_t counter, const uint32_t *nonce, uint32_t *out)
{
    orc_chacha20_block(key, counter, nonce, out);
}
u64 orc_api_stream(u64 seed, uint32_t tag, u64 sub, u64 idx) { return orc_stream(seed, tag, sub, idx); }
u64 orc_api_residue(double x, u64 q) { return orc_residue_of_double(x, q); }
int orc_api_galois_of_rot(const orc_params *P, int r) { return orc_galois_of_rot(P, r); }

orc_keys *orc_api_keygen(const orc_params *P, u64 seed, int h, const int *galois, int n, int relin)
{
    return orc_keygen(P, seed, h, galois, n, relin);
}
void orc_api_keys_free(orc_keys *K) { orc_keys_free(K); }
void orc_api_secret(const orc_params *P, const orc_keys *K, int64_t *out) { memcpy(out, K->s_coeff, sizeof(int64_t) * P->n); }
void orc_api_pk(const orc_params *P, const orc_keys *K, u64 *out)
{
    memcpy(out, K->pk, sizeof(u64) * 2 * (size_t)P->n_q * P->n);
}
/* [dnum][2][n_q+n_p][N] */
int orc_api_swk(const orc_params *P, const orc_keys *K, int galois, u64 *out)
{
    const orc_swk *k = orc_find_key(K, galois);
    if (!k) return -1;
    memcpy(out, k->k, sizeof(u64) * (size_t)P->dnum * 2 * (P->n_q + P->n_p) * P->n);
    return 0;
}

void orc_api_encode(const orc_params *P, const double *re, const double *im, double scale, int level, u64 *out)
{
    orc_encode_coeffs(P, re, im, scale, level, out);
}
double orc_api_encode_naive(const orc_params *P, const double *re, const double *im, double scale, int t)
{
    return orc_encode_naive_coeff(P, re, im, scale, t);
}

/* decrypt and decode with the canonical scale of the ciphertext's level,
 * from the q_0 residue (centred). */
void orc_api_decrypt_decode(const orc_params *P, const orc_keys *K, const orc_ct *c, double *re, double *im)
{
    int N = P->n;
    u64 *m = malloc(sizeof(u64) * (size_t)(c->level + 1) * N);
    orc_decrypt(P, K, c, m);
    i128 *co = malloc(sizeof(i128) * N);
    u64 q0 = P->prime[0];
    for (int t = 0; t < N; t++) co[t] = m[t] > q0 / 2 ? (i128)m[t] - (i128)q0 : (i128)m[t];
    orc_decode_coeffs(P, co, P->scale[c->level], re, im);
    free(co);
    free(m);
}
void orc_api_decrypt(const orc_params *P, const orc_keys *K, const orc_ct *c, u64 *out) { orc_decrypt(P, K, c, out); }

orc_ct *orc_api_encrypt(const orc_params *P, const orc_keys *K, const u64 *pt, int level, u64 seed, u64 idx, int use_sk)
{
    return use_sk ? orc_encrypt_sk(P, K, pt, level, seed, idx) : orc_encrypt_pk(P, K, pt, level, seed, idx);
}

orc_ct *orc_api_ct_import(const orc_params *P, int level, int ncomp, const u64 *w)
{
    orc_ct *c = orc_ct_alloc(P, level, ncomp);
    memcpy(c->a, w, sizeof(u64) * (size_t)ncomp * (level + 1) * P->n);
    return c;
}
void orc_api_ct_export(const orc_params *P, const orc_ct *c, u64 *w)
{
    memcpy(w, c->a, sizeof(u64) * (size_t)c->ncomp * (c->level + 1) * P->n);
}
int orc_api_ct_level(const orc_ct *c) { return c->level; }
int orc_api_ct_ncomp(const orc_ct *c) { return c->ncomp; }
void orc_api_ct_free(orc_ct *c) { orc_ct_release(c); }

enum { OP_ADD, OP_SUB, OP_MULT, OP_TENSOR, OP_RELIN, OP_RESCALE, OP_LEVEL_DOWN, OP_MULT_CONST,
       OP_ADD_CONST, OP_MULT_INT, OP_ROTATE, OP_CONJ, OP_GALOIS };

orc_ct *orc_api_op(const orc_params *P, const orc_keys *K, int op, const orc_ct *a, const orc_ct *b, double c, int i)
{
    switch (op) {
    case OP_ADD: return orc_op_add(P, a, b);
    case OP_SUB: return orc_op_sub(P, a, b);
    case OP_MULT: return orc_op_mult(P, K, a, b);
    case OP_TENSOR: return orc_op_tensor(P, a, b);
    case OP_RELIN: return orc_op_relin(P, K, a);
    case OP_RESCALE: return orc_op_rescale(P, a);
    case OP_LEVEL_DOWN: return orc_op_level_down(P, a, i);
    case OP_MULT_CONST: return orc_op_mult_const(P, a, c, i);
    case OP_ADD_CONST: return orc_op_add_const(P, a, c);
    case OP_MULT_INT: return orc_op_mult_int(P, a, (int64_t)i);
    case OP_ROTATE: return orc_op_rotate(P, K, a, i);
    case OP_CONJ: return orc_op_conjugate(P, K, a);
    case OP_GALOIS: return orc_op_galois(P, K, a, i);
    }
    return NULL;
}

orc_ct *orc_api_mult_pt(const orc_params *P, const orc_ct *a, const double *re, const double *im, int target)
{
    return orc_op_mult_pt(P, a, re, im, target);
}

int orc_api_keyswitch(const orc_params *P, const orc_keys *K, int galois, int level, const u64 *d, u64 *o0, u64 *o1)
{
    const orc_swk *k = orc_find_key(K, galois);
    if (!k) return -1;
    orc_keyswitch(P, k, level, d, o0, o1);
    return 0;
}

/* digit-parallel key switch pieces */
int orc_api_ks_partial(const orc_params *P, const orc_keys *K, int galois, int level, const u64 *d, int j0, int j1,
                       u64 *acc)
{
    const orc_swk *k = orc_find_key(K, galois);
    if (!k) return -1;
    orc_ks_partial(P, k, level, d, j0, j1, acc);
    return 0;
}
void orc_api_ks_finish(const orc_params *P, int level, const u64 *acc, u64 *o0, u64 *o1)
{
    orc_ks_finish(P, level, acc, o0, o1);
}

/* C16: hoisted rotations of one ciphertext; out[n] (NULL on a missing key) */
int orc_api_rotate_hoisted(const orc_params *P, const orc_keys *K, const orc_ct *a, const int *rots, int n,
                           orc_ct **out)
{
    return orc_op_rotate_hoisted(P, K, a, rots, n, out);
}

/* x holds alpha x (G28); gain multiplies the series (C13) */
orc_ct *orc_api_cheb(const orc_params *P, const orc_keys *K, const orc_ct *x, int deg, double a, double b, const double *c,
                     double gain)
{
    orc_cheb p = {deg, a, b, c};
    return orc_eval_cheb(P, K, x, &p, gain);
}
/* G28 input contract: the Softmax reads x encoded at Delta_level * alpha_exp */
double orc_api_softmax_input_scale(const orc_params *P, double a, double b, int level)
{
    return P->scale[level] * (2.0 / (b - a));
}
int orc_api_cheb_depth(int deg) { return orc_cheb_depth(deg); }

/* polys: n_poly = 1 + k entries (exp first), degs/as/bs arrays, coeffs concatenated */
int orc_api_softmax(const orc_params *P, const orc_keys *K, int n, int m, int k, int variant,
                    const int *degs, const double *as, const double *bs, const double *coeffs,
                    orc_ct *const *in, orc_ct **out, int newton)
{
    orc_cheb *polys = malloc(sizeof(orc_cheb) * (k + 1));
    const double *cp = coeffs;
    for (int i = 0; i <= k; i++) {
        polys[i].deg = degs[i];
        polys[i].a = as[i];
        polys[i].b = bs[i];
        polys[i].c = cp;
        cp += degs[i] + 1;
    }
    orc_softmax_desc d = {n, m, k, variant, &polys[0], &polys[1], NULL, NULL, newton};
    int rc = orc_softmax(P, K, &d, in, out);
    free(polys);
    return rc;
}

/* OpenMP threads of the oracle (bench's single-thread baseline) */
void orc_api_set_threads(int n) { omp_set_num_threads(n < 1 ? 1 : n); }
int orc_api_max_threads(void) { return omp_get_max_threads(); }

void orc_api_ledger(long *out) { memcpy(out, orc_ledger, sizeof(orc_ledger)); }
void orc_api_ledger_reset(void)
{
    memset(orc_ledger, 0, sizeof(orc_ledger));
    memset(orc_ks_level, 0, sizeof(orc_ks_level));
}
void orc_api_ks_levels(long *out) { memcpy(out, orc_ks_level, sizeof(orc_ks_level)); }

/* ---------------------------------------------------------------- bootstrapping */
typedef struct orc_bts_set orc_bts_set;
orc_bts_set *orc_bts_set_new(const orc_params *P, int K, int r, int n_cts, int n_stc, int arcsine, int deg,
                             const double *coeffs, int out_level);
void orc_bts_set_free(orc_bts_set *S);
int orc_bts_rotations(const orc_params *P, int n_cts, int n_stc, int *out, int max);
int orc_bts_exponent(const orc_params *P, int arcsine, double bound);
orc_ct *orc_bootstrap(const orc_params *P, const orc_keys *K, const orc_ct *in, void *ctx, double bound);

orc_ct *orc_api_newton(const orc_params *P, const orc_keys *K, const orc_ct *xh, const orc_ct *y)
{
    return orc_newton_invsqrt_step(P, K, xh, y);
}

void *orc_api_bts_new(const orc_params *P, int K, int r, int n_cts, int n_stc, int arcsine, int deg,
                      const double *coeffs, int out_level)
{
    return orc_bts_set_new(P, K, r, n_cts, n_stc, arcsine, deg, coeffs, out_level);
}
void orc_api_bts_free(void *p) { orc_bts_set_free(p); }
int orc_api_bts_rotations(const orc_params *P, int n_cts, int n_stc, int *out, int max)
{
    return orc_bts_rotations(P, n_cts, n_stc, out, max);
}
int orc_api_bts_exponent(const orc_params *P, int arcsine, double bound) { return orc_bts_exponent(P, arcsine, bound); }
orc_ct *orc_api_bootstrap(const orc_params *P, const orc_keys *K, const orc_ct *in, void *bts, double bound)
{
    return orc_bootstrap(P, K, in, bts, bound);
}
int orc_api_softmax_bts(const orc_params *P, const orc_keys *K, int n, int m, int k, int variant,
                        const int *degs, const double *as, const double *bs, const double *coeffs,
                        orc_ct *const *in, orc_ct **out, void *bts, int newton)
{
    orc_cheb *polys = malloc(sizeof(orc_cheb) * (k + 1));
    const double *cp = coeffs;
    for (int i = 0; i <= k; i++) {
        polys[i].deg = degs[i];
        polys[i].a = as[i];
        polys[i].b = bs[i];
        polys[i].c = cp;
        cp += degs[i] + 1;
    }
    orc_softmax_desc d = {n, m, k, variant, &polys[0], &polys[1], bts ? orc_bootstrap : NULL, bts, newton};
    int rc = orc_softmax(P, K, &d, in, out);
    free(polys);
    return rc;
}

extern int orc_bts_debug_stop;
void orc_api_bts_debug_stop(int s) { orc_bts_debug_stop = s; }
extern int orc_bts_debug_skip_raise;
void orc_api_bts_debug_skip_raise(int s) { orc_bts_debug_skip_raise = s; }

extern int orc_trace_on, orc_trace_n;
extern int orc_trace[512][4];
void orc_api_trace(int on) { orc_trace_on = on; orc_trace_n = 0; }
int orc_api_trace_get(int *out, int max)
{
    int n = orc_trace_n < max ? orc_trace_n : max;
    memcpy(out, orc_trace, sizeof(int) * 4 * n);
    return n;
}

/* bench.py --impl reference: the Softmax schedule with a bootstrap STUB that
 * returns an all-zero ciphertext at out_level (and counts LG_BTS) -- the op
 * inventory of a step (key switches per level, bootstrap count) without the
 * bootstraps' own work, which is timed separately.  Data-independent
 * schedule (G12 reads levels only); never used for parity. */
static int g_stub_out_level;
static orc_ct *bts_stub(const orc_params *P, const orc_keys *K, const orc_ct *c, void *ctx, double bound)
{
    (void)K; (void)c; (void)ctx; (void)bound;
    orc_ledger[LG_BTS]++;
    return orc_ct_alloc(P, g_stub_out_level, 2);
}
int orc_api_softmax_inventory(const orc_params *P, const orc_keys *K, int n, int m, int k, int variant,
                              const int *degs, const double *as, const double *bs, const double *coeffs,
                              orc_ct *const *in, orc_ct **out, int out_level, int newton)
{
    orc_cheb *polys = malloc(sizeof(orc_cheb) * (k + 1));
    const double *cp = coeffs;
    for (int i = 0; i <= k; i++) {
        polys[i].deg = degs[i];
        polys[i].a = as[i];
        polys[i].b = bs[i];
        polys[i].c = cp;
        cp += degs[i] + 1;
    }
    g_stub_out_level = out_level;
    orc_softmax_desc d = {n, m, k, variant, &polys[0], &polys[1], bts_stub, NULL, newton};
    int rc = orc_softmax(P, K, &d, in, out);
    free(polys);
    return rc;
}
