/*
 * oracle/bts.c -- real-slot CKKS bootstrapping of the oracle.
 * TEST INFRASTRUCTURE ONLY (see orc.h).
 *
 * PAPER.md 281-283 and 429-440 require bootstrapping (BTS) but give none of
 * its internals (HEaaN FGb, PAPER.md 386-393).  DESIGN.md reading G11 fixes a
 * textbook CoeffToSlot-first bootstrap specialised to real slot values (all
 * Softmax data are real):
 *   0. pre-scale: x *= 2^e, e = clamp(floor(log2 q0 - cap - log2 Delta_0 - log2 B), 0, 30)
 *      (cap = 8 with the arcsine step, 12 without; B = caller's bound on |z|);
 *   1. drop to level 0; ModRaise to level L (centred lift of the q_0 residues);
 *   2. CoeffToSlot: n_cts sparse linear transforms (groups of inverse special-
 *      FFT stages), slot p then holds kappa (c_j + i c_{j+N0}) / q_0, j = brv(p);
 *   3. v = w + conj(w) - 1/(4(K+2))  (real part, mapped onto [-1, 1]);
 *   4. EvalMod: Chebyshev series of cos(2 pi (K+2) v / 2^r), r double angles
 *      -> s = sin(2 pi c_j / q_0);  optional arcsine step s <- s + s^3/6;
 *   5. SlotToCoeff: n_stc transforms (groups of special-FFT stages) with the
 *      factor q_0 / (4 pi Delta_out 2^e) and D = diag(1, 2, ..., 2) (real-message
 *      identity z = Re(V D m_lo)), then out = x + conj(x).
 * Each linear transform is a baby-step/giant-step diagonal evaluation landing
 * at the canonical scale of the next level (one rescale).
 */
#include "orc.h"
#include <math.h>
#include <quadmath.h>
#include <stdlib.h>
#include <string.h>

void orc_encode_coeffs_q(const orc_params *P, const __float128 *re, const __float128 *im, double scale, int level,
                         u64 *out);
void orc_encode_coeffs_q_pq(const orc_params *P, const __float128 *re, const __float128 *im, double scale, int level,
                            u64 *out);

typedef __float128 f128;
typedef struct { f128 re, im; } qz;

static qz qmul(qz a, qz b) { qz r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; return r; }
static qz qdiv(qz a, qz b)
{
    f128 d = b.re * b.re + b.im * b.im;
    qz r = {(a.re * b.re + a.im * b.im) / d, (a.im * b.re - a.re * b.im) / d};
    return r;
}

/* a sparse matrix in diagonal form: diag[d][p] = A[p][(p + d) mod N0] */
typedef struct {
    int n0;
    char *present;   /* [n0] */
    qz **diag;       /* [n0] -> vector or NULL */
} dmat;

static dmat *dm_new(int n0)
{
    dmat *m = calloc(1, sizeof(*m));
    m->n0 = n0;
    m->present = calloc(n0, 1);
    m->diag = calloc(n0, sizeof(qz *));
    return m;
}
static void dm_free(dmat *m)
{
    if (!m) return;
    for (int d = 0; d < m->n0; d++) free(m->diag[d]);
    free(m->diag);
    free(m->present);
    free(m);
}
static void dm_add(dmat *m, int d, int p, qz v)
{
    d = ((d % m->n0) + m->n0) % m->n0;
    if (!m->present[d]) {
        m->present[d] = 1;
        m->diag[d] = calloc(m->n0, sizeof(qz));
    }
    m->diag[d][p].re += v.re;
    m->diag[d][p].im += v.im;
}

/* special-FFT stage of length len (or its inverse): for block i, j < len/2,
 * p = i + j:  out[p] = in[p] + xi in[p+h],  out[p+h] = in[p] - xi in[p+h],
 * xi = exp(2 pi i ((5^j mod 4 len) (2N / 4 len)) / 2N). */
static dmat *stage(int log_n, int len, int inverse)
{
    int N = 1 << log_n, n0 = N / 2, h = len / 2, q4 = 4 * len;
    dmat *m = dm_new(n0);
    u64 g = 1;
    for (int j = 0; j < h; j++) {
        u64 e = (g % (u64)q4) * (u64)(2 * N / q4);
        f128 ang = 2 * M_PIq * (f128)e / (f128)(2 * N);
        qz xi = {cosq(ang), sinq(ang)}, one = {1, 0}, half = {0.5, 0};
        for (int i = 0; i < n0; i += len) {
            int p = i + j;
            if (!inverse) {
                qz mxi = {-xi.re, -xi.im};
                dm_add(m, 0, p, one);
                dm_add(m, h, p, xi);
                dm_add(m, -h, p + h, one);
                dm_add(m, 0, p + h, mxi);
            } else {
                qz ix = qdiv(half, xi), mix = {-ix.re, -ix.im};
                dm_add(m, 0, p, half);
                dm_add(m, h, p, half);
                dm_add(m, -h, p + h, ix);
                dm_add(m, 0, p + h, mix);
            }
        }
        g = (g * 5) % (2ull * N);
    }
    return m;
}

/* C = A B :  diag_d(C)[p] = sum_{e+f=d} diag_e(A)[p] diag_f(B)[(p+e) mod N0] */
static dmat *compose(const dmat *A, const dmat *B)
{
    int n0 = A->n0;
    dmat *C = dm_new(n0);
    for (int e = 0; e < n0; e++) {
        if (!A->present[e]) continue;
        for (int f = 0; f < n0; f++) {
            if (!B->present[f]) continue;
            int d = (e + f) % n0;
            for (int p = 0; p < n0; p++) dm_add(C, d, p, qmul(A->diag[e][p], B->diag[f][(p + e) % n0]));
        }
    }
    return C;
}

static void dm_scale_cols(dmat *m, const f128 *s)  /* m <- m diag(s) */
{
    for (int d = 0; d < m->n0; d++) {
        if (!m->present[d]) continue;
        for (int p = 0; p < m->n0; p++) {
            f128 f = s[(p + d) % m->n0];
            m->diag[d][p].re *= f;
            m->diag[d][p].im *= f;
        }
    }
}

/* ------------------------------------------------------------ plan */
#define ORC_MAXG 8

typedef struct {
    int level;           /* input level of this transform          */
    int u, b1;           /* step unit, baby size                   */
    int n_terms;
    int *g, *b;          /* per term: giant index, baby index      */
    u64 **pt;            /* per term: NTT residues, level+1 limbs  */
} ltrans;

typedef struct {
    int K, r, n_cts, n_stc, arcsine, out_level;
} orc_bts_cfg;

typedef struct {
    const orc_params *P;
    orc_bts_cfg cfg;
    int e;
    const orc_cheb *cosp;
    ltrans cts[ORC_MAXG], stc[ORC_MAXG];
} orc_bts_plan;

/* all plans of one parameter set, one per pre-scaling exponent e */
#define ORC_BTS_EMAX 30
typedef struct {
    const orc_params *P;
    orc_bts_cfg cfg;
    orc_cheb cosp;
    double *coeffs;
    orc_bts_plan *plan[ORC_BTS_EMAX + 1];
} orc_bts_set;

static int ilog2i(int x) { int t = 0; while ((1 << t) < x) t++; return t; }

/* split s stages into g groups, the earlier groups not smaller */
static void group_sizes(int s, int g, int *sz)
{
    int rem = s;
    for (int k = g, i = 0; k >= 1; k--, i++) { sz[i] = (rem + k - 1) / k; rem -= sz[i]; }
}

/* encode a transform at input level `level` */
static void make_ltrans(const orc_params *P, const dmat *m, int level, int u, int r, ltrans *T)
{
    int n0 = P->n / 2, N = P->n;
    T->level = level;
    T->u = u;
    T->b1 = 1 << (r < 4 ? r : 4);  /* baby size 2^min(r, 4) (G11) */
    int cnt = 0;
    for (int d = 0; d < n0; d++) cnt += m->present[d];
    T->n_terms = cnt;
    T->g = malloc(sizeof(int) * cnt);
    T->b = malloc(sizeof(int) * cnt);
    T->pt = calloc(cnt, sizeof(u64 *));
    int *dl = malloc(sizeof(int) * cnt);
    for (int d = 0, k = 0; d < n0; d++)
        if (m->present[d]) {
            int idx = d / u;
            T->g[k] = idx / T->b1;
            T->b[k] = idx % T->b1;
            dl[k++] = d;
        }
    double sc = (P->scale[level - 1] * (double)P->prime[level]) / P->scale[level];
    {   /* warm the encoder's twiddle cache before the parallel loop */
        double *z = calloc(n0, sizeof(double));
        u64 *tmp = malloc(sizeof(u64) * N);
        orc_encode_coeffs(P, z, z, 1.0, 0, tmp);
        free(z);
        free(tmp);
    }
    #pragma omp parallel for schedule(dynamic)
    for (int k = 0; k < cnt; k++) {
        int G = (T->g[k] * T->b1 * u) % n0;
        f128 *re = malloc(sizeof(f128) * n0), *im = malloc(sizeof(f128) * n0);
        const qz *v = m->diag[dl[k]];
        for (int p = 0; p < n0; p++) {           /* rot(diag, -G)_p = diag_{p - G} */
            qz x = v[((p - G) % n0 + n0) % n0];
            re[p] = x.re;
            im[p] = x.im;
        }
        /* C17: plaintexts in the extended basis Q_level u P */
        int ntg = level + 1 + P->n_p;
        u64 *pt = malloc(sizeof(u64) * (size_t)ntg * N);
        orc_encode_coeffs_q_pq(P, re, im, sc, level, pt);
        for (int gi = 0; gi < ntg; gi++)
            orc_ntt_fwd(P, gi <= level ? gi : P->n_q + (gi - level - 1), pt + (size_t)gi * N);
        T->pt[k] = pt;
        free(re);
        free(im);
    }
    free(dl);
}

static void free_ltrans(ltrans *T)
{
    for (int k = 0; k < T->n_terms; k++) free(T->pt[k]);
    free(T->pt);
    free(T->g);
    free(T->b);
}

static void add_group_rotations(int n0, int ngroups, int *out, int *cnt, int max)
{
    int s = ilog2i(n0), sz[ORC_MAXG], first = 0;
    group_sizes(s, ngroups, sz);
    for (int gi = 0; gi < ngroups; gi++) {
        int u = 1 << first, r = sz[gi], b1 = 1 << (r < 4 ? r : 4);
        int span = (1 << r) - 1;  /* idx in [-span, span] mod n0/u */
        int mod = n0 / u;
        for (int idx = -span; idx <= span; idx++) {
            int id = ((idx % mod) + mod) % mod;
            int rots[2] = {(id % b1) * u, (id / b1) * b1 * u};
            for (int t = 0; t < 2; t++) {
                int rr = rots[t] % n0;
                if (!rr) continue;
                int dup = 0;
                for (int i = 0; i < *cnt; i++) if (out[i] == rr) dup = 1;
                if (!dup && *cnt < max) out[(*cnt)++] = rr;
            }
        }
        first += r;
    }
}

/* the rotations (left, slots) a plan needs: babies b u, giants g b1 u of the
 * SlotToCoeff groups, then of the CoeffToSlot groups (same stage grouping
 * rule; duplicates removed in first-seen order) */
int orc_bts_rotations(const orc_params *P, int n_cts, int n_stc, int *out, int max)
{
    int cnt = 0;
    add_group_rotations(P->n / 2, n_stc, out, &cnt, max);
    add_group_rotations(P->n / 2, n_cts, out, &cnt, max);
    return cnt;
}

static dmat *group_matrix(const orc_params *P, int first, int size, int inverse)
{
    dmat *acc = NULL;
    for (int t = 0; t < size; t++) {
        int i = inverse ? first + size - 1 - t : first + t;  /* inverse: largest stage first */
        dmat *S = stage(P->log_n, 2 << i, inverse);
        if (!acc) acc = S;
        else { dmat *x = compose(S, acc); dm_free(S); dm_free(acc); acc = x; }
    }
    return acc;
}

/* e: the input is multiplied by 2^e before ModRaise (message pre-scaling,
 * DESIGN.md G11); SlotToCoeff divides it back. */
static orc_bts_plan *plan_new(const orc_params *P, const orc_bts_cfg *cfg, const orc_cheb *cosp, int e)
{
    orc_bts_plan *B = calloc(1, sizeof(*B));
    B->P = P;
    B->cfg = *cfg;
    B->e = e;
    B->cosp = cosp;
    int n0 = P->n / 2, s = ilog2i(n0), L = P->L;
    int sz[ORC_MAXG], first[ORC_MAXG];
    /* SlotToCoeff: groups in stage order; first transform composed with diag(lambda D) */
    group_sizes(s, cfg->n_stc, sz);
    for (int gi = 0, st = 0; gi < cfg->n_stc; st += sz[gi], gi++) {
        dmat *m = group_matrix(P, st, sz[gi], 0);
        if (gi == 0) {
            f128 lam = (f128)P->prime[0] / (4 * M_PIq * (f128)P->scale[cfg->out_level] * ldexpq(1, e));
            f128 *dv = malloc(sizeof(f128) * n0);
            for (int p = 0; p < n0; p++) dv[p] = p == 0 ? lam : 2 * lam;
            dm_scale_cols(m, dv);
            free(dv);
        }
        make_ltrans(P, m, cfg->out_level + cfg->n_stc - gi, 1 << st, sz[gi], &B->stc[gi]);
        dm_free(m);
    }
    /* CoeffToSlot: inverse groups, largest stages first; factor kappa Delta_L / q0 first */
    group_sizes(s, cfg->n_cts, sz);
    for (int gi = 0, st = 0; gi < cfg->n_cts; st += sz[gi], gi++) first[gi] = st;
    for (int k = 0; k < cfg->n_cts; k++) {
        int gi = cfg->n_cts - 1 - k;
        dmat *m = group_matrix(P, first[gi], sz[gi], 1);
        if (k == 0) {
            f128 f = ((f128)P->scale[L] / (f128)P->prime[0]) / (2 * (f128)(cfg->K + 2));
            f128 *fv = malloc(sizeof(f128) * n0);
            for (int p = 0; p < n0; p++) fv[p] = f;
            dm_scale_cols(m, fv);
            free(fv);
        }
        make_ltrans(P, m, L - k, 1 << first[gi], sz[gi], &B->cts[k]);
        dm_free(m);
    }
    return B;
}

static void plan_free(orc_bts_plan *B)
{
    if (!B) return;
    for (int k = 0; k < B->cfg.n_cts; k++) free_ltrans(&B->cts[k]);
    for (int k = 0; k < B->cfg.n_stc; k++) free_ltrans(&B->stc[k]);
    free(B);
}

/* prime index of limb g of the extended basis Q_level u P */
static int ext_prime(const orc_params *P, int nl, int g) { return g < nl ? g : P->n_q + (g - nl); }

/* C17 double-hoisted BSGS (C17), ct (2 comps) -> transform at
 * level T->level, landing at level-1.  Every intermediate lives in the
 * extended basis Q_l u P ("PQ", ntg = l+1+np limbs, a value v stands for P v):
 *   R_0 = P x; R_b = (P sigma_b(c0) + <sigma_b(ModUp(c1)), evk_b>_0,
 *                     <sigma_b(ModUp(c1)), evk_b>_1)  (one ModUp, no ModDown)
 *   inner_g = sum_b pt_{g,b} (.) R_b  (plaintexts encoded in PQ)
 *   giant g != 0:  b' = ModDown(inner_g,1);  Rot = (sigma_g(inner_g,0) +
 *                  <ModUp(sigma_g(b')), evk_g>_0, <...>_1)   (no ModDown)
 *   out = ModDown+rescale by P q_l (C8) of inner_0 + sum_g Rot_g. */
static orc_ct *apply_ltrans(const orc_params *P, const orc_keys *K, const orc_ct *ct0, const ltrans *T)
{
    int N = P->n, n0 = N / 2, l = T->level, nl = l + 1, np = P->n_p, ntg = nl + np;
    size_t W = (size_t)2 * ntg * N;   /* one PQ ciphertext */
    orc_ct *x = orc_op_level_down(P, ct0, l);
    unsigned *perm = malloc(sizeof(unsigned) * N);
    u64 *R[64] = {0};
    int present[64] = {0};
    for (int k = 0; k < T->n_terms; k++) present[T->b[k]] = 1;
    if (present[0]) {             /* R_0 = P x: Q limbs x (P mod q_i), P limbs 0 */
        R[0] = calloc(W, sizeof(u64));
        for (int c = 0; c < 2; c++)
            for (int i = 0; i < nl; i++) {
                u64 q = P->prime[i];
                const u64 *s = LIMB(P, x, c, i);
                u64 *o = R[0] + ((size_t)c * ntg + i) * N;
                for (int t = 0; t < N; t++) o[t] = orc_mul(s[t], P->p_mod_q[i], q);
            }
    }
    int any = 0;
    for (int b = 1; b < 64; b++) any |= present[b];
    u64 *ext = any ? orc_ks_modup(P, l, LIMB(P, x, 1, 0)) : NULL;
    for (int b = 1; b < 64; b++) {    /* babies in increasing b */
        if (!present[b]) continue;
        int k = orc_galois_of_rot(P, b * T->u);
        const orc_swk *key = orc_find_key(K, k);
        if (!key) return NULL;
        orc_galois_perm(P, k, perm);
        R[b] = malloc(sizeof(u64) * W);
        orc_ks_inner(P, key, l, ext, perm, R[b]);
        for (int i = 0; i < nl; i++) {      /* + P sigma_b(c0) on the Q limbs */
            u64 q = P->prime[i];
            const u64 *c0 = LIMB(P, x, 0, i);
            u64 *o = R[b] + (size_t)i * N;
            for (int t = 0; t < N; t++) o[t] = orc_add(o[t], orc_mul(c0[perm[t]], P->p_mod_q[i], q), q);
        }
        ORC_COUNT_KS(l);
        orc_ledger[LG_ROT]++;
    }
    free(ext);
    int maxg = 0;
    for (int k = 0; k < T->n_terms; k++) if (T->g[k] > maxg) maxg = T->g[k];
    u64 *acc = calloc(W, sizeof(u64)), *inner = malloc(sizeof(u64) * W);
    u64 *bq = malloc(sizeof(u64) * (size_t)nl * N), *sb = malloc(sizeof(u64) * (size_t)nl * N);
    u64 *rot = malloc(sizeof(u64) * W);
    for (int g = 0; g <= maxg; g++) {
        int have = 0;
        memset(inner, 0, sizeof(u64) * W);
        for (int k = 0; k < T->n_terms; k++) {
            if (T->g[k] != g) continue;
            have = 1;
            const u64 *Rb = R[T->b[k]];
            for (int gi = 0; gi < ntg; gi++) {
                u64 q = P->prime[ext_prime(P, nl, gi)];
                const u64 *m = T->pt[k] + (size_t)gi * N;
                for (int c = 0; c < 2; c++) {
                    u64 *o = inner + ((size_t)c * ntg + gi) * N;
                    const u64 *sv = Rb + ((size_t)c * ntg + gi) * N;
                    for (int t = 0; t < N; t++) o[t] = orc_add(o[t], orc_mul(sv[t], m[t], q), q);
                }
            }
            orc_ledger[LG_PMULT]++;
        }
        if (!have) continue;
        const u64 *add = inner;
        if (g != 0) {
            int k = orc_galois_of_rot(P, (g * T->b1 * T->u) % n0);
            const orc_swk *key = orc_find_key(K, k);
            if (!key) return NULL;
            orc_galois_perm(P, k, perm);
            orc_ks_moddown1(P, l, inner + (size_t)ntg * N, bq);     /* b' = ModDown(inner_1) */
            for (int i = 0; i < nl; i++)                            /* sigma_g(b') */
                for (int t = 0; t < N; t++) sb[(size_t)i * N + t] = bq[(size_t)i * N + perm[t]];
            u64 *e2 = orc_ks_modup(P, l, sb);
            orc_ks_inner(P, key, l, e2, NULL, rot);
            free(e2);
            for (int gi = 0; gi < ntg; gi++) {                      /* + sigma_g(inner_0), all PQ limbs */
                u64 q = P->prime[ext_prime(P, nl, gi)];
                const u64 *a0 = inner + (size_t)gi * N;
                u64 *o = rot + (size_t)gi * N;
                for (int t = 0; t < N; t++) o[t] = orc_add(o[t], a0[perm[t]], q);
            }
            ORC_COUNT_KS(l);
            orc_ledger[LG_ROT]++;
            add = rot;
        }
        for (int c = 0; c < 2; c++)
            for (int gi = 0; gi < ntg; gi++) {
                u64 q = P->prime[ext_prime(P, nl, gi)];
                u64 *o = acc + ((size_t)c * ntg + gi) * N;
                const u64 *sv = add + ((size_t)c * ntg + gi) * N;
                for (int t = 0; t < N; t++) o[t] = orc_add(o[t], sv[t], q);
            }
    }
    orc_ct *out = orc_ct_alloc(P, l - 1, 2);
    orc_ks_moddown_rescale(P, l, acc, LIMB(P, out, 0, 0), LIMB(P, out, 1, 0));
    orc_ledger[LG_RESCALE]++;
    for (int b = 0; b < 64; b++) free(R[b]);
    free(acc);
    free(inner);
    free(bq);
    free(sb);
    free(rot);
    free(perm);
    orc_ct_release(x);
    return out;
}

/* ModRaise: the q_0 residues of both components, centred, lifted to Q_L */
static orc_ct *mod_raise(const orc_params *P, const orc_ct *ct)
{
    int N = P->n, L = P->L;
    orc_ct *r = orc_ct_alloc(P, L, 2);
    u64 q0 = P->prime[0];
    u64 *x = malloc(sizeof(u64) * N);
    for (int c = 0; c < 2; c++) {
        memcpy(x, LIMB(P, ct, c, 0), sizeof(u64) * N);
        orc_ntt_inv(P, 0, x);
        #pragma omp parallel for
        for (int i = 0; i <= L; i++) {
            u64 q = P->prime[i];
            u64 *o = LIMB(P, r, c, i);
            for (int t = 0; t < N; t++) {
                u64 v = x[t];
                if (v <= (q0 - 1) / 2) o[t] = v % q;
                else o[t] = orc_sub(0, (q0 - v) % q, q);
            }
            orc_ntt_fwd(P, i, o);
        }
    }
    free(x);
    return r;
}

/* G11 pre-scaling exponent for a message bound B. */
int orc_bts_exponent(const orc_params *P, int arcsine, double bound)
{
    double cap = arcsine ? 8.0 : 12.0;
    double e = floor(log2((double)P->prime[0]) - cap - log2(P->scale[0]) - log2(bound));
    if (e < 0) e = 0;
    if (e > ORC_BTS_EMAX) e = ORC_BTS_EMAX;
    return (int)e;
}

/* the chain the plan needs: L = out + n_stc + 2 arcsine + r + depth(cos) + n_cts */
orc_bts_set *orc_bts_set_new(const orc_params *P, int K, int r, int n_cts, int n_stc, int arcsine, int deg,
                             const double *coeffs, int out_level)
{
    if (n_cts < 1 || n_cts > ORC_MAXG || n_stc < 1 || n_stc > ORC_MAXG) return NULL;
    if (out_level + n_stc + (arcsine ? 2 : 1) + r + orc_cheb_depth(deg) + n_cts != P->L) return NULL;
    orc_bts_set *S = calloc(1, sizeof(*S));
    S->P = P;
    S->cfg.K = K;
    S->cfg.r = r;
    S->cfg.n_cts = n_cts;
    S->cfg.n_stc = n_stc;
    S->cfg.arcsine = arcsine != 0;
    S->cfg.out_level = out_level;
    S->coeffs = malloc(sizeof(double) * (deg + 1));
    memcpy(S->coeffs, coeffs, sizeof(double) * (deg + 1));
    S->cosp.deg = deg;
    S->cosp.a = -1.0;
    S->cosp.b = 1.0;
    S->cosp.c = S->coeffs;
    return S;
}

void orc_bts_set_free(orc_bts_set *S)
{
    if (!S) return;
    for (int e = 0; e <= ORC_BTS_EMAX; e++) plan_free(S->plan[e]);
    free(S->coeffs);
    free(S);
}

int orc_bts_debug_stop = -1;       /* test hook: return the intermediate after this stage */
int orc_bts_debug_skip_raise = 0;  /* test hook: input is already at level L */
#define STOP(st, ct) if (orc_bts_debug_stop == (st)) return ct;

orc_ct *orc_bootstrap(const orc_params *P, const orc_keys *K, const orc_ct *in, void *ctx, double bound)
{
    orc_bts_set *BS = ctx;
    const orc_bts_cfg *cf = &BS->cfg;
    int e = orc_bts_exponent(P, cf->arcsine, bound);
    if (!BS->plan[e]) BS->plan[e] = plan_new(P, cf, &BS->cosp, e);
    const orc_bts_plan *B = BS->plan[e];
    int conj = 2 * P->n - 1;
    orc_ct *c0 = e ? orc_op_mult_int(P, in, (int64_t)1 << e) : orc_ct_copy(P, in);
    orc_ct *low = orc_ct_alloc(P, 0, 2);
    for (int c = 0; c < 2; c++) memcpy(LIMB(P, low, c, 0), LIMB(P, c0, c, 0), sizeof(u64) * P->n);
    orc_ct_release(c0);
    orc_ct *x = orc_bts_debug_skip_raise ? orc_ct_copy(P, in) : mod_raise(P, low);
    orc_ct_release(low);
    STOP(0, x);
    for (int k = 0; k < cf->n_cts; k++) {
        orc_ct *t = apply_ltrans(P, K, x, &B->cts[k]);
        orc_ct_release(x);
        if (!t) return NULL;
        x = t;
        STOP(1 + k, x);
    }
    orc_ct *cj = orc_op_galois(P, K, x, conj);
    if (!cj) return NULL;
    orc_ct *v = orc_op_add(P, x, cj);
    orc_ct_release(x);
    orc_ct_release(cj);
    orc_ct *v2 = orc_op_add_const(P, v, -1.0 / (4.0 * (cf->K + 2)));
    orc_ct_release(v);
    STOP(10, v2);
    /* C18 EvalMod: the cosine series is even (Jacobi-Anger: odd coefficients
     * are 0), p(v) = sum_k c_2k T_2k(v) = sum_k c_2k T_k(w), w = T_2(v) = 2 v^2 - 1:
     * one HMult and a series of half the degree on w (same depth, C13) */
    orc_ct *s;
    int even = B->cosp->deg >= 2;
    for (int i = 1; i <= B->cosp->deg; i += 2) even &= B->cosp->c[i] == 0.0;
    if (even) {
        orc_ct *vv = orc_op_mult(P, K, v2, v2);
        orc_ct *vv2 = orc_op_mult_int(P, vv, 2);
        orc_ct *w = orc_op_add_const(P, vv2, -1.0);
        orc_ct_release(vv);
        orc_ct_release(vv2);
        int hd = B->cosp->deg / 2;
        double *hc = malloc(sizeof(double) * (hd + 1));
        for (int k = 0; k <= hd; k++) hc[k] = B->cosp->c[2 * k];
        orc_cheb hp = {hd, -1.0, 1.0, hc};
        s = orc_eval_cheb_unit(P, K, w, &hp);
        orc_ct_release(w);
        free(hc);
    } else {
        s = orc_eval_cheb_unit(P, K, v2, B->cosp);
    }
    orc_ct_release(v2);
    STOP(11, s);
    for (int i = 0; i < cf->r; i++) {
        orc_ct *m = orc_op_mult(P, K, s, s);
        orc_ct *m2 = orc_op_mult_int(P, m, 2);
        orc_ct_release(s);
        orc_ct_release(m);
        s = orc_op_add_const(P, m2, -1.0);
        orc_ct_release(m2);
    }
    /* gamma = Delta_out / Delta_in: the input message m was encoded at the scale
     * of its own level, SlotToCoeff normalises by Delta_out (G11) */
    double gamma = P->scale[cf->out_level] / P->scale[in->level];
    if (cf->arcsine) {   /* s <- gamma (s + (1/6) s^3)  (arcsin(s) to O(s^5)) */
        orc_ct *s6 = orc_op_mult_const(P, s, gamma / 6.0, s->level - 1);
        orc_ct *t = orc_op_mult(P, K, s, s);
        orc_ct *u = orc_op_mult(P, K, s6, t);
        orc_ct *sg = orc_op_mult_const(P, s, gamma, u->level);
        orc_ct *w = orc_op_add(P, sg, u);
        orc_ct_release(s6);
        orc_ct_release(t);
        orc_ct_release(u);
        orc_ct_release(sg);
        orc_ct_release(s);
        s = w;
    } else {             /* s <- gamma s (one level) */
        orc_ct *sg = orc_op_mult_const(P, s, gamma, s->level - 1);
        orc_ct_release(s);
        s = sg;
    }
    STOP(12, s);
    for (int k = 0; k < cf->n_stc; k++) {
        orc_ct *t = apply_ltrans(P, K, s, &B->stc[k]);
        orc_ct_release(s);
        if (!t) return NULL;
        s = t;
        STOP(20 + k, s);
    }
    cj = orc_op_galois(P, K, s, conj);
    if (!cj) return NULL;
    orc_ct *out = orc_op_add(P, s, cj);
    orc_ct_release(s);
    orc_ct_release(cj);
    orc_ledger[LG_BTS]++;
    return out;
}

/* test hook (tests/test_oracle_bts_transforms.py): the dense float matrix of
 * the special-FFT stage group [first, first + size) of ring degree 2^log_n,
 * forward (SlotToCoeff) or inverse (CoeffToSlot), as the plan builds it
 * before its scaling factors: A[p][c] = diag_{(c - p) mod N0}[p]. */
void orc_api_sfft_group(int log_n, int first, int size, int inverse, double *re, double *im)
{
    orc_params P0;
    memset(&P0, 0, sizeof(P0));
    P0.log_n = log_n;
    P0.n = 1 << log_n;
    dmat *m = group_matrix(&P0, first, size, inverse);
    int n0 = m->n0;
    memset(re, 0, sizeof(double) * n0 * n0);
    memset(im, 0, sizeof(double) * n0 * n0);
    for (int d = 0; d < n0; d++) {
        if (!m->present[d]) continue;
        for (int p = 0; p < n0; p++) {
            re[(size_t)p * n0 + (p + d) % n0] = (double)m->diag[d][p].re;
            im[(size_t)p * n0 + (p + d) % n0] = (double)m->diag[d][p].im;
        }
    }
    dm_free(m);
}
