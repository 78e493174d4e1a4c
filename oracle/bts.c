/*
 * oracle/bts.c -- real-slot CKKS bootstrapping of the oracle.
 * TEST INFRASTRUCTURE ONLY (see orc.h).
 *
 * PAPER.md 281-283 and 429-440 require bootstrapping (BTS) but give none of
 * its internals (HEaaN FGb, PAPER.md 386-393).  DESIGN.md reading G11 fixes a
 * textbook CoeffToSlot-first bootstrap specialised to real slot values (all
 * Softmax data are real):
 *   1. drop to level 0; ModRaise to level L (centred lift of the q_0 residues);
 *   2. CoeffToSlot: three sparse linear transforms (groups of inverse special-
 *      FFT stages), slot p then holds kappa (c_j + i c_{j+N0}) / q_0, j = brv(p);
 *   3. v = w + conj(w) - 1/(4(K+2))  (real part, mapped onto [-1, 1]);
 *   4. EvalMod: Chebyshev series of cos(2 pi (K+2) v / 2^r), r double angles
 *      -> sin(2 pi c_j / q_0) ~ 2 pi m_j / q_0;
 *   5. SlotToCoeff: three transforms (groups of special-FFT stages) with the
 *      factor q_0 / (4 pi Delta_out) and D = diag(1, 2, ..., 2) (real-message
 *      identity z = Re(V D m_lo)), then out = x + conj(x).
 * Each linear transform is a baby-step/giant-step diagonal evaluation landing
 * at the canonical scale of the next level (one rescale).
 */
#include "orc.h"
#include <math.h>
#include <quadmath.h>
#include <stdlib.h>
#include <string.h>

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
typedef struct {
    int level;           /* input level of this transform          */
    int u, b1;           /* step unit, baby size                   */
    int n_terms;
    int *g, *b;          /* per term: giant index, baby index      */
    u64 **pt;            /* per term: NTT residues, level+1 limbs  */
} ltrans;

typedef struct {
    const orc_params *P;
    int K, r, e;
    const orc_cheb *cosp;
    ltrans cts[3], stc[3];
    int out_level;
} orc_bts_plan;

/* all plans of one parameter set, one per pre-scaling exponent e */
#define ORC_BTS_EMAX 30
typedef struct {
    const orc_params *P;
    int K, r, out_level;
    orc_cheb cosp;
    double *coeffs;
    orc_bts_plan *plan[ORC_BTS_EMAX + 1];
} orc_bts_set;

static int ilog2i(int x) { int t = 0; while ((1 << t) < x) t++; return t; }

static void group_sizes(int s, int *sz)
{
    int rem = s;
    for (int k = 3, i = 0; k >= 1; k--, i++) { sz[i] = (rem + k - 1) / k; rem -= sz[i]; }
}

/* encode a transform at input level `level` */
static void make_ltrans(const orc_params *P, const dmat *m, int level, int u, int r, ltrans *T)
{
    int n0 = P->n / 2, N = P->n;
    T->level = level;
    T->u = u;
    T->b1 = 1 << ((r + 2) / 2);   /* 2^ceil((r+1)/2) */
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
        double *re = malloc(sizeof(double) * n0), *im = malloc(sizeof(double) * n0);
        const qz *v = m->diag[dl[k]];
        for (int p = 0; p < n0; p++) {           /* rot(diag, -G)_p = diag_{p - G} */
            qz x = v[((p - G) % n0 + n0) % n0];
            re[p] = (double)x.re;
            im[p] = (double)x.im;
        }
        u64 *pt = malloc(sizeof(u64) * (size_t)(level + 1) * N);
        orc_encode_coeffs(P, re, im, sc, level, pt);
        for (int i = 0; i <= level; i++) orc_ntt_fwd(P, i, pt + (size_t)i * N);
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

/* the rotations (left, slots) a plan needs: babies b u, giants g b1 u */
int orc_bts_rotations(const orc_params *P, int *out, int max)
{
    int n0 = P->n / 2, s = ilog2i(n0), sz[3], cnt = 0, first = 0;
    group_sizes(s, sz);
    for (int gi = 0; gi < 3; gi++) {
        int u = 1 << first, r = sz[gi], b1 = 1 << ((r + 2) / 2);
        int span = (1 << r) - 1;  /* idx in [-span, span] mod n0/u */
        int mod = n0 / u;
        for (int idx = -span; idx <= span; idx++) {
            int id = ((idx % mod) + mod) % mod;
            int rots[2] = {(id % b1) * u, (id / b1) * b1 * u};
            for (int t = 0; t < 2; t++) {
                int rr = rots[t] % n0;
                if (!rr) continue;
                int dup = 0;
                for (int i = 0; i < cnt; i++) if (out[i] == rr) dup = 1;
                if (!dup && cnt < max) out[cnt++] = rr;
            }
        }
        first += r;
    }
    return cnt;
}

/* e: the input is multiplied by 2^e before ModRaise (message pre-scaling,
 * DESIGN.md G11); SlotToCoeff divides it back. */
orc_bts_plan *orc_bts_plan_new(const orc_params *P, int K, int r, const orc_cheb *cosp, int out_level, int e)
{
    orc_bts_plan *B = calloc(1, sizeof(*B));
    B->e = e;
    B->P = P;
    B->K = K;
    B->r = r;
    B->cosp = cosp;
    B->out_level = out_level;
    int N = P->n, n0 = N / 2, s = ilog2i(n0), sz[3];
    group_sizes(s, sz);
    int L = P->L;
    dmat *grp[3];
    int first[3];
    for (int gi = 0, st = 0; gi < 3; gi++) {
        first[gi] = st;
        dmat *acc = NULL;
        for (int i = st; i < st + sz[gi]; i++) {
            dmat *S = stage(P->log_n, 2 << i, 0);
            if (!acc) acc = S;
            else { dmat *t = compose(S, acc); dm_free(S); dm_free(acc); acc = t; }
        }
        grp[gi] = acc;
        st += sz[gi];
    }
    /* SlotToCoeff: M_0 diag(lambda D), M_1, M_2 at levels out+3, out+2, out+1 */
    f128 lam = (f128)P->prime[0] / (4 * M_PIq * (f128)P->scale[out_level] * ldexpq(1, e));
    f128 *dv = malloc(sizeof(f128) * n0);
    for (int p = 0; p < n0; p++) dv[p] = p == 0 ? lam : 2 * lam;
    dm_scale_cols(grp[0], dv);
    free(dv);
    for (int gi = 0; gi < 3; gi++) make_ltrans(P, grp[gi], out_level + 3 - gi, 1 << first[gi], sz[gi], &B->stc[gi]);
    for (int gi = 0; gi < 3; gi++) dm_free(grp[gi]);
    /* CoeffToSlot: inverse groups in reverse order, factor kappa Delta_L / q0 first */
    for (int k = 0; k < 3; k++) {
        int gi = 2 - k;
        dmat *acc = NULL;
        for (int i = first[gi] + sz[gi] - 1; i >= first[gi]; i--) {
            dmat *S = stage(P->log_n, 2 << i, 1);
            if (!acc) acc = S;
            else { dmat *t = compose(S, acc); dm_free(S); dm_free(acc); acc = t; }
        }
        if (k == 0) {
            f128 f = ((f128)P->scale[L] / (f128)P->prime[0]) / (2 * (f128)(K + 2));
            f128 *fv = malloc(sizeof(f128) * n0);
            for (int p = 0; p < n0; p++) fv[p] = f;
            dm_scale_cols(acc, fv);
            free(fv);
        }
        make_ltrans(P, acc, L - k, 1 << first[gi], sz[gi], &B->cts[k]);
        dm_free(acc);
    }
    return B;
}

void orc_bts_plan_free(orc_bts_plan *B)
{
    if (!B) return;
    for (int k = 0; k < 3; k++) { free_ltrans(&B->cts[k]); free_ltrans(&B->stc[k]); }
    free(B);
}

/* ct (level T->level, 2 comps) -> transform, landing at level-1 */
static orc_ct *apply_ltrans(const orc_params *P, const orc_keys *K, const orc_ct *ct0, const ltrans *T)
{
    int N = P->n, n0 = N / 2, l = T->level;
    orc_ct *ct = orc_op_level_down(P, ct0, l);
    /* baby rotations */
    orc_ct *R[64] = {0};
    for (int k = 0; k < T->n_terms; k++) {
        int b = T->b[k];
        if (R[b]) continue;
        R[b] = b == 0 ? orc_ct_copy(P, ct) : orc_op_rotate(P, K, ct, b * T->u);
        if (!R[b]) return NULL;
    }
    int maxg = 0;
    for (int k = 0; k < T->n_terms; k++) if (T->g[k] > maxg) maxg = T->g[k];
    orc_ct *acc = orc_ct_alloc(P, l, 2);
    for (int g = 0; g <= maxg; g++) {
        orc_ct *inner = NULL;
        for (int k = 0; k < T->n_terms; k++) {
            if (T->g[k] != g) continue;
            if (!inner) inner = orc_ct_alloc(P, l, 2);
            const orc_ct *Rb = R[T->b[k]];
            for (int i = 0; i <= l; i++) {
                u64 q = P->prime[i];
                const u64 *m = T->pt[k] + (size_t)i * N;
                for (int c = 0; c < 2; c++) {
                    u64 *o = LIMB(P, inner, c, i);
                    const u64 *s = LIMB(P, Rb, c, i);
                    for (int t = 0; t < N; t++) o[t] = orc_add(o[t], orc_mul(s[t], m[t], q), q);
                }
            }
            orc_ledger[LG_PMULT]++;
        }
        if (!inner) continue;
        if (g != 0) {
            orc_ct *rot = orc_op_rotate(P, K, inner, (g * T->b1 * T->u) % n0);
            orc_ct_release(inner);
            if (!rot) return NULL;
            inner = rot;
        }
        for (int i = 0; i <= l; i++) {
            u64 q = P->prime[i];
            for (int c = 0; c < 2; c++) {
                u64 *o = LIMB(P, acc, c, i);
                const u64 *s = LIMB(P, inner, c, i);
                for (int t = 0; t < N; t++) o[t] = orc_add(o[t], s[t], q);
            }
        }
        orc_ct_release(inner);
    }
    for (int b = 0; b < 64; b++) orc_ct_release(R[b]);
    orc_ct_release(ct);
    orc_ct *out = orc_op_rescale(P, acc);
    orc_ct_release(acc);
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

int orc_bts_debug_stop = -1;  /* test hook: return the intermediate after this stage */
int orc_bts_debug_skip_raise = 0;  /* test hook: input is already at level L */
#define STOP(st, ct) if (orc_bts_debug_stop == (st)) return ct;

/* G11 pre-scaling exponent for a message bound B:
 * e = floor(log2 q_0 - 12 - log2 Delta_0 - log2 B) clamped to [0, 30], so that
 * |2^e m| <= 2^-12 q_0 and sin(2 pi y) ~ 2 pi y stays accurate. */
int orc_bts_exponent(const orc_params *P, double bound)
{
    double e = floor(log2((double)P->prime[0]) - 12.0 - log2(P->scale[0]) - log2(bound));
    if (e < 0) e = 0;
    if (e > ORC_BTS_EMAX) e = ORC_BTS_EMAX;
    return (int)e;
}

orc_bts_set *orc_bts_set_new(const orc_params *P, int K, int r, int deg, const double *coeffs, int out_level)
{
    orc_bts_set *S = calloc(1, sizeof(*S));
    S->P = P;
    S->K = K;
    S->r = r;
    S->out_level = out_level;
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
    for (int e = 0; e <= ORC_BTS_EMAX; e++) orc_bts_plan_free(S->plan[e]);
    free(S->coeffs);
    free(S);
}

orc_ct *orc_bootstrap(const orc_params *P, const orc_keys *K, const orc_ct *in, void *ctx, double bound)
{
    orc_bts_set *BS = ctx;
    int e = orc_bts_exponent(P, bound);
    if (!BS->plan[e]) BS->plan[e] = orc_bts_plan_new(P, BS->K, BS->r, &BS->cosp, BS->out_level, e);
    const orc_bts_plan *B = BS->plan[e];
    int conj = 2 * P->n - 1;
    orc_ct *c0 = e ? orc_op_mult_int(P, in, (int64_t)1 << e) : orc_ct_copy(P, in);
    orc_ct *low = orc_ct_alloc(P, 0, 2);
    for (int c = 0; c < 2; c++) memcpy(LIMB(P, low, c, 0), LIMB(P, c0, c, 0), sizeof(u64) * P->n);
    orc_ct_release(c0);
    orc_ct *x = orc_bts_debug_skip_raise ? orc_ct_copy(P, in) : mod_raise(P, low);
    orc_ct_release(low);
    STOP(0, x);
    for (int k = 0; k < 3; k++) {
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
    orc_ct *v2 = orc_op_add_const(P, v, -1.0 / (4.0 * (B->K + 2)));
    orc_ct_release(v);
    STOP(4, v2);
    orc_ct *s = orc_eval_cheb_unit(P, K, v2, B->cosp);
    orc_ct_release(v2);
    STOP(5, s);
    for (int i = 0; i < B->r; i++) {
        orc_ct *m = orc_op_mult(P, K, s, s);
        orc_ct *m2 = orc_op_mult_int(P, m, 2);
        orc_ct_release(s);
        orc_ct_release(m);
        s = orc_op_add_const(P, m2, -1.0);
        orc_ct_release(m2);
    }
    STOP(6, s);
    for (int k = 0; k < 3; k++) {
        orc_ct *t = apply_ltrans(P, K, s, &B->stc[k]);
        orc_ct_release(s);
        if (!t) return NULL;
        s = t;
        STOP(7 + k, s);
    }
    cj = orc_op_galois(P, K, s, conj);
    if (!cj) return NULL;
    orc_ct *out = orc_op_add(P, s, cj);
    orc_ct_release(s);
    orc_ct_release(cj);
    orc_ledger[LG_BTS]++;
    return out;
}
