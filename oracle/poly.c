/*
 * oracle/poly.c -- homomorphic evaluation of a Chebyshev series (C13).
 * TEST INFRASTRUCTURE ONLY (see orc.h).
 *
 * PAPER.md 2.2.4 (lines 330-336): "a polynomial of degree d can be evaluated
 * using ceil(log(d+1)) multiplicative levels" and O(sqrt d) ct-ct products;
 * PAPER.md 424-425: degrees 2^t - 1 "maximize accuracy for a fixed-level
 * budget of t".  DESIGN.md C13 (round 2, level-exact) fixes the tree both
 * sides follow:
 *   input  W encrypts w = alpha x, alpha = 2/(b-a) (the caller folds the
 *          affine map's factor into what it feeds in, G28);
 *          T_1 = u = W + beta, beta = -(a+b)/(b-a) (a constant add, no level);
 *   gain   the series is multiplied by g: c_i <- g c_i before the split;
 *   t = ceil(log2(d+1)), baby size B = 2^ceil(t/2) (B = 2 when d <= 1),
 *          T_i = 2 T_a T_b - T_{a-b} with a = 2^(ceil(log2 i)-1), b = i-a,
 *          giants T_B .. T_{2^(t-1)} by doubling;
 *   rec(p, target): a LEAF when deg p < B and every T_i it reads sits at
 *          level >= target+1; otherwise split at g = 2^(ceil(log2(deg+1))-1):
 *          p = q T_g + r (q_0 = c_g, q_k = 2 c_{g+k}, r_{g-k} = c_{g-k} - c_{g+k}),
 *          out = rec(q, target+1) * T_g + rec(r, target)  (T_g a baby when g < B);
 *   leaf:  rescale(sum_i rint(c_i sc_i) T_i |target+1) + c_0  (one rescale);
 *   target = level(W) - t: depth exactly ceil(log2(d+1)) (1 for d <= 1).
 * A leaf never reads a basis element at its own target level, so the deepest
 * baby of every leaf gets its coefficient one level above it: the split
 * recurses until that holds (down to c_0 + c_1 T_1 if needed).
 */
#include "orc.h"
#include <stdlib.h>
#include <string.h>

static int ceil_log2(int x) { int t = 0; while ((1 << t) < x) t++; return t; }

int orc_cheb_depth(int deg) { return deg <= 1 ? 1 : ceil_log2(deg + 1); }

typedef struct {
    const orc_params *P;
    const orc_keys *K;
    int B, t;
    orc_ct **T;    /* baby steps T_0..T_{B-1} (T_0 unused) */
    orc_ct **G;    /* giants: G[j] = T_{B 2^j} */
} ev_t;

static orc_ct *leaf(ev_t *E, const double *c, int d, int target)
{
    const orc_params *P = E->P;
    int N = P->n;
    orc_ct *acc = orc_ct_alloc(P, target + 1, 2);
    for (int i = 1; i <= d; i++) {
        if (c[i] == 0.0) continue;
        orc_ct *Ti = E->T[i];
        double sc = (P->scale[target] * (double)P->prime[target + 1]) / P->scale[Ti->level];
        double v = c[i] * sc;
        for (int l = 0; l <= target + 1; l++) {
            u64 q = P->prime[l], C = orc_residue_of_double(v, q);
            for (int k = 0; k < 2; k++) {
                u64 *o = LIMB(P, acc, k, l);
                const u64 *s = LIMB(P, Ti, k, l);
                for (int x = 0; x < N; x++) o[x] = orc_add(o[x], orc_mul(s[x], C, q), q);
            }
        }
        orc_ledger[LG_CMULT]++;
    }
    orc_ct *r = orc_op_rescale(P, acc);
    orc_ct_release(acc);
    orc_ct *r2 = orc_op_add_const(P, r, c[0]);
    orc_ct_release(r);
    return r2;
}

/* a leaf may read T_1..T_d only if they all lie above its target level */
static int leaf_ok(const ev_t *E, int d, int target)
{
    if (d >= E->B) return 0;
    for (int i = 1; i <= (d > 0 ? d : 1); i++)
        if (E->T[i]->level < target + 1) return 0;
    return 1;
}

static orc_ct *rec(ev_t *E, const double *c, int d, int target)
{
    if (leaf_ok(E, d, target)) return leaf(E, c, d, target);
    int g = 1 << (ceil_log2(d + 1) - 1);
    double *q = malloc(sizeof(double) * (d - g + 1));
    double *r = malloc(sizeof(double) * g);
    q[0] = c[g];
    for (int k = 1; k <= d - g; k++) q[k] = 2.0 * c[g + k];
    for (int j = 0; j < g; j++) r[j] = c[j];
    for (int k = 1; k <= d - g; k++) r[g - k] = c[g - k] - c[g + k];
    orc_ct *Q = rec(E, q, d - g, target + 1);
    const orc_ct *Tg = g < E->B ? E->T[g] : E->G[ceil_log2(g / E->B)];
    orc_ct *QT = orc_op_mult(E->P, E->K, Q, Tg);
    orc_ct *R = rec(E, r, g - 1, target);
    orc_ct *out = orc_op_add(E->P, QT, R);
    orc_ct_release(Q);
    orc_ct_release(QT);
    orc_ct_release(R);
    free(q);
    free(r);
    return out;
}

/* 2 X^2 - 1 */
static orc_ct *cheb_double(const orc_params *P, const orc_keys *K, const orc_ct *x)
{
    orc_ct *s = orc_op_mult(P, K, x, x);
    orc_ct *s2 = orc_op_mult_int(P, s, 2);
    orc_ct *r = orc_op_add_const(P, s2, -1.0);
    orc_ct_release(s);
    orc_ct_release(s2);
    return r;
}

orc_ct *orc_eval_cheb_unit(const orc_params *P, const orc_keys *K, const orc_ct *u, const orc_cheb *p)
{
    int d = p->deg;
    ev_t E = {P, K, 0, 0, NULL, NULL};
    E.t = ceil_log2(d + 1);
    E.B = 1 << ((E.t + 1) / 2);
    if (d <= 1) E.B = 2;
    E.T = calloc(E.B, sizeof(orc_ct *));
    E.T[1] = orc_ct_copy(P, u);
    for (int i = 2; i < E.B; i++) {
        int a = 1 << (ceil_log2(i) - 1), b = i - a;
        if (a == b) {
            E.T[i] = cheb_double(P, K, E.T[a]);
        } else {
            orc_ct *m = orc_op_mult(P, K, E.T[a], E.T[b]);
            orc_ct *m2 = orc_op_mult_int(P, m, 2);
            E.T[i] = orc_op_sub(P, m2, E.T[a - b]);
            orc_ct_release(m);
            orc_ct_release(m2);
        }
    }
    int ng = E.t - ceil_log2(E.B);
    if (ng < 0) ng = 0;
    E.G = calloc(ng > 0 ? ng : 1, sizeof(orc_ct *));
    for (int j = 0; j < ng; j++) E.G[j] = cheb_double(P, K, j == 0 ? E.T[E.B / 2] : E.G[j - 1]);
    int target = u->level - orc_cheb_depth(d);
    orc_ct *out = rec(&E, p->c, d, target);
    for (int i = 1; i < E.B; i++) orc_ct_release(E.T[i]);
    for (int j = 0; j < ng; j++) orc_ct_release(E.G[j]);
    free(E.T);
    free(E.G);
    return out;
}

/* G28: W already holds alpha x; u = W + beta costs no level.  The series is
 * scaled by `gain` (the caller's output gain) before the C13 split. */
orc_ct *orc_eval_cheb(const orc_params *P, const orc_keys *K, const orc_ct *w, const orc_cheb *p, double gain)
{
    double *c = malloc(sizeof(double) * (p->deg + 1));
    for (int i = 0; i <= p->deg; i++) c[i] = gain * p->c[i];
    orc_cheb g = {p->deg, p->a, p->b, c};
    orc_ct *out;
    if (p->a == -1.0 && p->b == 1.0) {
        out = orc_eval_cheb_unit(P, K, w, &g);
    } else {
        double beta = -(p->a + p->b) / (p->b - p->a);
        orc_ct *u = orc_op_add_const(P, w, beta);
        out = orc_eval_cheb_unit(P, K, u, &g);
        orc_ct_release(u);
    }
    free(c);
    return out;
}
