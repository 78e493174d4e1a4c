/*
 * oracle/softmax.c -- the paper's Softmax over packed CKKS ciphertexts.
 * TEST INFRASTRUCTURE ONLY (see orc.h).
 *
 *   Alg 1 (normalize-and-square)  PAPER.md 776-787 [sec 3.3, alg:Softmax]
 *   Alg 2 (auxiliary thread)      PAPER.md 904-921 [sec 3.4.1, alg:AuxThread]
 *   Alg B (version B)             PAPER.md 168-181 [sec 4.3, alg:Softmax1B],
 *                                 exponent read as -1/2^j (G4)
 *   square-and-normalize          PAPER.md 757-765 [sec 3.3, remark]: variant 2,
 *                                 mu_j = (sum y^2)^-1, y <- mu_j y^2 (G26)
 *   t-th power, t = 3             PAPER.md 1645-1663 [App. C]: variant 3,
 *                                 mu_j = (sum y^3)^-1, y <- mu_j y^3 (G27)
 *   packings                      PAPER.md 94-131 [sec 4.1-4.2]
 *   many-ciphertext aux sum       DESIGN.md C15 / G6 (sum of tensors, one relin)
 *   bootstrap placement           PAPER.md 429-440 [sec 5.1.3], rule G12
 *   level-exact polynomials       PAPER.md 330-336 (ceil(log(d+1)) levels) via
 *                                 the C13 tree; the affine map's factor folded
 *                                 into gains (G28): the input holds
 *                                 alpha_exp x, the main thread carries g_j, the
 *                                 masks the compensating factors
 *
 * Unified packing: m ciphertexts, nb = n/m coordinate
 * blocks per ciphertext, stride = N0/nb; instance o (o < stride) of
 * coordinate block b lives in slot b*stride + o.
 */
#include "orc.h"
#include <stdlib.h>
#include <string.h>
#include <math.h>

enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_ELEVEL = 2, ORC_EKEY = 3 };

static int ilog2(int x) { int t = 0; while ((1 << t) < x) t++; return t; }

static void swap_in(orc_ct **slot, orc_ct *v) { orc_ct_release(*slot); *slot = v; }

/* test hook (tests/test_oracle_levels.py): the level before and after each
 * step of the schedule, to pin the level budget against PAPER.md's depth
 * tables (tab:depth_main 964-979, tab:depth_aux_thread 1032-1058) */
enum { TR_EXP, TR_SQUARE, TR_POLY, TR_MASK, TR_MAIN, TR_BTS_MAIN, TR_BTS_AUX, TR_LAMBDA };
int orc_trace_on = 0, orc_trace_n = 0;
int orc_trace[512][4];   /* {event, iteration j, level in, level out} */
static void trace(int ev, int j, int lin, int lout)
{
    if (!orc_trace_on || orc_trace_n >= 512) return;
    orc_trace[orc_trace_n][0] = ev;
    orc_trace[orc_trace_n][1] = j;
    orc_trace[orc_trace_n][2] = lin;
    orc_trace[orc_trace_n][3] = lout;
    orc_trace_n++;
}

/* S <- S + Rot(S, sign * stride * 2^i) for i < log2(nb) */
static int rot_sum(const orc_params *P, const orc_keys *K, orc_ct **S, int nb, int stride, int sign)
{
    for (int i = 0; (1 << i) < nb; i++) {
        orc_ct *r = orc_op_rotate(P, K, *S, sign * stride * (1 << i));
        if (!r) return ORC_EKEY;
        swap_in(S, orc_op_add(P, *S, r));
        orc_ct_release(r);
    }
    return ORC_OK;
}

static int bts_or_fail(const orc_params *P, const orc_keys *K, const orc_softmax_desc *d, orc_ct **c, double bound)
{
    if (!d->bts) return ORC_ELEVEL;
    orc_ct *b = d->bts(P, K, *c, d->bts_ctx, bound);
    if (!b) return ORC_ELEVEL;
    swap_in(c, b);
    return ORC_OK;
}

/* PAPER.md 1313-1316: z1 = (x/2) y; z2 = y y; z3 = (3/2) y; return z3 - z1 z2.
 * xh = x/2 is computed once by the caller.  Levels (C11, C12): z1 at
 * min(l(xh), l(y)) - 1, z2 at l(y) - 1, z1 z2 one below the lower of the two,
 * z3 multiplied straight to that level, so the step costs 2 levels. */
orc_ct *orc_newton_invsqrt_step(const orc_params *P, const orc_keys *K, const orc_ct *xh, const orc_ct *y)
{
    orc_ct *z1 = orc_op_mult(P, K, xh, y);
    orc_ct *z2 = orc_op_mult(P, K, y, y);
    orc_ct *p = orc_op_mult(P, K, z1, z2);
    orc_ct *z3 = orc_op_mult_const(P, y, 1.5, p->level);
    orc_ct *r = orc_op_sub(P, z3, p);
    orc_ct_release(z1); orc_ct_release(z2); orc_ct_release(p); orc_ct_release(z3);
    return r;
}

/* C13 (level-exact): a polynomial costs ceil(log2(d+1)) levels; its affine
 * map is folded into the gains below (G28) */
static int poly_cost(const orc_cheb *p) { return orc_cheb_depth(p->deg); }

static double alpha_of(const orc_cheb *p) { return 2.0 / (p->b - p->a); }
static double root2k(double x, int k)   /* x^(1/2^k) by k correctly rounded square roots */
{
    for (int i = 0; i < k; i++) x = sqrt(x);
    return x;
}

/* G28 gains (G28).  Every polynomial reads alpha x instead of x.  The
 * main thread carries y'_j = g_j y_j so that the aux sum of iteration j+1 is
 * S' = alpha_{j+1} S (g_j^e = alpha_{j+1}, e = 2, or 3 for the cube variant);
 * the exp polynomial's output gain is g_0; the mask of iteration j carries
 * mu_j, the factor that turns the true lambda_j into the gain the next main
 * update needs; g_k = 1 (the output is y itself).  alpha_j belongs to
 * inv_poly[j-1].
 *   Alg 1:           mu_j = sqrt(g_j) / g_{j-1}        (y_j = (mu_j lambda_j y_{j-1})^2)
 *   square-and-norm: mu_j = g_j / g_{j-1}^2             (y_j = mu_j lambda_j y_{j-1}^2)
 *   cube-and-norm:   mu_j = g_j / g_{j-1}^3             (y_j = mu_j lambda_j y_{j-1}^3)
 *   version B:       lambda carries c_j = alpha_{j+1}^(1/2^(j+1)) / g_0 (c_k = 1/g_0,
 *                    c_0 = 1), so (c_j g_0 Lambda_j y0)^(2^j) = sqrt(alpha_{j+1}) y^(j);
 *                    mu_j = c_j / c_{j-1}. */
static void gains(const orc_softmax_desc *d, double *g, double *mu, double *c)
{
    int k = d->k;
    for (int j = 0; j <= k; j++) {
        double a = j < k ? alpha_of(&d->inv_poly[j]) : 1.0;
        g[j] = j == k ? 1.0 : d->variant == 3 ? cbrt(a) : sqrt(a);
    }
    c[0] = 1.0;
    mu[0] = 1.0;
    for (int j = 1; j <= k; j++) {
        if (d->variant == 1) {
            c[j] = j < k ? root2k(alpha_of(&d->inv_poly[j]), j + 1) / g[0] : 1.0 / g[0];
            mu[j] = c[j] / c[j - 1];
        } else {
            c[j] = 1.0;
            if (d->variant == 0) mu[j] = sqrt(g[j]) / g[j - 1];
            else if (d->variant == 2) mu[j] = g[j] / (g[j - 1] * g[j - 1]);
            else mu[j] = g[j] / (g[j - 1] * g[j - 1] * g[j - 1]);
        }
    }
}

int orc_softmax(const orc_params *P, const orc_keys *K, const orc_softmax_desc *d, orc_ct *const *x, orc_ct **out)
{
    int m = d->m, n = d->n, N0 = P->n / 2;
    if (m < 1 || n % m || d->variant < 0 || d->variant > 3 || d->newton < 0 || (d->newton > 0 && d->variant != 0))
        return ORC_EINVAL;
    /* the cube variant's main update consumes 3 levels (y^2, y^3, mu y^3) */
    int main_need = d->variant == 3 ? 3 : 2;
    /* Alg 1 and square-and-normalize share the schedule (variant 0 / 2) */
    int alg1 = d->variant != 1;
    int nb = n / m;
    if ((nb & (nb - 1)) || nb > N0) return ORC_EINVAL;
    int stride = N0 / nb;
    int rc = ORC_OK;
    orc_ct **y0 = calloc(m, sizeof(orc_ct *)), **y = calloc(m, sizeof(orc_ct *));
    orc_ct *lam = NULL, *S = NULL, *lj = NULL;
    orc_ct **w = NULL;  /* G27: the squares y_c^2 of the current iteration */
    double *mask = calloc(N0, sizeof(double));
    double *g = calloc(d->k + 1, sizeof(double)), *mu = calloc(d->k + 1, sizeof(double));
    double *cb = calloc(d->k + 1, sizeof(double));
    gains(d, g, mu, cb);

    /* y^(0) = exp(x / 2^k)  (Alg 1 line 1; Alg B line 2); x arrives as
     * alpha_exp x (G28), y0 leaves with gain g_0 */
    for (int c = 0; c < m; c++) {
        if (x[c]->level < poly_cost(d->exp_poly)) { rc = ORC_ELEVEL; goto done; }
        y0[c] = orc_eval_cheb(P, K, x[c], d->exp_poly, g[0]);
        if (c == 0) trace(TR_EXP, 0, x[c]->level, y0[c]->level);
        y[c] = orc_ct_copy(P, y0[c]);
    }
    for (int j = 1; j <= d->k; j++) {
        const orc_cheb *ip = &d->inv_poly[j - 1];
        /* Alg 1 main thread needs 1 (aux square) + 2 levels; bootstrap y (G12 c) */
        if (alg1 && y[0]->level < main_need) {
            for (int c = 0; c < m; c++) if ((rc = bts_or_fail(P, K, d, &y[c], 1.0 * g[j - 1]))) goto done;
            trace(TR_BTS_MAIN, j, -1, y[0]->level);
        }
        if (y[0]->level < 1) { rc = ORC_ELEVEL; goto done; }
        /* ---- auxiliary thread (Alg 2) ---- */
        /* step 1 + C15: S = relin(sum_c tensor(y_c, y_c)) with its rescale (C8);
         * G27: S = relin(sum_c tensor(w_c, y_c)), w_c = y_c^2 */
        orc_ct *acc = NULL;
        w = d->variant == 3 ? calloc(m, sizeof(orc_ct *)) : NULL;
        for (int c = 0; c < m; c++) {
            if (w) w[c] = orc_op_mult(P, K, y[c], y[c]);
            orc_ct *t = w ? orc_op_tensor(P, w[c], y[c]) : orc_op_tensor(P, y[c], y[c]);
            if (!acc) acc = t;
            else { orc_ct *s2 = orc_op_add(P, acc, t); orc_ct_release(acc); orc_ct_release(t); acc = s2; }
        }
        S = orc_op_relin_rescale(P, K, acc);
        trace(TR_SQUARE, j, y[0]->level, S->level);
        orc_ct_release(acc);
        /* steps 3-5: sum over the coordinate blocks (rotations by -stride 2^i) */
        if ((rc = rot_sum(P, K, &S, nb, stride, -1))) goto done;
        /* G12 (a): bootstrap before step 6 if the rest of the aux thread would
         * leave lambda below the main level.  Main level: Alg 1 -- the level of
         * y (keeps the main thread from bootstrapping), at j = k only the 2
         * levels of the last update; version B -- the levels its update
         * consumes, j + 2 (lambda y0, j squarings, one left for the next aux
         * square) or k + 1 at j = k, capped by y0's level (G12) */
        int need_b = j < d->k ? j + 2 : d->k + 1;
        int main_a = j < d->k ? y[0]->level : (y[0]->level < 2 ? y[0]->level : 2);
        int main_level = alg1 ? main_a : (y0[0]->level < need_b ? y0[0]->level : need_b);
        int need = poly_cost(ip) + 1 + ((d->variant == 1 && j > 1) ? 1 : 0);
        /* G24: Newton steps after the last polynomial read x/2 (one level below
         * S), 2 levels each, then the mask: S must also supply 2 t + 2 levels */
        int nt = j == d->k ? d->newton : 0;
        if (nt > 0 && 2 * nt + 2 > need) need = 2 * nt + 2;
        if (S->level - need < main_level) {
            if (d->bts) {
                if ((rc = bts_or_fail(P, K, d, &S, alpha_of(ip) * ip->b))) goto done;
                trace(TR_BTS_AUX, j, -1, S->level);
            }
            else if (S->level - need < 0) { rc = ORC_ELEVEL; goto done; }
        }
        /* step 6: InvSqrt (Alg 1) or x^(-1/2^j) (Alg B, G4) */
        lj = orc_eval_cheb(P, K, S, ip, 1.0);   /* S holds alpha_j S (G28) */
        trace(TR_POLY, j, S->level, lj->level);
        if (nt > 0) {
            /* G24 (n): bootstrap the seed when the Newton steps and the mask
             * would leave lambda below the main level */
            int top = lj->level < S->level - 1 ? lj->level : S->level - 1;
            if (top - 2 * nt - 1 < main_level && d->bts) {
                if ((rc = bts_or_fail(P, K, d, &lj, 1.1 / sqrt(ip->a)))) goto done;
                top = lj->level < S->level - 1 ? lj->level : S->level - 1;
            }
            if (top - 2 * nt - 1 < 0) { rc = ORC_ELEVEL; goto done; }
            orc_ct *xh = orc_op_mult_const(P, S, 0.5 / alpha_of(ip), S->level - 1);   /* x/2 from alpha x */
            for (int t = 0; t < nt; t++) swap_in(&lj, orc_newton_invsqrt_step(P, K, xh, lj));
            orc_ct_release(xh);
        }
        orc_ct_release(S); S = NULL;
        /* Alg B line 5, taken BEFORE the mask: lambda_j holds its value in every
         * coordinate block (S was summed over all of them), so the product
         * lambda * lambda_j is the new lambda everywhere */
        if (d->variant == 1 && j > 1) {
            orc_ct *t = orc_op_mult(P, K, lam, lj);
            trace(TR_LAMBDA, j, lj->level < lam->level ? lj->level : lam->level, t->level);
            orc_ct_release(lj);
            lj = t;
        }
        /* G12 (b): bootstrap lambda_j (version B: the product) BEFORE the mask
         * when the mask would leave it below the main level: the broadcast then
         * copies block 0's value, so every coordinate of an instance sees the
         * same bootstrapping error (a common factor the next normalisation
         * absorbs) instead of an independent one per slot */
        if (lj->level - 1 < main_level && d->bts) {
            double bound = d->variant >= 2 ? 1.1 / ip->a : (d->variant == 1 && j > 1) ? 1.5 * cb[j - 1] : 1.1 / sqrt(ip->a);
            if ((rc = bts_or_fail(P, K, d, &lj, bound))) goto done;
            trace(TR_BTS_AUX, j, -1, lj->level);
        }
        /* step 7: mask block 0 (G10), carrying the gain factor mu_j (G28) */
        if (lj->level < 1) { rc = ORC_ELEVEL; goto done; }
        for (int s2 = 0; s2 < stride; s2++) mask[s2] = mu[j];
        int lvm = lj->level;
        swap_in(&lj, orc_op_mult_pt(P, lj, mask, NULL, lj->level - 1));
        trace(TR_MASK, j, lvm, lj->level);
        /* steps 8-10: broadcast back (rotations by +stride 2^i) */
        if ((rc = rot_sum(P, K, &lj, nb, stride, +1))) goto done;
        orc_ct_release(lam);
        lam = lj; lj = NULL;
        /* ---- main thread ---- */
        if (lam->level < 1) { rc = ORC_ELEVEL; goto done; }
        int main_in = y[0]->level;
        for (int c = 0; c < m; c++) {
            if (d->variant == 0) {
                orc_ct *z = orc_op_mult(P, K, lam, y[c]);        /* Alg 1 line 4 */
                /* G12 (c'): bootstrap the normalised z (|z| <= 1 + alpha, larger
                 * than y) when its square would leave y below the 2 levels the
                 * next iteration needs */
                if (d->bts && j < d->k && z->level - 1 < 2) {
                    orc_ct *zb = d->bts(P, K, z, d->bts_ctx, 1.1 * sqrt(g[j]));
                    if (!zb) { orc_ct_release(z); rc = ORC_ELEVEL; goto done; }
                    orc_ct_release(z);
                    z = zb;
                }
                swap_in(&y[c], orc_op_mult(P, K, z, z));          /* Alg 1 line 5 */
                orc_ct_release(z);
            } else if (d->variant == 2) {
                orc_ct *w2 = orc_op_mult(P, K, y[c], y[c]);       /* square ...      */
                swap_in(&y[c], orc_op_mult(P, K, lam, w2));       /* ... and normalize */
                orc_ct_release(w2);
            } else if (d->variant == 3) {
                orc_ct *y3 = orc_op_mult(P, K, w[c], y[c]);       /* cube ...        */
                swap_in(&y[c], orc_op_mult(P, K, lam, y3));       /* ... and normalize */
                orc_ct_release(y3);
            } else {
                orc_ct *z = orc_op_mult(P, K, lam, y0[c]);       /* Alg B line 6 */
                for (int s = 0; s < j; s++) {                     /* Alg B line 7 */
                    if (z->level < 1) { orc_ct_release(z); rc = ORC_ELEVEL; goto done; }
                    orc_ct *z2 = orc_op_mult(P, K, z, z);
                    orc_ct_release(z);
                    z = z2;
                }
                swap_in(&y[c], z);
            }
        }
        {
            /* the main update read lambda and y (Alg 1, variants 2/3) or y0 (Alg B) */
            int src = d->variant == 1 ? y0[0]->level : main_in;
            trace(TR_MAIN, j, lam->level < src ? lam->level : src, y[0]->level);
        }
        if (w) {
            for (int c = 0; c < m; c++) orc_ct_release(w[c]);
            free(w);
            w = NULL;
        }
    }
    for (int c = 0; c < m; c++) { out[c] = y[c]; y[c] = NULL; }
done:
    if (w) {
        for (int c = 0; c < m; c++) orc_ct_release(w[c]);
        free(w);
    }
    for (int c = 0; c < m; c++) { orc_ct_release(y0[c]); orc_ct_release(y[c]); }
    free(y0); free(y); free(mask); free(g); free(mu); free(cb);
    orc_ct_release(lam); orc_ct_release(S); orc_ct_release(lj);
    return rc;
}
