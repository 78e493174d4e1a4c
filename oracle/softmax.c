/*
 * oracle/softmax.c -- the paper's Softmax over packed CKKS ciphertexts.
 * TEST INFRASTRUCTURE ONLY (see orc.h).
 *
 *   Alg 1 (normalize-and-square)  PAPER.md 776-787 [sec 3.3, alg:Softmax]
 *   Alg 2 (auxiliary thread)      PAPER.md 904-921 [sec 3.4.1, alg:AuxThread]
 *   Alg B (version B)             PAPER.md 168-181 [sec 4.3, alg:Softmax1B],
 *                                 exponent read as -1/2^j (G4)
 *   packings                      PAPER.md 94-131 [sec 4.1-4.2]
 *   many-ciphertext aux sum       DESIGN.md C15 / G6 (sum of tensors, one relin)
 *   bootstrap placement           PAPER.md 429-440 [sec 5.1.3], rule G12
 *
 * Unified packing: m ciphertexts, nb = n/m coordinate
 * blocks per ciphertext, stride = N0/nb; instance o (o < stride) of
 * coordinate block b lives in slot b*stride + o.
 */
#include "orc.h"
#include <stdlib.h>
#include <string.h>
#include <math.h>

typedef orc_ct *(*orc_bts_fn)(const orc_params *, const orc_keys *, const orc_ct *, void *, double);

typedef struct {
    int n, m, k, variant;           /* variant 0 = Alg 1, 1 = Alg B */
    const orc_cheb *exp_poly;       /* exp(x/2^k) on [-M, 0]         */
    const orc_cheb *inv_poly;       /* k polys, one per iteration     */
    orc_bts_fn bts;                 /* NULL: no bootstrapping         */
    void *bts_ctx;
} orc_softmax_desc;

enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_ELEVEL = 2, ORC_EKEY = 3 };

static int ilog2(int x) { int t = 0; while ((1 << t) < x) t++; return t; }

static void swap_in(orc_ct **slot, orc_ct *v) { orc_ct_release(*slot); *slot = v; }

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

static int poly_cost(const orc_cheb *p)
{
    return orc_cheb_depth(p->deg) + ((p->a == -1.0 && p->b == 1.0) ? 0 : 1);
}

int orc_softmax(const orc_params *P, const orc_keys *K, const orc_softmax_desc *d, orc_ct *const *x, orc_ct **out)
{
    int m = d->m, n = d->n, N0 = P->n / 2;
    if (m < 1 || n % m) return ORC_EINVAL;
    int nb = n / m;
    if ((nb & (nb - 1)) || nb > N0) return ORC_EINVAL;
    int stride = N0 / nb;
    int rc = ORC_OK;
    orc_ct **y0 = calloc(m, sizeof(orc_ct *)), **y = calloc(m, sizeof(orc_ct *));
    orc_ct *lam = NULL, *S = NULL, *lj = NULL;
    double *mask = calloc(N0, sizeof(double));
    for (int s = 0; s < stride; s++) mask[s] = 1.0;       /* G10: block 0 */

    /* y^(0) = exp(x / 2^k)  (Alg 1 line 1; Alg B line 2) */
    for (int c = 0; c < m; c++) {
        if (x[c]->level < poly_cost(d->exp_poly)) { rc = ORC_ELEVEL; goto done; }
        y0[c] = orc_eval_cheb(P, K, x[c], d->exp_poly);
        y[c] = orc_ct_copy(P, y0[c]);
    }
    for (int j = 1; j <= d->k; j++) {
        const orc_cheb *ip = &d->inv_poly[j - 1];
        /* Alg 1 main thread needs 1 (aux square) + 2 levels; bootstrap y (G12 c) */
        if (d->variant == 0 && y[0]->level < 2) {
            for (int c = 0; c < m; c++) if ((rc = bts_or_fail(P, K, d, &y[c], 1.0))) goto done;
        }
        if (y[0]->level < 1) { rc = ORC_ELEVEL; goto done; }
        /* ---- auxiliary thread (Alg 2) ---- */
        /* step 1 + C15: S = relin(sum_c tensor(y_c, y_c)) with its rescale (C8) */
        orc_ct *acc = NULL;
        for (int c = 0; c < m; c++) {
            orc_ct *t = orc_op_tensor(P, y[c], y[c]);
            if (!acc) acc = t;
            else { orc_ct *s2 = orc_op_add(P, acc, t); orc_ct_release(acc); orc_ct_release(t); acc = s2; }
        }
        S = orc_op_relin_rescale(P, K, acc);
        orc_ct_release(acc);
        /* steps 3-5: sum over the coordinate blocks (rotations by -stride 2^i) */
        if ((rc = rot_sum(P, K, &S, nb, stride, -1))) goto done;
        /* G12 (a): bootstrap before step 6 if the rest of the aux thread would
         * leave lambda below the main level.  Main level: Alg 1 -- the level of
         * y (keeps the main thread from bootstrapping); version B -- the levels
         * its update consumes, j + 2 (lambda y0, j squarings, one left for the
         * next aux square) or k + 1 at j = k, capped by y0's level (G12) */
        int need_b = j < d->k ? j + 2 : d->k + 1;
        int main_level = d->variant == 0 ? y[0]->level : (y0[0]->level < need_b ? y0[0]->level : need_b);
        int need = poly_cost(ip) + 1 + ((d->variant == 1 && j > 1) ? 1 : 0);
        if (S->level - need < main_level) {
            if (d->bts) { if ((rc = bts_or_fail(P, K, d, &S, ip->b))) goto done; }
            else if (S->level - need < 0) { rc = ORC_ELEVEL; goto done; }
        }
        /* step 6: InvSqrt (Alg 1) or x^(-1/2^j) (Alg B, G4) */
        lj = orc_eval_cheb(P, K, S, ip);
        orc_ct_release(S); S = NULL;
        /* step 7: mask block 0 */
        if (lj->level < 1) { rc = ORC_ELEVEL; goto done; }
        swap_in(&lj, orc_op_mult_pt(P, lj, mask, NULL, lj->level - 1));
        /* steps 8-10: broadcast back (rotations by +stride 2^i) */
        if ((rc = rot_sum(P, K, &lj, nb, stride, +1))) goto done;
        if (d->variant == 1 && j > 1) {
            orc_ct *t = orc_op_mult(P, K, lam, lj);      /* Alg B line 5 */
            orc_ct_release(lam); orc_ct_release(lj); lj = NULL;
            lam = t;
        } else {
            orc_ct_release(lam);
            lam = lj; lj = NULL;
        }
        /* G12 (b): bootstrap lambda again if it ended below the main level */
        if (lam->level < main_level && d->bts) {
            if ((rc = bts_or_fail(P, K, d, &lam, d->variant == 1 ? 1.5 : 1.1 / sqrt(ip->a)))) goto done;
        }
        /* ---- main thread ---- */
        for (int c = 0; c < m; c++) {
            if (d->variant == 0) {
                orc_ct *z = orc_op_mult(P, K, lam, y[c]);        /* Alg 1 line 4 */
                swap_in(&y[c], orc_op_mult(P, K, z, z));          /* Alg 1 line 5 */
                orc_ct_release(z);
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
    }
    for (int c = 0; c < m; c++) { out[c] = y[c]; y[c] = NULL; }
done:
    for (int c = 0; c < m; c++) { orc_ct_release(y0[c]); orc_ct_release(y[c]); }
    free(y0); free(y); free(mask);
    orc_ct_release(lam); orc_ct_release(S); orc_ct_release(lj);
    return rc;
}
