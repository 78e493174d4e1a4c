// softmax.cpp -- the paper's Softmax over packed ciphertexts (product side).
//
//   Alg 1 normalize-and-square   PAPER.md 776-787 [sec 3.3, alg:Softmax]
//   Alg 2 auxiliary thread       PAPER.md 904-921 [sec 3.4.1, alg:AuxThread]
//   version B                    PAPER.md 168-181 [sec 4.3], exponent -1/2^j (G4)
//   square-and-normalize         PAPER.md 757-765 [sec 3.3, remark], variant 2:
//                                mu_j = (sum y^2)^-1, y <- mu_j y^2 (G26)
//   t-th power, t = 3            PAPER.md 1645-1663 [App. C], variant 3:
//                                mu_j = (sum y^3)^-1, y <- mu_j y^3 (G27)
//   one / many ciphertexts       PAPER.md 94-131 [sec 4.1-4.2]
//   shared aux sum               DESIGN.md C15 / G6: sum_c tensor(y_c, y_c)
//                                exactly mod q, ONE relin + rescale
//   bootstrap placement          PAPER.md 429-440 [sec 5.1.3], rule G12
//   Newton inverse square root   PAPER.md 1311-1327 [App. A] (G22 reading of
//                                the printed step), after the last polynomial
//                                of Alg 1 when d->newton > 0 (G24)
//
// Sharding: rank r owns ciphertexts [r m/G, (r+1) m/G).
// The only exchange is the degree-2 partial aux sum of each iteration; the
// gathered partials are added mod q (exact, order-free), so every rank runs
// the replicated aux thread on identical words and all outputs are identical
// to the single-GPU run.
#include <math.h>

#include <algorithm>
#include <vector>

#include "hs_internal.h"

namespace {

int poly_cost(const hs_poly *p) { return cheb_depth(p->deg) + ((p->a == -1.0 && p->b == 1.0) ? 0 : 1); }

void rot_sum(const hs_keys *K, CtP &S, int nb, int stride, int sign, cudaStream_t st)
{
    for (int i = 0; (1 << i) < nb; i++) {
        CtP r = ev_rotate(K, S.get(), sign * stride * (1 << i), st);
        S = ev_add(S.get(), r.get(), false, st);
    }
}

[[noreturn]] void level_error(const char *what) { throw HsError(HS_ELEVEL, std::string("softmax: ") + what); }

// PAPER.md 1313-1316: z1 = (x/2) y; z2 = y y; z3 = (3/2) y; y' = z3 - z1 z2
// (2 levels; z3 multiplied straight to the level of z1 z2, C12)
CtP newton_step(const hs_keys *K, const hs_ct *xh, const hs_ct *y, cudaStream_t st)
{
    CtP z1 = ev_mult(K, xh, y, st);
    CtP z2 = ev_mult(K, y, y, st);
    CtP p = ev_mult(K, z1.get(), z2.get(), st);
    CtP z3 = ev_mult_const(y, 1.5, p->level, st);
    return ev_add(z3.get(), p.get(), true, st);
}

}  // namespace

hs_status softmax_run(hs_ctx *c, const hs_keys *K, const hs_softmax_desc *d, const hs_ct *const *in,
                      size_t m_local, cudaStream_t st, hs_ct **out)
{
    const hs_params *P = c->P;
    const int N0 = P->n / 2;
    const int m = d->m, n = d->n, world = d->world < 1 ? 1 : d->world;
    if (m < 1 || n < 1 || n % m || d->k < 1 || !d->exp_poly || !d->inv_poly || d->variant < 0 || d->variant > 3 ||
        d->newton < 0 || (d->newton > 0 && d->variant != 0))
        throw HsError(HS_EINVAL, "softmax: bad descriptor");
    // Alg 1, square-and-normalize and cube-and-normalize share the schedule
    const bool alg1 = d->variant != 1;
    const int main_need = d->variant == 3 ? 3 : 2;  // levels of the main update
    if (m % world || (size_t)(m / world) != m_local) throw HsError(HS_EINVAL, "softmax: m_local != m / world");
    if (d->comm && comm_world(d->comm) != world)
        throw HsError(HS_EINVAL, "softmax: communicator size != world");
    if (world > 1 && !d->exchange && !d->comm)
        throw HsError(HS_EINVAL, "softmax: world > 1 needs a communicator or an exchange callback");
    const int nb = n / m;
    if ((nb & (nb - 1)) || nb > N0) throw HsError(HS_EINVAL, "softmax: n/m must be a power of two <= N0");
    const int stride = N0 / nb;
    const int ml = (int)m_local;
    for (int i = 0; i < ml; i++)
        if (!in[i] || in[i]->ncomp != 2 || in[i]->level != in[0]->level)
            throw HsError(HS_EINVAL, "softmax: inputs must be degree-1 ciphertexts at one level");
    std::vector<double> mask(N0, 0.0);
    for (int s = 0; s < stride; s++) mask[s] = 1.0;  // G10: coordinate block 0

    // the main thread keeps this rank's ml ciphertexts as ONE batch: every op
    // below runs once over all of them (same schedule as per ciphertext)
    if (in[0]->level < poly_cost(d->exp_poly)) level_error("input level too low for exp");
    CtP xb = ct_gather(in, ml, st);
    // y^(0) = exp(x / 2^k)
    CtP y0 = ev_cheb(K, xb.get(), d->exp_poly, st);
    xb.reset();
    CtP y = ct_copy(y0.get(), st);
    CtP lam;
    for (int j = 1; j <= d->k; j++) {
        const hs_poly *ip = &d->inv_poly[j - 1];
        // G12 (c): Alg 1 main thread needs 1 (aux square) + 2 levels
        if (alg1 && y->level < main_need) {
            if (!d->bts) level_error("main thread needs bootstrapping (not available)");
            std::vector<CtP> parts(ml);
            std::vector<const hs_ct *> ptrs(ml);
            for (int i = 0; i < ml; i++) {
                CtP one = ct_slice(y.get(), i, st);
                parts[i] = ev_bootstrap(K, d->bts, one.get(), 1.0, st);
                ptrs[i] = parts[i].get();
            }
            y = ct_gather(ptrs.data(), ml, st);
        }
        if (y->level < 1) level_error("main thread out of levels");
        // ---- auxiliary thread: S = relin(sum tensor(y, y)) -> rescale (C15)
        // G27: S = relin(sum_c tensor(w_c, y_c)) with w_c = y_c^2 (kept for the main update)
        CtP w = d->variant == 3 ? ev_mult(K, y.get(), y.get(), st) : CtP();
        CtP acc = w ? ev_tensor_sum2(w.get(), y.get(), st) : ev_tensor_sum(y.get(), st);
        if (world > 1 || d->comm) {
            const size_t words = acc->limbs() * P->n;
            DBuf gathered(words * world, st);
            if (d->comm) comm_all_gather(d->comm, acc->d, gathered.p, words, st);  // native NCCL
            else if (d->exchange(d->exchange_user, acc->d, gathered.p, words, st) != 0)
                throw HsError(HS_ENCCL, "softmax: exchange callback failed");
            // sum in rank order (exact modular addition)
            HS_CUDA(cudaMemcpyAsync(acc->d, gathered.p, words * 8, cudaMemcpyDeviceToDevice, st));
            for (int r = 1; r < world; r++)
                k_add(c, acc->d, gathered.p + r * words, acc->d, (int)acc->limbs(), acc->level + 1, false, st);
        }
        CtP S = ev_relin_rescale(K, acc.get(), st);  // C8: one division by P q_l
        acc.reset();
        rot_sum(K, S, nb, stride, -1, st);
        // main level (G12): Alg 1 -- y's level (the 2 levels of the
        // last update at j = k); version B -- the levels its update consumes,
        // j + 2 (k + 1 at j = k), capped by y0's
        const int need_b = j < d->k ? j + 2 : d->k + 1;
        const int main_a = j < d->k ? y->level : std::min(y->level, 2);
        const int main_level = alg1 ? main_a : std::min(y0->level, need_b);
        int need = poly_cost(ip) + 1 + ((d->variant == 1 && j > 1) ? 1 : 0);
        // G24: Newton steps after the last polynomial read x/2 (one level
        // below S), 2 levels each, then the mask: S supplies 2 t + 2 levels too
        const int nt = j == d->k ? d->newton : 0;
        if (nt > 0) need = std::max(need, 2 * nt + 2);
        // G12 (a): bootstrap before the inverse square root when the rest of the
        // aux thread would leave lambda below the main operand's level
        if (S->level - need < main_level) {
            if (d->bts) S = ev_bootstrap(K, d->bts, S.get(), ip->b, st);
            else if (S->level - need < 0) level_error("aux thread needs bootstrapping");
        }
        CtP lj = ev_cheb(K, S.get(), ip, st);
        if (nt > 0) {
            // G24 (n): bootstrap the seed when the Newton steps and the mask
            // would leave lambda below the main level
            int top = std::min(lj->level, S->level - 1);
            if (top - 2 * nt - 1 < main_level && d->bts) {
                lj = ev_bootstrap(K, d->bts, lj.get(), 1.1 / sqrt(ip->a), st);
                top = std::min(lj->level, S->level - 1);
            }
            if (top - 2 * nt - 1 < 0) level_error("Newton steps out of levels");
            CtP xh = ev_mult_const(S.get(), 0.5, S->level - 1, st);
            for (int t = 0; t < nt; t++) lj = newton_step(K, xh.get(), lj.get(), st);
        }
        S.reset();
        // Alg B line 5, taken BEFORE the mask: lambda_j holds its value in every
        // coordinate block (S was summed over all of them), so lambda * lambda_j
        // is the new lambda everywhere
        if (d->variant == 1 && j > 1) lj = ev_mult(K, lam.get(), lj.get(), st);
        // G12 (b): bootstrap lambda_j (version B: the product) BEFORE the mask
        // when the mask would leave it below the main level -- the broadcast
        // then gives every coordinate of an instance block 0's value, one
        // common bootstrapping error per instance (absorbed by the next
        // normalisation) instead of an independent one per slot
        if (lj->level - 1 < main_level && d->bts) {
            const double bound =
                d->variant >= 2 ? 1.1 / ip->a : (d->variant == 1 && j > 1) ? 1.5 : 1.1 / sqrt(ip->a);
            lj = ev_bootstrap(K, d->bts, lj.get(), bound, st);
        }
        if (lj->level < 1) level_error("no level for the mask");
        lj = ev_mult_pt(lj.get(), mask.data(), nullptr, lj->level - 1, st);
        rot_sum(K, lj, nb, stride, +1, st);
        lam = std::move(lj);
        // ---- main thread (lam broadcast against the batch)
        if (lam->level < 1) level_error("lambda out of levels");
        if (d->variant == 0) {
            CtP z = ev_mult(K, lam.get(), y.get(), st);
            // G12 (c'): bootstrap the normalised z (|z| <= 1 + alpha, larger
            // than y) when its square would leave y below the 2 levels the
            // next iteration needs
            if (d->bts && j < d->k && z->level - 1 < 2) {
                std::vector<CtP> parts(ml);
                std::vector<const hs_ct *> ptrs(ml);
                for (int i = 0; i < ml; i++) {
                    CtP one = ct_slice(z.get(), i, st);
                    parts[i] = ev_bootstrap(K, d->bts, one.get(), 1.1, st);
                    ptrs[i] = parts[i].get();
                }
                z = ct_gather(ptrs.data(), ml, st);
            }
            y = ev_mult(K, z.get(), z.get(), st);
        } else if (d->variant == 2) {
            CtP w2 = ev_mult(K, y.get(), y.get(), st);
            y = ev_mult(K, lam.get(), w2.get(), st);
        } else if (d->variant == 3) {
            CtP y3 = ev_mult(K, w.get(), y.get(), st);
            y = ev_mult(K, lam.get(), y3.get(), st);
        } else {
            CtP z = ev_mult(K, lam.get(), y0.get(), st);
            for (int s = 0; s < j; s++) {
                if (z->level < 1) level_error("version B squaring out of levels");
                z = ev_mult(K, z.get(), z.get(), st);
            }
            y = std::move(z);
        }
    }
    std::vector<CtP> res(ml);
    for (int i = 0; i < ml; i++) res[i] = ct_slice(y.get(), i, st);
    for (int i = 0; i < ml; i++) out[i] = res[i].release();
    return HS_OK;
}
