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

// C13 level-exact: a polynomial costs ceil(log2(d+1)) levels, its affine
// factor rides in the gains below (G28)
int poly_cost(const hs_poly *p) { return cheb_depth(p->deg); }

double affine_alpha(const hs_poly *p) { return 2.0 / (p->b - p->a); }

// x^(1/2^k): k square roots (each correctly rounded)
double root_pow2(double x, int k)
{
    for (int i = 0; i < k; i++) x = sqrt(x);
    return x;
}

// DESIGN.md G28.  Each polynomial reads alpha x (alpha = 2/(b-a)).  The main
// thread carries y'_j = gain[j] * y_j with gain[j]^e = alpha of the next
// iteration's polynomial (e = 2; 3 for the cube variant), so the aux sum is
// fed to the polynomial as alpha S; gain[0] is the exp polynomial's output
// gain, gain[k] = 1.  The mask of iteration j multiplies the true lambda_j by
// mask[j], producing the next main gain:
//   Alg 1  y_j = (mask_j lambda_j y'_{j-1})^2        mask_j = sqrt(g_j) / g_{j-1}
//   sq-n   y_j = mask_j lambda_j y'_{j-1}^2          mask_j = g_j / g_{j-1}^2
//   cube   y_j = mask_j lambda_j y'_{j-1}^3          mask_j = g_j / g_{j-1}^3
//   Alg B  lambda carries c_j = alpha_{j+1}^(2^-(j+1)) / g_0 (c_0 = 1,
//          c_k = 1 / g_0), mask_j = c_j / c_{j-1}
struct Gains {
    std::vector<double> g, mask, c;
    Gains(const hs_softmax_desc *d) : g(d->k + 1), mask(d->k + 1, 1.0), c(d->k + 1, 1.0)
    {
        const int k = d->k;
        for (int j = 0; j < k; j++) {
            const double a = affine_alpha(&d->inv_poly[j]);
            g[j] = d->variant == 3 ? cbrt(a) : sqrt(a);
        }
        g[k] = 1.0;
        for (int j = 1; j <= k; j++) {
            switch (d->variant) {
            case 1:
                c[j] = j < k ? root_pow2(affine_alpha(&d->inv_poly[j]), j + 1) / g[0] : 1.0 / g[0];
                mask[j] = c[j] / c[j - 1];
                break;
            case 0: mask[j] = sqrt(g[j]) / g[j - 1]; break;
            case 2: mask[j] = g[j] / (g[j - 1] * g[j - 1]); break;
            default: mask[j] = g[j] / (g[j - 1] * g[j - 1] * g[j - 1]); break;
            }
        }
    }
};

[[noreturn]] void level_error(const char *what) { throw HsError(HS_ELEVEL, std::string("softmax: ") + what); }

// ------------------------------------------------------------ executors
// The schedule below (softmax_body) is written ONCE against an executor E:
// RealEx runs every op on the device; SymEx only tracks levels, batch sizes
// and op counts (the planner).  Both take every decision
// from the same level arithmetic, so a plan's bootstrap placement is exactly
// the one the device run makes.

struct RealEx {
    typedef hs_ct T;
    typedef ::CtP Ct;
    hs_ctx *c;
    const hs_keys *K;
    const hs_softmax_desc *d;
    cudaStream_t st;
    bool has_bts() const { return d->bts != nullptr; }
    void check_exchange(int world) const
    {
        if (d->comm && comm_world(d->comm) != world)
            throw HsError(HS_EINVAL, "softmax: communicator size != world");
        if (world > 1 && !d->exchange && !d->comm)
            throw HsError(HS_EINVAL, "softmax: world > 1 needs a communicator or an exchange callback");
    }
    // digit-split the aux thread's key switches (d->aux_split)
    void aux_split(bool on)
    {
        if (!d->aux_split) return;
        if (on) {
            hs_ctx::KsSplit S;
            const int world = d->world < 1 ? 1 : d->world;
            if (world > 1) {
                S.rank = d->rank;
                S.world = world;
                S.comm = d->comm;
                S.ex = d->exchange;
                S.user = d->exchange_user;
            } else {
                S.emulate = d->aux_split >= 2 ? d->aux_split : 0;
            }
            c->ks_split = S;
            c->ks_split_on = world > 1 || S.emulate >= 2;
        } else {
            c->ks_split_on = false;
        }
    }
    Ct gather(const T *const *in, int n) { return ct_gather(in, n, st); }
    Ct copy(const T *x) { return ct_copy(x, st); }
    Ct cheb(const T *x, const hs_poly *p, double gain) { return ev_cheb(K, x, p, gain, st); }
    Ct mult(const T *a, const T *b) { return ev_mult(K, a, b, st); }
    Ct mult_const(const T *a, double v, int target) { return ev_mult_const(a, v, target, st); }
    Ct mult_pt(const T *a, const double *re, int target) { return ev_mult_pt(a, re, nullptr, target, st); }
    Ct add(const T *a, const T *b, bool sub) { return ev_add(a, b, sub, st); }
    Ct rotate(const T *a, int r) { return ev_rotate(K, a, r, st); }
    Ct tensor_sum(const T *y) { return ev_tensor_sum(y, st); }
    Ct tensor_sum2(const T *w, const T *y) { return ev_tensor_sum2(w, y, st); }
    Ct relin_rescale(const T *a) { return ev_relin_rescale(K, a, st); }
    Ct bootstrap(const T *a, double bound) { return ev_bootstrap(K, d->bts, a, bound, st); }
    // every member of a batch bootstrapped on its own, then re-batched
    Ct bootstrap_each(const T *y, double bound)
    {
        const int b = y->batch;
        std::vector<Ct> parts(b);
        std::vector<const hs_ct *> ptrs(b);
        for (int i = 0; i < b; i++) {
            Ct one = ct_slice(y, i, st);
            parts[i] = ev_bootstrap(K, d->bts, one.get(), bound, st);
            ptrs[i] = parts[i].get();
        }
        return ct_gather(ptrs.data(), b, st);
    }
    // hs_ctx_debug_domain: decrypt the aux sum (it holds alpha S, G28) and
    // check every slot against the polynomial's interval
    void domain_check(const T *S, const hs_poly *p)
    {
        if (!c->debug_keys) return;
        const hs_params *P = c->P;
        const size_t N = P->n;
        std::vector<u64> m((size_t)(S->level + 1) * N);
        CtP one = ct_slice(S, 0, st);
        ev_decrypt(c->debug_keys, one.get(), m.data(), st);
        std::vector<double> re(N / 2), im(N / 2);
        hs_decode_impl(P, m.data(), P->scale[S->level], re.data(), im.data());
        const double alpha = 2.0 / (p->b - p->a), tol = (p->b - p->a) / 64.0;
        for (size_t j = 0; j < N / 2; j++) {
            const double v = re[j] / alpha;
            if (!(v >= p->a - tol && v <= p->b + tol))
                throw HsError(HS_EDOMAIN, "softmax: aux sum outside the polynomial interval (input outside [-M, 0]?)");
        }
    }
    // all-gather of the partial aux sums, added in rank order (exact)
    void exchange(T *acc, int world)
    {
        const size_t words = acc->limbs() * c->P->n;
        DBuf gathered(words * world, st);
        if (d->comm) comm_all_gather(d->comm, acc->d, gathered.p, words, st);  // native NCCL
        else if (d->exchange(d->exchange_user, acc->d, gathered.p, words, st) != 0)
            throw HsError(HS_ENCCL, "softmax: exchange callback failed");
        HS_CUDA(cudaMemcpyAsync(acc->d, gathered.p, words * 8, cudaMemcpyDeviceToDevice, st));
        for (int r = 1; r < world; r++)
            k_add(c, acc->d, gathered.p + r * words, acc->d, (int)acc->limbs(), acc->level + 1, false, st);
    }
};

// A ciphertext of the planner: level, components, batch members.
struct SymCt {
    int level, ncomp, batch;
};

// Level semantics of every op (C8, C9, C11, C12; poly.cpp eval_unit; bts.cpp
// out_level) plus a cost model in units of ONE HMult+relin+rescale of one
// ciphertext at level 12.
struct SymEx {
    typedef SymCt T;
    typedef std::unique_ptr<SymCt> Ct;
    const hs_params *P;
    int bts_out;  // < 0: no bootstrapping
    hs_softmax_sched *s;
    bool has_bts() const { return bts_out >= 0; }
    void check_exchange(int) const {}
    static Ct mk(int level, int ncomp, int batch) { return Ct(new SymCt{level, ncomp, batch}); }
    // limb-NTTs of one key switch at level l (ModUp iNTT + NTT, ModDown iNTT + NTT)
    double ks_work(int l) const
    {
        const int a = P->alpha, nl = l + 1, beta = (nl + a - 1) / a;
        return (double)beta * (nl + a) + 2.0 * a + 2.0 * nl;
    }
    // batched ops amortise keys and launches: 64 members cost ~40 (measured
    // HMult ops/s at batch 64 vs 1, profiles/r01_bench_full.json)
    static double beff(int b) { return b / (1.0 + 0.1 * log2((double)b)); }
    double ks_cost(int l, int b) const { return ks_work(l) / ks_work(12) * beff(b); }
    Ct gather(const T *const *in, int n) { return mk(in[0]->level, in[0]->ncomp, n); }
    Ct copy(const T *x) { return mk(x->level, x->ncomp, x->batch); }
    Ct cheb(const T *x, const hs_poly *p, double)
    {
        const int cost = poly_cost(p);
        if (x->level < cost) throw HsError(HS_ELEVEL, "polynomial deeper than the remaining levels");
        // ~2 sqrt(d+1) + log2(d+1) non-scalar products (PAPER.md 330-336) at the mid level
        const double mults = 2.0 * sqrt(p->deg + 1.0) + log2(p->deg + 1.0);
        s->poly_evals += 1;
        s->cost += mults * ks_cost(x->level - cost / 2, x->batch);
        return mk(x->level - cost, 2, x->batch);
    }
    Ct mult(const T *a, const T *b)
    {
        const int l = std::min(a->level, b->level);
        if (l < 1) throw HsError(HS_ELEVEL, "no level left for a product");
        const int bt = std::max(a->batch, b->batch);
        s->hmult += bt;
        s->cost += ks_cost(l, bt);
        return mk(l - 1, 2, bt);
    }
    Ct mult_const(const T *a, double, int target) { return mk(target, a->ncomp, a->batch); }
    Ct mult_pt(const T *a, const double *, int target) { return mk(target, a->ncomp, a->batch); }
    Ct add(const T *a, const T *b, bool) { return mk(std::min(a->level, b->level), a->ncomp, std::max(a->batch, b->batch)); }
    Ct rotate(const T *a, int)
    {
        s->rotations += a->batch;
        s->cost += ks_cost(a->level, a->batch);
        return mk(a->level, a->ncomp, a->batch);
    }
    Ct tensor_sum(const T *y) { return mk(y->level, 3, 1); }
    Ct tensor_sum2(const T *w, const T *y) { return mk(std::min(w->level, y->level), 3, 1); }
    Ct relin_rescale(const T *a)
    {
        s->cost += ks_cost(a->level, 1);
        return mk(a->level - 1, 2, 1);
    }
    Ct bootstrap(const T *a, double)
    {
        s->bts_aux += a->batch;
        s->cost += HS_SCHED_BTS_COST * a->batch;
        return mk(bts_out, 2, a->batch);
    }
    Ct bootstrap_each(const T *y, double)
    {
        s->bts_main += y->batch;
        s->cost += HS_SCHED_BTS_COST * y->batch;
        return mk(bts_out, 2, y->batch);
    }
    void exchange(T *, int) { s->exchanges += 1; }
    void domain_check(const T *, const hs_poly *) {}
    void aux_split(bool) {}
};

// RAII: the aux thread's digit split is on between construction and end()
// (or the scope's exit, also on an exception)
template <class E>
struct AuxScope {
    E &ex;
    bool on;
    explicit AuxScope(E &e) : ex(e), on(true) { ex.aux_split(true); }
    void end()
    {
        if (on) ex.aux_split(false);
        on = false;
    }
    ~AuxScope() { end(); }
};

template <class E>
void rot_sum(E &ex, typename E::Ct &S, int nb, int stride, int sign)
{
    for (int i = 0; (1 << i) < nb; i++) {
        typename E::Ct r = ex.rotate(S.get(), sign * stride * (1 << i));
        S = ex.add(S.get(), r.get(), false);
    }
}

// PAPER.md 1313-1316: z1 = (x/2) y; z2 = y y; z3 = (3/2) y; y' = z3 - z1 z2
// (2 levels; z3 multiplied straight to the level of z1 z2, C12)
template <class E>
typename E::Ct newton_step(E &ex, const typename E::T *xh, const typename E::T *y)
{
    typename E::Ct z1 = ex.mult(xh, y);
    typename E::Ct z2 = ex.mult(y, y);
    typename E::Ct p = ex.mult(z1.get(), z2.get());
    typename E::Ct z3 = ex.mult_const(y, 1.5, p->level);
    return ex.add(z3.get(), p.get(), true);
}

template <class E>
typename E::Ct softmax_body(E &ex, const hs_params *P, const hs_softmax_desc *d, const typename E::T *const *in,
                            size_t m_local)
{
    typedef typename E::Ct CtP;
    const int N0 = P->n / 2;
    const int m = d->m, n = d->n, world = d->world < 1 ? 1 : d->world;
    if (m < 1 || n < 1 || n % m || d->k < 1 || !d->exp_poly || !d->inv_poly || d->variant < 0 || d->variant > 3 ||
        d->newton < 0 || (d->newton > 0 && d->variant != 0))
        throw HsError(HS_EINVAL, "softmax: bad descriptor");
    // Alg 1, square-and-normalize and cube-and-normalize share the schedule
    const bool alg1 = d->variant != 1;
    const int main_need = d->variant == 3 ? 3 : 2;  // levels of the main update
    if (m % world || (size_t)(m / world) != m_local) throw HsError(HS_EINVAL, "softmax: m_local != m / world");
    if (d->aux_split < 0 || (d->aux_split == 1 && world == 1) || (d->aux_split >= 2 && world > 1) ||
        d->aux_split > 64)
        throw HsError(HS_EINVAL, "softmax: aux_split must be 0, 1 (world > 1) or an emulated rank count >= 2");
    ex.check_exchange(world);
    const int nb = n / m;
    if ((nb & (nb - 1)) || nb > N0) throw HsError(HS_EINVAL, "softmax: n/m must be a power of two <= N0");
    const int stride = N0 / nb;
    const int ml = (int)m_local;
    for (int i = 0; i < ml; i++)
        if (!in[i] || in[i]->ncomp != 2 || in[i]->level != in[0]->level)
            throw HsError(HS_EINVAL, "softmax: inputs must be degree-1 ciphertexts at one level");
    std::vector<double> mask(N0, 0.0);  // G10: coordinate block 0, value G28's mask_j
    const Gains gn(d);

    // the main thread keeps this rank's ml ciphertexts as ONE batch: every op
    // below runs once over all of them (same schedule as per ciphertext)
    if (in[0]->level < poly_cost(d->exp_poly)) level_error("input level too low for exp");
    CtP xb = ex.gather(in, ml);
    // y^(0) = exp(x / 2^k): x arrives as alpha_exp x, y0 leaves with gain g_0 (G28)
    CtP y0 = ex.cheb(xb.get(), d->exp_poly, gn.g[0]);
    xb.reset();
    CtP y = ex.copy(y0.get());
    CtP lam;
    for (int j = 1; j <= d->k; j++) {
        const hs_poly *ip = &d->inv_poly[j - 1];
        // G12 (c): Alg 1 main thread needs 1 (aux square) + 2 levels
        if (alg1 && y->level < main_need) {
            if (!ex.has_bts()) level_error("main thread needs bootstrapping (not available)");
            y = ex.bootstrap_each(y.get(), 1.0 * gn.g[j - 1]);
        }
        if (y->level < 1) level_error("main thread out of levels");
        // ---- auxiliary thread: S = relin(sum tensor(y, y)) -> rescale (C15)
        // G27: S = relin(sum_c tensor(w_c, y_c)) with w_c = y_c^2 (kept for the main update)
        CtP w = d->variant == 3 ? ex.mult(y.get(), y.get()) : CtP();
        CtP acc = w ? ex.tensor_sum2(w.get(), y.get()) : ex.tensor_sum(y.get());
        if (world > 1 || d->comm) ex.exchange(acc.get(), world);
        // the aux thread proper: its key switches may be digit-split (d->aux_split)
        AuxScope<E> aux_scope(ex);
        CtP S = ex.relin_rescale(acc.get());  // C8: one division by P q_l
        acc.reset();
        rot_sum(ex, S, nb, stride, -1);
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
            if (ex.has_bts()) S = ex.bootstrap(S.get(), affine_alpha(ip) * ip->b);
            else if (S->level - need < 0) level_error("aux thread needs bootstrapping");
        }
        ex.domain_check(S.get(), ip);
        CtP lj = ex.cheb(S.get(), ip, 1.0);  // S holds alpha_j S (G28)
        if (nt > 0) {
            // G24 (n): bootstrap the seed when the Newton steps and the mask
            // would leave lambda below the main level
            int top = std::min(lj->level, S->level - 1);
            if (top - 2 * nt - 1 < main_level && ex.has_bts()) {
                lj = ex.bootstrap(lj.get(), 1.1 / sqrt(ip->a));
                top = std::min(lj->level, S->level - 1);
            }
            if (top - 2 * nt - 1 < 0) level_error("Newton steps out of levels");
            CtP xh = ex.mult_const(S.get(), 0.5 / affine_alpha(ip), S->level - 1);  // x/2 from alpha x
            for (int t = 0; t < nt; t++) lj = newton_step(ex, xh.get(), lj.get());
        }
        S.reset();
        // Alg B line 5, taken BEFORE the mask: lambda_j holds its value in every
        // coordinate block (S was summed over all of them), so lambda * lambda_j
        // is the new lambda everywhere
        if (d->variant == 1 && j > 1) lj = ex.mult(lam.get(), lj.get());
        // G12 (b): bootstrap lambda_j (version B: the product) BEFORE the mask
        // when the mask would leave it below the main level -- the broadcast
        // then gives every coordinate of an instance block 0's value, one
        // common bootstrapping error per instance (absorbed by the next
        // normalisation) instead of an independent one per slot
        if (lj->level - 1 < main_level && ex.has_bts()) {
            const double bound =
                d->variant >= 2 ? 1.1 / ip->a : (d->variant == 1 && j > 1) ? 1.5 * gn.c[j - 1] : 1.1 / sqrt(ip->a);
            lj = ex.bootstrap(lj.get(), bound);
        }
        if (lj->level < 1) level_error("no level for the mask");
        for (int s = 0; s < stride; s++) mask[s] = gn.mask[j];
        lj = ex.mult_pt(lj.get(), mask.data(), lj->level - 1);
        rot_sum(ex, lj, nb, stride, +1);
        lam = std::move(lj);
        aux_scope.end();
        // ---- main thread (lam broadcast against the batch)
        if (lam->level < 1) level_error("lambda out of levels");
        if (d->variant == 0) {
            CtP z = ex.mult(lam.get(), y.get());
            // G12 (c'): bootstrap the normalised z (|z| <= 1 + alpha, larger
            // than y) when its square would leave y below the 2 levels the
            // next iteration needs
            if (ex.has_bts() && j < d->k && z->level - 1 < 2) {
                z = ex.bootstrap_each(z.get(), 1.1 * sqrt(gn.g[j]));
            }
            y = ex.mult(z.get(), z.get());
        } else if (d->variant == 2) {
            CtP w2 = ex.mult(y.get(), y.get());
            y = ex.mult(lam.get(), w2.get());
        } else if (d->variant == 3) {
            CtP y3 = ex.mult(w.get(), y.get());
            y = ex.mult(lam.get(), y3.get());
        } else {
            CtP z = ex.mult(lam.get(), y0.get());
            for (int s = 0; s < j; s++) {
                if (z->level < 1) level_error("version B squaring out of levels");
                z = ex.mult(z.get(), z.get());
            }
            y = std::move(z);
        }
    }
    return y;
}

}  // namespace

hs_status softmax_run(hs_ctx *c, const hs_keys *K, const hs_softmax_desc *d, const hs_ct *const *in,
                      size_t m_local, cudaStream_t st, hs_ct **out)
{
    // the G28 input contract: an input declared at another scale than the
    // Softmax reads is rejected (C11)
    if (d && d->exp_poly && d->exp_poly->b > d->exp_poly->a)
        for (size_t i = 0; i < m_local; i++) {
            if (!in[i] || in[i]->scale == 0.0) continue;
            const double want = c->P->scale[in[i]->level] * (2.0 / (d->exp_poly->b - d->exp_poly->a));
            if (fabs(in[i]->scale / want - 1.0) > ldexp(1.0, -40))
                throw HsError(HS_ESCALE, "softmax: input not encoded at hs_softmax_input_scale (G28)");
        }
    RealEx ex{c, K, d, st};
    CtP y = softmax_body(ex, c->P, d, in, m_local);
    const int ml = (int)m_local;
    std::vector<CtP> res(ml);
    for (int i = 0; i < ml; i++) res[i] = ct_slice(y.get(), i, st);
    for (int i = 0; i < ml; i++) out[i] = res[i].release();
    return HS_OK;
}

void softmax_schedule(const hs_params *P, const hs_softmax_desc *d, int in_level, size_t m_local, int bts_out_level,
                      hs_softmax_sched *s)
{
    *s = hs_softmax_sched{};
    if (m_local < 1 || in_level < 0 || in_level > P->L) throw HsError(HS_EINVAL, "schedule: bad input level / m_local");
    if (bts_out_level > P->L) throw HsError(HS_EINVAL, "schedule: bootstrap output level above the chain");
    SymEx ex{P, bts_out_level, s};
    std::vector<SymCt> cts(m_local, SymCt{in_level, 2, 1});
    std::vector<const SymCt *> ptrs(m_local);
    for (size_t i = 0; i < m_local; i++) ptrs[i] = &cts[i];
    SymEx::Ct y = softmax_body(ex, P, d, ptrs.data(), m_local);
    s->out_level = y->level;
}
