// poly.cpp -- Chebyshev-series evaluation on ciphertexts (C13).
//
// PAPER.md 330-336 (sec 2.2.4): a degree-d polynomial costs ceil(log(d+1))
// levels and O(sqrt d) ct-ct products; PAPER.md 424-425: degrees 2^t - 1 for a
// budget of t levels.  The exact tree (shared with the oracle as a written
// convention, not as code; C13, round 2 level-exact form):
//   the input W holds alpha x (alpha = 2/(b-a)); T_1 = u = W + beta,
//   beta = -(a+b)/(b-a), a constant add (G28);
//   coefficients scaled by the caller's gain first: c_i <- g c_i;
//   t = ceil(log2(d+1)); baby size B = 2^ceil(t/2) (B = 2 when d <= 1);
//   T_i = 2 T_a T_b - T_{a-b} (a = 2^(ceil(log2 i)-1), b = i-a; a == b:
//   2 T_a^2 - 1); giants G_j = T_{B 2^j} by doubling;
//   rec(p, target): LEAF when deg < B and every T_1..T_deg lies at level >=
//     target+1; else split at g = 2^(ceil(log2(deg+1))-1):
//     q_0 = c_g, q_k = 2 c_{g+k};  r_j = c_j, r_{g-k} = c_{g-k} - c_{g+k};
//     out = rec(q, target+1) * T_g + rec(r, target)  (T_g a baby when g < B)
//   leaf: rescale(sum_i rint(c_i sc_i) T_i|target+1) + c_0   (one rescale)
//   target = level(W) - t: exactly ceil(log2(d+1)) levels (1 for d <= 1).
#include <map>
#include <vector>

#include "hs_internal.h"

static int clog2(int x)
{
    int t = 0;
    while ((1 << t) < x) t++;
    return t;
}

int cheb_depth(int deg) { return deg <= 1 ? 1 : clog2(deg + 1); }

namespace {

struct Basis {
    const hs_keys *K;
    cudaStream_t st;
    int B;
    std::vector<CtP> T;  // T[0] unused
    std::vector<CtP> G;
    // level-downs already made (a basis ciphertext is lowered to the same
    // level by several products / subtractions; the same op, done once)
    std::map<std::pair<const hs_ct *, int>, CtP> low;
    const hs_ct *at(const hs_ct *x, int level)
    {
        if (x->level == level) return x;
        auto key = std::make_pair(x, level);
        auto it = low.find(key);
        if (it != low.end()) return it->second.get();
        return (low[key] = ev_level_down(x, level, st)).get();
    }
};

CtP dbl_minus_one(const hs_keys *K, const hs_ct *x, cudaStream_t st)
{
    CtP s = ev_mult(K, x, x, st);
    CtP s2 = ev_mult_int(s.get(), 2, st);
    return ev_add_const(s2.get(), -1.0, st);
}

CtP leaf(Basis &E, const std::vector<double> &c, int target)
{
    std::vector<const hs_ct *> terms;
    std::vector<double> coef;
    for (size_t i = 1; i < c.size(); i++) {
        terms.push_back(E.T[i].get());
        coef.push_back(c[i]);
    }
    if (terms.empty()) {
        terms.push_back(E.T[1].get());
        coef.push_back(0.0);
    }
    CtP s = ev_mult_const_sum(terms, coef, target, E.st);
    return ev_add_const(s.get(), c[0], E.st);
}

// a leaf reads T_1..T_d (T_1 for a constant) one level above its target
bool leaf_ok(const Basis &E, int d, int target)
{
    if (d >= E.B) return false;
    for (int i = 1; i <= std::max(d, 1); i++)
        if (E.T[i]->level < target + 1) return false;
    return true;
}

CtP rec(Basis &E, const std::vector<double> &c, int target)
{
    const int d = (int)c.size() - 1;
    if (leaf_ok(E, d, target)) return leaf(E, c, target);
    const int g = 1 << (clog2(d + 1) - 1);
    std::vector<double> q(d - g + 1), r(c.begin(), c.begin() + g);
    q[0] = c[g];
    for (int k = 1; k <= d - g; k++) {
        q[k] = 2.0 * c[g + k];
        r[g - k] = c[g - k] - c[g + k];
    }
    CtP Q = rec(E, q, target + 1);
    const hs_ct *Gj = g < E.B ? E.T[g].get() : E.G[clog2(g / E.B)].get();
    CtP QT = ev_mult(E.K, Q.get(), Gj->level > Q->level ? E.at(Gj, Q->level) : Gj, E.st);
    CtP R = rec(E, r, target);
    return ev_add(QT.get(), R.get(), false, E.st);
}

CtP eval_unit(const hs_keys *K, const hs_ct *u, const hs_poly *p, double gain, cudaStream_t st)
{
    const int d = p->deg;
    Basis E{K, st, 0, {}, {}};
    const int t = clog2(d + 1);
    E.B = d <= 1 ? 2 : 1 << ((t + 1) / 2);
    const int ng = std::max(0, t - clog2(E.B));
    // baby steps in waves: wave a computes T_{a+1} .. T_{2a} (plus T_B = G_0
    // when giants are needed), all products T_a T_b at T_a's level, as ONE
    // batched HMult (the same words as one product at a time)
    const int top = ng > 0 ? E.B : E.B - 1;
    E.T.resize(top + 1);
    E.T[1] = ct_copy(u, st);
    // (an input that is itself a batch -- the main thread's m ciphertexts --
    // runs the members of a wave one after the other)
    const int per = u->batch == 1 ? E.B : 1;
    for (int a = 1; a < top; a *= 2) {
        const int i1 = std::min(2 * a, top);
        for (int i0 = a + 1; i0 <= i1; i0 += per) {
            const int i2 = std::min(i1, i0 + per - 1);
            std::vector<const hs_ct *> ops;
            for (int i = i0; i <= i2; i++) {
                const hs_ct *tb = E.T[i - a].get();
                if (tb->level > E.T[a]->level) tb = E.at(tb, E.T[a]->level);
                ops.push_back(tb);
            }
            CtP bb = ops.size() == 1 ? CtP() : ct_gather(ops.data(), (int)ops.size(), st);
            CtP m = ev_mult(K, E.T[a].get(), bb ? bb.get() : ops[0], st);
            CtP m2 = ev_mult_int(m.get(), 2, st);
            for (int i = i0; i <= i2; i++) {
                CtP v = ops.size() == 1 ? std::move(m2) : ct_view(m2.get(), i - i0);
                const int b = i - a;
                E.T[i] = a == b ? ev_add_const(v.get(), -1.0, st)
                                : ev_add(v.get(), E.at(E.T[a - b].get(), v->level), true, st);
            }
        }
    }
    if (ng > 0) {
        E.G.push_back(std::move(E.T[E.B]));
        E.T.resize(E.B);
    }
    for (int j = 1; j < ng; j++) E.G.push_back(dbl_minus_one(K, E.G[j - 1].get(), st));
    const int target = u->level - cheb_depth(d);
    if (target < 0) throw HsError(HS_ELEVEL, "polynomial deeper than the remaining levels");
    std::vector<double> c(p->coeffs, p->coeffs + d + 1);
    for (double &v : c) v *= gain;
    return rec(E, c, target);
}

}  // namespace

CtP ev_cheb(const hs_keys *K, const hs_ct *w, const hs_poly *p, double gain, cudaStream_t st)
{
    if (!p || p->deg < 1 || !p->coeffs || !(p->b > p->a)) throw HsError(HS_EINVAL, "bad polynomial");
    if (p->a == -1.0 && p->b == 1.0) return eval_unit(K, w, p, gain, st);
    // G28: w already holds alpha x; the shift is a constant add (no level)
    const double beta = -(p->a + p->b) / (p->b - p->a);
    CtP u = ev_add_const(w, beta, st);
    return eval_unit(K, u.get(), p, gain, st);
}
