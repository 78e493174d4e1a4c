// bts.cpp -- real-slot CKKS bootstrapping on the GPU (reading G11).
//
// PAPER.md 281-283 / 429-440 need bootstrapping but give no internals (the
// paper calls HEaaN's FGb BTS, PAPER.md 386-393).  Conventions shared with
// the oracle only in writing:
//   e = clamp(floor(log2 q0 - cap - log2 Delta_0 - log2 bound), 0, 30), cap = 8
//       with the arcsine step else 12;  x *= 2^e
//   drop to level 0; ModRaise (centred lift of the q0 residues) to level L
//   CoeffToSlot: inverse special-FFT stages in n_cts groups (largest stages
//                first), the first transform scaled by (Delta_L / q0) / (2 (K+2))
//   v = w + conj(w) - 1/(4 (K+2)); EvalMod = cos series on [-1,1], r x (2c^2-1);
//   arcsine step s <- s + (1/6) s^3 (s6 = mult_const(s, 1/6), t = s*s, s + s6*t)
//   SlotToCoeff: special-FFT stages in n_stc groups, the first composed with
//                diag(lambda, 2 lambda, ..., 2 lambda), lambda = q0/(4 pi Delta_out 2^e)
//   out = x + conj(x)
// Each transform: diagonals d (mod N0, structural presence), step unit u =
// 2^(first stage index of the group), baby size b1 = 2^min(r, 4),
// idx = d/u, giant g = idx / b1, baby b = idx % b1;
//   out = rescale( sum_g Rot( sum_b pt_{g,b} (.) Rot(ct, b u), g b1 u ) ),
// pt_{g,b} = encode(rot(diag_d, -g b1 u)) at the landing scale of the level.
#include <math.h>
#include <omp.h>
#include <quadmath.h>

#include <algorithm>
#include <map>
#include <vector>

#include "hs_internal.h"

typedef __float128 f128;

namespace {

struct Qc {
    f128 re = 0, im = 0;
};
inline Qc operator*(Qc a, Qc b) { return Qc{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }

// sparse N0 x N0 matrix by diagonals: D[d][p] = A[p][(p+d) mod N0]
struct DiagMat {
    int n0;
    std::vector<std::vector<Qc>> D;
    explicit DiagMat(int n) : n0(n), D(n) {}
    void add(int d, int p, Qc v)
    {
        d = ((d % n0) + n0) % n0;
        if (D[d].empty()) D[d].assign(n0, Qc{});
        D[d][p].re += v.re;
        D[d][p].im += v.im;
    }
};

DiagMat fft_stage(int log_n, int len, bool inverse)
{
    const int N = 1 << log_n, n0 = N / 2, h = len / 2, q4 = 4 * len;
    DiagMat m(n0);
    u64 g = 1;
    for (int j = 0; j < h; j++, g = g * 5 % (2ull * N)) {
        f128 ang = 2 * M_PIq * (f128)((g % q4) * (u64)(2 * N / q4)) / (f128)(2 * N);
        Qc xi{cosq(ang), sinq(ang)};
        f128 den = xi.re * xi.re + xi.im * xi.im;
        Qc hinv{0.5q * xi.re / den, -0.5q * xi.im / den};  // 1/(2 xi)
        for (int i = 0; i < n0; i += len) {
            const int p = i + j;
            if (!inverse) {
                m.add(0, p, Qc{1, 0});
                m.add(h, p, xi);
                m.add(-h, p + h, Qc{1, 0});
                m.add(0, p + h, Qc{-xi.re, -xi.im});
            } else {
                m.add(0, p, Qc{0.5q, 0});
                m.add(h, p, Qc{0.5q, 0});
                m.add(-h, p + h, hinv);
                m.add(0, p + h, Qc{-hinv.re, -hinv.im});
            }
        }
    }
    return m;
}

DiagMat matmul(const DiagMat &A, const DiagMat &B)
{
    const int n0 = A.n0;
    DiagMat C(n0);
    for (int e = 0; e < n0; e++) {
        if (A.D[e].empty()) continue;
        for (int f = 0; f < n0; f++) {
            if (B.D[f].empty()) continue;
            const int d = (e + f) % n0;
            for (int p = 0; p < n0; p++) C.add(d, p, A.D[e][p] * B.D[f][(p + e) % n0]);
        }
    }
    return C;
}

void scale_columns(DiagMat &m, const std::vector<f128> &s)
{
    for (int d = 0; d < m.n0; d++)
        if (!m.D[d].empty())
            for (int p = 0; p < m.n0; p++) {
                f128 f = s[(p + d) % m.n0];
                m.D[d][p].re *= f;
                m.D[d][p].im *= f;
            }
}

std::vector<int> group_sizes(int s, int g)
{
    std::vector<int> sz;
    int rem = s;
    for (int k = g; k >= 1; k--) {
        sz.push_back((rem + k - 1) / k);
        rem -= sz.back();
    }
    return sz;
}

int ilog2(int x)
{
    int t = 0;
    while ((1 << t) < x) t++;
    return t;
}

// product of the stages [first, first+size): forward in stage order, inverse
// largest stage first
DiagMat group_matrix(int log_n, int first, int size, bool inverse)
{
    DiagMat acc(1 << (log_n - 1));
    for (int t = 0; t < size; t++) {
        const int i = inverse ? first + size - 1 - t : first + t;
        DiagMat S = fft_stage(log_n, 2 << i, inverse);
        acc = t ? matmul(S, acc) : S;
    }
    return acc;
}

struct LinTrans {
    int level = 0, unit = 1, b1 = 1;
    std::vector<int> g, b;
    u64 *pts = nullptr;  // [terms][level+1][N] NTT-domain plaintexts
    LinTrans() {}
    LinTrans(const LinTrans &) = delete;
    ~LinTrans() { dev_free_persist(pts); }
};

// C17: plaintexts in the extended basis Q_level u P ([terms][ntg][N], NTT
// domain, Montgomery form) for the double-hoisted BSGS
void build_lintrans(hs_ctx *c, const DiagMat &m, int level, int unit, int r, LinTrans &T)
{
    const hs_params *P = c->P;
    const int n0 = P->n / 2, N = P->n, nl = level + 1, ntg = nl + P->n_p;
    T.level = level;
    T.unit = unit;
    T.b1 = 1 << std::min(r, 4);  // baby size 2^min(r, 4) (G11)
    std::vector<int> ds;
    for (int d = 0; d < n0; d++)
        if (!m.D[d].empty()) {
            ds.push_back(d);
            T.g.push_back((d / unit) / T.b1);
            T.b.push_back((d / unit) % T.b1);
        }
    const int nt = (int)ds.size();
    const double sc = (P->scale[level - 1] * (double)P->prime[level]) / P->scale[level];
    std::vector<u64> host((size_t)nt * ntg * N);
#pragma omp parallel for schedule(dynamic)
    for (int k = 0; k < nt; k++) {
        const int G = (T.g[k] * T.b1 * unit) % n0;
        std::vector<f128> re(n0), im(n0);
        const std::vector<Qc> &v = m.D[ds[k]];
        for (int p = 0; p < n0; p++) {
            const Qc &x = v[((p - G) % n0 + n0) % n0];
            re[p] = x.re;
            im[p] = x.im;
        }
        hs_encode_impl_q(P, re.data(), im.data(), sc, level, host.data() + (size_t)k * ntg * N, true);
    }
    T.pts = (decltype(T.pts))dev_alloc_persist(host.size() * 8);
    HS_CUDA(cudaMemcpy(T.pts, host.data(), host.size() * 8, cudaMemcpyHostToDevice));
    PrimeMap pm;
    pm.n = ntg;
    for (int i = 0; i < ntg; i++) pm.p[i] = (unsigned char)(i < nl ? i : P->n_q + (i - nl));
    k_ntt(c, T.pts, nt * ntg, pm, false, nullptr);
    // Montgomery form pt 2^64 mod p: the fused BSGS kernel sums 128-bit
    // products and lands with one REDC
    u64 r64[HS_MAXP];
    for (int i = 0; i < ntg; i++) r64[i] = P->pk[pm.p[i]].r64;
    k_mul_scalar_pm(c, T.pts, T.pts, r64, nt * ntg, pm, nullptr);
    HS_CUDA(cudaDeviceSynchronize());
}

void add_group_rotations(int n0, int ngroups, std::vector<int> &rots)
{
    std::vector<int> sz = group_sizes(ilog2(n0), ngroups);
    int first = 0;
    for (int gi = 0; gi < ngroups; gi++) {
        const int u = 1 << first, r = sz[gi], b1 = 1 << std::min(r, 4), span = (1 << r) - 1, mod = n0 / u;
        for (int idx = -span; idx <= span; idx++) {
            int id = ((idx % mod) + mod) % mod;
            for (int rr : {(id % b1) * u, (id / b1) * b1 * u}) {
                rr %= n0;
                if (rr && std::find(rots.begin(), rots.end(), rr) == rots.end()) rots.push_back(rr);
            }
        }
        first += r;
    }
}

}  // namespace

struct hs_bts {
    hs_ctx *ctx = nullptr;
    int K = 0, r = 0, out_level = 0, n_cts = 0, n_stc = 0, arcsine = 0;
    std::vector<double> cos_coeffs, half_coeffs;
    hs_poly cos_poly{}, half_poly{};
    bool even = false;  // C18: odd coefficients all 0 -> evaluate on T_2(x)
    std::vector<std::unique_ptr<LinTrans>> cts;                   // shared by every e
    std::map<int, std::vector<std::unique_ptr<LinTrans>>> stc;    // per pre-scaling exponent e
    std::mutex mu;
};

int bts_exponent(const hs_params *P, int arcsine, double bound)
{
    double cap = arcsine ? 8.0 : 12.0;
    // dev diagnostic: HS_BTS_CAP overrides the headroom (the oracle keeps 8 / 12)
    if (const char *v = getenv("HS_BTS_CAP")) cap = atof(v);
    double e = floor(log2((double)P->prime[0]) - cap - log2(P->scale[0]) - log2(bound));
    return (int)std::min(30.0, std::max(0.0, e));
}

int bts_rotations(const hs_params *P, int n_cts, int n_stc, int32_t *out, int max)
{
    std::vector<int> rots;
    add_group_rotations(P->n / 2, n_stc, rots);
    add_group_rotations(P->n / 2, n_cts, rots);
    int cnt = 0;
    for (int v : rots) {
        if (out && cnt < max) out[cnt] = v;
        cnt++;
    }
    return cnt;
}

static void ensure_cts(hs_bts *B)
{
    if (!B->cts.empty()) return;
    hs_ctx *c = B->ctx;
    const hs_params *P = c->P;
    const int n0 = P->n / 2, L = P->L;
    std::vector<int> sz = group_sizes(ilog2(n0), B->n_cts), first(B->n_cts);
    for (int gi = 0, st = 0; gi < B->n_cts; st += sz[gi], gi++) first[gi] = st;
    for (int k = 0; k < B->n_cts; k++) {
        const int gi = B->n_cts - 1 - k;
        DiagMat m = group_matrix(P->log_n, first[gi], sz[gi], true);
        if (k == 0) {
            f128 f = ((f128)P->scale[L] / (f128)P->prime[0]) / (2 * (f128)(B->K + 2));
            scale_columns(m, std::vector<f128>(n0, f));
        }
        B->cts.emplace_back(new LinTrans);
        build_lintrans(c, m, L - k, 1 << first[gi], sz[gi], *B->cts.back());
    }
}

static std::vector<std::unique_ptr<LinTrans>> &ensure_stc(hs_bts *B, int e)
{
    auto it = B->stc.find(e);
    if (it != B->stc.end()) return it->second;
    hs_ctx *c = B->ctx;
    const hs_params *P = c->P;
    const int n0 = P->n / 2;
    std::vector<int> sz = group_sizes(ilog2(n0), B->n_stc);
    std::vector<std::unique_ptr<LinTrans>> &T = B->stc[e];
    for (int gi = 0, st = 0; gi < B->n_stc; st += sz[gi], gi++) {
        DiagMat m = group_matrix(P->log_n, st, sz[gi], false);
        if (gi == 0) {
            f128 lam = (f128)P->prime[0] / (4 * M_PIq * (f128)P->scale[B->out_level] * ldexpq(1, e));
            std::vector<f128> dv(n0, 2 * lam);
            dv[0] = lam;
            scale_columns(m, dv);
        }
        T.emplace_back(new LinTrans);
        build_lintrans(c, m, B->out_level + B->n_stc - gi, 1 << st, sz[gi], *T.back());
    }
    return T;
}

// C17 double-hoisted BSGS (C17; same words as the oracle's
// apply_ltrans).  Every intermediate lives in the extended basis Q_l u P
// (ntg limbs per component, a value v standing for P v):
//   R_0 = P x;  R_b = (P sigma_b(c0) + <sigma_b(ModUp c1), evk_b>_0, <.>_1)
//   (one ModUp, one inner-product launch for all babies, NO ModDown);
//   inner_g = sum_b pt_{g,b} (.) R_b (one fused kernel, PQ plaintexts);
//   giants g != 0 (one batch): b' = ModDown(inner_g,1), Rot = (sigma_g(inner_g,0)
//   + <ModUp(sigma_g b'), evk_g>_0, <.>_1) (no ModDown);
//   out = ModDown + rescale by P q_l (C8) of inner_0 + sum Rot_g.
static CtP apply(const hs_keys *K, const hs_ct *in, const LinTrans &T, cudaStream_t st)
{
    hs_ctx *c = K->ctx;
    const hs_params *P = c->P;
    const size_t N = P->n;
    const int n0 = (int)N / 2, l = T.level, nl = l + 1, np = P->n_p, ntg = nl + np;
    const size_t W = (size_t)2 * ntg * N;  // one extended-basis ciphertext
    CtP lowered;
    const hs_ct *x = in;
    if (in->level != l) {
        lowered = ev_level_down(in, l, st);
        x = lowered.get();
    }
    PrimeMap pq;  // Q_l u P
    pq.n = ntg;
    for (int i = 0; i < ntg; i++) pq.p[i] = (unsigned char)(i < nl ? i : P->n_q + (i - nl));
    // ---- babies
    std::vector<int> bs, rots;
    for (int b = 1; b < T.b1; b++)
        if (std::find(T.b.begin(), T.b.end(), b) != T.b.end()) {
            bs.push_back(b);
            rots.push_back(b * T.unit);
        }
    std::vector<const u64 *> R(T.b1, nullptr);
    DBuf r0, hb;
    if (std::find(T.b.begin(), T.b.end(), 0) != T.b.end()) {  // R_0 = P x
        r0.alloc(W, st);
        u64 pmq[HS_MAXP];
        for (int i = 0; i < nl; i++) pmq[i] = P->p_mod_q[i];
        const PrimeMap pql = pmap_range(0, nl);
        for (int comp = 0; comp < 2; comp++) {
            k_mul_scalar_pm(c, x->limb(comp, 0), r0.p + (size_t)comp * ntg * N, pmq, nl, pql, st);
            HS_CUDA(cudaMemsetAsync(r0.p + ((size_t)comp * ntg + nl) * N, 0, (size_t)np * N * 8, st));
        }
        R[0] = r0.p;
    }
    if (!bs.empty()) {
        const int nb = (int)bs.size();
        std::vector<const u64 *> keys(nb);
        std::vector<const unsigned *> perms(nb);
        for (int i = 0; i < nb; i++) {
            const int k = hs_galois_elt(P, rots[i]);
            const SwKey *key = K->find(k);
            if (!key) throw HsError(HS_EKEY, "switching key for rotation " + std::to_string(rots[i]) + " missing");
            keys[i] = key->k;
            perms[i] = galois_table(c, k);
        }
        ModUpBuf m;
        ks_modup(c, l, 1, x->limb(1, 0), nl * N, m, st);
        hb.alloc((size_t)nb * W, st);
        k_ks_inner_h(c, x->limb(1, 0), m.ext.p, m.off, m.nd, keys.data(), perms.data(), nb, hb.p, l, m.beta, st,
                     x->limb(0, 0));
        for (int i = 0; i < nb; i++) R[bs[i]] = hb.p + (size_t)i * W;
        c->ledger[HS_LG_KS] += nb;
        c->ledger[HS_LG_ROT] += nb;
    }
    // ---- inner sums of every giant (increasing g; negative diagonals wrap)
    std::vector<int> gs(T.g.begin(), T.g.end());
    std::sort(gs.begin(), gs.end());
    gs.erase(std::unique(gs.begin(), gs.end()), gs.end());
    const int G = (int)gs.size();
    std::vector<int> tk((size_t)G * T.b1, -1);
    for (size_t k = 0; k < T.g.size(); k++) {
        const int gi = (int)(std::lower_bound(gs.begin(), gs.end(), T.g[k]) - gs.begin());
        tk[(size_t)gi * T.b1 + T.b[k]] = (int)k;
    }
    DBuf inners((size_t)G * W, st);
    k_bsgs_inner(c, R.data(), T.b1, T.pts, tk.data(), G, ntg, inners.p, st, nl);
    c->ledger[HS_LG_PMULT] += (int64_t)T.g.size();
    // ---- giants g != 0 as one batch
    const int g0 = gs[0] == 0 ? 1 : 0, ng = G - g0;
    // the accumulator is giant 0's inner sum in place (or the first rotated
    // giant's buffer when there is no giant 0): no copy
    u64 *acc = g0 ? inners.p : nullptr;
    DBuf rot;
    if (ng > 0) {
        const u64 *gin = inners.p + (size_t)g0 * W;
        // b'_g = ModDown(inner_g component 1): rows with stride W, out [ng][nl][N]
        DBuf bq((size_t)ng * nl * N, st);
        {
            DBuf z((size_t)ng * np * N, st);
            const BconvTab &md = bconv_moddown(c, l);
            const BconvTab *mdt = &md;
            k_ntt_inv_from(c, z.p, gin + ((size_t)ntg + nl) * N, W, np, ng * np, pmap_range(P->n_q, np), st,
                           bconv_ninv(c, &mdt, 1, ((long)l << 8) | 251));
            DBuf conv((size_t)ng * nl * N, st);
            k_bconv(c, md, z.p, N, conv.p, N, ng, (size_t)np * N, (size_t)nl * N, st, true);
            const u64 *a1 = gin + (size_t)ntg * N;
            if (!k_ntt_moddown(c, conv.p, a1, W, bq.p, 2 * (size_t)nl * N, nullptr, 0, 0, nl, nullptr, ng, st)) {
                k_ntt(c, conv.p, ng * nl, pmap_range(0, nl), false, st);
                k_moddown_final_b(c, a1, W, conv.p, nl, bq.p, 2 * (size_t)nl * N, nullptr, 0, 0, nullptr, ng, st);
            }
        }
        // sigma_g on b'_g (Q) and on inner_g component 0 (Q u P)
        std::vector<const u64 *> keys(ng);
        DBuf sb((size_t)ng * nl * N, st), sa((size_t)ng * ntg * N, st);
        for (int i = 0; i < ng; i++) {
            const int k = hs_galois_elt(P, (gs[g0 + i] * T.b1 * T.unit) % n0);
            const SwKey *key = K->find(k);
            if (!key) throw HsError(HS_EKEY, "switching key for a giant rotation missing");
            keys[i] = key->k;
            const unsigned *perm = galois_table(c, k);
            k_permute(c, bq.p + (size_t)i * nl * N, sb.p + (size_t)i * nl * N, perm, nl, st);
            k_permute(c, gin + (size_t)i * W, sa.p + (size_t)i * ntg * N, perm, ntg, st);
        }
        ModUpBuf m;
        ks_modup(c, l, ng, sb.p, (size_t)nl * N, m, st);
        rot.alloc((size_t)ng * W, st);
        k_ks_inner_m(c, sb.p, (size_t)nl * N, m.ext.p, m.off, m.nd, keys.data(), ng, rot.p, l, m.beta, st);
        for (int i = 0; i < ng; i++) {
            u64 *ri = rot.p + (size_t)i * W;
            k_add_pm(c, ri, sa.p + (size_t)i * ntg * N, ri, ntg, pq, st);  // + sigma_g(inner_g,0)
            if (i == 0 && !g0) acc = ri;
            else k_add_pm(c, acc, ri, acc, 2 * ntg, pq, st);
        }
        c->ledger[HS_LG_KS] += ng;
        c->ledger[HS_LG_ROT] += ng;
    }
    CtP out = ct_new(c, l - 1, 2, st);
    ks_moddown_rescale(c, l, 1, acc, out->d, out->ct_words(), st);
    c->ledger[HS_LG_RESCALE]++;
    return out;
}

CtP ev_bootstrap(const hs_keys *K, hs_bts *B, const hs_ct *in, double bound, cudaStream_t st)
{
    hs_ctx *c = K->ctx;
    const hs_params *P = c->P;
    const size_t N = P->n;
    const int L = P->L, conj = 2 * P->n - 1;
    if (in->ncomp != 2) throw HsError(HS_EINVAL, "bootstrap needs a degree-1 ciphertext");
    const int e = bts_exponent(P, B->arcsine, bound);
    std::vector<std::unique_ptr<LinTrans>> *stc;
    {
        std::lock_guard<std::mutex> g(B->mu);
        ensure_cts(B);
        stc = &ensure_stc(B, e);
    }
    // dev diagnostic: HS_BTS_PHASES=1 prints per-phase device time (eager calls only)
    struct Phases {
        bool on = false;
        cudaStream_t st = nullptr;
        std::vector<cudaEvent_t> ev;
        std::vector<const char *> nm;
        void mark(const char *n)
        {
            if (!on) return;
            cudaEvent_t e;
            cudaEventCreate(&e);
            cudaEventRecord(e, st);
            ev.push_back(e);
            nm.push_back(n);
        }
        ~Phases()
        {
            if (!on) return;
            cudaEventSynchronize(ev.back());
            for (size_t i = 1; i < ev.size(); i++) {
                float ms = 0;
                cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
                fprintf(stderr, "bts phase %-10s %8.3f ms\n", nm[i], ms);
            }
            for (auto e : ev) cudaEventDestroy(e);
        }
    } ph;
    {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(st, &cs);
        ph.on = getenv("HS_BTS_PHASES") && cs == cudaStreamCaptureStatusNone;
        ph.st = st;
    }
    ph.mark("start");
    CtP x = e ? ev_mult_int(in, (int64_t)1 << e, st) : ct_copy(in, st);
    // ModRaise of the q0 residues
    DBuf low(2 * N, st);
    HS_CUDA(cudaMemcpy2DAsync(low.p, N * 8, x->d, (x->level + 1) * N * 8, N * 8, 2, cudaMemcpyDeviceToDevice, st));
    PrimeMap p0;
    p0.n = 1;
    p0.p[0] = 0;
    k_ntt(c, low.p, 2, p0, true, st);
    x = ct_new(c, L, 2, st);
    k_modraise(c, low.p, x->d, L + 1, st);
    k_ntt(c, x->d, 2 * (L + 1), pmap_range(0, L + 1), false, st);
    ph.mark("modraise");
    for (auto &T : B->cts) {
        x = apply(K, x.get(), *T, st);
        ph.mark("cts-group");
    }
    CtP cj = ev_galois(K, x.get(), conj, st);
    x = ev_add(x.get(), cj.get(), false, st);
    x = ev_add_const(x.get(), -1.0 / (4.0 * (B->K + 2)), st);
    ph.mark("conj");
    if (B->even) {  // C18: even series, w = T_2(x), half the degree on w
        CtP m = ev_mult(K, x.get(), x.get(), st);
        CtP m2 = ev_mult_int(m.get(), 2, st);
        CtP w = ev_add_const(m2.get(), -1.0, st);
        x = ev_cheb(K, w.get(), &B->half_poly, 1.0, st);
    } else {
        x = ev_cheb(K, x.get(), &B->cos_poly, 1.0, st);
    }
    ph.mark("cos-cheb");
    for (int i = 0; i < B->r; i++) {
        CtP m = ev_mult(K, x.get(), x.get(), st);
        m = ev_mult_int(m.get(), 2, st);
        x = ev_add_const(m.get(), -1.0, st);
    }
    // gamma = Delta_out / Delta_in: the message was encoded at its own level's
    // scale; SlotToCoeff normalises by Delta_out
    const double gamma = P->scale[B->out_level] / P->scale[in->level];
    if (B->arcsine) {  // gamma (s + (1/6) s^3)
        CtP s6 = ev_mult_const(x.get(), gamma / 6.0, x->level - 1, st);
        CtP t = ev_mult(K, x.get(), x.get(), st);
        CtP u = ev_mult(K, s6.get(), t.get(), st);
        CtP sg = ev_mult_const(x.get(), gamma, u->level, st);
        x = ev_add(sg.get(), u.get(), false, st);
    } else {  // gamma s
        x = ev_mult_const(x.get(), gamma, x->level - 1, st);
    }
    ph.mark("dbl+arcsin");
    for (auto &T : *stc) {
        x = apply(K, x.get(), *T, st);
        ph.mark("stc-group");
    }
    cj = ev_galois(K, x.get(), conj, st);
    ph.mark("conj");
    c->ledger[HS_LG_BTS]++;
    return ev_add(x.get(), cj.get(), false, st);
}

// ------------------------------------------------------------------ C ABI
extern "C" {

hs_status hs_bts_create(hs_ctx *c, const hs_bts_desc *d, hs_bts **out)
{
    try {
        if (!c || !d || !out || !d->cos_poly || !d->cos_poly->coeffs || d->cos_poly->deg < 1 || d->r < 0 ||
            d->K < 1 || d->n_cts < 1 || d->n_cts > 8 || d->n_stc < 1 || d->n_stc > 8)
            throw HsError(HS_EINVAL, "hs_bts_create: bad descriptor");
        const hs_params *P = c->P;
        const int need =
            d->out_level + d->n_stc + (d->arcsine ? 2 : 1) + d->r + cheb_depth(d->cos_poly->deg) + d->n_cts;
        if (d->out_level < 0 || need != P->L)
            throw HsError(HS_ELEVEL, "hs_bts_create: chain top must be out + n_stc + 2 arcsine + r + depth + n_cts");
        std::unique_ptr<hs_bts> B(new hs_bts);
        B->ctx = c;
        B->K = d->K;
        B->r = d->r;
        B->out_level = d->out_level;
        B->n_cts = d->n_cts;
        B->n_stc = d->n_stc;
        B->arcsine = d->arcsine != 0;
        B->cos_coeffs.assign(d->cos_poly->coeffs, d->cos_poly->coeffs + d->cos_poly->deg + 1);
        B->cos_poly = hs_poly{d->cos_poly->deg, -1.0, 1.0, B->cos_coeffs.data()};
        B->even = d->cos_poly->deg >= 2;
        for (int i = 1; i <= d->cos_poly->deg; i += 2) B->even = B->even && d->cos_poly->coeffs[i] == 0.0;
        for (int k = 0; k <= d->cos_poly->deg / 2; k++) B->half_coeffs.push_back(d->cos_poly->coeffs[2 * k]);
        B->half_poly = hs_poly{d->cos_poly->deg / 2, -1.0, 1.0, B->half_coeffs.data()};
        *out = B.release();
        return HS_OK;
    } catch (const HsError &e) {
        return e.code;
    } catch (const std::exception &e) {
        return HS_EINVAL;
    }
}

void hs_bts_destroy(hs_bts *b) { delete b; }
int hs_bts_rotations(const hs_params *p, int n_cts, int n_stc, int32_t *out, int max)
{
    return bts_rotations(p, n_cts, n_stc, out, max);
}
int hs_bts_exponent(const hs_params *p, int arcsine, double bound) { return bts_exponent(p, arcsine, bound); }

}  // extern "C"
