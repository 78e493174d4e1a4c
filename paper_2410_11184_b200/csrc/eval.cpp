// eval.cpp -- host orchestration of the CKKS evaluator on one GPU.
//
// Every operation follows the oracle's written conventions:
//   C5 randomness, C6 Enc/Dec, C7 hybrid key switching, C8 HMult,
//   C9 rescale, C10 rotations, C11 operand levels, C12 canonical scales.
// Ciphertexts live in HBM limb-major [batch][comp][limb][N], NTT domain.  A
// batch holds several ciphertexts at one level (the Softmax main thread keeps
// its m/world ciphertexts as one batch): every op then runs as one launch per
// kernel over the whole batch, and the key switch reads each evaluation-key
// limb once per batch tile.  A batch-1 operand broadcasts against a batch.
// All temporaries are stream-ordered (cudaMallocAsync), so an op enqueues
// work and returns without synchronising.
#include <math.h>

#include <cstring>

#include "hs_internal.h"

enum { TAG_SK = 1, TAG_PK_A = 2, TAG_PK_E = 3, TAG_KSK_A = 4, TAG_KSK_E = 5,
       TAG_ENC_V = 6, TAG_ENC_E0 = 7, TAG_ENC_E1 = 8, TAG_ENC_A = 9 };
static const int ETA_ERR = 21, ETA_V = 1;

// ------------------------------------------------------------------ memory
// Default pool: the device's stream-ordered pool (cudaMallocAsync) for
// temporaries and ciphertexts, cudaMalloc for long-lived tables.  With an
// allocator hook (hs_context_create_ex) both go through the hook, except
// inside a CUDA-graph capture (graph-owned memory nodes).  Each hook
// allocation is recorded with a copy of its hook so that the free finds it.
namespace {
struct HookRec {
    hs_allocator a;
    size_t bytes;
};
std::mutex g_hook_mu;
std::map<void *, HookRec> g_hook_ptrs;
thread_local AllocHook tl_hook;
thread_local int tl_capturing = 0;

bool capturing(cudaStream_t st)
{
    if (tl_capturing) return true;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
}

void *hook_alloc(size_t bytes, cudaStream_t st)
{
    void *p = tl_hook.a.alloc(bytes, (void *)st, tl_hook.a.user);
    if (!p) throw HsError(HS_ENOMEM, "allocator hook returned NULL");
    std::lock_guard<std::mutex> g(g_hook_mu);
    g_hook_ptrs[p] = HookRec{tl_hook.a, bytes};
    return p;
}

bool hook_take(void *p, HookRec &r)
{
    std::lock_guard<std::mutex> g(g_hook_mu);
    auto it = g_hook_ptrs.find(p);
    if (it == g_hook_ptrs.end()) return false;
    r = it->second;
    g_hook_ptrs.erase(it);
    return true;
}
}  // namespace

void alloc_hook_set(const AllocHook &h) { tl_hook = h; }
void alloc_capturing(bool on) { tl_capturing += on ? 1 : -1; }

u64 *dev_alloc(size_t words, cudaStream_t st)
{
    void *p = nullptr;
    if (words == 0) words = 1;
    if (tl_hook.on && !capturing(st)) return (u64 *)hook_alloc(words * sizeof(u64), st);
    cudaError_t e = cudaMallocAsync(&p, words * sizeof(u64), st);
    if (e != cudaSuccess) throw HsError(e == cudaErrorMemoryAllocation ? HS_ENOMEM : HS_ECUDA,
                                        std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
    return (u64 *)p;
}

void dev_free(void *p, cudaStream_t st)
{
    if (!p) return;
    HookRec r;
    if (hook_take(p, r))
        r.a.free(p, r.bytes, (void *)st, r.a.user);
    else
        cudaFreeAsync(p, st);
}

void *dev_alloc_persist(size_t bytes)
{
    if (bytes == 0) bytes = 8;
    if (tl_hook.on && !tl_capturing) return hook_alloc(bytes, nullptr);
    void *p = nullptr;
    HS_CUDA(cudaMalloc(&p, bytes));
    return p;
}

void dev_free_persist(void *p)
{
    if (!p) return;
    HookRec r;
    if (hook_take(p, r))
        r.a.free(p, r.bytes, nullptr, r.a.user);
    else
        cudaFree(p);
}

hs_ctx::~hs_ctx()
{
    cudaDeviceSynchronize();
    for (auto &kv : bconv) {
        dev_free_persist(kv.second.dev);
        dev_free_persist(kv.second.mma);
    }
    for (auto &kv : galois_perm) dev_free_persist(kv.second);
    for (auto &kv : bconv_ninv) dev_free_persist(kv.second);
    for (auto &kv : pt_cache) dev_free_persist(kv.second);
    for (auto e : kprof_ev) cudaEventDestroy(e);
    dev_free_persist(T.tw);
}

hs_keys::~hs_keys()
{
    cudaDeviceSynchronize();
    dev_free_persist(s_ntt);
    dev_free_persist(pk);
    for (auto &k : swk) dev_free_persist(k.k);
}

hs_ct::~hs_ct()
{
    if (d && owns) dev_free(d, st);
}

size_t hs_ct::ct_words() const { return (size_t)ncomp * (level + 1) * ctx->P->n; }
u64 *hs_ct::limb(int comp, int i) const { return d + ((size_t)comp * (level + 1) + i) * ctx->P->n; }
u64 *hs_ct::at(int b, int comp, int i) const { return d + (((size_t)b * ncomp + comp) * (level + 1) + i) * ctx->P->n; }

CtP ct_new(hs_ctx *c, int level, int ncomp, cudaStream_t st, int batch)
{
    CtP r(new hs_ct);
    r->ctx = c;
    r->level = level;
    r->ncomp = ncomp;
    r->batch = batch;
    r->st = st;
    r->d = dev_alloc((size_t)batch * ncomp * (level + 1) * c->P->n, st);
    return r;
}

CtP ct_copy(const hs_ct *a, cudaStream_t st)
{
    CtP r = ct_new(a->ctx, a->level, a->ncomp, st, a->batch);
    HS_CUDA(cudaMemcpyAsync(r->d, a->d, a->limbs() * a->ctx->P->n * 8, cudaMemcpyDeviceToDevice, st));
    return r;
}

// keep limbs 0..level of every row
CtP ct_drop(const hs_ct *a, int level, cudaStream_t st)
{
    if (level == a->level) return ct_copy(a, st);
    hs_ctx *c = a->ctx;
    CtP r = ct_new(c, level, a->ncomp, st, a->batch);
    size_t N = c->P->n;
    HS_CUDA(cudaMemcpy2DAsync(r->d, (level + 1) * N * 8, a->d, (a->level + 1) * N * 8, (level + 1) * N * 8, a->rows(),
                              cudaMemcpyDeviceToDevice, st));
    return r;
}

CtP ct_gather(const hs_ct *const *cts, int n, cudaStream_t st)
{
    const hs_ct *a = cts[0];
    CtP r = ct_new(a->ctx, a->level, a->ncomp, st, n);
    for (int b = 0; b < n; b++) {
        if (cts[b]->level != a->level || cts[b]->ncomp != a->ncomp || cts[b]->batch != 1)
            throw HsError(HS_EINVAL, "gather: ciphertexts differ in level or shape");
        HS_CUDA(cudaMemcpyAsync(r->d + b * a->ct_words(), cts[b]->d, a->ct_words() * 8, cudaMemcpyDeviceToDevice, st));
    }
    return r;
}

// non-owning view of batch member b (valid while a lives)
CtP ct_view(const hs_ct *a, int b)
{
    CtP r(new hs_ct);
    r->ctx = a->ctx;
    r->level = a->level;
    r->ncomp = a->ncomp;
    r->batch = 1;
    r->st = a->st;
    r->d = a->d + b * a->ct_words();
    r->owns = false;
    return r;
}

CtP ct_slice(const hs_ct *a, int b, cudaStream_t st)
{
    CtP r = ct_new(a->ctx, a->level, a->ncomp, st, 1);
    HS_CUDA(cudaMemcpyAsync(r->d, a->d + b * a->ct_words(), a->ct_words() * 8, cudaMemcpyDeviceToDevice, st));
    return r;
}

// ------------------------------------------------------------------ tables
// BConv target constants are stored in Montgomery form c 2^64 mod q: the
// kernels sum y_a c'_a in 128 bits and one REDC (T 2^-64 mod q) lands on
// sum y_a c_a mod q directly.
static u64 mont(u64 v, u64 q) { return (u64)(((u128)v << 64) % q); }

// B-operand fragments of the tensor-core BConv (kernels.cu bconv_mma_kernel).
// The conversion sum_a y_a c_ab (c_ab in Montgomery form, mod p_b) is split
// into bytes: y_a = sum_u y_au 2^8u and c'_aub = 2^8u c_ab mod p_b =
// sum_v c'_aubv 2^8v, so sum_a y_a c_ab == sum_v 2^8v D_bv (mod p_b) with
// D_bv = sum_(a,u) y_au c'_aubv -- an exact u8 x u8 -> s32 product with
// K = (a, u) (8 sources x 8 bytes) and N = (b, v).  Fragment of lane
// (g = lane / 4, t = lane % 4), k-step s, register r: the 4 bytes
// k = 16 r + 4 t + i (i = 0..3) of column v = g, i.e. source a = 4 s + 2 r +
// t / 2, bytes u = 4 (t % 2) + i.
void bconv_build_mma(BconvTab &t, const std::vector<u64> &h, const hs_params *P)
{
    if (t.n_src > 8) return;
    std::vector<uint32_t> f((size_t)t.n_dst * 2 * 32 * 2, 0);
    for (int b = 0; b < t.n_dst; b++) {
        const u64 p = P->prime[t.dst[b]];
        for (int s = 0; s < 2; s++)
            for (int lane = 0; lane < 32; lane++)
                for (int r = 0; r < 2; r++) {
                    const int g = lane >> 2, tg = lane & 3, a = 4 * s + 2 * r + (tg >> 1);
                    uint32_t reg = 0;
                    if (a < t.n_src) {
                        const u64 cm = h[2 * t.n_src + 2 * ((size_t)a * t.n_dst + b)];
                        for (int i = 0; i < 4; i++) {
                            const int u = 4 * (tg & 1) + i;
                            const u64 cu = (u64)(((u128)cm << (8 * u)) % p);
                            reg |= (uint32_t)((cu >> (8 * g)) & 0xff) << (8 * i);
                        }
                    }
                    f[(((size_t)b * 2 + s) * 32 + lane) * 2 + r] = reg;
                }
    }
    t.mma = (uint32_t *)dev_alloc_persist(f.size() * 4);
    HS_CUDA(cudaMemcpy(t.mma, f.data(), f.size() * 4, cudaMemcpyHostToDevice));
}

const BconvTab &bconv_modup(hs_ctx *c, int level, int digit)
{
    std::lock_guard<std::mutex> g(c->mu);
    long key = ((long)level << 8) | digit;
    auto it = c->bconv.find(key);
    if (it != c->bconv.end()) return it->second;
    const hs_params *P = c->P;
    BconvTab t;
    int nl = level + 1, lo = digit * P->alpha, hi = std::min((digit + 1) * P->alpha, nl);
    for (int i = lo; i < hi; i++) t.src.push_back(i);
    for (int i = 0; i < nl; i++)
        if (i < lo || i >= hi) t.dst.push_back(i);
    for (int k = 0; k < P->n_p; k++) t.dst.push_back(P->n_q + k);
    t.n_src = (int)t.src.size();
    t.n_dst = (int)t.dst.size();
    std::vector<u64> h(2 * t.n_src + 2 * (size_t)t.n_src * t.n_dst);
    for (int a = 0; a < t.n_src; a++) {
        u64 qa = P->prime[t.src[a]], qh = 1;
        for (int b = 0; b < t.n_src; b++)
            if (b != a) qh = hs_mulmod(qh, P->prime[t.src[b]] % qa, qa);
        h[2 * a] = hs_invmod(qh, qa);
        h[2 * a + 1] = hs_shoup_const(h[2 * a], qa);
        for (int d = 0; d < t.n_dst; d++) {
            u64 p = P->prime[t.dst[d]], v = 1;
            for (int b = 0; b < t.n_src; b++)
                if (b != a) v = hs_mulmod(v, P->prime[t.src[b]] % p, p);
            size_t ci = 2 * t.n_src + 2 * ((size_t)a * t.n_dst + d);
            h[ci] = mont(v, p);  // kernel accumulates 128-bit, one REDC
            h[ci + 1] = hs_shoup_const(v, p);
        }
    }
    t.dev = (decltype(t.dev))dev_alloc_persist(h.size() * 8);
    HS_CUDA(cudaMemcpy(t.dev, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
    bconv_build_mma(t, h, P);
    return c->bconv[key] = t;
}

const BconvTab &bconv_moddown(hs_ctx *c, int level)
{
    std::lock_guard<std::mutex> g(c->mu);
    long key = ((long)level << 8) | 255;
    auto it = c->bconv.find(key);
    if (it != c->bconv.end()) return it->second;
    const hs_params *P = c->P;
    BconvTab t;
    for (int k = 0; k < P->n_p; k++) t.src.push_back(P->n_q + k);
    for (int i = 0; i <= level; i++) t.dst.push_back(i);
    t.n_src = (int)t.src.size();
    t.n_dst = (int)t.dst.size();
    t.centred = true;
    // [n_src](inv, inv_sh), [n_src][n_dst](c, c_sh), then [n_dst] P mod q (centred correction)
    std::vector<u64> h(2 * t.n_src + 2 * (size_t)t.n_src * t.n_dst + t.n_dst);
    for (int a = 0; a < t.n_src; a++) {
        u64 pa = P->prime[t.src[a]], ph = 1;
        for (int b = 0; b < t.n_src; b++)
            if (b != a) ph = hs_mulmod(ph, P->prime[t.src[b]] % pa, pa);
        h[2 * a] = hs_invmod(ph, pa);
        h[2 * a + 1] = hs_shoup_const(h[2 * a], pa);
        for (int d = 0; d < t.n_dst; d++) {
            u64 q = P->prime[t.dst[d]], v = 1;
            for (int b = 0; b < t.n_src; b++)
                if (b != a) v = hs_mulmod(v, P->prime[t.src[b]] % q, q);
            size_t ci = 2 * t.n_src + 2 * ((size_t)a * t.n_dst + d);
            h[ci] = mont(v, q);  // kernel accumulates 128-bit, one REDC
            h[ci + 1] = hs_shoup_const(v, q);
        }
    }
    for (int d = 0; d < t.n_dst; d++) h[2 * t.n_src + 2 * (size_t)t.n_src * t.n_dst + d] = P->p_mod_q[t.dst[d]];
    t.dev = (decltype(t.dev))dev_alloc_persist(h.size() * 8);
    HS_CUDA(cudaMemcpy(t.dev, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
    bconv_build_mma(t, h, P);
    return c->bconv[key] = t;
}

// C8 fused ModDown + rescale: centred BConv from the sources {q_level,
// p_0..p_{np-1}} (S = P q_level) to q_0..q_{level-1}; correction S mod q_i.
const BconvTab &bconv_moddown_rescale(hs_ctx *c, int level)
{
    std::lock_guard<std::mutex> g(c->mu);
    long key = ((long)level << 8) | 254;
    auto it = c->bconv.find(key);
    if (it != c->bconv.end()) return it->second;
    const hs_params *P = c->P;
    BconvTab t;
    t.src.push_back(level);
    for (int k = 0; k < P->n_p; k++) t.src.push_back(P->n_q + k);
    for (int i = 0; i < level; i++) t.dst.push_back(i);
    t.n_src = (int)t.src.size();
    t.n_dst = (int)t.dst.size();
    t.centred = true;
    std::vector<u64> h(2 * t.n_src + 2 * (size_t)t.n_src * t.n_dst + t.n_dst);
    for (int a = 0; a < t.n_src; a++) {
        u64 sa = P->prime[t.src[a]], sh = 1;
        for (int b = 0; b < t.n_src; b++)
            if (b != a) sh = hs_mulmod(sh, P->prime[t.src[b]] % sa, sa);
        h[2 * a] = hs_invmod(sh, sa);
        h[2 * a + 1] = hs_shoup_const(h[2 * a], sa);
        for (int d = 0; d < t.n_dst; d++) {
            u64 q = P->prime[t.dst[d]], v = 1;
            for (int b = 0; b < t.n_src; b++)
                if (b != a) v = hs_mulmod(v, P->prime[t.src[b]] % q, q);
            size_t ci = 2 * t.n_src + 2 * ((size_t)a * t.n_dst + d);
            h[ci] = mont(v, q);  // kernel accumulates 128-bit, one REDC
            h[ci + 1] = hs_shoup_const(v, q);
        }
    }
    for (int d = 0; d < t.n_dst; d++) {
        u64 q = P->prime[t.dst[d]];
        h[2 * t.n_src + 2 * (size_t)t.n_src * t.n_dst + d] = hs_mulmod(P->p_mod_q[t.dst[d]], P->prime[level] % q, q);
    }
    t.dev = (decltype(t.dev))dev_alloc_persist(h.size() * 8);
    HS_CUDA(cudaMemcpy(t.dev, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
    bconv_build_mma(t, h, P);
    return c->bconv[key] = t;
}

const u64 *bconv_ninv(hs_ctx *c, const BconvTab *const *tabs, int n_tabs, long key)
{
    {
        std::lock_guard<std::mutex> g(c->mu);
        auto it = c->bconv_ninv.find(key);
        if (it != c->bconv_ninv.end()) return it->second;
    }
    const hs_params *P = c->P;
    const int np = P->n_q + P->n_p;
    std::vector<u64> h(2 * (size_t)np, 0);
    for (int t = 0; t < n_tabs; t++) {
        const BconvTab &T = *tabs[t];
        for (int a = 0; a < T.n_src; a++) {
            const int pi = T.src[a];
            const u64 q = P->prime[pi];
            // qhat_a^-1 as the table holds it, times N^-1
            u64 qh = 1;
            for (int b = 0; b < T.n_src; b++)
                if (b != a) qh = hs_mulmod(qh, P->prime[T.src[b]] % q, q);
            const u64 v = hs_mulmod(hs_invmod(qh, q), P->n_inv[pi], q);
            h[2 * pi] = v;
            h[2 * pi + 1] = hs_shoup_const(v, q);
        }
    }
    u64 *d = (u64 *)dev_alloc_persist(h.size() * 8);
    HS_CUDA(cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
    std::lock_guard<std::mutex> g(c->mu);
    auto it = c->bconv_ninv.find(key);
    if (it != c->bconv_ninv.end()) {  // another thread won the race
        dev_free_persist(d);
        return it->second;
    }
    return c->bconv_ninv[key] = d;
}

// C10: out[i] = in[perm[i]], perm[i] = brv(((2 brv(i) + 1) k mod 2N - 1) / 2)
const unsigned *galois_table(hs_ctx *c, int k)
{
    std::lock_guard<std::mutex> g(c->mu);
    auto it = c->galois_perm.find(k);
    if (it != c->galois_perm.end()) return it->second;
    const hs_params *P = c->P;
    int N = P->n, lg = P->log_n;
    auto brv = [lg](unsigned x) {
        unsigned r = 0;
        for (int i = 0; i < lg; i++, x >>= 1) r = (r << 1) | (x & 1);
        return r;
    };
    std::vector<unsigned> h(N);
    u64 two_n = 2ull * N;
    for (int i = 0; i < N; i++) {
        u64 e = 2ull * brv((unsigned)i) + 1;
        h[i] = brv((unsigned)(((e * (u64)k) % two_n - 1) / 2));
    }
    unsigned *d;
    d = (decltype(d))dev_alloc_persist(N * sizeof(unsigned));
    HS_CUDA(cudaMemcpy(d, h.data(), N * sizeof(unsigned), cudaMemcpyHostToDevice));
    return c->galois_perm[k] = d;
}

// ------------------------------------------------------------------ key switching (C7)
// ModUp of B polynomials d_b = d + b*d_stride (level+1 limbs, NTT domain):
// digit j's extension to every target prime but its own, block [B][nd_j][N].
// the ModUp union of a level's digit tables (every Q prime of the level is
// a source of exactly one digit)
static const u64 *modup_ninv(hs_ctx *c, int level)
{
    const hs_params *P = c->P;
    const int nl = level + 1, beta = (nl + P->alpha - 1) / P->alpha;
    const BconvTab *tabs[HS_MAXDIG];
    for (int j = 0; j < beta; j++) tabs[j] = &bconv_modup(c, level, j);
    return bconv_ninv(c, tabs, beta, ((long)level << 8) | 250);
}

void ks_modup(hs_ctx *c, int level, int B, const u64 *d, size_t d_stride, ModUpBuf &m, cudaStream_t st)
{
    const hs_params *P = c->P;
    const size_t N = P->n;
    const int nl = level + 1, alpha = P->alpha;
    m.beta = (nl + alpha - 1) / alpha;
    // coefficient form of every d_b: [B][nl][N]
    DBuf x((size_t)B * nl * N, st);
    k_ntt_inv_from(c, x.p, d, d_stride, nl, B * nl, pmap_range(0, nl), st, modup_ninv(c, level));
    size_t tot = 0;
    for (int j = 0; j < m.beta; j++) {
        const BconvTab &tab = bconv_modup(c, level, j);
        m.off[j] = tot;
        m.nd[j] = tab.n_dst;
        tot += (size_t)B * tab.n_dst * N;
    }
    m.ext.alloc(tot, st);
    if (B == 1 && tot / N <= 256 && m.beta <= 12) {
        // one polynomial: every digit in ONE BConv launch and ONE NTT launch
        // (bigger grids than beta small launches; same words)
        const BconvTab *tabs[16];
        PrimeMap pm;
        pm.n = 0;
        for (int j = 0; j < m.beta; j++) {
            tabs[j] = &bconv_modup(c, level, j);
            for (int i = 0; i < tabs[j]->n_dst; i++) pm.p[pm.n++] = (unsigned char)tabs[j]->dst[i];
        }
        k_bconv_modup_multi(c, tabs, m.off, m.beta, x.p, m.ext.p, st, true);
        k_ntt(c, m.ext.p, pm.n, pm, false, st);
        return;
    }
    for (int j = 0; j < m.beta; j++) {
        const BconvTab &tab = bconv_modup(c, level, j);
        u64 *e = m.ext.p + m.off[j];
        k_bconv(c, tab, x.p + (size_t)tab.src[0] * N, N, e, N, B, (size_t)nl * N, (size_t)tab.n_dst * N, st, true);
        PrimeMap pm;
        pm.n = tab.n_dst;
        for (int i = 0; i < tab.n_dst; i++) pm.p[i] = (unsigned char)tab.dst[i];
        k_ntt(c, e, B * tab.n_dst, pm, false, st);
    }
}

// ModDown of B accumulators acc [B][2][ntg][N]: iNTT of the P limbs, centred
// BConv P -> Q_l, NTT, out_b = add_b + (acc - conv) P^{-1}
void ks_moddown(hs_ctx *c, int level, int B, const u64 *acc, u64 *out, size_t out_stride, const u64 *add,
                size_t add_stride, int add_comps, cudaStream_t st)
{
    const hs_params *P = c->P;
    const size_t N = P->n;
    const int nl = level + 1, np = P->n_p, ntg = nl + np;
    DBuf z((size_t)B * 2 * np * N, st);
    const BconvTab &md = bconv_moddown(c, level);
    const BconvTab *mdt = &md;
    k_ntt_inv_from(c, z.p, acc + (size_t)nl * N, ntg * N, np, 2 * B * np, pmap_range(P->n_q, np), st,
                   bconv_ninv(c, &mdt, 1, ((long)level << 8) | 251));
    DBuf conv((size_t)B * 2 * nl * N, st);
    k_bconv(c, md, z.p, N, conv.p, N, 2 * B, (size_t)np * N, (size_t)nl * N, st, true);
    const size_t ar = (size_t)ntg * N;
    if (k_ntt_moddown(c, conv.p, acc, ar, out, out_stride, add, add_stride, add_comps, nl, nullptr, 2 * B, st)) return;
    k_ntt(c, conv.p, 2 * B * nl, pmap_range(0, nl), false, st);
    k_moddown_final_b(c, acc, ar, conv.p, nl, out, out_stride, add, add_stride, add_comps, nullptr, 2 * B, st);
}

// C8 fused ModDown + rescale of B accumulators acc [B][2][ntg][N] (basis
// Q_level u P): ONE centred BConv from {q_level, p_0..} to q_0..q_{level-1},
// out_b = (acc - conv) (P q_level)^-1 at level - 1 (out: [B][2][level][N]).
void ks_moddown_rescale(hs_ctx *c, int level, int B, const u64 *acc, u64 *out, size_t out_stride, cudaStream_t st)
{
    const hs_params *P = c->P;
    const size_t N = P->n;
    const int nl = level + 1, np = P->n_p, ntg = nl + np, ns = np + 1;
    // the sources q_level, p_0.. are acc limbs level .. ntg-1 of every row
    DBuf z((size_t)B * 2 * ns * N, st);
    PrimeMap pz;
    pz.n = ns;
    pz.p[0] = (unsigned char)level;
    for (int k = 0; k < np; k++) pz.p[1 + k] = (unsigned char)(P->n_q + k);
    const BconvTab &md = bconv_moddown_rescale(c, level);
    const BconvTab *mdt = &md;
    k_ntt_inv_from(c, z.p, acc + (size_t)level * N, ntg * N, ns, 2 * B * ns, pz, st,
                   bconv_ninv(c, &mdt, 1, ((long)level << 8) | 252));
    DBuf conv((size_t)B * 2 * level * N, st);
    k_bconv(c, md, z.p, N, conv.p, N, 2 * B, (size_t)ns * N, (size_t)level * N, st, true);
    std::vector<u64> inv(level);
    for (int i = 0; i < level; i++) {
        const u64 q = P->prime[i];
        inv[i] = hs_invmod(hs_mulmod(P->p_mod_q[i], P->prime[level] % q, q), q);
    }
    const size_t ar = (size_t)ntg * N;
    if (k_ntt_moddown(c, conv.p, acc, ar, out, out_stride, nullptr, 0, 0, level, inv.data(), 2 * B, st)) return;
    k_ntt(c, conv.p, 2 * B * level, pmap_range(0, level), false, st);
    k_moddown_final_b(c, acc, ar, conv.p, level, out, out_stride, nullptr, 0, 0, inv.data(), 2 * B, st);
}

// Digit-parallel key switch: rank r of G runs ModUp and
// the evaluation-key inner product for its digits only; the partial
// accumulators are summed mod q (exact, order-free: the C7 accumulator is a
// sum over the digits mod q) and moved down once.  Only the digits' own limbs
// are brought to coefficient form.
void ks_partial(const hs_keys *K, const SwKey *key, int level, const u64 *d, int j0, int j1, u64 *acc,
                cudaStream_t st, const u64 *dadd, size_t dadd_stride)
{
    hs_ctx *c = K->ctx;
    const hs_params *P = c->P;
    const size_t N = P->n;
    const int nl = level + 1, alpha = P->alpha, beta = (nl + alpha - 1) / alpha;
    if (j0 < 0 || j1 > beta || j0 > j1) throw HsError(HS_EINVAL, "key switch: digit range out of [0, beta]");
    const int ntg = nl + P->n_p;
    if (j0 == j1) {
        if (!dadd) {
            HS_CUDA(cudaMemsetAsync(acc, 0, (size_t)2 * ntg * N * 8, st));
            return;
        }
        // no digits: the C8 P*d term alone
        size_t off0[HS_MAXDIG] = {0};
        int nd0[HS_MAXDIG] = {0};
        k_ks_inner_b(c, d, (size_t)nl * N, nullptr, off0, nd0, key->k, acc, level, j1, 1, st, dadd, dadd_stride, j0);
        return;
    }
    const int lo0 = j0 * alpha, hi1 = std::min(j1 * alpha, nl), cnt = hi1 - lo0;
    DBuf x((size_t)cnt * N, st);
    k_ntt_inv_from(c, x.p, d + (size_t)lo0 * N, (size_t)cnt * N, cnt, cnt, pmap_range(lo0, cnt), st,
                   modup_ninv(c, level));
    ModUpBuf m;
    m.beta = j1;
    size_t tot = 0;
    for (int j = j0; j < j1; j++) {
        const BconvTab &tab = bconv_modup(c, level, j);
        m.off[j] = tot;
        m.nd[j] = tab.n_dst;
        tot += (size_t)tab.n_dst * N;
    }
    m.ext.alloc(tot, st);
    for (int j = j0; j < j1; j++) {
        const BconvTab &tab = bconv_modup(c, level, j);
        u64 *e = m.ext.p + m.off[j];
        k_bconv(c, tab, x.p + (size_t)(tab.src[0] - lo0) * N, N, e, N, 1, (size_t)cnt * N, (size_t)tab.n_dst * N, st,
                true);
        PrimeMap pm;
        pm.n = tab.n_dst;
        for (int i = 0; i < tab.n_dst; i++) pm.p[i] = (unsigned char)tab.dst[i];
        k_ntt(c, e, tab.n_dst, pm, false, st);
    }
    k_ks_inner_b(c, d, (size_t)nl * N, m.ext.p, m.off, m.nd, key->k, acc, level, j1, 1, st, dadd, dadd_stride, j0);
}

bool ks_sum_fits(const hs_params *P, int world)
{
    u64 mx = 0;
    for (u64 q : P->prime) mx = std::max(mx, q);
    return (u128)world * (mx - 1) < ((u128)1 << 64);
}

void ks_split_acc(hs_ctx *c, const hs_keys *K, const SwKey *key, int level, const u64 *d, const u64 *dadd,
                  size_t dadd_stride, u64 *acc, cudaStream_t st)
{
    const hs_params *P = c->P;
    const size_t N = P->n;
    const int nl = level + 1, beta = (nl + P->alpha - 1) / P->alpha, ntg = nl + P->n_p;
    const size_t words = (size_t)2 * ntg * N;
    const hs_ctx::KsSplit &S = c->ks_split;
    auto range = [&](int r, int G, int &j0, int &j1) {
        j0 = (int)((long)r * beta / G);
        j1 = (int)((long)(r + 1) * beta / G);
    };
    int j0, j1;
    if (S.emulate >= 2) {
        DBuf part(words, st);
        for (int r = 0; r < S.emulate; r++) {
            range(r, S.emulate, j0, j1);
            ks_partial(K, key, level, d, j0, j1, r == 0 ? acc : part.p, st, r == 0 ? dadd : nullptr,
                       dadd_stride);
            if (r > 0) ks_acc_add(c, level, acc, part.p, st);
        }
        return;
    }
    range(S.rank, S.world, j0, j1);
    if (S.comm && ks_sum_fits(P, S.world)) {
        // uint64 sum all-reduce (exact: world * q < 2^64), then mod q -- moves
        // ~2x the accumulator per rank instead of world x
        ks_partial(K, key, level, d, j0, j1, acc, st, S.rank == 0 ? dadd : nullptr, dadd_stride);
        comm_all_reduce_u64(S.comm, acc, words, st);
        PrimeMap pm;
        pm.n = ntg;
        for (int g = 0; g < ntg; g++) pm.p[g] = (unsigned char)(g < nl ? g : P->n_q + (g - nl));
        k_mod_pm(c, acc, 2 * ntg, pm, st);
        return;
    }
    DBuf part(words, st), gathered(words * S.world, st);
    // the C8 P*d term rides with rank 0's share
    ks_partial(K, key, level, d, j0, j1, part.p, st, S.rank == 0 ? dadd : nullptr, dadd_stride);
    if (S.comm) comm_all_gather(S.comm, part.p, gathered.p, words, st);
    else if (S.ex(S.user, part.p, gathered.p, words, st) != 0)
        throw HsError(HS_ENCCL, "aux key switch: exchange callback failed");
    HS_CUDA(cudaMemcpyAsync(acc, gathered.p, words * 8, cudaMemcpyDeviceToDevice, st));
    for (int r = 1; r < S.world; r++) ks_acc_add(c, level, acc, gathered.p + r * words, st);
}

void ks_acc_add(hs_ctx *c, int level, u64 *acc, const u64 *other, cudaStream_t st)
{
    const hs_params *P = c->P;
    const int nl = level + 1, ntg = nl + P->n_p;
    PrimeMap pm;
    pm.n = ntg;
    for (int g = 0; g < ntg; g++) pm.p[g] = (unsigned char)(g < nl ? g : P->n_q + (g - nl));
    k_add_pm(c, acc, other, acc, 2 * ntg, pm, st);
}

// B polynomials d_b = d + b*d_stride (level+1 limbs each, NTT domain);
// out_b = out + b*out_stride gets (ks0, ks1) (+ add_b's first add_comps components).
void ev_keyswitch_b(const hs_keys *K, const SwKey *key, int level, int B, const u64 *d, size_t d_stride, u64 *out,
                    size_t out_stride, const u64 *add, size_t add_stride, int add_comps, cudaStream_t st)
{
    hs_ctx *c = K->ctx;
    const hs_params *P = c->P;
    const size_t N = P->n;
    const int ntg = level + 1 + P->n_p;
    DBuf acc((size_t)B * 2 * ntg * N, st);
    if (B == 1 && c->ks_split_on) {
        // digit-parallel key switch of a single-ciphertext op
        ks_split_acc(c, K, key, level, d, nullptr, 0, acc.p, st);
    } else {
        ModUpBuf m;
        ks_modup(c, level, B, d, d_stride, m, st);
        // inner product with the evaluation key: acc[B][2][ntg][N]
        k_ks_inner_b(c, d, d_stride, m.ext.p, m.off, m.nd, key->k, acc.p, level, m.beta, B, st);
    }
    ks_moddown(c, level, B, acc.p, out, out_stride, add, add_stride, add_comps, st);
    c->ledger[HS_LG_KS] += B;
}

// C16: rotations rots[0..R) of ONE degree-1 ciphertext from a single ModUp of
// its c1 (hoisting); returns a batch of R ciphertexts, batch r = Rot(a, rots[r]).
CtP ev_rotate_hoisted(const hs_keys *K, const hs_ct *a, const int *rots, int R, cudaStream_t st)
{
    hs_ctx *c = K->ctx;
    const hs_params *P = c->P;
    const size_t N = P->n;
    const int l = a->level, nl = l + 1, ntg = nl + P->n_p;
    if (a->ncomp != 2 || a->batch != 1) throw HsError(HS_EINVAL, "hoisted rotation needs one degree-1 ciphertext");
    if (R < 1 || R > HS_MAXROT) throw HsError(HS_EINVAL, "hoisted rotation: bad rotation count");
    std::vector<const u64 *> keys(R);
    std::vector<const unsigned *> perms(R);
    for (int r = 0; r < R; r++) {
        const int k = hs_galois_elt(P, rots[r]);
        const SwKey *key = K->find(k);
        if (!key) throw HsError(HS_EKEY, "switching key for rotation " + std::to_string(rots[r]) + " missing");
        keys[r] = key->k;
        perms[r] = galois_table(c, k);
    }
    const u64 *c1 = a->limb(1, 0);
    ModUpBuf m;
    ks_modup(c, l, 1, c1, nl * N, m, st);
    DBuf acc((size_t)R * 2 * ntg * N, st);
    k_ks_inner_h(c, c1, m.ext.p, m.off, m.nd, keys.data(), perms.data(), R, acc.p, l, m.beta, st);
    // sigma_r(c0) as the added component 0 of each output
    DBuf c0p((size_t)R * nl * N, st);
    for (int r = 0; r < R; r++) k_permute(c, a->limb(0, 0), c0p.p + (size_t)r * nl * N, perms[r], nl, st);
    CtP out = ct_new(c, l, 2, st, R);
    ks_moddown(c, l, R, acc.p, out->d, out->ct_words(), c0p.p, (size_t)nl * N, 1, st);
    c->ledger[HS_LG_KS] += R;
    c->ledger[HS_LG_ROT] += R;
    return out;
}

void ev_keyswitch(const hs_keys *K, const SwKey *key, int level, const u64 *d, u64 *out0, u64 *out1,
                  const u64 *add0, const u64 *add1, cudaStream_t st)
{
    // (out0, out1) and (add0, add1) as separate pointers: the hooks' layout
    const size_t N = K->ctx->P->n, nl = level + 1;
    DBuf o(2 * nl * N, st), a(add0 || add1 ? 2 * nl * N : 0, st);
    int add_comps = 0;
    if (add0 || add1) {
        HS_CUDA(cudaMemsetAsync(a.p, 0, 2 * nl * N * 8, st));
        if (add0) HS_CUDA(cudaMemcpyAsync(a.p, add0, nl * N * 8, cudaMemcpyDeviceToDevice, st));
        if (add1) HS_CUDA(cudaMemcpyAsync(a.p + nl * N, add1, nl * N * 8, cudaMemcpyDeviceToDevice, st));
        add_comps = 2;
    }
    ev_keyswitch_b(K, key, level, 1, d, nl * N, o.p, 2 * nl * N, add_comps ? a.p : nullptr, 2 * nl * N, add_comps,
                   st);
    HS_CUDA(cudaMemcpyAsync(out0, o.p, nl * N * 8, cudaMemcpyDeviceToDevice, st));
    HS_CUDA(cudaMemcpyAsync(out1, o.p + nl * N, nl * N * 8, cudaMemcpyDeviceToDevice, st));
}

// ------------------------------------------------------------------ arithmetic
CtP ev_rescale(const hs_ct *a, cudaStream_t st)
{
    hs_ctx *c = a->ctx;
    const size_t N = c->P->n;
    const int l = a->level, rows = (int)a->rows();
    if (l < 1) throw HsError(HS_ELEVEL, "rescale at level 0");
    DBuf last((size_t)rows * N, st);
    HS_CUDA(cudaMemcpy2DAsync(last.p, N * 8, a->d + (size_t)l * N, (l + 1) * N * 8, N * 8, rows,
                              cudaMemcpyDeviceToDevice, st));
    PrimeMap pm;
    pm.n = 1;
    pm.p[0] = (unsigned char)l;
    k_ntt(c, last.p, rows, pm, true, st);
    DBuf w((size_t)rows * l * N, st);
    CtP r = ct_new(c, l - 1, a->ncomp, st, a->batch);
    if (!k_ntt_rescale(c, last.p, w.p, a->d, r->d, rows, l, st)) {
        k_rescale_prep(c, last.p, w.p, rows, l, st);
        k_ntt(c, w.p, rows * l, pmap_range(0, l), false, st);
        k_rescale_final(c, a->d, w.p, r->d, rows, l, st);
    }
    c->ledger[HS_LG_RESCALE] += a->batch;
    return r;
}

// C12 landing constant: sc = (Delta_target q_{target+1}) / Delta_level
static double landing_scale(const hs_params *P, int level, int target)
{
    return (P->scale[target] * (double)P->prime[target + 1]) / P->scale[level];
}

static void residues(const hs_params *P, double v, int n, u64 *out)
{
    for (int i = 0; i < n; i++) out[i] = hs_residue_of_double(v, P->prime[i]);
}

CtP ev_mult_const(const hs_ct *a, double v, int target, cudaStream_t st)
{
    hs_ctx *c = a->ctx;
    const hs_params *P = c->P;
    if (target < 0 || target >= a->level) throw HsError(HS_ELEVEL, "mult_const: target level must be below the input");
    const int nl = target + 2;
    u64 s[HS_MAXP];
    residues(P, v * landing_scale(P, a->level, target), nl, s);
    c->ledger[HS_LG_CMULT] += a->batch;
    if (P->log_n == 16) {
        // drop + scale + rescale without a pass over the whole ciphertext: only
        // the dropped limb l = target+1 is scaled here; the NTT-fused rescale
        // multiplies limbs 0..target by s_i in its epilogue (same words)
        const size_t N = P->n;
        const int l = target + 1, rows = (int)a->rows();
        DBuf last((size_t)rows * N, st);
        HS_CUDA(cudaMemcpy2DAsync(last.p, N * 8, a->d + (size_t)l * N, (a->level + 1) * N * 8, N * 8, rows,
                                  cudaMemcpyDeviceToDevice, st));
        PrimeMap pl;
        pl.n = 1;
        pl.p[0] = (unsigned char)l;
        k_mul_scalar_pm(c, last.p, last.p, &s[l], rows, pl, st);
        k_ntt(c, last.p, rows, pl, true, st);
        DBuf w((size_t)rows * l * N, st);
        CtP r = ct_new(c, target, a->ncomp, st, a->batch);
        k_ntt_rescale(c, last.p, w.p, a->d, r->d, rows, l, st, s, (a->level + 1) * N);
        c->ledger[HS_LG_RESCALE] += a->batch;
        return r;
    }
    CtP d = ct_new(c, target + 1, a->ncomp, st, a->batch);
    k_mul_scalar_s(c, a->d, d->d, s, (int)a->rows(), nl, a->level + 1, nl, false, st);  // drop + scale
    return ev_rescale(d.get(), st);
}

CtP ev_level_down(const hs_ct *a, int target, cudaStream_t st)
{
    if (target == a->level) return ct_copy(a, st);
    if (target > a->level) throw HsError(HS_ELEVEL, "level_down to a higher level");
    a->ctx->ledger[HS_LG_LEVELDOWN] += a->batch;
    return ev_mult_const(a, 1.0, target, st);
}

static void match(const hs_ct *a, const hs_ct *b, CtP &ta, CtP &tb, const hs_ct *&ra, const hs_ct *&rb,
                  cudaStream_t st)
{
    ra = a;
    rb = b;
    if (a->level > b->level) {
        ta = ev_level_down(a, b->level, st);
        ra = ta.get();
    } else if (b->level > a->level) {
        tb = ev_level_down(b, a->level, st);
        rb = tb.get();
    }
}

static int out_batch(const hs_ct *a, const hs_ct *b)
{
    if (a->batch != b->batch && a->batch != 1 && b->batch != 1)
        throw HsError(HS_EINVAL, "operand batches must match or one must be 1");
    return std::max(a->batch, b->batch);
}

CtP ev_add(const hs_ct *a, const hs_ct *b, bool sub, cudaStream_t st)
{
    if (a->ncomp != b->ncomp) throw HsError(HS_EINVAL, "add: component counts differ");
    const int B = out_batch(a, b);
    CtP ta, tb;
    const hs_ct *ra, *rb;
    match(a, b, ta, tb, ra, rb, st);
    CtP r = ct_new(a->ctx, ra->level, ra->ncomp, st, B);
    k_add_b(a->ctx, ra->d, (int)ra->rows(), rb->d, (int)rb->rows(), r->d, (int)r->rows(), ra->level + 1, sub, st);
    return r;
}

CtP ev_mult_int(const hs_ct *a, int64_t v, cudaStream_t st)
{
    const hs_params *P = a->ctx->P;
    u64 s[HS_MAXP];
    for (int i = 0; i <= a->level; i++) {
        int64_t m = v % (int64_t)P->prime[i];
        s[i] = (u64)(m < 0 ? m + (int64_t)P->prime[i] : m);
    }
    CtP r = ct_new(a->ctx, a->level, a->ncomp, st, a->batch);
    k_mul_scalar(a->ctx, a->d, r->d, s, (int)a->limbs(), a->level + 1, st);
    return r;
}

CtP ev_add_const(const hs_ct *a, double v, cudaStream_t st)
{
    const hs_params *P = a->ctx->P;
    u64 s[HS_MAXP];
    residues(P, v * P->scale[a->level], a->level + 1, s);
    CtP r = ct_copy(a, st);
    k_add_scalar_b(a->ctx, r->d, s, a->batch, a->ncomp, a->level + 1, st);
    return r;
}

CtP ev_mult_pt(const hs_ct *a, const double *re, const double *im, int target, cudaStream_t st)
{
    hs_ctx *c = a->ctx;
    const hs_params *P = c->P;
    if (target < 0 || target >= a->level) throw HsError(HS_ELEVEL, "mult_pt: target level must be below the input");
    const size_t N = P->n;
    const int nl = target + 2;
    // encoded plaintexts are cached per (slot content, input level, target):
    // the Softmax mask is re-used every iteration
    u64 h = 1469598103934665603ull;
    auto mix = [&h](const double *v, size_t n) {
        const unsigned char *p = (const unsigned char *)v;
        for (size_t i = 0; i < n * 8; i++) h = (h ^ p[i]) * 1099511628211ull;
    };
    mix(re, N / 2);
    if (im) mix(im, N / 2);
    else h ^= 0x9e3779b97f4a7c15ull;
    const std::pair<u64, long> key(h, ((long)a->level << 16) | target);
    u64 *m;
    {
        std::lock_guard<std::mutex> g(c->mu);
        auto it = c->pt_cache.find(key);
        m = it == c->pt_cache.end() ? nullptr : it->second;
    }
    if (!m) {
        std::vector<u64> pt((size_t)nl * N);
        hs_encode_impl(P, re, im, landing_scale(P, a->level, target), target + 1, pt.data());
        m = (decltype(m))dev_alloc_persist(pt.size() * 8);
        HS_CUDA(cudaMemcpy(m, pt.data(), pt.size() * 8, cudaMemcpyHostToDevice));
        k_ntt(c, m, nl, pmap_range(0, nl), false, st);
        std::lock_guard<std::mutex> g(c->mu);
        c->pt_cache[key] = m;
    }
    CtP d = ct_drop(a, target + 1, st);
    k_mul_pointwise(c, d->d, m, d->d, (int)d->limbs(), nl, nl, st);
    c->ledger[HS_LG_PMULT] += a->batch;
    return ev_rescale(d.get(), st);
}

CtP ev_tensor(const hs_ct *a, const hs_ct *b, cudaStream_t st)
{
    if (a->ncomp != 2 || b->ncomp != 2) throw HsError(HS_EINVAL, "tensor needs degree-1 ciphertexts");
    const int B = out_batch(a, b);
    CtP ta, tb;
    const hs_ct *ra, *rb;
    match(a, b, ta, tb, ra, rb, st);
    if (ra->batch < rb->batch) std::swap(ra, rb);  // the tensor is symmetric: broadcast the second operand
    CtP r = ct_new(a->ctx, ra->level, 3, st, B);
    k_tensor_b(a->ctx, ra->d, rb->d, r->d, B, ra->level + 1, rb->batch, st);
    a->ctx->ledger[HS_LG_TENSOR] += B;
    return r;
}

CtP ev_tensor_sum(const hs_ct *a, cudaStream_t st)
{
    if (a->ncomp != 2) throw HsError(HS_EINVAL, "tensor_sum needs degree-1 ciphertexts");
    CtP r = ct_new(a->ctx, a->level, 3, st, 1);
    k_tensor_sum(a->ctx, a->d, r->d, a->batch, a->level + 1, st);
    a->ctx->ledger[HS_LG_TENSOR] += a->batch;
    return r;
}

// sum_b a_b (x) c_b over the members of two batches (C15 with distinct
// operands; the higher-level operand is brought down as in every product)
CtP ev_tensor_sum2(const hs_ct *a, const hs_ct *b, cudaStream_t st)
{
    if (a->ncomp != 2 || b->ncomp != 2 || a->batch != b->batch)
        throw HsError(HS_EINVAL, "tensor_sum2 needs two degree-1 batches of one size");
    CtP ta, tb;
    const hs_ct *ra, *rb;
    match(a, b, ta, tb, ra, rb, st);
    CtP r = ct_new(a->ctx, ra->level, 3, st, 1);
    k_tensor_sum2(a->ctx, ra->d, rb->d, r->d, a->batch, ra->level + 1, st);
    a->ctx->ledger[HS_LG_TENSOR] += a->batch;
    return r;
}

CtP ev_relin(const hs_keys *K, const hs_ct *d, cudaStream_t st)
{
    const SwKey *rk = K->find(0);
    if (!rk) throw HsError(HS_EKEY, "relinearisation key missing");
    if (d->ncomp != 3) throw HsError(HS_EINVAL, "relin needs a degree-2 ciphertext");
    CtP r = ct_new(d->ctx, d->level, 2, st, d->batch);
    const size_t w3 = d->ct_words();
    ev_keyswitch_b(K, rk, d->level, d->batch, d->limb(2, 0), w3, r->d, r->ct_words(), d->d, w3, 2, st);
    return r;
}

// C8: relinearise + rescale as ONE division of (P d + sum ModUp(d2) evk) by
// P q_level (the P d term rides in the evk inner product); output level - 1.
CtP ev_relin_rescale(const hs_keys *K, const hs_ct *d, cudaStream_t st)
{
    const SwKey *rk = K->find(0);
    if (!rk) throw HsError(HS_EKEY, "relinearisation key missing");
    if (d->ncomp != 3) throw HsError(HS_EINVAL, "relin needs a degree-2 ciphertext");
    if (d->level < 1) throw HsError(HS_ELEVEL, "rescale at level 0");
    hs_ctx *c = d->ctx;
    const hs_params *P = c->P;
    const size_t N = P->n;
    const int l = d->level, B = d->batch, ntg = l + 1 + P->n_p;
    const size_t w3 = d->ct_words();
    DBuf acc((size_t)B * 2 * ntg * N, st);
    if (B == 1 && c->ks_split_on) {
        ks_split_acc(c, K, rk, l, d->limb(2, 0), d->d, w3, acc.p, st);
    } else {
        ModUpBuf m;
        ks_modup(c, l, B, d->limb(2, 0), w3, m, st);
        k_ks_inner_b(c, d->limb(2, 0), w3, m.ext.p, m.off, m.nd, rk->k, acc.p, l, m.beta, B, st, d->d, w3);
    }
    CtP r = ct_new(c, l - 1, 2, st, B);
    ks_moddown_rescale(c, l, B, acc.p, r->d, r->ct_words(), st);
    c->ledger[HS_LG_KS] += B;
    c->ledger[HS_LG_RESCALE] += B;
    return r;
}

CtP ev_mult(const hs_keys *K, const hs_ct *a, const hs_ct *b, cudaStream_t st)
{
    CtP t = ev_tensor(a, b, st);
    K->ctx->ledger[HS_LG_HMULT] += t->batch;
    return ev_relin_rescale(K, t.get(), st);
}

CtP ev_galois(const hs_keys *K, const hs_ct *a, int k, cudaStream_t st)
{
    const SwKey *key = K->find(k);
    if (!key) throw HsError(HS_EKEY, "switching key for Galois element " + std::to_string(k) + " missing");
    if (a->ncomp != 2) throw HsError(HS_EINVAL, "rotation needs a degree-1 ciphertext");
    hs_ctx *c = a->ctx;
    CtP s = ct_new(c, a->level, 2, st, a->batch);
    k_permute(c, a->d, s->d, galois_table(c, k), (int)a->limbs(), st);
    CtP r = ct_new(c, a->level, 2, st, a->batch);
    const size_t w = a->ct_words();
    ev_keyswitch_b(K, key, a->level, a->batch, s->limb(1, 0), w, r->d, w, s->d, w, 1, st);
    c->ledger[HS_LG_ROT] += a->batch;
    return r;
}

// out_b = Rot(a_b, rots[b]) for every member of the batch a, as ONE batched
// key switch with a key per member (the BTS giant steps); words identical to
// rotating each member alone.
CtP ev_rotate_multi(const hs_keys *K, const hs_ct *a, const int *rots, cudaStream_t st)
{
    hs_ctx *c = a->ctx;
    const hs_params *P = c->P;
    const size_t N = P->n;
    const int B = a->batch, l = a->level, nl = l + 1, ntg = nl + P->n_p;
    if (a->ncomp != 2) throw HsError(HS_EINVAL, "rotation needs a degree-1 ciphertext");
    if (B < 1 || B > HS_MAXROT) throw HsError(HS_EINVAL, "rotate_multi: batch out of range");
    const size_t w = a->ct_words();
    std::vector<const u64 *> keys(B);
    CtP s = ct_new(c, l, 2, st, B);
    for (int b = 0; b < B; b++) {
        const int k = hs_galois_elt(P, rots[b]);
        const SwKey *key = K->find(k);
        if (!key) throw HsError(HS_EKEY, "switching key for rotation " + std::to_string(rots[b]) + " missing");
        keys[b] = key->k;
        k_permute(c, a->d + b * w, s->d + b * w, galois_table(c, k), 2 * nl, st);
    }
    ModUpBuf m;
    ks_modup(c, l, B, s->limb(1, 0), w, m, st);
    DBuf acc((size_t)B * 2 * ntg * N, st);
    k_ks_inner_m(c, s->limb(1, 0), w, m.ext.p, m.off, m.nd, keys.data(), B, acc.p, l, m.beta, st);
    CtP r = ct_new(c, l, 2, st, B);
    ks_moddown(c, l, B, acc.p, r->d, w, s->d, w, 1, st);
    c->ledger[HS_LG_KS] += B;
    c->ledger[HS_LG_ROT] += B;
    return r;
}

CtP ev_rotate(const hs_keys *K, const hs_ct *a, int r, cudaStream_t st)
{
    return ev_galois(K, a, hs_galois_elt(K->ctx->P, r), st);
}

// sum_i coef_i * terms_i landing at `target` with ONE rescale (C13 leaves):
// every term is dropped to target+1 and multiplied by rint(coef_i * sc_i).
CtP ev_mult_const_sum(const std::vector<const hs_ct *> &terms, const std::vector<double> &coef, int target,
                      cudaStream_t st)
{
    hs_ctx *c = terms[0]->ctx;
    const hs_params *P = c->P;
    const size_t N = P->n;
    const int nl = target + 2;
    int B = 1;
    for (auto t : terms) B = std::max(B, t->batch);
    CtP acc = ct_new(c, target + 1, 2, st, B);
    // every nonzero term in one pass per 16 (k_lin_comb): sum_i rint(c_i sc_i) T_i
    std::vector<const u64 *> ptr;
    std::vector<int> rl;
    std::vector<std::vector<u64>> sc;
    for (size_t i = 0; i < terms.size(); i++) {
        if (coef[i] == 0.0) continue;
        const hs_ct *t = terms[i];
        if (t->level < target + 1) throw HsError(HS_ELEVEL, "leaf term below its landing level");
        if (t->batch != B) throw HsError(HS_EINVAL, "leaf terms must share the batch");
        sc.emplace_back(HS_MAXP);
        residues(P, coef[i] * landing_scale(P, t->level, target), nl, sc.back().data());
        ptr.push_back(t->d);
        rl.push_back(t->level + 1);
        c->ledger[HS_LG_CMULT] += B;
    }
    if (ptr.empty()) {
        HS_CUDA(cudaMemsetAsync(acc->d, 0, acc->limbs() * N * 8, st));
    } else {
        const int rows = (int)acc->rows();
        for (size_t j0 = 0; j0 < ptr.size(); j0 += 16) {
            const int nt = (int)std::min<size_t>(16, ptr.size() - j0);
            std::vector<const u64 *> sp(nt);
            for (int j = 0; j < nt; j++) sp[j] = sc[j0 + j].data();
            k_lin_comb(c, ptr.data() + j0, rl.data() + j0, sp.data(), nt, acc->d, rows, nl, nl, j0 > 0, st);
        }
    }
    return ev_rescale(acc.get(), st);
}

// ------------------------------------------------------------------ keys (C5, C6, C7)
static void sample_secret(const hs_params *P, u64 seed, int h, std::vector<int64_t> &s)
{
    int N = P->n;
    std::vector<int> pos(N);
    for (int i = 0; i < N; i++) pos[i] = i;
    s.assign(N, 0);
    for (int i = 0; i < h; i++) {
        u64 w = hs_stream_word(seed, TAG_SK, 0, 2 * (u64)i);
        int j = i + (int)(w % (u64)(N - i));
        std::swap(pos[i], pos[j]);
        s[pos[i]] = (hs_stream_word(seed, TAG_SK, 0, 2 * (u64)i + 1) & 1) ? -1 : 1;
    }
}

// e (CBD eta) in coefficient form -> NTT residues over primes [0, n)
static void error_poly(hs_ctx *c, u64 seed, uint32_t tag, u64 sub, int eta, u64 *out, int n, cudaStream_t st)
{
    DBuf e(c->P->n, st);
    k_cbd(c, (int64_t *)e.p, seed, tag, sub, eta, st);
    k_signed_to_rns(c, (const int64_t *)e.p, out, n, pmap_range(0, n), st);
    k_ntt(c, out, n, pmap_range(0, n), false, st);
}

hs_keys *keys_generate(hs_ctx *c, u64 seed, int h, const int32_t *galois, size_t n_galois, int relin, cudaStream_t st)
{
    const hs_params *P = c->P;
    const size_t N = P->n;
    const int nt = P->n_q + P->n_p, nq = P->n_q;
    std::unique_ptr<hs_keys> K(new hs_keys);
    K->ctx = c;
    if (h < 1 || h > P->n) throw HsError(HS_EINVAL, "secret Hamming weight out of range");
    sample_secret(P, seed, h, K->s_coeff);
    K->s_ntt = (decltype(K->s_ntt))dev_alloc_persist((size_t)nt * N * 8);
    {
        DBuf sc(N, st);
        HS_CUDA(cudaMemcpyAsync(sc.p, K->s_coeff.data(), N * 8, cudaMemcpyHostToDevice, st));
        k_signed_to_rns(c, (const int64_t *)sc.p, K->s_ntt, nt, pmap_range(0, nt), st);
        k_ntt(c, K->s_ntt, nt, pmap_range(0, nt), false, st);
        HS_CUDA(cudaStreamSynchronize(st));
    }
    // pk = (-a s + e, a) over Q_L
    K->pk = (decltype(K->pk))dev_alloc_persist((size_t)2 * nq * N * 8);
    {
        u64 *b = K->pk, *a = K->pk + (size_t)nq * N;
        k_uniform(c, a, nq, pmap_range(0, nq), seed, TAG_PK_A, 0, 0, st);
        error_poly(c, seed, TAG_PK_E, 0, ETA_ERR, b, nq, st);
        DBuf as((size_t)nq * N, st);
        k_mul_pointwise(c, a, K->s_ntt, as.p, nq, nq, nq, st);
        k_add(c, b, as.p, b, nq, nq, true, st);
    }
    // switching keys: relin (s' = s^2) then one per Galois element (s' = sigma_k(s))
    std::vector<int> ids;
    if (relin) ids.push_back(0);
    for (size_t i = 0; i < n_galois; i++) ids.push_back(galois[i]);
    DBuf sp((size_t)nt * N, st), as((size_t)nt * N, st);
    for (int id : ids) {
        if (id == 0) k_mul_pointwise(c, K->s_ntt, K->s_ntt, sp.p, nt, nt, nt, st);
        else k_permute(c, K->s_ntt, sp.p, galois_table(c, id), nt, st);
        SwKey key;
        key.galois = id;
        // generated component-planar ([dnum][2][nt][N]) in a scratch buffer,
        // stored interleaved ([dnum][nt][N][2]: one 16-byte load per word pair)
        DBuf planar((size_t)P->dnum * 2 * nt * N, st);
        key.k = (decltype(key.k))dev_alloc_persist((size_t)P->dnum * 2 * nt * N * 8);
        for (int j = 0; j < P->dnum; j++) {
            u64 sub = (u64)id * 256 + (u64)j;
            u64 *k0 = planar.p + (size_t)(2 * j) * nt * N, *k1 = planar.p + (size_t)(2 * j + 1) * nt * N;
            k_uniform(c, k1, nt, pmap_range(0, nt), seed, TAG_KSK_A, sub, 0, st);
            error_poly(c, seed, TAG_KSK_E, sub, ETA_ERR, k0, nt, st);
            k_mul_pointwise(c, k1, K->s_ntt, as.p, nt, nt, nt, st);
            k_add(c, k0, as.p, k0, nt, nt, true, st);
            u64 g[HS_MAXP];
            for (int i = 0; i < nq; i++) g[i] = (i / P->alpha == j) ? P->p_mod_q[i] : 0;
            k_mac_scalar(c, k0, sp.p, g, nq, nq, st);
        }
        k_interleave2(c, planar.p, key.k, P->dnum, nt * N, st);
        K->swk.push_back(key);
    }
    HS_CUDA(cudaStreamSynchronize(st));
    return K.release();
}

CtP ev_encrypt(const hs_keys *K, const u64 *pt_host, int level, u64 seed, u64 idx, bool use_sk, cudaStream_t st)
{
    hs_ctx *c = K->ctx;
    const hs_params *P = c->P;
    const size_t N = P->n;
    const int nl = level + 1;
    if (level < 0 || level > P->L) throw HsError(HS_EINVAL, "encrypt: level out of range");
    DBuf m((size_t)nl * N, st);
    HS_CUDA(cudaMemcpyAsync(m.p, pt_host, (size_t)nl * N * 8, cudaMemcpyHostToDevice, st));
    k_ntt(c, m.p, nl, pmap_range(0, nl), false, st);
    CtP r = ct_new(c, level, 2, st);
    u64 *c0 = r->limb(0, 0), *c1 = r->limb(1, 0);
    DBuf tmp((size_t)nl * N, st);
    if (use_sk && !K->s_ntt) throw HsError(HS_EKEY, "encrypt: this key set holds no secret (hs_keys_upload)");
    if (!use_sk && !K->pk) throw HsError(HS_EKEY, "encrypt: this key set holds no public key");
    if (use_sk) {
        k_uniform(c, c1, nl, pmap_range(0, nl), seed, TAG_ENC_A, idx, 0, st);
        error_poly(c, seed, TAG_ENC_E0, idx, ETA_ERR, c0, nl, st);
        k_mul_pointwise(c, c1, K->s_ntt, tmp.p, nl, nl, nl, st);
        k_add(c, c0, tmp.p, c0, nl, nl, true, st);
        k_add(c, c0, m.p, c0, nl, nl, false, st);
    } else {
        DBuf v((size_t)nl * N, st);
        error_poly(c, seed, TAG_ENC_V, idx, ETA_V, v.p, nl, st);
        error_poly(c, seed, TAG_ENC_E0, idx, ETA_ERR, c0, nl, st);
        error_poly(c, seed, TAG_ENC_E1, idx, ETA_ERR, c1, nl, st);
        const u64 *b = K->pk, *a = K->pk + (size_t)P->n_q * N;
        k_mul_pointwise(c, v.p, b, tmp.p, nl, nl, nl, st);
        k_add(c, c0, tmp.p, c0, nl, nl, false, st);
        k_add(c, c0, m.p, c0, nl, nl, false, st);
        k_mul_pointwise(c, v.p, a, tmp.p, nl, nl, nl, st);
        k_add(c, c1, tmp.p, c1, nl, nl, false, st);
    }
    HS_CUDA(cudaStreamSynchronize(st));  // host pt lifetime
    return r;
}

void ev_decrypt(const hs_keys *K, const hs_ct *ct, u64 *host_out, cudaStream_t st)
{
    hs_ctx *c = K->ctx;
    const size_t N = c->P->n;
    const int nl = ct->level + 1;
    if (ct->batch != 1) throw HsError(HS_EINVAL, "decrypt one ciphertext at a time");
    if (!K->s_ntt) throw HsError(HS_EKEY, "decrypt: this key set holds no secret (hs_keys_upload)");
    DBuf m((size_t)nl * N, st);
    k_mul_pointwise(c, ct->limb(1, 0), K->s_ntt, m.p, nl, nl, nl, st);
    k_add(c, m.p, ct->limb(0, 0), m.p, nl, nl, false, st);
    k_ntt(c, m.p, nl, pmap_range(0, nl), true, st);
    HS_CUDA(cudaMemcpyAsync(host_out, m.p, (size_t)nl * N * 8, cudaMemcpyDeviceToHost, st));
    HS_CUDA(cudaStreamSynchronize(st));
}
