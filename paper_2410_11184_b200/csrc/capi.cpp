// capi.cpp -- the extern "C" boundary (include/hesoftmax.h).  No exception
// crosses it: every entry point converts HsError / std::exception into an
// hs_status and a thread-local message.
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "hs_internal.h"

static thread_local std::string g_err;
static std::mutex g_active_mu;
// per device: __constant__ memory is per device (one module image each)
static const hs_params *g_active[HS_MAXDEV] = {nullptr};

#define HS_TRY try {
#define HS_CATCH                                              \
    }                                                         \
    catch (const HsError &e) {                                \
        g_err = e.what();                                     \
        return e.code;                                        \
    }                                                         \
    catch (const std::bad_alloc &) {                          \
        g_err = "host allocation failed";                     \
        return HS_ENOMEM;                                     \
    }                                                         \
    catch (const std::exception &e) {                         \
        g_err = e.what();                                     \
        return HS_EINVAL;                                     \
    }

static cudaStream_t S(void *s) { return (cudaStream_t)s; }

// The prime constants live in __constant__ memory of the module; make sure they
// hold this context's parameter set before enqueueing work.
static void activate(hs_ctx *c)
{
    std::lock_guard<std::mutex> g(g_active_mu);
    if (c->device < 0 || c->device >= HS_MAXDEV) throw HsError(HS_EINVAL, "device index out of range");
    HS_CUDA(cudaSetDevice(c->device));
    if (g_active[c->device] != c->P) {
        HS_CUDA(cudaDeviceSynchronize());
        upload_prime_constants(c->P);
        g_active[c->device] = c->P;
    }
    alloc_hook_set(c->alloc);
}

void check_scales(const hs_ct *a, const hs_ct *b)
{
    const hs_params *P = a->ctx->P;
    for (const hs_ct *x : {a, b}) {
        if (x->scale == 0.0) continue;
        const double canon = P->scale[x->level];
        if (fabs(x->scale / canon - 1.0) > ldexp(1.0, -40))
            throw HsError(HS_ESCALE, "operand declared at a non-canonical scale (C11)");
    }
}

extern "C" {

const char *hs_last_error(void) { return g_err.c_str(); }

hs_status hs_ckks_params(const hs_params_desc *d, hs_params **out)
{
    HS_TRY
    if (!out) throw HsError(HS_EINVAL, "out is NULL");
    std::unique_ptr<hs_params> P(new hs_params);
    hs_build_params(d, P.get());
    *out = P.release();
    return HS_OK;
    HS_CATCH
}

void hs_params_destroy(hs_params *p)
{
    std::lock_guard<std::mutex> g(g_active_mu);
    for (auto &a : g_active)
        if (a == p) a = nullptr;
    delete p;
}
int hs_params_log_n(const hs_params *p) { return p->log_n; }
int hs_params_n_q(const hs_params *p) { return p->n_q; }
int hs_params_n_p(const hs_params *p) { return p->n_p; }
hs_status hs_params_primes(const hs_params *p, uint64_t *out)
{
    if (!p || !out) return HS_EINVAL;
    memcpy(out, p->prime.data(), p->prime.size() * 8);
    return HS_OK;
}
uint64_t hs_params_psi(const hs_params *p, int i) { return p->psi.at(i); }
double hs_params_scale(const hs_params *p, int level) { return p->scale.at(level); }
int hs_galois_of_rot(const hs_params *p, int r) { return hs_galois_elt(p, r); }

hs_status hs_context_create_ex(const hs_params *p, int device, const hs_allocator *alloc, hs_ctx **out)
{
    HS_TRY
    if (!p || !out) throw HsError(HS_EINVAL, "NULL argument");
    if (alloc && (!alloc->alloc) != (!alloc->free))
        throw HsError(HS_EINVAL, "hs_allocator: alloc and free must both be set");
    int ndev = 0;
    HS_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw HsError(HS_EINVAL, "no such CUDA device");
    HS_CUDA(cudaSetDevice(device));
    std::unique_ptr<hs_ctx> c(new hs_ctx);
    c->P = p;
    c->device = device;
    if (alloc && alloc->alloc) {
        c->alloc.a = *alloc;
        c->alloc.on = true;
    }
    // the twiddle tables below already go through the hook; the thread's
    // current hook is cleared again on every exit (activate() sets it per call)
    struct HookOff {
        ~HookOff() { alloc_hook_set(AllocHook{}); }
    } hook_off;
    alloc_hook_set(c->alloc);
    const int np = p->n_q + p->n_p;
    const size_t N = p->n;
    // [np][4][N] integer twiddles, [np](N^-1, Shoup), then [np][2][N] the
    // twiddles as doubles for the FP64 NTT path (primes < 2^43, kernels.cu)
    std::vector<u64> h((size_t)np * 4 * N + 2 * np + (size_t)np * 2 * N);
    // device layout per prime: (w, w') pairs of the forward table, then of the
    // inverse table -- one 16-byte load per butterfly
    for (int i = 0; i < np; i++)
        for (int half = 0; half < 2; half++)
            for (size_t k = 0; k < N; k++) {
                h[(size_t)i * 4 * N + half * 2 * N + 2 * k] = p->tw[i][half * 2 * N + k];
                h[(size_t)i * 4 * N + half * 2 * N + 2 * k + 1] = p->tw[i][half * 2 * N + N + k];
            }
    for (int i = 0; i < np; i++) {
        h[(size_t)np * 4 * N + 2 * i] = p->n_inv[i];
        h[(size_t)np * 4 * N + 2 * i + 1] = p->n_inv_sh[i];
    }
    const size_t foff = (size_t)np * 4 * N + 2 * np;
    for (int i = 0; i < np; i++)
        if (p->prime[i] < (1ull << 43))
            for (int half = 0; half < 2; half++)
                for (size_t k = 0; k < N; k++) {
                    const double w = (double)p->tw[i][half * 2 * N + k];  // exact: w < 2^43
                    memcpy(&h[foff + (size_t)i * 2 * N + half * N + k], &w, 8);
                }
    c->T.tw = (decltype(c->T.tw))dev_alloc_persist(h.size() * 8);
    HS_CUDA(cudaMemcpy(c->T.tw, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
    // keep freed stream-ordered memory in the pool (no release back to the OS)
    cudaMemPool_t pool;
    HS_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    HS_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    activate(c.get());
    *out = c.release();
    return HS_OK;
    HS_CATCH
}

hs_status hs_context_create(const hs_params *p, int device, hs_ctx **out)
{
    return hs_context_create_ex(p, device, nullptr, out);
}

void hs_context_destroy(hs_ctx *c)
{
    delete c;
    alloc_hook_set(AllocHook{});
}

hs_status hs_ckks_keygen(hs_ctx *c, uint64_t seed, int h, const int32_t *galois, size_t n_galois, int relin,
                         void *stream, hs_keys **out)
{
    HS_TRY
    if (!c || !out || (n_galois && !galois)) throw HsError(HS_EINVAL, "NULL argument");
    activate(c);
    *out = keys_generate(c, seed, h, galois, n_galois, relin, S(stream));
    return HS_OK;
    HS_CATCH
}

void hs_keys_destroy(hs_keys *k) { delete k; }

hs_status hs_keys_export_swk(hs_ctx *c, const hs_keys *k, int galois, uint64_t *host_out)
{
    HS_TRY
    const SwKey *key = k->find(galois);
    if (!key) throw HsError(HS_EKEY, "no such switching key");
    const hs_params *P = c->P;
    HS_CUDA(cudaDeviceSynchronize());
    // stored interleaved [dnum][nt][N][2]; exported planar [dnum][2][nt][N]
    const size_t W = (size_t)(P->n_q + P->n_p) * P->n;
    std::vector<uint64_t> tmp((size_t)P->dnum * 2 * W);
    HS_CUDA(cudaMemcpy(tmp.data(), key->k, tmp.size() * 8, cudaMemcpyDeviceToHost));
    for (int j = 0; j < P->dnum; j++)
        for (size_t w = 0; w < W; w++) {
            host_out[((size_t)j * 2 + 0) * W + w] = tmp[((size_t)j * W + w) * 2 + 0];
            host_out[((size_t)j * 2 + 1) * W + w] = tmp[((size_t)j * W + w) * 2 + 1];
        }
    return HS_OK;
    HS_CATCH
}

hs_status hs_keys_export_secret(hs_ctx *c, const hs_keys *k, int64_t *host_out)
{
    HS_TRY
    if (!k || !host_out) throw HsError(HS_EINVAL, "NULL argument");
    if (!k->s_ntt) throw HsError(HS_EKEY, "this key set holds no secret (hs_keys_upload)");
    memcpy(host_out, k->s_coeff.data(), k->s_coeff.size() * 8);
    (void)c;
    return HS_OK;
    HS_CATCH
}

hs_status hs_ckks_keygen_host(const hs_params *p, uint64_t seed, int h, const int32_t *galois, size_t n_galois,
                              int relin, hs_secret_key **sk, hs_public_key **pk, hs_eval_keys **evk)
{
    HS_TRY
    if (!p || !sk || !pk || !evk || (n_galois && !galois)) throw HsError(HS_EINVAL, "NULL argument");
    keygen_host(p, seed, h, galois, n_galois, relin, sk, pk, evk);
    return HS_OK;
    HS_CATCH
}

hs_status hs_keys_upload(hs_ctx *c, const hs_public_key *pk, const hs_eval_keys *evk, void *stream, hs_keys **out)
{
    HS_TRY
    if (!c || !evk || !out) throw HsError(HS_EINVAL, "NULL argument");
    activate(c);
    *out = keys_upload(c, pk, evk, S(stream));
    return HS_OK;
    HS_CATCH
}

hs_status hs_ckks_decrypt_host(const hs_secret_key *sk, const uint64_t *words, int level, int ncomp, uint64_t *out)
{
    HS_TRY
    if (!sk || !words || !out) throw HsError(HS_EINVAL, "NULL argument");
    decrypt_host(sk, words, level, ncomp, out);
    return HS_OK;
    HS_CATCH
}

hs_status hs_secret_key_export(const hs_secret_key *sk, int64_t *out)
{
    HS_TRY
    if (!sk || !out) throw HsError(HS_EINVAL, "NULL argument");
    const std::vector<int64_t> &s = secret_coeffs(sk);
    memcpy(out, s.data(), s.size() * 8);
    return HS_OK;
    HS_CATCH
}

size_t hs_eval_keys_count(const hs_eval_keys *e) { return e ? evk_count(e) : 0; }

hs_status hs_eval_keys_export(const hs_eval_keys *e, int galois, uint64_t *out)
{
    HS_TRY
    if (!e || !out) throw HsError(HS_EINVAL, "NULL argument");
    for (size_t i = 0; i < evk_count(e); i++)
        if (evk_galois(e, i) == galois) {
            const std::vector<u64> &w = evk_words(e, i);
            memcpy(out, w.data(), w.size() * 8);
            return HS_OK;
        }
    throw HsError(HS_EKEY, "no such switching key");
    HS_CATCH
}

hs_status hs_public_key_export(const hs_public_key *pk, uint64_t *out)
{
    HS_TRY
    if (!pk || !out) throw HsError(HS_EINVAL, "NULL argument");
    const std::vector<u64> &w = pk_words(pk);
    memcpy(out, w.data(), w.size() * 8);
    return HS_OK;
    HS_CATCH
}

void hs_secret_key_destroy(hs_secret_key *sk) { secret_destroy(sk); }
void hs_public_key_destroy(hs_public_key *pk) { pk_destroy(pk); }
void hs_eval_keys_destroy(hs_eval_keys *e) { evk_destroy(e); }

hs_status hs_ckks_encode(const hs_params *p, const double *re, const double *im, size_t n_slots, int level,
                         double scale, uint64_t *out)
{
    HS_TRY
    if (!p || !re || !out || n_slots != (size_t)p->n / 2 || level < 0 || level > p->L || !(scale > 0))
        throw HsError(HS_EINVAL, "encode: bad arguments (n_slots must be N/2)");
    double mx = 0;
    for (size_t i = 0; i < n_slots; i++) {
        mx = std::max(mx, std::fabs(re[i]));
        if (im) mx = std::max(mx, std::fabs(im[i]));
    }
    double logq = 0;
    for (int i = 0; i <= level; i++) logq += std::log2((double)p->prime[i]);
    if (mx > 0 && (std::log2(mx * scale) + 1 >= logq || mx * scale >= 0x1p100))
        throw HsError(HS_EOVERFLOW, "encode: |Delta v| too large for Q_level");
    hs_encode_impl(p, re, im, scale, level, out);
    return HS_OK;
    HS_CATCH
}

hs_status hs_ckks_decode(const hs_params *p, const uint64_t *q0c, double scale, double *re, double *im, size_t n_slots)
{
    HS_TRY
    if (!p || !q0c || !re || n_slots != (size_t)p->n / 2) throw HsError(HS_EINVAL, "decode: bad arguments");
    hs_decode_impl(p, q0c, scale, re, im);
    return HS_OK;
    HS_CATCH
}

// PAPER.md 94-131 packing, unified: nb = n/m blocks per
// ciphertext, stride = N0/nb; instance o, coordinate i -> ciphertext i / nb,
// slot (i % nb) stride + o.
static void check_pack(size_t L, size_t n, size_t m, size_t n0)
{
    if (!m || !n || n % m) throw HsError(HS_EINVAL, "pack: n must be a multiple of m");
    size_t nb = n / m;
    if ((nb & (nb - 1)) || nb > n0 || L > n0 / nb || L == 0) throw HsError(HS_EINVAL, "pack: sizes not divisible");
}

hs_status hs_pack(const double *x, size_t L, size_t n, size_t m, size_t n0, double *slots)
{
    HS_TRY
    check_pack(L, n, m, n0);
    size_t nb = n / m, stride = n0 / nb;
    memset(slots, 0, m * n0 * 8);
    for (size_t i = 0; i < n; i++)
        for (size_t o = 0; o < L; o++) slots[(i / nb) * n0 + (i % nb) * stride + o] = x[o * n + i];
    return HS_OK;
    HS_CATCH
}

hs_status hs_unpack(const double *slots, size_t L, size_t n, size_t m, size_t n0, double *x)
{
    HS_TRY
    check_pack(L, n, m, n0);
    size_t nb = n / m, stride = n0 / nb;
    for (size_t i = 0; i < n; i++)
        for (size_t o = 0; o < L; o++) x[o * n + i] = slots[(i / nb) * n0 + (i % nb) * stride + o];
    return HS_OK;
    HS_CATCH
}

hs_status hs_ckks_encrypt(hs_ctx *c, const hs_keys *k, const uint64_t *pt, int level, uint64_t seed,
                          uint64_t ct_index, int use_sk, void *stream, hs_ct **out)
{
    HS_TRY
    if (!c || !k || !pt || !out) throw HsError(HS_EINVAL, "NULL argument");
    activate(c);
    *out = ev_encrypt(k, pt, level, seed, ct_index, use_sk != 0, S(stream)).release();
    return HS_OK;
    HS_CATCH
}

hs_status hs_ckks_decrypt(hs_ctx *c, const hs_keys *k, const hs_ct *ct, uint64_t *host_out, void *stream)
{
    HS_TRY
    if (!c || !k || !ct || !host_out) throw HsError(HS_EINVAL, "NULL argument");
    activate(c);
    ev_decrypt(k, ct, host_out, S(stream));
    return HS_OK;
    HS_CATCH
}

hs_status hs_ct_import(hs_ctx *c, int level, int ncomp, const uint64_t *words, int on_device, void *stream,
                       hs_ct **out)
{
    HS_TRY
    if (!c || !words || !out || level < 0 || level > c->P->L || ncomp < 1 || ncomp > 3)
        throw HsError(HS_EINVAL, "ct_import: bad arguments");
    activate(c);
    CtP r = ct_new(c, level, ncomp, S(stream));
    HS_CUDA(cudaMemcpyAsync(r->d, words, r->limbs() * c->P->n * 8,
                            on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, S(stream)));
    if (!on_device) HS_CUDA(cudaStreamSynchronize(S(stream)));
    *out = r.release();
    return HS_OK;
    HS_CATCH
}

hs_status hs_ct_gather(hs_ctx *c, const hs_ct *const *cts, int n, void *stream, hs_ct **out)
{
    HS_TRY
    if (!c || !cts || !out || n < 1) throw HsError(HS_EINVAL, "ct_gather: bad arguments");
    for (int i = 0; i < n; i++)
        if (!cts[i]) throw HsError(HS_EINVAL, "ct_gather: NULL member");
    activate(c);
    *out = ct_gather(cts, n, S(stream)).release();
    return HS_OK;
    HS_CATCH
}

int hs_ct_batch(const hs_ct *ct) { return ct ? ct->batch : 0; }

hs_status hs_ct_member(hs_ctx *c, const hs_ct *batch, int i, void *stream, hs_ct **out)
{
    HS_TRY
    if (!c || !batch || !out || i < 0 || i >= batch->batch) throw HsError(HS_EINVAL, "ct_member: bad index");
    activate(c);
    *out = ct_slice(batch, i, S(stream)).release();
    return HS_OK;
    HS_CATCH
}

hs_status hs_ct_write(hs_ctx *c, hs_ct *ct, const uint64_t *words, int on_device, void *stream)
{
    HS_TRY
    if (!c || !ct || !words) throw HsError(HS_EINVAL, "ct_write: NULL argument");
    activate(c);
    HS_CUDA(cudaMemcpyAsync(ct->d, words, ct->limbs() * c->P->n * 8,
                            on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, S(stream)));
    return HS_OK;
    HS_CATCH
}

hs_status hs_ct_export(hs_ctx *c, const hs_ct *ct, uint64_t *words, int on_device, void *stream)
{
    HS_TRY
    if (!c || !ct || !words) throw HsError(HS_EINVAL, "NULL argument");
    HS_CUDA(cudaMemcpyAsync(words, ct->d, ct->limbs() * c->P->n * 8,
                            on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, S(stream)));
    if (!on_device) HS_CUDA(cudaStreamSynchronize(S(stream)));
    return HS_OK;
    HS_CATCH
}

int hs_ct_level(const hs_ct *ct) { return ct->level; }
int hs_ct_ncomp(const hs_ct *ct) { return ct->ncomp; }
void hs_ct_destroy(hs_ct *ct) { delete ct; }

hs_status hs_op(hs_ctx *c, const hs_keys *k, int op, const hs_ct *a, const hs_ct *b, double cst, int i, void *stream,
                hs_ct **out)
{
    HS_TRY
    if (!c || !a || !out) throw HsError(HS_EINVAL, "NULL argument");
    activate(c);
    cudaStream_t st = S(stream);
    CtP r;
    auto need_b = [&]() { if (!b) throw HsError(HS_EINVAL, "second operand missing"); };
    auto need_k = [&]() { if (!k) throw HsError(HS_EKEY, "keys missing"); };
    // C11: the library computes at canonical scales; an operand declared at
    // another scale (hs_ct_set_scale) cannot be combined
    if (b) check_scales(a, b);
    else check_scales(a, a);
    switch (op) {
    case HS_OP_ADD: need_b(); r = ev_add(a, b, false, st); break;
    case HS_OP_SUB: need_b(); r = ev_add(a, b, true, st); break;
    case HS_OP_MULT: need_b(); need_k(); r = ev_mult(k, a, b, st); break;
    case HS_OP_TENSOR: need_b(); r = ev_tensor(a, b, st); break;
    case HS_OP_RELIN: need_k(); r = ev_relin(k, a, st); break;
    case HS_OP_RESCALE: r = ev_rescale(a, st); break;
    case HS_OP_LEVEL_DOWN: r = ev_level_down(a, i, st); break;
    case HS_OP_MULT_CONST: r = ev_mult_const(a, cst, i, st); break;
    case HS_OP_ADD_CONST: r = ev_add_const(a, cst, st); break;
    case HS_OP_MULT_INT: r = ev_mult_int(a, i, st); break;
    case HS_OP_ROTATE: need_k(); r = ev_rotate(k, a, i, st); break;
    case HS_OP_CONJ: need_k(); r = ev_galois(k, a, 2 * c->P->n - 1, st); break;
    case HS_OP_GALOIS: need_k(); r = ev_galois(k, a, i, st); break;
    default: throw HsError(HS_EINVAL, "unknown op");
    }
    *out = r.release();
    return HS_OK;
    HS_CATCH
}

hs_status hs_mult_pt(hs_ctx *c, const hs_ct *a, const double *re, const double *im, int target, void *stream,
                     hs_ct **out)
{
    HS_TRY
    if (!c || !a || !re || !out) throw HsError(HS_EINVAL, "NULL argument");
    activate(c);
    *out = ev_mult_pt(a, re, im, target, S(stream)).release();
    return HS_OK;
    HS_CATCH
}

hs_status hs_rotate_hoisted(hs_ctx *c, const hs_keys *k, const hs_ct *a, const int32_t *rots, int n, void *stream,
                            hs_ct **out)
{
    HS_TRY
    if (!c || !k || !a || !rots || !out || n < 1 || n > HS_MAXROT) throw HsError(HS_EINVAL, "bad arguments");
    activate(c);
    cudaStream_t st = S(stream);
    std::vector<int> r(rots, rots + n);
    CtP hb = ev_rotate_hoisted(k, a, r.data(), n, st);
    std::vector<CtP> res(n);
    for (int i = 0; i < n; i++) res[i] = ct_slice(hb.get(), i, st);
    for (int i = 0; i < n; i++) out[i] = res[i].release();
    return HS_OK;
    HS_CATCH
}

hs_status hs_keyswitch(hs_ctx *c, const hs_keys *k, int galois, int level, const uint64_t *d, uint64_t *out0,
                       uint64_t *out1, void *stream)
{
    HS_TRY
    if (!c || !k || !d || !out0 || !out1 || level < 0 || level > c->P->L) throw HsError(HS_EINVAL, "bad arguments");
    const SwKey *key = k->find(galois);
    if (!key) throw HsError(HS_EKEY, "no such switching key");
    activate(c);
    ev_keyswitch(k, key, level, d, out0, out1, nullptr, nullptr, S(stream));
    return HS_OK;
    HS_CATCH
}

hs_status hs_keyswitch_partial(hs_ctx *c, const hs_keys *k, int galois, int level, const uint64_t *d, int digit_begin,
                               int digit_end, uint64_t *acc, void *stream)
{
    HS_TRY
    if (!c || !k || !d || !acc || level < 0 || level > c->P->L) throw HsError(HS_EINVAL, "bad arguments");
    const SwKey *key = k->find(galois);
    if (!key) throw HsError(HS_EKEY, "no such switching key");
    activate(c);
    ks_partial(k, key, level, d, digit_begin, digit_end, acc, S(stream));
    return HS_OK;
    HS_CATCH
}

hs_status hs_ks_acc_add(hs_ctx *c, int level, uint64_t *acc, const uint64_t *other, void *stream)
{
    HS_TRY
    if (!c || !acc || !other || level < 0 || level > c->P->L) throw HsError(HS_EINVAL, "bad arguments");
    activate(c);
    ks_acc_add(c, level, acc, other, S(stream));
    return HS_OK;
    HS_CATCH
}

static void ks_finish_to(hs_ctx *c, int level, const u64 *acc, u64 *out0, u64 *out1, cudaStream_t st)
{
    const size_t N = c->P->n, w = (size_t)(level + 1) * N;
    DBuf out(2 * w, st);
    ks_moddown(c, level, 1, acc, out.p, 2 * w, nullptr, 0, 0, st);
    HS_CUDA(cudaMemcpyAsync(out0, out.p, w * 8, cudaMemcpyDeviceToDevice, st));
    HS_CUDA(cudaMemcpyAsync(out1, out.p + w, w * 8, cudaMemcpyDeviceToDevice, st));
}

hs_status hs_keyswitch_finish(hs_ctx *c, int level, const uint64_t *acc, uint64_t *out0, uint64_t *out1, void *stream)
{
    HS_TRY
    if (!c || !acc || !out0 || !out1 || level < 0 || level > c->P->L) throw HsError(HS_EINVAL, "bad arguments");
    activate(c);
    ks_finish_to(c, level, acc, out0, out1, S(stream));
    return HS_OK;
    HS_CATCH
}

hs_status hs_keyswitch_sharded(hs_ctx *c, const hs_keys *k, int galois, int level, const uint64_t *d, int rank,
                               int world, hs_comm *comm, hs_exchange_fn exchange, void *user, uint64_t *out0,
                               uint64_t *out1, void *stream)
{
    HS_TRY
    if (!c || !k || !d || !out0 || !out1 || level < 0 || level > c->P->L || world < 1 || rank < 0 || rank >= world)
        throw HsError(HS_EINVAL, "bad arguments");
    if (world > 1 && !comm && !exchange) throw HsError(HS_EINVAL, "world > 1 needs a communicator or an exchange");
    if (comm && comm_world(comm) != world) throw HsError(HS_EINVAL, "communicator size != world");
    const SwKey *key = k->find(galois);
    if (!key) throw HsError(HS_EKEY, "no such switching key");
    activate(c);
    cudaStream_t st = S(stream);
    const hs_params *P = c->P;
    const size_t N = P->n;
    const int nl = level + 1, beta = (nl + P->alpha - 1) / P->alpha, ntg = nl + P->n_p;
    const size_t words = (size_t)2 * ntg * N;
    // rank r owns the digits [r beta / world, (r + 1) beta / world)
    const int j0 = (int)((long)rank * beta / world), j1 = (int)((long)(rank + 1) * beta / world);
    if (comm && ks_sum_fits(P, world)) {
        // uint64 sum all-reduce + mod q (exact while world * q < 2^64)
        DBuf acc(words, st);
        ks_partial(k, key, level, d, j0, j1, acc.p, st);
        comm_all_reduce_u64(comm, acc.p, words, st);
        PrimeMap pm;
        pm.n = ntg;
        for (int g = 0; g < ntg; g++) pm.p[g] = (unsigned char)(g < nl ? g : P->n_q + (g - nl));
        k_mod_pm(c, acc.p, 2 * ntg, pm, st);
        ks_finish_to(c, level, acc.p, out0, out1, st);
        c->ledger[HS_LG_KS] += 1;
        return HS_OK;
    }
    DBuf part(words, st), gathered(words * world, st);
    ks_partial(k, key, level, d, j0, j1, part.p, st);
    if (world == 1) {
        HS_CUDA(cudaMemcpyAsync(gathered.p, part.p, words * 8, cudaMemcpyDeviceToDevice, st));
    } else if (comm) {
        comm_all_gather(comm, part.p, gathered.p, words, st);
    } else if (exchange(user, part.p, gathered.p, words, st) != 0) {
        throw HsError(HS_ENCCL, "key switch: exchange callback failed");
    }
    for (int r = 1; r < world; r++) ks_acc_add(c, level, gathered.p, gathered.p + r * words, st);
    ks_finish_to(c, level, gathered.p, out0, out1, st);
    c->ledger[HS_LG_KS] += 1;
    return HS_OK;
    HS_CATCH
}

hs_status hs_ntt(hs_ctx *c, int prime_index, int n_limbs, uint64_t *data, int inverse, void *stream)
{
    HS_TRY
    if (!c || !data || prime_index < 0 || n_limbs < 1 || prime_index + n_limbs > c->P->n_q + c->P->n_p)
        throw HsError(HS_EINVAL, "ntt: bad limb range");
    activate(c);
    k_ntt(c, data, n_limbs, pmap_range(prime_index, n_limbs), inverse != 0, S(stream));
    return HS_OK;
    HS_CATCH
}

hs_status hs_cheb(hs_ctx *c, const hs_keys *k, const hs_ct *x, const hs_poly *p, double gain, void *stream,
                  hs_ct **out)
{
    HS_TRY
    if (!c || !k || !x || !p || !out) throw HsError(HS_EINVAL, "NULL argument");
    activate(c);
    *out = ev_cheb(k, x, p, gain, S(stream)).release();
    return HS_OK;
    HS_CATCH
}

int hs_cheb_depth(int deg) { return cheb_depth(deg); }

double hs_softmax_input_scale(const hs_params *p, const hs_softmax_desc *d, int level)
{
    if (!p || !d || !d->exp_poly || level < 0 || level > p->L || !(d->exp_poly->b > d->exp_poly->a)) return 0.0;
    return p->scale[level] * (2.0 / (d->exp_poly->b - d->exp_poly->a));
}

hs_status hs_softmax_encrypt_input(hs_ctx *c, const hs_keys *k, const hs_softmax_desc *d, const double *slots,
                                   int level, uint64_t seed, uint64_t ct_index, void *stream, hs_ct **out)
{
    HS_TRY
    if (!c || !k || !d || !d->exp_poly || !slots || !out) throw HsError(HS_EINVAL, "NULL argument");
    const hs_params *P = c->P;
    if (level < 0 || level > P->L || !(d->exp_poly->b > d->exp_poly->a)) throw HsError(HS_EINVAL, "bad level / exp");
    activate(c);
    cudaStream_t st = S(stream);
    const double s_in = P->scale[level] * (2.0 / (d->exp_poly->b - d->exp_poly->a));
    // one level up at scale s_in q_{level+1}, then one rescale: the fresh
    // encryption noise is divided by q_{level+1} (G28)
    const int up = level < P->L ? level + 1 : level;
    const double sc = up > level ? s_in * (double)P->prime[up] : s_in;
    std::vector<u64> pt((size_t)(up + 1) * P->n);
    hs_encode_impl(P, slots, nullptr, sc, up, pt.data());
    CtP ct = ev_encrypt(k, pt.data(), up, seed, ct_index, false, st);
    if (up > level) ct = ev_rescale(ct.get(), st);
    *out = ct.release();
    return HS_OK;
    HS_CATCH
}

hs_status hs_softmax_input_level(const hs_params *p, const hs_softmax_desc *d, size_t m_local, int bts_out_level,
                                 int *level)
{
    HS_TRY
    if (!p || !d || !level) throw HsError(HS_EINVAL, "NULL argument");
    const int top = (bts_out_level >= 0 ? bts_out_level : p->L) - 1;
    double best = HUGE_VAL;
    int pick = -1;
    for (int l = 0; l <= top; l++) {
        hs_softmax_sched s;
        try {
            softmax_schedule(p, d, l, m_local, bts_out_level, &s);
        } catch (const HsError &e) {
            if (e.code == HS_ELEVEL) continue;
            throw;
        }
        if (s.cost < best) {
            best = s.cost;
            pick = l;
        }
    }
    if (pick < 0) throw HsError(HS_ELEVEL, "no input level fits the schedule");
    *level = pick;
    return HS_OK;
    HS_CATCH
}

hs_status hs_softmax_one_ctxt(hs_ctx *c, const hs_keys *k, const hs_softmax_desc *d, const hs_ct *in, void *stream,
                              hs_ct **out)
{
    HS_TRY
    if (!c || !k || !d || !in || !out) throw HsError(HS_EINVAL, "NULL argument");
    if (d->m != 1) throw HsError(HS_EINVAL, "one_ctxt needs m = 1");
    activate(c);
    return softmax_run(c, k, d, &in, 1, S(stream), out);
    HS_CATCH
}

hs_status hs_softmax_many_ctxt(hs_ctx *c, const hs_keys *k, const hs_softmax_desc *d, const hs_ct *const *in,
                               size_t m_local, void *stream, hs_ct **out)
{
    HS_TRY
    if (!c || !k || !d || !in || !out) throw HsError(HS_EINVAL, "NULL argument");
    activate(c);
    return softmax_run(c, k, d, in, m_local, S(stream), out);
    HS_CATCH
}

hs_status hs_ct_set_scale(hs_ct *ct, double scale)
{
    HS_TRY
    if (!ct || !(scale >= 0.0)) throw HsError(HS_EINVAL, "bad ciphertext or scale");
    ct->scale = scale;
    return HS_OK;
    HS_CATCH
}

double hs_ct_scale(const hs_ct *ct)
{
    if (!ct) return 0.0;
    return ct->scale != 0.0 ? ct->scale : ct->ctx->P->scale[ct->level];
}

hs_status hs_ctx_debug_domain(hs_ctx *c, const hs_keys *k)
{
    HS_TRY
    if (!c) throw HsError(HS_EINVAL, "NULL context");
    if (k && !k->s_ntt) throw HsError(HS_EKEY, "the domain check decrypts: keys with the secret needed");
    c->debug_keys = k;
    return HS_OK;
    HS_CATCH
}

hs_status hs_softmax_schedule(const hs_params *p, const hs_softmax_desc *d, int in_level, size_t m_local,
                              int bts_out_level, hs_softmax_sched *out)
{
    HS_TRY
    if (!p || !d || !out) throw HsError(HS_EINVAL, "NULL argument");
    softmax_schedule(p, d, in_level, m_local, bts_out_level, out);
    return HS_OK;
    HS_CATCH
}

hs_status hs_softmax_choose(const hs_params *p, const hs_softmax_desc *cands, size_t n, int in_level,
                            size_t m_local, int bts_out_level, size_t *best, hs_softmax_sched *sched)
{
    HS_TRY
    if (!p || !cands || !best || n == 0) throw HsError(HS_EINVAL, "NULL argument or no candidate");
    double best_cost = HUGE_VAL;
    size_t bi = n;
    for (size_t i = 0; i < n; i++) {
        hs_softmax_sched s{};
        try {
            softmax_schedule(p, &cands[i], in_level, m_local, bts_out_level, &s);
        } catch (const HsError &e) {
            if (e.code != HS_ELEVEL) throw;
            s = hs_softmax_sched{};
            s.cost = HUGE_VAL;
        }
        if (sched) sched[i] = s;
        if (s.cost < best_cost) best_cost = s.cost, bi = i;
    }
    if (bi == n) throw HsError(HS_ELEVEL, "softmax_choose: no candidate fits the modulus chain");
    *best = bi;
    return HS_OK;
    HS_CATCH
}

}  // extern "C"

extern "C" {

hs_status hs_comm_unique_id(uint8_t uid[128])
{
    HS_TRY
    if (!uid) throw HsError(HS_EINVAL, "NULL argument");
    comm_unique_id(uid);
    return HS_OK;
    HS_CATCH
}

hs_status hs_comm_init(hs_ctx *c, int rank, int world, const uint8_t uid[128], hs_comm **out)
{
    HS_TRY
    if (!c || !uid || !out || world < 1 || rank < 0 || rank >= world) throw HsError(HS_EINVAL, "bad communicator");
    activate(c);
    *out = comm_create(rank, world, uid);
    return HS_OK;
    HS_CATCH
}

void hs_comm_destroy(hs_comm *comm) { comm_destroy(comm); }

}  // extern "C"

struct hs_plan {
    hs_ctx *c = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    std::vector<hs_ct *> outs;
    int64_t ledger_delta[HS_LG_COUNT] = {0};
    ~hs_plan()
    {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        for (hs_ct *o : outs) delete o;
    }
};

extern "C" {

hs_status hs_softmax_plan_create(hs_ctx *c, const hs_keys *k, const hs_softmax_desc *d, const hs_ct *const *in,
                                 size_t m_local, void *stream, hs_plan **out)
{
    HS_TRY
    if (!c || !k || !d || !in || !out || m_local < 1) throw HsError(HS_EINVAL, "NULL argument");
    if (d->world > 1 && !d->comm)
        throw HsError(HS_EINVAL, "plans capture a sharded Softmax only with a native communicator (hs_comm_init)");
    activate(c);
    cudaStream_t user = S(stream);
    std::unique_ptr<hs_plan> p(new hs_plan);
    p->c = c;
    std::vector<hs_ct *> tmp(m_local, nullptr);
    // 1. eager warm-up: builds every table / cached plaintext the graph reads
    const bool prof = c->kprof_on;
    c->kprof_on = false;
    int64_t led0[HS_LG_COUNT];
    memcpy(led0, c->ledger, sizeof(led0));
    hs_status s = softmax_run(c, k, d, in, m_local, user, tmp.data());
    if (s != HS_OK) return s;
    HS_CUDA(cudaStreamSynchronize(user));
    for (size_t i = 0; i < m_local; i++) {
        hs_ct *o = new hs_ct;
        o->ctx = c;
        o->level = tmp[i]->level;
        o->ncomp = tmp[i]->ncomp;
        o->batch = 1;
        o->st = user;
        o->d = dev_alloc(o->ct_words(), user);
        p->outs.push_back(o);
        delete tmp[i];
    }
    HS_CUDA(cudaStreamSynchronize(user));
    memcpy(c->ledger, led0, sizeof(led0));
    // 2. capture on a private stream (the legacy stream cannot capture)
    cudaStream_t cs;
    HS_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    c->kprof_on = prof;
    // scratch inside the graph is graph-owned: bypass the allocator hook
    alloc_capturing(true);
    struct CapOff {
        ~CapOff() { alloc_capturing(false); }
    } cap_off;
    HS_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    try {
        s = softmax_run(c, k, d, in, m_local, cs, tmp.data());
        if (s == HS_OK)
            for (size_t i = 0; i < m_local; i++) {
                HS_CUDA(cudaMemcpyAsync(p->outs[i]->d, tmp[i]->d, p->outs[i]->ct_words() * 8,
                                        cudaMemcpyDeviceToDevice, cs));
                delete tmp[i];  // stream-ordered free, inside the graph
            }
    } catch (...) {
        cudaGraph_t g;
        cudaStreamEndCapture(cs, &g);
        if (g) cudaGraphDestroy(g);
        cudaStreamDestroy(cs);
        c->kprof_on = prof;
        throw;
    }
    HS_CUDA(cudaStreamEndCapture(cs, &p->graph));
    cudaStreamDestroy(cs);
    for (int i = 0; i < HS_LG_COUNT; i++) p->ledger_delta[i] = c->ledger[i] - led0[i];
    memcpy(c->ledger, led0, sizeof(led0));
    if (s != HS_OK) return s;
    HS_CUDA(cudaGraphInstantiate(&p->exec, p->graph, 0));
    *out = p.release();
    return HS_OK;
    HS_CATCH
}

hs_status hs_plan_run(hs_plan *p, void *stream)
{
    HS_TRY
    if (!p) throw HsError(HS_EINVAL, "NULL plan");
    activate(p->c);
    HS_CUDA(cudaGraphLaunch(p->exec, S(stream)));
    for (int i = 0; i < HS_LG_COUNT; i++) p->c->ledger[i] += p->ledger_delta[i];
    return HS_OK;
    HS_CATCH
}

size_t hs_plan_n_outputs(const hs_plan *p) { return p ? p->outs.size() : 0; }
const hs_ct *hs_plan_output(const hs_plan *p, size_t i) { return p && i < p->outs.size() ? p->outs[i] : nullptr; }
void hs_plan_destroy(hs_plan *p)
{
    if (p) cudaDeviceSynchronize();
    delete p;
}

hs_status hs_bootstrap(hs_ctx *c, const hs_keys *k, hs_bts *b, const hs_ct *in, double bound, void *stream,
                       hs_ct **out)
{
    HS_TRY
    if (!c || !k || !b || !in || !out || !(bound > 0)) throw HsError(HS_EINVAL, "bad arguments");
    activate(c);
    *out = ev_bootstrap(k, b, in, bound, S(stream)).release();
    return HS_OK;
    HS_CATCH
}

hs_status hs_ledger_get(hs_ctx *c, int64_t *out, int n)
{
    if (!c || !out) return HS_EINVAL;
    for (int i = 0; i < n && i < HS_LG_COUNT; i++) out[i] = c->ledger[i];
    return HS_OK;
}

hs_status hs_ledger_reset(hs_ctx *c)
{
    if (!c) return HS_EINVAL;
    memset(c->ledger, 0, sizeof(c->ledger));
    return HS_OK;
}

}  // extern "C"
