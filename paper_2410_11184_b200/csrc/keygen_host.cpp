// keygen_host.cpp -- host-side key generation, upload and decryption
// (PAPER.md 262-271 [sec 2.2.1]: KeyGen hands sk, pk, evk and the rotation
// keys to the user; the evaluator receives only the public material).
//
// hs_ckks_keygen_host produces, on the host and from the counter-based
// ChaCha20 stream of DESIGN.md C5, exactly the words the device keygen
// (eval.cpp keys_generate) and the oracle produce: secret s (Hamming weight h,
// partial Fisher-Yates), pk = (-a s + e, a) over Q_L (C6), and switching keys
// evk_j = (-a_j s + e_j + [i in D_j] (P mod q_i) s', a_j) over Q_L u P (C7)
// for s' = s^2 (relinearisation) and s' = sigma_k(s) (Galois element k).
// hs_keys_upload builds a device key set from pk + evk only: it holds no
// secret, so the evaluating context can run every Softmax / bootstrap
// operation but not decrypt.  hs_ckks_decrypt_host decrypts exported words
// with the host secret.
#include <omp.h>

#include <algorithm>
#include <cstring>

#include "hs_internal.h"

namespace {

enum { TAG_SK = 1, TAG_PK_A = 2, TAG_PK_E = 3, TAG_KSK_A = 4, TAG_KSK_E = 5 };
const int ETA_ERR = 21;

inline u64 add_q(u64 a, u64 b, u64 q)
{
    u64 s = a + b;
    return s >= q ? s - q : s;
}
inline u64 sub_q(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
inline u64 shoup(u64 a, u64 w, u64 wsh, u64 q)
{
    u64 h = (u64)(((u128)a * wsh) >> 64);
    u64 r = a * w - h * q;
    return r >= q ? r - q : r;
}

// C3 on the host: Cooley-Tukey with the bit-reversed psi table (tw[m + i]),
// natural-order input, bit-reversed evaluation order out; the inverse is
// Gentleman-Sande with psi^-1 and a final N^-1.
void ntt_host(const hs_params *P, int pi, u64 *a, bool inverse)
{
    const int N = P->n;
    const u64 q = P->prime[pi];
    const u64 *tw = P->tw[pi].data();
    if (!inverse) {
        for (int m = 1, t = N / 2; m < N; m *= 2, t /= 2)
            for (int i = 0; i < m; i++) {
                const u64 w = tw[m + i], ws = tw[N + m + i];
                for (int j = 2 * i * t; j < 2 * i * t + t; j++) {
                    const u64 u = a[j], v = shoup(a[j + t], w, ws, q);
                    a[j] = add_q(u, v, q);
                    a[j + t] = sub_q(u, v, q);
                }
            }
    } else {
        for (int m = N / 2, t = 1; m >= 1; m /= 2, t *= 2)
            for (int i = 0; i < m; i++) {
                const u64 w = tw[2 * N + m + i], ws = tw[3 * N + m + i];
                for (int j = 2 * i * t; j < 2 * i * t + t; j++) {
                    const u64 u = a[j], v = a[j + t];
                    a[j] = add_q(u, v, q);
                    a[j + t] = shoup(sub_q(u, v, q), w, ws, q);
                }
            }
        for (int j = 0; j < N; j++) a[j] = shoup(a[j], P->n_inv[pi], P->n_inv_sh[pi], q);
    }
}

u64 signed_mod(int64_t x, u64 q)
{
    if (x >= 0) return (u64)x % q;
    u64 r = (u64)(-(x + 1)) % q;
    return q - 1 - r;
}

// C5 uniform mod q, prime index pi: sample t uses stream words 2 (pi N + t)
// and 2 (pi N + t) + 1 as w0, w1; value (w1 2^64 + w0) mod q.
void uniform_limb(const hs_params *P, u64 seed, uint32_t tag, u64 sub, int pi, u64 *out)
{
    const int N = P->n;
    const u64 q = P->prime[pi];
    uint32_t key[8] = {(uint32_t)seed, (uint32_t)(seed >> 32), tag, (uint32_t)sub, (uint32_t)(sub >> 32), 0, 0, 0};
    uint32_t nonce[3] = {0, 0, 0}, w[16];
    const u64 base = (u64)pi * N;
    for (int t = 0; t < N; t += 4) {
        hs_chacha20_block(key, (uint32_t)((base + t) >> 2), nonce, w);
        for (int s = 0; s < 4; s++) {
            const u64 w0 = (u64)w[4 * s] | ((u64)w[4 * s + 1] << 32);
            const u64 w1 = (u64)w[4 * s + 2] | ((u64)w[4 * s + 3] << 32);
            out[t + s] = (u64)((((u128)w1 << 64) | w0) % q);
        }
    }
}

// C5 centred binomial: coefficient t uses stream word t
void cbd(const hs_params *P, u64 seed, uint32_t tag, u64 sub, int eta, int64_t *out)
{
    const int N = P->n;
    uint32_t key[8] = {(uint32_t)seed, (uint32_t)(seed >> 32), tag, (uint32_t)sub, (uint32_t)(sub >> 32), 0, 0, 0};
    uint32_t nonce[3] = {0, 0, 0}, w[16];
    const u64 m = (1ull << eta) - 1;
    for (int b = 0; b < N / 8; b++) {
        hs_chacha20_block(key, (uint32_t)b, nonce, w);
        for (int s = 0; s < 8; s++) {
            const u64 x = (u64)w[2 * s] | ((u64)w[2 * s + 1] << 32);
            out[b * 8 + s] = (int64_t)__builtin_popcountll(x & m) - (int64_t)__builtin_popcountll((x >> eta) & m);
        }
    }
}

// e in NTT form over primes [0, n)
void error_ntt(const hs_params *P, u64 seed, uint32_t tag, u64 sub, int n, u64 *out)
{
    const int N = P->n;
    std::vector<int64_t> e(N);
    cbd(P, seed, tag, sub, ETA_ERR, e.data());
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; i++) {
        u64 *o = out + (size_t)i * N;
        for (int t = 0; t < N; t++) o[t] = signed_mod(e[t], P->prime[i]);
        ntt_host(P, i, o, false);
    }
}

std::vector<unsigned> galois_perm_host(const hs_params *P, int k)
{
    const int N = P->n, lg = P->log_n;
    auto brv = [lg](unsigned x) {
        unsigned r = 0;
        for (int i = 0; i < lg; i++, x >>= 1) r = (r << 1) | (x & 1);
        return r;
    };
    std::vector<unsigned> h(N);
    for (int i = 0; i < N; i++) {
        const u64 e = 2ull * brv((unsigned)i) + 1;
        h[i] = brv((unsigned)(((e * (u64)k) % (2ull * N) - 1) / 2));
    }
    return h;
}

}  // namespace

struct hs_secret_key {
    const hs_params *P;
    std::vector<int64_t> s;    // coefficients
    std::vector<u64> s_ntt;    // [n_q + n_p][N]
};
struct hs_public_key {
    const hs_params *P;
    std::vector<u64> w;        // [2][n_q][N] NTT domain: (b, a)
};
struct hs_eval_keys {
    const hs_params *P;
    std::vector<int> galois;                 // 0 = relinearisation
    std::vector<std::vector<u64>> k;         // planar [dnum][2][n_q + n_p][N]
};

static void sample_secret_host(const hs_params *P, u64 seed, int h, std::vector<int64_t> &s)
{
    const int N = P->n;
    std::vector<int> pos(N);
    for (int i = 0; i < N; i++) pos[i] = i;
    s.assign(N, 0);
    for (int i = 0; i < h; i++) {
        const u64 w = hs_stream_word(seed, TAG_SK, 0, 2 * (u64)i);
        const int j = i + (int)(w % (u64)(N - i));
        std::swap(pos[i], pos[j]);
        s[pos[i]] = (hs_stream_word(seed, TAG_SK, 0, 2 * (u64)i + 1) & 1) ? -1 : 1;
    }
}

void keygen_host(const hs_params *P, u64 seed, int h, const int32_t *galois, size_t n_galois, int relin,
                 hs_secret_key **sk_out, hs_public_key **pk_out, hs_eval_keys **evk_out)
{
    if (h < 1 || h > P->n) throw HsError(HS_EINVAL, "secret Hamming weight out of range");
    const int N = P->n, nq = P->n_q, nt = P->n_q + P->n_p;
    std::unique_ptr<hs_secret_key> sk(new hs_secret_key);
    sk->P = P;
    sample_secret_host(P, seed, h, sk->s);
    sk->s_ntt.assign((size_t)nt * N, 0);
    std::vector<u64> s_sh((size_t)nt * N);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < nt; i++) {
        u64 *o = sk->s_ntt.data() + (size_t)i * N;
        for (int t = 0; t < N; t++) o[t] = signed_mod(sk->s[t], P->prime[i]);
        ntt_host(P, i, o, false);
        for (int t = 0; t < N; t++) s_sh[(size_t)i * N + t] = hs_shoup_const(o[t], P->prime[i]);
    }
    // pk = (-a s + e, a) over Q_L (C6)
    std::unique_ptr<hs_public_key> pk(new hs_public_key);
    pk->P = P;
    pk->w.assign((size_t)2 * nq * N, 0);
    {
        u64 *b = pk->w.data(), *a = b + (size_t)nq * N;
        error_ntt(P, seed, TAG_PK_E, 0, nq, b);
#pragma omp parallel for schedule(static)
        for (int i = 0; i < nq; i++) {
            const u64 q = P->prime[i];
            u64 *ai = a + (size_t)i * N, *bi = b + (size_t)i * N;
            uniform_limb(P, seed, TAG_PK_A, 0, i, ai);
            const u64 *si = sk->s_ntt.data() + (size_t)i * N, *ss = s_sh.data() + (size_t)i * N;
            for (int t = 0; t < N; t++) bi[t] = sub_q(bi[t], shoup(ai[t], si[t], ss[t], q), q);
        }
    }
    // switching keys (C7): relin (s' = s^2) first, then one per Galois element
    std::unique_ptr<hs_eval_keys> evk(new hs_eval_keys);
    evk->P = P;
    std::vector<int> ids;
    if (relin) ids.push_back(0);
    for (size_t i = 0; i < n_galois; i++) ids.push_back(galois[i]);
    std::vector<u64> sp((size_t)nt * N);
    for (int id : ids) {
        if (id == 0) {
            for (size_t x = 0; x < sp.size(); x++)
                sp[x] = shoup(sk->s_ntt[x], sk->s_ntt[x], s_sh[x], P->prime[x / N]);
        } else {
            const std::vector<unsigned> perm = galois_perm_host(P, id);
            for (int i = 0; i < nt; i++)
                for (int t = 0; t < N; t++) sp[(size_t)i * N + t] = sk->s_ntt[(size_t)i * N + perm[t]];
        }
        std::vector<u64> key((size_t)P->dnum * 2 * nt * N);
        for (int j = 0; j < P->dnum; j++) {
            const u64 sub = (u64)id * 256 + (u64)j;
            u64 *k0 = key.data() + (size_t)(2 * j) * nt * N, *k1 = key.data() + (size_t)(2 * j + 1) * nt * N;
            error_ntt(P, seed, TAG_KSK_E, sub, nt, k0);
#pragma omp parallel for schedule(static)
            for (int i = 0; i < nt; i++) {
                const u64 q = P->prime[i];
                u64 *a = k1 + (size_t)i * N, *b = k0 + (size_t)i * N;
                uniform_limb(P, seed, TAG_KSK_A, sub, i, a);
                const u64 *si = sk->s_ntt.data() + (size_t)i * N, *ss = s_sh.data() + (size_t)i * N;
                const u64 g = (i < nq && i / P->alpha == j) ? P->p_mod_q[i] : 0;
                const u64 gs = hs_shoup_const(g, q);
                for (int t = 0; t < N; t++) {
                    u64 v = sub_q(b[t], shoup(a[t], si[t], ss[t], q), q);
                    if (g) v = add_q(v, shoup(sp[(size_t)i * N + t], g, gs, q), q);
                    b[t] = v;
                }
            }
        }
        evk->galois.push_back(id);
        evk->k.push_back(std::move(key));
    }
    *sk_out = sk.release();
    *pk_out = pk.release();
    *evk_out = evk.release();
}

// device key set from the public material only (no secret)
hs_keys *keys_upload(hs_ctx *c, const hs_public_key *pk, const hs_eval_keys *evk, cudaStream_t st)
{
    const hs_params *P = c->P;
    if (!evk || evk->P != P || (pk && pk->P != P)) throw HsError(HS_EINVAL, "keys belong to another parameter set");
    const size_t N = P->n;
    const int nt = P->n_q + P->n_p;
    std::unique_ptr<hs_keys> K(new hs_keys);
    K->ctx = c;
    if (pk) {
        K->pk = (decltype(K->pk))dev_alloc_persist(pk->w.size() * 8);
        HS_CUDA(cudaMemcpyAsync(K->pk, pk->w.data(), pk->w.size() * 8, cudaMemcpyHostToDevice, st));
    }
    const size_t words = (size_t)P->dnum * 2 * nt * N;
    DBuf planar(words, st);
    for (size_t i = 0; i < evk->k.size(); i++) {
        SwKey key;
        key.galois = evk->galois[i];
        key.k = (decltype(key.k))dev_alloc_persist(words * 8);
        HS_CUDA(cudaMemcpyAsync(planar.p, evk->k[i].data(), words * 8, cudaMemcpyHostToDevice, st));
        k_interleave2(c, planar.p, key.k, P->dnum, nt * N, st);
        K->swk.push_back(key);
    }
    HS_CUDA(cudaStreamSynchronize(st));
    return K.release();
}

// m = c0 + c1 s over the ciphertext's level+1 limbs, coefficient residues out
void decrypt_host(const hs_secret_key *sk, const u64 *words, int level, int ncomp, u64 *out)
{
    const hs_params *P = sk->P;
    const int N = P->n;
    if (level < 0 || level > P->L || ncomp < 2) throw HsError(HS_EINVAL, "decrypt: bad level / components");
#pragma omp parallel for schedule(static)
    for (int i = 0; i <= level; i++) {
        const u64 q = P->prime[i];
        const u64 *c0 = words + (size_t)i * N, *c1 = words + ((size_t)(level + 1) + i) * N;
        const u64 *s = sk->s_ntt.data() + (size_t)i * N;
        u64 *o = out + (size_t)i * N;
        for (int t = 0; t < N; t++) o[t] = add_q(c0[t], hs_mulmod(c1[t], s[t], q), q);
        if (ncomp == 3) {
            const u64 *c2 = words + ((size_t)2 * (level + 1) + i) * N;
            for (int t = 0; t < N; t++) o[t] = add_q(o[t], hs_mulmod(hs_mulmod(c2[t], s[t], q), s[t], q), q);
        }
        ntt_host(P, i, o, true);
    }
}

void host_ntt_limb(const hs_params *P, int pi, u64 *a, bool inverse) { ntt_host(P, pi, a, inverse); }

const std::vector<int64_t> &secret_coeffs(const hs_secret_key *sk) { return sk->s; }
const hs_params *secret_params(const hs_secret_key *sk) { return sk->P; }
size_t evk_count(const hs_eval_keys *e) { return e->galois.size(); }
int evk_galois(const hs_eval_keys *e, size_t i) { return e->galois.at(i); }
const std::vector<u64> &evk_words(const hs_eval_keys *e, size_t i) { return e->k.at(i); }
const std::vector<u64> &pk_words(const hs_public_key *p) { return p->w; }
void secret_destroy(hs_secret_key *s) { delete s; }
void pk_destroy(hs_public_key *p) { delete p; }
void evk_destroy(hs_eval_keys *e) { delete e; }
