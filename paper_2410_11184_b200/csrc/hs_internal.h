// hs_internal.h -- internal declarations of libhesoftmax (product side).
//
// Layers:
//   tables.cpp   host RNS tables: primes (C1), psi (C2), twiddles with Shoup
//                companions, canonical scales (C12), BConv constants
//   rng.cu       ChaCha20 counter stream + samplers on the device (C5)
//   ntt.cu       negacyclic NTT / iNTT kernels (C3)
//   kernels.cu   elementwise, tensor, automorphism, rescale, BConv, evk dot
//   eval.cu      evaluator: key switch (C7), HMult (C8), rescale (C9),
//                rotation (C10), constants (C12), keys, encrypt/decrypt
//   poly.cpp     Chebyshev BSGS evaluation (C13)
//   softmax.cpp  Alg 1 / Alg 2 / Alg B driver, packing (C14, C15)
//   encode.cpp   quad-precision canonical embedding (C4), host
//   capi.cpp     extern "C" boundary (include/hesoftmax.h)
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hesoftmax.h"

typedef uint64_t u64;
typedef unsigned __int128 u128;

#define HS_MAXP 64
#define HS_MAXDEV 64  // devices tracked by the per-device constant upload (capi.cpp)
#define HS_MAXDIG 16  // key-switch digits (ModUpBuf / KsArgB hold 16 offsets)
#define HS_MAXROT 64  // rotations served by one hoisted ModUp (C16)

// ------------------------------------------------------------------ errors
struct HsError : std::runtime_error {
    hs_status code;
    HsError(hs_status c, const std::string &m) : std::runtime_error(m), code(c) {}
};
#define HS_CUDA(x)                                                                            \
    do {                                                                                      \
        cudaError_t _e = (x);                                                                 \
        if (_e != cudaSuccess)                                                                \
            throw HsError(HS_ECUDA, std::string(#x) + ": " + cudaGetErrorString(_e));         \
    } while (0)
#define HS_CHECK_LAUNCH() HS_CUDA(cudaGetLastError())

// ------------------------------------------------------------------ per-prime constants
// Shoup: x*w mod q = x*w - hi(x*wsh)*q (+ one correction), wsh = floor(w 2^64 / q).
// Reduction of a 128-bit T < q 2^64: Montgomery REDC (qinv = -q^{-1} mod 2^64)
// gives T 2^-64 mod q, then a Shoup multiply by r64 = 2^64 mod q restores T mod q.
struct PrimeK {
    u64 q, qinv, r64, r64sh;
};

// ------------------------------------------------------------------ host parameters
struct hs_params {
    int log_n = 0, n = 0, n_q = 0, n_p = 0, L = 0, alpha = 0, dnum = 0;
    std::vector<u64> prime, psi;
    std::vector<double> scale;                 // canonical scale per level (C12)
    std::vector<PrimeK> pk;                    // per prime
    std::vector<std::vector<u64>> tw;          // per prime: [psi_rev | psi_rev_sh | ipsi_rev | ipsi_rev_sh]
    std::vector<u64> n_inv, n_inv_sh;
    std::vector<u64> p_mod_q, p_inv_mod_q;     // per Q prime
};

u64 hs_mulmod(u64 a, u64 b, u64 q);
u64 hs_powmod(u64 a, u64 e, u64 q);
u64 hs_invmod(u64 a, u64 q);
u64 hs_shoup_const(u64 w, u64 q);
u64 hs_residue_of_double(double x, u64 q);
void hs_build_params(const hs_params_desc *d, hs_params *P);
int hs_galois_elt(const hs_params *P, int r);

// ------------------------------------------------------------------ device context
struct DevTables {
    u64 *tw = nullptr;          // [nprimes][4][N]
    PrimeK *pk = nullptr;       // device copy (also in __constant__ via cudaMemcpyToSymbol)
};

struct BconvTab {               // ModUp digit (level, digit) or ModDown (level)
    int n_src = 0, n_dst = 0;
    bool centred = false;       // ModDown: centred source terms (unbiased, C7)
    std::vector<int> src, dst;  // global prime indices
    u64 *dev = nullptr;         // [n_src](inv, inv_sh) then [n_src][n_dst](c, c_sh)
    // tensor-core form (n_src <= 8, kernels.cu bconv_mma_kernel): the B-operand
    // fragments of mma.m16n8k32 u8, [n_dst][2 k-steps][32 lanes] x 2 u32
    uint32_t *mma = nullptr;
};
void bconv_build_mma(BconvTab &t, const std::vector<u64> &h, const hs_params *P);

// Allocator hook of hs_context_create_ex.  activate() makes the context's
// hook current for the calling thread; every allocation records which hook
// (if any) served it, so a free always goes back to its own allocator.
struct AllocHook {
    hs_allocator a{};
    bool on = false;
};

struct hs_ctx {
    const hs_params *P = nullptr;
    int device = 0;
    AllocHook alloc;                         // hs_context_create_ex
    DevTables T;
    std::map<long, BconvTab> bconv;          // key: (level << 8 | digit), digit 255 = ModDown
    std::map<int, unsigned *> galois_perm;   // device permutation tables
    std::map<long, u64 *> bconv_ninv;        // folded inverse-NTT scales (bconv_ninv)
    std::map<std::pair<u64, long>, u64 *> pt_cache;  // (content hash, level pair) -> NTT plaintext
    std::map<const u64 *, CUtensorMap> key_tmaps;     // TMA tensor maps of switching keys (kernels.cu)
    std::mutex mu;
    int64_t ledger[HS_LG_COUNT] = {0};
    const hs_keys *debug_keys = nullptr;  // hs_ctx_debug_domain: keys WITH the secret
    // digit-parallel key switching of single-ciphertext ops (SURVEY 8(f) rank
    // 1), switched on by the Softmax driver around its aux thread
    struct KsSplit {
        int rank = 0, world = 1, emulate = 0;  // emulate = G: every rank's share in turn
        hs_comm *comm = nullptr;
        hs_exchange_fn ex = nullptr;
        void *user = nullptr;
    } ks_split;
    bool ks_split_on = false;
    bool kprof_on = false;
    std::vector<cudaEvent_t> kprof_ev;       // pairs (start, end)
    std::vector<int> kprof_id;
    std::vector<double> kprof_bytes;
    size_t kprof_used = 0;
    ~hs_ctx();
};

struct SwKey {
    int galois = 0;
    u64 *k = nullptr;           // [dnum][n_q+n_p][N][2]: (b, a) word pairs interleaved
};

struct hs_keys {
    hs_ctx *ctx = nullptr;
    std::vector<int64_t> s_coeff;
    u64 *s_ntt = nullptr;       // [n_q+n_p][N]
    u64 *pk = nullptr;          // [2][n_q][N]
    std::vector<SwKey> swk;
    ~hs_keys();
    const SwKey *find(int galois) const {
        for (auto &k : swk)
            if (k.galois == galois) return &k;
        return nullptr;
    }
};

// One ciphertext, or a batch of `batch` ciphertexts at the same level sharing
// one allocation [batch][ncomp][level+1][N] (the main thread of the
// many-ciphertext Softmax runs its 64 ciphertexts as one batch).
struct hs_ct {
    hs_ctx *ctx = nullptr;
    int level = 0, ncomp = 0, batch = 1;
    u64 *d = nullptr;           // [batch][ncomp][level+1][N]
    cudaStream_t st = nullptr;  // stream the buffer is ordered on
    bool owns = true;           // false: a view into another ciphertext's buffer
    double scale = 0.0;         // declared encoding scale (hs_ct_set_scale); 0 = the
                                // canonical scale of its level (C11, C12)
    ~hs_ct();
    size_t rows() const { return (size_t)batch * ncomp; }
    size_t limbs() const { return rows() * (level + 1); }
    size_t ct_words() const;    // words of one ciphertext of the batch
    u64 *limb(int comp, int i) const;
    u64 *at(int b, int comp, int i) const;
};

// ------------------------------------------------------------------ memory
void alloc_hook_set(const AllocHook &h);     // thread-local current hook
void alloc_capturing(bool on);               // inside a CUDA-graph capture: bypass the hook
u64 *dev_alloc(size_t words, cudaStream_t st);   // stream-ordered
void dev_free(void *p, cudaStream_t st);
void *dev_alloc_persist(size_t bytes);           // long-lived (tables, keys, caches)
void dev_free_persist(void *p);
struct DBuf {                   // stream-ordered scratch buffer
    u64 *p = nullptr;
    cudaStream_t st = nullptr;
    DBuf() {}
    DBuf(size_t words, cudaStream_t s) : p(dev_alloc(words, s)), st(s) {}
    ~DBuf() { if (p) dev_free(p, st); }
    void alloc(size_t words, cudaStream_t s)
    {
        if (p) dev_free(p, st);
        p = dev_alloc(words, s);
        st = s;
    }
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
};

// ModUp result of the hybrid key switch (C7): digit j's extension to every
// target prime but its own, block [B][nd_j][N] at ext + off[j]
struct ModUpBuf {
    DBuf ext;
    size_t off[HS_MAXDIG];
    int nd[HS_MAXDIG];
    int beta = 0;
};

// ------------------------------------------------------------------ kernel profiling (kprof.cpp)
// When enabled, every launcher records CUDA events around its kernel on the
// launching stream plus the launch's algorithmic bytes;
// hs_kprof_collect aggregates them per kernel class.
enum { KID_NTT, KID_ADD, KID_SCALAR, KID_PTMUL, KID_TENSOR, KID_PERMUTE, KID_RESCALE, KID_BCONV, KID_KS_INNER,
       KID_MODDOWN, KID_RNG, KID_MODRAISE, KID_KS_HOIST, KID_COUNT };
struct KTimer {
    hs_ctx *c;
    int id;
    double bytes;
    cudaStream_t st;
    int slot;
    bool ext = false;  // recorded under stream capture (graph event nodes)
    KTimer(hs_ctx *c, int id, double bytes, cudaStream_t st);
    ~KTimer();
};

// ------------------------------------------------------------------ kernel launchers (kernels.cu / ntt.cu / rng.cu)
struct PrimeMap {               // prime index of limb l = p[l % n]
    int n;
    unsigned char p[256];
};
PrimeMap pmap_range(int first, int count);

// ninv (optional, inverse only): per-prime (scale, Shoup) pairs replacing N^-1 --
// the BConv's q-hat^-1 folded into the inverse transform (bconv_ninv)
void k_ntt(hs_ctx *c, u64 *data, int n_limbs, const PrimeMap &pm, bool inverse, cudaStream_t st,
           const u64 *ninv = nullptr);
void k_ntt_inv_from(hs_ctx *c, u64 *dst, const u64 *src, size_t sstr, int srows, int n_limbs, const PrimeMap &pm,
                    cudaStream_t st, const u64 *ninv = nullptr);
void k_add(hs_ctx *c, const u64 *a, const u64 *b, u64 *o, int n_limbs, int period, bool sub, cudaStream_t st);
void k_neg(hs_ctx *c, const u64 *a, u64 *o, int n_limbs, int period, cudaStream_t st);
void k_mul_scalar(hs_ctx *c, const u64 *a, u64 *o, const u64 *host_scal, int n_limbs, int period, cudaStream_t st);
void k_add_scalar(hs_ctx *c, u64 *a, const u64 *host_scal, int n_limbs, cudaStream_t st);
void k_mul_pointwise(hs_ctx *c, const u64 *a, const u64 *b, u64 *o, int n_limbs, int period_a, int period_b,
                     cudaStream_t st);
void k_mac_scalar(hs_ctx *c, u64 *acc, const u64 *a, const u64 *host_scal, int n_limbs, int period, cudaStream_t st);
void k_tensor(hs_ctx *c, const u64 *a, const u64 *b, u64 *o, int nl, cudaStream_t st);
void k_permute(hs_ctx *c, const u64 *a, u64 *o, const unsigned *perm, int n_limbs, cudaStream_t st);
void k_rescale_prep(hs_ctx *c, const u64 *last, u64 *w, int ncomp, int level, cudaStream_t st);
void k_rescale_final(hs_ctx *c, const u64 *a, const u64 *w, u64 *o, int ncomp, int level, cudaStream_t st);
// prescaled: the sources already hold [x_a qhat_a^-1]_{q_a} (inverse NTT with
// the tables' bconv_ninv), so the conversion skips that first step
void k_bconv(hs_ctx *c, const BconvTab &tab, const u64 *src, size_t src_stride, u64 *dst, size_t dst_stride,
             int batch, size_t batch_src_stride, size_t batch_dst_stride, cudaStream_t st, bool prescaled = false);
void k_bconv_modup_multi(hs_ctx *c, const BconvTab *const *tabs, const size_t *dst_off, int n_dig, const u64 *x,
                         u64 *o, cudaStream_t st, bool prescaled = false);
// [n_q + n_p] (N^-1 qhat_a^-1 mod q_a, Shoup) for the sources of the given
// tables (other entries 0): the inverse-NTT scale that leaves the BConv input
// prescaled; cached per (kind, level)
const u64 *bconv_ninv(hs_ctx *c, const BconvTab *const *tabs, int n_tabs, long key);
void k_ks_inner(hs_ctx *c, const u64 *d, const u64 *ext, const u64 *key, u64 *acc, int level, int beta,
                cudaStream_t st);
void k_moddown_final(hs_ctx *c, const u64 *acc, const u64 *conv, u64 *o0, u64 *o1, const u64 *add0,
                     const u64 *add1, int level, cudaStream_t st);
void upload_prime_constants(const hs_params *P);
bool ntt_fp_enabled();  // FP64 NTT path for primes < 2^43 (HS_NTT_FP=0: off)
bool k_ntt_rescale(hs_ctx *c, const u64 *last, u64 *w, const u64 *a, u64 *o, int rows, int l, cudaStream_t st,
                   const u64 *scal = nullptr, size_t a_row = 0);
bool k_ntt_moddown(hs_ctx *c, u64 *conv, const u64 *acc, size_t acc_row, u64 *o, size_t o_stride, const u64 *add,
                   size_t add_stride, int add_comps, int nt, const u64 *inv, int rows, cudaStream_t st);
void k_mul_scalar_pm(hs_ctx *c, const u64 *a, u64 *o, const u64 *host_scal, int n_limbs, const PrimeMap &pm,
                     cudaStream_t st);
void k_add_pm(hs_ctx *c, const u64 *a, const u64 *b, u64 *o, int n_limbs, const PrimeMap &pm, cudaStream_t st);
void k_bsgs_inner(hs_ctx *c, const u64 *const *R, int b1, const u64 *pts, const int *tk, int G, int nl, u64 *out,
                  cudaStream_t st, int nlq = -1);
void k_mac_pt(hs_ctx *c, u64 *acc, const u64 *a, const u64 *pt, int nl, int la, cudaStream_t st);
// batched ciphertext kernels ([B][ncomp][nl][N]; "rows" = B * ncomp)
void k_add_b(hs_ctx *c, const u64 *a, int a_rows, const u64 *b, int b_rows, u64 *o, int rows, int nl, bool sub,
             cudaStream_t st);
void k_mul_scalar_s(hs_ctx *c, const u64 *a, u64 *o, const u64 *host_scal, int rows, int nl, int a_rl, int o_rl,
                    bool accumulate, cudaStream_t st);
void k_add_scalar_b(hs_ctx *c, u64 *a, const u64 *host_scal, int B, int ncomp, int nl, cudaStream_t st);
// o[d][w][c] = planar[d][c][w]: [D][2][W] -> [D][W][2] (switching-key layout)
void k_interleave2(hs_ctx *c, const u64 *planar, u64 *o, int D, size_t W, cudaStream_t st);
void k_lin_comb(hs_ctx *c, const u64 *const *a, const int *a_rl, const u64 *const *host_scal, int n_terms, u64 *o,
                int rows, int nl, int o_rl, bool accumulate, cudaStream_t st);
void k_tensor_b(hs_ctx *c, const u64 *a, const u64 *b, u64 *o, int B, int nl, int b_batch, cudaStream_t st);
void k_tensor_sum(hs_ctx *c, const u64 *a, u64 *o, int B, int nl, cudaStream_t st);
void k_tensor_sum2(hs_ctx *c, const u64 *a, const u64 *b, u64 *o, int B, int nl, cudaStream_t st);
void k_ks_inner_b(hs_ctx *c, const u64 *d, size_t d_stride, const u64 *ext, const size_t *off, const int *nd,
                  const u64 *key, u64 *acc, int level, int beta, int B, cudaStream_t st, const u64 *dadd = nullptr,
                  size_t dadd_stride = 0, int j0 = 0);
void k_ks_inner_m(hs_ctx *c, const u64 *d, size_t d_stride, const u64 *ext, const size_t *off, const int *nd,
                  const u64 *const *keys, int B, u64 *acc, int level, int beta, cudaStream_t st);
void k_ks_inner_h(hs_ctx *c, const u64 *d, const u64 *ext, const size_t *off, const int *nd, const u64 *const *keys,
                  const unsigned *const *perms, int R, u64 *acc, int level, int beta, cudaStream_t st,
                  const u64 *c0add = nullptr);
void k_moddown_final_b(hs_ctx *c, const u64 *acc, size_t acc_row, const u64 *conv, int nt, u64 *o, size_t o_stride,
                       const u64 *add, size_t add_stride, int add_comps, const u64 *inv, int rows, cudaStream_t st);
void k_modraise(hs_ctx *c, const u64 *x, u64 *o, int nl, cudaStream_t st);
void k_signed_to_rns(hs_ctx *c, const int64_t *v, u64 *o, int n_limbs, const PrimeMap &pm, cudaStream_t st);
void k_uniform(hs_ctx *c, u64 *o, int n_limbs, const PrimeMap &pm, u64 seed, uint32_t tag, u64 sub,
               int limb_index0, cudaStream_t st);
void k_cbd(hs_ctx *c, int64_t *o, u64 seed, uint32_t tag, u64 sub, int eta, cudaStream_t st);

const BconvTab &bconv_modup(hs_ctx *c, int level, int digit);
const BconvTab &bconv_moddown(hs_ctx *c, int level);
const unsigned *galois_table(hs_ctx *c, int k);
void count_kernel(hs_ctx *c, int n = 1);

// host ChaCha20 (C5) for the sequential secret sampler
void hs_chacha20_block(const uint32_t key[8], uint32_t counter, const uint32_t nonce[3], uint32_t out[16]);
u64 hs_stream_word(u64 seed, uint32_t tag, u64 sub, u64 idx);

// ------------------------------------------------------------------ evaluator (eval.cu)
typedef std::unique_ptr<hs_ct> CtP;
CtP ct_new(hs_ctx *c, int level, int ncomp, cudaStream_t st, int batch = 1);
CtP ct_copy(const hs_ct *a, cudaStream_t st);
CtP ct_drop(const hs_ct *a, int level, cudaStream_t st);
CtP ct_gather(const hs_ct *const *cts, int n, cudaStream_t st);        // n single cts -> one batch
CtP ct_view(const hs_ct *a, int b);
CtP ct_slice(const hs_ct *a, int b, cudaStream_t st);                  // ciphertext b of a batch
CtP ev_tensor_sum(const hs_ct *a, cudaStream_t st);                     // sum_b tensor(a_b, a_b)
CtP ev_tensor_sum2(const hs_ct *a, const hs_ct *b, cudaStream_t st);    // sum_b tensor(a_b, b_b)
void ev_keyswitch_b(const hs_keys *K, const SwKey *key, int level, int B, const u64 *d, size_t d_stride, u64 *out,
                    size_t out_stride, const u64 *add, size_t add_stride, int add_comps, cudaStream_t st);
CtP ev_add(const hs_ct *a, const hs_ct *b, bool sub, cudaStream_t st);
CtP ev_level_down(const hs_ct *a, int target, cudaStream_t st);
CtP ev_rescale(const hs_ct *a, cudaStream_t st);
CtP ev_tensor(const hs_ct *a, const hs_ct *b, cudaStream_t st);
CtP ev_relin(const hs_keys *K, const hs_ct *d, cudaStream_t st);
CtP ev_mult(const hs_keys *K, const hs_ct *a, const hs_ct *b, cudaStream_t st);
CtP ev_mult_int(const hs_ct *a, int64_t v, cudaStream_t st);
CtP ev_add_const(const hs_ct *a, double v, cudaStream_t st);
CtP ev_mult_const(const hs_ct *a, double v, int target, cudaStream_t st);
CtP ev_mult_pt(const hs_ct *a, const double *re, const double *im, int target, cudaStream_t st);
CtP ev_galois(const hs_keys *K, const hs_ct *a, int k, cudaStream_t st);
CtP ev_rotate(const hs_keys *K, const hs_ct *a, int r, cudaStream_t st);
CtP ev_rotate_multi(const hs_keys *K, const hs_ct *a, const int *rots, cudaStream_t st);
CtP ev_rotate_hoisted(const hs_keys *K, const hs_ct *a, const int *rots, int R, cudaStream_t st);
void ks_modup(hs_ctx *c, int level, int B, const u64 *d, size_t d_stride, ModUpBuf &m, cudaStream_t st);
void ks_moddown_rescale(hs_ctx *c, int level, int B, const u64 *acc, u64 *out, size_t out_stride, cudaStream_t st);
const BconvTab &bconv_moddown_rescale(hs_ctx *c, int level);
CtP ev_relin_rescale(const hs_keys *K, const hs_ct *d, cudaStream_t st);
// digit-parallel key switch: ModUp + inner product of
// the digits [j0, j1) only -> acc [2][ntg][N]; acc += other (mod q, basis Q_l u P)
void ks_partial(const hs_keys *K, const SwKey *key, int level, const u64 *d, int j0, int j1, u64 *acc,
                cudaStream_t st, const u64 *dadd = nullptr, size_t dadd_stride = 0);
// the full accumulator of one key switch through the context's active split
// (this rank's digits + all-gather + rank-order sum, or emulated)
void ks_split_acc(hs_ctx *c, const hs_keys *K, const SwKey *key, int level, const u64 *d, const u64 *dadd,
                  size_t dadd_stride, u64 *acc, cudaStream_t st);
void ks_acc_add(hs_ctx *c, int level, u64 *acc, const u64 *other, cudaStream_t st);
void ks_moddown(hs_ctx *c, int level, int B, const u64 *acc, u64 *out, size_t out_stride, const u64 *add,
                size_t add_stride, int add_comps, cudaStream_t st);
void ev_keyswitch(const hs_keys *K, const SwKey *key, int level, const u64 *d, u64 *out0, u64 *out1,
                  const u64 *add0, const u64 *add1, cudaStream_t st);
CtP ev_mult_const_sum(const std::vector<const hs_ct *> &terms, const std::vector<double> &coef, int target,
                      cudaStream_t st);

// keys / enc / dec
hs_keys *keys_generate(hs_ctx *c, u64 seed, int h, const int32_t *galois, size_t n_galois, int relin,
                       cudaStream_t st);
CtP ev_encrypt(const hs_keys *K, const u64 *pt_host, int level, u64 seed, u64 idx, bool use_sk, cudaStream_t st);
void ev_decrypt(const hs_keys *K, const hs_ct *ct, u64 *host_out, cudaStream_t st);

// keygen_host.cpp (host KeyGen, upload, host decryption)
void keygen_host(const hs_params *P, u64 seed, int h, const int32_t *galois, size_t n_galois, int relin,
                 hs_secret_key **sk, hs_public_key **pk, hs_eval_keys **evk);
hs_keys *keys_upload(hs_ctx *c, const hs_public_key *pk, const hs_eval_keys *evk, cudaStream_t st);
void decrypt_host(const hs_secret_key *sk, const u64 *words, int level, int ncomp, u64 *out);
void host_ntt_limb(const hs_params *P, int pi, u64 *a, bool inverse);
const std::vector<int64_t> &secret_coeffs(const hs_secret_key *sk);
const hs_params *secret_params(const hs_secret_key *sk);
size_t evk_count(const hs_eval_keys *e);
int evk_galois(const hs_eval_keys *e, size_t i);
const std::vector<u64> &evk_words(const hs_eval_keys *e, size_t i);
const std::vector<u64> &pk_words(const hs_public_key *p);
void secret_destroy(hs_secret_key *s);
void pk_destroy(hs_public_key *p);
void evk_destroy(hs_eval_keys *e);

// encode.cpp
void hs_encode_impl(const hs_params *P, const double *re, const double *im, double scale, int level, u64 *out);
void hs_encode_impl_q(const hs_params *P, const __float128 *re, const __float128 *im, double scale, int level,
                      u64 *out, bool with_p = false);
void hs_decode_impl(const hs_params *P, const u64 *q0_coeffs, double scale, double *re, double *im);

// poly.cpp
CtP ev_cheb(const hs_keys *K, const hs_ct *w, const hs_poly *p, double gain, cudaStream_t st);
int cheb_depth(int deg);

// bts.cpp
CtP ev_bootstrap(const hs_keys *K, hs_bts *B, const hs_ct *in, double bound, cudaStream_t st);
int bts_exponent(const hs_params *P, int arcsine, double bound);
int bts_rotations(const hs_params *P, int n_cts, int n_stc, int32_t *out, int max);

// softmax.cpp
// comm.cpp: NCCL (dlopen'ed) for the sharded aux sum
void comm_unique_id(uint8_t uid[128]);
hs_comm *comm_create(int rank, int world, const uint8_t uid[128]);
void comm_destroy(hs_comm *comm);
int comm_world(const hs_comm *c);
void comm_all_gather(const hs_comm *c, const u64 *partial, u64 *gathered, size_t words, cudaStream_t st);
void comm_all_reduce_u64(const hs_comm *c, u64 *buf, size_t words, cudaStream_t st);
// x <- x mod q limb by limb (x < 2^64; prime of limb l = pm.p[l % pm.n])
void k_mod_pm(hs_ctx *c, u64 *a, int n_limbs, const PrimeMap &pm, cudaStream_t st);
// true when a uint64 sum of world accumulators stays below 2^64 (then an
// NCCL all-reduce + mod q replaces the all-gather of the digit split)
bool ks_sum_fits(const hs_params *P, int world);
void check_scales(const hs_ct *a, const hs_ct *b);  // C11: HS_ESCALE on a mismatch
hs_status softmax_run(hs_ctx *c, const hs_keys *K, const hs_softmax_desc *d, const hs_ct *const *in,
                      size_t m_local, cudaStream_t st, hs_ct **out);
void softmax_schedule(const hs_params *P, const hs_softmax_desc *d, int in_level, size_t m_local, int bts_out_level,
                      hs_softmax_sched *s);
