/*
 * hesoftmax.h -- C ABI of the B200-native RNS-CKKS Softmax library
 * (libhesoftmax.so, built from paper_2410_11184_b200/csrc).
 *
 * The calls follow the paper's problem statement (arXiv 2410.11184,
 * PAPER.md):
 *   - CKKS functionalities KeyGen / Enc / Dec / Add / Mult / Rot
 *     (PAPER.md 262-271, sec 2.2.1);
 *   - Softmax of x in [-M, 0]^n with parameter k (PAPER.md 688-691, 776-787);
 *   - L Softmax packed in one ciphertext (PAPER.md 94-111, sec 4.1) or in m
 *     ciphertexts with one shared auxiliary ciphertext (PAPER.md 113-131,
 *     sec 4.2), Alg 1 or version B (PAPER.md 168-181).
 * Every convention the paper leaves open (primes, NTT order, randomness,
 * key switching, rescale rounding, scales, polynomial evaluation tree,
 * schedule) is fixed in DESIGN.md (C1-C15, G1-G23); results are
 * word-for-word identical to the CPU oracle under those conventions.
 *
 * Conventions of this header:
 *   - No C++ exception crosses the ABI; every call returns hs_status.
 *     On failure hs_last_error() (thread-local) describes the cause and
 *     *out parameters are left untouched.
 *   - Handles are opaque and freed by the matching *_destroy (NULL is a no-op).
 *   - "stream" is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  Device work is enqueued on it; calls that return host data
 *     synchronise that stream.
 *   - Ciphertext words are uint64 residues in [0, q_i), limb-major
 *     [component][limb][N], NTT (evaluation) domain: limb i of a level-l
 *     ciphertext is reduced mod q_i, i = 0..l.
 *   - Plaintext words (encode output, decrypt output) are coefficient-domain
 *     residues [limb][N].
 *   - The scale of a ciphertext is implicit: the canonical scale of its
 *     level (C12, hs_params_scale).
 */
#ifndef HESOFTMAX_H
#define HESOFTMAX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HS_OK = 0,
    HS_EINVAL = 1,     /* bad argument, inconsistent sizes, packing not divisible */
    HS_ELEVEL = 2,     /* the planned schedule does not fit the modulus chain     */
    HS_EKEY = 3,       /* a required rotation / relinearisation key is missing    */
    HS_ESCALE = 4,     /* scale mismatch                                          */
    HS_EOVERFLOW = 5,  /* |round(Delta v)| too large for the modulus              */
    HS_EDOMAIN = 6,    /* debug: decrypted intermediate outside its interval       */
    HS_ENOMEM = 7,
    HS_ECUDA = 8,
    HS_ENCCL = 9       /* collective failure (exchange callback or NCCL)          */
} hs_status;

typedef struct hs_params hs_params;   /* host tables (primes, twiddles, BConv)  */
typedef struct hs_ctx hs_ctx;         /* one GPU: device tables, pools, ledger  */
typedef struct hs_keys hs_keys;       /* device key set (public + evaluation keys,
                                         and the secret only when generated on the
                                         device by hs_ckks_keygen)              */
typedef struct hs_secret_key hs_secret_key; /* host: the client's secret s         */
typedef struct hs_public_key hs_public_key; /* host: pk = (-a s + e, a)            */
typedef struct hs_eval_keys hs_eval_keys;   /* host: relinearisation + Galois keys */
typedef struct hs_ct hs_ct;           /* a device ciphertext                    */

/* Last error message of the calling thread ("" if none). */
const char *hs_last_error(void);

/* ------------------------------------------------------------ parameters */
/* q_bits[l]: bit size of q_l (sized primes) or the target size (derived
 * primes); p_bits[k]: special primes; alpha: primes per key-switching digit;
 * log2_anchor[l] != 0 pins Delta_l = 2^anchor (top level must be anchored).
 * Prime selection is DESIGN.md C1, psi C2, canonical scales C12.
 * HS_EINVAL if sizes are inconsistent or no prime can be found. */
typedef struct {
    int log_n;
    int n_q;
    const int *q_bits;
    int n_p;
    const int *p_bits;
    int alpha;
    const int *log2_anchor;
} hs_params_desc;

hs_status hs_ckks_params(const hs_params_desc *d, hs_params **out);
void hs_params_destroy(hs_params *p);
int hs_params_log_n(const hs_params *p);
int hs_params_n_q(const hs_params *p);
int hs_params_n_p(const hs_params *p);
/* out: n_q + n_p primes, Q primes first. */
hs_status hs_params_primes(const hs_params *p, uint64_t *out);
uint64_t hs_params_psi(const hs_params *p, int prime_index);
double hs_params_scale(const hs_params *p, int level);
/* Galois element 5^r mod 2N of a left rotation by r slots (G1). */
int hs_galois_of_rot(const hs_params *p, int r);

/* ------------------------------------------------------------ context */
/* One GPU context: uploads the twiddle tables of p to `device`.  Device
 * memory comes from the device's default stream-ordered pool
 * (cudaMallocAsync / cudaMalloc).  HS_EINVAL: NULL argument or no such
 * device; HS_ECUDA / HS_ENOMEM from the runtime.  p must outlive the context. */
hs_status hs_context_create(const hs_params *p, int device, hs_ctx **out);

/* Allocator hook ("library-owned device memory goes through
 * alloc", e.g. bound to torch's caching allocator so that the library and
 * the framework around it share one pool).
 *   alloc(bytes, stream, user): return device memory of >= bytes usable in
 *     stream order on `stream` (a cudaStream_t as void*, NULL = legacy
 *     default stream), or NULL on failure (the call then fails with
 *     HS_ENOMEM).  Long-lived objects (twiddle / BConv / Galois tables,
 *     keys, cached plaintexts, bootstrap transforms) are allocated with
 *     stream NULL and freed only after a device synchronisation.
 *   free(ptr, bytes, stream, user): release ptr in stream order on `stream`
 *     (the stream of the last use the library knows of).
 * Every object created under the context (keys, ciphertexts, plans' input
 * and output ciphertexts, bootstrap caches) allocates through the hook.
 * Exception: scratch memory of work captured into a CUDA graph
 * (hs_softmax_plan_create) is graph-owned (cudaMallocAsync memory nodes) and
 * never reaches the hook.  The hook struct is copied; its functions must stay
 * callable until the last object allocated through them is destroyed, and
 * must not call back into this library.  alloc == NULL selects the default
 * pool (same as hs_context_create).  Errors as hs_context_create;
 * HS_EINVAL when exactly one of alloc / free is NULL. */
typedef struct hs_allocator {
    void *(*alloc)(size_t bytes, void *stream, void *user);
    void (*free)(void *ptr, size_t bytes, void *stream, void *user);
    void *user;
} hs_allocator;
hs_status hs_context_create_ex(const hs_params *p, int device, const hs_allocator *alloc, hs_ctx **out);
void hs_context_destroy(hs_ctx *c);

/* ------------------------------------------------------------ keys (C5-C7) */
/* Client / server split (PAPER.md 262-271 [sec 2.2.1]: KeyGen(lambda, S) ->
 * pk, sk, evk, rotation keys; Enc, Dec with sk; Mult / Rot with evk).
 *
 * hs_ckks_keygen_host runs KeyGen on the HOST (no device, thread-safe), from
 * the counter-based ChaCha20 stream of DESIGN.md C5 keyed by `seed`: secret s
 * of Hamming weight h (C5), pk = (-a s + e, a) over Q_L (C6), and the
 * switching keys of C7 -- relinearisation (s' = s^2) if relin != 0, then one
 * per Galois element galois[0..n_galois) (s' = sigma_k(s)).  The words equal
 * those of hs_ckks_keygen and of the oracle for the same seed.  Outputs are
 * host objects owned by the caller (hs_*_destroy).  HS_EINVAL if h is not in
 * [1, N] or a pointer is NULL.
 *
 * hs_keys_upload builds a device key set from pk (nullable: then no public-key
 * encryption) and evk only: it holds NO secret -- hs_ckks_decrypt, secret-key
 * encryption and hs_keys_export_secret return HS_EKEY on it -- and serves every
 * evaluation (scheme ops, bootstrapping, Softmax).  Synchronous; the host
 * objects may be destroyed afterwards.  HS_EINVAL if they belong to another
 * parameter set.
 *
 * hs_ckks_decrypt_host: words = ncomp x (level+1) x N ciphertext words (NTT
 * domain, host, e.g. from hs_ct_export), out = (level+1) x N coefficient
 * residues of c0 + c1 s (+ c2 s^2 when ncomp = 3).  Host only. */
hs_status hs_ckks_keygen_host(const hs_params *p, uint64_t seed, int h, const int32_t *galois, size_t n_galois,
                              int relin, hs_secret_key **sk, hs_public_key **pk, hs_eval_keys **evk);
hs_status hs_keys_upload(hs_ctx *c, const hs_public_key *pk, const hs_eval_keys *evk, void *stream,
                         hs_keys **out);
hs_status hs_ckks_decrypt_host(const hs_secret_key *sk, const uint64_t *words, int level, int ncomp,
                               uint64_t *out);
/* test hooks on the host objects: secret coefficients (N int64); number of
 * switching keys; switching key of Galois element `galois` (0 = relin) as
 * planar [dnum][2][n_q+n_p][N] (HS_EKEY if absent); pk words [2][n_q][N]. */
hs_status hs_secret_key_export(const hs_secret_key *sk, int64_t *out);
size_t hs_eval_keys_count(const hs_eval_keys *e);
hs_status hs_eval_keys_export(const hs_eval_keys *e, int galois, uint64_t *out);
hs_status hs_public_key_export(const hs_public_key *pk, uint64_t *out);
void hs_secret_key_destroy(hs_secret_key *sk);
void hs_public_key_destroy(hs_public_key *pk);
void hs_eval_keys_destroy(hs_eval_keys *e);

/* Device keygen (tests and benches: one call builds a full key set, secret
 * included, on the evaluating GPU): the same words as hs_ckks_keygen_host.
 * Immutable after creation. */
hs_status hs_ckks_keygen(hs_ctx *c, uint64_t seed, int h, const int32_t *galois, size_t n_galois,
                         int relin, void *stream, hs_keys **out);
void hs_keys_destroy(hs_keys *k);
/* Test hooks: copy a switching key ([dnum][2][n_q+n_p][N], galois 0 = relin)
 * or the secret (N int64 coefficients) to host memory.  HS_EKEY if absent. */
hs_status hs_keys_export_swk(hs_ctx *c, const hs_keys *k, int galois, uint64_t *host_out);
hs_status hs_keys_export_secret(hs_ctx *c, const hs_keys *k, int64_t *host_out);

/* ------------------------------------------------------------ encode / decode (C4) */
/* Canonical-embedding encode of n_slots = N/2 complex slots (im may be NULL)
 * at `scale`, coefficients rounded half-even from a quad-precision
 * evaluation; out = (level+1) x N coefficient residues (host). */
hs_status hs_ckks_encode(const hs_params *p, const double *re, const double *im, size_t n_slots,
                         int level, double scale, uint64_t *out);
/* Decode the q_0 residues (N coefficients, centred) at `scale`. */
hs_status hs_ckks_decode(const hs_params *p, const uint64_t *q0_coeffs, double scale, double *re,
                         double *im, size_t n_slots);
/* Packing (PAPER.md 94-131): x[L][n] (row-major) into m
 * slot vectors of N0 = N/2 (row-major [m][N0]); padding lanes hold x = 0 (G9).
 * HS_EINVAL unless n % m == 0, n/m a power of two <= N0 and L <= N0 m / n. */
hs_status hs_pack(const double *x, size_t L, size_t n, size_t m, size_t n0, double *slots);
hs_status hs_unpack(const double *slots, size_t L, size_t n, size_t m, size_t n0, double *x);

/* ------------------------------------------------------------ encrypt / decrypt (C6) */
/* pt: (level+1) x N coefficient residues in host memory.  use_sk != 0 selects
 * secret-key encryption (tests).  Randomness: C5 stream keyed by (seed,
 * ct_index). */
hs_status hs_ckks_encrypt(hs_ctx *c, const hs_keys *k, const uint64_t *pt, int level, uint64_t seed,
                          uint64_t ct_index, int use_sk, void *stream, hs_ct **out);
/* m = c0 + c1 s (coefficient residues, (level+1) x N, host). */
hs_status hs_ckks_decrypt(hs_ctx *c, const hs_keys *k, const hs_ct *ct, uint64_t *host_out, void *stream);

/* ------------------------------------------------------------ ciphertexts */
/* words: ncomp x (level+1) x N uint64, on the device if on_device else host. */
hs_status hs_ct_import(hs_ctx *c, int level, int ncomp, const uint64_t *words, int on_device, void *stream,
                       hs_ct **out);
hs_status hs_ct_export(hs_ctx *c, const hs_ct *ct, uint64_t *words, int on_device, void *stream);
/* Overwrite an existing ciphertext's words (same layout as import) with a
 * stream-ordered copy; no synchronisation: host words must stay valid until
 * the stream passes this point (pinned memory makes the copy asynchronous).
 * Used to refresh a plan's bound inputs. */
hs_status hs_ct_write(hs_ctx *c, hs_ct *ct, const uint64_t *words, int on_device, void *stream);
/* Batched ciphertexts: n ciphertexts of one level and shape copied into ONE
 * batch handle ([n][ncomp][level+1][N]); every hs_op on a batch runs each
 * kernel once over all members (key switches read each evaluation-key limb
 * once per batch tile) and a batch-1 operand broadcasts against a batch.
 * hs_ct_batch returns the member count; hs_ct_member copies member i out. */
hs_status hs_ct_gather(hs_ctx *c, const hs_ct *const *cts, int n, void *stream, hs_ct **out);
int hs_ct_batch(const hs_ct *ct);
hs_status hs_ct_member(hs_ctx *c, const hs_ct *batch, int i, void *stream, hs_ct **out);
int hs_ct_level(const hs_ct *ct);
/* Declared encoding scale (C11).  The library computes at the canonical scale
 * Delta_level of every level (C12) and ciphertexts carry no scale of their
 * own; a caller that encoded a ciphertext at another scale declares it here
 * (0 = canonical, the default).  hs_op returns HS_ESCALE for an operand
 * declared at a scale other than Delta_level (relative 2^-40, C11); the
 * Softmax entry points return HS_ESCALE for an input declared at a scale other
 * than hs_softmax_input_scale.  hs_ct_scale returns the declared scale, else
 * Delta_level. */
hs_status hs_ct_set_scale(hs_ct *ct, double scale);
double hs_ct_scale(const hs_ct *ct);
int hs_ct_ncomp(const hs_ct *ct);
void hs_ct_destroy(hs_ct *ct);

/* ------------------------------------------------------------ scheme operations */
typedef enum {
    HS_OP_ADD = 0, HS_OP_SUB = 1,
    HS_OP_MULT = 2,        /* tensor -> relin -> rescale (C8)                    */
    HS_OP_TENSOR = 3, HS_OP_RELIN = 4, HS_OP_RESCALE = 5,
    HS_OP_LEVEL_DOWN = 6,  /* i = target level (C12 landing)                      */
    HS_OP_MULT_CONST = 7,  /* c = real constant, i = target level                 */
    HS_OP_ADD_CONST = 8,   /* c = real constant                                   */
    HS_OP_MULT_INT = 9,    /* i = integer                                         */
    HS_OP_ROTATE = 10,     /* i = left rotation (G1)                              */
    HS_OP_CONJ = 11,
    HS_OP_GALOIS = 12      /* i = Galois element                                  */
} hs_op_code;

hs_status hs_op(hs_ctx *c, const hs_keys *k, int op, const hs_ct *a, const hs_ct *b, double cst, int i,
                void *stream, hs_ct **out);
/* C16 hoisted rotations (C16; Halevi-Shoup hoisting, used by the
 * bootstrapping linear transforms' baby steps): out[r] = Rot(a, rots[r]) for
 * r < n (1 <= n <= 64), all computed from ONE ModUp of a's c1.  Each output
 * decrypts like hs_op(HS_OP_ROTATE) but its words differ (bit-exact with the
 * oracle's orc_op_rotate_hoisted, not with a plain rotation).  a: one
 * degree-1 ciphertext; out[]: n new ciphertexts owned by the caller
 * (hs_ct_destroy).  HS_EKEY if a rotation key is missing (no output written). */
hs_status hs_rotate_hoisted(hs_ctx *c, const hs_keys *k, const hs_ct *a, const int32_t *rots, int n, void *stream,
                            hs_ct **out);
/* slot-vector multiply landing at level `target` (C12). */
hs_status hs_mult_pt(hs_ctx *c, const hs_ct *a, const double *re, const double *im, int target, void *stream,
                     hs_ct **out);
/* Hybrid key switch of one (level+1)-limb polynomial (device pointers). */
hs_status hs_keyswitch(hs_ctx *c, const hs_keys *k, int galois, int level, const uint64_t *d,
                       uint64_t *out0, uint64_t *out1, void *stream);
/* Digit-parallel key switching (PAPER.md 118-121 and
 * 608-614: the shared aux ciphertext and its bootstraps are the serial part
 * of the many-ciphertext Softmax).  The C7 key switch of d (level+1 limbs,
 * NTT domain, device) is split over its beta = ceil((level+1)/alpha) digits:
 *   hs_keyswitch_partial: ModUp and the evaluation-key inner product of the
 *     digits [digit_begin, digit_end) only -> acc = 2 x (level+1+n_p) limbs
 *     (components 0, 1; basis q_0..q_level, p_0..p_{n_p-1}; device; residues
 *     reduced).  An empty range writes zeros.  HS_EINVAL outside [0, beta].
 *   hs_ks_acc_add: acc += other mod q, limb by limb (exact: the accumulator is
 *     a sum over the digits mod q, so any partition's partials add up to the
 *     full one, word for word).
 *   hs_keyswitch_finish: ModDown of a summed accumulator -> out0, out1
 *     ((level+1) limbs each): the same words as hs_keyswitch.
 *   hs_keyswitch_sharded: rank `rank` of `world` computes its digit share
 *     [rank beta / world, (rank+1) beta / world) and combines the partials --
 *     with a native NCCL communicator `comm`, an in-place uint64 sum
 *     all-reduce followed by a reduction mod q (exact while world * q < 2^64,
 *     e.g. world <= 8 with 61-bit primes; otherwise an all-gather), with the
 *     `exchange` callback of the Softmax descriptor's contract an all-gather
 *     added in rank order -- and finishes; every rank ends with
 *     hs_keyswitch's words.  HS_ENCCL on an exchange failure. */
hs_status hs_keyswitch_partial(hs_ctx *c, const hs_keys *k, int galois, int level, const uint64_t *d, int digit_begin,
                               int digit_end, uint64_t *acc, void *stream);
hs_status hs_ks_acc_add(hs_ctx *c, int level, uint64_t *acc, const uint64_t *other, void *stream);
hs_status hs_keyswitch_finish(hs_ctx *c, int level, const uint64_t *acc, uint64_t *out0, uint64_t *out1, void *stream);
/* Forward / inverse negacyclic NTT (C3) of n_limbs consecutive device limbs,
 * limb j reduced mod prime (prime_index + j). */
hs_status hs_ntt(hs_ctx *c, int prime_index, int n_limbs, uint64_t *data, int inverse, void *stream);

/* ------------------------------------------------------------ polynomials (C13) */
typedef struct {
    int deg;
    double a, b;            /* interval; Chebyshev variable u = (2x-a-b)/(b-a) */
    const double *coeffs;   /* deg+1 Chebyshev coefficients                     */
} hs_poly;

/* gain * p(x) for a ciphertext x that holds alpha * x, alpha = 2/(b-a)
 * (G28: the affine map's factor is folded into the input, its shift
 * is a constant add).  Consumes exactly hs_cheb_depth(deg) = ceil(log2(deg+1))
 * levels (1 for deg 1; PAPER.md 330-336 [sec 2.2.4]) with the C13 tree.
 * HS_ELEVEL if x->level is lower, HS_EINVAL on a bad polynomial; the output is
 * library-owned (hs_ct_destroy). */
hs_status hs_cheb(hs_ctx *c, const hs_keys *k, const hs_ct *x, const hs_poly *p, double gain, void *stream,
                  hs_ct **out);
int hs_cheb_depth(int deg);

/* ------------------------------------------------------------ bootstrapping (G11) */
/* Real-slot CoeffToSlot-first bootstrapping:
 * ModRaise -> n_cts CoeffToSlot transforms -> real part -> EvalMod (Chebyshev
 * series of cos(2 pi (K+2) v / 2^r), r double angles, optional arcsine step
 * s + s^3/6) -> n_stc SlotToCoeff transforms -> real part.  The output lands at
 * out_level; the chain top must be
 *   out_level + n_stc + 2 arcsine + r + hs_cheb_depth(cos_poly->deg) + n_cts.
 * Needs the relinearisation key, the conjugation key (Galois 2N-1) and the
 * rotations listed by hs_bts_rotations.  HS_ELEVEL if the chain does not fit. */
typedef struct hs_bts hs_bts;
typedef struct {
    int K;                    /* bound on |I| after ModRaise                   */
    int r;                    /* double-angle steps                            */
    const hs_poly *cos_poly;  /* Chebyshev series on [-1, 1]                    */
    int out_level;
    int n_cts, n_stc;         /* number of CoeffToSlot / SlotToCoeff transforms */
    int arcsine;              /* 1: arcsine correction (2 levels)              */
} hs_bts_desc;

hs_status hs_bts_create(hs_ctx *c, const hs_bts_desc *d, hs_bts **out);
void hs_bts_destroy(hs_bts *b);
/* left-rotation amounts the transforms need (count returned; out may be NULL) */
int hs_bts_rotations(const hs_params *p, int n_cts, int n_stc, int32_t *out, int max);
/* pre-scaling exponent for a message bound (G11) */
int hs_bts_exponent(const hs_params *p, int arcsine, double bound);
/* bound: upper bound on |slot values| of `in` (selects the pre-scaling). */
hs_status hs_bootstrap(hs_ctx *c, const hs_keys *k, hs_bts *b, const hs_ct *in, double bound, void *stream,
                       hs_ct **out);

/* ------------------------------------------------------------ Softmax */
/* Exchange callback for the sharded many-ciphertext case:
 * called with the device buffer of this rank's partial aux sum (`words`
 * uint64 per rank) and must leave in `gathered` (world * words uint64,
 * device) the partial sums of all ranks in rank order, e.g. an NCCL
 * all-gather issued by the caller on `stream`.  Return 0 on success. */
typedef int (*hs_exchange_fn)(void *user, const uint64_t *partial, uint64_t *gathered, size_t words,
                              void *stream);

/* Library-owned NCCL communicator for the sharded many-ciphertext Softmax
 * (SURVEY 8(b) hs_comm_init).  Rank 0 calls
 * hs_comm_unique_id and the caller broadcasts the 128 bytes (e.g. with
 * torch.distributed); every rank then calls hs_comm_init on its own context.
 * NCCL is loaded at run time (libnccl.so.2); HS_ENCCL if it is missing or a
 * collective fails.  The aux-sum exchange then runs as ncclAllGather on the
 * Softmax stream, which CUDA-graph plans capture (hs_softmax_plan_create). */
typedef struct hs_comm hs_comm;
hs_status hs_comm_unique_id(uint8_t uid[128]);
hs_status hs_comm_init(hs_ctx *c, int rank, int world, const uint8_t uid[128], hs_comm **out);
/* hs_keyswitch_sharded: see the digit-parallel key switching block above. */
hs_status hs_keyswitch_sharded(hs_ctx *c, const hs_keys *k, int galois, int level, const uint64_t *d, int rank,
                               int world, hs_comm *comm, hs_exchange_fn exchange, void *user, uint64_t *out0,
                               uint64_t *out1, void *stream);
void hs_comm_destroy(hs_comm *comm);

typedef struct {
    int n;                    /* Softmax dimension                                  */
    int m;                    /* GLOBAL number of main-thread ciphertexts (1: one-ctxt) */
    int k;                    /* iterations (PAPER.md 821)                          */
    int variant;              /* 0 = Alg 1 (normalize-and-square), 1 = version B,
                                 2 = square-and-normalize (PAPER.md 757-765, G26),
                                 3 = cube-and-normalize (PAPER.md 1645-1663, G27)   */
    const hs_poly *exp_poly;  /* exp(x/2^k) on [-M, 0]                              */
    const hs_poly *inv_poly;  /* k polynomials: x^-1/2 (Alg 1), x^-1/2^j (version B),
                                 x^-1 (square- / cube-and-normalize)                 */
    int world, rank;          /* sharding of the m ciphertexts (1, 0 = one GPU)     */
    hs_exchange_fn exchange;  /* required when world > 1                            */
    void *exchange_user;
    hs_bts *bts;              /* NULL: no bootstrapping (HS_ELEVEL when needed)     */
    int newton;               /* Alg 1 only: Newton steps y (3 - x y^2)/2 after the
                                 LAST inverse-square-root polynomial, which is then a
                                 seed (PAPER.md 1311-1327 [App. A]; G24);
                                 0 = none.  HS_EINVAL if < 0 or with version B       */
    hs_comm *comm;            /* native exchange (hs_comm_init; NULL = use exchange).
                                 Its size must equal world; with world == 1 a
                                 one-rank communicator still runs the exchange   */
    int aux_split;            /* SURVEY 8(f) rank 1 / DESIGN.md section 7: 1 = every
                                 key switch of the shared aux thread (the aux-sum
                                 relinearisation, rotate-and-sum, polynomial and
                                 lambda products, the bootstraps' EvalMod products
                                 and conjugations) is digit-split over the world
                                 ranks (hs_keyswitch_sharded semantics, through
                                 comm / exchange); words identical to aux_split = 0.
                                 G >= 2 with world == 1: single-process emulation
                                 (every rank's digit share in turn, then the
                                 rank-order modular sum).  0 = off              */
} hs_softmax_desc;

/* Input contract (G28): every input ciphertext holds x encoded at
 * scale hs_softmax_input_scale(p, d, level) = Delta_level * 2/(b-a) of
 * d->exp_poly's interval [a, b] (the exp polynomial's affine factor folded
 * into the encoding, so the Softmax spends exactly the levels of PAPER.md's
 * depth tables).  Returns 0 on a NULL argument or a level outside the chain. */
double hs_softmax_input_scale(const hs_params *p, const hs_softmax_desc *d, int level);
/* The client-side input step of G28: encode the N/2 real slots (one packed
 * ciphertext, hs_pack) at level+1 with scale hs_softmax_input_scale(level) *
 * q_{level+1}, encrypt with the public key (C5/C6 stream keyed by seed and
 * ct_index, as hs_ckks_encrypt) and rescale once, landing at `level` with the
 * fresh encryption noise divided by q_{level+1} (x keeps ~log2(q) more bits
 * than an encryption straight at the input scale; at level = L it encrypts
 * at `level` directly).  HS_EINVAL on a bad level, HS_EKEY without pk. */
hs_status hs_softmax_encrypt_input(hs_ctx *c, const hs_keys *k, const hs_softmax_desc *d, const double *slots,
                                   int level, uint64_t seed, uint64_t ct_index, void *stream, hs_ct **out);
/* Planner choice of the input level: the level in
 * [0, top - 1] (top = bts_out_level, or the chain top without bootstrapping)
 * whose hs_softmax_schedule cost is lowest -- the main thread needs only the
 * levels its updates consume (G12), and every level above them
 * makes each batched main-thread product dearer.  Host only.  HS_ELEVEL if
 * no level fits. */
hs_status hs_softmax_input_level(const hs_params *p, const hs_softmax_desc *d, size_t m_local, int bts_out_level,
                                 int *level);

/* Debug domain check (SPEC's "domain" error; HS_EDOMAIN): with keys that hold
 * the secret (hs_ckks_keygen), every eager Softmax on this context decrypts
 * the aux sum before each inverse-square-root polynomial and returns
 * HS_EDOMAIN if a slot lies outside the polynomial's interval [a, b] (widened
 * by 1/64 of its width) -- e.g. an input outside [-M, 0].  NULL disables it.
 * Debug only: it synchronises the stream and cannot run inside a plan.  The
 * keys must outlive the setting (the context keeps the pointer; pass NULL
 * before destroying them).  HS_EKEY for keys without the secret. */
hs_status hs_ctx_debug_domain(hs_ctx *c, const hs_keys *k);

/* One ciphertext (m = 1). */
hs_status hs_softmax_one_ctxt(hs_ctx *c, const hs_keys *k, const hs_softmax_desc *d, const hs_ct *in,
                              void *stream, hs_ct **out);
/* m_local = m / world ciphertexts of this rank (contiguous shard). */
hs_status hs_softmax_many_ctxt(hs_ctx *c, const hs_keys *k, const hs_softmax_desc *d, const hs_ct *const *in,
                               size_t m_local, void *stream, hs_ct **out);

/* ------------------------------------------------------------ schedule planner */
/* The bootstrap placement of the paper is prose (PAPER.md 429-440
 * [sec 5.1.3]; G12) and its cost lever is where the bootstraps fall
 * (PAPER.md 285-295, 608-614 [sec 5.2.2]: ~80 % of Alg 1's time, 27 % of
 * version B's at 64 ciphertexts).  hs_softmax_schedule runs the Softmax
 * driver's schedule -- the SAME code hs_softmax_many_ctxt runs, instantiated
 * with a level-only executor -- on the host, without a device or keys, and
 * reports where it bootstraps and what it costs.  Arguments: p the parameter
 * set; d a Softmax descriptor (d->bts, exchange and comm are ignored; world
 * and rank are read); in_level the inputs' level; m_local this rank's
 * ciphertexts (m / world); bts_out_level the level a bootstrap returns
 * (hs_bts_desc.out_level; < 0 = no bootstrapping).  Host only, thread-safe.
 * HS_ELEVEL if the schedule does not fit (as the device run would return),
 * HS_EINVAL on a bad descriptor.
 *
 * cost: a model in units of ONE HMult+relin+rescale of one ciphertext at
 * level 12 of P16: every key switch at level l costs
 * its limb-NTT count relative to level 12, a batch of b members costs
 * b / (1 + 0.1 log2 b) members (measured batch-64 gain 1.6x), a Chebyshev
 * polynomial of degree d costs 2 sqrt(d+1) + log2(d+1) products (PAPER.md
 * 330-336) and a bootstrap HS_SCHED_BTS_COST (measured 22.6 ms per bootstrap vs
 * 0.228 ms per HMult at level 12 on one B200, profiles/r01_bench_full.json). */
#define HS_SCHED_BTS_COST 99.0
typedef struct {
    int out_level;   /* level of the Softmax output                               */
    int bts_main;    /* main-thread bootstraps (one per ciphertext of this rank)   */
    int bts_aux;     /* bootstraps of the auxiliary ciphertext                    */
    int hmult;       /* driver-level ciphertext products, batch members counted
                        (polynomial-internal products are in `cost` only)          */
    int rotations;   /* rotate-and-sum rotations, batch members counted            */
    int poly_evals;  /* Chebyshev evaluations                                      */
    int exchanges;   /* aux-sum all-gathers (world > 1)                            */
    double cost;     /* modelled cost (see above)                                  */
} hs_softmax_sched;
hs_status hs_softmax_schedule(const hs_params *p, const hs_softmax_desc *d, int in_level, size_t m_local,
                              int bts_out_level, hs_softmax_sched *out);
/* Automatic variant selection (Alg 1 vs version B vs the normalisation
 * variants, PAPER.md 585-614 tab:SMmany): plans each of the n candidate
 * descriptors (each with its own variant, k and polynomials) and returns in
 * *best the index of the cheapest one that fits; sched (n entries, nullable)
 * receives every plan, cost = HUGE_VAL for one that does not fit.
 * HS_ELEVEL if none fits, HS_EINVAL on a bad candidate or n == 0. */
hs_status hs_softmax_choose(const hs_params *p, const hs_softmax_desc *cands, size_t n, int in_level,
                            size_t m_local, int bts_out_level, size_t *best, hs_softmax_sched *sched);

/* ------------------------------------------------------------ replayable plans (CUDA graphs) */
/* A plan is one hs_softmax_many_ctxt call captured into a CUDA
 * graph: every kernel of the Softmax runs again at each hs_plan_run, with no
 * host work between launches.  The plan is BOUND to the m_local input
 * ciphertexts `in` (their device words are read at every run -- refresh them
 * with hs_ct_write before a run) and owns m_local output
 * ciphertexts (hs_plan_output; valid until hs_plan_destroy, overwritten by each
 * run).  Creation runs the Softmax once eagerly (warming every table the graph
 * needs) and once under capture.  The inputs and the descriptor's objects
 * (keys, polynomials, bts) must outlive the plan.  Each run adds the captured
 * call's ledger counts.  If kernel profiling is on at creation, the graph
 * records the per-kernel events and hs_kprof_collect after a run reports that
 * run.  A sharded plan (world > 1) needs the native communicator d->comm
 * (hs_comm_init; the NCCL all-gather is captured into the graph, and the
 * communicator must outlive the plan): HS_EINVAL for world > 1 with only an
 * exchange callback. */
typedef struct hs_plan hs_plan;
hs_status hs_softmax_plan_create(hs_ctx *c, const hs_keys *k, const hs_softmax_desc *d, const hs_ct *const *in,
                                 size_t m_local, void *stream, hs_plan **out);
hs_status hs_plan_run(hs_plan *p, void *stream);
size_t hs_plan_n_outputs(const hs_plan *p);
const hs_ct *hs_plan_output(const hs_plan *p, size_t i);
void hs_plan_destroy(hs_plan *p);

/* ------------------------------------------------------------ kernel profiling (bench hooks) */
/* When enabled, every kernel launch is bracketed by CUDA events on its stream
 * and tagged with its algorithmic bytes.  collect
 * synchronises the device and returns, per kernel class (0 NTT, 1 add,
 * 2 scalar, 3 pt-mult, 4 tensor, 5 permute, 6 rescale, 7 bconv, 8 ks-inner,
 * 9 moddown, 10 rng, 11 modraise, 12 hoisted ks-inner), [launches, total ms,
 * total bytes].  Enabling starts a new recording; disabling keeps the slots so
 * a plan captured while enabled can replay into them (its event nodes). */
hs_status hs_kprof_enable(hs_ctx *c, int on);
hs_status hs_kprof_collect(hs_ctx *c, double *out, int n_classes);

/* ------------------------------------------------------------ ledger (D8) */
/* HS_LG_NTT counts limb transforms; HS_LG_NTT_FP those of them that ran on
 * the FP64 butterflies (N = 2^16, primes < 2^43). */
enum { HS_LG_HMULT, HS_LG_TENSOR, HS_LG_KS, HS_LG_ROT, HS_LG_RESCALE, HS_LG_CMULT, HS_LG_PMULT,
       HS_LG_LEVELDOWN, HS_LG_BTS, HS_LG_NTT, HS_LG_KERNELS, HS_LG_NTT_FP, HS_LG_COUNT };
hs_status hs_ledger_get(hs_ctx *c, int64_t *out, int n);
hs_status hs_ledger_reset(hs_ctx *c);

#ifdef __cplusplus
}
#endif
#endif
