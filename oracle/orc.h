/*
 * oracle/orc.h -- internal header of the CPU ORACLE.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load liborc.so.  The oracle shares no code,
 * header, table or constant generator with paper_2410_11184_b200/.
 *
 * It is a plain, slow, obviously-correct C implementation of RNS-CKKS and of
 * the paper's Softmax (arXiv 2410.11184, PAPER.md).  Every convention the
 * paper leaves open is fixed in DESIGN.md section "Conventions" (C1..C15,
 * G1..G23); each function cites the passage or reading it follows.
 */
#ifndef ORC_H
#define ORC_H
#include <stdint.h>
#include <stddef.h>

typedef uint64_t u64;
typedef unsigned __int128 u128;
typedef __int128 i128;

#define ORC_MAXP 64

typedef struct {
    int log_n, n;             /* ring degree N = 2^log_n                   */
    int n_q, n_p;             /* number of Q primes (levels 0..n_q-1), P primes */
    int L;                    /* top level = n_q - 1                        */
    int alpha, dnum;          /* hybrid key-switch digit size, #digits at top */
    u64 prime[ORC_MAXP];      /* q_0..q_L then p_0..p_{alpha-1}              */
    u64 psi[ORC_MAXP];        /* C2 primitive 2N-th root                    */
    u64 *psi_rev[ORC_MAXP];   /* psi^{brv(k)}, k < N                        */
    u64 *ipsi_rev[ORC_MAXP];  /* psi^{-brv(k)}                              */
    u64 n_inv[ORC_MAXP];
    double scale[ORC_MAXP];   /* canonical scale Delta_l per level (C12)    */
    u64 p_mod_q[ORC_MAXP];    /* P mod q_i                                  */
    u64 p_inv_mod_q[ORC_MAXP];/* P^{-1} mod q_i                             */
} orc_params;

/* A ciphertext: ncomp components, each (level+1) limbs of N words,
 * limb-major, NTT (evaluation) domain.  Scale is implicit: the canonical
 * scale of its level (C12). */
typedef struct {
    int level, ncomp;
    u64 *a;                   /* ncomp * (level+1) * N */
} orc_ct;

typedef struct {
    int galois;               /* 0 = relinearisation key, else Galois element */
    int dnum;
    u64 *k;                   /* [dnum][2][n_q + n_p][N] NTT domain          */
} orc_swk;

typedef struct {
    int64_t *s_coeff;         /* ternary secret, coefficient domain          */
    u64 *s_ntt;               /* [n_q+n_p][N]                                 */
    u64 *pk;                  /* [2][n_q][N]                                  */
    int n_swk;
    orc_swk *swk;             /* relin + rotation/conjugation keys           */
} orc_keys;

/* ledger (D8): op counts, exported for tests */
enum { LG_HMULT, LG_TENSOR, LG_KS, LG_ROT, LG_RESCALE, LG_CMULT, LG_PMULT,
       LG_LEVELDOWN, LG_BTS, LG_NTT, LG_COUNT };
extern long orc_ledger[LG_COUNT];
/* key switches per level (bench.py --impl reference: the op inventory the
 * oracle's timed samples are weighted by) */
extern long orc_ks_level[ORC_MAXP];
#define ORC_COUNT_KS(lvl) do { orc_ledger[LG_KS]++; orc_ks_level[(lvl)]++; } while (0)

/* arith.c */
u64 orc_mul(u64 a, u64 b, u64 q);
u64 orc_add(u64 a, u64 b, u64 q);
u64 orc_sub(u64 a, u64 b, u64 q);
u64 orc_pow(u64 a, u64 e, u64 q);
u64 orc_inv(u64 a, u64 q);
int orc_is_prime(u64 n);
u64 orc_residue_of_double(double x, u64 q);
unsigned orc_brv(unsigned x, int bits);

/* ntt.c */
void orc_ntt_fwd(const orc_params *P, int pi, u64 *a);
void orc_ntt_inv(const orc_params *P, int pi, u64 *a);
void orc_ntt_naive(const orc_params *P, int pi, u64 *a);
void orc_galois_perm(const orc_params *P, int k, unsigned *perm);

/* rng.c */
void orc_chacha20_block(const uint32_t key[8], uint32_t counter, const uint32_t nonce[3], uint32_t out[16]);
u64 orc_stream(u64 seed, uint32_t tag, u64 sub, u64 idx);
u64 orc_uniform_mod(u64 seed, uint32_t tag, u64 sub, u64 idx2, u64 q);
int orc_cbd(u64 w, int eta);

/* ckks.c */
orc_ct *orc_ct_alloc(const orc_params *P, int level, int ncomp);
orc_ct *orc_ct_copy(const orc_params *P, const orc_ct *c);
void orc_ct_release(orc_ct *c);
#define LIMB(P, ct, comp, i) ((ct)->a + ((size_t)(comp) * ((ct)->level + 1) + (i)) * (P)->n)

orc_ct *orc_op_add(const orc_params *P, const orc_ct *a, const orc_ct *b);
orc_ct *orc_op_sub(const orc_params *P, const orc_ct *a, const orc_ct *b);
orc_ct *orc_op_level_down(const orc_params *P, const orc_ct *a, int target);
orc_ct *orc_op_rescale(const orc_params *P, const orc_ct *a);
orc_ct *orc_op_tensor(const orc_params *P, const orc_ct *a, const orc_ct *b);
orc_ct *orc_op_relin(const orc_params *P, const orc_keys *K, const orc_ct *d);
orc_ct *orc_op_relin_rescale(const orc_params *P, const orc_keys *K, const orc_ct *d);
orc_ct *orc_op_mult(const orc_params *P, const orc_keys *K, const orc_ct *a, const orc_ct *b);
orc_ct *orc_op_mult_int(const orc_params *P, const orc_ct *a, int64_t c);
orc_ct *orc_op_add_const(const orc_params *P, const orc_ct *a, double c);
orc_ct *orc_op_mult_const(const orc_params *P, const orc_ct *a, double c, int target);
orc_ct *orc_op_mult_pt(const orc_params *P, const orc_ct *a, const double *re, const double *im, int target);
orc_ct *orc_op_galois(const orc_params *P, const orc_keys *K, const orc_ct *a, int k);
orc_ct *orc_op_rotate(const orc_params *P, const orc_keys *K, const orc_ct *a, int r);
orc_ct *orc_op_conjugate(const orc_params *P, const orc_keys *K, const orc_ct *a);
int orc_op_rotate_hoisted(const orc_params *P, const orc_keys *K, const orc_ct *a, const int *rots, int n,
                          orc_ct **out);
void orc_keyswitch(const orc_params *P, const orc_swk *key, int level, const u64 *d, u64 *out0, u64 *out1);
/* key-switch pieces (C7): ModUp -> [beta][ntg][N]; inner product (perm NULL
 * or a Galois permutation of the extended digits) -> acc [2][ntg][N]; ModDown
 * of one component; fused ModDown + rescale by P q_level (C8) */
u64 *orc_ks_modup(const orc_params *P, int level, const u64 *d);
void orc_ks_inner(const orc_params *P, const orc_swk *key, int level, const u64 *ext, const unsigned *perm,
                  u64 *acc);
void orc_ks_moddown1(const orc_params *P, int level, const u64 *A, u64 *out);
void orc_ks_moddown_rescale(const orc_params *P, int level, const u64 *acc, u64 *out0, u64 *out1);
/* digit-parallel key switch: partial accumulator of the
 * digits [j0, j1); ModDown of a summed accumulator */
void orc_ks_inner_digits(const orc_params *P, const orc_swk *key, int level, const u64 *ext, int j0, int j1,
                         u64 *acc);
void orc_ks_partial(const orc_params *P, const orc_swk *key, int level, const u64 *d, int j0, int j1, u64 *acc);
void orc_ks_finish(const orc_params *P, int level, const u64 *acc, u64 *out0, u64 *out1);
const orc_swk *orc_find_key(const orc_keys *K, int galois);
int orc_galois_of_rot(const orc_params *P, int r);

/* encode.c (quad precision, C4) */
void orc_encode_coeffs(const orc_params *P, const double *re, const double *im, double scale, int level, u64 *out);
void orc_decode_coeffs(const orc_params *P, const i128 *coeff, double scale, double *re, double *im);

/* poly.c (C13) */
typedef struct { int deg; double a, b; const double *c; } orc_cheb;
int orc_cheb_depth(int deg);
orc_ct *orc_eval_cheb(const orc_params *P, const orc_keys *K, const orc_ct *w, const orc_cheb *p, double gain);
orc_ct *orc_eval_cheb_unit(const orc_params *P, const orc_keys *K, const orc_ct *u, const orc_cheb *p);

/* softmax.c (Alg 1 / Alg 2 / version B, C14, G12, G24) */
typedef orc_ct *(*orc_bts_fn)(const orc_params *, const orc_keys *, const orc_ct *, void *, double);
typedef struct {
    int n, m, k, variant;           /* 0 = Alg 1, 1 = Alg B, 2 = square-and-normalize  */
    const orc_cheb *exp_poly;       /* exp(x/2^k) on [-M, 0]                            */
    const orc_cheb *inv_poly;       /* k polys, one per iteration                       */
    orc_bts_fn bts;                 /* NULL: no bootstrapping                           */
    void *bts_ctx;
    int newton;                     /* Alg 1: Newton steps after the LAST poly (G24)    */
} orc_softmax_desc;
int orc_softmax(const orc_params *P, const orc_keys *K, const orc_softmax_desc *d, orc_ct *const *x, orc_ct **out);
orc_ct *orc_newton_invsqrt_step(const orc_params *P, const orc_keys *K, const orc_ct *xh, const orc_ct *y);

#endif
