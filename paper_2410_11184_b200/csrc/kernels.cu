// kernels.cu -- all device code of libhesoftmax (sm_100a).
//
// 64-bit modular arithmetic: Shoup multiplication by constants (twiddles,
// BConv constants, scalars) and REDC-based reduction of 128-bit values
// T < q 2^64 for variable x variable products and lazy accumulations
// (tensor, evaluation-key inner product).  All results are canonical
// residues in [0, q), so every kernel is bit-identical to the oracle's
// plain `%` arithmetic.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "hs_internal.h"

__constant__ PrimeK c_pk[HS_MAXP];
// FP64 NTT path (ntt16, primes < 2^43): word offset of the double twiddle
// table inside the context's table allocation, and the switch (HS_NTT_FP=0 off)
__constant__ unsigned long long c_twf_off;
__constant__ int c_ntt_fp;

void upload_prime_constants(const hs_params *P)
{
    HS_CUDA(cudaMemcpyToSymbol(c_pk, P->pk.data(), sizeof(PrimeK) * P->pk.size()));
    const int np = P->n_q + P->n_p;
    const unsigned long long off = (unsigned long long)np * 4 * P->n + 2ull * np;
    HS_CUDA(cudaMemcpyToSymbol(c_twf_off, &off, sizeof(off)));
    const int on = ntt_fp_enabled() ? 1 : 0;
    HS_CUDA(cudaMemcpyToSymbol(c_ntt_fp, &on, sizeof(on)));
}

bool ntt_fp_enabled()
{
    static const bool on = !getenv("HS_NTT_FP") || atoi(getenv("HS_NTT_FP")) != 0;
    return on;
}

// ------------------------------------------------------------------ modular helpers
__device__ __forceinline__ u64 d_add(u64 a, u64 b, u64 q)
{
    u64 s = a + b;
    return s >= q ? s - q : s;
}
__device__ __forceinline__ u64 d_sub(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
__device__ __forceinline__ u64 d_shoup(u64 a, u64 w, u64 wsh, u64 q)
{
    u64 h = __umul64hi(a, wsh);
    u64 r = a * w - h * q;
    return r >= q ? r - q : r;
}
// T = hi 2^64 + lo < q 2^64  ->  T mod q
__device__ __forceinline__ u64 d_reduce128(u64 hi, u64 lo, const PrimeK &k)
{
    u64 m = lo * k.qinv;
    u64 t = hi + __umul64hi(m, k.q) + (lo != 0);
    if (t >= k.q) t -= k.q;
    return d_shoup(t, k.r64, k.r64sh, k.q);
}
__device__ __forceinline__ u64 d_mulmod(u64 a, u64 b, const PrimeK &k) { return d_reduce128(__umul64hi(a, b), a * b, k); }
// Montgomery REDC alone: T = hi 2^64 + lo < q 2^64  ->  T 2^-64 mod q (for
// sums against constants stored as c 2^64 mod q)
__device__ __forceinline__ u64 d_redc(u64 hi, u64 lo, const PrimeK &k)
{
    u64 m = lo * k.qinv;
    u64 t = hi + __umul64hi(m, k.q) + (lo != 0);
    return t >= k.q ? t - k.q : t;
}
// (hi:lo) += a*b as one 32-bit multiply-add carry chain: the four partial
// products are formed once (mul.lo + mul.hi on 64 bits would form the low ones
// twice) -- 8 IMAD-class instructions, no IMAD.WIDE
__device__ __forceinline__ void mac128(u64 &hi, u64 &lo, u64 a, u64 b)
{
    asm("{\n\t"
        ".reg .u32 a0, a1, b0, b1, r0, r1, r2, r3;\n\t"
        "mov.b64 {a0, a1}, %2;\n\t"
        "mov.b64 {b0, b1}, %3;\n\t"
        "mov.b64 {r0, r1}, %0;\n\t"
        "mov.b64 {r2, r3}, %1;\n\t"
        "mad.lo.cc.u32 r0, a0, b0, r0;\n\t"
        "madc.hi.cc.u32 r1, a0, b0, r1;\n\t"
        "madc.lo.cc.u32 r2, a1, b1, r2;\n\t"
        "madc.hi.u32 r3, a1, b1, r3;\n\t"
        "mad.lo.cc.u32 r1, a0, b1, r1;\n\t"
        "madc.hi.cc.u32 r2, a0, b1, r2;\n\t"
        "addc.u32 r3, r3, 0;\n\t"
        "mad.lo.cc.u32 r1, a1, b0, r1;\n\t"
        "madc.hi.cc.u32 r2, a1, b0, r2;\n\t"
        "addc.u32 r3, r3, 0;\n\t"
        "mov.b64 %0, {r0, r1};\n\t"
        "mov.b64 %1, {r2, r3};\n\t"
        "}"
        : "+l"(lo), "+l"(hi)
        : "l"(a), "l"(b));
}

PrimeMap pmap_range(int first, int count)
{
    PrimeMap m;
    m.n = count;
    for (int i = 0; i < count; i++) m.p[i] = (unsigned char)(first + i);
    return m;
}

void count_kernel(hs_ctx *c, int n)
{
    c->ledger[HS_LG_KERNELS] += n;
}

// ------------------------------------------------------------------ NTT (C3)
// N = N1 * N2, index j = r * N2 + col.  Forward Cooley-Tukey stages with
// half-span t >= N2 pair rows (phase "cols"), t < N2 pair within a row
// (phase "rows").  Stage with half-span t uses twiddle table[N/(2t) + j/(2t)].
// Inverse = Gentleman-Sande in the reverse stage order with the psi^-1 table
// and a final N^-1 (fused into the last phase).
struct NttGeom {
    int log_n, log_n1, log_n2;
};

template <bool INV>
__global__ void __launch_bounds__(256) ntt_cols_kernel(u64 *data, PrimeMap pm, const u64 *__restrict__ tw, NttGeom g,
                                                      int C, const u64 *__restrict__ ninv)
{
    extern __shared__ u64 sm[];
    const int N = 1 << g.log_n, N1 = 1 << g.log_n1, N2 = 1 << g.log_n2;
    const int limb = blockIdx.y;
    const int pi = pm.p[limb % pm.n];
    const PrimeK k = c_pk[pi];
    const u64 q = k.q;
    u64 *a = data + (size_t)limb * N;
    const u64 *w = tw + (size_t)pi * 4 * N + (INV ? 2 * N : 0);  // (w, w') pairs
    const int c0 = blockIdx.x * C;
    const int tot = N1 * C;
    for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
        int r = idx / C, c = idx - r * C;
        sm[idx] = a[(size_t)r * N2 + c0 + c];
    }
    __syncthreads();
    const int half = tot >> 1;
    if (!INV) {
        for (int tr = N1 >> 1, m = 1; tr >= 1; tr >>= 1, m <<= 1) {
            for (int b = threadIdx.x; b < half; b += blockDim.x) {
                int c = b % C, rb = b / C;
                int grp = rb / tr, rl = grp * 2 * tr + (rb - grp * tr), rh = rl + tr;
                u64 W = w[2 * (m + grp)], Ws = w[2 * (m + grp) + 1];
                u64 U = sm[rl * C + c], V = d_shoup(sm[rh * C + c], W, Ws, q);
                sm[rl * C + c] = d_add(U, V, q);
                sm[rh * C + c] = d_sub(U, V, q);
            }
            __syncthreads();
        }
    } else {
        for (int tr = 1, m = N1 >> 1; tr < N1; tr <<= 1, m >>= 1) {
            for (int b = threadIdx.x; b < half; b += blockDim.x) {
                int c = b % C, rb = b / C;
                int grp = rb / tr, rl = grp * 2 * tr + (rb - grp * tr), rh = rl + tr;
                u64 W = w[2 * (m + grp)], Ws = w[2 * (m + grp) + 1];
                u64 U = sm[rl * C + c], V = sm[rh * C + c];
                sm[rl * C + c] = d_add(U, V, q);
                sm[rh * C + c] = d_shoup(d_sub(U, V, q), W, Ws, q);
            }
            __syncthreads();
        }
    }
    const u64 ni = INV ? ninv[2 * pi] : 0, nis = INV ? ninv[2 * pi + 1] : 0;
    for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
        int r = idx / C, c = idx - r * C;
        u64 v = sm[idx];
        if (INV) v = d_shoup(v, ni, nis, q);
        a[(size_t)r * N2 + c0 + c] = v;
    }
}

template <bool INV>
__global__ void __launch_bounds__(256) ntt_rows_kernel(u64 *data, PrimeMap pm, const u64 *__restrict__ tw, NttGeom g,
                                                      int R)
{
    extern __shared__ u64 sm[];
    const int N = 1 << g.log_n, N2 = 1 << g.log_n2;
    const int limb = blockIdx.y;
    const int pi = pm.p[limb % pm.n];
    const PrimeK k = c_pk[pi];
    const u64 q = k.q;
    u64 *a = data + (size_t)limb * N + (size_t)blockIdx.x * R * N2;
    const u64 *w = tw + (size_t)pi * 4 * N + (INV ? 2 * N : 0);  // (w, w') pairs
    const int tot = R * N2;
    const int row0 = blockIdx.x * R;
    for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) sm[idx] = a[idx];
    __syncthreads();
    const int half = tot >> 1, hrow = N2 >> 1;
    if (!INV) {
        for (int t = N2 >> 1; t >= 1; t >>= 1) {
            const int m = N / (2 * t);
            for (int b = threadIdx.x; b < half; b += blockDim.x) {
                int row = b / hrow, bb = b - row * hrow;
                int gl = bb / t, lo = gl * 2 * t + (bb - gl * t);
                int grp = (row0 + row) * (N2 / (2 * t)) + gl;
                u64 W = w[2 * (m + grp)], Ws = w[2 * (m + grp) + 1];
                int il = row * N2 + lo, ih = il + t;
                u64 U = sm[il], V = d_shoup(sm[ih], W, Ws, q);
                sm[il] = d_add(U, V, q);
                sm[ih] = d_sub(U, V, q);
            }
            __syncthreads();
        }
    } else {
        for (int t = 1; t < N2; t <<= 1) {
            const int m = N / (2 * t);
            for (int b = threadIdx.x; b < half; b += blockDim.x) {
                int row = b / hrow, bb = b - row * hrow;
                int gl = bb / t, lo = gl * 2 * t + (bb - gl * t);
                int grp = (row0 + row) * (N2 / (2 * t)) + gl;
                u64 W = w[2 * (m + grp)], Ws = w[2 * (m + grp) + 1];
                int il = row * N2 + lo, ih = il + t;
                u64 U = sm[il], V = sm[ih];
                sm[il] = d_add(U, V, q);
                sm[ih] = d_shoup(d_sub(U, V, q), W, Ws, q);
            }
            __syncthreads();
        }
    }
    for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) a[idx] = sm[idx];
}

// ------------------------------------------------------------------ fast NTT for N = 2^16
// Two kernels of 8 stages each (index j = r*256 + e).  Inside a kernel every
// thread keeps 8 words in registers and runs 3 butterfly stages on them
// (radix 8), exchanging through shared memory between rounds 8 / 8 / 4
// stages-per-round = 3 + 3 + 2.  Stage with half-span t on element j uses the
// twiddle tw[N/(2t) + j/(2t)] (Cooley-Tukey forward, Gentleman-Sande inverse).
namespace ntt16 {
constexpr int LOGN = 16, N = 1 << LOGN;
// CTAs per SM the two passes are compiled for at 4-wide tiles (128 threads:
// register cap 64; wider tiles scale it down): measured 121.7 ms of NTT per config-3 step vs 124.5 uncapped and
// 123.0 / 125.8 at 9 / 10 (spills)
#ifndef NTT_MINB
#define NTT_MINB 8
#endif

struct Tw {
    const ulonglong2 *__restrict__ w;  // (twiddle, Shoup companion) pairs
    u64 q, q2;                         // q, 2q
};

// Harvey's lazy butterflies (q < 2^62): a Shoup product without its final
// correction lies in [0, 2q) for any 64-bit input.  Forward values stay in
// [0, 4q), inverse values in [0, 2q); the last stage of each transform
// reduces to [0, q), so the words leaving k_ntt are canonical.
//
// The Shoup quotient drops its a0*s0 partial product (a = a1 2^32 + a0,
// s = s1 2^32 + s0): the estimate hi' = a1 s1 + floor((a1 s0 + a0 s1) / 2^32)
// is floor(a s / 2^64) or one less, so a w - hi' q lies in [0, 3q) (all our
// primes are < 2^61: 3q < 2^64) and one conditional subtraction of 2q brings
// it back to [0, 2q).  Three 32x32 products instead of four in the quotient
// (tools/bfly_lab.cu: 0.86 vs 0.81 T butterflies/s).
__device__ __forceinline__ u64 shoup_lazy3(u64 a, u64 w, u64 ws, u64 q)
{
    u64 r;
    asm("{\n\t"
        ".reg .u32 a0, a1, w0, w1, s0, s1, n0, n1, t0, t1, t2, h0, h1, r0, r1;\n\t"
        "mov.b64 {a0, a1}, %1;\n\t"
        "mov.b64 {w0, w1}, %2;\n\t"
        "mov.b64 {s0, s1}, %3;\n\t"
        "mov.b64 {n0, n1}, %4;\n\t"
        "mul.lo.u32 t0, a1, s0;\n\t"
        "mul.hi.u32 t1, a1, s0;\n\t"
        "mad.lo.cc.u32 t0, a0, s1, t0;\n\t"
        "madc.hi.cc.u32 t1, a0, s1, t1;\n\t"
        "addc.u32 t2, 0, 0;\n\t"
        "mad.lo.cc.u32 h0, a1, s1, t1;\n\t"
        "madc.hi.u32 h1, a1, s1, t2;\n\t"
        "mul.lo.u32 r0, a0, w0;\n\t"
        "mul.hi.u32 r1, a0, w0;\n\t"
        "mad.lo.u32 r1, a0, w1, r1;\n\t"
        "mad.lo.u32 r1, a1, w0, r1;\n\t"
        "mad.lo.cc.u32 r0, h0, n0, r0;\n\t"
        "madc.hi.u32 r1, h0, n0, r1;\n\t"
        "mad.lo.u32 r1, h0, n1, r1;\n\t"
        "mad.lo.u32 r1, h1, n0, r1;\n\t"
        "mov.b64 %0, {r0, r1};\n\t"
        "}"
        : "=l"(r)
        : "l"(a), "l"(w), "l"(ws), "l"(0 - q));
    const u64 q2 = 2 * q;
    return r >= q2 ? r - q2 : r;
}
__device__ __forceinline__ void bfly_ct(u64 &a, u64 &b, const Tw &T, int idx)
{
    const ulonglong2 W = __ldg(T.w + idx);
    const u64 X = a >= T.q2 ? a - T.q2 : a;
    const u64 V = shoup_lazy3(b, W.x, W.y, T.q);
    a = X + V;
    b = X + T.q2 - V;
}
__device__ __forceinline__ void bfly_gs(u64 &a, u64 &b, const Tw &T, int idx)
{
    const ulonglong2 W = __ldg(T.w + idx);
    const u64 U = a, V = b, s = U + V;
    a = s >= T.q2 ? s - T.q2 : s;
    b = shoup_lazy3(U + T.q2 - V, W.x, W.y, T.q);
}
// [0, 4q) -> [0, q)
__device__ __forceinline__ u64 reduce4(u64 v, const Tw &T)
{
    v = v >= T.q2 ? v - T.q2 : v;
    return v >= T.q ? v - T.q : v;
}

// FP64 butterflies for primes 2^36 < q < 2^43 (the P16 user levels).  B200's
// FP64 pipe is separate from the integer multiply pipe and, for these primes,
// exact: values are SIGNED integers |x| < 2^48 held in doubles; hi + lo = b w
// exactly (FMA); qe = round(hi / q) by the 1.5 2^52 trick (|hi/q| < 2^51,
// error below 2^-3); t = hi - qe q is exact (FMA), r = t + lo is exact and
// |r| < 0.7 q (|lo| <= 2^38).  The forward butterfly keeps signed values
// (a + V, a - V: growth below q per stage, < 12 q after 16 stages); the
// inverse one re-centres its sum each stage.  Words between the two passes are
// the signed values as int64; the outputs are canonical.  Same words as the
// integer path (tools/bfly_lab.cu: 1.16 vs 0.85 T butterflies/s at q = 2^42
// for the first, unsigned version).
struct TwF {
    const double *__restrict__ w;  // twiddles as doubles (exact)
    double q, q2, qinv;
};
// b w mod q as a signed representative in (-q, q)
__device__ __forceinline__ double f_mulmod_s(double b, double w, const TwF &T)
{
    const double M = 6755399441055744.0;  // 1.5 * 2^52
    const double hi = b * w;
    const double lo = fma(b, w, -hi);
    const double qe = fma(hi, T.qinv, M) - M;
    return fma(-qe, T.q, hi) + lo;
}
// canonical b w mod q
__device__ __forceinline__ double f_mulmod(double b, double w, const TwF &T)
{
    const double r = f_mulmod_s(b, w, T);
    return r < 0.0 ? r + T.q : r;
}
// x mod q centred: |result| < 0.6 q for |x| < 2^51
__device__ __forceinline__ double f_red(double x, const TwF &T)
{
    const double M = 6755399441055744.0;
    const double qe = fma(x, T.qinv, M) - M;
    return fma(-qe, T.q, x);
}
__device__ __forceinline__ void bfly_ct(double &a, double &b, const TwF &T, int idx)
{
    const double V = f_mulmod_s(b, __ldg(T.w + idx), T);
    b = a - V;
    a = a + V;
}
__device__ __forceinline__ void bfly_gs(double &a, double &b, const TwF &T, int idx)
{
    const double W = __ldg(T.w + idx);
    const double U = a, V = b;
    a = f_red(U + V, T);
    b = f_mulmod_s(U - V, W, T);
}
__device__ __forceinline__ u64 reduce4(double v, const TwF &T)
{
    const double r = f_red(v, T);
    return (u64)(r < 0.0 ? r + T.q : r);
}
// word <-> working value
__device__ __forceinline__ void to_v(u64 &d, u64 x) { d = x; }
__device__ __forceinline__ void to_v(double &d, u64 x) { d = (double)(long long)x; }  // canonical or signed inter-pass word
// inverse output: canonical x N^-1
struct NiI {
    u64 ni, nis;
};
struct NiF {
    double ni;
};
__device__ __forceinline__ u64 scale_out(u64 x, const NiI &n, const Tw &T) { return d_shoup(x, n.ni, n.nis, T.q); }
__device__ __forceinline__ u64 scale_out(double x, const NiF &n, const TwF &T) { return (u64)f_mulmod(x, n.ni, T); }
// values between the passes -> u64 words (integer path: [0, 4q); FP64 path:
// signed, two's complement)
__device__ __forceinline__ u64 to_word(u64 x) { return x; }
__device__ __forceinline__ u64 to_word(double x) { return (u64)(long long)x; }  // signed inter-pass word

// x[k] = element j0 + k s (j0 = block start + offset, block start multiple of 8s)
template <class V, class TW>
__device__ __forceinline__ void radix8_fwd(V x[8], int j0, int s, const TW &T)
{
    int m = N / (8 * s), g = j0 / (8 * s);
    for (int k = 0; k < 4; k++) bfly_ct(x[k], x[k + 4], T, m + g);
    m <<= 1;
    g <<= 1;
    bfly_ct(x[0], x[2], T, m + g);
    bfly_ct(x[1], x[3], T, m + g);
    bfly_ct(x[4], x[6], T, m + g + 1);
    bfly_ct(x[5], x[7], T, m + g + 1);
    m <<= 1;
    g <<= 1;
    for (int k = 0; k < 4; k++) bfly_ct(x[2 * k], x[2 * k + 1], T, m + g + k);
}
template <class V, class TW>
__device__ __forceinline__ void radix8_inv(V x[8], int j0, int s, const TW &T)
{
    int m = N / (2 * s), g = j0 / (2 * s);
    for (int k = 0; k < 4; k++) bfly_gs(x[2 * k], x[2 * k + 1], T, m + g + k);
    m >>= 1;
    g >>= 1;
    bfly_gs(x[0], x[2], T, m + g);
    bfly_gs(x[1], x[3], T, m + g);
    bfly_gs(x[4], x[6], T, m + g + 1);
    bfly_gs(x[5], x[7], T, m + g + 1);
    m >>= 1;
    g >>= 1;
    for (int k = 0; k < 4; k++) bfly_gs(x[k], x[k + 4], T, m + g);
}
// x[k] = element j0 + k s, block start multiple of 4s
template <class V, class TW>
__device__ __forceinline__ void radix4_fwd(V x[4], int j0, int s, const TW &T)
{
    int m = N / (4 * s), g = j0 / (4 * s);
    bfly_ct(x[0], x[2], T, m + g);
    bfly_ct(x[1], x[3], T, m + g);
    m <<= 1;
    g <<= 1;
    bfly_ct(x[0], x[1], T, m + g);
    bfly_ct(x[2], x[3], T, m + g + 1);
}
template <class V, class TW>
__device__ __forceinline__ void radix4_inv(V x[4], int j0, int s, const TW &T)
{
    int m = N / (2 * s), g = j0 / (2 * s);
    bfly_gs(x[0], x[1], T, m + g);
    bfly_gs(x[2], x[3], T, m + g + 1);
    m >>= 1;
    g >>= 1;
    bfly_gs(x[0], x[2], T, m + g);
    bfly_gs(x[1], x[3], T, m + g);
}

__device__ __forceinline__ Tw twiddles(const u64 *tw, int pi, bool inv)
{
    const u64 *base = tw + (size_t)pi * 4 * N + (inv ? 2 * N : 0);
    const u64 q = c_pk[pi].q;
    return Tw{reinterpret_cast<const ulonglong2 *>(base), q, 2 * q};
}
__device__ __forceinline__ bool fp_prime(int pi)
{
    const u64 q = c_pk[pi].q;
    return c_ntt_fp && q < (1ull << 43) && q > (1ull << 36);
}
__device__ __forceinline__ TwF twiddles_f(const u64 *tw, int pi, bool inv)
{
    const double *base = reinterpret_cast<const double *>(tw + c_twf_off) + (size_t)pi * 2 * N + (inv ? N : 0);
    const double q = (double)c_pk[pi].q;
    return TwF{base, q, 2.0 * q, __ddiv_rn(1.0, q)};
}

// Fused prologue / epilogue of a FORWARD transform (limb = row * E.l + i):
//   MODE 1 (rescale, C9): cols loads centred(last_row) mod q_i from the row's
//     dropped limb in coefficient form; rows stores
//     o[row ostr + i N + e] = (ain[row astr + i N + e] - v) q_l^-1
//   MODE 2 (ModDown, C7): rows stores, with row = 2 b + comp,
//     o[b ostr + (comp l + i) N + e] = [add] + (ain[row astr + i N + e] - v) P^-1
// MODE 0 is the plain transform.
struct NttEpi {
    const u64 *last, *ain, *add;
    u64 *o;
    size_t astr, ostr, addstr;
    int l, lq, add_comps;
    u64 inv[HS_MAXP], inv_sh[HS_MAXP];
    u64 rsh[HS_MAXP];  // MODE 1: floor(2^64 / q_i) (Shoup reduction of x < 2^64 by q_i)
    int scaled;        // MODE 1: the input limbs are multiplied by scl_i first (fused mult_const)
    u64 scl[HS_MAXP], scl_sh[HS_MAXP];
    // MODE 3 (inverse, out of place): rows reads limb t from
    // src + (t / srows) sstr + (t % srows) N instead of data (no staging copy)
    const u64 *src;
    size_t sstr;
    int srows;
};

// Phase over the high 8 index bits (half-spans 2^15..2^8): C columns x 256 rows
// per CTA of 32 C threads (thread = column tid % C, row index rid = tid / C).
// The body is generic in the working value (u64 with Shoup butterflies, or
// double with the FP64 butterflies for primes < 2^43): the kernel picks one
// per limb (uniform per CTA).
// Shared-memory swizzle of the butterfly rounds: element a lives at
// a ^ ((5 (a >> 4)) & 15).  With 8-byte words the three access patterns of
// each pass (stride-32 rows, the radix-8 4-groups, the radix-4 quads) all hit
// 16 distinct 8-byte bank pairs per half warp -- 2 wavefronts per 32 lanes,
// the minimum -- where the plain layout needed 8 for the last two patterns
// (ncu: shared-load wavefronts 4x the ideal).  A bijection on every aligned
// block of 16 (it XORs the low 4 bits with a function of the higher ones).
__device__ __forceinline__ int swz(int a) { return a ^ ((5 * (a >> 4)) & 15); }

template <bool INV, int C, int MODE, bool TMA, class V, class TW, class NI>
__device__ __forceinline__ void cols_body(u64 *a, int limb, const TW &T, const NI &ni, V *sm, u64 *smw,
                                          const NttEpi &E)
{
    const int tid = threadIdx.x, col = tid % C, rid = tid / C, c = blockIdx.x * C + col;
    // the TMA tile arrives in the plain layout; otherwise the swizzled one
#define SWC(i) (TMA ? (i) : swz(i))
    V x[8];
    if (!INV) {
        // round 1: rows r0 + 32k, s = 32 rows
        const int r0 = rid;
        if (MODE == 1) {
            // x = centred(last) mod q_i, last = the row's dropped limb mod q_l
            const int row = limb / E.l;
            const u64 *src = E.last + (size_t)row * N;
            const u64 ql = c_pk[E.lq].q, half = (ql - 1) / 2, rsh = E.rsh[limb - row * E.l];
            const u64 q = (u64)T.q;
#pragma unroll
            for (int k = 0; k < 8; k++) {
                // |centred v| mod q by a Shoup step with w = 1, sign restored
                const u64 v = src[(r0 + 32 * k) * 256 + c];
                const bool neg = v > half;
                const u64 sv = neg ? ql - v : v;
                u64 r = sv - __umul64hi(sv, rsh) * q;
                r = r >= q ? r - q : r;
                to_v(x[k], (neg && r) ? q - r : r);
            }
        } else if (TMA) {
#pragma unroll
            for (int k = 0; k < 8; k++) to_v(x[k], smw[SWC((r0 + 32 * k) * C + col)]);
        } else {
#pragma unroll
            for (int k = 0; k < 8; k++) to_v(x[k], a[(r0 + 32 * k) * 256 + c]);
        }
        radix8_fwd(x, r0 * 256 + c, 32 * 256, T);
#pragma unroll
        for (int k = 0; k < 8; k++) sm[SWC((r0 + 32 * k) * C + col)] = x[k];
        __syncthreads();
        // round 2: rows b*32 + sub + 4k, s = 4 rows
        const int b = rid >> 2, sub = rid & 3;
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = sm[SWC((b * 32 + sub + 4 * k) * C + col)];
        radix8_fwd(x, (b * 32 + sub) * 256 + c, 4 * 256, T);
#pragma unroll
        for (int k = 0; k < 8; k++) sm[SWC((b * 32 + sub + 4 * k) * C + col)] = x[k];
        __syncthreads();
        // round 3: rows 4q + k (two groups per thread), s = 1 row; the words
        // between the passes stay in [0, 4q)
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int q = rid + 32 * h;
            V y[4];
#pragma unroll
            for (int k = 0; k < 4; k++) y[k] = sm[SWC((4 * q + k) * C + col)];
            radix4_fwd(y, 4 * q * 256 + c, 256, T);
#pragma unroll
            for (int k = 0; k < 4; k++) {
                if (TMA)
                    smw[SWC((4 * q + k) * C + col)] = to_word(y[k]);
                else
                    a[(4 * q + k) * 256 + c] = to_word(y[k]);
            }
        }
    } else {
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int q = rid + 32 * h;
            V y[4];
#pragma unroll
            for (int k = 0; k < 4; k++) to_v(y[k], TMA ? smw[SWC((4 * q + k) * C + col)] : a[(4 * q + k) * 256 + c]);
            radix4_inv(y, 4 * q * 256 + c, 256, T);
#pragma unroll
            for (int k = 0; k < 4; k++) sm[SWC((4 * q + k) * C + col)] = y[k];
        }
        __syncthreads();
        const int b = rid >> 2, sub = rid & 3;
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = sm[SWC((b * 32 + sub + 4 * k) * C + col)];
        radix8_inv(x, (b * 32 + sub) * 256 + c, 4 * 256, T);
#pragma unroll
        for (int k = 0; k < 8; k++) sm[SWC((b * 32 + sub + 4 * k) * C + col)] = x[k];
        __syncthreads();
        const int r0 = rid;
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = sm[SWC((r0 + 32 * k) * C + col)];
        radix8_inv(x, r0 * 256 + c, 32 * 256, T);
#pragma unroll
        for (int k = 0; k < 8; k++) {
            if (TMA)
                smw[SWC((r0 + 32 * k) * C + col)] = scale_out(x[k], ni, T);
            else
                a[(r0 + 32 * k) * 256 + c] = scale_out(x[k], ni, T);
        }
    }
}
#undef SWC

// TMA = 1: the CTA's 256 x C tile arrives by one cp.async.bulk.tensor load
// into shared memory and leaves by one tensor store (tensor map over the
// limbs as a [256 n_limbs][256] u64 array, box (C, 256)): the strided
// 32-byte column segments no longer cost L1 wavefronts (the pass was
// L1-bound).
template <bool INV, int C, int MODE = 0, bool TMA = false>
__global__ void __launch_bounds__(32 * C, NTT_MINB * 4 / C) cols(u64 *data, PrimeMap pm, const u64 *__restrict__ tw,
                                               const u64 *__restrict__ ninv, const __grid_constant__ NttEpi E,
                                               const __grid_constant__ CUtensorMap tm)
{
    __shared__ __align__(128) u64 sm[256 * C];
    __shared__ __align__(8) u64 bar;
    const int limb = blockIdx.y, pi = pm.p[limb % pm.n];
    u64 *a = data + (size_t)limb * N;
    const unsigned ssm = (unsigned)__cvta_generic_to_shared(sm), sbar = (unsigned)__cvta_generic_to_shared(&bar);
    const int cx = blockIdx.x * C, cy = limb * 256;
    if (TMA) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(256 * C * 8)
                         : "memory");
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                "[%4];" ::"r"(ssm),
                "l"(reinterpret_cast<uint64_t>(&tm)), "r"(cx), "r"(cy), "r"(sbar)
                : "memory");
        }
        asm volatile(
            "{\n\t.reg .pred P;\n\t"
            "NTT_TMA_WAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t"
            "@!P bra NTT_TMA_WAIT_%=;\n\t}" ::"r"(sbar)
            : "memory");
    }
    if (fp_prime(pi)) {
        const TwF T = twiddles_f(tw, pi, INV);
        const NiF ni{INV ? (double)ninv[2 * pi] : 0.0};
        cols_body<INV, C, MODE, TMA>(a, limb, T, ni, reinterpret_cast<double *>(sm), sm, E);
    } else {
        const Tw T = twiddles(tw, pi, INV);
        const NiI ni{INV ? ninv[2 * pi] : 0, INV ? ninv[2 * pi + 1] : 0};
        cols_body<INV, C, MODE, TMA>(a, limb, T, ni, sm, sm, E);
    }
    if (TMA) {
        // the tile's words are in shared memory: make them visible to the
        // async proxy, then one thread stores the tile and waits until the
        // bulk store has read it (the CTA's shared memory must outlive it)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                             reinterpret_cast<uint64_t>(&tm)),
                         "r"(cx), "r"(cy), "r"(ssm)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
    }
}

// Phase over the low 8 index bits (half-spans 2^7..1): R rows of 256 per CTA of
// 32 R threads (one warp per row).
template <bool INV, int R, int MODE, class V, class TW>
__device__ __forceinline__ void rows_body(u64 *data, int limb, const TW &T, V *sm, const NttEpi &E)
{
    const int row0 = blockIdx.x * R;
    u64 *a = data + (size_t)limb * N + (size_t)row0 * 256;
    const int tid = threadIdx.x, row = tid >> 5;
    const int jrow = (row0 + row) * 256;
    const u64 qw = (u64)T.q;
    V x[8];
    if (!INV) {
        const int e0 = tid & 31;
#pragma unroll
        for (int k = 0; k < 8; k++) to_v(x[k], a[row * 256 + e0 + 32 * k]);
        radix8_fwd(x, jrow + e0, 32, T);
#pragma unroll
        for (int k = 0; k < 8; k++) sm[swz(row * 256 + e0 + 32 * k)] = x[k];
        __syncthreads();
        const int b = (tid >> 2) & 7, sub = tid & 3;
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = sm[swz(row * 256 + b * 32 + sub + 4 * k)];
        radix8_fwd(x, jrow + b * 32 + sub, 4, T);
#pragma unroll
        for (int k = 0; k < 8; k++) sm[swz(row * 256 + b * 32 + sub + 4 * k)] = x[k];
        __syncthreads();
        // last round: each thread ends with 4 consecutive words, stored
        // straight to global memory as two 16-byte stores (no smem pass)
        const int crow = MODE ? limb / E.l : 0, li = MODE ? limb - crow * E.l : 0;
        const size_t eb = (size_t)row0 * 256;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int q = (tid & 31) + 32 * h;
            V yv[4];
#pragma unroll
            for (int k = 0; k < 4; k++) yv[k] = sm[swz(row * 256 + 4 * q + k)];
            radix4_fwd(yv, jrow + 4 * q, 1, T);
            const int i0 = row * 256 + 4 * q;
            u64 y[4];
#pragma unroll
            for (int k = 0; k < 4; k++) y[k] = reduce4(yv[k], T);
            if (MODE == 0) {
                ulonglong2 *dst = reinterpret_cast<ulonglong2 *>(a + i0);
                dst[0] = make_ulonglong2(y[0], y[1]);
                dst[1] = make_ulonglong2(y[2], y[3]);
            } else {
                const u64 *in = E.ain + crow * E.astr + (size_t)li * N + eb + i0;
                const ulonglong2 in0 = reinterpret_cast<const ulonglong2 *>(in)[0];
                const ulonglong2 in1 = reinterpret_cast<const ulonglong2 *>(in)[1];
                const u64 iv[4] = {in0.x, in0.y, in1.x, in1.y};
                const u64 inv = E.inv[li], ish = E.inv_sh[li];
                u64 ov[4];
                u64 *o;
                if (MODE == 1) {
                    o = E.o + crow * E.ostr + (size_t)li * N + eb + i0;
                    if (E.scaled) {
                        const u64 sc = E.scl[li], scs = E.scl_sh[li];
#pragma unroll
                        for (int k = 0; k < 4; k++)
                            ov[k] = d_shoup(d_sub(d_shoup(iv[k], sc, scs, qw), y[k], qw), inv, ish, qw);
                    } else {
#pragma unroll
                        for (int k = 0; k < 4; k++) ov[k] = d_shoup(d_sub(iv[k], y[k], qw), inv, ish, qw);
                    }
                } else {
                    const int bb = crow >> 1, comp = crow & 1;
                    const size_t ci = ((size_t)comp * E.l + li) * N + eb + i0;
                    o = E.o + bb * E.ostr + ci;
#pragma unroll
                    for (int k = 0; k < 4; k++) ov[k] = d_shoup(d_sub(iv[k], y[k], qw), inv, ish, qw);
                    if (comp < E.add_comps) {
                        const ulonglong2 *ad = reinterpret_cast<const ulonglong2 *>(E.add + bb * E.addstr + ci);
                        const ulonglong2 a0 = ad[0], a1 = ad[1];
                        ov[0] = d_add(ov[0], a0.x, qw);
                        ov[1] = d_add(ov[1], a0.y, qw);
                        ov[2] = d_add(ov[2], a1.x, qw);
                        ov[3] = d_add(ov[3], a1.y, qw);
                    }
                }
                reinterpret_cast<ulonglong2 *>(o)[0] = make_ulonglong2(ov[0], ov[1]);
                reinterpret_cast<ulonglong2 *>(o)[1] = make_ulonglong2(ov[2], ov[3]);
            }
        }
    } else {
        // first round straight from global memory (two 16-byte loads of 4
        // consecutive words per group)
        const u64 *ra = a;
        if (MODE == 3) ra = E.src + (size_t)(limb / E.srows) * E.sstr + (size_t)(limb % E.srows) * N + (size_t)row0 * 256;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int q = (tid & 31) + 32 * h;
            const ulonglong2 *src = reinterpret_cast<const ulonglong2 *>(ra + row * 256 + 4 * q);
            const ulonglong2 v0 = src[0], v1 = src[1];
            V y[4];
            to_v(y[0], v0.x);
            to_v(y[1], v0.y);
            to_v(y[2], v1.x);
            to_v(y[3], v1.y);
            radix4_inv(y, jrow + 4 * q, 1, T);
#pragma unroll
            for (int k = 0; k < 4; k++) sm[swz(row * 256 + 4 * q + k)] = y[k];
        }
        __syncthreads();
        const int b = (tid >> 2) & 7, sub = tid & 3;
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = sm[swz(row * 256 + b * 32 + sub + 4 * k)];
        radix8_inv(x, jrow + b * 32 + sub, 4, T);
#pragma unroll
        for (int k = 0; k < 8; k++) sm[swz(row * 256 + b * 32 + sub + 4 * k)] = x[k];
        __syncthreads();
        const int e0 = tid & 31;
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = sm[swz(row * 256 + e0 + 32 * k)];
        radix8_inv(x, jrow + e0, 32, T);
#pragma unroll
        for (int k = 0; k < 8; k++) a[row * 256 + e0 + 32 * k] = to_word(x[k]);
    }
}

template <bool INV, int R, int MODE = 0>
__global__ void __launch_bounds__(32 * R, NTT_MINB * 4 / R) rows(u64 *data, PrimeMap pm, const u64 *__restrict__ tw,
                                               const __grid_constant__ NttEpi E)
{
    __shared__ u64 sm[R * 256];
    const int limb = blockIdx.y, pi = pm.p[limb % pm.n];
    if (fp_prime(pi))
        rows_body<INV, R, MODE>(data, limb, twiddles_f(tw, pi, INV), reinterpret_cast<double *>(sm), E);
    else
        rows_body<INV, R, MODE>(data, limb, twiddles(tw, pi, INV), sm, E);
}
// tensor map of `n_limbs` contiguous limbs as a [256 n_limbs][256] u64 array,
// box (C, 256): the cols pass's TMA tile.  false (plain loads) when the
// driver entry point is missing or HS_NTT_TMA=0.
bool cols_tmap(CUtensorMap *m, const u64 *data, int n_limbs, int C)
{
    static const bool on = !getenv("HS_NTT_TMA") || atoi(getenv("HS_NTT_TMA")) != 0;
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    memset(m, 0, sizeof(*m));
    if (!on || !encode || ((uintptr_t)data & 15)) return false;
    const cuuint64_t dims[2] = {256, (cuuint64_t)256 * n_limbs};
    const cuuint64_t strides[1] = {256 * 8};
    const cuuint32_t box[2] = {(cuuint32_t)C, 256};
    const cuuint32_t estr[2] = {1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<u64 *>(data), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int C, int R>
void launch(u64 *data, int n_limbs, const PrimeMap &pm, bool inverse, const u64 *tw, const u64 *ninv,
            cudaStream_t st)
{
    const dim3 gc(256 / C, n_limbs), gr(256 / R, n_limbs);
    NttEpi E{};
    CUtensorMap tm;
    const bool tma = cols_tmap(&tm, data, n_limbs, C);
    if (!inverse) {
        if (tma)
            cols<false, C, 0, true><<<gc, 32 * C, 0, st>>>(data, pm, tw, ninv, E, tm);
        else
            cols<false, C><<<gc, 32 * C, 0, st>>>(data, pm, tw, ninv, E, tm);
        rows<false, R><<<gr, 32 * R, 0, st>>>(data, pm, tw, E);
    } else {
        rows<true, R><<<gr, 32 * R, 0, st>>>(data, pm, tw, E);
        if (tma)
            cols<true, C, 0, true><<<gc, 32 * C, 0, st>>>(data, pm, tw, ninv, E, tm);
        else
            cols<true, C><<<gc, 32 * C, 0, st>>>(data, pm, tw, ninv, E, tm);
    }
}

// inverse transform of n_limbs limbs read from a strided source (MODE 3)
// into the contiguous dst [n_limbs][N]
void launch_inv_from(u64 *dst, const u64 *src, size_t sstr, int srows, int n_limbs, const PrimeMap &pm,
                     const u64 *tw, const u64 *ninv, cudaStream_t st)
{
    NttEpi E{};
    E.src = src;
    E.sstr = sstr;
    E.srows = srows;
    rows<true, 4, 3><<<dim3(64, n_limbs), 128, 0, st>>>(dst, pm, tw, E);
    CUtensorMap tm;
    if (cols_tmap(&tm, dst, n_limbs, 4))
        cols<true, 4, 0, true><<<dim3(64, n_limbs), 128, 0, st>>>(dst, pm, tw, ninv, E, tm);
    else
        cols<true, 4><<<dim3(64, n_limbs), 128, 0, st>>>(dst, pm, tw, ninv, E, tm);
}

// tile width (columns per cols-CTA = rows per rows-CTA); HS_NTT_TILE=4|8|16
// overrides for experiments
int tile()
{
    static int t = [] {
        const char *e = getenv("HS_NTT_TILE");
        int v = e ? atoi(e) : 4;  // measured best: 4 (1.12 us/limb fwd vs 1.33 at 16)
        return (v == 4 || v == 8 || v == 16) ? v : 4;
    }();
    return t;
}
}  // namespace ntt16

// ledger: limb transforms, and how many of them ran on the FP64 butterflies
static void lg_ntt(hs_ctx *c, int n_limbs, const PrimeMap &pm, bool n16)
{
    c->ledger[HS_LG_NTT] += n_limbs;
    if (!n16 || !ntt_fp_enabled()) return;
    int per = 0;
    for (int i = 0; i < pm.n; i++) {
        const u64 q = c->P->prime[pm.p[i]];
        per += q < (1ull << 43) && q > (1ull << 36);
    }
    c->ledger[HS_LG_NTT_FP] += (int64_t)(n_limbs / pm.n) * per;
    for (int i = 0; i < n_limbs % pm.n; i++) {
        const u64 q = c->P->prime[pm.p[i]];
        c->ledger[HS_LG_NTT_FP] += q < (1ull << 43) && q > (1ull << 36);
    }
}

// Rescale of `rows` rows at level l (C9) around ONE forward transform:
// w (scratch, rows*l limbs) = NTT(centred(last) mod q_i) with the lift fused
// into the first pass, o = (a - w) q_l^-1 fused into the second.  last: the
// rows' dropped limbs in coefficient form [rows][N]; a: rows of a_row words
// (default (l+1) N), limbs 0..l-1 read; o: [rows][l][N].  scal (optional):
// a_i is multiplied by scal_i first -- a constant multiplication fused into
// the rescale that follows it (C12).  N = 2^16 only (returns false otherwise).
bool k_ntt_rescale(hs_ctx *c, const u64 *last, u64 *w, const u64 *a, u64 *o, int rows, int l, cudaStream_t st,
                   const u64 *scal, size_t a_row)
{
    const hs_params *P = c->P;
    if (P->log_n != 16) return false;
    const int N = P->n, n_limbs = rows * l;
    KTimer _kt(c, KID_NTT, (double)n_limbs * N * 16, st);
    ntt16::NttEpi E{};
    E.last = last;
    E.ain = a;
    E.o = o;
    E.astr = a_row ? a_row : (size_t)(l + 1) * N;
    E.scaled = scal != nullptr;
    for (int i = 0; scal && i < l; i++) {
        E.scl[i] = scal[i];
        E.scl_sh[i] = hs_shoup_const(scal[i], P->prime[i]);
    }
    E.ostr = (size_t)l * N;
    E.l = l;
    E.lq = l;
    const u64 ql = P->prime[l];
    for (int i = 0; i < l; i++) {
        E.inv[i] = hs_invmod(ql % P->prime[i], P->prime[i]);
        E.inv_sh[i] = hs_shoup_const(E.inv[i], P->prime[i]);
        E.rsh[i] = (u64)((((u128)1) << 64) / P->prime[i]);
    }
    const PrimeMap pm = pmap_range(0, l);
    const u64 *ninv = c->T.tw + (size_t)(P->n_q + P->n_p) * 4 * N;
    CUtensorMap tm0;
    memset(&tm0, 0, sizeof(tm0));
    ntt16::cols<false, 4, 1><<<dim3(64, n_limbs), 128, 0, st>>>(w, pm, c->T.tw, ninv, E, tm0);
    ntt16::rows<false, 4, 1><<<dim3(64, n_limbs), 128, 0, st>>>(w, pm, c->T.tw, E);
    HS_CHECK_LAUNCH();
    lg_ntt(c, n_limbs, pm, true);
    count_kernel(c, 2);
    return true;
}

// ModDown tail (C7): the forward transform of conv [rows][nt][N] (BConv of
// the special limbs) with out = add + (acc - NTT(conv)) inv fused into its
// second pass.  Row r = 2 b + comp reads acc + r acc_row and writes
// o + b o_stride + (comp nt + i) N (so o_stride = 2 nt N lays rows out
// contiguously); inv NULL = P^-1 mod q_i (plain ModDown), else e.g.
// (P q_l)^-1 for the fused relin + rescale (C8).  N = 2^16 only.
bool k_ntt_moddown(hs_ctx *c, u64 *conv, const u64 *acc, size_t acc_row, u64 *o, size_t o_stride, const u64 *add,
                   size_t add_stride, int add_comps, int nt, const u64 *inv, int rows, cudaStream_t st)
{
    const hs_params *P = c->P;
    if (P->log_n != 16) return false;
    const int N = P->n, n_limbs = rows * nt;
    KTimer _kt(c, KID_NTT, (double)n_limbs * N * 16, st);
    ntt16::NttEpi E{};
    E.ain = acc;
    E.add = add;
    E.o = o;
    E.astr = acc_row;
    E.ostr = o_stride;
    E.addstr = add_stride;
    E.add_comps = add ? add_comps : 0;
    E.l = nt;
    for (int i = 0; i < nt; i++) {
        E.inv[i] = inv ? inv[i] : P->p_inv_mod_q[i];
        E.inv_sh[i] = hs_shoup_const(E.inv[i], P->prime[i]);
    }
    const PrimeMap pm = pmap_range(0, nt);
    const u64 *ninv = c->T.tw + (size_t)(P->n_q + P->n_p) * 4 * N;
    CUtensorMap tm;
    if (ntt16::cols_tmap(&tm, conv, n_limbs, 4))
        ntt16::cols<false, 4, 0, true><<<dim3(64, n_limbs), 128, 0, st>>>(conv, pm, c->T.tw, ninv, E, tm);
    else
        ntt16::cols<false, 4, 0><<<dim3(64, n_limbs), 128, 0, st>>>(conv, pm, c->T.tw, ninv, E, tm);
    ntt16::rows<false, 4, 2><<<dim3(64, n_limbs), 128, 0, st>>>(conv, pm, c->T.tw, E);
    HS_CHECK_LAUNCH();
    lg_ntt(c, n_limbs, pm, true);
    count_kernel(c, 2);
    return true;
}

void k_ntt(hs_ctx *c, u64 *data, int n_limbs, const PrimeMap &pm, bool inverse, cudaStream_t st, const u64 *ninv_o)
{
    KTimer _kt(c, KID_NTT, (double)n_limbs * c->P->n * 16, st);
    if (n_limbs <= 0) return;
    const hs_params *P = c->P;
    if (P->log_n == 16) {
        const u64 *ninv = ninv_o && inverse ? ninv_o : c->T.tw + (size_t)(P->n_q + P->n_p) * 4 * P->n;
        switch (ntt16::tile()) {
        case 4: ntt16::launch<4, 4>(data, n_limbs, pm, inverse, c->T.tw, ninv, st); break;
        case 8: ntt16::launch<8, 8>(data, n_limbs, pm, inverse, c->T.tw, ninv, st); break;
        default: ntt16::launch<16, 16>(data, n_limbs, pm, inverse, c->T.tw, ninv, st); break;
        }
        HS_CHECK_LAUNCH();
        lg_ntt(c, n_limbs, pm, true);
        count_kernel(c, 2);
        return;
    }
    NttGeom g;
    g.log_n = P->log_n;
    g.log_n2 = P->log_n / 2;
    g.log_n1 = P->log_n - g.log_n2;
    const int N1 = 1 << g.log_n1, N2 = 1 << g.log_n2;
    const int C = N2 < 16 ? N2 : 16;
    const int R = (2048 / N2) > 0 ? (2048 / N2 < N1 ? 2048 / N2 : N1) : 1;
    dim3 gc(N2 / C, n_limbs), gr(N1 / R, n_limbs);
    size_t smc = (size_t)N1 * C * 8, smr = (size_t)R * N2 * 8;
    const u64 *ninv = ninv_o && inverse ? ninv_o : c->T.tw + (size_t)(P->n_q + P->n_p) * 4 * P->n;
    if (!inverse) {
        ntt_cols_kernel<false><<<gc, 256, smc, st>>>(data, pm, c->T.tw, g, C, ninv);
        ntt_rows_kernel<false><<<gr, 256, smr, st>>>(data, pm, c->T.tw, g, R);
    } else {
        ntt_rows_kernel<true><<<gr, 256, smr, st>>>(data, pm, c->T.tw, g, R);
        ntt_cols_kernel<true><<<gc, 256, smc, st>>>(data, pm, c->T.tw, g, C, ninv);
    }
    HS_CHECK_LAUNCH();
    lg_ntt(c, n_limbs, pm, false);
    count_kernel(c, 2);
}

// dst [n_limbs][N] = iNTT of limb t of src + (t / srows) sstr + (t % srows) N
// (the staging copy of ModUp / ModDown folded into the first pass)
void k_ntt_inv_from(hs_ctx *c, u64 *dst, const u64 *src, size_t sstr, int srows, int n_limbs, const PrimeMap &pm,
                    cudaStream_t st, const u64 *ninv_o)
{
    if (n_limbs <= 0) return;
    const hs_params *P = c->P;
    const size_t N = P->n;
    if (P->log_n != 16) {
        HS_CUDA(cudaMemcpy2DAsync(dst, srows * N * 8, src, sstr * 8, srows * N * 8, n_limbs / srows,
                                  cudaMemcpyDeviceToDevice, st));
        k_ntt(c, dst, n_limbs, pm, true, st, ninv_o);
        return;
    }
    KTimer _kt(c, KID_NTT, (double)n_limbs * N * 16, st);
    const u64 *ninv = ninv_o ? ninv_o : c->T.tw + (size_t)(P->n_q + P->n_p) * 4 * N;
    ntt16::launch_inv_from(dst, src, sstr, srows, n_limbs, pm, c->T.tw, ninv, st);
    HS_CHECK_LAUNCH();
    lg_ntt(c, n_limbs, pm, true);
    count_kernel(c, 2);
}

// ------------------------------------------------------------------ elementwise
#define GRID_LIMBS(n_limbs, N) dim3(((N) + 255) / 256, (n_limbs))

__global__ void add_kernel(const u64 *a, const u64 *b, u64 *o, int N, int period, int sub)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    int l = blockIdx.y;
    u64 q = c_pk[l % period].q;
    size_t x = (size_t)l * N + t;
    o[x] = sub ? d_sub(a[x], b[x], q) : d_add(a[x], b[x], q);
}

void k_add(hs_ctx *c, const u64 *a, const u64 *b, u64 *o, int n_limbs, int period, bool sub, cudaStream_t st)
{
    KTimer _kt(c, KID_ADD, (double)n_limbs * c->P->n * 24, st);
    int N = c->P->n;
    add_kernel<<<GRID_LIMBS(n_limbs, N), 256, 0, st>>>(a, b, o, N, period, sub ? 1 : 0);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

__global__ void neg_kernel(const u64 *a, u64 *o, int N, int period)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    int l = blockIdx.y;
    u64 q = c_pk[l % period].q;
    size_t x = (size_t)l * N + t;
    o[x] = a[x] ? q - a[x] : 0;
}

void k_neg(hs_ctx *c, const u64 *a, u64 *o, int n_limbs, int period, cudaStream_t st)
{
    KTimer _kt(c, KID_ADD, (double)n_limbs * c->P->n * 16, st);
    int N = c->P->n;
    neg_kernel<<<GRID_LIMBS(n_limbs, N), 256, 0, st>>>(a, o, N, period);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

struct ScalarArg {
    u64 v[HS_MAXP], vs[HS_MAXP];
};

static ScalarArg make_scalars(const hs_params *P, const u64 *host_scal, int count)
{
    ScalarArg s;
    for (int i = 0; i < count; i++) {
        s.v[i] = host_scal[i];
        s.vs[i] = hs_shoup_const(host_scal[i], P->prime[i]);
    }
    return s;
}

__global__ void mul_scalar_kernel(const u64 *a, u64 *o, ScalarArg s, int N, int period)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    int l = blockIdx.y, i = l % period;
    size_t x = (size_t)l * N + t;
    o[x] = d_shoup(a[x], s.v[i], s.vs[i], c_pk[i].q);
}

void k_mul_scalar(hs_ctx *c, const u64 *a, u64 *o, const u64 *host_scal, int n_limbs, int period, cudaStream_t st)
{
    KTimer _kt(c, KID_SCALAR, (double)n_limbs * c->P->n * 16, st);
    int N = c->P->n;
    mul_scalar_kernel<<<GRID_LIMBS(n_limbs, N), 256, 0, st>>>(a, o, make_scalars(c->P, host_scal, period), N, period);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

// Elementwise ops on limbs of any basis: limb l is reduced mod the prime
// pm.p[l % pm.n] (the extended basis Q_l u P of the double-hoisted BSGS, C17).
__global__ void mul_scalar_pm_kernel(const u64 *a, u64 *o, ScalarArg s, PrimeMap pm, int N)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    const int l = blockIdx.y, i = l % pm.n;
    const size_t x = (size_t)l * N + t;
    o[x] = d_shoup(a[x], s.v[i], s.vs[i], c_pk[pm.p[i]].q);
}

void k_mul_scalar_pm(hs_ctx *c, const u64 *a, u64 *o, const u64 *host_scal, int n_limbs, const PrimeMap &pm,
                     cudaStream_t st)
{
    KTimer _kt(c, KID_SCALAR, (double)n_limbs * c->P->n * 16, st);
    ScalarArg s;
    for (int i = 0; i < pm.n; i++) {
        s.v[i] = host_scal[i];
        s.vs[i] = hs_shoup_const(host_scal[i], c->P->prime[pm.p[i]]);
    }
    int N = c->P->n;
    mul_scalar_pm_kernel<<<GRID_LIMBS(n_limbs, N), 256, 0, st>>>(a, o, s, pm, N);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

__global__ void add_pm_kernel(const u64 *a, const u64 *b, u64 *o, PrimeMap pm, int N)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    const int l = blockIdx.y;
    const size_t x = (size_t)l * N + t;
    o[x] = d_add(a[x], b[x], c_pk[pm.p[l % pm.n]].q);
}

__global__ void mod_pm_kernel(u64 *a, PrimeMap pm, int N)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    const int l = blockIdx.y;
    const PrimeK k = c_pk[pm.p[l % pm.n]];
    u64 *x = a + (size_t)l * N + t;
    *x = d_reduce128(0, *x, k);  // x < 2^64 < q 2^64: exact x mod q
}

void k_mod_pm(hs_ctx *c, u64 *a, int n_limbs, const PrimeMap &pm, cudaStream_t st)
{
    KTimer _kt(c, KID_ADD, (double)n_limbs * c->P->n * 16, st);
    int N = c->P->n;
    mod_pm_kernel<<<GRID_LIMBS(n_limbs, N), 256, 0, st>>>(a, pm, N);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

void k_add_pm(hs_ctx *c, const u64 *a, const u64 *b, u64 *o, int n_limbs, const PrimeMap &pm, cudaStream_t st)
{
    KTimer _kt(c, KID_ADD, (double)n_limbs * c->P->n * 24, st);
    int N = c->P->n;
    add_pm_kernel<<<GRID_LIMBS(n_limbs, N), 256, 0, st>>>(a, b, o, pm, N);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

__global__ void mac_scalar_kernel(u64 *acc, const u64 *a, ScalarArg s, int N, int period)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    int l = blockIdx.y, i = l % period;
    size_t x = (size_t)l * N + t;
    u64 q = c_pk[i].q;
    acc[x] = d_add(acc[x], d_shoup(a[x], s.v[i], s.vs[i], q), q);
}

void k_mac_scalar(hs_ctx *c, u64 *acc, const u64 *a, const u64 *host_scal, int n_limbs, int period, cudaStream_t st)
{
    KTimer _kt(c, KID_SCALAR, (double)n_limbs * c->P->n * 24, st);
    int N = c->P->n;
    mac_scalar_kernel<<<GRID_LIMBS(n_limbs, N), 256, 0, st>>>(acc, a, make_scalars(c->P, host_scal, period), N,
                                                              period);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

__global__ void add_scalar_kernel(u64 *a, ScalarArg s, int N)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    int l = blockIdx.y;
    size_t x = (size_t)l * N + t;
    a[x] = d_add(a[x], s.v[l], c_pk[l].q);
}

void k_add_scalar(hs_ctx *c, u64 *a, const u64 *host_scal, int n_limbs, cudaStream_t st)
{
    KTimer _kt(c, KID_SCALAR, (double)n_limbs * c->P->n * 16, st);
    int N = c->P->n;
    ScalarArg s;
    for (int i = 0; i < n_limbs; i++) s.v[i] = host_scal[i];
    add_scalar_kernel<<<GRID_LIMBS(n_limbs, N), 256, 0, st>>>(a, s, N);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

__global__ void mul_pointwise_kernel(const u64 *a, const u64 *b, u64 *o, int N, int pa, int pb)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    int l = blockIdx.y, i = l % pa;
    const PrimeK k = c_pk[i];
    o[(size_t)l * N + t] = d_mulmod(a[(size_t)l * N + t], b[(size_t)(l % pb) * N + t], k);
}

void k_mul_pointwise(hs_ctx *c, const u64 *a, const u64 *b, u64 *o, int n_limbs, int period_a, int period_b,
                     cudaStream_t st)
{
    KTimer _kt(c, KID_PTMUL, (double)n_limbs * c->P->n * 24, st);
    int N = c->P->n;
    mul_pointwise_kernel<<<GRID_LIMBS(n_limbs, N), 256, 0, st>>>(a, b, o, N, period_a, period_b);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

// (a0,a1) x (b0,b1) -> (a0b0, a0b1 + a1b0, a1b1); nl limbs per component
__global__ void tensor_kernel(const u64 *a, const u64 *b, u64 *o, int N, int nl)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    int l = blockIdx.y;
    const PrimeK k = c_pk[l];
    size_t s = (size_t)nl * N, x = (size_t)l * N + t;
    u64 a0 = a[x], a1 = a[s + x], b0 = b[x], b1 = b[s + x];
    o[x] = d_mulmod(a0, b0, k);
    u64 hi = 0, lo = 0;
    mac128(hi, lo, a0, b1);
    mac128(hi, lo, a1, b0);
    o[s + x] = d_reduce128(hi, lo, k);
    o[2 * s + x] = d_mulmod(a1, b1, k);
}

void k_tensor(hs_ctx *c, const u64 *a, const u64 *b, u64 *o, int nl, cudaStream_t st)
{
    KTimer _kt(c, KID_TENSOR, (double)nl * c->P->n * 56, st);
    int N = c->P->n;
    tensor_kernel<<<GRID_LIMBS(nl, N), 256, 0, st>>>(a, b, o, N, nl);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

__global__ void permute_kernel(const u64 *a, u64 *o, const unsigned *perm, int N)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    size_t l = blockIdx.y;
    o[l * N + t] = a[l * N + perm[t]];
}

void k_permute(hs_ctx *c, const u64 *a, u64 *o, const unsigned *perm, int n_limbs, cudaStream_t st)
{
    KTimer _kt(c, KID_PERMUTE, (double)n_limbs * c->P->n * 16, st);
    int N = c->P->n;
    permute_kernel<<<GRID_LIMBS(n_limbs, N), 256, 0, st>>>(a, o, perm, N);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

// ------------------------------------------------------------------ rescale (C9)
// last: [ncomp][N] coefficient form of the dropped limb (mod q_level);
// w[comp][i][t] = centred(last) mod q_i, i < level.
__global__ void rescale_prep_kernel(const u64 *last, u64 *w, int N, int level)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    int i = blockIdx.y, comp = blockIdx.z;
    const PrimeK k = c_pk[i];
    const u64 ql = c_pk[level].q, q = k.q;
    u64 x = last[(size_t)comp * N + t];
    u64 v;
    // x mod q by REDC + Shoup (x < 2^61 < q 2^64), not a 64-bit division
    if (x <= (ql - 1) / 2) v = d_reduce128(0, x, k);
    else {
        u64 r = d_reduce128(0, ql - x, k);
        v = r ? q - r : 0;
    }
    w[((size_t)comp * level + i) * N + t] = v;
}

void k_rescale_prep(hs_ctx *c, const u64 *last, u64 *w, int ncomp, int level, cudaStream_t st)
{
    KTimer _kt(c, KID_RESCALE, (double)ncomp * (1 + level) * c->P->n * 8, st);
    int N = c->P->n;
    rescale_prep_kernel<<<dim3((N + 255) / 256, level, ncomp), 256, 0, st>>>(last, w, N, level);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

struct RescaleArg {
    u64 inv[HS_MAXP], inv_sh[HS_MAXP];
};

__global__ void rescale_final_kernel(const u64 *a, const u64 *w, u64 *o, RescaleArg r, int N, int level)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    int i = blockIdx.y, comp = blockIdx.z;
    u64 q = c_pk[i].q;
    u64 x = a[((size_t)comp * (level + 1) + i) * N + t];
    u64 y = w[((size_t)comp * level + i) * N + t];
    o[((size_t)comp * level + i) * N + t] = d_shoup(d_sub(x, y, q), r.inv[i], r.inv_sh[i], q);
}

void k_rescale_final(hs_ctx *c, const u64 *a, const u64 *w, u64 *o, int ncomp, int level, cudaStream_t st)
{
    KTimer _kt(c, KID_RESCALE, (double)ncomp * level * c->P->n * 24, st);
    const hs_params *P = c->P;
    RescaleArg r;
    u64 ql = P->prime[level];
    for (int i = 0; i < level; i++) {
        r.inv[i] = hs_invmod(ql % P->prime[i], P->prime[i]);
        r.inv_sh[i] = hs_shoup_const(r.inv[i], P->prime[i]);
    }
    int N = P->n;
    rescale_final_kernel<<<dim3((N + 255) / 256, level, ncomp), 256, 0, st>>>(a, w, o, r, N, level);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

// ------------------------------------------------------------------ basis conversion (C7)
// y_a = x_a * inv_a mod src_a;  out_b = sum_a y_a * c_ab mod dst_b
struct BconvArg {
    int n_src, n_dst, centred, prescaled;
    unsigned char src[16], dst[HS_MAXP];
};

// centred (ModDown, C7): a term y_a > (q_a-1)/2 stands for y_a - q_a, so the
// target loses one (prod of sources) per such term (table entry pm[b]).
// grid: (N/256, batch, target groups of BCONV_TG).  The sum over the n_src <= 7
// sources of y_a * c_ab (each < 2^61 p) stays below p 2^64, so it is
// accumulated in 128 bits and reduced once (REDC + Shoup, d_reduce128).
#define BCONV_TG 16  // targets per thread (y and the centring sum computed once per 16; 8: +2.6 ms/step)
// NS = number of source primes (compile time: y[] stays in registers and the
// source loops unroll, the NS constants of a target load together)
template <int NS>
__global__ void __launch_bounds__(256) bconv_kernel(const u64 *__restrict__ x, size_t xs, u64 *__restrict__ o,
                                                    size_t os, const __grid_constant__ BconvArg A, const u64 *__restrict__ tab, int N,
                                                    size_t bxs, size_t bos)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    x += blockIdx.y * bxs;
    o += blockIdx.y * bos;
    u64 y[NS];
    double f = 0.0;  // C7 exact centred conversion: v = round(sum_a y_a / s_a)
#pragma unroll
    for (int a = 0; a < NS; a++) {
        const PrimeK k = c_pk[A.src[a]];
        const u64 xa = x[(size_t)a * xs + t];
        y[a] = A.prescaled ? xa : d_shoup(xa, __ldg(tab + 2 * a), __ldg(tab + 2 * a + 1), k.q);
        if (A.centred) f = __dadd_rn(f, __ddiv_rn(__ull2double_rn(y[a]), __ull2double_rn(k.q)));
    }
    const int neg = A.centred ? (int)floor(__dadd_rn(f, 0.5)) : 0;
    const u64 *cm = tab + 2 * NS;
    const u64 *pm = cm + 2 * (size_t)NS * A.n_dst;
    const int b0 = blockIdx.z * BCONV_TG, b1 = min(b0 + BCONV_TG, A.n_dst);
    for (int b = b0; b < b1; b++) {
        const PrimeK k = c_pk[A.dst[b]];
        u64 c[NS];
#pragma unroll
        for (int a = 0; a < NS; a++) c[a] = __ldg(cm + 2 * ((size_t)a * A.n_dst + b));
        // constants in Montgomery form; more than 7 sources fold through one
        // extra REDC after the 7th term (the 128-bit bound needs n_src q < 2^64)
        u64 hi = 0, lo = 0, part = 0;
#pragma unroll
        for (int a = 0; a < NS; a++) {
            mac128(hi, lo, y[a], c[a]);
            if (NS > 7 && a == 6) {
                part = d_redc(hi, lo, k);
                hi = lo = 0;
            }
        }
        u64 s = d_redc(hi, lo, k);
        if (NS > 7) s = d_add(s, part, k.q);
        if (A.centred) {
            const u64 pmb = __ldg(pm + b);
            for (int kk = 0; kk < neg; kk++) s = d_sub(s, pmb, k.q);
        }
        o[(size_t)b * os + t] = s;
    }
}

// Tensor-core BConv (same words as bconv_kernel).  The byte-split identity
// of eval.cpp bconv_build_mma turns the conversion of a 128-coefficient tile
// into u8 x u8 -> s32 products on mma.sync m16n8k32: M = 16 coefficients per
// warp, K = 32 bytes (4 sources x 8 bytes) per k-step, N = 8 bytes v of one
// target.  D_bv < 64 * 255^2 < 2^22, so sum_v 2^8v D_bv < 2^79 < p 2^64 is
// reduced by one REDC (constants in Montgomery form).  The four lanes holding
// the v's of one output stage their partials in shared memory, so that each
// lane reduces one (coefficient, target) output.  The integer-pipe
// work per output falls from n_src 128-bit multiply-adds to one REDC: the
// products move to the tensor cores.
#define BCM_TILE 128
#define BCM_LD (BCM_TILE + 8)  // padded source row (u64): conflict-free fragment loads
__device__ __forceinline__ void mma_u8(int d[4], const uint32_t a[4], uint2 b)
{
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b.x), "r"(b.y));
}

// the conversion's sources / targets as seen by one CTA (pointers into the
// launch's __grid_constant__ argument)
struct BcView {
    const unsigned char *src, *dst;
    int n_src, n_dst, prescaled;
};

template <bool CENTRED>
__device__ __forceinline__ void bconv_mma_body(const u64 *__restrict__ x, size_t xs, u64 *__restrict__ o, size_t os,
                                               const BcView A, const u64 *__restrict__ tab,
                                               const uint2 *__restrict__ frag, int N)
{
    __shared__ u64 sy[8 * BCM_LD];
    __shared__ int sneg[BCM_TILE];
    __shared__ __align__(16) uint32_t spart[8 * 128];  // per warp: [32 outputs][4 partials]
    __shared__ ulonglong2 sk[HS_MAXP];                  // per target: (q, -q^-1 mod 2^64)
    __shared__ u64 spm[CENTRED ? HS_MAXP : 1];
    const int n_base = blockIdx.x * BCM_TILE, tid = threadIdx.x;
    if (tid < A.n_dst) {
        const PrimeK k = c_pk[A.dst[tid]];
        sk[tid] = make_ulonglong2(k.q, k.qinv);
        if (CENTRED) spm[tid] = __ldg(tab + 2 * A.n_src + 2 * (size_t)A.n_src * A.n_dst + tid);
    }
    // y_a = x_a inv_a mod q_a for the tile (sources >= n_src are zero)
    for (int idx = tid; idx < 8 * BCM_TILE; idx += 256) {
        const int a = idx / BCM_TILE, n = idx % BCM_TILE;
        u64 y = 0;
        if (a < A.n_src && n_base + n < N) {
            const u64 xa = x[(size_t)a * xs + n_base + n];
            y = A.prescaled ? xa : d_shoup(xa, __ldg(tab + 2 * a), __ldg(tab + 2 * a + 1), c_pk[A.src[a]].q);
        }
        sy[a * BCM_LD + n] = y;
    }
    __syncthreads();
    if (CENTRED && tid < BCM_TILE) {
        // C7 exact centred conversion: v = round(sum_a y_a / s_a), same order as bconv_kernel
        double f = 0.0;
        for (int a = 0; a < A.n_src; a++)
            f = __dadd_rn(f, __ddiv_rn(__ull2double_rn(sy[a * BCM_LD + tid]), __ull2double_rn(c_pk[A.src[a]].q)));
        sneg[tid] = (int)floor(__dadd_rn(f, 0.5));
    }
    __syncthreads();
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, tg = lane & 3;
    const int r0 = warp * 16, half = tg & 1;
    const uint32_t *sy32 = reinterpret_cast<const uint32_t *>(sy);
    uint32_t af[2][4];
#pragma unroll
    for (int s = 0; s < 2; s++) {
        const int a0 = 4 * s + (tg >> 1), a1 = a0 + 2;
        af[s][0] = sy32[(a0 * BCM_LD + r0 + g) * 2 + half];
        af[s][1] = sy32[(a0 * BCM_LD + r0 + g + 8) * 2 + half];
        af[s][2] = sy32[(a1 * BCM_LD + r0 + g) * 2 + half];
        af[s][3] = sy32[(a1 * BCM_LD + r0 + g + 8) * 2 + half];
    }
    const bool two = A.n_src > 4;
    const int row = r0 + (lane & 15), n = n_base + row;  // this lane's output coefficient
    const int neg = CENTRED ? sneg[row] : 0;
    uint32_t *sp = spart + warp * 128;
    u64 *op = o + (size_t)(lane >> 4) * os + n;  // output (target b + lane / 16, coefficient n)
    const bool nok = n < N;
    for (int b = 0; b < A.n_dst; b += 2, op += 2 * os) {
        int d0[4] = {0, 0, 0, 0}, d1[4] = {0, 0, 0, 0};
        mma_u8(d0, af[0], __ldg(frag + ((size_t)b * 2) * 32 + lane));
        if (two) mma_u8(d0, af[1], __ldg(frag + ((size_t)b * 2 + 1) * 32 + lane));
        if (b + 1 < A.n_dst) {
            mma_u8(d1, af[0], __ldg(frag + ((size_t)(b + 1) * 2) * 32 + lane));
            if (two) mma_u8(d1, af[1], __ldg(frag + ((size_t)(b + 1) * 2 + 1) * 32 + lane));
        }
        // partial of this lane's two v's (v = 2 tg, weight 2^(16 tg)) for its four
        // (target, row) outputs; staged per warp so that lane L then reduces
        // output (target b + L / 16, row r0 + L % 16) from one 16-byte load
        __syncwarp();
        sp[(g) * 4 + tg] = (uint32_t)d0[0] + ((uint32_t)d0[1] << 8);
        sp[(8 + g) * 4 + tg] = (uint32_t)d0[2] + ((uint32_t)d0[3] << 8);
        sp[(16 + g) * 4 + tg] = (uint32_t)d1[0] + ((uint32_t)d1[1] << 8);
        sp[(24 + g) * 4 + tg] = (uint32_t)d1[2] + ((uint32_t)d1[3] << 8);
        __syncwarp();
        const uint4 w = reinterpret_cast<const uint4 *>(sp)[lane];
        const int bb = b + (lane >> 4);
        if (bb < A.n_dst && nok) {
            const u64 lo0 = (u64)w.x + ((u64)w.y << 16) + ((u64)w.z << 32);
            const u64 lo = lo0 + ((u64)w.w << 48);
            const u64 hi = (u64)(w.w >> 16) + (lo < lo0 ? 1 : 0);
            const ulonglong2 kq = sk[bb];
            // REDC: (hi 2^64 + lo + m q) / 2^64, m = lo (-q^-1) mod 2^64
            const u64 m = lo * kq.y;
            u64 r = hi + __umul64hi(m, kq.x) + (lo != 0);
            r = r >= kq.x ? r - kq.x : r;
            if (CENTRED) {
                const u64 pmb = spm[bb];
                for (int kk = 0; kk < neg; kk++) r = r >= pmb ? r - pmb : r + kq.x - pmb;
            }
            *op = r;
        }
    }
}


template <bool CENTRED>
__global__ void __launch_bounds__(256, 8) bconv_mma_kernel(const u64 *__restrict__ x, size_t xs, u64 *__restrict__ o,
                                                        size_t os, const __grid_constant__ BconvArg A, const u64 *__restrict__ tab,
                                                        const uint2 *__restrict__ frag, int N, size_t bxs, size_t bos)
{
    bconv_mma_body<CENTRED>(x + blockIdx.y * bxs, xs, o + blockIdx.y * bos, os,
                            BcView{A.src, A.dst, A.n_src, A.n_dst, A.prescaled}, tab, frag, N);
}

// All ModUp digits of ONE polynomial in one launch (grid.y = digit): digit j
// converts x limbs [src0_j, src0_j + n_src_j) to its n_dst_j targets at
// o + dst_off_j.  Non-centred (ModUp).  Up to 8 sources, unrolled with guards.
struct BconvMultiArg {
    int n_dig, prescaled;
    struct Dig {
        const u64 *tab;
        const uint2 *frag;  // tensor-core fragments (bconv_mma_multi_kernel) or NULL
        int n_src, n_dst, src0;
        size_t dst_off;
        unsigned char src[8], dst[HS_MAXP];
    } d[12];
};

__global__ void __launch_bounds__(256) bconv_multi_kernel(const u64 *__restrict__ x, u64 *__restrict__ o,
                                                          const __grid_constant__ BconvMultiArg A, int N)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    const BconvMultiArg::Dig &D = A.d[blockIdx.y];
    const int b0 = blockIdx.z * BCONV_TG, b1 = min(b0 + BCONV_TG, D.n_dst);
    if (b0 >= b1) return;
    const u64 *tab = D.tab;
    u64 y[8];
#pragma unroll
    for (int a = 0; a < 8; a++)
        if (a < D.n_src) {
            const PrimeK k = c_pk[D.src[a]];
            const u64 xa = x[(size_t)(D.src0 + a) * N + t];
            y[a] = A.prescaled ? xa : d_shoup(xa, __ldg(tab + 2 * a), __ldg(tab + 2 * a + 1), k.q);
        }
    const u64 *cm = tab + 2 * D.n_src;
    for (int b = b0; b < b1; b++) {
        const PrimeK k = c_pk[D.dst[b]];
        u64 hi = 0, lo = 0;
#pragma unroll
        for (int a = 0; a < 7; a++)
            if (a < D.n_src) mac128(hi, lo, y[a], __ldg(cm + 2 * ((size_t)a * D.n_dst + b)));
        u64 r = d_redc(hi, lo, k);  // constants in Montgomery form
        if (D.n_src > 7) {          // 8th source: its own REDC (n_src q < 2^64 bound)
            hi = lo = 0;
            mac128(hi, lo, y[7], __ldg(cm + 2 * ((size_t)7 * D.n_dst + b)));
            r = d_add(r, d_redc(hi, lo, k), k.q);
        }
        o[D.dst_off + (size_t)b * N + t] = r;
    }
}

// All ModUp digits of one polynomial, tensor-core form where it pays (digits of
// >= 4 primes; the CTA geometry of bconv_mma_kernel, grid.y = digit); the
// smaller digits run a plain 128-bit multiply-add loop on the same geometry
// (thread = coefficient tid % 128, targets tid / 128, tid / 128 + 2, ...).
__global__ void __launch_bounds__(256) bconv_mma_multi_kernel(const u64 *__restrict__ x, u64 *__restrict__ o,
                                                              const __grid_constant__ BconvMultiArg A, int N)
{
    const BconvMultiArg::Dig &D = A.d[blockIdx.y];
    if (D.frag && D.n_src >= 4) {
        bconv_mma_body<false>(x + (size_t)D.src0 * N, N, o + D.dst_off, N,
                              BcView{D.src, D.dst, D.n_src, D.n_dst, A.prescaled}, D.tab, D.frag, N);
        return;
    }
    const int t = blockIdx.x * BCM_TILE + (threadIdx.x & (BCM_TILE - 1));
    if (t >= N) return;
    u64 y[8];
#pragma unroll
    for (int a = 0; a < 8; a++)
        if (a < D.n_src) {
            const u64 xa = x[(size_t)(D.src0 + a) * N + t];
            y[a] = A.prescaled ? xa : d_shoup(xa, __ldg(D.tab + 2 * a), __ldg(D.tab + 2 * a + 1), c_pk[D.src[a]].q);
        }
    const u64 *cm = D.tab + 2 * D.n_src;
    for (int b = threadIdx.x / BCM_TILE; b < D.n_dst; b += 2) {
        const PrimeK k = c_pk[D.dst[b]];
        u64 hi = 0, lo = 0;
#pragma unroll
        for (int a = 0; a < 7; a++)
            if (a < D.n_src) mac128(hi, lo, y[a], __ldg(cm + 2 * ((size_t)a * D.n_dst + b)));
        u64 r = d_redc(hi, lo, k);
        if (D.n_src > 7) {
            hi = lo = 0;
            mac128(hi, lo, y[7], __ldg(cm + 2 * ((size_t)7 * D.n_dst + b)));
            r = d_add(r, d_redc(hi, lo, k), k.q);
        }
        o[D.dst_off + (size_t)b * N + t] = r;
    }
}

void k_bconv_modup_multi(hs_ctx *c, const BconvTab *const *tabs, const size_t *dst_off, int n_dig, const u64 *x,
                         u64 *o, cudaStream_t st, bool prescaled)
{
    const int N = c->P->n;
    if (n_dig < 1 || n_dig > 12) throw HsError(HS_EINVAL, "bconv_multi: digit count out of range");
    BconvMultiArg A;
    A.n_dig = n_dig;
    A.prescaled = prescaled ? 1 : 0;
    double bytes = 0;
    int maxg = 1;
    for (int j = 0; j < n_dig; j++) {
        const BconvTab &t = *tabs[j];
        if (t.n_src > 8 || t.centred) throw HsError(HS_EINVAL, "bconv_multi: ModUp digits of at most 8 primes only");
        A.d[j].tab = t.dev;
        A.d[j].frag = reinterpret_cast<const uint2 *>(t.mma);
        A.d[j].n_src = t.n_src;
        A.d[j].n_dst = t.n_dst;
        A.d[j].src0 = t.src[0];
        A.d[j].dst_off = dst_off[j];
        for (int i = 0; i < t.n_src; i++) A.d[j].src[i] = (unsigned char)t.src[i];
        for (int i = 0; i < t.n_dst; i++) A.d[j].dst[i] = (unsigned char)t.dst[i];
        bytes += (double)(t.n_src + t.n_dst) * N * 8;
        maxg = std::max(maxg, (t.n_dst + BCONV_TG - 1) / BCONV_TG);
    }
    KTimer _kt(c, KID_BCONV, bytes, st);
    static const bool mma_on = !getenv("HS_BCONV_MMA") || atoi(getenv("HS_BCONV_MMA")) != 0;
    bool any_mma = false;
    for (int j = 0; j < n_dig; j++) any_mma = any_mma || (A.d[j].frag && A.d[j].n_src >= 4);
    if (mma_on && any_mma)
        bconv_mma_multi_kernel<<<dim3((N + BCM_TILE - 1) / BCM_TILE, n_dig), 256, 0, st>>>(x, o, A, N);
    else
        bconv_multi_kernel<<<dim3((N + 255) / 256, n_dig, maxg), 256, 0, st>>>(x, o, A, N);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

void k_bconv(hs_ctx *c, const BconvTab &tab, const u64 *src, size_t src_stride, u64 *dst, size_t dst_stride,
             int batch, size_t bss, size_t bds, cudaStream_t st, bool prescaled)
{
    KTimer _kt(c, KID_BCONV, (double)batch * (tab.n_src + tab.n_dst) * c->P->n * 8, st);
    BconvArg A;
    A.n_src = tab.n_src;
    A.n_dst = tab.n_dst;
    A.centred = tab.centred ? 1 : 0;
    A.prescaled = prescaled ? 1 : 0;
    for (int i = 0; i < tab.n_src; i++) A.src[i] = (unsigned char)tab.src[i];
    for (int i = 0; i < tab.n_dst; i++) A.dst[i] = (unsigned char)tab.dst[i];
    if (tab.n_src > 9) throw HsError(HS_EINVAL, "bconv: more than 9 source primes");
    int N = c->P->n;
    static const bool mma_on = !getenv("HS_BCONV_MMA") || atoi(getenv("HS_BCONV_MMA")) != 0;
    // measured: the tensor-core form wins for ModUp digits of
    // >= 4 sources; single-prime digits and the centred ModDown stay on bconv_kernel
    if (tab.mma && mma_on && !tab.centred && tab.n_src >= 4) {
        const dim3 g2((N + BCM_TILE - 1) / BCM_TILE, batch);
        const uint2 *fr = reinterpret_cast<const uint2 *>(tab.mma);
        if (tab.centred)
            bconv_mma_kernel<true><<<g2, 256, 0, st>>>(src, src_stride, dst, dst_stride, A, tab.dev, fr, N, bss, bds);
        else
            bconv_mma_kernel<false><<<g2, 256, 0, st>>>(src, src_stride, dst, dst_stride, A, tab.dev, fr, N, bss, bds);
        HS_CHECK_LAUNCH();
        count_kernel(c);
        return;
    }
    const dim3 grid((N + 255) / 256, batch, (tab.n_dst + BCONV_TG - 1) / BCONV_TG);
    switch (tab.n_src) {
#define BCONV_CASE(ns) \
    case ns: bconv_kernel<ns><<<grid, 256, 0, st>>>(src, src_stride, dst, dst_stride, A, tab.dev, N, bss, bds); break;
        BCONV_CASE(1) BCONV_CASE(2) BCONV_CASE(3) BCONV_CASE(4) BCONV_CASE(5) BCONV_CASE(6) BCONV_CASE(7)
        BCONV_CASE(8) BCONV_CASE(9)
#undef BCONV_CASE
    default: throw HsError(HS_EINVAL, "bconv: source count out of range");
    }
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

// ------------------------------------------------------------------ key-switch inner product (C7)
// targets g = 0..level (q_g) then level+1..level+alpha (p_{g-level-1}).
// digit j covers Q primes [j alpha, min((j+1) alpha, level+1)); for g in
// digit j the extended value is d itself, otherwise ext[j][g'] with g' = g
// (g < lo) or g - dn (g >= hi).  key: [dnum][2][n_q+n_p][N].
struct KsArg {
    int level, beta, alpha, n_q, n_t;
};

__global__ void ks_inner_kernel(const u64 *__restrict__ d, const u64 *__restrict__ ext,
                                const u64 *__restrict__ key, u64 *acc, KsArg A, int N)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    int g = blockIdx.y;
    const int nl = A.level + 1;
    const int pi = g < nl ? g : A.n_q + (g - nl);
    const PrimeK k = c_pk[pi];
    const size_t ntot = (size_t)A.n_q + A.n_t;  // primes in key layout
    u64 h0 = 0, l0 = 0, h1 = 0, l1 = 0;
    for (int j = 0; j < A.beta; j++) {
        int lo = j * A.alpha, hi = min((j + 1) * A.alpha, nl), dn = hi - lo;
        u64 v;
        if (g >= lo && g < hi) v = d[(size_t)g * N + t];
        else {
            int gg = g < lo ? g : g - dn;
            v = ext[((size_t)j * (nl + A.alpha) + gg) * N + t];
        }
        const ulonglong2 kk = reinterpret_cast<const ulonglong2 *>(key)[((size_t)j * ntot + pi) * N + t];
        u64 k0 = kk.x, k1 = kk.y;
        mac128(h0, l0, v, k0);
        mac128(h1, l1, v, k1);
    }
    acc[(size_t)g * N + t] = d_reduce128(h0, l0, k);
    acc[((size_t)(nl + A.alpha) + g) * N + t] = d_reduce128(h1, l1, k);
}

void k_ks_inner(hs_ctx *c, const u64 *d, const u64 *ext, const u64 *key, u64 *acc, int level, int beta,
                cudaStream_t st)
{
    KTimer _kt(c, KID_KS_INNER, ((double)beta * (level + 1 + c->P->n_p) * 24 + 2.0 * (level + 1 + c->P->n_p) * 8) * c->P->n, st);
    const hs_params *P = c->P;
    KsArg A{level, beta, P->alpha, P->n_q, P->n_p};
    int N = P->n;
    ks_inner_kernel<<<dim3((N + 255) / 256, level + 1 + P->n_p), 256, 0, st>>>(d, ext, key, acc, A, N);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

// out_c[i] = add_c[i] + (acc_c[i] - conv_c[i]) P^{-1} mod q_i  (add_c may be null)
struct MdArg {
    u64 pinv[HS_MAXP], pinv_sh[HS_MAXP];
    int level, alpha;
    u64 *o0, *o1;
    const u64 *a0, *a1;
};

__global__ void moddown_final_kernel(const u64 *acc, const u64 *conv, MdArg A, int N)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    int i = blockIdx.y, comp = blockIdx.z;
    const int nl = A.level + 1;
    u64 q = c_pk[i].q;
    u64 a = acc[((size_t)comp * (nl + A.alpha) + i) * N + t];
    u64 b = conv[((size_t)comp * nl + i) * N + t];
    u64 v = d_shoup(d_sub(a, b, q), A.pinv[i], A.pinv_sh[i], q);
    const u64 *ad = comp ? A.a1 : A.a0;
    size_t oi = (size_t)i * N + t;
    if (ad) v = d_add(v, ad[oi], q);
    (comp ? A.o1 : A.o0)[oi] = v;
}

void k_moddown_final(hs_ctx *c, const u64 *acc, const u64 *conv, u64 *o0, u64 *o1, const u64 *add0,
                     const u64 *add1, int level, cudaStream_t st)
{
    KTimer _kt(c, KID_MODDOWN, (double)(level + 1) * c->P->n * 8 * (6 + (add0 ? 1 : 0) + (add1 ? 1 : 0)), st);
    const hs_params *P = c->P;
    MdArg A;
    for (int i = 0; i <= level; i++) {
        A.pinv[i] = P->p_inv_mod_q[i];
        A.pinv_sh[i] = hs_shoup_const(P->p_inv_mod_q[i], P->prime[i]);
    }
    A.level = level;
    A.alpha = P->n_p;
    A.o0 = o0;
    A.o1 = o1;
    A.a0 = add0;
    A.a1 = add1;
    int N = P->n;
    moddown_final_kernel<<<dim3((N + 255) / 256, level + 1, 2), 256, 0, st>>>(acc, conv, A, N);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

// ------------------------------------------------------------------ randomness (C5)
__host__ __device__ __forceinline__ uint32_t rotl32(uint32_t x, int n) { return (x << n) | (x >> (32 - n)); }
#define CHQR(a, b, c, d)                  \
    a += b; d ^= a; d = rotl32(d, 16);    \
    c += d; b ^= c; b = rotl32(b, 12);    \
    a += b; d ^= a; d = rotl32(d, 8);     \
    c += d; b ^= c; b = rotl32(b, 7);

__host__ __device__ void chacha_block(const uint32_t key[8], uint32_t ctr, const uint32_t nonce[3], uint32_t o[16])
{
    uint32_t s[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u, key[0], key[1], key[2], key[3],
                      key[4],      key[5],      key[6],      key[7],      ctr,    nonce[0], nonce[1], nonce[2]};
    uint32_t x[16];
    for (int i = 0; i < 16; i++) x[i] = s[i];
    for (int r = 0; r < 10; r++) {
        CHQR(x[0], x[4], x[8], x[12]);
        CHQR(x[1], x[5], x[9], x[13]);
        CHQR(x[2], x[6], x[10], x[14]);
        CHQR(x[3], x[7], x[11], x[15]);
        CHQR(x[0], x[5], x[10], x[15]);
        CHQR(x[1], x[6], x[11], x[12]);
        CHQR(x[2], x[7], x[8], x[13]);
        CHQR(x[3], x[4], x[9], x[14]);
    }
    for (int i = 0; i < 16; i++) o[i] = x[i] + s[i];
}

void hs_chacha20_block(const uint32_t key[8], uint32_t counter, const uint32_t nonce[3], uint32_t out[16])
{
    chacha_block(key, counter, nonce, out);
}

u64 hs_stream_word(u64 seed, uint32_t tag, u64 sub, u64 idx)
{
    uint32_t key[8] = {(uint32_t)seed, (uint32_t)(seed >> 32), tag, (uint32_t)sub, (uint32_t)(sub >> 32), 0, 0, 0};
    uint32_t nonce[3] = {0, 0, 0}, o[16];
    chacha_block(key, (uint32_t)(idx >> 3), nonce, o);
    int w = (int)(idx & 7);
    return (u64)o[2 * w] | ((u64)o[2 * w + 1] << 32);
}

// uniform mod q: sample idx2 = pi*N + t uses stream words 2 idx2, 2 idx2 + 1,
// value = (w1 2^64 + w0) mod q.  One ChaCha block = 4 samples.
__global__ void uniform_kernel(u64 *o, PrimeMap pm, u64 seed, uint32_t tag, u64 sub, int N)
{
    int blk = blockIdx.x * blockDim.x + threadIdx.x;  // block within limb
    if (blk * 4 >= N) return;
    int l = blockIdx.y, pi = pm.p[l % pm.n];
    const PrimeK k = c_pk[pi];
    uint32_t key[8] = {(uint32_t)seed, (uint32_t)(seed >> 32), tag, (uint32_t)sub, (uint32_t)(sub >> 32), 0, 0, 0};
    uint32_t nonce[3] = {0, 0, 0}, w[16];
    u64 idx2_0 = (u64)pi * N + (u64)blk * 4;
    chacha_block(key, (uint32_t)(idx2_0 >> 2), nonce, w);
    for (int s = 0; s < 4; s++) {
        u64 w0 = (u64)w[4 * s] | ((u64)w[4 * s + 1] << 32);
        u64 w1 = (u64)w[4 * s + 2] | ((u64)w[4 * s + 3] << 32);
        u64 h = d_reduce128(0, w1, k);
        o[(size_t)l * N + blk * 4 + s] = d_reduce128(h, w0, k);
    }
}

void k_uniform(hs_ctx *c, u64 *o, int n_limbs, const PrimeMap &pm, u64 seed, uint32_t tag, u64 sub, int,
               cudaStream_t st)
{
    KTimer _kt(c, KID_RNG, (double)n_limbs * c->P->n * 8, st);
    int N = c->P->n;
    int nb = N / 4;
    uniform_kernel<<<dim3((nb + 127) / 128, n_limbs), 128, 0, st>>>(o, pm, seed, tag, sub, N);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

// centred binomial: coefficient t uses stream word t
__global__ void cbd_kernel(int64_t *o, u64 seed, uint32_t tag, u64 sub, int eta, int N)
{
    int blk = blockIdx.x * blockDim.x + threadIdx.x;
    if (blk * 8 >= N) return;
    uint32_t key[8] = {(uint32_t)seed, (uint32_t)(seed >> 32), tag, (uint32_t)sub, (uint32_t)(sub >> 32), 0, 0, 0};
    uint32_t nonce[3] = {0, 0, 0}, w[16];
    chacha_block(key, (uint32_t)blk, nonce, w);
    u64 m = (1ull << eta) - 1;
    for (int s = 0; s < 8; s++) {
        u64 x = (u64)w[2 * s] | ((u64)w[2 * s + 1] << 32);
        o[blk * 8 + s] = (int64_t)__popcll(x & m) - (int64_t)__popcll((x >> eta) & m);
    }
}

void k_cbd(hs_ctx *c, int64_t *o, u64 seed, uint32_t tag, u64 sub, int eta, cudaStream_t st)
{
    KTimer _kt(c, KID_RNG, (double)c->P->n * 8, st);
    int N = c->P->n;
    cbd_kernel<<<(N / 8 + 127) / 128, 128, 0, st>>>(o, seed, tag, sub, eta, N);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

__global__ void signed_to_rns_kernel(const int64_t *v, u64 *o, PrimeMap pm, int N)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    int l = blockIdx.y;
    u64 q = c_pk[pm.p[l % pm.n]].q;
    int64_t x = v[t];
    u64 r = x >= 0 ? (u64)x % q : (u64)(-(x + 1)) % q;  // |x| - 1 for negatives avoids overflow
    if (x < 0) r = q - 1 - r;
    o[(size_t)l * N + t] = r;
}

void k_signed_to_rns(hs_ctx *c, const int64_t *v, u64 *o, int n_limbs, const PrimeMap &pm, cudaStream_t st)
{
    KTimer _kt(c, KID_RNG, (double)(n_limbs + 1) * c->P->n * 8, st);
    int N = c->P->n;
    signed_to_rns_kernel<<<GRID_LIMBS(n_limbs, N), 256, 0, st>>>(v, o, pm, N);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

// ------------------------------------------------------------------ batched ciphertext kernels
// A batch of B ciphertexts is one allocation [B][ncomp][nl][N]; a "row" is one
// (ciphertext, component) pair of nl limbs.  Second operands may be broadcast
// (b_rows < rows: row r uses b row r % b_rows).

// two adjacent words per thread (16-byte loads / stores)
__global__ void add_b_kernel(const u64 *a, const u64 *b, u64 *o, int N, int nl, int a_rows, int b_rows, int sub)
{
    int t = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (t >= N) return;
    int i = blockIdx.y, r = blockIdx.z;
    u64 q = c_pk[i].q;
    size_t x = ((size_t)(r % a_rows) * nl + i) * N + t, y = ((size_t)(r % b_rows) * nl + i) * N + t;
    const ulonglong2 va = *reinterpret_cast<const ulonglong2 *>(a + x);
    const ulonglong2 vb = *reinterpret_cast<const ulonglong2 *>(b + y);
    ulonglong2 vo;
    vo.x = sub ? d_sub(va.x, vb.x, q) : d_add(va.x, vb.x, q);
    vo.y = sub ? d_sub(va.y, vb.y, q) : d_add(va.y, vb.y, q);
    *reinterpret_cast<ulonglong2 *>(o + ((size_t)r * nl + i) * N + t) = vo;
}

void k_add_b(hs_ctx *c, const u64 *a, int a_rows, const u64 *b, int b_rows, u64 *o, int rows, int nl, bool sub,
             cudaStream_t st)
{
    KTimer _kt(c, KID_ADD, (double)rows * nl * c->P->n * 24, st);
    int N = c->P->n;
    add_b_kernel<<<dim3((N / 2 + 255) / 256, nl, rows), 256, 0, st>>>(a, b, o, N, nl, a_rows, b_rows, sub ? 1 : 0);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

// o[r][i] = a[r][i] * s_i, rows of a/o with their own limb strides (drop + scale in one pass)
__global__ void mul_scalar_s_kernel(const u64 *a, u64 *o, ScalarArg s, int N, int a_rl, int o_rl, int acc)
{
    int t = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (t >= N) return;
    int i = blockIdx.y, r = blockIdx.z;
    u64 q = c_pk[i].q;
    const ulonglong2 va = *reinterpret_cast<const ulonglong2 *>(a + ((size_t)r * a_rl + i) * N + t);
    ulonglong2 v;
    v.x = d_shoup(va.x, s.v[i], s.vs[i], q);
    v.y = d_shoup(va.y, s.v[i], s.vs[i], q);
    ulonglong2 *op = reinterpret_cast<ulonglong2 *>(o + ((size_t)r * o_rl + i) * N + t);
    if (acc) {
        const ulonglong2 vo = *op;
        v.x = d_add(vo.x, v.x, q);
        v.y = d_add(vo.y, v.y, q);
    }
    *op = v;
}

void k_mul_scalar_s(hs_ctx *c, const u64 *a, u64 *o, const u64 *host_scal, int rows, int nl, int a_rl, int o_rl,
                    bool accumulate, cudaStream_t st)
{
    KTimer _kt(c, KID_SCALAR, (double)rows * nl * c->P->n * (accumulate ? 24 : 16), st);
    int N = c->P->n;
    mul_scalar_s_kernel<<<dim3((N / 2 + 255) / 256, nl, rows), 256, 0, st>>>(a, o, make_scalars(c->P, host_scal, nl), N,
                                                                          a_rl, o_rl, accumulate ? 1 : 0);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

// o = [o +] sum_j s_j a_j over up to 16 terms in ONE pass (Chebyshev leaves,
// C13): each term read once, 128-bit accumulation against Montgomery-form
// scalars (s 2^64 mod q; 16 q^2 < q 2^64 for q < 2^60), one REDC.  Term j
// element (row r, limb i, t) at a_j + (r a_rl[j] + i) N + t; o rows of o_rl.
struct LinCombArg {
    const u64 *a[16];
    int a_rl[16];
    int n, acc;
    u64 s[16][HS_MAXP];
};

__global__ void __launch_bounds__(256) lin_comb_kernel(u64 *__restrict__ o, const __grid_constant__ LinCombArg A,
                                                       int N, int o_rl)
{
    const int t = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (t >= N) return;
    const int i = blockIdx.y, r = blockIdx.z;
    const PrimeK k = c_pk[i];
    u64 h0 = 0, l0 = 0, h1 = 0, l1 = 0;
    for (int j = 0; j < A.n; j++) {
        const ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(A.a[j] + ((size_t)r * A.a_rl[j] + i) * N + t);
        const u64 sm = A.s[j][i];
        mac128(h0, l0, v.x, sm);
        mac128(h1, l1, v.y, sm);
    }
    ulonglong2 *op = reinterpret_cast<ulonglong2 *>(o + ((size_t)r * o_rl + i) * N + t);
    ulonglong2 w = make_ulonglong2(d_redc(h0, l0, k), d_redc(h1, l1, k));
    if (A.acc) {
        const ulonglong2 vo = *op;
        w.x = d_add(vo.x, w.x, k.q);
        w.y = d_add(vo.y, w.y, k.q);
    }
    *op = w;
}

__global__ void interleave2_kernel(const u64 *planar, u64 *o, size_t W)
{
    const size_t w = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= W) return;
    const size_t d = blockIdx.y;
    reinterpret_cast<ulonglong2 *>(o)[d * W + w] = make_ulonglong2(planar[(d * 2) * W + w], planar[(d * 2 + 1) * W + w]);
}

void k_interleave2(hs_ctx *c, const u64 *planar, u64 *o, int D, size_t W, cudaStream_t st)
{
    interleave2_kernel<<<dim3((unsigned)((W + 255) / 256), D), 256, 0, st>>>(planar, o, W);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

void k_lin_comb(hs_ctx *c, const u64 *const *a, const int *a_rl, const u64 *const *host_scal, int n_terms, u64 *o,
                int rows, int nl, int o_rl, bool accumulate, cudaStream_t st)
{
    const hs_params *P = c->P;
    if (n_terms < 1 || n_terms > 16) throw HsError(HS_EINVAL, "lin_comb: 1..16 terms");
    KTimer _kt(c, KID_SCALAR, (double)rows * nl * P->n * 8 * (n_terms + 1 + (accumulate ? 1 : 0)), st);
    LinCombArg A;
    A.n = n_terms;
    A.acc = accumulate ? 1 : 0;
    for (int j = 0; j < n_terms; j++) {
        A.a[j] = a[j];
        A.a_rl[j] = a_rl[j];
        for (int i = 0; i < nl; i++) {
            const u64 q = P->prime[i];
            A.s[j][i] = (u64)((((unsigned __int128)(host_scal[j][i] % q)) << 64) % q);
        }
    }
    const int N = P->n;
    lin_comb_kernel<<<dim3((N / 2 + 255) / 256, nl, rows), 256, 0, st>>>(o, A, N, o_rl);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

// comp 0 of each of B ciphertexts += s_i
__global__ void add_scalar_b_kernel(u64 *a, ScalarArg s, int N, int nl, int row_stride)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    int i = blockIdx.y, b = blockIdx.z;
    size_t x = ((size_t)b * row_stride + i) * N + t;
    a[x] = d_add(a[x], s.v[i], c_pk[i].q);
}

void k_add_scalar_b(hs_ctx *c, u64 *a, const u64 *host_scal, int B, int ncomp, int nl, cudaStream_t st)
{
    KTimer _kt(c, KID_SCALAR, (double)B * nl * c->P->n * 16, st);
    int N = c->P->n;
    ScalarArg s;
    for (int i = 0; i < nl; i++) s.v[i] = host_scal[i];
    add_scalar_b_kernel<<<dim3((N + 255) / 256, nl, B), 256, 0, st>>>(a, s, N, nl, ncomp * nl);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

// o[b] = tensor(a[b], bb[b % b_batch]); a/bb: [.][2][nl][N], o: [B][3][nl][N]
__global__ void tensor_b_kernel(const u64 *a, const u64 *bb, u64 *o, int N, int nl, int b_batch)
{
    int t = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (t >= N) return;
    int l = blockIdx.y, b = blockIdx.z;
    const PrimeK k = c_pk[l];
    size_t s = (size_t)nl * N, x = (size_t)l * N + t;
    const u64 *A = a + (size_t)b * 2 * s, *Bp = bb + (size_t)(b % b_batch) * 2 * s;
    u64 *O = o + (size_t)b * 3 * s;
    const ulonglong2 a0 = *reinterpret_cast<const ulonglong2 *>(A + x), a1 = *reinterpret_cast<const ulonglong2 *>(A + s + x);
    const ulonglong2 b0 = *reinterpret_cast<const ulonglong2 *>(Bp + x), b1 = *reinterpret_cast<const ulonglong2 *>(Bp + s + x);
    ulonglong2 o0, o1, o2;
    o0.x = d_mulmod(a0.x, b0.x, k);
    o0.y = d_mulmod(a0.y, b0.y, k);
    u64 hi = 0, lo = 0;
    mac128(hi, lo, a0.x, b1.x);
    mac128(hi, lo, a1.x, b0.x);
    o1.x = d_reduce128(hi, lo, k);
    hi = lo = 0;
    mac128(hi, lo, a0.y, b1.y);
    mac128(hi, lo, a1.y, b0.y);
    o1.y = d_reduce128(hi, lo, k);
    o2.x = d_mulmod(a1.x, b1.x, k);
    o2.y = d_mulmod(a1.y, b1.y, k);
    *reinterpret_cast<ulonglong2 *>(O + x) = o0;
    *reinterpret_cast<ulonglong2 *>(O + s + x) = o1;
    *reinterpret_cast<ulonglong2 *>(O + 2 * s + x) = o2;
}

// o[b] = (a0^2, 2 a0 a1, a1^2): the square, reading each operand once
__global__ void square_b_kernel(const u64 *a, u64 *o, int N, int nl)
{
    int t = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (t >= N) return;
    int l = blockIdx.y, b = blockIdx.z;
    const PrimeK k = c_pk[l];
    size_t s = (size_t)nl * N, x = (size_t)l * N + t;
    const u64 *A = a + (size_t)b * 2 * s;
    u64 *O = o + (size_t)b * 3 * s;
    const ulonglong2 a0 = *reinterpret_cast<const ulonglong2 *>(A + x), a1 = *reinterpret_cast<const ulonglong2 *>(A + s + x);
    ulonglong2 o0, o1, o2;
    o0.x = d_mulmod(a0.x, a0.x, k);
    o0.y = d_mulmod(a0.y, a0.y, k);
    o1.x = d_mulmod(a0.x, a1.x, k);
    o1.y = d_mulmod(a0.y, a1.y, k);
    o1.x = d_add(o1.x, o1.x, k.q);
    o1.y = d_add(o1.y, o1.y, k.q);
    o2.x = d_mulmod(a1.x, a1.x, k);
    o2.y = d_mulmod(a1.y, a1.y, k);
    *reinterpret_cast<ulonglong2 *>(O + x) = o0;
    *reinterpret_cast<ulonglong2 *>(O + s + x) = o1;
    *reinterpret_cast<ulonglong2 *>(O + 2 * s + x) = o2;
}

void k_tensor_b(hs_ctx *c, const u64 *a, const u64 *b, u64 *o, int B, int nl, int b_batch, cudaStream_t st)
{
    const bool sq = a == b && b_batch == B;
    KTimer _kt(c, KID_TENSOR, (double)B * nl * c->P->n * (sq ? 40 : 56), st);
    int N = c->P->n;
    if (sq) square_b_kernel<<<dim3((N / 2 + 255) / 256, nl, B), 256, 0, st>>>(a, o, N, nl);
    else tensor_b_kernel<<<dim3((N / 2 + 255) / 256, nl, B), 256, 0, st>>>(a, b, o, N, nl, b_batch);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

// o = sum_b tensor(a[b], a[b])  (C15 aux sum, exact mod q in any order)
__global__ void tensor_sum_kernel(const u64 *a, u64 *o, int N, int nl, int B)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    int l = blockIdx.y;
    const PrimeK k = c_pk[l];
    size_t s = (size_t)nl * N, x = (size_t)l * N + t;
    u64 d0 = 0, d1 = 0, d2 = 0;
    for (int b = 0; b < B; b++) {
        const u64 *A = a + (size_t)b * 2 * s;
        u64 a0 = A[x], a1 = A[s + x];
        d0 = d_add(d0, d_mulmod(a0, a0, k), k.q);
        u64 p = d_mulmod(a0, a1, k);
        d1 = d_add(d1, d_add(p, p, k.q), k.q);
        d2 = d_add(d2, d_mulmod(a1, a1, k), k.q);
    }
    o[x] = d0;
    o[s + x] = d1;
    o[2 * s + x] = d2;
}

void k_tensor_sum(hs_ctx *c, const u64 *a, u64 *o, int B, int nl, cudaStream_t st)
{
    KTimer _kt(c, KID_TENSOR, (double)(2 * B + 3) * nl * c->P->n * 8, st);
    int N = c->P->n;
    tensor_sum_kernel<<<dim3((N + 255) / 256, nl), 256, 0, st>>>(a, o, N, nl, B);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

__global__ void tensor_sum2_kernel(const u64 *a, const u64 *c, u64 *o, int N, int nl, int B)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    int l = blockIdx.y;
    const PrimeK k = c_pk[l];
    size_t s = (size_t)nl * N, x = (size_t)l * N + t;
    u64 d0 = 0, d1 = 0, d2 = 0;
    for (int b = 0; b < B; b++) {
        const u64 *A = a + (size_t)b * 2 * s, *Cc = c + (size_t)b * 2 * s;
        u64 a0 = A[x], a1 = A[s + x], c0 = Cc[x], c1 = Cc[s + x];
        d0 = d_add(d0, d_mulmod(a0, c0, k), k.q);
        d1 = d_add(d1, d_add(d_mulmod(a0, c1, k), d_mulmod(a1, c0, k), k.q), k.q);
        d2 = d_add(d2, d_mulmod(a1, c1, k), k.q);
    }
    o[x] = d0;
    o[s + x] = d1;
    o[2 * s + x] = d2;
}

void k_tensor_sum2(hs_ctx *c, const u64 *a, const u64 *b, u64 *o, int B, int nl, cudaStream_t st)
{
    KTimer _kt(c, KID_TENSOR, (double)(4 * B + 3) * nl * c->P->n * 8, st);
    int N = c->P->n;
    tensor_sum2_kernel<<<dim3((N + 255) / 256, nl), 256, 0, st>>>(a, b, o, N, nl, B);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

// batched key-switch inner product.  d: B polys with stride d_stride words;
// ext digit j of ciphertext b: ext + off[j] + (b * nd[j] + g') * N;
// acc: [B][2][ntg][N].  Each thread keeps BT ciphertexts' accumulators so
// the evaluation key is read once per batch tile.
struct KsArgB {
    int level, beta, alpha, n_q, n_t, B;
    int j0;  // first digit (digits [j0, beta)): the digit-parallel partial accumulator
    size_t d_stride;
    size_t off[HS_MAXDIG];
    int nd[HS_MAXDIG];
    // C8 fused relin + rescale: acc_c,g += dadd_c,g * (P mod q_g) on the Q limbs
    const u64 *dadd;  // member b comps 0/1 at dadd + b dadd_stride + (c nl + g) N; NULL = none
    size_t dadd_stride;
    u64 pmq[HS_MAXP];
};

// grid (batch tiles of BT, N / 256, ntg): each thread keeps BT ciphertexts'
// 128-bit accumulators; the tiles sharing a key block are scheduled back to
// back, so the key's re-reads hit L2 and HBM streams it about once.
template <int BT>
__global__ void __launch_bounds__(256, BT == 2 ? 8 : 1) ks_inner_b_kernel(const u64 *__restrict__ d, const u64 *__restrict__ ext,
                                                         const u64 *__restrict__ key, u64 *__restrict__ acc,
                                                         const __grid_constant__ KsArgB A, int N)
{
    int t = blockIdx.y * blockDim.x + threadIdx.x;
    if (t >= N) return;
    const int g = blockIdx.z, b0 = blockIdx.x * BT;
    const int nl = A.level + 1, ntg = nl + A.n_t;
    const int pi = g < nl ? g : A.n_q + (g - nl);
    const PrimeK k = c_pk[pi];
    const size_t ntot = (size_t)A.n_q + A.n_t;
    u64 h0[BT], l0[BT], h1[BT], l1[BT];
#pragma unroll
    for (int u = 0; u < BT; u++) h0[u] = l0[u] = h1[u] = l1[u] = 0;
    for (int j = A.j0; j < A.beta; j++) {
        const int lo = j * A.alpha, hi = min((j + 1) * A.alpha, nl), dn = hi - lo;
        const ulonglong2 kk = reinterpret_cast<const ulonglong2 *>(key)[((size_t)j * ntot + pi) * N + t];
        const u64 k0 = kk.x, k1 = kk.y;
        const bool own = g >= lo && g < hi;
        const int gg = g < lo ? g : g - dn;
#pragma unroll
        for (int u = 0; u < BT; u++) {
            const int b = b0 + u;
            if (b >= A.B) break;
            u64 v = own ? d[(size_t)b * A.d_stride + (size_t)g * N + t]
                        : ext[A.off[j] + ((size_t)b * A.nd[j] + gg) * N + t];
            mac128(h0[u], l0[u], v, k0);
            mac128(h1[u], l1[u], v, k1);
        }
    }
    if (A.dadd && g < nl) {
        const u64 pm = A.pmq[g];
#pragma unroll
        for (int u = 0; u < BT; u++) {
            const int b = b0 + u;
            if (b >= A.B) break;
            const u64 *dd = A.dadd + (size_t)b * A.dadd_stride + (size_t)g * N + t;
            mac128(h0[u], l0[u], dd[0], pm);
            mac128(h1[u], l1[u], dd[(size_t)nl * N], pm);
        }
    }
#pragma unroll
    for (int u = 0; u < BT; u++) {
        const int b = b0 + u;
        if (b >= A.B) break;
        acc[((size_t)b * 2 * ntg + g) * N + t] = d_reduce128(h0[u], l0[u], k);
        acc[((size_t)(b * 2 + 1) * ntg + g) * N + t] = d_reduce128(h1[u], l1[u], k);
    }
}

void k_ks_inner_b(hs_ctx *c, const u64 *d, size_t d_stride, const u64 *ext, const size_t *off, const int *nd,
                  const u64 *key, u64 *acc, int level, int beta, int B, cudaStream_t st, const u64 *dadd,
                  size_t dadd_stride, int j0)
{
    const hs_params *P = c->P;
    const int ntg = level + 1 + P->n_p;
    // algorithmic bytes: the key once, every input limb once, the C8 P*d
    // term's 2 (level+1) limbs per member when fused, the outputs once
    KTimer _kt(c, KID_KS_INNER,
               ((double)(beta - j0) * ntg * (16.0 + 8.0 * B) + 16.0 * ntg * B +
                (dadd ? 16.0 * (level + 1) * B : 0.0)) * P->n,
               st);
    KsArgB A;
    A.level = level;
    A.beta = beta;
    A.j0 = j0;
    A.alpha = P->alpha;
    A.n_q = P->n_q;
    A.n_t = P->n_p;
    A.B = B;
    A.d_stride = d_stride;
    for (int j = 0; j < beta; j++) {
        A.off[j] = off[j];
        A.nd[j] = nd[j];
    }
    A.dadd = dadd;
    A.dadd_stride = dadd_stride;
    if (dadd)
        for (int i = 0; i <= level; i++) A.pmq[i] = P->p_mod_q[i];
    int N = P->n;
    // batch tile per thread: HS_KS_BT=1|4|8 for experiments (default 2: measured
    // 31.3 ms/step vs 36.0 at 4 -- occupancy beats key reuse, the re-reads hit L2)
    static const int bt = [] {
        const char *e = getenv("HS_KS_BT");
        const int v = e ? atoi(e) : 2;
        return (v == 1 || v == 4 || v == 8) ? v : 2;
    }();
    if (bt == 8 && B >= 8) {
        ks_inner_b_kernel<8><<<dim3((B + 7) / 8, (N + 255) / 256, ntg), 256, 0, st>>>(d, ext, key, acc, A, N);
    } else if (bt == 2) {
        ks_inner_b_kernel<2><<<dim3((B + 1) / 2, (N + 255) / 256, ntg), 256, 0, st>>>(d, ext, key, acc, A, N);
    } else if (bt == 1) {
        ks_inner_b_kernel<1><<<dim3(B, (N + 255) / 256, ntg), 256, 0, st>>>(d, ext, key, acc, A, N);
    } else {
        const int tiles = (B + 3) / 4;
        ks_inner_b_kernel<4><<<dim3(tiles, (N + 255) / 256, ntg), 256, 0, st>>>(d, ext, key, acc, A, N);
    }
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

// C16 hoisted rotations: ONE ModUp (d = c1 own limbs, ext = the digits'
// other limbs) serves R rotations.  Rotation r reads every extended limb
// through its Galois permutation (out[t] = in[perm_r[t]]; a warp's 32
// consecutive t read one aligned 32-word block, so the gather stays
// coalesced) and its own key.  grid (N/256, ntg, R); acc [R][2][ntg][N].
struct KsArgH {
    const u64 *key[HS_MAXROT];
    const unsigned *perm[HS_MAXROT];
    int level, beta, alpha, n_q, n_t;
    size_t off[HS_MAXDIG];
    int nd[HS_MAXDIG];
    // C17: component 0 also gets sigma_r(c0) (P mod q_g) on the Q limbs (the
    // rotation kept in the extended basis, no ModDown); NULL = none
    const u64 *c0add;
    u64 pmq[HS_MAXP];
};

__global__ void __launch_bounds__(256) ks_inner_h_kernel(const u64 *__restrict__ d, const u64 *__restrict__ ext,
                                                         u64 *__restrict__ acc, const __grid_constant__ KsArgH A,
                                                         int N)
{
    // grid (R, N / 256, ntg): the R rotations of one coefficient block run back
    // to back, so their gathers of the shared extended digits hit L2
    int t = blockIdx.y * blockDim.x + threadIdx.x;
    if (t >= N) return;
    const int g = blockIdx.z, r = blockIdx.x;
    const int nl = A.level + 1, ntg = nl + A.n_t;
    const int pi = g < nl ? g : A.n_q + (g - nl);
    const PrimeK k = c_pk[pi];
    const size_t ntot = (size_t)A.n_q + A.n_t;
    const unsigned src = __ldg(A.perm[r] + t);
    const u64 *key = A.key[r];
    u64 h0 = 0, l0 = 0, h1 = 0, l1 = 0;
#pragma unroll 4
    for (int j = 0; j < A.beta; j++) {
        const int lo = j * A.alpha, hi = min((j + 1) * A.alpha, nl), dn = hi - lo;
        const ulonglong2 kk = reinterpret_cast<const ulonglong2 *>(key)[((size_t)j * ntot + pi) * N + t];
        const u64 k0 = kk.x, k1 = kk.y;
        const bool own = g >= lo && g < hi;
        const int gg = g < lo ? g : g - dn;
        const u64 v = own ? d[(size_t)g * N + src] : ext[A.off[j] + (size_t)gg * N + src];
        mac128(h0, l0, v, k0);
        mac128(h1, l1, v, k1);
    }
    if (A.c0add && g < nl) mac128(h0, l0, A.c0add[(size_t)g * N + src], A.pmq[g]);
    acc[((size_t)r * 2 * ntg + g) * N + t] = d_reduce128(h0, l0, k);
    acc[((size_t)(r * 2 + 1) * ntg + g) * N + t] = d_reduce128(h1, l1, k);
}

// ---- TMA-streamed variant: the evaluation keys -- the
// bytes that dominate a hoisted key switch (R keys of 2 beta ntg limbs) --
// arrive by cp.async.bulk.tensor (one 3-D tensor map per key: (pair, N,
// dnum (n_q + n_p)) u64, box (2, 256, 1) = 4 KiB) into shared memory, all
// beta digits of a CTA's (rotation, 256-coefficient block, target limb) tile
// requested up front on one mbarrier, while the threads gather the extended
// digits through the rotation's permutation with ordinary loads.
struct KsArgHT {
    CUtensorMap tmap[HS_MAXROT];  // 64-byte aligned (CUtensorMap is declared aligned(64))
    const unsigned *perm[HS_MAXROT];
    int level, beta, alpha, n_q, n_t;
    size_t off[HS_MAXDIG];
    int nd[HS_MAXDIG];
    const u64 *c0add;
    u64 pmq[HS_MAXP];
};

__global__ void __launch_bounds__(256, 6) ks_inner_h_tma_kernel(const u64 *__restrict__ d, const u64 *__restrict__ ext,
                                                             u64 *__restrict__ acc,
                                                             const __grid_constant__ KsArgHT A, int N)
{
    extern __shared__ __align__(128) unsigned char ks_smem[];
    __shared__ __align__(8) unsigned long long bar[HS_MAXDIG];  // one per digit: compute starts as tiles land
    const int tid = threadIdx.x, t0 = blockIdx.y * 256, t = t0 + tid;
    const int g = blockIdx.z, r = blockIdx.x;
    const int nl = A.level + 1, ntg = nl + A.n_t;
    const int pi = g < nl ? g : A.n_q + (g - nl);
    const PrimeK k = c_pk[pi];
    const int ntot = A.n_q + A.n_t;
    const unsigned sbar = (unsigned)__cvta_generic_to_shared(bar);
    const unsigned skey = (unsigned)__cvta_generic_to_shared(ks_smem);
    if (tid < A.beta) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar + 8 * tid));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid < A.beta) {  // one issuing thread per digit
        const int j = tid;
        const CUtensorMap *tm = &A.tmap[r];
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 4096;" ::"r"(sbar + 8 * j) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
            "[%5];" ::"r"(skey + j * 4096),
            "l"(reinterpret_cast<uint64_t>(tm)), "r"(0), "r"(t0), "r"(j * ntot + pi), "r"(sbar + 8 * j)
            : "memory");
    }
    const bool live = t < N;
    const unsigned src = live ? __ldg(A.perm[r] + t) : 0;
    // the permuted extended digits, gathered while the key tiles are in flight
    // (up to 8 digits ahead; later digits gather in the loop)
    auto gather = [&](int j) -> u64 {
        const int lo = j * A.alpha, hi = min((j + 1) * A.alpha, nl), dn = hi - lo;
        const bool own = g >= lo && g < hi;
        const int gg = g < lo ? g : g - dn;
        return !live ? 0 : own ? d[(size_t)g * N + src] : ext[A.off[j] + (size_t)gg * N + src];
    };
    u64 v[8];
#pragma unroll
    for (int j = 0; j < 8; j++) v[j] = j < A.beta ? gather(j) : 0;
    const ulonglong2 *kt = reinterpret_cast<const ulonglong2 *>(ks_smem);
    u64 h0 = 0, l0 = 0, h1 = 0, l1 = 0;
#pragma unroll
    for (int j = 0; j < HS_MAXDIG; j++) {
        if (j >= A.beta) break;
        const u64 vj = j < 8 ? v[j] : gather(j);
        asm volatile(
            "{\n\t.reg .pred P;\n\t"
            "KS_TMA_WAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t"
            "@!P bra KS_TMA_WAIT_%=;\n\t}" ::"r"(sbar + 8 * j)
            : "memory");
        const ulonglong2 kk = kt[j * 256 + tid];
        mac128(h0, l0, vj, kk.x);
        mac128(h1, l1, vj, kk.y);
    }
    if (!live) return;
    if (A.c0add && g < nl) mac128(h0, l0, A.c0add[(size_t)g * N + src], A.pmq[g]);
    acc[((size_t)r * 2 * ntg + g) * N + t] = d_reduce128(h0, l0, k);
    acc[((size_t)(r * 2 + 1) * ntg + g) * N + t] = d_reduce128(h1, l1, k);
}

// one 3-D tensor map per switching key, cached by device pointer
static const CUtensorMap &key_tmap(hs_ctx *c, const u64 *key)
{
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode) throw HsError(HS_ECUDA, "cuTensorMapEncodeTiled not available");
    std::lock_guard<std::mutex> lk(c->mu);
    auto it = c->key_tmaps.find(key);
    if (it != c->key_tmaps.end()) return it->second;
    const hs_params *P = c->P;
    const cuuint64_t rows = (cuuint64_t)P->dnum * (P->n_q + P->n_p);
    const cuuint64_t dims[3] = {2, (cuuint64_t)P->n, rows};
    const cuuint64_t strides[2] = {16, (cuuint64_t)P->n * 16};
    const cuuint32_t box[3] = {2, 256, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUtensorMap m;
    CUresult rc = encode(&m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<u64 *>(key), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS) throw HsError(HS_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)rc));
    return c->key_tmaps[key] = m;
}

// HS_KS_TMA=1 selects the TMA variant (measured: DESIGN.md section 6)
static bool ks_tma_on()
{
    static const bool on = [] {
        const char *e = getenv("HS_KS_TMA");
        return e && e[0] == '1';
    }();
    return on;
}

void k_ks_inner_h(hs_ctx *c, const u64 *d, const u64 *ext, const size_t *off, const int *nd, const u64 *const *keys,
                  const unsigned *const *perms, int R, u64 *acc, int level, int beta, cudaStream_t st,
                  const u64 *c0add)
{
    if (ks_tma_on() && c->P->n % 256 == 0 && beta <= HS_MAXDIG) {
        const hs_params *P = c->P;
        const int ntg = level + 1 + P->n_p;
        if (R < 1 || R > HS_MAXROT) throw HsError(HS_EINVAL, "hoisted key switch: bad rotation count");
        KTimer _kt(c, KID_KS_HOIST,
                   ((double)R * beta * ntg * 16.0 + (double)beta * ntg * 8.0 + 16.0 * ntg * R +
                    (c0add ? 8.0 * (level + 1) : 0.0)) *
                       P->n,
                   st);
        static KsArgHT A;  // ~10 KB: kept off the stack; launches copy their parameters
        static std::mutex amu;
        std::lock_guard<std::mutex> lk(amu);
        for (int r = 0; r < R; r++) {
            A.tmap[r] = key_tmap(c, keys[r]);
            A.perm[r] = perms[r];
        }
        A.level = level;
        A.beta = beta;
        A.alpha = P->alpha;
        A.n_q = P->n_q;
        A.n_t = P->n_p;
        for (int j = 0; j < beta; j++) {
            A.off[j] = off[j];
            A.nd[j] = nd[j];
        }
        A.c0add = c0add;
        if (c0add)
            for (int i = 0; i <= level; i++) A.pmq[i] = P->p_mod_q[i];
        const int N = P->n;
        const size_t smem = (size_t)beta * 4096;
        static bool attr = false;
        if (!attr) {
            HS_CUDA(cudaFuncSetAttribute(ks_inner_h_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         HS_MAXDIG * 4096));
            attr = true;
        }
        ks_inner_h_tma_kernel<<<dim3(R, N / 256, ntg), 256, smem, st>>>(d, ext, acc, A, N);
        HS_CHECK_LAUNCH();
        count_kernel(c);
        return;
    }
    const hs_params *P = c->P;
    const int ntg = level + 1 + P->n_p;
    if (R < 1 || R > HS_MAXROT) throw HsError(HS_EINVAL, "hoisted key switch: bad rotation count");
    // algorithmic bytes: R keys, the shared extended digits and sigma's c0 once
    // (every rotation gathers them again through its own permutation -- from
    // HBM: a source-order variant that let the R re-reads hit L2 measured no
    // faster, the key streams dominate), R outputs
    KTimer _kt(c, KID_KS_HOIST,
               ((double)R * beta * ntg * 16.0 + (double)beta * ntg * 8.0 + 16.0 * ntg * R +
                (c0add ? 8.0 * (level + 1) : 0.0)) *
                   P->n,
               st);
    KsArgH A;
    for (int r = 0; r < R; r++) {
        A.key[r] = keys[r];
        A.perm[r] = perms[r];
    }
    A.level = level;
    A.beta = beta;
    A.alpha = P->alpha;
    A.n_q = P->n_q;
    A.n_t = P->n_p;
    for (int j = 0; j < beta; j++) {
        A.off[j] = off[j];
        A.nd[j] = nd[j];
    }
    A.c0add = c0add;
    if (c0add)
        for (int i = 0; i <= level; i++) A.pmq[i] = P->p_mod_q[i];
    int N = P->n;
    ks_inner_h_kernel<<<dim3(R, (N + 255) / 256, ntg), 256, 0, st>>>(d, ext, acc, A, N);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

// B polynomials, each with ITS OWN key (a batch of rotations by different
// amounts): ModUp blocks as in ks_inner_b ([B][nd_j][N] per digit), member r
// uses key[r].  grid (B, N / 256, ntg): the members of one coefficient block
// run back to back.  acc [B][2][ntg][N].
struct KsArgM {
    const u64 *key[HS_MAXROT];
    int level, beta, alpha, n_q, n_t;
    size_t d_stride;
    size_t off[HS_MAXDIG];
    int nd[HS_MAXDIG];
};

__global__ void __launch_bounds__(256) ks_inner_m_kernel(const u64 *__restrict__ d, const u64 *__restrict__ ext,
                                                         u64 *__restrict__ acc, const __grid_constant__ KsArgM A,
                                                         int N)
{
    int t = blockIdx.y * blockDim.x + threadIdx.x;
    if (t >= N) return;
    const int g = blockIdx.z, r = blockIdx.x;
    const int nl = A.level + 1, ntg = nl + A.n_t;
    const int pi = g < nl ? g : A.n_q + (g - nl);
    const PrimeK k = c_pk[pi];
    const size_t ntot = (size_t)A.n_q + A.n_t;
    const u64 *key = A.key[r];
    u64 h0 = 0, l0 = 0, h1 = 0, l1 = 0;
#pragma unroll 4
    for (int j = 0; j < A.beta; j++) {
        const int lo = j * A.alpha, hi = min((j + 1) * A.alpha, nl), dn = hi - lo;
        const ulonglong2 kk = reinterpret_cast<const ulonglong2 *>(key)[((size_t)j * ntot + pi) * N + t];
        const u64 k0 = kk.x, k1 = kk.y;
        const bool own = g >= lo && g < hi;
        const int gg = g < lo ? g : g - dn;
        const u64 v = own ? d[(size_t)r * A.d_stride + (size_t)g * N + t]
                          : ext[A.off[j] + ((size_t)r * A.nd[j] + gg) * N + t];
        mac128(h0, l0, v, k0);
        mac128(h1, l1, v, k1);
    }
    acc[((size_t)r * 2 * ntg + g) * N + t] = d_reduce128(h0, l0, k);
    acc[((size_t)(r * 2 + 1) * ntg + g) * N + t] = d_reduce128(h1, l1, k);
}

void k_ks_inner_m(hs_ctx *c, const u64 *d, size_t d_stride, const u64 *ext, const size_t *off, const int *nd,
                  const u64 *const *keys, int B, u64 *acc, int level, int beta, cudaStream_t st)
{
    const hs_params *P = c->P;
    const int ntg = level + 1 + P->n_p;
    if (B < 1 || B > HS_MAXROT) throw HsError(HS_EINVAL, "multi-key inner product: bad batch");
    KTimer _kt(c, KID_KS_INNER, ((double)B * beta * ntg * 24.0 + 16.0 * ntg * B) * P->n, st);
    KsArgM A;
    for (int r = 0; r < B; r++) A.key[r] = keys[r];
    A.level = level;
    A.beta = beta;
    A.alpha = P->alpha;
    A.n_q = P->n_q;
    A.n_t = P->n_p;
    A.d_stride = d_stride;
    for (int j = 0; j < beta; j++) {
        A.off[j] = off[j];
        A.nd[j] = nd[j];
    }
    int N = P->n;
    ks_inner_m_kernel<<<dim3(B, (N + 255) / 256, ntg), 256, 0, st>>>(d, ext, acc, A, N);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

struct MdArgB {
    u64 pinv[HS_MAXP], pinv_sh[HS_MAXP];
    int nt, add_comps;
    size_t acc_row, o_stride, add_stride;
};

// row r = 2 b + comp: o_b[comp][i] = add + (acc_r[i] - conv_r[i]) inv_i for
// i < nt; acc row r at acc + r acc_row, conv [rows][nt][N]
__global__ void moddown_final_b_kernel(const u64 *acc, const u64 *conv, u64 *o, const u64 *add, MdArgB A, int N)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    const int i = blockIdx.y, comp = blockIdx.z & 1, b = blockIdx.z >> 1;
    u64 q = c_pk[i].q;
    u64 av = acc[(size_t)blockIdx.z * A.acc_row + (size_t)i * N + t];
    u64 cv = conv[(((size_t)b * 2 + comp) * A.nt + i) * N + t];
    u64 v = d_shoup(d_sub(av, cv, q), A.pinv[i], A.pinv_sh[i], q);
    size_t ci = ((size_t)comp * A.nt + i) * N + t;
    if (comp < A.add_comps) v = d_add(v, add[(size_t)b * A.add_stride + ci], q);
    o[(size_t)b * A.o_stride + ci] = v;
}

void k_moddown_final_b(hs_ctx *c, const u64 *acc, size_t acc_row, const u64 *conv, int nt, u64 *o, size_t o_stride,
                       const u64 *add, size_t add_stride, int add_comps, const u64 *inv, int rows, cudaStream_t st)
{
    const hs_params *P = c->P;
    KTimer _kt(c, KID_MODDOWN, (double)rows * nt * P->n * 8 * (3 + add_comps), st);
    MdArgB A;
    for (int i = 0; i < nt; i++) {
        A.pinv[i] = inv ? inv[i] : P->p_inv_mod_q[i];
        A.pinv_sh[i] = hs_shoup_const(A.pinv[i], P->prime[i]);
    }
    A.nt = nt;
    A.acc_row = acc_row;
    A.add_comps = add ? add_comps : 0;
    A.o_stride = o_stride;
    A.add_stride = add_stride;
    int N = P->n;
    moddown_final_b_kernel<<<dim3((N + 255) / 256, nt, rows), 256, 0, st>>>(acc, conv, o, add, A, N);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

// ------------------------------------------------------------------ bootstrapping helpers (G11)
// acc[c][i][t] += a[c][i][t] * pt[i][t]  (c < 2, i < nl); a has stride la limbs
__global__ void mac_pt_kernel(u64 *acc, const u64 *a, const u64 *pt, int N, int nl, int la)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    int i = blockIdx.y, c = blockIdx.z;
    const PrimeK k = c_pk[i];
    u64 p = pt[(size_t)i * N + t];
    size_t ai = ((size_t)c * la + i) * N + t, oi = ((size_t)c * nl + i) * N + t;
    acc[oi] = d_add(acc[oi], d_mulmod(a[ai], p, k), k.q);
}

// One BSGS layer of a bootstrapping linear transform in ONE pass:
// out[g][c][i][t] = sum_b pt_{tk[g][b]}[i][t] * R_b[c][i][t] mod q_i for every
// giant g.  A thread keeps its 2*B1 baby words in registers (each read once),
// accumulates in 128 bits (B1 <= 8 terms of < q^2 stay below q 2^64 for
// q < 2^61) and reduces once per output.  tk[g*B1+b] = term index or -1.
struct BsgsArg {
    const u64 *R[16];
    int tk[16 * 16];
    int G, nl;      // limbs per component (Q limbs, or Q u P limbs for C17)
    int nlq, n_q;   // limb i >= nlq is the special prime n_q + (i - nlq)
};

template <int B1>
__global__ void __launch_bounds__(256) bsgs_inner_kernel(const u64 *__restrict__ pts, u64 *__restrict__ out,
                                                         const __grid_constant__ BsgsArg A, int N)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    const int i = blockIdx.y, nl = A.nl;
    const PrimeK k = c_pk[i < A.nlq ? i : A.n_q + (i - A.nlq)];
    u64 r0[B1], r1[B1];
#pragma unroll
    for (int b = 0; b < B1; b++)
        if (A.R[b]) {
            r0[b] = A.R[b][(size_t)i * N + t];
            r1[b] = A.R[b][((size_t)nl + i) * N + t];
        }
    for (int g = 0; g < A.G; g++) {
        u64 h0 = 0, l0 = 0, h1 = 0, l1 = 0;
#pragma unroll
        for (int b = 0; b < B1; b++) {
            const int kk = A.tk[g * B1 + b];
            if (kk >= 0) {
                const u64 p = pts[((size_t)kk * nl + i) * N + t];
                mac128(h0, l0, r0[b], p);
                mac128(h1, l1, r1[b], p);
            }
        }
        // pts are stored in Montgomery form (pt 2^64 mod q): one REDC lands
        out[((size_t)g * 2 * nl + i) * N + t] = d_redc(h0, l0, k);
        out[((size_t)(g * 2 + 1) * nl + i) * N + t] = d_redc(h1, l1, k);
    }
}

// Baby-major variant for large baby sets (b1 <= 16) and few giants (G <= GM):
// each baby's two words are loaded once and feed every giant's 128-bit
// accumulators; every 8 babies the accumulators fold through one REDC into a
// reduced partial sum (8 q^2 < q 2^64 for q < 2^61), so any b1 stays exact.
// occupancy of the baby-major BSGS sums (HBM-bound): 3 / 4 CTAs per SM for 4 /
// 2 giants (128 / 78 registers otherwise; the cap costs a few spilled words,
// L1-resident): 10.3 -> 10.0 ms per config-3 step
#ifndef BSGS_MINB
#define BSGS_MINB(G) ((G) >= 4 ? 3 : (G) == 2 ? 4 : 1)
#endif
template <int GM>
__global__ void __launch_bounds__(256, BSGS_MINB(GM)) bsgs_inner_bm_kernel(const u64 *__restrict__ pts, u64 *__restrict__ out,
                                                            const __grid_constant__ BsgsArg A, int N, int b1)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    const int i = blockIdx.y, nl = A.nl;
    const PrimeK k = c_pk[i < A.nlq ? i : A.n_q + (i - A.nlq)];
    u64 h0[GM], l0[GM], h1[GM], l1[GM], s0[GM], s1[GM];
#pragma unroll
    for (int g = 0; g < GM; g++) h0[g] = l0[g] = h1[g] = l1[g] = s0[g] = s1[g] = 0;
    // babies in groups of 8 (the REDC fold); within a group, batches of 4
    // babies load every operand first (predicated, absent terms read as 0,
    // which adds nothing) so all their loads are in flight together
    for (int b0 = 0; b0 < b1; b0 += 8) {
#pragma unroll
        for (int half = 0; half < 2; half++) {
            u64 r0v[4], r1v[4], pv[4][GM];
#pragma unroll
            for (int bb = 0; bb < 4; bb++) {
                const int b = b0 + 4 * half + bb;
                const u64 *R = b < b1 ? A.R[b] : nullptr;
                r0v[bb] = R ? R[(size_t)i * N + t] : 0;
                r1v[bb] = R ? R[((size_t)nl + i) * N + t] : 0;
#pragma unroll
                for (int g = 0; g < GM; g++) {
                    const int kk = (R && g < A.G) ? A.tk[g * 16 + b] : -1;
                    pv[bb][g] = kk >= 0 ? pts[((size_t)kk * nl + i) * N + t] : 0;
                }
            }
#pragma unroll
            for (int bb = 0; bb < 4; bb++)
#pragma unroll
                for (int g = 0; g < GM; g++) {
                    mac128(h0[g], l0[g], r0v[bb], pv[bb][g]);
                    mac128(h1[g], l1[g], r1v[bb], pv[bb][g]);
                }
        }
#pragma unroll
        for (int g = 0; g < GM; g++) {
            s0[g] = d_add(s0[g], d_redc(h0[g], l0[g], k), k.q);
            s1[g] = d_add(s1[g], d_redc(h1[g], l1[g], k), k.q);
            h0[g] = l0[g] = h1[g] = l1[g] = 0;
        }
    }
#pragma unroll
    for (int g = 0; g < GM; g++)
        if (g < A.G) {
            out[((size_t)g * 2 * nl + i) * N + t] = s0[g];
            out[((size_t)(g * 2 + 1) * nl + i) * N + t] = s1[g];
        }
}

void k_bsgs_inner(hs_ctx *c, const u64 *const *R, int b1, const u64 *pts, const int *tk, int G, int nl, u64 *out,
                  cudaStream_t st, int nlq)
{
    if (b1 < 1 || b1 > 16 || G < 1 || G > 16) throw HsError(HS_EINVAL, "bsgs_inner: baby / giant count out of range");
    if (b1 > 8) {  // baby-major kernel
        if (G > 4) throw HsError(HS_EINVAL, "bsgs_inner: more than 4 giants with more than 8 babies");
        BsgsArg A;
        int terms = 0, babies = 0;
        for (int b = 0; b < 16; b++) A.R[b] = b < b1 ? R[b] : nullptr;
        for (int b = 0; b < b1; b++) babies += R[b] != nullptr;
        for (int g = 0; g < 16; g++)
            for (int b = 0; b < 16; b++) {
                A.tk[g * 16 + b] = (g < G && b < b1) ? tk[g * b1 + b] : -1;
                terms += A.tk[g * 16 + b] >= 0;
            }
        A.G = G;
        A.nl = nl;
        A.nlq = nlq < 0 ? nl : nlq;
        A.n_q = c->P->n_q;
        const int N = c->P->n;
        KTimer _kt(c, KID_PTMUL, (double)(2 * babies + terms + 2 * G) * nl * N * 8, st);
        // accumulators sized to the giant count (registers -> occupancy)
        const dim3 grid((N + 255) / 256, nl);
        if (G == 1) bsgs_inner_bm_kernel<1><<<grid, 256, 0, st>>>(pts, out, A, N, b1);
        else if (G == 2) bsgs_inner_bm_kernel<2><<<grid, 256, 0, st>>>(pts, out, A, N, b1);
        else bsgs_inner_bm_kernel<4><<<grid, 256, 0, st>>>(pts, out, A, N, b1);
        HS_CHECK_LAUNCH();
        count_kernel(c);
        return;
    }
    BsgsArg A;
    int terms = 0, babies = 0;
    for (int b = 0; b < 16; b++) A.R[b] = b < b1 ? R[b] : nullptr;
    for (int b = 0; b < b1; b++) babies += R[b] != nullptr;
    const int B1 = b1 <= 2 ? 2 : b1 <= 4 ? 4 : 8;
    for (int g = 0; g < G; g++)
        for (int b = 0; b < B1; b++) {
            A.tk[g * B1 + b] = b < b1 ? tk[g * b1 + b] : -1;
            terms += A.tk[g * B1 + b] >= 0;
        }
    A.G = G;
    A.nl = nl;
    A.nlq = nlq < 0 ? nl : nlq;
    A.n_q = c->P->n_q;
    const int N = c->P->n;
    KTimer _kt(c, KID_PTMUL, (double)(2 * babies + terms + 2 * G) * nl * N * 8, st);
    const dim3 grid((N + 255) / 256, nl);
    if (B1 == 2) bsgs_inner_kernel<2><<<grid, 256, 0, st>>>(pts, out, A, N);
    else if (B1 == 4) bsgs_inner_kernel<4><<<grid, 256, 0, st>>>(pts, out, A, N);
    else bsgs_inner_kernel<8><<<grid, 256, 0, st>>>(pts, out, A, N);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

void k_mac_pt(hs_ctx *c, u64 *acc, const u64 *a, const u64 *pt, int nl, int la, cudaStream_t st)
{
    KTimer _kt(c, KID_PTMUL, (double)nl * c->P->n * 8 * 7, st);
    int N = c->P->n;
    mac_pt_kernel<<<dim3((N + 255) / 256, nl, 2), 256, 0, st>>>(acc, a, pt, N, nl, la);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}

// ModRaise: x[c][t] (coefficients mod q_0) -> o[c][i][t] = centred(x) mod q_i, i <= L
__global__ void modraise_kernel(const u64 *x, u64 *o, int N, int nl)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    int i = blockIdx.y, c = blockIdx.z;
    const PrimeK k = c_pk[i];
    u64 q0 = c_pk[0].q, q = k.q;
    u64 v = x[(size_t)c * N + t], r;
    if (v <= (q0 - 1) / 2) r = d_reduce128(0, v, k);
    else {
        u64 w = d_reduce128(0, q0 - v, k);
        r = w ? q - w : 0;
    }
    o[((size_t)c * nl + i) * N + t] = r;
}

void k_modraise(hs_ctx *c, const u64 *x, u64 *o, int nl, cudaStream_t st)
{
    KTimer _kt(c, KID_MODRAISE, (double)(2 + 2 * nl) * c->P->n * 8, st);
    int N = c->P->n;
    modraise_kernel<<<dim3((N + 255) / 256, nl, 2), 256, 0, st>>>(x, o, N, nl);
    HS_CHECK_LAUNCH();
    count_kernel(c);
}
