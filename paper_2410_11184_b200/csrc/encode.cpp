// encode.cpp -- canonical-embedding encode / decode on the host (C4).
//
// PAPER.md 248-253: CKKS messages are C^{N/2}; slot j is the evaluation of
// the plaintext polynomial at zeta^(5^j mod 2N), zeta = exp(i pi / N).
// encode: m_t = rint( Delta (2/N) Re sum_j z_j zeta^(-g_j t) ),  g_j = 5^j mod 2N
// computed as a length-2N DFT in __float128 (decimation in frequency) so the
// rounding decision is made on a value accurate to ~2^-100 relative.
#include <quadmath.h>

#include <vector>

#include "hs_internal.h"

typedef __float128 f128;

namespace {

struct Cq {
    f128 re, im;
};

struct Twiddles {
    int log_n2 = -1;
    std::vector<Cq> w;  // exp(-2 pi i k / n2), k < n2/2
};

Twiddles &twiddles(int log_n2)
{
    static thread_local Twiddles T;
    if (T.log_n2 != log_n2) {
        int n2 = 1 << log_n2;
        T.w.resize(n2 / 2);
        for (int k = 0; k < n2 / 2; k++) {
            f128 a = -2 * M_PIq * (f128)k / (f128)n2;
            T.w[k].re = cosq(a);
            T.w[k].im = sinq(a);
        }
        T.log_n2 = log_n2;
    }
    return T;
}

// Decimation-in-frequency radix-2 DFT, natural order in, natural order out
// (bit-reversal permutation at the end).  sign < 0: exp(-..), > 0: exp(+..).
void dft(std::vector<Cq> &a, int log_n2, int sign)
{
    const int n2 = 1 << log_n2;
    const Twiddles &T = twiddles(log_n2);
    for (int len = n2; len >= 2; len >>= 1) {
        const int half = len >> 1, step = n2 / len;
        for (int s = 0; s < n2; s += len)
            for (int k = 0; k < half; k++) {
                Cq w = T.w[k * step];
                if (sign > 0) w.im = -w.im;
                Cq u = a[s + k], v = a[s + k + half];
                a[s + k] = Cq{u.re + v.re, u.im + v.im};
                f128 dr = u.re - v.re, di = u.im - v.im;
                a[s + k + half] = Cq{dr * w.re - di * w.im, dr * w.im + di * w.re};
            }
    }
    for (int i = 0, j = 0; i < n2; i++) {
        if (i < j) std::swap(a[i], a[j]);
        int bit = n2 >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j |= bit;
    }
}

}  // namespace

static void encode_from(const hs_params *P, std::vector<Cq> &a, double scale, int level, u64 *out, bool with_p = false);

void hs_encode_impl(const hs_params *P, const double *re, const double *im, double scale, int level, u64 *out)
{
    const int N = P->n, n0 = N / 2, n2 = 2 * N;
    std::vector<Cq> a(n2, Cq{0, 0});
    u64 g = 1;
    for (int j = 0; j < n0; j++) {
        a[g] = Cq{(f128)re[j], im ? (f128)im[j] : (f128)0};
        g = g * 5 % (u64)n2;
    }
    encode_from(P, a, scale, level, out);
}

// quad-precision slot values (bootstrapping diagonals, G11)
void hs_encode_impl_q(const hs_params *P, const __float128 *re, const __float128 *im, double scale, int level,
                      u64 *out, bool with_p)
{
    const int N = P->n, n0 = N / 2, n2 = 2 * N;
    std::vector<Cq> a(n2, Cq{0, 0});
    u64 g = 1;
    for (int j = 0; j < n0; j++) {
        a[g] = Cq{re[j], im[j]};
        g = g * 5 % (u64)n2;
    }
    encode_from(P, a, scale, level, out, with_p);
}

// with_p: also the residues mod p_0..p_{np-1} after the level+1 Q limbs (the
// extended basis of the double-hoisted BSGS plaintexts, C17)
static void encode_from(const hs_params *P, std::vector<Cq> &a, double scale, int level, u64 *out, bool with_p)
{
    const int N = P->n, lg = P->log_n + 1;
    dft(a, lg, -1);
    const f128 f = (f128)scale * 2 / (f128)N;
    for (int t = 0; t < N; t++) {
        f128 v = rintq(a[t].re * f);
        __int128 m = (__int128)v;
        for (int i = 0; i <= level; i++) {
            __int128 q = (__int128)P->prime[i], r = m % q;
            out[(size_t)i * N + t] = (u64)(r < 0 ? r + q : r);
        }
        for (int k = 0; with_p && k < P->n_p; k++) {
            __int128 q = (__int128)P->prime[P->n_q + k], r = m % q;
            out[(size_t)(level + 1 + k) * N + t] = (u64)(r < 0 ? r + q : r);
        }
    }
}

void hs_decode_impl(const hs_params *P, const u64 *q0c, double scale, double *re, double *im)
{
    const int N = P->n, n0 = N / 2, n2 = 2 * N, lg = P->log_n + 1;
    const u64 q0 = P->prime[0];
    std::vector<Cq> a(n2, Cq{0, 0});
    for (int t = 0; t < N; t++) a[t].re = q0c[t] > q0 / 2 ? -(f128)(q0 - q0c[t]) : (f128)q0c[t];
    dft(a, lg, +1);
    u64 g = 1;
    for (int j = 0; j < n0; j++) {
        re[j] = (double)(a[g].re / (f128)scale);
        if (im) im[j] = (double)(a[g].im / (f128)scale);
        g = g * 5 % (u64)n2;
    }
}
