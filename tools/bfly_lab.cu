// bfly_lab.cu -- dev tool: the arithmetic ceiling of a 64-bit Shoup butterfly
// on this GPU (registers only, no memory), to compare with the NTT kernels'
// achieved butterflies/s.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;

__device__ __forceinline__ u64 shoup_lazy(u64 a, u64 w, u64 ws, u64 q) { return a * w - __umul64hi(a, ws) * q; }

// the same value from 32-bit multiply-add chains (nq = 2^64 - q)
__device__ __forceinline__ u64 shoup_lazy_ptx(u64 a, u64 w, u64 ws, u64 nq)
{
    u64 r;
    asm("{\n\t"
        ".reg .u32 a0, a1, w0, w1, s0, s1, n0, n1, t0, t1, t2, r0, r1;\n\t"
        "mov.b64 {a0, a1}, %1;\n\t"
        "mov.b64 {w0, w1}, %2;\n\t"
        "mov.b64 {s0, s1}, %3;\n\t"
        "mov.b64 {n0, n1}, %4;\n\t"
        "mul.hi.u32 t0, a0, s0;\n\t"
        "mad.lo.cc.u32 t0, a0, s1, t0;\n\t"
        "madc.hi.u32 t1, a0, s1, 0;\n\t"
        "mad.lo.cc.u32 t0, a1, s0, t0;\n\t"
        "madc.hi.cc.u32 t1, a1, s0, t1;\n\t"
        "madc.hi.u32 t2, a1, s1, 0;\n\t"
        "mad.lo.cc.u32 t1, a1, s1, t1;\n\t"
        "addc.u32 t2, t2, 0;\n\t"
        "mul.lo.u32 r0, a0, w0;\n\t"
        "mul.hi.u32 r1, a0, w0;\n\t"
        "mad.lo.u32 r1, a0, w1, r1;\n\t"
        "mad.lo.u32 r1, a1, w0, r1;\n\t"
        "mad.lo.cc.u32 r0, t1, n0, r0;\n\t"
        "madc.hi.u32 r1, t1, n0, r1;\n\t"
        "mad.lo.u32 r1, t1, n1, r1;\n\t"
        "mad.lo.u32 r1, t2, n0, r1;\n\t"
        "mov.b64 %0, {r0, r1};\n\t"
        "}"
        : "=l"(r)
        : "l"(a), "l"(w), "l"(ws), "l"(nq));
    return r;
}

// Shoup with the quotient's a0*s0 partial product dropped: hi' in {hi - 1, hi},
// so the result lies in [0, 3q) (q < 2^61 keeps 3q < 2^64)
__device__ __forceinline__ u64 shoup_approx(u64 a, u64 w, u64 ws, u64 nq)
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
        : "l"(a), "l"(w), "l"(ws), "l"(nq));
    return r;
}

// 64-bit a + b and a - b as explicit 32-bit carry chains (ALU pipe adds)
__device__ __forceinline__ u64 add64(u64 a, u64 b)
{
    u64 r;
    asm("{\n\t.reg .u32 a0, a1, b0, b1;\n\tmov.b64 {a0, a1}, %1;\n\tmov.b64 {b0, b1}, %2;\n\t"
        "add.cc.u32 a0, a0, b0;\n\taddc.u32 a1, a1, b1;\n\tmov.b64 %0, {a0, a1};\n\t}"
        : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 sub64(u64 a, u64 b)
{
    u64 r;
    asm("{\n\t.reg .u32 a0, a1, b0, b1;\n\tmov.b64 {a0, a1}, %1;\n\tmov.b64 {b0, b1}, %2;\n\t"
        "sub.cc.u32 a0, a0, b0;\n\tsubc.u32 a1, a1, b1;\n\tmov.b64 %0, {a0, a1};\n\t}"
        : "=l"(r) : "l"(a), "l"(b));
    return r;
}

template <int ILP, int PTX>
__global__ void bfly_loop(u64 *out, u64 q, u64 w0, u64 ws0, int iters)
{
    u64 x[2 * ILP];
    for (int i = 0; i < 2 * ILP; i++) x[i] = (threadIdx.x * 7919ull + i * 104729ull) % q;
    const u64 q2 = 2 * q;
    u64 w = w0 + threadIdx.x, ws = ws0 + threadIdx.x;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < ILP; i++) {
            u64 &a = x[2 * i], &b = x[2 * i + 1];
            if (PTX == 2) {
                const u64 X = a >= q2 ? a - q2 : a;
                u64 V = shoup_approx(b, w, ws, 0 - q);
                V = V >= q2 ? V - q2 : V;
                a = X + V;
                b = X + q2 - V;
            } else if (PTX) {
                const u64 X = a >= q2 ? sub64(a, q2) : a;
                const u64 V = shoup_lazy(b, w, ws, q);
                a = add64(X, V);
                b = sub64(add64(X, q2), V);
            } else {
                const u64 X = a >= q2 ? a - q2 : a;
                const u64 V = shoup_lazy(b, w, ws, q);
                a = X + V;
                b = X + q2 - V;
            }
        }
        w += 2;
    }
    u64 s = 0;
    for (int i = 0; i < 2 * ILP; i++) s ^= x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void check(u64 *bad, u64 q, u64 seed)
{
    u64 x = seed + threadIdx.x + blockIdx.x * 977ull;
    for (int i = 0; i < 256; i++) {
        x = x * 6364136223846793005ull + 1442695040888963407ull;
        u64 a = x % (4 * q), w = (x >> 7) % q;
        u64 ws = (u64)(((unsigned __int128)w << 64) / q);
        u64 r1 = shoup_lazy(a, w, ws, q), r2 = shoup_lazy_ptx(a, w, ws, 0 - q);
        if (r1 != r2) atomicAdd(bad, 1ull);
        u64 r3 = shoup_approx(a, w, ws, 0 - q);
        if (r3 >= 3 * q || r3 % q != r1 % q) atomicAdd(bad + 1, 1ull);
    }
}


// FP64 butterfly for q < 2^43 (values held as doubles, exact integers < 2^53):
// hi + lo = b w exactly (FMA), quotient estimate by the magic-number rounding
// of hi/q (off by at most one), t = hi - qe q exact (FMA), r = t + lo in
// (-q, 2q), one correction to [0, 2q).  Everything runs on the FP64 pipe
// except the selects.
__device__ __forceinline__ double fmodmul(double b, double w, double qd, double qinv)
{
    const double M = 6755399441055744.0;  // 1.5 * 2^52
    const double hi = b * w;
    const double lo = fma(b, w, -hi);
    const double qe = fma(hi, qinv, M) - M;
    const double t = fma(-qe, qd, hi);
    const double r = t + lo;
    return r < 0.0 ? r + qd : r;
}

// signed variant (the kernels' butterfly): V = b w mod q in (-q, q), a +- V,
// no range corrections inside a pass
__device__ __forceinline__ double fmodmul_s(double b, double w, double qd, double qinv)
{
    const double M = 6755399441055744.0;
    const double hi = b * w;
    const double lo = fma(b, w, -hi);
    const double qe = fma(hi, qinv, M) - M;
    return fma(-qe, qd, hi) + lo;
}
__device__ __forceinline__ double fred(double x, double qd, double qinv)
{
    const double M = 6755399441055744.0;
    const double qe = fma(x, qinv, M) - M;
    return fma(-qe, qd, x);
}

template <int ILP, int MODE>  // MODE 0: FP64 only; 1: half the pairs integer, half FP64; 2: signed FP64
__global__ void bfly_fp(u64 *out, u64 q, u64 w0, u64 ws0, int iters)
{
    double x[2 * ILP];
    u64 y[2 * ILP];
    const double qd = (double)q, qinv = 1.0 / qd, q2d = 2.0 * qd;
    for (int i = 0; i < 2 * ILP; i++) {
        y[i] = (threadIdx.x * 7919ull + i * 104729ull) % q;
        x[i] = (double)y[i];
    }
    const u64 q2 = 2 * q;
    u64 w = w0 + threadIdx.x, ws = ws0 + threadIdx.x;
    double wd = (double)(w % q);
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < ILP; i++) {
            if (MODE == 1 && (i & 1)) {
                u64 &a = y[2 * i], &b = y[2 * i + 1];
                const u64 X = a >= q2 ? a - q2 : a;
                u64 V = shoup_approx(b, w, ws, 0 - q);
                V = V >= q2 ? V - q2 : V;
                a = X + V;
                b = X + q2 - V;
            } else if (MODE == 2) {
                // 8 stages of signed butterflies, then a re-centring (the
                // kernels' per-pass pattern)
                double &a = x[2 * i], &b = x[2 * i + 1];
                const double V = fmodmul_s(b, wd, qd, qinv);
                b = a - V;
                a = a + V;
                if ((it & 7) == 7) {
                    a = fred(a, qd, qinv);
                    b = fred(b, qd, qinv);
                }
            } else {
                double &a = x[2 * i], &b = x[2 * i + 1];
                const double X = a >= q2d ? a - q2d : a;
                const double V = fmodmul(b, wd, qd, qinv);
                a = X + V;
                b = (X + q2d) - V;
            }
        }
        w += 2;
        wd += 2.0;
    }
    u64 s = 0;
    for (int i = 0; i < 2 * ILP; i++) s ^= (u64)x[i] ^ y[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void check_fp(u64 *bad, u64 q, u64 seed)
{
    const double qd = (double)q, qinv = 1.0 / qd;
    u64 x = seed + threadIdx.x + blockIdx.x * 977ull;
    for (int i = 0; i < 256; i++) {
        x = x * 6364136223846793005ull + 1442695040888963407ull;
        u64 a = x % (4 * q), w = (x >> 7) % q;
        const double r = fmodmul((double)a, (double)w, qd, qinv);
        const u64 want = (u64)(((unsigned __int128)a * w) % q);
        if (!(r >= 0.0 && r < 2.0 * qd) || ((u64)r) % q != want) atomicAdd(bad, 1ull);
    }
}

template <int ILP, int MODE>
void run_fp(const char *name, u64 *out, u64 q, u64 w, u64 ws, int threads, int bpsm)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096, blocks = 148 * bpsm;
    bfly_fp<ILP, MODE><<<blocks, threads>>>(out, q, w, ws, 16);
    cudaEventRecord(e0);
    bfly_fp<ILP, MODE><<<blocks, threads>>>(out, q, w, ws, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double bf = (double)blocks * threads * iters * ILP;
    printf("%-10s ILP%d %4d thr x %d/SM: %.3f T bfly/s\n", name, ILP, threads, bpsm, bf / ms / 1e9);
}

template <int ILP, int PTX>
void run(const char *name, u64 *out, u64 q, u64 w, u64 ws, int threads, int bpsm)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096, blocks = 148 * bpsm;
    bfly_loop<ILP, PTX><<<blocks, threads>>>(out, q, w, ws, 16);
    cudaEventRecord(e0);
    bfly_loop<ILP, PTX><<<blocks, threads>>>(out, q, w, ws, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double bf = (double)blocks * threads * iters * ILP;
    printf("%-10s ILP%d %4d thr x %d/SM: %.3f T bfly/s\n", name, ILP, threads, bpsm, bf / ms / 1e9);
}

int main()
{
    const u64 q = 0x1fffffffffe00001ull;
    const u64 w = 123456789123ull % q;
    const u64 ws = (u64)(((unsigned __int128)w << 64) / q);
    u64 *out, *bad;
    cudaMalloc(&out, 148 * 64 * 1024 * 8);
    cudaMalloc(&bad, 16);
    cudaMemset(bad, 0, 16);
    for (u64 qq : {q, 0xfffffffffc0001ull, 0x3ffffffffe0001ull}) check<<<1024, 256>>>(bad, qq, 12345);
    u64 nb[2] = {0, 0};
    cudaMemcpy(nb, bad, 16, cudaMemcpyDeviceToHost);
    printf("ptx shoup mismatches: %llu, approx out of range / wrong: %llu\n", nb[0], nb[1]);
    run<4, 0>("compiler", out, q, w, ws, 256, 4);
    run<4, 1>("ptx-adds", out, q, w, ws, 256, 4);
    run<4, 2>("approx", out, q, w, ws, 256, 4);
    run<8, 0>("compiler", out, q, w, ws, 256, 4);
    run<8, 2>("approx", out, q, w, ws, 256, 4);
    run<4, 0>("compiler", out, q, w, ws, 512, 2);
    run<4, 2>("approx", out, q, w, ws, 512, 2);
    // FP64 butterflies for a 42-bit prime (the P16 user levels)
    const u64 q42 = 0x3fffffa0001ull;  // 2^42 - 0x5ffff: any odd modulus < 2^43 for timing
    const u64 w42 = 123456789ull % q42, ws42 = (u64)(((unsigned __int128)w42 << 64) / q42);
    cudaMemset(bad, 0, 16);
    for (u64 qq : {q42, 0x7fffffe0001ull, 0x1fffffc0001ull}) check_fp<<<1024, 256>>>(bad, qq, 999);
    cudaMemcpy(nb, bad, 16, cudaMemcpyDeviceToHost);
    printf("fp64 modmul wrong: %llu\n", nb[0]);
    run<4, 2>("approx42", out, q42, w42, ws42, 256, 4);
    run_fp<4, 0>("fp64", out, q42, w42, ws42, 256, 4);
    run_fp<8, 0>("fp64", out, q42, w42, ws42, 256, 4);
    run_fp<4, 2>("fp64-signed", out, q42, w42, ws42, 256, 4);
    run_fp<8, 2>("fp64-signed", out, q42, w42, ws42, 256, 4);
    run_fp<4, 1>("hybrid", out, q42, w42, ws42, 256, 4);
    run_fp<8, 1>("hybrid", out, q42, w42, ws42, 256, 4);
    return 0;
}
