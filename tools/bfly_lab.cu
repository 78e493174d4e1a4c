// bfly_lab.cu -- dev tool: the arithmetic ceiling of a 64-bit Shoup butterfly
// on this GPU (registers only, no memory), to compare with the NTT kernels'
// achieved butterflies/s.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;

__device__ __forceinline__ u64 shoup_lazy(u64 a, u64 w, u64 ws, u64 q) { return a * w - __umul64hi(a, ws) * q; }

template <int ILP>
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
            const u64 X = a >= q2 ? a - q2 : a;
            const u64 V = shoup_lazy(b, w, ws, q);
            a = X + V;
            b = X + q2 - V;
        }
        w += 2;
    }
    u64 s = 0;
    for (int i = 0; i < 2 * ILP; i++) s ^= x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main()
{
    const u64 q = 0x1fffffffffe00001ull;  // 61-bit NTT-friendly prime shape
    const u64 w = 123456789123ull % q;
    const u64 ws = (u64)(((unsigned __int128)w << 64) / q);
    u64 *out;
    cudaMalloc(&out, 148 * 64 * 1024 * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int threads : {256, 512, 1024}) {
        for (int blocks_per_sm : {1, 2, 4, 8}) {
            if (threads * blocks_per_sm > 2048) continue;
            const int blocks = 148 * blocks_per_sm;
            bfly_loop<4><<<blocks, threads>>>(out, q, w, ws, 16);
            cudaEventRecord(e0);
            bfly_loop<4><<<blocks, threads>>>(out, q, w, ws, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double bf = (double)blocks * threads * iters * 4;
            printf("ILP4 threads %4d x %d/SM: %.3f T bfly/s  (=> %.3f us per 2^16 NTT limb)\n", threads,
                   blocks_per_sm, bf / ms / 1e9, 524288.0 / (bf / ms / 1e9) * 1e-3 * 1e3 / 1e3);
        }
    }
    for (int threads : {512, 1024}) {
        const int blocks = 148 * (2048 / threads);
        bfly_loop<2><<<blocks, threads>>>(out, q, w, ws, iters);
        cudaEventRecord(e0);
        bfly_loop<2><<<blocks, threads>>>(out, q, w, ws, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double bf = (double)blocks * threads * iters * 2;
        printf("ILP2 threads %4d full occ: %.3f T bfly/s\n", threads, bf / ms / 1e9);
    }
    return 0;
}
