// Engine microbenchmarks on sm_100a (SURVEY §8(d) "engine ceilings"):
// per-SM throughput of IMMA.16832 (mma.sync m16n8k32 u8), emulated
// mma.sync m16n8k256 b1 and.popc, POPC, LOP3.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb scripts/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096

__global__ void k_imma(int* out, int seed) {
    uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    int c[4][4] = {};
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
            asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+r"(c[q][0]), "+r"(c[q][1]), "+r"(c[q][2]), "+r"(c[q][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    int s = 0;
    for (int q = 0; q < 4; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
    if (s == 0x12345) out[0] = s;
}

__global__ void k_bmma(int* out, int seed) {
    uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    int c[4][4] = {};
    for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
            asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+r"(c[q][0]), "+r"(c[q][1]), "+r"(c[q][2]), "+r"(c[q][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    int s = 0;
    for (int q = 0; q < 4; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
    if (s == 0x12345) out[0] = s;
}

__global__ void k_popc(int* out, int seed) {
    uint32_t x[8];
    for (int i = 0; i < 8; ++i) x[i] = (seed + threadIdx.x) * (2 * i + 1);
    uint32_t acc[8] = {};
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) { acc[i] += __popc(x[i] ^ it); }
    }
    uint32_t s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 0x12345) out[0] = s;
}

__global__ void k_lop3(int* out, int seed) {
    uint32_t x[8];
    for (int i = 0; i < 8; ++i) x[i] = (seed + threadIdx.x) * (2 * i + 1);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[i]) : "r"(x[(i + 1) & 7]), "r"(it));
        }
    }
    uint32_t s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 0x12345) out[0] = s;
}

template <typename K>
float run(K kern, int blocks, int threads, int* d) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    kern<<<blocks, threads>>>(d, 1);
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(d, 2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

int main() {
    int* d; cudaMalloc(&d, 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double ghz = clk / 1e6;
    for (int threads : {128, 256, 512, 1024}) {
        int blocks = sms * 2;
        double warps = (double)blocks * threads / 32;
        float ms = run(k_imma, blocks, threads, d);
        double n = warps * ITERS * 4;    // mma.sync per warp
        printf("IMMA.16832 u8  threads=%4d: %.3f ms  %.3f mma/clk/SM (at %.2f GHz)  %.1f TOPS\n", threads, ms,
               n / (ms * 1e-3) / sms / (ghz * 1e9), ghz, n * 16 * 8 * 32 * 2 / (ms * 1e-3) / 1e12);
        ms = run(k_bmma, blocks, threads, d);
        n = warps * (ITERS / 8) * 4;
        printf("b1 m16n8k256 (emul) thr=%4d: %.3f ms  %.3f mma/clk/SM\n", threads, ms,
               n / (ms * 1e-3) / sms / (ghz * 1e9));
        ms = run(k_popc, blocks, threads, d);
        n = (double)blocks * threads * ITERS * 8;
        printf("POPC           threads=%4d: %.3f ms  %.1f popc/clk/SM\n", threads, ms, n / (ms * 1e-3) / sms / (ghz * 1e9));
        ms = run(k_lop3, blocks, threads, d);
        printf("LOP3           threads=%4d: %.3f ms  %.1f lop3/clk/SM\n", threads, ms, n / (ms * 1e-3) / sms / (ghz * 1e9));
    }
    return 0;
}
