// mxf4_mb.cu -- microbenchmark: tcgen05.mma kind::mxf4.block_scale (M=128, K=64) rate on
// sm_100a with the A operand from TMEM (TS) or from SMEM (SS), alone and while 4 other
// warps keep the A-producing path busy (tcgen05.st into TMEM, or st.shared into SMEM),
// plus an alternating TS/SS issue.  One CTA per SM on all SMs; cycles per MMA from
// clock64 on the issuing thread (CTA 0).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                     smem_u32(b)),
                 "r"(ph)
                 : "memory");
}
// K-major, no swizzle: core matrix 8 rows x 16 B, LBO 128 B (K-adjacent), SBO 256 B (next 8 rows)
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
           ((uint64_t)1 << 46);
}

// MODE: 0 = TS (A in TMEM), 1 = SS (A in SMEM), 2 = alternate TS / SS
// LOAD: 0 = none, 1 = 4 warps tcgen05.st.32x32b.x32 (TMEM), 2 = 4 warps st.shared.v4 (SMEM)
template <int MODE, int N, int LOAD>
__global__ void __launch_bounds__(160, 1) rate(long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* sA = sm;                    // 8 A tiles of 128 x 32 B (SS)
    uint8_t* sB = sm + 8 * 4096;         // B: 256 x 32 B
    uint8_t* sX = sB + 8192;             // st.shared target: 16 KiB
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tb;
    __shared__ volatile int stop;
    __shared__ unsigned long long nst;
    const int w = threadIdx.x >> 5;
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < 8 * 4096 + 8192; i += blockDim.x) sm[i] = (uint8_t)0x22;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        stop = 0;
        nst = 0;
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t t = tb;
    // scale factors at column 480 (SFA) and 488 (SFB): 1.0
    if (w >= 1) {
        const uint32_t s7 = 0x7F7F7F7Fu;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                         t + ((uint32_t)((w & 3) * 32) << 16) + 480),
                     "r"(s7));
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // TMEM map: A ring [0,128), D [256, 256 + N) (N <= 224 here; N = 256 uses [224, 480))
    const uint32_t dcol = N <= 224 ? 256 : 224;
    if (w == 0) {
        if (threadIdx.x == 0) {
            const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | (8u << 24);
            const uint64_t bd = desc(smem_u32(sB));
            long long t0 = clock64();
            for (int i = 0; i < iters; ++i) {
                const uint32_t acc = i > 0;
                const bool ts = MODE == 0 || (MODE == 2 && (i & 1));
                if (ts)
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %3, [%5], [%6], p;\n}\n" ::"r"(
                                     t + dcol),
                                 "r"(t + (uint32_t)((i & 7) * 8)), "l"(bd), "r"(idesc), "r"(acc), "r"(t + 480),
                                 "r"(t + 488));
                else
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(
                                     t + dcol),
                                 "l"(desc(smem_u32(sA + (i & 7) * 4096))), "l"(bd), "r"(idesc), "r"(acc),
                                 "r"(t + 480), "r"(t + 488));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&bar)));
            mbar_wait(&bar, 0);
            long long t1 = clock64();
            stop = 1;
            if (blockIdx.x == 0) out[0] = t1 - t0;
        }
    } else if (LOAD == 1) {
        const uint32_t ta = t + ((uint32_t)((w & 3) * 32) << 16) + 128;   // cols [128, 256)
        uint32_t v[32];
        for (int i = 0; i < 32; ++i) v[i] = threadIdx.x * 33 + i;
        long long n = 0;
        while (!stop) {
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta + (uint32_t)((n & 3) * 32)),
                "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
                "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
                "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
                : "memory");
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            ++n;
        }
        if ((threadIdx.x & 31) == 0) atomicAdd(&nst, (unsigned long long)n * 4096ull);   // bytes per warp-op
    } else if (LOAD == 2) {
        const uint32_t base = smem_u32(sX) + (uint32_t)(threadIdx.x - 32) * 16;
        long long n = 0;
        while (!stop) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(base + (uint32_t)(k * 2048)),
                             "r"((uint32_t)n), "r"((uint32_t)k), "r"(3u), "r"(4u)
                             : "memory");
            ++n;
        }
        if ((threadIdx.x & 31) == 0) atomicAdd(&nst, (unsigned long long)n * 8ull * 512ull);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[1] = (long long)nst;
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

template <class K>
void run(const char* name, K k, int iters) {
    long long* d;
    cudaMalloc(&d, 16);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = 8 * 4096 + 8192 + 16384;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<sms, 160, smem>>>(d, iters);
    k<<<sms, 160, smem>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[2] = {0, 0};
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-40s %s cycles/mma = %6.1f   side-load bytes/cycle = %6.1f\n", name,
           e == cudaSuccess ? "" : cudaGetErrorString(e), (double)h[0] / iters, h[0] ? (double)h[1] / h[0] : 0.0);
    cudaFree(d);
}

int main() {
    const int it = 4096;
    run("mxf4 TS N8", rate<0, 8, 0>, it);
    run("mxf4 TS N16", rate<0, 16, 0>, it);
    run("mxf4 TS N32", rate<0, 32, 0>, it);
    run("mxf4 TS N64", rate<0, 64, 0>, it);
    run("mxf4 TS N128", rate<0, 128, 0>, it);
    run("mxf4 TS N256", rate<0, 256, 0>, it);
    run("mxf4 SS N8", rate<1, 8, 0>, it);
    run("mxf4 SS N16", rate<1, 16, 0>, it);
    run("mxf4 SS N64", rate<1, 64, 0>, it);
    run("mxf4 SS N128", rate<1, 128, 0>, it);
    run("mxf4 SS N256", rate<1, 256, 0>, it);
    run("mxf4 TS/SS alternating N16", rate<2, 16, 0>, it);
    run("mxf4 TS N16 + 4 warps tcgen05.st", rate<0, 16, 1>, it);
    run("mxf4 SS N16 + 4 warps tcgen05.st", rate<1, 16, 1>, it);
    run("mxf4 TS N16 + 4 warps st.shared", rate<0, 16, 2>, it);
    run("mxf4 SS N16 + 4 warps st.shared", rate<1, 16, 2>, it);
    run("mxf4 alt N16 + 4 warps tcgen05.st", rate<2, 16, 1>, it);
    run("mxf4 alt N16 + 4 warps st.shared", rate<2, 16, 2>, it);
    run("mxf4 TS N256 + 4 warps tcgen05.st", rate<0, 256, 1>, it);
    run("mxf4 SS N256 + 4 warps st.shared", rate<1, 256, 2>, it);
    return 0;
}
