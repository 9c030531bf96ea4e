// tc_mb.cu -- microbenchmarks of the tcgen05 pieces the MMA engine uses (sm_100a):
//   (1) back-to-back tcgen05.mma.kind::i8 M=128, A from TMEM, N in {8..256}
//   (2) same with A from SMEM (SS)
//   (3) tcgen05.st.32x32b.x32 throughput, with and without wait::st per store
//   (4) round trip: st -> wait::st -> fence -> mbarrier arrive -> MMA -> commit -> mbarrier
// One CTA per SM on all SMs; cycles from clock64 on thread 0; 4 warps.
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
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
           ((uint64_t)1 << 46);
}

template <int N, bool A_TMEM>
__global__ void __launch_bounds__(128, 1) mma_rate(long long* out, int iters) {
    __shared__ __align__(1024) uint8_t sB[256 * 32];
    __shared__ __align__(1024) uint8_t sA[128 * 32];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tb;
    const int w = threadIdx.x >> 5;
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < 256 * 32; i += 128) sB[i] = (uint8_t)i;
    for (int i = threadIdx.x; i < 128 * 32; i += 128) sA[i] = (uint8_t)(i * 7);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t t = tb;
    if (threadIdx.x == 0) {
        const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
        const uint64_t bd = desc(smem_u32(sB));
        const uint64_t ad = desc(smem_u32(sA));
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t acc = i > 0;
            if (A_TMEM)
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(
                                 t + 256),
                             "r"(t + (uint32_t)((i & 7) * 8)), "l"(bd), "r"(idesc), "r"(acc));
            else
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                                 t + 256),
                             "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

template <int N>
__global__ void __launch_bounds__(128, 1) mma_rate_f4(long long* out, int iters) {
    __shared__ __align__(1024) uint8_t sB[256 * 32];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tb;
    const int w = threadIdx.x >> 5;
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < 256 * 32; i += 128) sB[i] = (uint8_t)0x22;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t t = tb;
    const uint32_t s7 = 0x7F7F7F7Fu;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                     t + ((uint32_t)(w * 32) << 16) + 480),
                 "r"(s7));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 0) {
        const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | (8u << 24);
        const uint64_t bd = desc(smem_u32(sB));
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t acc = i > 0;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %3, [%5], [%6], p;\n}\n" ::"r"(
                             t + 256),
                         "r"(t + (uint32_t)((i & 7) * 8)), "l"(bd), "r"(idesc), "r"(acc), "r"(t + 480), "r"(t + 488));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

template <bool WAIT>
__global__ void __launch_bounds__(128, 1) st_rate(long long* out, int iters) {
    __shared__ uint32_t tb;
    const int w = threadIdx.x >> 5;
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t t = tb + ((uint32_t)(w * 32) << 16);
    uint32_t v[32];
    for (int i = 0; i < 32; ++i) v[i] = threadIdx.x * 33 + i;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
            "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(t + (uint32_t)((i & 7) * 32)),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
            "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
            "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
            "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
            : "memory");
        if (WAIT) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        v[i & 31] += 1;
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

// MMA (TS or SS, N=16) back-to-back while warps 1..4 store to TMEM continuously.
template <bool A_TMEM, bool STORES>
__global__ void __launch_bounds__(160, 1) mma_vs_st(long long* out, int iters) {
    __shared__ __align__(1024) uint8_t sB[256 * 32];
    __shared__ __align__(1024) uint8_t sA[128 * 32];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tb;
    __shared__ volatile int stop;
    __shared__ long long nst;
    const int w = threadIdx.x >> 5;
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) sB[i] = (uint8_t)i;
    for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) sA[i] = (uint8_t)(i * 7);
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
    if (w == 0) {
        if (threadIdx.x == 0) {
            const uint32_t idesc = (2u << 4) | ((uint32_t)(16 >> 3) << 17) | (8u << 24);
            const uint64_t bd = desc(smem_u32(sB));
            const uint64_t ad = desc(smem_u32(sA));
            long long t0 = clock64();
            for (int i = 0; i < iters; ++i) {
                const uint32_t acc = i > 0;
                if (A_TMEM)
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(
                                     t + 448),
                                 "r"(t + (uint32_t)((i & 7) * 8)), "l"(bd), "r"(idesc), "r"(acc));
                else
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                                     t + 448),
                                 "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
            mbar_wait(&bar, 0);
            long long t1 = clock64();
            stop = 1;
            if (blockIdx.x == 0) out[0] = t1 - t0;
        }
    } else if (STORES) {
        const uint32_t ta = t + ((uint32_t)((w & 3) * 32) << 16) + 128;
        uint32_t v[32];
        for (int i = 0; i < 32; ++i) v[i] = threadIdx.x * 33 + i;
        long long n = 0;
        while (!stop) {
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta + (uint32_t)((n & 7) * 32)),
                "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
                "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
                "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
                : "memory");
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            ++n;
        }
        if ((threadIdx.x & 31) == 0) atomicAdd((unsigned long long*)&nst, (unsigned long long)n);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[1] = nst;
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

// ping-pong between warp 1 (producer role) and warp 0 (MMA role) through two mbarriers;
// KIND 0: plain arrive both ways; 1: return via tcgen05.commit (no MMA); 2: 4 MMAs + commit.
template <int KIND>
__global__ void __launch_bounds__(64, 1) pingpong(long long* out, int iters) {
    __shared__ __align__(1024) uint8_t sB[16 * 32];
    __shared__ __align__(8) uint64_t full, empty;
    __shared__ uint32_t tb;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < 16 * 32; i += 64) sB[i] = 0;
    if (threadIdx.x == 0) {
        mbar_init(&full, 1);
        mbar_init(&empty, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t t = tb;
    long long t0 = clock64();
    if (w == 1) {
        for (int i = 0; i < iters; ++i) {
            if (i > 0) mbar_wait(&empty, (i - 1) & 1);
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full)) : "memory");
        }
        mbar_wait(&empty, (iters - 1) & 1);
    } else {
        const uint32_t idesc = (2u << 4) | ((uint32_t)(16 >> 3) << 17) | (8u << 24);
        const uint64_t bd = desc(smem_u32(sB));
        for (int i = 0; i < iters; ++i) {
            mbar_wait(&full, i & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (lane == 0) {
                if (KIND == 0) {
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty)) : "memory");
                } else {
                    if (KIND == 2)
                        for (int q = 0; q < 4; ++q)
                            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(
                                             t + 256),
                                         "r"(t + (uint32_t)(q * 8)), "l"(bd), "r"(idesc), "r"(1));
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                        smem_u32(&empty)));
                }
            }
            __syncwarp();
        }
    }
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 32) out[0] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

// cta_group::2 (M = 256 across a CTA pair) mxf4 TS rate, N = 16
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma2_rate(long long* out, int iters) {
    __shared__ __align__(1024) uint8_t sB[256 * 32];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tb;
    const int w = threadIdx.x >> 5;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    for (int i = threadIdx.x; i < 256 * 32; i += 128) sB[i] = (uint8_t)0x22;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t t = tb;
    const uint32_t s7 = 0x7F7F7F7Fu;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                     t + ((uint32_t)(w * 32) << 16) + 480),
                 "r"(s7));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (rank == 0 && threadIdx.x == 0) {
        const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(16 >> 3) << 17) | (1u << 23) | (16u << 24);
        const uint64_t bd = desc(smem_u32(sB));
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t acc = i > 0;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %3, [%5], [%6], p;\n}\n" ::"r"(
                             t + 256),
                         "r"(t + (uint32_t)((i & 7) * 8)), "l"(bd), "r"(idesc), "r"(acc), "r"(t + 480), "r"(t + 488));
        }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                         smem_u32(&bar)),
                     "h"((uint16_t)3));
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    if (rank == 1 && threadIdx.x == 0) mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::before_thread_sync;");
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(t));
}

template <class K>
void run64(const char* name, K k, int iters) {
    long long* d;
    cudaMalloc(&d, 8);
    k<<<148, 64>>>(d, iters);
    k<<<148, 64>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-36s %s cycles/roundtrip = %.1f\n", name, e == cudaSuccess ? "" : cudaGetErrorString(e), (double)h / iters);
    cudaFree(d);
}

void run2(const char* name, void (*k)(long long*, int), int iters) {
    long long* d;
    cudaMalloc(&d, 16);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    k<<<sms, 160>>>(d, iters);
    k<<<sms, 160>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[2] = {0, 0};
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-36s %s cycles/mma = %.1f   warp-stores during run = %lld (%.1f cycles per store per SM)\n", name,
           e == cudaSuccess ? "" : cudaGetErrorString(e), (double)h[0] / iters, h[1],
           h[1] ? (double)h[0] / h[1] : 0.0);
    cudaFree(d);
}

template <class K>
void run(const char* name, K k, int iters, double per) {
    long long* d;
    cudaMalloc(&d, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    k<<<sms, 128>>>(d, iters);
    k<<<sms, 128>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-36s %s cycles/op = %.1f\n", name, e == cudaSuccess ? "" : cudaGetErrorString(e), (double)h / iters / per);
    cudaFree(d);
}

int main() {
    const int it = 4096;
    {
        long long* d;
        cudaMalloc(&d, 8);
        mma2_rate<<<148, 128>>>(d, it);
        mma2_rate<<<148, 128>>>(d, it);
        cudaError_t e = cudaDeviceSynchronize();
        long long h = 0;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("%-36s %s cycles/op = %.1f (M=256 over 2 SMs)\n", "mma mxf4 TS cta_group::2 N16",
               e == cudaSuccess ? "" : cudaGetErrorString(e), (double)h / it);
    }
    run64("pingpong plain arrive", pingpong<0>, it);
    run64("pingpong commit (no mma)", pingpong<1>, it);
    run64("pingpong 4 mma + commit", pingpong<2>, it);
    run("mma mxf4 TS M128 N8", mma_rate_f4<8>, it, 1);
    run("mma mxf4 TS M128 N16", mma_rate_f4<16>, it, 1);
    run("mma mxf4 TS M128 N32", mma_rate_f4<32>, it, 1);
    run("mma mxf4 TS M128 N256", mma_rate_f4<256>, it, 1);
    run("mma i8 TS M128 N8", mma_rate<8, true>, it, 1);
    run("mma i8 TS M128 N16", mma_rate<16, true>, it, 1);
    run("mma i8 TS M128 N32", mma_rate<32, true>, it, 1);
    run("mma i8 TS M128 N64", mma_rate<64, true>, it, 1);
    run("mma i8 TS M128 N128", mma_rate<128, true>, it, 1);
    run("mma i8 TS M128 N256", mma_rate<256, true>, it, 1);
    run("mma i8 SS M128 N16", mma_rate<16, false>, it, 1);
    run("mma i8 SS M128 N64", mma_rate<64, false>, it, 1);
    run("mma i8 SS M128 N256", mma_rate<256, false>, it, 1);
    run("tmem st x32 (no wait)  per warp-op", st_rate<false>, it, 1);
    run("tmem st x32 (wait each) per warp-op", st_rate<true>, it, 1);
    run2("mma TS N16 alone", mma_vs_st<true, false>, it);
    run2("mma TS N16 + 4 warps st", mma_vs_st<true, true>, it);
    run2("mma SS N16 + 4 warps st", mma_vs_st<false, true>, it);
    return 0;
}
