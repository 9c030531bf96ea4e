// mxf4_data_mb.cu -- does the tcgen05.mma kind::mxf4.block_scale (M=128, K=64, TS) issue rate
// depend on the operand DATA, or on the B tile / scale / A column pattern of bitgemm_tc_kernel?
// A in TMEM (128 columns = 16 MMAs), B in SMEM (16 tiles of N x 32 B, K-major, no swizzle).
// DATA: 0 = zeros, 1 = random 0/1-layer nibbles (0b00hl) in A and random e2m1 digits in B,
//       2 = all-ones nibbles (0b0011) in A and max digits in B.
// BVAR: 0 = one B tile for all MMAs, 1 = B tile advances per MMA (as in the kernel).
// One CTA per SM, cycles per MMA on the issuing thread of CTA 0.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mxd mxf4_data_mb.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
           ((uint64_t)1 << 46);
}
__device__ __forceinline__ uint32_t hsh(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <int N, int DATA, int BVAR>
__global__ void __launch_bounds__(160, 1) rate(long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tb;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr uint32_t kBT = N * 32;                 // one MMA's B tile
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < 16 * (int)kBT; i += blockDim.x) {
        uint8_t v = 0;
        if (DATA == 1) {
            // e2m1 digit codes 2d for d in {-2..3}: 0, 2(1.0), 4(2.0), 5(3.0), 6(4.0), 7(6.0), 9(-0.5)...
            const uint32_t r = hsh(i * 2654435761u + 7);
            const uint8_t lut[8] = {0x0, 0x2, 0x4, 0x5, 0x6, 0x7, 0xC, 0xA};
            v = (uint8_t)(lut[r & 7] | (lut[(r >> 3) & 7] << 4));
        } else if (DATA == 2) {
            v = 0x77;
        }
        sm[i] = v;
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t t = tb;
    if (w >= 1) {
        // A columns [0, 128): 4 x32 stores per lane quarter; SF at 480/488 = 1.0 (0x7F)
        const uint32_t lq = (uint32_t)((w & 3) * 32) << 16;
        uint32_t v[32];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const uint32_t r = hsh((uint32_t)(threadIdx.x * 977 + c * 131 + i * 7919));
                v[i] = DATA == 1 ? (r & 0x33333333u) : (DATA == 2 ? 0x33333333u : 0u);
            }
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(t + lq + (uint32_t)(c * 32)),
                "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
                "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
                "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
                : "memory");
        }
        const uint32_t s7 = 0x7F7F7F7Fu;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                         t + lq + 480),
                     "r"(s7));
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 0) {
        const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | (8u << 24);
        const uint64_t bd = desc(su(sm));
        const uint32_t dcol = t + 256;
        long long t0 = clock64();
        for (int i = 0; i < iters; i += 16) {
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const uint32_t acc = (i + u) > 0;
                const uint64_t b = BVAR ? bd + (uint64_t)(u * (kBT / 16)) : bd;
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %3, [%5], [%6], p;\n}\n" ::"r"(
                                 dcol),
                             "r"(t + (uint32_t)(u * 8)), "l"(b), "r"(idesc), "r"(acc), "r"(t + 480), "r"(t + 488));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)));
        asm volatile("{\n.reg .pred p;\nW_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(
                         su(&bar))
                     : "memory");
        long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
    (void)lane;
}

template <class K>
void run(const char* name, K k, int iters) {
    long long* d;
    cudaMalloc(&d, 16);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = 16 * 64 * 32 + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<sms, 160, smem>>>(d, iters);
    k<<<sms, 160, smem>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-34s %s cycles/mma = %6.1f\n", name, e == cudaSuccess ? "" : cudaGetErrorString(e), (double)h / iters);
    cudaFree(d);
}

int main() {
    const int it = 8192;
    run("N8  zeros   same B", rate<8, 0, 0>, it);
    run("N8  zeros   B/mma", rate<8, 0, 1>, it);
    run("N8  random  same B", rate<8, 1, 0>, it);
    run("N8  random  B/mma", rate<8, 1, 1>, it);
    run("N8  max     B/mma", rate<8, 2, 1>, it);
    run("N16 zeros   B/mma", rate<16, 0, 1>, it);
    run("N16 random  B/mma", rate<16, 1, 1>, it);
    run("N16 max     B/mma", rate<16, 2, 1>, it);
    run("N64 random  B/mma", rate<64, 1, 1>, it);
    return 0;
}
