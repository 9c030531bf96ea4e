// tc_probe_2cta.cu -- semantics of tcgen05.mma.cta_group::2.kind::mxf4 (M = 256, N = 16)
// with A in TMEM: which rows of A each CTA's TMEM supplies and where B (the N x K
// operand) is read from.  CTA r of the pair holds A rows [128r, 128r+128) in its
// TMEM and its own B tile Br in SMEM (different data per CTA).  D is read back from
// both CTAs and compared against candidate interpretations.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
probe(const uint8_t* A, const uint8_t* Bm, float* D) {
    __shared__ __align__(1024) uint8_t sB[16 * 32];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tb;
    const int t = threadIdx.x, warp = t >> 5;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    const uint8_t* Br = Bm + rank * 16 * 32;
    for (int e = t; e < 16 * 32; e += 128) {
        const int n = e / 32, k = e % 32;
        sB[(n / 8) * 256 + (k / 16) * 128 + (n % 8) * 16 + (k % 16)] = Br[n * 32 + k];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = tb;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    uint32_t a[8];
    const uint8_t* Ar = A + (rank * 128 + t) * 32;
    for (int c = 0; c < 8; ++c) a[c] = Ar[4 * c] | (Ar[4 * c + 1] << 8) | (Ar[4 * c + 2] << 16) | ((uint32_t)Ar[4 * c + 3] << 24);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(base + lane_base),
                 "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
    const uint32_t s7 = 0x7F7F7F7Fu;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                     base + lane_base + 64),
                 "r"(s7));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (rank == 0 && t == 0) {
        const uint32_t saddr = smem_u32(sB);
        uint64_t desc = (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
                        ((uint64_t)1 << 46);
        const uint32_t idesc = (1u << 7) | (1u << 10) | ((16u >> 3) << 17) | (1u << 23) | ((256u >> 4) << 24);
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, 0, 0;\n"
            "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %3, [%4], [%5], p;\n}\n" ::"r"(
                base + 32),
            "r"(base), "l"(desc), "r"(idesc), "r"(base + 64), "r"(base + 72));
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&bar)),
            "h"((uint16_t)3));
    }
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
        smem_u32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t d[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
          "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
        : "r"(base + lane_base + 32));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int n = 0; n < 16; ++n) D[(rank * 128 + t) * 16 + n] = __uint_as_float(d[n]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 128;" ::"r"(base));
}

static float e2m1(int c) {
    static const float mag[8] = {0.f, 0.5f, 1.f, 1.5f, 2.f, 3.f, 4.f, 6.f};
    return (c & 8) ? -mag[c & 7] : mag[c & 7];
}
static double dot(const uint8_t* a, const uint8_t* b) {
    double s = 0;
    for (int k = 0; k < 32; ++k) s += e2m1(a[k] & 15) * e2m1(b[k] & 15) + e2m1(a[k] >> 4) * e2m1(b[k] >> 4);
    return s;
}

int main() {
    static uint8_t hA[256 * 32], hB[2 * 16 * 32];
    srand(5);
    for (auto& v : hA) v = rand() & 0x77;   // positive codes only
    for (auto& v : hB) v = rand() & 0x77;
    uint8_t *dA, *dB;
    float* dD;
    cudaMalloc(&dA, sizeof hA);
    cudaMalloc(&dB, sizeof hB);
    cudaMalloc(&dD, 256 * 16 * 4);
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
    probe<<<2, 128>>>(dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("CUDA error: %s\n", cudaGetErrorString(e));
        return 1;
    }
    static float hD[256 * 16];
    cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
    // candidates for B row n: H1 = B0[n] (leader only); H2 = n<8 ? B0[n] : B1[n-8]; H3 = n<8 ? B0[n] : B1[n]
    int bad[3] = {0, 0, 0};
    for (int m = 0; m < 256; ++m)
        for (int n = 0; n < 16; ++n) {
            const uint8_t* b1 = hB + n * 32;
            const uint8_t* b2 = n < 8 ? hB + n * 32 : hB + 16 * 32 + (n - 8) * 32;
            const uint8_t* b3 = n < 8 ? hB + n * 32 : hB + 16 * 32 + n * 32;
            const double got = hD[m * 16 + n];
            bad[0] += got != dot(hA + m * 32, b1);
            bad[1] += got != dot(hA + m * 32, b2);
            bad[2] += got != dot(hA + m * 32, b3);
        }
    printf("2-CTA mxf4 probe mismatches: H1 (B from leader only) %d, H2 (N split, first halves) %d, H3 (N split, same rows) %d\n",
           bad[0], bad[1], bad[2]);
    printf("D[0][0..3] = %g %g %g %g ; D[200][8] = %g\n", hD[0], hD[1], hD[2], hD[3], hD[200 * 16 + 8]);
    return 0;
}
