// tc_probe_f4.cu -- verifies tcgen05.mma.kind::mxf4.block_scale.scale_vec::2X with A in TMEM:
//   A (M=128 x K=64 e2m1, packed 2/byte) via tcgen05.st (lane = row, 8 columns),
//   B (N=16 x K=64 e2m1) in SMEM, K-major no-swizzle canonical layout (as the i8 probe),
//   scale factors (E8M0 = 0x7F = 1.0) filling TMEM columns for SFA / SFB,
//   D (f32) read back with tcgen05.ld.  Checks element order within a byte and the e2m1 code.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const uint8_t* A, const uint8_t* Bm, float* D) {
    __shared__ __align__(1024) uint8_t sB[16 * 32];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tb;
    const int t = threadIdx.x, warp = t >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    for (int e = t; e < 16 * 32; e += 128) {
        const int n = e / 32, k = e % 32;   // k = byte index (2 fp4 each)
        sB[(n / 8) * 256 + (k / 16) * 128 + (n % 8) * 16 + (k % 16)] = Bm[n * 32 + k];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = tb;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    uint32_t a[8];
    for (int c = 0; c < 8; ++c) {
        const uint8_t* p = A + t * 32 + 4 * c;
        a[c] = p[0] | (p[1] << 8) | (p[2] << 16) | ((uint32_t)p[3] << 24);
    }
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(base + lane_base),
                 "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
    // scale factors: columns 64..79 all 0x7F (E8M0 1.0)
    const uint32_t s7 = 0x7F7F7F7Fu;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                     base + lane_base + 64),
                 "r"(s7));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (t == 0) {
        const uint32_t saddr = smem_u32(sB);
        uint64_t desc = (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
                        ((uint64_t)1 << 46);
        const uint32_t idesc = (0u << 4) | (1u << 7) | (1u << 10) | ((16u >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, 0, 0;\n"
            "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %3, [%4], [%5], p;\n}\n" ::"r"(
                base + 32),
            "r"(base), "l"(desc), "r"(idesc), "r"(base + 64), "r"(base + 72));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
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
    for (int n = 0; n < 16; ++n) D[t * 16 + n] = __uint_as_float(d[n]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(base));
}

static float e2m1(int c) {
    static const float mag[8] = {0.f, 0.5f, 1.f, 1.5f, 2.f, 3.f, 4.f, 6.f};
    return (c & 8) ? -mag[c & 7] : mag[c & 7];
}

int main() {
    uint8_t hA[128 * 32], hB[16 * 32];
    srand(3);
    for (auto& v : hA) v = rand() & 0xFF;
    for (auto& v : hB) v = rand() & 0xFF;
    uint8_t *dA, *dB;
    float* dD;
    cudaMalloc(&dA, sizeof hA);
    cudaMalloc(&dB, sizeof hB);
    cudaMalloc(&dD, 128 * 16 * 4);
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
    probe<<<1, 128>>>(dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("CUDA error: %s\n", cudaGetErrorString(e));
        return 1;
    }
    float hD[128 * 16];
    cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
    int bad_lo = 0, bad_hi = 0;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 16; ++n) {
            double lo = 0, hi = 0;
            for (int k = 0; k < 32; ++k) {
                const uint8_t a = hA[m * 32 + k], b = hB[n * 32 + k];
                lo += e2m1(a & 15) * e2m1(b & 15) + e2m1(a >> 4) * e2m1(b >> 4);
                hi += e2m1(a & 15) * e2m1(b & 15) + e2m1(a >> 4) * e2m1(b >> 4);
            }
            if (lo != hD[m * 16 + n]) {
                if (bad_lo < 4) printf("m=%d n=%d got %f want %f\n", m, n, hD[m * 16 + n], lo);
                ++bad_lo;
            }
            (void)hi;
        }
    printf("mxf4 TS probe: %s (%d mismatches)\n", bad_lo ? "FAIL" : "OK", bad_lo);
    return bad_lo ? 2 : 0;
}
