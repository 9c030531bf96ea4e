// tc_probe.cu -- verifies the tcgen05 layout assumptions the MMA engine relies on:
//   * A (M=128 x K=32 u8) written to TMEM with tcgen05.st.32x32b.x8 (lane = row,
//     column c holds bytes k = 4c..4c+3);
//   * B (N=16 x K=32 u8) in shared memory, K-major SWIZZLE_NONE canonical layout
//     ((8,n),2):((16B,SBO),LBO) with LBO = 128 B, SBO = 256 B;
//   * instruction descriptor kind::i8 (u8 x u8 -> s32), M=128, N=16;
//   * D read back with tcgen05.ld.32x32b.x16 (lane = row, column = n).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tcp scripts/tc_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void probe(const uint8_t* A, const uint8_t* Bm, int32_t* D, int accumulate_twice) {
    __shared__ __align__(1024) uint8_t sB[512];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int t = threadIdx.x, warp = t >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "n"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    // B canonical K-major no-swizzle: offset(n,k) = (n/8)*256 + (k/16)*128 + (n%8)*16 + k%16
    for (int e = t; e < 16 * 32; e += blockDim.x) {
        const int n = e / 32, k = e % 32;
        sB[(n / 8) * 256 + (k / 16) * 128 + (n % 8) * 16 + (k % 16)] = Bm[n * 32 + k];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = tmem_base;
    // A row t -> lane t; 8 columns of 4 bytes
    uint32_t a[8];
    for (int c = 0; c < 8; ++c) {
        const uint8_t* p = A + t * 32 + 4 * c;
        a[c] = p[0] | (p[1] << 8) | (p[2] << 16) | ((uint32_t)p[3] << 24);
    }
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(base + lane_base),
                 "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (t == 0) {
        const uint32_t saddr = smem_u32(sB);
        uint64_t desc = 0;
        desc |= (uint64_t)((saddr >> 4) & 0x3FFF);
        desc |= (uint64_t)((128 >> 4) & 0x3FFF) << 16;   // LBO: K-adjacent core matrices
        desc |= (uint64_t)((256 >> 4) & 0x3FFF) << 32;   // SBO: N-adjacent 8-row groups
        desc |= (uint64_t)1 << 46;                        // version 1 (sm100)
        const uint32_t idesc = (2u << 4) | (0u << 7) | (0u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24);
        const uint32_t dcol = base + 32, acol = base;
        for (int rep = 0; rep < (accumulate_twice ? 2 : 1); ++rep) {
            const uint32_t acc = rep;
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(dcol),
                "r"(acol), "l"(desc), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&bar)));
    }
    // everyone waits for the MMA
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
            smem_u32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t d[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
          "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
        : "r"(base + lane_base + 32));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int n = 0; n < 16; ++n) D[t * 16 + n] = (int32_t)d[n];
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(64));
}

int main() {
    uint8_t hA[128 * 32], hB[16 * 32];
    srand(1);
    for (auto& v : hA) v = rand() & 0xFF;
    for (auto& v : hB) v = rand() & 0xFF;
    uint8_t *dA, *dB;
    int32_t* dD;
    cudaMalloc(&dA, sizeof hA);
    cudaMalloc(&dB, sizeof hB);
    cudaMalloc(&dD, 128 * 16 * 4);
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
    int bad_total = 0;
    for (int twice = 0; twice < 2; ++twice) {
        probe<<<1, 128>>>(dA, dB, dD, twice);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("CUDA error: %s\n", cudaGetErrorString(e));
            return 1;
        }
        int32_t hD[128 * 16];
        cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < 16; ++n) {
                int64_t ref = 0;
                for (int k = 0; k < 32; ++k) ref += (int)hA[m * 32 + k] * (int)hB[n * 32 + k];
                ref *= (twice ? 2 : 1);
                if (ref != hD[m * 16 + n]) {
                    if (bad < 5) printf("mismatch m=%d n=%d got %d want %lld\n", m, n, hD[m * 16 + n], (long long)ref);
                    ++bad;
                }
            }
        printf("tcgen05 i8 probe (accumulate=%d): %s (%d mismatches)\n", twice, bad ? "FAIL" : "OK", bad);
        bad_total += bad;
    }
    return bad_total ? 2 : 0;
}
