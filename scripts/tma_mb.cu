// tma_mb.cu -- streaming rate of TMA tile loads into an SMEM ring (one CTA per SM),
// consumer releases each stage immediately: the ceiling of the weight producer of
// pb_gemm_tc.cu.  Tensor {kwords, R, L} uint32, box {32, 128, 1}, 128B swizzle, as there.
#include <cuda.h>
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

// ORDER 0: tiles in memory order (k fastest, then rows, then layers);
// ORDER 1: the GEMM's order -- per (row tile, k chunk) unit all L layers, units contiguous per CTA.
template <int STAGES, int BOXW, int BOXR, int ORDER>
__global__ void __launch_bounds__(64, 1) stream(const __grid_constant__ CUtensorMap map, int kwords, int R, int L,
                                                 int* out, int reps = 1) {
    extern __shared__ __align__(1024) uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
    constexpr uint32_t kTile = BOXW * BOXR * 4;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const long long tiles_k = kwords / BOXW, tiles_r = R / BOXR;
    const long long total = tiles_k * tiles_r * L;
    const long long t0 = total * blockIdx.x / gridDim.x, t1 = total * (blockIdx.x + 1) / gridDim.x;
    if (warp == 0 && lane == 0) {
        int n = 0;
        for (int rp = 0; rp < reps; ++rp)
        for (long long t = t0; t < t1; ++t, ++n) {
            const int st = n % STAGES;
            mbar_wait(&empty[st], ((n / STAGES) & 1) ^ 1);
            long long l, rt, kt;
            if (ORDER == 0) {
                l = t / (tiles_k * tiles_r);
                const long long rem = t - l * tiles_k * tiles_r;
                rt = rem / tiles_k;
                kt = rem - rt * tiles_k;
            } else {
                const long long unit = t / L;
                l = t - unit * L;
                rt = unit / tiles_k;
                kt = unit - rt * tiles_k;
            }
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[st])), "r"(kTile)
                         : "memory");
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                "%4}], [%5];" ::"r"(smem_u32(sm + st * kTile)),
                "l"(&map), "r"((int)(kt * BOXW)), "r"((int)(rt * BOXR)), "r"((int)l), "r"(smem_u32(&full[st]))
                : "memory");
        }
    } else if (warp == 1 && lane == 0) {
        int n = 0;
        uint32_t acc = 0;
        for (int rp = 0; rp < reps; ++rp)
        for (long long t = t0; t < t1; ++t, ++n) {
            const int st = n % STAGES;
            mbar_wait(&full[st], (n / STAGES) & 1);
            acc += *reinterpret_cast<volatile uint32_t*>(sm + st * kTile + (n & 127) * 4);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
        }
        if (acc == 0x12345678) out[0] = 1;
    }
}


// 1-D bulk copies (cp.async.bulk, no tensor map) of contiguous TILE-byte blocks: the rate of a
// pre-tiled weight layout.  Each CTA streams its contiguous share `reps` times.
template <int STAGES, int TILE>
__global__ void __launch_bounds__(64, 1) stream1d(const uint8_t* src, long long bytes, int* out, int reps) {
    extern __shared__ __align__(1024) uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const long long total = bytes / TILE;
    const long long t0 = total * blockIdx.x / gridDim.x, t1 = total * (blockIdx.x + 1) / gridDim.x;
    if (warp == 0 && lane == 0) {
        int n = 0;
        for (int rp = 0; rp < reps; ++rp)
            for (long long t = t0; t < t1; ++t, ++n) {
                const int st = n % STAGES;
                mbar_wait(&empty[st], ((n / STAGES) & 1) ^ 1);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[st])), "r"(TILE)
                             : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                 smem_u32(sm + st * TILE)),
                             "l"(src + t * TILE), "r"(TILE), "r"(smem_u32(&full[st]))
                             : "memory");
            }
    } else if (warp == 1 && lane == 0) {
        int n = 0;
        uint32_t acc = 0;
        for (int rp = 0; rp < reps; ++rp)
            for (long long t = t0; t < t1; ++t, ++n) {
                const int st = n % STAGES;
                mbar_wait(&full[st], (n / STAGES) & 1);
                acc += *reinterpret_cast<volatile uint32_t*>(sm + st * TILE + (n & 127) * 4);
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
            }
        if (acc == 0x12345678) out[0] = 1;
    }
}
template <int STAGES, int TILE>
void run1d(const uint8_t* buf, long long bytes, int reps) {
    int* d;
    cudaMalloc(&d, 4);
    const size_t smem = STAGES * TILE + 1024;
    cudaFuncSetAttribute(stream1d<STAGES, TILE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int i = 0; i < 3; ++i) stream1d<STAGES, TILE><<<148, 64, smem>>>(buf, bytes, d, reps);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int it = 10;
    for (int i = 0; i < it; ++i) stream1d<STAGES, TILE><<<148, 64, smem>>>(buf, bytes, d, reps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("1d reps %2d stages %2d tile %6d B (%.1f MB): %.1f us  %.0f GB/s  %s\n", reps, STAGES, TILE, bytes / 1e6,
           ms * 1e3 / it, (double)bytes * reps / (ms * 1e-3 / it) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int STAGES, int BOXW, int BOXR, int ORDER = 0>
void run(void* buf, int kwords, int R, int L, int reps = 1) {
    static EncodeTiledFn enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    }
    CUtensorMap map;
    const cuuint64_t dims[3] = {(cuuint64_t)kwords, (cuuint64_t)R, (cuuint64_t)L};
    const cuuint64_t strides[2] = {(cuuint64_t)kwords * 4, (cuuint64_t)kwords * 4 * R};
    const cuuint32_t box[3] = {BOXW, BOXR, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        BOXW * 4 <= 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int* d;
    cudaMalloc(&d, 4);
    const size_t smem = STAGES * BOXW * BOXR * 4 + 1024;
    cudaFuncSetAttribute(stream<STAGES, BOXW, BOXR, ORDER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int i = 0; i < 3; ++i) stream<STAGES, BOXW, BOXR, ORDER><<<148, 64, smem>>>(map, kwords, R, L, d, reps);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int it = 10;
    for (int i = 0; i < it; ++i) stream<STAGES, BOXW, BOXR, ORDER><<<148, 64, smem>>>(map, kwords, R, L, d, reps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)kwords * 4 * R * L * reps;
    printf("reps %d order %d stages %2d box %3dx%3d (%5d B): %.1f us  %.0f GB/s  %s\n", reps, ORDER, STAGES, BOXW, BOXR, BOXW * BOXR * 4,
           ms * 1e3 / it, bytes / (ms * 1e-3 / it) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int kwords = 512, R = 16384, L = 8;   // the 16384 x 16384, L = 8 packed layer (268 MB)
    void* buf;
    cudaMalloc(&buf, (size_t)kwords * 4 * R * L);
    cudaMemset(buf, 1, (size_t)kwords * 4 * R * L);
    run<8, 32, 128, 0>(buf, kwords, R, L);
    run<8, 32, 128, 1>(buf, kwords, R, L);
    run<12, 32, 128, 1>(buf, kwords, R, L);
    run<8, 32, 128, 0>(buf, kwords, R, L);
    run<8, 32, 128, 1>(buf, kwords, R, L);
    // L2-resident (33.5 MB, streamed 8 times per launch): the TMA box rate without HBM
    run<8, 32, 128, 1>(buf, kwords, R, 2, 8);
    run<12, 32, 128, 1>(buf, kwords, R, 2, 8);
    run<12, 32, 64, 1>(buf, kwords, R, 2, 8);
    run<12, 32, 32, 1>(buf, kwords, R, 2, 8);
    run<12, 32, 128, 1>(buf, kwords, R, 1, 16);
    const uint8_t* b8 = static_cast<const uint8_t*>(buf);
    run1d<12, 16384>(b8, 268435456ll, 1);
    run1d<12, 16384>(b8, 33554432ll, 8);
    run1d<12, 8192>(b8, 33554432ll, 8);
    run1d<6, 32768>(b8, 33554432ll, 8);
    run1d<12, 16384>(b8, 16777216ll, 16);
    return 0;
}
