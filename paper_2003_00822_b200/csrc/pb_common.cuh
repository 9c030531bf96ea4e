// pb_common.cuh -- small device helpers for the sm_100a kernels (product code).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pb {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 128-bit streaming load of packed weights: read once, do not pollute L1.
__device__ __forceinline__ uint4 ld_stream_u4(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// ---- mbarrier + 1-D TMA bulk copy (cp.async.bulk -> UBLKCP) ----
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared bulk copy, completion counted on `bar` (bytes % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Shift-weighted reduction scales: T_j and S_i as wrapping
// 64-bit integers.  All accumulation is done modulo 2^64, which is exact as
// long as the final value fits int64 (the G11 guard checked on the host).
__device__ __forceinline__ unsigned long long plane_scale(int a, int j) {
    const unsigned long long p = 1ull << (a - 1 - j);
    return j == 0 ? (0ull - p) : p;
}
__device__ __forceinline__ unsigned long long layer_scale(int L, int offset, int i) {
    if (i == 0) return offset ? (0ull - 2ull) : (0ull - (1ull << (L - 1)));
    return 1ull << (L - 1 - i);
}

// Dequant epilogue (reading G13): y = (float) ldexp((double)acc * s_w, -f_b),
// then bias / accumulate / fn in fp32.
__device__ __forceinline__ float dequant(long long acc, double scale, int f) {
    double t = __dmul_rn(__ll2double_rn(acc), scale);
    t = ldexp(t, -f);
    return __double2float_rn(t);
}
__device__ __forceinline__ float apply_fn(float v, int fn) {
    switch (fn) {
        case 1: return v > 0.f ? v : 0.f;
        case 2: return tanhf(v);
        case 3: return 1.f / (1.f + expf(-v));
        default: return v;
    }
}

}  // namespace pb
