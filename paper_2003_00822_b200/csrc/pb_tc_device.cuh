// pb_tc_device.cuh -- device building blocks shared by the sm_100a tensor-engine kernels
// (pb_gemm_tc.cu: the bitlayer GEMM; pb_lstm_tc.cu: the persistent LSTM recurrence):
// mbarrier / TMA / tcgen05 wrappers, the A-operand builder for the paired weight storage
// (two bitlayers per e2m1 nibble), pass bookkeeping, grid barriers on monotonic
// counters, and the epilogue's digit sums.  Product code only; nothing here is shared with
// oracle/.
#pragma once
#include <cuda.h>
#include <cstdint>
#include <cuda_runtime.h>

#include "pb_common.cuh"
#include "pb_internal.h"

namespace pb {

constexpr int kChunkWords = 32;               // K-chunk = one 128-byte swizzle row
constexpr int kActAutoFrac = -1024;           // == PB_ACT_AUTO
constexpr uint32_t kWTileBytes = kTcRows * kChunkWords * 4;   // 16 KiB weight tile (128 rows x 32 words)
constexpr uint32_t kSmemMax = 227 * 1024;                     // opt-in dynamic SMEM per CTA

// Tensor maps of the stored weights (pb.h pairs + canonical last layer), cached per thread
// (pb_gemm_tc.cu).
cudaError_t tc_weight_maps(const GemmArgs& g, CUtensorMap* pmap, CUtensorMap* smap);

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate, uint32_t sfa, uint32_t sfb) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %3, [%5], [%6], p;\n}\n" ::"r"(
            d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(sfa), "r"(sfb)
        : "memory");
}
// The same with A from SMEM (descriptor a_desc, the layout of b_desc below).
__device__ __forceinline__ void tc_mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate, uint32_t sfa, uint32_t sfb) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(
            d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(sfa), "r"(sfb)
        : "memory");
}
// K-major, no swizzle: core matrix = 8 rows x 16 B; LBO = 128 B (K-adjacent),
// SBO = 256 B (next 8 rows); version 1 (sm_100).
__device__ __forceinline__ uint64_t b_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
           ((uint64_t)1 << 46);
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}
// The shared::cluster address of `addr` in the CTA of cluster rank `rank` (DSMEM).
__device__ __forceinline__ uint32_t mapa_shared_u32(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ void st_tmem_x32(uint32_t addr, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
        "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
        "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
__device__ __forceinline__ void ld_tmem_x8(uint32_t addr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(addr)
                 : "memory");
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n"
        : "=r"(pred));
    return pred != 0;
}
template <int N>
__device__ __forceinline__ void ld_tmem_cols(uint32_t addr, uint32_t (&v)[N]) {
    static_assert(N % 8 == 0, "8-column granularity");
#pragma unroll
    for (int c = 0; c < N; c += 8) {
        uint32_t t[8];
        ld_tmem_x8(addr + c, t);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[c + e] = t[e];
    }
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// A registers from the stored weights (pb.h), 8 32-column blocks -> 32
// registers; register 4k + r holds in nibble e column 32k + 4e + r (the B
// operand's order, pb_act.cu):
//   KIND 0, a stored pair used whole: block k = words (P0, P1) = even / odd
//     columns as (lower, upper) bit pairs, so nibble e of A_r is already the
//     e2m1 code 1.0*upper + 0.5*lower of column 4e + r after one mask:
//       A_0 = P0 & 0x33333333, A_1 = P1 & .., A_2 = (P0 >> 2) & .., A_3 = (P1 >> 2) & ..
//   KIND 1, upper layer only (k_used odd): 0.5*upper (the pass unit becomes |S_upper|):
//       A_0 = (P0 >> 1) & 0x11111111, ..., A_3 = (P1 >> 3) & 0x11111111
//   KIND 2, canonical single layer (the last layer of an odd L): A_r = (w >> r) & 0x11111111.
// The sign layer (pass 0) carries its negative weight S_0 in the nibble's sign bit
// (sign_nibbles below), so every product is the signed integer term of sum_i S_i W_i and no
// correction term remains.
template <int KIND>
__device__ __forceinline__ void build_a(const uint4 (&q)[4], uint32_t xm, uint32_t (&v)[32]) {
    const uint32_t w[16] = {q[0].x, q[0].y, q[0].z, q[0].w, q[1].x, q[1].y, q[1].z, q[1].w,
                            q[2].x, q[2].y, q[2].z, q[2].w, q[3].x, q[3].y, q[3].z, q[3].w};
    constexpr uint32_t kM3 = 0x33333333u, kM1 = 0x11111111u;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if (KIND == 0) {
            const uint32_t p0 = w[2 * k], p1 = w[2 * k + 1];
            v[4 * k + 0] = (p0 ^ xm) & kM3;
            v[4 * k + 1] = (p1 ^ xm) & kM3;
            v[4 * k + 2] = ((p0 >> 2) ^ (xm >> 2)) & kM3;
            v[4 * k + 3] = ((p1 >> 2) ^ (xm >> 2)) & kM3;
        } else if (KIND == 1) {
            const uint32_t p0 = w[2 * k], p1 = w[2 * k + 1];
            v[4 * k + 0] = ((p0 >> 1) ^ (xm >> 1)) & kM1;
            v[4 * k + 1] = ((p1 >> 1) ^ (xm >> 1)) & kM1;
            v[4 * k + 2] = ((p0 >> 3) ^ (xm >> 3)) & kM1;
            v[4 * k + 3] = ((p1 >> 3) ^ (xm >> 3)) & kM1;
        } else {
            const uint32_t c = w[k];                       // words 0..7 only
            v[4 * k + 0] = (c ^ xm) & kM1;
            v[4 * k + 1] = ((c >> 1) ^ xm) & kM1;
            v[4 * k + 2] = ((c >> 2) ^ xm) & kM1;
            v[4 * k + 3] = ((c >> 3) ^ xm) & kM1;
        }
    }
}

// Pass 0 of a code: the sign layer's nibbles signed.  Per e2m1 nibble (bit 3 = sign):
//   KIND 0, (upper = sign W_0, lower = W_1): -1.0 W_0 + 0.5 W_1 in {0, 0.5, -1, -0.5}
//     = 0000 / 0001 / 1010 / 1001: bit 3 = U, bit 1 = U & ~L, bit 0 = L;
//   KIND 1 (the sign layer alone, k_used = 1): -0.5 W_0 (1001 or 0);
//   KIND 2 (L = 1): -0.5 W_0, or for the binary code 1 - 2 W_0 (offset 1): +-0.5.
template <int KIND>
__device__ __forceinline__ uint32_t sign_nibbles(uint32_t x, bool binary) {
    constexpr uint32_t kM1 = 0x11111111u, kM2 = 0x22222222u;
    if (KIND == 0) {
        const uint32_t u = x & kM2, l = x & kM1;
        return (u << 2) | (u & ~(l << 1)) | l;
    }
    return (x << 3) | (KIND == 2 && binary ? kM1 : x);
}

// One pass of one row.  Paired storage: the pass's 32 blocks are 64 words in
// two 16 KiB stages (t0: blocks 0..15, t1: 16..31); canonical: 32 words in one
// stage.  A stage's 8 chunks of the row are read from the swizzled tile (128B
// swizzle: chunk c of row m at c ^ (m & 7)) and the stage goes back to the TMA
// producer before its A registers are built and stored to TMEM (32 columns
// per 4 chunks).
template <int KIND, bool SMEM = false, bool WAITST = true>
__device__ __forceinline__ void convert_pass(uint32_t t0, uint32_t t1, uint32_t swz, uint32_t dst, uint32_t xm,
                                             int sgn, int dbg, uint64_t* rel0, uint64_t* rel1, int lane) {
    constexpr bool kPair = KIND <= 1;
    if (dbg == 4) {                             // profiling knob: the pipeline skeleton only
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(rel0);
            if (kPair) mbar_arrive(rel1);
        }
        return;
    }
#pragma unroll
    for (int t = 0; t < (kPair ? 2 : 1); ++t) {
        uint4 q[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) q[c] = lds128((t == 0 ? t0 : t1) + ((((uint32_t)c) ^ swz) << 4));
        __syncwarp();
        if (lane == 0) mbar_arrive(t == 0 ? rel0 : rel1);
#pragma unroll
        for (int h = 0; h < (kPair ? 2 : 4); ++h) {
            uint32_t v[32];
            if (kPair) {
                const uint4 qq[4] = {q[4 * h], q[4 * h + 1], q[4 * h + 2], q[4 * h + 3]};
                build_a<KIND>(qq, xm, v);
            } else {
                const uint4 qq[4] = {q[2 * h], q[2 * h + 1], q[2 * h], q[2 * h + 1]};
                build_a<KIND>(qq, xm, v);
            }
            if (sgn) {                          // warp-uniform: pass 0 only
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = sign_nibbles<KIND>(v[i], sgn == 2);
            }
            const int b4 = kPair ? 2 * t + h : h;
            if (SMEM) {
                // A in SMEM for an SS MMA (K-major, no swizzle, the layout of b_desc): dst is this
                // row's core-matrix line; MMA uu = 4 b4 + j at uu * 4 KiB, its K halves 128 B apart
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t ad = dst + (uint32_t)((4 * b4 + j) * 4096);
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(ad), "r"(v[8 * j]), "r"(v[8 * j + 1]),
                                 "r"(v[8 * j + 2]), "r"(v[8 * j + 3])
                                 : "memory");
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(ad + 128u), "r"(v[8 * j + 4]),
                                 "r"(v[8 * j + 5]), "r"(v[8 * j + 6]), "r"(v[8 * j + 7])
                                 : "memory");
                }
            } else if (dbg != 1 && dbg != 3) {
                st_tmem_x32(dst + (uint32_t)(32 * b4), v);
                // the next build_a rewrites registers this asynchronous store reads: wait for it
                // first (measured: without this wait the wide batched path lost an A row
                // intermittently -- a few rows of one pass, 2-8% of C4 B=128 calls -- depending on
                // how ptxas scheduled the register reuse).  The batch-1 GEMM, where a wait per
                // store costs 2-3 us per call, uses convert_pass_ka instead
                if (WAITST) tmem_st_wait();
            }
            else if (v[0] == 0x12345 && v[3] == 0x777)
                asm volatile("trap;");   // keep the ALU work alive
        }
    }
}

// tcgen05.wait::st that keeps the 32 source registers of the store it waits for live up to this
// point, so the compiler cannot give them to other values while that store may still read them.
__device__ __forceinline__ void tmem_st_wait_keep(const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.wait::st.sync.aligned;" ::"r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
        "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
        "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
        "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
// convert_pass for the batch-1 GEMM (TMEM destination, no sign nibbles): the 4 A stores of a
// pass alternate two register sets; store k waits for store k - 1 (its registers kept live) after
// building k's registers, so the build overlaps the previous store and no source register is
// rewritten while a store may read it; one wait per pass is exposed (the last store's).
template <int KIND>
__device__ __forceinline__ void convert_pass_ka(uint32_t t0, uint32_t t1, uint32_t swz, uint32_t dst, uint32_t xm,
                                                int dbg, uint64_t* rel0, uint64_t* rel1, int lane) {
    constexpr bool kPair = KIND <= 1;
    if (dbg == 4) {                             // profiling knob: the pipeline skeleton only
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(rel0);
            if (kPair) mbar_arrive(rel1);
        }
        return;
    }
    const bool store = dbg != 1 && dbg != 3;
    uint32_t va[32], vb[32];
#pragma unroll
    for (int t = 0; t < (kPair ? 2 : 1); ++t) {
        uint4 q[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) q[c] = lds128((t == 0 ? t0 : t1) + ((((uint32_t)c) ^ swz) << 4));
        __syncwarp();
        if (lane == 0) mbar_arrive(t == 0 ? rel0 : rel1);
#pragma unroll
        for (int h = 0; h < (kPair ? 2 : 4); ++h) {
            const int k = kPair ? 2 * t + h : h;              // store index (compile time)
            uint32_t(&v)[32] = (k & 1) ? vb : va;
            if (kPair) {
                const uint4 qq[4] = {q[4 * h], q[4 * h + 1], q[4 * h + 2], q[4 * h + 3]};
                build_a<KIND>(qq, xm, v);
            } else {
                const uint4 qq[4] = {q[2 * h], q[2 * h + 1], q[2 * h], q[2 * h + 1]};
                build_a<KIND>(qq, xm, v);
            }
            if (k > 0) tmem_st_wait_keep((k & 1) ? va : vb);
            if (store) st_tmem_x32(dst + (uint32_t)(32 * k), v);
            else if (v[0] == 0x12345 && v[3] == 0x777) asm volatile("trap;");
        }
    }
    tmem_st_wait_keep(vb);                                    // the last store (k = 3)
}

// Least significant layer of pass ps (the pass's unit weight is |S_lo|).
__device__ __host__ __forceinline__ int pass_lo(int k_used, int ps) {
    return (2 * ps + 1 < k_used) ? 2 * ps + 1 : 2 * ps;
}
// Accumulator region of pass ps, its block-scale exponent s (weight 2^s
// relative to the region's least significant layer) and whether it opens
// the region (first MMA overwrites).
__device__ __forceinline__ void pass_region_g(int Gp, int passes, int k_used, int ps, int& region, int& s,
                                              bool& first) {
    region = ps / Gp;
    int last = (region + 1) * Gp - 1;
    if (last > passes - 1) last = passes - 1;
    s = pass_lo(k_used, last) - pass_lo(k_used, ps);
    first = (ps == region * Gp);
}
// |S_i|: 2^(L-1-i), the unit of a pass whose least significant layer is i.  The
// binary code 1 - 2 W_0 (offset 1) is carried whole by its +-0.5 nibbles: unit 1.
// Complemented sign layer (xm, the tensor engine's batch path): the binary layer's unit is
// |S_0| = 2, with the correction (o - |S_0|) sum_c x_q in the epilogue.
__device__ __forceinline__ unsigned long long layer_mag(int L, int offset, int i, bool complement = false) {
    if (i == 0 && offset) return complement ? 2ull : 1ull;
    return 1ull << (L - 1 - i);
}

__device__ __forceinline__ void red_add_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_shared_u64(uint32_t a, unsigned long long v) {
    asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_shared_u64(uint32_t a) {
    unsigned long long v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
    return v;
}
// Grid barriers on monotonic 64-bit counters in the workspace: every barrier
// instance adds exactly kGridStride in total (CTA 0 adds kGridStride - (G-1), the
// others 1) with one fire-and-forget red.release each, so nothing is reset and no
// arrival waits for a returned value.  A CTA reads the counter after its PDL wait
// (every earlier call has completed, and no instance of this call can complete
// before this CTA arrives): the instance's base is that value rounded down to a
// multiple of kGridStride, and it is complete once the counter reaches base + stride.
constexpr unsigned long long kGridStride = 1ull << 20;
__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// Relaxed gpu-scope 64-bit access (single-copy atomic): tagged values that validate themselves.
__device__ __forceinline__ unsigned long long ld_relaxed_gpu_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_gpu_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// Cross-rank wait (f2): spin on an arrival counter other GPUs add to; a peer that never
// arrives (a rank that died or diverged) ends the kernel with a trap after 30 s instead of
// hanging the device.
__device__ __forceinline__ void sys_wait(const unsigned long long* ctr, unsigned long long target) {
    long long t0 = 0;
    for (unsigned k = 0; ld_acquire_sys_u64(ctr) < target; ++k) {
        if ((k & 1023) == 1023) {
            long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t0 == 0) t0 = t;
            else if (t - t0 > 30000000000ll) asm volatile("trap;");
        }
    }
}
__device__ __forceinline__ unsigned long long grid_base(const int* ctr) {
    return ld_acquire_gpu_u64(reinterpret_cast<const unsigned long long*>(ctr)) & ~(kGridStride - 1);
}
__device__ __forceinline__ void grid_arrive(int* ctr) {
    const unsigned long long v = blockIdx.x == 0 ? kGridStride - (gridDim.x - 1) : 1ull;
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(ctr), "l"(v) : "memory");
}
__device__ __forceinline__ void grid_wait(const int* ctr, unsigned long long base) {
    const unsigned long long* c = reinterpret_cast<const unsigned long long*>(ctr);
    while (ld_acquire_gpu_u64(c) < base + kGridStride) {
    }
}
// An accumulator column as a signed integer (|D| < 2^24: exact in f32).
__device__ __forceinline__ unsigned long long d2i(uint32_t bits) {
    return (unsigned long long)(long long)__float2int_rn(__uint_as_float(bits));
}
// Epilogue digit sums for a compile-time even a = 2 ND (ND divides CG): CG accumulator
// columns hold CG / ND batch columns of the slice, digit k of column q at q * ND + k.  The
// digit weights U_k = 4^(ND-1-k) (pb_common.cuh; the sign rides in digit 0) are applied as
// shifts on independent terms (two interleaved partial sums, not one serial Horner chain),
// then the group weight wr; per-column totals go to s_tot [bc][128] (exact modulo 2^64).
template <int CG, int ND>
__device__ __forceinline__ void plane_sums_ca(uint32_t dreg, int nb, int m, uint32_t s_tot_s,
                                              unsigned long long wr, bool first) {
    static_assert(CG % ND == 0, "ND must divide the column group");
#pragma unroll 1
    for (int c0 = 0; c0 < nb * ND; c0 += CG) {
        uint32_t dv[CG];
        ld_tmem_cols<CG>(dreg + (uint32_t)c0, dv);
        tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < CG / ND; ++q) {
            unsigned long long s0 = 0, s1 = 0;
#pragma unroll
            for (int k = 0; k < ND; ++k) {
                const unsigned long long t = d2i(dv[q * ND + k]) << (2 * (ND - 1 - k));
                if (k & 1) s1 += t;
                else s0 += t;
            }
            const int bc = c0 / ND + q;
            if (bc < nb) {
                const uint32_t sa = s_tot_s + (uint32_t)(bc * kTcRows + m) * 8u;
                const unsigned long long t = (s0 + s1) * wr;
                st_shared_u64(sa, first ? t : t + ld_shared_u64(sa));
            }
        }
    }
}
// a in {8, 16, 32}: the compile-time form above; false for any other a.
template <int NPAD>
__device__ __forceinline__ bool plane_sums_dispatch(int a, uint32_t dreg, int nb, int m, uint32_t s_tot_s,
                                                    unsigned long long wr, bool first) {
    constexpr int CG = NPAD < 32 ? NPAD : 32;
    if (a == 8) {
        plane_sums_ca<CG, 4>(dreg, nb, m, s_tot_s, wr, first);
        return true;
    }
    if (a == 16) {
        plane_sums_ca<CG, 8>(dreg, nb, m, s_tot_s, wr, first);
        return true;
    }
    if constexpr (CG >= 16) {
        if (a == 32) {
            plane_sums_ca<CG, 16>(dreg, nb, m, s_tot_s, wr, first);
            return true;
        }
    }
    return false;
}


// E8M0 block scale factors in TMEM columns [sf_col, sf_col + 64) (warps of one lane-quarter
// set, warp & 3 = quarter): columns 0..3 = 1.0 (SFA), columns 4(1+s)..4(1+s)+3 = 2^s (SFB of
// passes with in-group weight 2^s); every byte of a column holds the same value.
__device__ __forceinline__ void store_scale_factors(uint32_t tmem, int warp, int sf_col) {
#pragma unroll
    for (int blk = 0; blk < 4; ++blk) {
        uint32_t v[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            const int col = blk * 16 + c, sidx = col / 4;   // sidx 0 = SFA, 1 + s = 2^s
            v[c] = 0x01010101u * (uint32_t)(127 + (sidx == 0 ? 0 : sidx - 1));
        }
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
                tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(sf_col + blk * 16)),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
            "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
            : "memory");
    }
}
// kind::mxf4 instruction descriptor: A, B = E2M1, scale format UE8M0, K = 64, M = 128, N = npad.
__host__ __device__ constexpr uint32_t mxf4_idesc(int npad) {
    return (1u << 7) | (1u << 10) | ((uint32_t)(npad >> 3) << 17) | (1u << 23) | ((uint32_t)(kTcRows >> 4) << 24);
}
// Exact f32 accumulation bound: passes per accumulator group for K padded columns
// (|D| < 3 K 2^G <= 2^24, pb_gemm_tc.cu make_plan), at most 7 (SFB exponents 0..13).
inline int tc_group_passes(int64_t kwords) {
    int k = 0;
    while (((int64_t)1 << k) < 3 * kwords * 32) ++k;
    int G = 24 - k;
    if (G > 15) G = 15;
    return G / 2;
}

}  // namespace pb
