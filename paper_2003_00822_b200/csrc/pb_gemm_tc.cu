// pb_gemm_tc.cu -- steps a3-a5 on the 5th-generation tensor cores (engine MMA).
//
// The 0/1 products of P:205-206 (W_i[r,c] AND X_j[b,c], summed over c) are
// computed by tcgen05.mma.kind::mxf4.block_scale (packed e2m1 x e2m1 -> f32,
// SASS UTCOMMA) with TWO adjacent bitlayers stacked in every A nibble -- the
// "multiple bitlayers may be stacked together" option of P:206:
//   * e2m1 nibbles 0b00hl are exactly 1.0*h + 0.5*l, so the nibble of column
//     c holds the bits of layers (i, i+1) of column c; B holds each plane bit
//     as 2.0 (pb_act.cu), so every product is (2 W_i + W_{i+1}) * x_bit --
//     the two layers' relative weight S_i / S_{i+1} = 2;
//   * the sign layer (S_0 < 0) is carried as its complement with weight
//     |S_0| plus the exact correction -|S_0| * sum_c x_q (since
//     -|S_0| s = |S_0| (1 - s) - |S_0|), so every layer weight is a positive
//     power of two and the layers pair up as (0,1), (2,3), ...;
//   * the passes of a group ride on the E8M0 block scale of B (2^s, exact),
//     so a whole group accumulates into one TMEM accumulator
//     D_g = sum_pass 2^s (2 C_hi + C_lo), exact in f32 while K * 2^G <= 2^24
//     (G = layers per group).
// Plane weights T_j, the group weights and the sign correction are applied in
// the exact int64 epilogue, as in the POPC engine.
//
// Building A (per pair of words hi, lo and register r = 0..3, nibble e =
// column 4e + r):  ((hi >> (r-1)) & 0x22222222) | ((lo >> r) & 0x11111111),
// stored with tcgen05.st.32x32b (lane = row).
//
// Why this shape (measured on B200, scripts/tc_mb.cu): an M=128
// tcgen05 MMA costs ~55 cycles for any N <= 64 (an M=256 CTA-pair MMA costs the
// same on two SMs), so weight bits per MMA set the rate: kind::i8 with byte
// operands carries 32 bits per row, kind::mxf4 nibbles with one layer carry
// 64, two stacked layers 128.  The issuing warp blocks on each MMA, so
// barrier round trips between MMAs are paid serially; an A slot therefore
// holds a whole 32-word pass (16 MMAs) per handshake, and the two converter
// h-sets take alternate passes.
//
// Work decomposition: stream-K over units (128-row tile, 32-word K-chunk);
// each CTA (one per SM, persistent) walks a contiguous unit range; each B chunk
// staged in SMEM serves all k_used layers of the chunk.  A CTA that
// covers a whole tile writes y directly; a CTA holding part of a tile parks
// its int64 sums in its own slot and bumps the tile's arrival counter; the
// last arriving CTA sums the slots of all contributors (fixed order, exact)
// and resets the counter, so the workspace is left as it was found.
//
// Warp roles (11 warps):
//   warp 0      weight producer: TMA (cp.async.bulk.tensor.3d, 128B swizzle)
//               of 128-row x 32-word bitlayer tiles into an 8-stage SMEM ring;
//               starts before the activation kernel finishes (PDL);
//   warp 1      TMEM allocator and MMA issuer (one elected lane);
//   warp 2      B producer: 1-D bulk copies of the plane tiles (after PDL wait);
//   warps 3..10 converters: thread = weight row; read the row's words of the
//               pass's one or two tiles from the swizzled SMEM ring, build A,
//               tcgen05.st it into the TMEM A ring (software-pipelined: a slot
//               is published while the next is built); warps 3..6 also run
//               the epilogue.
#include <cuda.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "pb_common.cuh"
#include "pb_internal.h"

namespace pb {
namespace {

constexpr int kConvWarps = 8;                 // 2 h-sets of 4 warps (one per TMEM lane quarter)
constexpr int kHSets = kConvWarps / 4;
constexpr int kConv0 = 3;                     // first converter warp
constexpr int kThreads = 32 * (kConv0 + kConvWarps);
constexpr int kMaxSlots = 4;                  // A ring: up to 4 slots x 128 TMEM columns (16 MMAs each)
constexpr int kMaxRegions = 4;                // TMEM accumulators: sign layer + magnitude groups
constexpr int kChunkWords = 32;               // K-chunk = one 128-byte swizzle row
constexpr int kWStages = 8;                   // weight tile ring
constexpr uint32_t kWTileBytes = kTcRows * kChunkWords * 4;   // 16 KiB
constexpr uint32_t kBStageMax = (kChunkWords / 2) * kTcMaxN * 32;   // 16 KiB
constexpr uint32_t kTotBytes = kTcMaxN * kTcRows * 8;          // epilogue per-row, per-batch int64 sums
constexpr uint32_t kSmemBytes = 1024 + 1024 + kWStages * kWTileBytes + 2 * kBStageMax + kTotBytes;

struct Bars {
    uint64_t a_full[kMaxSlots], a_empty[kMaxSlots];   // a_full: the 4 warps of one h-set
    uint64_t w_full[kWStages], w_empty[kWStages];
    uint64_t b_full[2], b_empty[2];
    uint64_t d_full, d_empty;
    uint32_t tmem_base;
    int last_flag;
};

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
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 8 words of the hi layer and 8 of the lo layer -> 32 nibble registers (file
// header).  MODE 0: pair; 1: pair, hi = sign layer (complemented); 2: lo alone
// (hi = 0); 3: lo alone and it is the sign layer (complemented).
template <int MODE>
__device__ __forceinline__ void build_a(const uint4 h0, const uint4 h1, const uint4 l0, const uint4 l1,
                                        uint32_t (&v)[32]) {
    const uint32_t hs[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
    const uint32_t ls[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
#pragma unroll
    for (int uu = 0; uu < 8; ++uu) {
        const uint32_t lo = (MODE == 3) ? ~ls[uu] : ls[uu];
        if (MODE >= 2) {
            v[uu * 4 + 0] = lo & 0x11111111u;
            v[uu * 4 + 1] = (lo >> 1) & 0x11111111u;
            v[uu * 4 + 2] = (lo >> 2) & 0x11111111u;
            v[uu * 4 + 3] = (lo >> 3) & 0x11111111u;
        } else {
            const uint32_t hi = (MODE == 1) ? ~hs[uu] : hs[uu];
            v[uu * 4 + 0] = ((hi << 1) & 0x22222222u) | (lo & 0x11111111u);
            v[uu * 4 + 1] = (hi & 0x22222222u) | ((lo >> 1) & 0x11111111u);
            v[uu * 4 + 2] = ((hi >> 1) & 0x22222222u) | ((lo >> 2) & 0x11111111u);
            v[uu * 4 + 3] = ((hi >> 2) & 0x22222222u) | ((lo >> 3) & 0x11111111u);
        }
    }
}

// One pass of one row: 4 x (8 hi + 8 lo words from the swizzled SMEM tiles ->
// 32 A registers -> tcgen05.st of 32 TMEM columns).
template <int MODE>
__device__ __forceinline__ void convert_pass(uint32_t thi, uint32_t tlo, uint32_t swz, uint32_t dst, int dbg) {
#pragma unroll 1
    for (int b4 = 0; b4 < 4; ++b4) {
        // 128B swizzle: 16-byte chunk c of row m lives at chunk c ^ (m & 7)
        const uint32_t c0 = (((uint32_t)(2 * b4)) ^ swz) << 4;
        const uint32_t c1 = (((uint32_t)(2 * b4 + 1)) ^ swz) << 4;
        const uint4 l0 = lds128(tlo + c0), l1 = lds128(tlo + c1);
        uint4 h0 = l0, h1 = l1;
        if (MODE <= 1) {
            h0 = lds128(thi + c0);
            h1 = lds128(thi + c1);
        }
        uint32_t v[32];
        build_a<MODE>(h0, h1, l0, l1, v);
        if (dbg != 1 && dbg != 3)
            st_tmem_x32(dst + (uint32_t)(32 * b4), v);
        else if (v[0] == 0x12345 && v[3] == 0x777)
            asm volatile("trap;");   // keep the ALU work alive
    }
}

// Profiling (PB_TC_DEBUG=5): accumulate cycles spent in each wait site.
#define TWAIT(bar, ph, slotid)                                   \
    do {                                                         \
        if (p.prof) {                                            \
            const long long _t0 = clock64();                     \
            mbar_wait(bar, ph);                                  \
            prof[slotid] += clock64() - _t0;                     \
        } else {                                                 \
            mbar_wait(bar, ph);                                  \
        }                                                        \
    } while (0)

// Host-chosen decomposition and TMEM map: [0, 128*slots) A ring,
// [sf_col, sf_col + 64): columns 0..3 = SFA (1.0), columns 4(1+s).. = SFB 2^s
// (scale-factor operands are addressed at 4-column granularity);
// [d_col, d_col + regions*NPAD): one accumulator per group of passes.
struct TcPlan {
    int tiles;        // ceil(R / 128)
    int chunks;       // 32-word K-chunks per tile
    long long units;  // tiles * chunks
    int slots, sf_col, d_col;
    int passes;       // ceil(k_used / 2): layer pairs (0,1), (2,3), ...
    int Gp;           // passes per accumulator group (<= G/2 layers pairs, K * 2^G <= 2^24)
    int regions;      // ceil(passes / Gp)
    int dbg;          // profiling knob (env PB_TC_DEBUG): 1 = no A store, 2 = no MMA, 3 = neither,
                      // 6 = per-CTA timeline
    int prof;         // env PB_TC_PROF: print wait-cycle totals of CTA 0
};

// Least significant layer of pass ps (the pass's unit weight is |S_lo|).
__device__ __host__ __forceinline__ int pass_lo(int k_used, int ps) {
    return (2 * ps + 1 < k_used) ? 2 * ps + 1 : 2 * ps;
}
// Accumulator region of pass ps, its block-scale exponent s (weight 2^s
// relative to the region's least significant layer) and whether it opens
// the region (first MMA overwrites).
__device__ __forceinline__ void pass_region(const TcPlan& p, int k_used, int ps, int& region, int& s, bool& first) {
    region = ps / p.Gp;
    int last = (region + 1) * p.Gp - 1;
    if (last > p.passes - 1) last = p.passes - 1;
    s = pass_lo(k_used, last) - pass_lo(k_used, ps);
    first = (ps == region * p.Gp);
}
// |S_i|: 2^(L-1-i); the binary layer (offset 1) has |S_0| = 2.
__device__ __forceinline__ unsigned long long layer_mag(int L, int offset, int i) {
    if (i == 0 && offset) return 2ull;
    return 1ull << (L - 1 - i);
}

// A CTA's units [u0, u1) split into segments of one row tile: [kcA, kcB) of tile rt.
struct Seg {
    int rt, kcA, kcB;
    long long next;
};
__device__ __forceinline__ Seg segment(const TcPlan& p, long long u, long long u1) {
    Seg s;
    s.rt = (int)(u / p.chunks);
    s.kcA = (int)(u - (long long)s.rt * p.chunks);
    long long ue = (long long)(s.rt + 1) * p.chunks;
    if (ue > u1) ue = u1;
    s.kcB = s.kcA + (int)(ue - u);
    s.next = ue;
    return s;
}

template <int NPAD>
__global__ void __launch_bounds__(kThreads, 1)
bitgemm_tc_kernel(const GemmArgs g, const TcPlan p, const __grid_constant__ CUtensorMap wmap)
{
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment for the 128B-swizzled TMA tiles
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Bars& bars = *reinterpret_cast<Bars*>(smem);
    uint8_t* wtile0 = smem + 1024;
    uint8_t* btile0 = wtile0 + kWStages * kWTileBytes;
    unsigned long long* s_tot = reinterpret_cast<unsigned long long*>(btile0 + 2 * kBStageMax);  // [b][128]
    constexpr uint32_t kBTile = NPAD * 32;                    // one MMA's B (64 columns)
    constexpr uint32_t kBStage = (kChunkWords / 2) * kBTile;  // one K-chunk (16 MMAs)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long G = gridDim.x;
    long long prof[5] = {0, 0, 0, 0, 0};
    const long long t_start = clock64();
    long long g_start;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_start));
    const long long u0 = p.units * blockIdx.x / G, u1 = p.units * (blockIdx.x + 1) / G;

    if (threadIdx.x == 0) {
        for (int s = 0; s < p.slots; ++s) {
            mbar_init(&bars.a_full[s], 4);               // the 4 converter warps of one h-set
            mbar_init(&bars.a_empty[s], 1);
        }
        for (int s = 0; s < kWStages; ++s) {
            mbar_init(&bars.w_full[s], 1);
            mbar_init(&bars.w_empty[s], 4);              // the h-set that converts the tile
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bars.b_full[s], 1);
            mbar_init(&bars.b_empty[s], 1);
        }
        mbar_init(&bars.d_full, 1);
        mbar_init(&bars.d_empty, 4);
        fence_mbar_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(&wmap) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            smem_u32(&bars.tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars.tmem_base;
    if (warp >= kConv0 && warp < kConv0 + 4) {
        // E8M0 block scale factors: columns 0..3 = 1.0 (SFA), columns 4(1+s)..4(1+s)+3 = 2^s
        // (SFB of layers with in-group weight 2^s); every byte of a column holds the same value
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
                    tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(p.sf_col + blk * 16)),
                "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
                : "memory");
        }
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_trigger();

    if (warp == 0) {
        // ------------------------------------------------ weight tile producer (no PDL wait:
        // the packed weights do not depend on the activation kernel)
        int tc = 0;
        for (long long u = u0; u < u1;) {
            const Seg sg = segment(p, u, u1);
            for (int kc = sg.kcA; kc < sg.kcB; ++kc)
                for (int i = 0; i < g.k_used; ++i, ++tc) {
                    const int st = tc % kWStages;
                    TWAIT(&bars.w_empty[st], (uint32_t)(((tc / kWStages) & 1) ^ 1), 0);
                    if (elect_one()) {
                        mbar_arrive_expect_tx(&bars.w_full[st], kWTileBytes);
                        tma_load_3d(wtile0 + st * kWTileBytes, &wmap, kc * kChunkWords, sg.rt * kTcRows, i,
                                    &bars.w_full[st]);
                    }
                    __syncwarp();
                }
            u = sg.next;
        }
    } else if (warp == 2) {
        // ------------------------------------------------ B (plane tile) producer
        pdl_wait();
        int cc = 0;
        for (long long u = u0; u < u1;) {
            const Seg sg = segment(p, u, u1);
            for (int kc = sg.kcA; kc < sg.kcB; ++kc, ++cc) {
                const int st = cc & 1;
                mbar_wait(&bars.b_empty[st], (uint32_t)(((cc >> 1) & 1) ^ 1));
                if (elect_one()) {
                    mbar_arrive_expect_tx(&bars.b_full[st], kBStage);
                    bulk_g2s(btile0 + st * kBStage, g.bexp + (int64_t)kc * kBStage, kBStage, &bars.b_full[st]);
                }
                __syncwarp();
            }
            u = sg.next;
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer: the whole warp walks the
        // schedule (warp-uniform values stay in uniform registers), one elected lane issues.
        // kind::mxf4: A, B = E2M1 (1), scale format UE8M0 (bit 23), K = 64, M = 128
        const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(NPAD >> 3) << 17) | (1u << 23) |
                               ((uint32_t)(kTcRows >> 4) << 24);
        const uint32_t sfa = tmem + p.sf_col;
        uint32_t slot = 0, phase = 0;
        int cc = 0, seg = 0;
        for (long long u = u0; u < u1; ++seg) {
            const Seg sg = segment(p, u, u1);
            if (seg > 0) mbar_wait(&bars.d_empty, (uint32_t)((seg - 1) & 1));
            tc_fence_after();
            for (int kc = sg.kcA; kc < sg.kcB; ++kc, ++cc) {
                const int st = cc & 1;
                TWAIT(&bars.b_full[st], (uint32_t)((cc >> 1) & 1), 1);
                tc_fence_after();
                const uint64_t bdesc0 = b_desc(smem_u32(btile0 + st * kBStage));
                for (int ps = 0; ps < p.passes; ++ps) {
                    int region, sexp;
                    bool first;
                    pass_region(p, g.k_used, ps, region, sexp, first);
                    const uint32_t dcol = tmem + (uint32_t)(p.d_col + region * NPAD);
                    const uint32_t sfb = tmem + (uint32_t)(p.sf_col + 4 * (1 + sexp));
                    const bool open = first && kc == sg.kcA;
                    TWAIT(&bars.a_full[slot], phase, 2);
                    tc_fence_after();
                    if (p.dbg == 2 || p.dbg == 3) {
                        if (elect_one()) tc_commit(&bars.a_empty[slot]);
                    } else if (elect_one()) {
                        // descriptor start address advances in 16 B units: one B tile = NPAD*32 B
                        const uint32_t a0 = tmem + slot * 128;
#pragma unroll
                        for (int uu = 0; uu < 16; ++uu)
                            tc_mma(dcol, a0 + 8 * uu, bdesc0 + uu * (kBTile / 16), idesc,
                                   (uu == 0 && open) ? 0u : 1u, sfa, sfb);
                        tc_commit(&bars.a_empty[slot]);
                    }
                    __syncwarp();
                    if (++slot == (uint32_t)p.slots) {
                        slot = 0;
                        phase ^= 1;
                    }
                }
                if (elect_one()) tc_commit(&bars.b_empty[st]);
                __syncwarp();
            }
            if (elect_one()) tc_commit(&bars.d_full);
            __syncwarp();
            u = sg.next;
        }
    } else {
        // ------------------------------------------------ converters (+ epilogue)
        const int cw = warp - kConv0;
        const int h = cw >> 2;                 // h-set: 0 = warps 3..6 (also the epilogue), 1 = warps 7..10
        const int q = warp & 3;                // TMEM lane quarter this warp may access
        const int m = q * 32 + lane;           // row within the tile
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const uint32_t wtile_s = smem_u32(wtile0) + (uint32_t)m * 128;
        const uint32_t swz = (uint32_t)(m & 7);
        int tc = 0, pc = 0, seg = 0;
        // passes (kc, ps) in issue order; h-set h converts passes pc = h, h + 2, ...; pass pc
        // uses A slot pc % slots; its tiles are tc (hi, if paired) and tc + 1 (or tc alone)
        int slot = h % p.slots, sphase = (h / p.slots) & 1;
        // software pipeline: the TMEM stores of one pass drain while the next is awaited
        int pend_slot = -1;
        auto publish = [&]() {
            if (pend_slot >= 0) {
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars.a_full[pend_slot]);
                pend_slot = -1;
            }
        };
        for (long long u = u0; u < u1; ++seg) {
            const Seg sg = segment(p, u, u1);
            const int64_t row = (int64_t)sg.rt * kTcRows + m;
            const bool row_ok = row < g.R;
            for (int kc = sg.kcA; kc < sg.kcB; ++kc) {
                for (int ps = 0; ps < p.passes; ++ps, ++pc) {
                    const bool paired = 2 * ps + 1 < g.k_used;
                    const int ntile = paired ? 2 : 1;
                    if ((pc & 1) != h) {
                        tc += ntile;
                        continue;
                    }
                    const int st_hi = tc % kWStages, st_lo = (tc + ntile - 1) % kWStages;
                    TWAIT(&bars.w_full[st_hi], (uint32_t)((tc / kWStages) & 1), 3);
                    if (paired)
                        TWAIT(&bars.w_full[st_lo], (uint32_t)(((tc + 1) / kWStages) & 1), 3);
                    const uint32_t thi = wtile_s + (uint32_t)st_hi * kWTileBytes;
                    const uint32_t tlo = wtile_s + (uint32_t)st_lo * kWTileBytes;
                    publish();                          // previous pass's A is in TMEM: tell the MMA
                    TWAIT(&bars.a_empty[slot], (uint32_t)(sphase ^ 1), 4);
                    tc_fence_after();
                    const int mode = paired ? (ps == 0 ? 1 : 0) : (ps == 0 ? 3 : 2);
                    const uint32_t dst = tmem + lane_off + (uint32_t)(slot * 128);
                    switch (mode) {
                        case 0: convert_pass<0>(thi, tlo, swz, dst, p.dbg); break;
                        case 1: convert_pass<1>(thi, tlo, swz, dst, p.dbg); break;
                        case 2: convert_pass<2>(thi, tlo, swz, dst, p.dbg); break;
                        default: convert_pass<3>(thi, tlo, swz, dst, p.dbg); break;
                    }
                    __syncwarp();                       // this warp's words are in TMEM-bound registers
                    if (lane == 0) {
                        mbar_arrive(&bars.w_empty[st_hi]);
                        if (paired) mbar_arrive(&bars.w_empty[st_lo]);
                    }
                    tc += ntile;
                    pend_slot = slot;
                    slot += 2;
                    while (slot >= p.slots) {
                        slot -= p.slots;
                        sphase ^= 1;
                    }
                }
            }
            publish();

            if (h == 0) {
                // ---------------- epilogue: fold the accumulators into exact int64
                mbar_wait(&bars.d_full, (uint32_t)(seg & 1));
                tc_fence_after();
                pdl_wait();
                // tot_b = sum_j T_j sum_r |S_lo(r)| D_r[b*a + j] (+ the sign correction below);
                // lo(r) = least significant layer of group r
                for (int b = 0; b < g.B; ++b) s_tot[b * kTcRows + m] = 0;
                for (int r = 0; r < p.regions; ++r) {
                    int last = (r + 1) * p.Gp - 1;
                    if (last > p.passes - 1) last = p.passes - 1;
                    const unsigned long long wr = layer_mag(g.L, g.offset, pass_lo(g.k_used, last));
#pragma unroll 1
                    for (int c = 0; c < NPAD; c += 8) {
                        uint32_t t8[8];
                        ld_tmem_x8(tmem + lane_off + (uint32_t)(p.d_col + r * NPAD + c), t8);
                        tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const int n = c + e, b = n / g.a, j = n - b * g.a;
                            if (b < g.B)
                                s_tot[b * kTcRows + m] +=
                                    plane_scale(g.a, j) *
                                    (wr * (unsigned long long)__float2uint_rn(__uint_as_float(t8[e])));
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars.d_empty);
                auto tot_of = [&](int b) -> unsigned long long { return s_tot[b * kTcRows + m]; };
                const bool whole = (sg.kcA == 0 && sg.kcB == p.chunks);
                bool finalize = whole;
                if (!whole) {
                    // partial tile: park this CTA's sums in its slot (first segment of
                    // the range -> slot 0, otherwise it is the last -> slot 1)
                    const int myslot = (u == u0) ? 0 : 1;
                    unsigned long long* sl = g.slots + (((int64_t)blockIdx.x * 2 + myslot) * g.B) * kTcRows;
                    for (int b = 0; b < g.B; ++b) sl[b * kTcRows + m] = tot_of(b);
                    __threadfence();
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    if (cw == 0 && lane == 0) {
                        const int add = sg.kcB - sg.kcA;
                        const int old = atomicAdd(&g.counters[sg.rt], add);
                        const int last = (old + add == p.chunks);
                        if (last) g.counters[sg.rt] = 0;      // every call leaves the counters zero
                        bars.last_flag = last;
                    }
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    finalize = bars.last_flag != 0;
                    if (finalize) __threadfence();
                }
                if (finalize && row_ok) {
                    for (int b = 0; b < g.B; ++b) {
                        unsigned long long t;
                        if (whole) {
                            t = tot_of(b);
                        } else {
                            // sum the slots of every CTA whose unit range meets this tile
                            t = 0;
                            const long long t0u = (long long)sg.rt * p.chunks, t1u = t0u + p.chunks;
                            long long c = (t0u * G) / p.units;
                            while (c > 0 && p.units * c / G > t0u) --c;
                            while (p.units * (c + 1) / G <= t0u) ++c;
                            for (; c < G && p.units * c / G < t1u; ++c) {
                                const long long cu0 = p.units * c / G, cu1 = p.units * (c + 1) / G;
                                if (cu1 <= cu0) continue;
                                const int sslot = (cu0 >= t0u) ? 0 : 1;
                                t += __ldcg(g.slots + (((int64_t)c * 2 + sslot) * g.B + b) * kTcRows + m);
                            }
                        }
                        {
                            // (o - |S_0|) * sum_c x_q: the binary offset (o = 1) and the
                            // complemented sign layer (file header)
                            unsigned long long sx = 0;
                            for (int pp = 0; pp < g.nsplit; ++pp)
                                sx += (unsigned long long)g.xsum[(int64_t)b * kMaxSplit + pp];
                            t += ((unsigned long long)g.offset - layer_mag(g.L, g.offset, 0)) * sx;
                        }
                        const long long accv = (long long)t;
                        const int64_t o = (int64_t)b * g.R + row;
                        if (g.acc) g.acc[o] = accv;
                        float yv = dequant(accv, g.scale, g.f[b]);
                        if (g.bias) yv += g.bias[row];
                        if (g.accumulate) yv += g.y[o];
                        g.y[o] = apply_fn(yv, g.fn);
                    }
                }
            }
            u = sg.next;
        }
    }

    if (p.prof && blockIdx.x == 0 && lane == 0)
        printf("warp %d total %lld  w_empty %lld b_full %lld a_full %lld w_full %lld a_empty %lld\n", warp,
               clock64() - t_start, prof[0], prof[1], prof[2], prof[3], prof[4]);
    if (p.dbg == 6 && warp == 1 && lane == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        printf("cta %d sm %u units %lld cycles %lld end_ns %lld start_ns %lld\n", blockIdx.x, smid, u1 - u0,
               clock64() - t_start, gt, g_start);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

cudaError_t make_weight_map(const GemmArgs& g, CUtensorMap* map)
{
    static EncodeTiledFn encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
        encode = reinterpret_cast<EncodeTiledFn>(fn);
    }
    // bits[L][R][kwords] uint32 as a 3-D tensor {kwords, R, L}; box {32 words, 128 rows, 1}.
    // Out-of-range rows / words (tile tails) are filled with zeros by the TMA unit.
    const cuuint64_t dims[3] = {(cuuint64_t)g.kwords, (cuuint64_t)g.R, (cuuint64_t)g.L};
    const cuuint64_t strides[2] = {(cuuint64_t)g.kwords * 4, (cuuint64_t)g.kwords * 4 * (cuuint64_t)g.R};
    const cuuint32_t box[3] = {kChunkWords, kTcRows, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<uint32_t*>(g.bits), dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

int ceil_log2_i(int64_t v) {
    int k = 0;
    while (((int64_t)1 << k) < v) ++k;
    return k;
}

// The plan for a shape, or false when the tensor engine does not cover it.
bool make_plan(const GemmArgs& g, int npad, TcPlan& p)
{
    if (npad <= 0 || g.kwords <= 0 || g.R <= 0 || g.B <= 0 || g.L > 16) return false;
    p.tiles = (int)((g.R + kTcRows - 1) / kTcRows);
    if (p.tiles > kMaxTiles) return false;
    p.chunks = (int)((g.kwords + kChunkWords - 1) / kChunkWords);
    p.units = (long long)p.tiles * p.chunks;
    // exact f32 accumulation: a group of G layers sums to < K * 2^G <= 2^24
    int G = 24 - ceil_log2_i(g.kwords * 32);
    if (G > 15) G = 15;                           // SFB exponents 0..13 fit the 64-column SF area
    p.Gp = G / 2;
    if (p.Gp < 1) return false;
    p.passes = (g.k_used + 1) / 2;
    p.regions = (p.passes + p.Gp - 1) / p.Gp;
    if (p.regions > kMaxRegions) return false;
    p.d_col = 512 - (p.regions * npad + 31) / 32 * 32;
    p.sf_col = p.d_col - 64;
    p.slots = p.sf_col / 128;
    if (p.slots > kMaxSlots) p.slots = kMaxSlots;
    if (p.slots < 2) return false;
    return true;
}

template <int NPAD>
cudaError_t launch_t(const GemmArgs& g, cudaStream_t s)
{
    static int sms = 0;
    static bool attr = false;
    static int dbg = -1, prof = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const char* ev = getenv("PB_TC_DEBUG");
        dbg = ev ? atoi(ev) : 0;
        ev = getenv("PB_TC_PROF");
        prof = ev ? atoi(ev) : 0;
    }
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(bitgemm_tc_kernel<NPAD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)kSmemBytes);
        if (e != cudaSuccess) return e;
        cudaFuncSetAttribute(bitgemm_tc_kernel<NPAD>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             (int)cudaSharedmemCarveoutMaxShared);
        attr = true;
    }
    TcPlan p;
    if (!make_plan(g, NPAD, p)) return cudaErrorNotSupported;
    CUtensorMap map;
    cudaError_t e = make_weight_map(g, &map);
    if (e != cudaSuccess) return e;
    p.dbg = dbg;
    p.prof = prof;
    long long grid = p.units < sms ? p.units : sms;
    if (grid > kMaxCtas) grid = kMaxCtas;

    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = la;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, bitgemm_tc_kernel<NPAD>, g, p, map);
}

}  // namespace

bool tc_supported(const GemmArgs& g)
{
    TcPlan p;
    return make_plan(g, g.npad, p);
}

cudaError_t launch_gemm_tc(const GemmArgs& g, cudaStream_t s)
{
    switch (g.npad) {
        case 8: return launch_t<8>(g, s);
        case 16: return launch_t<16>(g, s);
        case 32: return launch_t<32>(g, s);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace pb
