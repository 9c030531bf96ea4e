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
// Building A from the paired storage (include/pb.h): each 2-bit field of a
// stored pair word is already the e2m1 code 1.0*upper + 0.5*lower, so a register
// of 8 nibbles is one mask (+ shift) of a stored word (build_a below), stored
// with tcgen05.st.32x32b (lane = row).
//
// Why this shape (measured on B200, scripts/tc_mb.cu): an M=128
// tcgen05 MMA costs ~55 cycles for any N <= 64 (an M=256 CTA-pair MMA costs the
// same on two SMs), so weight bits per MMA set the rate: kind::i8 with byte
// operands carries 32 bits per row, kind::mxf4 nibbles with one layer carry
// 64, two stacked layers 128.  The issuing warp blocks on each MMA, so an A
// slot holds a whole pass (16 MMAs) per handshake, and the two converter
// h-sets take alternate passes.
//
// Work decomposition (TcPlan): units = (128-row tile, 1024-column K-chunk, all
// k_used layers).  Default static schedule: CTA i of G = min(U, #SMs) owns units
// [iU/G, (i+1)U/G); a segment (the CTA's units within one tile) that is a whole
// tile is finalised from the CTA's own sums, a tile shared with a neighbouring
// CTA is summed exactly with red.add.u64 and finalised by the contributor that
// completes its chunk count (atom.acq_rel), which also re-zeroes the sums and
// the counter, so the workspace is left as it was found.  PB_TC_STATIC=0 selects
// dynamic claims with an end-of-work grid barrier instead.  Local mode (LOCAL = true, its own
// instantiation): with at most one unit per SM every CTA builds its only B chunk itself, so the
// grid-wide B slices and their barrier are skipped, the sign correction uses the chunk's own
// sum of x_q, and with 2-4 K-chunks the tile's chunks form a cluster that sums over DSMEM.
//
// Warp roles (15 warps, 480 threads, one CTA per SM):
//   warp 0       schedule + weight producer: TMA (cp.async.bulk.tensor.3d, 128B
//                swizzle) of 128-row x 32-word tiles of the pair rows into a
//                12-13-stage SMEM ring, from kernel start (before the PDL wait);
//   warp 1       TMEM allocator and MMA issuer (one elected lane);
//   warp 2       B producer: 1-D bulk copies of the plane tiles; the fused path's
//                grid barrier that publishes the B slices;
//   warps 3..10  converters (2 h-sets of 4): thread = weight row; read the pass's
//                tiles from the swizzled ring, build A, tcgen05.st into the TMEM
//                A ring (a slot is published while the next pass's tiles arrive);
//   warps 11..14 fused prologue (a1-a2: max|x|, f_b, the B slice, the first
//                chunk) and the epilogue (TMEM drain, Horner plane sums, exact
//                int64 tile sums, dequant / bias / fn / LSTM cell / peer stores).
#include <cuda.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <mutex>

#include "pb_common.cuh"
#include "pb_internal.h"
#include "pb_tc_device.cuh"

namespace pb {
namespace {

constexpr int kConvWarps = 8;                 // 2 h-sets of 4 warps (one per TMEM lane quarter)
constexpr int kConv0 = 3;                     // first converter warp
constexpr int kEpi0 = kConv0 + kConvWarps;    // first epilogue warp (4: one per TMEM lane quarter)
constexpr int kEpiWarps = 4;
constexpr int kThreads = 32 * (kEpi0 + kEpiWarps);
constexpr int kQDepth = 16;                   // work-item queue (warp 0 -> every other role)
constexpr int kMaxSlots = 4;                  // A ring: up to 4 slots x 128 TMEM columns (16 MMAs each)
constexpr int kMaxRegions = 4;                // TMEM accumulators: sign layer + magnitude groups
constexpr int kMaxBStages = 4;                // B (plane tile) ring: 2, or 4 when a unit is short
#ifndef PB_MAX_WSTAGES
#define PB_MAX_WSTAGES 16
#endif
#ifndef PB_TIMELINE
#define PB_TIMELINE 0
#endif
constexpr bool kTimeline = PB_TIMELINE;        // per-CTA timeline / wait profiling (pb_debug_timeline)
#define TLP(g) (kTimeline ? (g).tl : nullptr)
constexpr int kMaxWStages = PB_MAX_WSTAGES;   // weight tile ring (stages sized per launch from free SMEM)
constexpr uint32_t kHdrBytes = 4096;                          // struct Bars
// dynamic SMEM: [align slack][Bars][W ring: wstages x 16 KiB][B: 2 stages][s_tot: B x 128 int64]

struct Bars {
    uint64_t a_full[kMaxSlots], a_empty[kMaxSlots];   // a_full: the 4 warps of one h-set
    uint64_t w_full[kMaxWStages], w_empty[kMaxWStages];
    uint64_t b_full[kMaxBStages], b_empty[kMaxBStages];
    uint64_t d_full[2], d_empty[2];           // double-buffered accumulators (segment parity)
    uint64_t q_full[kQDepth], q_empty[kQDepth];
    int2 q[kQDepth];                          // work items: units [x, y); x < 0 = no more work
    uint64_t x_ready;                        // fused path: bars.xsum written (warp 2)
    int fin_tile;                            // static schedule: shared tile this CTA completed (-1: none)
    uint64_t slice_done;                     // fused path: this CTA's slice of B written (epilogue warps)
    uint64_t pro_done;                       // fused path: first chunk's B built (converters resume)
    uint64_t red_full;                       // local cluster mode (leader): the partners' sums arrived
    unsigned long long gbase;                // fused path: prologue grid-barrier counter base (grid_base)
    uint32_t tmem_base;
    int last_flag;
    long long t_b, t_mma0, t_mend, t_cend;   // diagnostics timeline (globaltimer ns)
    long long t_eseg[3], t_ebar[2];          // tail: last segment wake/drained/added; end barrier arrive/exit
    long long t_c0, t_cv[4];                 // first chunk built; converter warp 3's first pass
    long long t_c0s[2];                      // first chunk: x loads issued, f_b available
    // fused activation prologue
    float red[kEpiWarps * kTcMaxB];          // per-warp partial max|x[b,:]| (prologue warps)
    int f[kTcMaxB];                          // f_b
    double fsc[kTcMaxB];                     // s_w 2^-f_b (dequant scale of column b)
    unsigned long long xs[kTcMaxB];          // this CTA's sum of x_q[b, slice]
    unsigned long long xsum[kTcMaxB];        // sum_c x_q[b, c] over all CTAs
    // split path (planes by the activation kernel): f_b and sum_c x_q of the current segment's
    // batch columns, staged once per segment, double-buffered by segment parity
    double ssc[2][kTcMaxB];                  // s_w 2^-f_b
    unsigned long long sxs[2][kTcMaxB];
};
static_assert(sizeof(Bars) <= kHdrBytes, "Bars must fit the SMEM header");

// Profiling (PB_TC_DEBUG=5): accumulate cycles spent in each wait site.
#define TWAIT(bar, ph, slotid)                                   \
    do {                                                         \
        if (kTimeline && p.prof) {                               \
            const long long _t0 = gtimer();                      \
            mbar_wait(bar, ph);                                  \
            prof[slotid] += gtimer() - _t0;                      \
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
    int slices;       // batch slices of g.bs columns (wide mode; 1 otherwise): unit u covers global
                      // tile gt = u / chunks = slice * tiles + row tile, K-chunk u % chunks
    int chunks;       // 32-word K-chunks per tile
    long long units;  // tiles * chunks
    int slots, sf_col, d_col;
    int wstages;      // weight tile ring depth
    int bstages;      // B (plane tile) ring depth: a B copy is an L2 round trip, hidden only
                      // when the stages cover it (units of 1-2 passes take ~0.5-1 us of MMAs)
    int passes;       // ceil(k_used / 2): layer pairs (0,1), (2,3), ...
    int Gp;           // passes per accumulator group (<= G/2 layers pairs, K * 2^G <= 2^24)
    int dsingle;      // narrow with one accumulator set (as wide mode): see make_plan
    int regions;      // ceil(passes / Gp)
    int Gu;           // units per work item (dynamic claims)
    int gs;           // static schedule: grid size; ustat: units split statically (the rest is
    long long ustat;  // claimed dynamically, Gu per claim, to even out the CTAs' finishing times)
    int stat;         // static schedule: CTA i owns units [i*U/G, (i+1)*U/G) (one item each, no
                      // claims); a segment covering a whole tile is finalised from its own sums, a
                      // tile split between CTAs is summed exactly (red.add) and finalised by the
                      // contributor that completes its chunk count -- no end-of-work barrier
    long long items;  // ceil(units / Gu)
    int dbg;          // profiling knob (env PB_TC_DEBUG, or PB_TC_KNOB with the timeline on): 1 = no A
                      // store, 2 = no MMA, 3 = neither, 4 = skeleton (converters skip LDS/ALU too),
                      // 6 = per-CTA timeline; bits 64 = converters never hold for the prologue,
                      // 128 = no local mode, 256 = publish each A pass at once (no deferral)
    int prof;         // env PB_TC_PROF: print wait-cycle totals of CTA 0
    int local;        // fused path, one unit per CTA: its only B chunk is built in place, so no
                      // grid-wide B slices, no grid barrier; the sign correction uses the chunk's
                      // own sum of x_q (the correction is linear in the chunks)
    int clu;          // local mode, 2..8 K-chunks: a tile's chunks are one thread-block cluster; the
                      // partners st.async their exact sums into the leader's SMEM (rank 0)
};

// Units [u0, u1) of work item `item`: the static schedule splits the units evenly over
// the grid (one item per CTA); the dynamic one hands out Gu units per claim.
__device__ __forceinline__ void item_units(const TcPlan& p, long long item, long long& u0, long long& u1) {
    if (p.stat && item < p.gs) {
        u0 = item * p.ustat / p.gs;
        u1 = (item + 1) * p.ustat / p.gs;
    } else if (p.stat) {                     // the dynamic tail: Gu units per claim
        u0 = p.ustat + (item - p.gs) * p.Gu;
        u1 = u0 + p.Gu;
        if (u1 > p.units) u1 = p.units;
    } else {
        u0 = item * p.Gu;
        u1 = u0 + p.Gu;
        if (u1 > p.units) u1 = p.units;
    }
}
// Wide mode: the shared-tile sum slot of global tile gt (static schedule).  Every CTA
// boundary floor(jU/G) that falls strictly inside the tile's units makes it shared; all
// contributors name it by the first such boundary j = ceil((gt*chunks + 1) G / U), so the
// sums need G + 1 slots instead of one per tile.
__device__ __forceinline__ int shared_slot(const TcPlan& p, long long gt) {
    const long long t1 = gt * p.chunks + 1;
    return (int)((t1 * p.gs + p.ustat - 1) / p.ustat);
}
// K-chunk of the CTA's first (static) unit.
__device__ __forceinline__ int first_kc(const TcPlan& p) {
    long long u0, u1;
    item_units(p, blockIdx.x, u0, u1);
    return (int)(u0 % p.chunks);
}
__device__ __forceinline__ void pass_region(const TcPlan& p, int k_used, int ps, int& region, int& s, bool& first) {
    pass_region_g(p.Gp, p.passes, k_used, ps, region, s, first);
}
// Fused steps a1-a2 (same arithmetic as pb_act.cu), run at
// kernel start by the 4 epilogue warps (128 threads, bar 5; idle until their first
// segment) while warp 0 streams weight tiles and the converters already build A
// from them (A does not depend on x):
//   1. one load wave: max|x[b,:]| over all of x (every CTA re-reads the
//      L2-resident B*K floats), plus the values of the CTA's first chunk and of
//      its slice of the grid-wide B operand;
//   2. f_b (reading G8);
//   3. the CTA's 1/G slice of the (b, word) items of B into the workspace tiles
//      + its sum of x_q, published by warp 2's grid barrier (which then runs
//      while step 4 does);
//   4. the CTA's first chunk kc0 of B, built straight into B stage 0, so the
//      first MMAs wait neither for the grid barrier nor a copy.
template <int NPAD, bool LOCAL>
__device__ __forceinline__ void fused_prologue(const GemmArgs& g, const TcPlan& p, Bars& bars, int pt,
                                               uint8_t* bstage0, int kc0) {
    constexpr int kPW = kEpiWarps;                     // 4 warps
    constexpr int kPT = 32 * kPW;
    constexpr int kCx = 8;                             // first-chunk values prefetched per thread
    const int pw = pt >> 5, lane = pt & 31;
    const int nd = act_digits(g.a);                    // digit rows per batch column
    long long tpw = 0, tmax = 0, tc0 = 0, ttr = 0, tfb = 0, tcg = 0, cyc_ballot = 0, cyc_put = 0;
    pdl_wait();                                        // x may be the previous kernel's output
    if TLP(g) tpw = gtimer();
    const int B = (int)g.B;
    if (pt == 0) bars.gbase = grid_base(g.gbar);
    // first-chunk items it = b * 32 + local word; warp pw takes pw, pw + 4, ...
    const int nci = B * kChunkWords;
    auto chunk_x = [&](int it) -> float {
        const int b = it / kChunkWords;
        const int64_t c = 32 * ((int64_t)kc0 * kChunkWords + (it - b * kChunkWords)) + lane;
        return (it < nci && c < g.K) ? __ldg(g.x + (int64_t)b * g.K + c) : 0.f;
    };
    float cx[kCx];
#pragma unroll
    for (int k = 0; k < kCx; ++k) cx[k] = chunk_x(pw + kPW * k);
    // slice items: words up to the last chunk's end (zero B for the K tail, where the
    // complemented sign layer is 1)
    // (32-bit index math: N = B * Wt < 2^31 is checked by make_plan)
    const uint32_t Wt = (uint32_t)p.chunks * kChunkWords, N = (uint32_t)B * Wt;
    const uint32_t G = gridDim.x;
    const uint32_t nq = N / G, nr = N - nq * G;        // floor(N * c / G) without 64-bit division
    const uint32_t i0 = nq * blockIdx.x + nr * blockIdx.x / G, i1 = nq * (blockIdx.x + 1) + nr * (blockIdx.x + 1) / G;
    auto item_x = [&](uint32_t it) -> float {
        const uint32_t b = it / Wt;
        const uint32_t c = 32 * (it - b * Wt) + lane;
        return c < (uint32_t)g.K ? __ldg(g.x + (int64_t)b * g.K + c) : 0.f;
    };
    const int ew = pw;
    const float xv0 = (i0 + ew < i1) ? item_x(i0 + ew) : 0.f;
    const float xv1 = (i0 + ew + kEpiWarps < i1) ? item_x(i0 + ew + kEpiWarps) : 0.f;
    // ---- a1 (part 1): max|x[b,:]|
    // (a literal act_frac -- Alg. 2's fixed 2^16 cast, P:195 -- needs no max)
    const bool vec = (g.K & 3) == 0 && (reinterpret_cast<uintptr_t>(g.x) & 15) == 0;
    for (int b = 0; b < (g.act_frac == kActAutoFrac ? B : 0); ++b) {
        const float* xb = g.x + (int64_t)b * g.K;
        float m = 0.f;
        if (vec) {
            const float4* x4 = reinterpret_cast<const float4*>(xb);
            const int64_t n4 = g.K / 4;
            for (int64_t c0 = pt; c0 < n4; c0 += 16 * kPT) {    // 16 loads in flight per thread
                float4 v[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const int64_t c = c0 + (int64_t)u * kPT;
                    v[u] = c < n4 ? __ldg(x4 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < 16; ++u)
                    m = fmaxf(m, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
            }
        } else {
#pragma unroll 1
            for (int64_t c = pt; c < g.K; c += kPT) m = fmaxf(m, fabsf(__ldg(xb + c)));
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) bars.red[pw * kTcMaxB + b] = m;
    }
    asm volatile("bar.sync 5, 128;" ::: "memory");
    if TLP(g) tmax = gtimer();
    if (pt < B) {
        float m = bars.red[pt];
#pragma unroll
        for (int w = 1; w < kPW; ++w) m = fmaxf(m, bars.red[w * kTcMaxB + pt]);
        bars.f[pt] = (g.act_frac == kActAutoFrac) ? act_frac_of(m, g.a) : g.act_frac;
        bars.fsc[pt] = col_scale(g.scale, bars.f[pt]);
        bars.xs[pt] = 0;
    }
    asm volatile("bar.sync 5, 128;" ::: "memory");
    if TLP(g) tfb = gtimer();
    // even a <= 16: digits by a per-lane nibble transpose (digit_regs_shfl, pb_common.cuh) and
    // 32-bit stores; otherwise one ballot per plane (digit_of_lane)
    const bool shfl = !(g.a & 1) && g.a <= 16;
    const uint32_t amask = g.a >= 32 ? ~0u : ((1u << g.a) - 1u);
    // ---- the CTA's slice of the grid-wide B operand first: warp 2's grid barrier that
    // publishes the slices for the later chunks then overlaps the first chunk's build
    int k = 0;
#pragma unroll 1
    for (uint32_t it = i0 + ew; it < ((LOCAL && p.local) ? i0 : i1); it += kEpiWarps, ++k) {
        const uint32_t b = it / Wt;
        const uint32_t w = it - b * Wt;
        const float v = k == 0 ? xv0 : (k == 1 ? xv1 : item_x(it));
        const long long q = act_cast(v, bars.f[b], g.a);
        if (shfl) {
            int dk;
            const uint32_t reg = digit_regs_shfl((uint32_t)q & amask, g.a, lane, dk);
            if (dk < nd)
                *reinterpret_cast<uint32_t*>(g.bexp + b_operand_offset(NPAD, w, b * nd + dk, lane & 3)) = reg;
        } else {
            uint32_t mine = 0;
            for (int j = 0; j < g.a; ++j) {
                const uint32_t wj = __ballot_sync(0xffffffffu, ((uint32_t)q >> (g.a - 1 - j)) & 1u);
                if (lane == j) mine = wj;
            }
            uint4 dv;
            if (digit_of_lane(mine, lane, g.a, dv)) put_b_operand(g.bexp, NPAD, w, b * nd + (lane >> 1), dv);
        }
        if (b == B - 1)
            for (int n = B * nd + lane; n < NPAD; n += 32) put_b_operand(g.bexp, NPAD, w, n, make_uint4(0, 0, 0, 0));
        long long xs = q;
#pragma unroll
        for (int o = 16; o; o >>= 1) xs += __shfl_xor_sync(0xffffffffu, xs, o);
        if (lane == 0) atomicAdd(&bars.xs[b], (unsigned long long)xs);
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    const int et = pt;
    if (et < B) {
        g.xsum[(int64_t)et * kXsumStride + blockIdx.x] = (long long)bars.xs[et];
        if (blockIdx.x == 0) g.f[et] = bars.f[et];
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if TLP(g) ttr = gtimer();
    // warp 2 arrives at the grid barrier for this CTA once its slice is written
    if (et == 0) mbar_arrive(&bars.slice_done);
    // ---- a1 (part 2) + a2 for the first chunk: cast and transpose kCx words per warp at a time
    // (the words itb + kPW k of batch column itb / 32: no branches inside a group), e2m1 B rows
    // straight into B stage 0
    const uint32_t bstage0_s = smem_u32(bstage0);
    auto chunk_group = [&](int itb, const float (&v)[kCx]) {
        const int b = itb / kChunkWords;              // kPW * kCx == kChunkWords: one column
        const int f = bars.f[b];
        uint32_t u[kCx];
        if (g.a <= 24 && f >= -126 && f <= 127) {
            // act_cast's exact fp32 form (pb_common.cuh)
            const float sc = __int_as_float((127 + f) << 23), lim = (float)(1 << (g.a - 1));
#pragma unroll
            for (int k = 0; k < kCx; ++k) u[k] = (uint32_t)__float2int_rz(fminf(fmaxf(v[k] * sc, -lim), lim - 1.0f));
        } else {
#pragma unroll   // (indexed registers: no local-memory array)
            for (int k = 0; k < kCx; ++k) u[k] = (uint32_t)act_cast(v[k], f, g.a);
        }
        if ((LOCAL && p.local)) {
            // the chunk's sum of x_q for column b (codes fit 32 bits: a <= 32)
            long long xs = 0;
#pragma unroll
            for (int k = 0; k < kCx; ++k) xs += (int32_t)u[k];
#pragma unroll
            for (int o = 16; o; o >>= 1) xs += __shfl_xor_sync(0xffffffffu, xs, o);
            if (lane == 0) atomicAdd(&bars.xs[b], (unsigned long long)xs);
        }
        const long long c1 = kTimeline ? clock64() : 0;
        if (shfl) {
            uint32_t reg[kCx];
            int dk = 0;
#pragma unroll
            for (int k = 0; k < kCx; ++k) reg[k] = digit_regs_shfl(u[k] & amask, g.a, lane, dk);
            if (dk < nd) {
#pragma unroll
                for (int k = 0; k < kCx; ++k)
                    asm volatile("st.shared.u32 [%0], %1;" ::"r"(bstage0_s + b_operand_offset(NPAD, itb - b * kChunkWords + kPW * k, b * nd + dk, lane & 3)),
                                 "r"(reg[k]) : "memory");
            }
        } else {
            uint32_t mm[kCx];
#pragma unroll
            for (int k = 0; k < kCx; ++k) mm[k] = 0;
#pragma unroll 1
            for (int j = 0; j < g.a; ++j) {
                const uint32_t bit = 1u << (g.a - 1 - j);
#pragma unroll
                for (int k = 0; k < kCx; ++k) {
                    const uint32_t w = __ballot_sync(0xffffffffu, (u[k] & bit) != 0);
                    if (lane == j) mm[k] = w;
                }
            }
#pragma unroll
            for (int k = 0; k < kCx; ++k) {
                uint4 dv;
                if (digit_of_lane(mm[k], lane, g.a, dv))
                    put_b_operand_smem(bstage0_s, NPAD, itb - b * kChunkWords + kPW * k, b * nd + (lane >> 1), dv);
            }
        }
        const long long c2 = kTimeline ? clock64() : 0;
        if (b == B - 1 && B * nd < NPAD) {
#pragma unroll 1
            for (int k = 0; k < kCx; ++k)
                for (int n = B * nd + lane; n < NPAD; n += 32)
                    put_b_operand_smem(bstage0_s, NPAD, itb - b * kChunkWords + kPW * k, n, make_uint4(0, 0, 0, 0));
        }
        if (kTimeline) {
            cyc_ballot += c2 - c1;
            cyc_put += clock64() - c2;
        }
    };
    static_assert(kPW * kCx == kChunkWords, "a chunk group covers one batch column");
    chunk_group(pw, cx);
#pragma unroll 1
    for (int itb = pw + kPW * kCx; itb < nci; itb += kPW * kCx) {
        float v[kCx];
#pragma unroll
        for (int k = 0; k < kCx; ++k) v[k] = chunk_x(itb + kPW * k);
        chunk_group(itb, v);
    }
    if TLP(g) tcg = gtimer();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic SMEM writes -> MMA operand reads
    asm volatile("bar.sync 5, 128;" ::: "memory");
    if (pt == 0) {
        mbar_arrive(&bars.b_full[0]);
        mbar_arrive(&bars.pro_done);
    }
    if ((LOCAL && p.local)) {
        // the chunk sums (bar 5 above ordered the atomics) are the epilogue's x_q sums
        if (pt < B) bars.xsum[pt] = bars.xs[pt];
        asm volatile("bar.sync 5, 128;" ::: "memory");
        if (pt == 0) mbar_arrive(&bars.x_ready);
    }
    if TLP(g) tc0 = gtimer();
    if (TLP(g) && et == 0) {
        long long* r = tl_record(TLP(g));
        if (r) {
            const long long rec[10] = {2, blockIdx.x, cyc_ballot, cyc_put, tpw, tmax, tc0, ttr, tfb, tcg};
            for (int q = 0; q < 10; ++q) r[q] = rec[q];
        }
    }
}

#ifndef PB_NARROW_KA
#define PB_NARROW_KA 1
#endif
// The converters' A build: the wide kernel waits each TMEM store; the batch-1 kernels alternate
// two register sets (convert_pass_ka) so no store's source registers are rewritten early.
template <int NPAD, int KIND>
__device__ __forceinline__ void convert_pass_gemm(uint32_t t0, uint32_t t1, uint32_t swz, uint32_t dst, uint32_t xm,
                                                  int dbg, uint64_t* r0, uint64_t* r1, int lane) {
    if constexpr (NPAD > kTcMaxN || !PB_NARROW_KA)
        convert_pass<KIND, false, (NPAD > kTcMaxN)>(t0, t1, swz, dst, xm, 0, dbg, r0, r1, lane);
    else
        convert_pass_ka<KIND>(t0, t1, swz, dst, xm, dbg, r0, r1, lane);
}

// Reads work item `it` from the queue slot (qi, qph) and releases the slot (each
// consuming warp arrives once).  Warp-uniform.
__device__ __forceinline__ int2 take_item(Bars& bars, int& qi, uint32_t& qph, int lane) {
    mbar_wait(&bars.q_full[qi], qph);
    const volatile int* vq = reinterpret_cast<volatile int*>(&bars.q[qi]);
    const int2 it = make_int2(vq[0], vq[1]);
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars.q_empty[qi]);
    if (++qi == kQDepth) {
        qi = 0;
        qph ^= 1;
    }
    return it;
}

template <int NPAD, bool LOCAL>
__global__ void __launch_bounds__(kThreads, 1)
bitgemm_tc_kernel(const GemmArgs g, const TcPlan p, const __grid_constant__ CUtensorMap pmap,
                  const __grid_constant__ CUtensorMap smap)
{
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment for the 128B-swizzled TMA tiles
    // 1024-byte aligned as an offset into smem_raw (not through an integer cast), so the compiler
    // keeps the shared window: every access through `bars` is LDS/STS, not a generic LD/ST
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    Bars& bars = *reinterpret_cast<Bars*>(smem);
    constexpr uint32_t kBTile = NPAD * 32;                    // one MMA's B (64 columns)
    constexpr uint32_t kBStage = (kChunkWords / 2) * kBTile;  // one K-chunk (16 MMAs)
    constexpr int kQConsumers = 2 + kConvWarps + kEpiWarps;   // warps 1, 2, converters, epilogue
    constexpr bool kWide = NPAD > kTcMaxN;                     // wide mode (split path, static schedule)
    uint8_t* wtile0 = smem + kHdrBytes;
    uint8_t* btile0 = wtile0 + p.wstages * kWTileBytes;
    const uint32_t s_tot_s = smem_u32(btile0 + p.bstages * kBStage);   // [b][128] u64 (B > 1)
    const uint32_t redbuf_s = s_tot_s + (uint32_t)g.bs * kTcRows * 8u;   // [clu-1][b][128] u64 (leader)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long G = gridDim.x;
    long long prof[5] = {0, 0, 0, 0, 0};
    const long long g_start = gtimer();
    bool cwaited = false;                      // local cluster mode: this thread waited the cluster barrier

    if (threadIdx.x == 0) {
        for (int s = 0; s < p.slots; ++s) {
            mbar_init(&bars.a_full[s], 4);               // the 4 converter warps of one h-set
            mbar_init(&bars.a_empty[s], 1);
        }
        for (int s = 0; s < p.wstages; ++s) {
            mbar_init(&bars.w_full[s], 1);
            mbar_init(&bars.w_empty[s], 4);              // the h-set that converts the tile
        }
        for (int s = 0; s < p.bstages; ++s) {
            mbar_init(&bars.b_full[s], 1);
            mbar_init(&bars.b_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bars.d_full[s], 1);
            mbar_init(&bars.d_empty[s], kEpiWarps);
        }
        for (int s = 0; s < kQDepth; ++s) {
            mbar_init(&bars.q_full[s], 1);
            mbar_init(&bars.q_empty[s], kQConsumers);
        }
        mbar_init(&bars.x_ready, 1);
        mbar_init(&bars.slice_done, 1);
        mbar_init(&bars.pro_done, 1);
        mbar_init(&bars.red_full, 1);
        if ((LOCAL ? p.clu : 0) && blockIdx.x % (LOCAL ? p.clu : 0) == 0)   // the leader expects every partner's sums
            mbar_arrive_expect_tx(&bars.red_full, (uint32_t)(((LOCAL ? p.clu : 0) - 1) * g.B * kTcRows * 8));
        fence_mbar_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(&pmap) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&smap) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            smem_u32(&bars.tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // local cluster mode: every thread arrives once (the leader's barrier inits are published);
    // the epilogue warps wait before their first DSMEM exchange, everyone else at the end
    if ((LOCAL ? p.clu : 0)) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    // warp 0 (whose thread 0 initialised the barriers) only arrives: its weight tiles start
    // streaming now, while the other warps wait for the TMEM allocation and the scale factors
    if (warp == 0) {
        __syncwarp();
        asm volatile("barrier.arrive 8, %0;" ::"n"(kThreads) : "memory");   // non-aligned (different code than bar 8 sync)
    } else {
        tc_fence_before();
        asm volatile("barrier.sync 8, %0;" ::"n"(kThreads) : "memory");
        tc_fence_after();
    }
    const uint32_t tmem = warp == 0 ? 0u : bars.tmem_base;
    if (warp >= kConv0 && warp < kConv0 + 4) {
        store_scale_factors(tmem, warp, p.sf_col);
        tmem_st_wait();
    }
    if (warp != 0) {
        tc_fence_before();
        asm volatile("bar.sync 9, %0;" ::"n"(kThreads - 32) : "memory");
        tc_fence_after();
    }
    pdl_trigger();

    int qi = 0;                 // work-item queue position (every role walks the same items)
    uint32_t qph = 0;
    if (warp == 0) {
        // ------------------------------------------------ work claims + weight tile producer.
        // Item blockIdx.x is static (its tiles stream before the PDL wait: the packed weights
        // do not depend on the previous kernel); later items are claimed from a global counter
        // once the previous call (which reset it) has completed.
        long long item = blockIdx.x;
        bool waited = false;
        int tc = 0;
        while (true) {
            mbar_wait(&bars.q_empty[qi], qph ^ 1);
            long long u0 = -1, u1 = 0;
            if (item < p.items) item_units(p, item, u0, u1);
            if (lane == 0) {
                bars.q[qi] = make_int2((int)u0, (int)u1);
                mbar_arrive(&bars.q_full[qi]);
            }
            __syncwarp();
            if (++qi == kQDepth) {
                qi = 0;
                qph ^= 1;
            }
            if (u0 < 0) break;
            for (long long u = u0; u < u1; ++u) {
                const long long gt = u / p.chunks;
                const int kc = (int)(u - gt * p.chunks), rt = (int)(gt % p.tiles);
                for (int ps = 0; ps < p.passes; ++ps) {
                    // a stored pair: two 32-word boxes of the pair row; else the canonical last layer
                    const bool stored_pair = 2 * ps + 1 < g.L;
                    for (int t = 0; t < (stored_pair ? 2 : 1); ++t, ++tc) {
                        const int st = tc % p.wstages;
                        TWAIT(&bars.w_empty[st], (uint32_t)(((tc / p.wstages) & 1) ^ 1), 0);
                        if (elect_one()) {
                            mbar_arrive_expect_tx(&bars.w_full[st], kWTileBytes);
                            if (stored_pair)
                                tma_load_3d(wtile0 + st * kWTileBytes, &pmap, kc * 2 * kChunkWords + t * kChunkWords,
                                            rt * kTcRows, ps, &bars.w_full[st]);
                            else
                                tma_load_3d(wtile0 + st * kWTileBytes, &smap, kc * kChunkWords, rt * kTcRows, 0,
                                            &bars.w_full[st]);
                        }
                        __syncwarp();
                    }
                }
            }
            if (!waited) {
                pdl_wait();
                waited = true;
            }
            long long nxt = 0;
            if (lane == 0) nxt = G + atomicAdd(&g.work[0], 1);
            item = __shfl_sync(0xffffffffu, nxt, 0);
        }
        if (!waited) pdl_wait();
        if (lane == 0) {
            // the last CTA to run out of work clears the counters for the next call
            __threadfence();
            if (atomicAdd(&g.work[1], 1) == (int)G - 1) {
                atomicExch(&g.work[0], 0);
                atomicExch(&g.work[1], 0);
            }
        }
    } else if (warp == 2) {
        // ------------------------------------------------ B (plane tile) producer
        // Fused path: the converters build the CTA's first chunk in stage 0 themselves
        // (no copy); later chunks are copied once the grid barrier has published them.
        if (!g.x) {
            pdl_wait();
            // the B tiles were written by the activation kernel (generic proxy); the bulk copies
            // below read them through the async proxy
            asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        bool published = false;
        auto wait_published = [&]() {
            if (g.x && !(LOCAL && p.local) && !published) {
                mbar_wait(&bars.slice_done, 0);                        // this CTA's slice is written
                // the CTA's slice writes are ordered before the arrival by the epilogue warps'
                // bar.sync + slice_done mbarrier and the cumulative release of the arrival
                if (lane == 0) {
                    grid_arrive(g.gbar);
                    grid_wait(g.gbar, bars.gbase);
                }
                __syncwarp();
                asm volatile("fence.proxy.async.global;" ::: "memory");   // generic writes -> bulk-copy reads
                if (TLP(g) && lane == 0) bars.t_b = gtimer();
                // sum_c x_q[b, c] from every CTA's partial, for the epilogue
#pragma unroll 1
                for (int b = 0; b < (int)g.B; ++b) {
                    unsigned long long t = 0;
                    const long long* xs = g.xsum + b * kXsumStride;
#pragma unroll 1
                    for (int c = lane; c < (int)G; c += 32) t += (unsigned long long)__ldcg(xs + c);
#pragma unroll
                    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
                    if (lane == 0) bars.xsum[b] = t;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars.x_ready);
                published = true;
            }
        };
        if (!g.x && TLP(g) && lane == 0) bars.t_b = gtimer();
        int cc = 0;
        while (true) {
            const int2 it = take_item(bars, qi, qph, lane);
            if (it.x < 0) break;
            for (int u = it.x; u < it.y; ++u, ++cc) {
                if (g.x && cc == 0) continue;                 // built in place by the converters
                wait_published();
                const int gt = u / p.chunks, kc = u - gt * p.chunks;
                const int sl = gt / p.tiles;                  // batch slice (wide mode)
                const int st = cc % p.bstages;
                mbar_wait(&bars.b_empty[st], (uint32_t)(((cc / p.bstages) & 1) ^ 1));
                if (elect_one()) {
                    mbar_arrive_expect_tx(&bars.b_full[st], kBStage);
                    bulk_g2s(btile0 + st * kBStage, g.bexp + ((int64_t)sl * p.chunks + kc) * kBStage, kBStage,
                             &bars.b_full[st]);
                }
                __syncwarp();
            }
        }
        wait_published();                                     // (a one-chunk CTA still joins bar 3)
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer: the whole warp walks the
        // schedule (warp-uniform values stay in uniform registers), one elected lane issues.
        // kind::mxf4: A, B = E2M1 (1), scale format UE8M0 (bit 23), K = 64, M = 128
        const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(NPAD >> 3) << 17) | (1u << 23) |
                               ((uint32_t)(kTcRows >> 4) << 24);
        const uint32_t sfa = tmem + p.sf_col;
        long long t_mma0 = 0;
        uint32_t slot = 0, phase = 0;
        int cc = 0, seg = 0;
        while (true) {
            const int2 it = take_item(bars, qi, qph, lane);
            if (it.x < 0) break;
            for (int u = it.x; u < it.y; ++seg) {
                // a segment: the item's units in one row tile, accumulated in D[seg & 1]
                const int gt = u / p.chunks;
                int ue = (gt + 1) * p.chunks;
                if (ue > it.y) ue = it.y;
                // narrow: D double-buffered by segment parity; wide: one D, drained per segment
                const bool d1 = kWide || p.dsingle;     // one accumulator set
                const int db = d1 ? 0 : (seg & 1);
                if (d1 ? seg >= 1 : seg >= 2)
                    TWAIT(&bars.d_empty[db], (uint32_t)((d1 ? seg - 1 : (seg >> 1) - 1) & 1), 0);
                tc_fence_after();
                const uint32_t dbase = tmem + (uint32_t)(p.d_col + db * p.regions * NPAD);
                for (const int us = u; u < ue; ++u, ++cc) {
                    const int st = cc % p.bstages;
                    TWAIT(&bars.b_full[st], (uint32_t)((cc / p.bstages) & 1), 1);
                    tc_fence_after();
                    const uint64_t bdesc0 = b_desc(smem_u32(btile0 + st * kBStage));
                    for (int ps = 0; ps < p.passes; ++ps) {
                        int region, sexp;
                        bool first;
                        pass_region(p, g.k_used, ps, region, sexp, first);
                        const uint32_t dcol = dbase + (uint32_t)(region * NPAD);
                        const uint32_t sfb = tmem + (uint32_t)(p.sf_col + 4 * (1 + sexp));
                        const bool open = first && u == us;
                        TWAIT(&bars.a_full[slot], phase, 2);
                        tc_fence_after();
                        if (TLP(g) && t_mma0 == 0) t_mma0 = gtimer();
                        if (p.dbg == 2 || p.dbg == 3 || p.dbg == 4) {
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
                if (elect_one()) tc_commit(&bars.d_full[db]);
                __syncwarp();
            }
        }
        if (TLP(g) && lane == 0) {
            bars.t_mma0 = t_mma0;
            bars.t_mend = gtimer();
        }
    } else if (warp < kEpi0) {
        // ------------------------------------------------ converters
        const int cw = warp - kConv0;
        const int h = cw >> 2;                 // h-set: 0 = warps 3..6, 1 = warps 7..10
        const int q = warp & 3;                // TMEM lane quarter this warp may access
        const int m = q * 32 + lane;           // row within the tile
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const uint32_t wtile_s = smem_u32(wtile0) + (uint32_t)m * 128;
        const uint32_t swz = (uint32_t)(m & 7);
        int tc = 0, pc = 0;
        // passes in issue order; h-set h converts passes pc = h, h + 2, ...; pass pc uses A slot
        // pc % slots; its tiles are tc and tc + 1 (a stored pair) or tc alone
        int slot = h % p.slots, sphase = (h / p.slots) & 1;
        // software pipeline: a pass's TMEM stores drain while the next pass's tiles are awaited
        int pend_slot = -1;
        int npub = 0;
        bool hold = g.x != nullptr && !(p.dbg & 64), converted = false;
        auto publish = [&]() {
            if (pend_slot >= 0) {
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars.a_full[pend_slot]);
                pend_slot = -1;
                if (TLP(g) && warp == kConv0 && lane == 0 && npub++ == 0) bars.t_cv[3] = gtimer();
            }
        };
        while (true) {
            const int2 it = take_item(bars, qi, qph, lane);
            if (it.x < 0) break;
            for (int u = it.x; u < it.y; ++u) {
                for (int ps = 0; ps < p.passes; ++ps, ++pc) {
                    const bool stored_pair = 2 * ps + 1 < g.L;
                    const bool use_lo = 2 * ps + 1 < g.k_used;
                    const int ntile = stored_pair ? 2 : 1;
                    if ((pc & 1) != h) {
                        tc += ntile;
                        continue;
                    }
                    const int st0 = tc % p.wstages, st1 = (tc + ntile - 1) % p.wstages;
                    if (TLP(g) && warp == kConv0 && lane == 0 && pc == 0) bars.t_cv[0] = gtimer();
                    TWAIT(&bars.w_full[st0], (uint32_t)((tc / p.wstages) & 1), 3);
                    if (stored_pair) TWAIT(&bars.w_full[st1], (uint32_t)(((tc + 1) / p.wstages) & 1), 3);
                    if (TLP(g) && warp == kConv0 && lane == 0 && pc == 0) bars.t_cv[1] = gtimer();
                    publish();                          // previous pass's A is in TMEM: tell the MMA
                    if (hold && pend_slot < 0 && converted) {   // this h-set's first pass is published
                        // fused path: after its first pass an h-set waits for the prologue (the
                        // epilogue warps' x wave and first B chunk), which it would otherwise
                        // slow down by competing for issue slots; the MMAs need both anyway
                        mbar_wait(&bars.pro_done, 0);
                        hold = false;
                    }
                    TWAIT(&bars.a_empty[slot], (uint32_t)(sphase ^ 1), 4);
                    tc_fence_after();
                    const int kind = stored_pair ? (use_lo ? 0 : 1) : 2;
                    // the sign layer's pass: complemented (folded into the mask op at no cost; the
                    // epilogue adds (o - |S_0|) sum_c x_q)
                    const uint32_t xm = ps == 0 ? (stored_pair ? 0xAAAAAAAAu : 0xFFFFFFFFu) : 0u;
                    const uint32_t t0 = wtile_s + (uint32_t)st0 * kWTileBytes;
                    const uint32_t t1 = wtile_s + (uint32_t)st1 * kWTileBytes;
                    const uint32_t dst = tmem + lane_off + (uint32_t)(slot * 128);
                    uint64_t* r0 = &bars.w_empty[st0];
                    uint64_t* r1 = &bars.w_empty[st1];
                    if (kind == 0)
                        convert_pass_gemm<NPAD, 0>(t0, t1, swz, dst, xm, p.dbg, r0, r1, lane);
                    else if (kind == 1)
                        convert_pass_gemm<NPAD, 1>(t0, t1, swz, dst, xm, p.dbg, r0, r1, lane);
                    else
                        convert_pass_gemm<NPAD, 2>(t0, t1, swz, dst, xm, p.dbg, r0, r1, lane);
                    if (TLP(g) && warp == kConv0 && lane == 0 && pc == 0) bars.t_cv[2] = gtimer();
                    tc += ntile;
                    converted = true;
                    pend_slot = slot;
                    if (p.dbg & 256) publish();           // experiment knob: no deferred publish
                    slot += 2;
                    while (slot >= p.slots) {
                        slot -= p.slots;
                        sphase ^= 1;
                    }
                }
            }
        }
        publish();
    } else {
        // ------------------------------------------------ epilogue: per segment, fold D into
        // exact int64 per-row sums; a whole tile writes y, a partial tile adds into the
        // tile's accumulator (integer: order-independent, exact) and the contributor that
        // completes the tile's chunk count finalises it.
        const int ew = warp - kEpi0;
        const int q = warp & 3;
        const int m = q * 32 + lane;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        // (o - |S_0|) sum_c x_q: binary offset + complemented sign layer; + the midpoint offset
        // 2^(L-k_used-1) sum_c x_q (pb_matmul_ex)
        const unsigned long long o_corr = (unsigned long long)g.offset - layer_mag(g.L, g.offset, 0, true) + g.mid;
        bool have_xsum = false;
        const int pt = threadIdx.x - kEpi0 * 32;      // 0..127
        const int nd = act_digits(g.a);               // activation digits per batch column
        int seg_b0 = 0, spar = 0;                     // current segment: first batch column, parity
        // split path: stage f_b and sum_c x_q (the activation kernel's per-CTA partials) of the
        // segment's nb columns in SMEM -- one round of loads per segment, not per row
        auto stage_cols = [&](int b0, int nb, int par) {
            if (!g.x && pt < nb) {
                const long long* xs = g.xsum + (int64_t)(b0 + pt) * kXsumStride;
                unsigned long long sx = 0;
                int pp = 0;
#pragma unroll 1
                for (; pp + 8 <= g.nsplit; pp += 8) {
                    long long v[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) v[k] = __ldcg(xs + pp + k);
#pragma unroll
                    for (int k = 0; k < 8; ++k) sx += (unsigned long long)v[k];
                }
                for (; pp < g.nsplit; ++pp) sx += (unsigned long long)__ldcg(xs + pp);
                bars.ssc[par][pt] = col_scale(g.scale, __ldcg(g.f + b0 + pt));
                bars.sxs[par][pt] = sx;
            }
        };
        auto xsum_of = [&](int b) -> unsigned long long {
            if (g.x) {
                if (!have_xsum) {
                    mbar_wait(&bars.x_ready, 0);
                    have_xsum = true;
                }
                return bars.xsum[b];
            }
            return bars.sxs[spar][b - seg_b0];
        };
        // a5: y = dequant(acc) (+ bias, + y when accumulating), then fn -- or, in cell mode
        // (pb_lstm_seq), the LSTM cell over the 4 gate rows of a hidden unit (lanes 4j..4j+3)
        auto preact = [&](int b, int64_t row, unsigned long long t) -> float {
            if (!(LOCAL && p.local)) t += o_corr * xsum_of(b);    // (o - |S_0|) sum_c x_q: binary offset + complemented sign layer
            const long long accv = (long long)t;
            const int64_t o = (int64_t)b * g.R + row;
            if (g.acc) g.acc[o] = accv;
            float yv = dequant_sc(accv, g.x ? bars.fsc[b] : bars.ssc[spar][b - seg_b0]);
            if (g.bias) yv += g.bias[row];
            if (g.accumulate) yv += g.y[o];
            return yv;
        };
        // the rest of a5 for one column given its pre-activation: fn and the y store (or the
        // peer stores), or in cell mode the LSTM cell (warp-uniform call: lane shuffles)
        auto finish_value = [&](int b, int64_t row, float pre) {
            if (!g.cell) {
                if (row < g.R) {
                    const float v = apply_fn(pre, g.fn);
                    if (g.nranks) {
                        // fused all-gather (f2): this row of y into every rank's y_full
                        const int64_t grow = g.row0 + row;
                        if (grow < g.R_total)
                            for (int q = 0; q < g.nranks; ++q) g.peer_y[q][(int64_t)b * g.R_total + grow] = v;
                    } else {
                        g.y[(int64_t)b * g.R + row] = v;
                    }
                }
                return;
            }
            const float v = pre;
            const int q0 = lane & ~3;
            const float gi = __shfl_sync(0xffffffffu, v, q0), gf = __shfl_sync(0xffffffffu, v, q0 + 1);
            const float gg = __shfl_sync(0xffffffffu, v, q0 + 2), go = __shfl_sync(0xffffffffu, v, q0 + 3);
            if ((lane & 3) == 0 && row < g.R) {
                const int64_t i = (int64_t)b * g.H + (row >> 2);
                float hn, cn;
                lstm_cell(gi, gf, gg, go, g.cell_c[i], hn, cn);
                g.cell_h[i] = hn;
                g.cell_c_out[i] = cn;
            }
        };
        auto finish_tile_row = [&](int b, int64_t row, unsigned long long t) {   // warp-uniform call
            finish_value(b, row, row < g.R ? preact(b, row, t) : 0.f);
        };
        // columns [b0, b0 + nb) of this thread's row, totals from get_t(local column): the
        // pre-activations of 8 columns at a time are independent chains (the FP64 conversion
        // and multiply have long latencies), then finished one column at a time
        // (the totals are this thread's s_tot slots [b][m]; each slot is reused for its
        // pre-activation, so the column loop needs no indexed registers)
        auto finish_cols = [&](int b0, int nb, int64_t row) {   // warp-uniform call
#pragma unroll 1
            for (int bg = 0; bg < nb; bg += 8) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t sa = s_tot_s + (uint32_t)((bg + k) * kTcRows + m) * 8u;
                    if (bg + k < nb && row < g.R)
                        asm volatile("st.shared.f32 [%0], %1;" ::"r"(sa), "f"(preact(b0 + bg + k, row, ld_shared_u64(sa)))
                                     : "memory");
                }
#pragma unroll 1
                for (int k = 0; k < 8 && bg + k < nb; ++k) {
                    float v;
                    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(s_tot_s + (uint32_t)((bg + k) * kTcRows + m) * 8u)
                                 : "memory");
                    finish_value(b0 + bg + k, row, row < g.R ? v : 0.f);
                }
            }
        };
        // a tile's exact sums from the workspace into s_tot (re-zeroing them), then finished
        auto finish_from_accbuf = [&](int b0, int nb, int64_t row, unsigned long long* ab) {
            if (!kWide && g.B == 1) {
                const unsigned long long t = __ldcg(ab);
                *ab = 0;                                          // leave the sums zero
                finish_tile_row(0, row, t);
                return;
            }
            for (int b = 0; b < nb; ++b) {
                st_shared_u64(s_tot_s + (uint32_t)(b * kTcRows + m) * 8u, __ldcg(ab + b * kTcRows));
                ab[b * kTcRows] = 0;                              // leave the sums zero
            }
            finish_cols(b0, nb, row);
        };
        if (g.x)
            fused_prologue<NPAD, LOCAL>(g, p, bars, threadIdx.x - kEpi0 * 32, btile0,
                                 first_kc(p));
        else
            pdl_wait();
        // end-of-work barrier base (after the PDL wait above: every earlier call is complete)
        const unsigned long long ebase = (ew == 0 && lane == 0) ? grid_base(g.ebar) : 0ull;
        // cross-rank barrier base (f2): every rank's previous call has completed (its kernel
        // waited for all ranks), and no rank can arrive for the next call before this one
        unsigned long long xbase = 0, rbase = 0;
        if (g.nranks && ew == 0 && lane == 0) {
            xbase = ld_acquire_sys_u64(g.local_ctr) & ~(kGridStride - 1);
            rbase = ld_acquire_sys_u64(g.local_ctr + 1) & ~(kGridStride - 1);
            // entry handshake: this rank's stream has reached the call (everything before it,
            // including readers of the previous y_full, is complete), so peers may now store
            // into this rank's y_full -- CTA 0 tells every rank (ready counter, word 1)
            if (blockIdx.x == 0)
                for (int q = 0; q < g.nranks; ++q)
                    asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(g.peer_ctr[q] + 1),
                                 "l"(kGridStride / (unsigned)g.nranks)
                                 : "memory");
        }
        if (g.nranks && p.stat) {
            // the static schedule finalises (and stores into every rank's y_full) from its first
            // segment on: wait until every rank has entered this call before any remote store
            if (ew == 0 && lane == 0) sys_wait(g.local_ctr + 1, rbase + kGridStride);
            asm volatile("bar.sync 1, 128;" ::: "memory");
        }
        int seg = 0;
        while (true) {
            const int2 it = take_item(bars, qi, qph, lane);
            if (it.x < 0) break;
            for (int u = it.x; u < it.y; ++seg) {
                const int gt = u / p.chunks, kcA = u - gt * p.chunks;
                const int sl = gt / p.tiles, rt = gt - sl * p.tiles;      // batch slice, row tile
                const int b0 = sl * g.bs;                                 // the slice's first column
                const int nb = (int)(g.B - b0 < g.bs ? g.B - b0 : g.bs);  // and its width
                int ue = (gt + 1) * p.chunks;
                if (ue > it.y) ue = it.y;
                const int kcB = kcA + (ue - u);
                const bool d1 = kWide || p.dsingle;
                const int db = d1 ? 0 : (seg & 1);
                mbar_wait(&bars.d_full[db], (uint32_t)((d1 ? seg : (seg >> 1)) & 1));
                tc_fence_after();
                long long te[4] = {0, 0, 0, 0}, tcy[3] = {0, 0, 0};
                if TLP(g) {
                    te[0] = gtimer();
                    tcy[0] = clock64();
                }
                // tot_b = sum_r |S_lo(r)| sum_j T_j D_r[b*a + j]; lo(r) = least significant layer of group
                // r.  The plane sum runs as Horner's rule (T_0 = -2^(a-1), T_j = 2^(a-1-j)):
                // h = -D[0]; h = 2h + D[j] -- branch-free, exact modulo 2^64.  B = 1 keeps the
                // total in a register; B > 1 parks per-column totals in SMEM (s_tot).
                unsigned long long tot1 = 0;
                for (int r = 0; r < p.regions; ++r) {
                    int last = (r + 1) * p.Gp - 1;
                    if (last > p.passes - 1) last = p.passes - 1;
                    const unsigned long long wr = layer_mag(g.L, g.offset, pass_lo(g.k_used, last), true);
                    const uint32_t dreg = tmem + lane_off + (uint32_t)(p.d_col + (db * p.regions + r) * NPAD);
                    if (!kWide && g.B == 1) {
                        // all of the region's columns in one batch of loads, one wait; digit
                        // Horner h = 4h + D_k (an odd a's lone last plane: 2h + D)
                        uint32_t dv[NPAD];
                        ld_tmem_cols<NPAD>(dreg, dv);
                        tmem_ld_wait();
                        if (TLP(g) && r == 0) {
                            te[3] = gtimer();
                            tcy[1] = clock64();
                        }
                        unsigned long long h = d2i(dv[0]);
#pragma unroll
                        for (int e = 1; e < NPAD; ++e) {
                            const unsigned long long v = d2i(dv[e]);
                            const int sh = (e == nd - 1 && (g.a & 1)) ? 1 : 2;
                            h = (e < nd) ? (h << sh) + v : h;
                        }
                        tot1 += h * wr;
                    } else if (plane_sums_dispatch<NPAD>(g.a, dreg, nb, m, s_tot_s, wr, r == 0)) {
                    } else {
                        // any other a: per batch column, serial digit Horner; wide: 32 columns
                        // per batch of loads
                        constexpr int kCG = kWide ? 32 : NPAD;
                        unsigned long long h = 0;
                        int j = 0, bc = 0;
#pragma unroll 1
                        for (int c0 = 0; c0 < NPAD && bc < nb; c0 += kCG) {
                            uint32_t dv[kCG];
                            ld_tmem_cols<kCG>(dreg + (uint32_t)c0, dv);
                            tmem_ld_wait();
                            if (TLP(g) && r == 0 && c0 == 0) {
                                te[3] = gtimer();
                                tcy[1] = clock64();
                            }
#pragma unroll
                            for (int e = 0; e < kCG; ++e) {
                                if (bc < nb) {
                                    const unsigned long long v = d2i(dv[e]);
                                    const int sh = (j == nd - 1 && (g.a & 1)) ? 1 : 2;
                                    h = j == 0 ? v : (h << sh) + v;
                                    if (++j == nd) {
                                        const uint32_t sa = s_tot_s + (uint32_t)(bc * kTcRows + m) * 8u;
                                        const unsigned long long t = h * wr;
                                        st_shared_u64(sa, r == 0 ? t : t + ld_shared_u64(sa));
                                        j = 0;
                                        ++bc;
                                    }
                                }
                            }
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars.d_empty[db]);
                if ((LOCAL && p.local)) {
                    // local mode: this chunk's (o - |S_0|) sum x_q joins the segment's partial
                    const unsigned long long x0 = xsum_of(0);
                    if (!kWide && g.B == 1) {
                        tot1 += o_corr * x0;
                    } else {
                        for (int b = 0; b < nb; ++b) {
                            const uint32_t sa = s_tot_s + (uint32_t)(b * kTcRows + m) * 8u;
                            st_shared_u64(sa, ld_shared_u64(sa) + o_corr * bars.xsum[b0 + b]);
                        }
                    }
                }
                stage_cols(b0, nb, seg & 1);
                seg_b0 = b0;
                spar = seg & 1;
                if (!g.x) asm volatile("bar.sync 1, 128;" ::: "memory");
                if TLP(g) {
                    te[1] = gtimer();
                    tcy[2] = clock64();
                }
                // exact integer adds into the tile's accumulator (order-independent); no
                // round trip here: tiles are finalised after the end-of-work grid barrier
                // shared-tile sums: narrow mode one slot per tile, wide mode one per CTA boundary
                const long long slot = kWide ? shared_slot(p, gt) : gt;
                unsigned long long* ab = g.accbuf + slot * g.bs * kTcRows + m;
                if (p.stat && kcA == 0 && kcB == p.chunks) {
                    // static schedule, the segment is the whole tile: y straight from the sums
                    const int64_t row = (int64_t)rt * kTcRows + m;
                    if (!kWide && g.B == 1)
                        finish_tile_row(0, row, tot1);
                    else
                        finish_cols(b0, nb, row);
                } else if ((LOCAL ? p.clu : 0)) {
                    // local cluster mode: one chunk per CTA, the tile's chunks are the cluster
                    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
                    if (kcA > 0) {
                        const uint32_t rb = mapa_shared_u32(redbuf_s + (uint32_t)(((kcA - 1) * g.bs * kTcRows + m) * 8), 0);
                        const uint32_t rbar = mapa_shared_u32(smem_u32(&bars.red_full), 0);
                        for (int b = 0; b < nb; ++b) {
                            const unsigned long long v = (!kWide && g.B == 1) ? tot1
                                : ld_shared_u64(s_tot_s + (uint32_t)(b * kTcRows + m) * 8u);
                            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(
                                             rb + (uint32_t)(b * kTcRows * 8)),
                                         "l"(v), "r"(rbar)
                                         : "memory");
                        }
                    } else {
                        asm volatile(
                            "{\n.reg .pred p;\nWC_%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], 0;\n"
                            "@!p bra WC_%=;\n}\n" ::"r"(smem_u32(&bars.red_full))
                            : "memory");
                        const int64_t row = (int64_t)rt * kTcRows + m;
                        if (!kWide && g.B == 1) {
                            for (int r = 1; r < (LOCAL ? p.clu : 0); ++r) tot1 += ld_shared_u64(redbuf_s + (uint32_t)(((r - 1) * g.bs * kTcRows + m) * 8));
                            finish_tile_row(0, row, tot1);
                        } else {
                            for (int b = 0; b < nb; ++b) {
                                const uint32_t sa = s_tot_s + (uint32_t)(b * kTcRows + m) * 8u;
                                unsigned long long t = ld_shared_u64(sa);
                                for (int r = 1; r < (LOCAL ? p.clu : 0); ++r)
                                    t += ld_shared_u64(redbuf_s + (uint32_t)((((r - 1) * g.bs + b) * kTcRows + m) * 8));
                                st_shared_u64(sa, t);
                            }
                            finish_cols(b0, nb, row);
                        }
                    }
                    cwaited = true;
                } else {
                    if (!kWide && g.B == 1) {
                        red_add_u64(ab, tot1);
                    } else {
                        for (int b = 0; b < nb; ++b)
                            red_add_u64(ab + b * kTcRows, ld_shared_u64(s_tot_s + (uint32_t)(b * kTcRows + m) * 8u));
                    }
                    if (p.stat) {
                        // a tile shared with neighbouring CTAs (at most two per CTA): count its
                        // chunks after the sums (the 128 threads' adds are ordered before thread
                        // 0's acq_rel by bar.sync: causality through the CTA barrier, as in a
                        // grid sync); the contributor that completes it finalises
                        asm volatile("bar.sync 1, 128;" ::: "memory");
                        if (ew == 0 && lane == 0) {
                            int old;
                            asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;"
                                         : "=r"(old)
                                         : "l"(g.counters + slot), "r"(kcB - kcA)
                                         : "memory");
                            bars.fin_tile = (old + (kcB - kcA) == p.chunks) ? rt : -1;
                        }
                        asm volatile("bar.sync 1, 128;" ::: "memory");
                        if (bars.fin_tile >= 0) {
                            const int64_t row = (int64_t)rt * kTcRows + m;
                            finish_from_accbuf(b0, nb, row, ab);
                            if (ew == 0 && lane == 0) g.counters[slot] = 0;
                        }
                    }
                }
                if (TLP(g) && ew == 0 && lane == 0) {
                    te[2] = gtimer();
                    bars.t_eseg[0] = te[0];
                    bars.t_eseg[1] = te[1];
                    bars.t_eseg[2] = te[2];
                    long long* rr = tl_record(TLP(g));
                    if (rr) {
                        const long long rec[10] = {3, blockIdx.x, seg, kcB - kcA, te[0], te[1], te[2], tcy[1] - tcy[0], te[3], tcy[2] - tcy[1]};
                        for (int k = 0; k < 10; ++k) rr[k] = rec[k];
                    }
                }
                u = ue;
            }
        }
        // ---- end-of-work grid barrier (the 128 threads' adds are ordered before the arrival by
        // bar.sync + thread 0's cumulative release), then this CTA finalises tiles
        // blockIdx.x, blockIdx.x + G, ...: y from the exact tile sums, accumulators re-zeroed
        if (!p.stat) {
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (ew == 0 && lane == 0) {
            if TLP(g) bars.t_ebar[0] = gtimer();
            grid_arrive(g.ebar);
            grid_wait(g.ebar, ebase);                // acquire; bar.sync passes it to the CTA
            if (g.nranks)                            // every rank has entered this call (f2)
                sys_wait(g.local_ctr + 1, rbase + kGridStride);   // (the static schedule waited above)
            if TLP(g) bars.t_ebar[1] = gtimer();
        }
        stage_cols(0, (int)g.B, seg & 1);         // (narrow: one slice of all B columns)
        seg_b0 = 0;
        spar = seg & 1;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        for (long long rt = blockIdx.x; rt < p.tiles; rt += G) {
            const int64_t row = rt * kTcRows + m;
            unsigned long long* ab = g.accbuf + rt * g.B * kTcRows + m;
            finish_from_accbuf(0, (int)g.B, row, ab);                // (every call leaves the sums zero)
        }
        }   // !p.stat
        if (g.nranks) {
            // every rank's y_full holds this CTA's rows once its counter has the arrival: each
            // rank's CTAs add kGridStride / nranks in total (CTA 0 the remainder), so a call
            // adds exactly kGridStride to every counter whatever the grid sizes
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (ew == 0 && lane == 0) {
                __threadfence_system();              // the CTA's remote y stores (ordered by bar.sync)
                const unsigned long long amt =
                    blockIdx.x == 0 ? kGridStride / (unsigned)g.nranks - (gridDim.x - 1) : 1ull;
                for (int q = 0; q < g.nranks; ++q)
                    asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(g.peer_ctr[q]), "l"(amt)
                                 : "memory");
                sys_wait(g.local_ctr, xbase + kGridStride);
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
        }
        if (TLP(g) && ew == 0 && lane == 0) bars.t_cend = gtimer();
    }

    if (kTimeline && p.prof && TLP(g) && lane == 0) {
        // wait totals (ns): w_empty, b_full, a_full, w_full, a_empty
        long long* r = tl_record(TLP(g));
        if (r) {
            const long long rec[10] = {4, blockIdx.x, warp, gtimer() - g_start, prof[0], prof[1], prof[2], prof[3],
                                       prof[4], 0};
            for (int k = 0; k < 10; ++k) r[k] = rec[k];
        }
    }
    if ((LOCAL ? p.clu : 0) && !cwaited) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    if (TLP(g) && warp == 1 && lane == 0) {
        long long* r = tl_record(TLP(g));
        if (r) {
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            const long long rec[10] = {1, blockIdx.x, smid, 0, g_start, bars.t_b, bars.t_mma0, bars.t_mend,
                                       bars.t_cend, gtimer()};
            for (int k = 0; k < 10; ++k) r[k] = rec[k];
        }
        long long* r6 = tl_record(TLP(g));
        if (r6) {
            const long long rec[10] = {6, blockIdx.x, bars.t_mend, bars.t_eseg[0], bars.t_eseg[1], bars.t_eseg[2],
                                       bars.t_ebar[0], bars.t_ebar[1], bars.t_cend, gtimer()};
            for (int k = 0; k < 10; ++k) r6[k] = rec[k];
        }
        long long* r5 = tl_record(TLP(g));
        if (r5) {
            const long long rec[10] = {5, blockIdx.x, bars.t_c0s[0], bars.t_c0s[1], bars.t_cv[0], bars.t_cv[1],
                                       bars.t_cv[2], bars.t_cv[3], bars.t_c0, 0};
            for (int k = 0; k < 10; ++k) r5[k] = rec[k];
        }
    }
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// Tensor maps of the stored weights (pb.h), box {32 words, 128 rows, 1}, 128B
// swizzle; out-of-range rows / words (tile tails) are filled with zeros:
//   pmap: the L/2 layer pairs as {2*kwords, R, L/2} (pair rows of 2*kwords words);
//   smap: the canonical last layer of an odd L as {kwords, R, 1}.
// A map the shape does not have is a copy of the other (never read).
cudaError_t make_weight_maps(const GemmArgs& g, CUtensorMap* pmap, CUtensorMap* smap)
{
    static EncodeTiledFn encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
        encode = reinterpret_cast<EncodeTiledFn>(fn);
    }
    const cuuint32_t box[3] = {kChunkWords, kTcRows, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    auto enc = [&](CUtensorMap* m, const uint32_t* base, cuuint64_t w, cuuint64_t depth) {
        const cuuint64_t dims[3] = {w, (cuuint64_t)g.R, depth};
        const cuuint64_t strides[2] = {w * 4, w * 4 * (cuuint64_t)g.R};
        return encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<uint32_t*>(base), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    CUresult r = CUDA_SUCCESS;
    if (g.L >= 2) r = enc(pmap, g.bits, 2 * (cuuint64_t)g.kwords, (cuuint64_t)(g.L / 2));
    if (r == CUDA_SUCCESS && (g.L & 1))
        r = enc(smap, g.bits + (int64_t)(g.L - 1) * g.R * g.kwords, (cuuint64_t)g.kwords, 1);
    if (g.L < 2) *pmap = *smap;
    if (!(g.L & 1)) *smap = *pmap;
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
    const bool wide = npad > kTcMaxN;
    if (npad <= 0 || g.kwords <= 0 || g.R <= 0 || g.B <= 0 || g.L > 16) return false;
    if (wide ? (npad != kTcWideN || g.x || g.nranks || g.bs < 1 || (int64_t)g.bs * act_digits(g.a) > npad)
             : (g.B > kTcMaxB))
        return false;
    p.tiles = (int)((g.R + kTcRows - 1) / kTcRows);
    if (!wide && p.tiles > kAccTiles) return false;
    p.chunks = (int)((g.kwords + kChunkWords - 1) / kChunkWords);
    p.slices = wide ? (int)((g.B + g.bs - 1) / g.bs) : 1;
    p.units = (long long)p.slices * p.tiles * p.chunks;
    if (p.units >= (1ll << 30)) return false;                  // int unit indices in the kernel
    // exact f32 accumulation: per pass and column |(2 hi + lo) d| <= 9 (signed activation
    // digits, |d| <= 3), so a group of G layers sums to |D| < 3 K 2^G <= 2^24
    int G = 24 - ceil_log2_i(3 * g.kwords * 32);
    if (G > 15) G = 15;                           // SFB exponents 0..13 fit the 64-column SF area
    p.Gp = G / 2;
    if (p.Gp < 1) return false;
    p.passes = (g.k_used + 1) / 2;
    p.regions = (p.passes + p.Gp - 1) / p.Gp;
    if (p.regions > kMaxRegions) return false;
    // narrow: two accumulator sets (segment parity); wide: one -- and narrow too when two
    // sets would leave fewer than two A slots (several groups at a wide N, e.g. L = 16 at K =
    // 2048 with 64 digit columns): a drained accumulator then blocks the next segment's MMAs,
    // but one launch covers twice the batch columns
    p.dsingle = 0;
    p.d_col = 512 - ((wide ? 1 : 2) * p.regions * npad + 31) / 32 * 32;
    if (!wide && (p.d_col - 64) / 128 < 2 && p.regions > 1) {
        p.dsingle = 1;
        p.d_col = 512 - (p.regions * npad + 31) / 32 * 32;
    }
    p.sf_col = p.d_col - 64;
    p.slots = p.sf_col / 128;
    if (p.slots > kMaxSlots) p.slots = kMaxSlots;
    if (p.slots < 2) return false;
    // work items of >= ~4 passes (so an item's epilogue keeps up with its MMAs)
    if ((long long)g.B * p.chunks * kChunkWords >= (1ll << 31)) return false;   // prologue index math
    p.Gu = (4 + p.passes - 1) / p.passes;
    p.stat = 0;
    p.items = (p.units + p.Gu - 1) / p.Gu;
    return true;
}

// Per-device launch state: SM count and whether the kernel's attributes are set (function
// attributes belong to the device's context, so one process driving several GPUs sets them on
// each).  Devices are few; the table is written once per (device, NPAD) under a mutex.
struct DevState {
    int sms = 0;
    bool attr[5] = {false, false, false, false, false};
};
constexpr int kMaxDevices = 64;
DevState g_dev[kMaxDevices];
std::mutex g_dev_mu;

// Tensor maps of recently used weight buffers (per thread, tiny LRU): encoding two
// CUtensorMaps costs a few microseconds of host time per un-graphed call otherwise.
struct MapEntry {
    const uint32_t* bits = nullptr;
    int64_t R = 0, kwords = 0;
    int L = 0, dev = -1;
    CUtensorMap pmap, smap;
    unsigned long long used = 0;
};
constexpr int kMapCache = 8;
thread_local MapEntry t_maps[kMapCache];
thread_local unsigned long long t_map_clock = 0;

cudaError_t weight_maps_cached(const GemmArgs& g, int dev, CUtensorMap* pmap, CUtensorMap* smap)
{
    MapEntry* victim = &t_maps[0];
    for (int i = 0; i < kMapCache; ++i) {
        MapEntry& e = t_maps[i];
        if (e.bits == g.bits && e.R == g.R && e.kwords == g.kwords && e.L == g.L && e.dev == dev) {
            e.used = ++t_map_clock;
            *pmap = e.pmap;
            *smap = e.smap;
            return cudaSuccess;
        }
        if (e.used < victim->used) victim = &e;
    }
    cudaError_t r = make_weight_maps(g, pmap, smap);
    if (r != cudaSuccess) return r;
    victim->bits = g.bits;
    victim->R = g.R;
    victim->kwords = g.kwords;
    victim->L = g.L;
    victim->dev = dev;
    victim->pmap = *pmap;
    victim->smap = *smap;
    victim->used = ++t_map_clock;
    return cudaSuccess;
}

template <int NPAD>
cudaError_t launch_t(const GemmArgs& g, cudaStream_t s)
{
    static int dbg = -1, prof = 0, bst_env = 0, stat_env = -1, dyn_pct = 0, clu_max = 4;   // 8-CTA clusters: 1.6x slower (co-scheduling)
    static std::once_flag env_once;
    std::call_once(env_once, [] {
        const char* ev = getenv("PB_TC_DEBUG");
        dbg = ev ? atoi(ev) : 0;
        ev = getenv("PB_TC_CLU");              // experiment knob: largest local-mode cluster (< 2: off)
        if (ev) clu_max = atoi(ev);
        ev = getenv("PB_TC_KNOB");             // profiling knob with the timeline on (PB_TC_DEBUG=6)
        if (ev) dbg = atoi(ev);
        ev = getenv("PB_TC_PROF");
        prof = ev ? atoi(ev) : 0;
        ev = getenv("PB_TC_BSTAGES");          // experiment knob: B ring depth
        bst_env = ev ? atoi(ev) : 0;
        ev = getenv("PB_TC_STATIC");           // comparison knob: 0 = dynamic stream-K claims
        stat_env = ev ? atoi(ev) : -1;
        ev = getenv("PB_TC_DYN");              // experiment knob: % of units claimed dynamically
        dyn_pct = ev ? atoi(ev) : 0;
    });
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    DevState& ds = g_dev[dev];
    constexpr int ai = NPAD == 8 ? 0 : (NPAD == 16 ? 1 : (NPAD == 32 ? 2 : (NPAD == 64 ? 3 : 4)));
    if (!ds.attr[ai] || !ds.sms) {
        std::lock_guard<std::mutex> lk(g_dev_mu);
        if (!ds.sms) {
            int n = 0;
            if ((e = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
            ds.sms = n;
        }
        if (!ds.attr[ai]) {
            e = cudaFuncSetAttribute(bitgemm_tc_kernel<NPAD, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kSmemMax);
            if (e != cudaSuccess) return e;
            cudaFuncSetAttribute(bitgemm_tc_kernel<NPAD, false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 (int)cudaSharedmemCarveoutMaxShared);
            if constexpr (NPAD <= kTcMaxN) {
                e = cudaFuncSetAttribute(bitgemm_tc_kernel<NPAD, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSmemMax);
                if (e != cudaSuccess) return e;
                cudaFuncSetAttribute(bitgemm_tc_kernel<NPAD, true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     (int)cudaSharedmemCarveoutMaxShared);
            }
            ds.attr[ai] = true;
        }
    }
    const int sms = ds.sms;
    TcPlan p;
    if (!make_plan(g, NPAD, p)) return cudaErrorNotSupported;
    if (stat_env != 0 || NPAD > kTcMaxN) {     // default: static (PB_TC_STATIC=0: dynamic claims)
        p.stat = 1;
        p.gs = (int)(p.units < sms ? p.units : sms);
        if (p.gs > kMaxCtas) p.gs = kMaxCtas;
        long long dyn = NPAD > kTcMaxN ? 0 : p.units * dyn_pct / 100;   // a dynamic tail of single-unit claims
                                                   // (narrow only: wide shared slots assume the static split)
        if (dyn < 0) dyn = 0;
        p.Gu = 1;
        p.ustat = p.units - dyn;
        if (p.ustat < p.gs) p.ustat = p.units < p.gs ? p.units : p.gs;
        // wide mode with few (slice, tile) pairs: one whole tile per CTA, so no tile is shared
        // and no partial sums go through atomics (the wide epilogue's dominant cost: 16
        // batch columns x 128 rows per shared tile)
        if (NPAD > kTcMaxN && p.chunks > 1 && (long long)p.slices * p.tiles <= sms && !dyn) {
            p.gs = (int)(p.slices * p.tiles);
            p.ustat = p.units;
        }
        p.items = p.gs + (p.units - p.ustat);
    }
    CUtensorMap pmap, smap;
    e = weight_maps_cached(g, dev, &pmap, &smap);
    if (e != cudaSuccess) return e;
    p.dbg = dbg;
    p.prof = prof;
    p.local = (g.x && p.stat && NPAD <= kTcMaxN && p.units <= p.gs && p.items == p.gs && !(dbg & 128)) ? 1 : 0;
    p.clu = (p.local && p.chunks >= 2 && p.chunks <= clu_max && p.gs % p.chunks == 0) ? p.chunks : 0;
    // weight ring: every 16 KiB stage the B stages and epilogue sums leave free
    p.bstages = (p.passes <= 2 && NPAD <= kTcMaxN) ? kMaxBStages : 2;
    if (bst_env) p.bstages = bst_env < 2 ? 2 : (bst_env > kMaxBStages ? kMaxBStages : bst_env);
    if (NPAD > kTcMaxN && p.bstages > 2) p.bstages = 2;        // 64 KiB per wide B stage
    const uint32_t fixed = 1024 + kHdrBytes + (uint32_t)p.bstages * (kChunkWords / 2) * NPAD * 32 + (uint32_t)g.bs * kTcRows * 8 +
                           (uint32_t)(p.clu ? p.clu - 1 : 0) * g.bs * kTcRows * 8;
    p.wstages = (int)((kSmemMax - fixed) / kWTileBytes);
    if (p.wstages > kMaxWStages) p.wstages = kMaxWStages;
    if (p.wstages < 4) return cudaErrorNotSupported;
    const uint32_t smem = fixed + (uint32_t)p.wstages * kWTileBytes;
    long long grid = p.stat ? p.gs : (p.items < sms ? p.items : sms);
    if (grid > kMaxCtas) grid = kMaxCtas;

    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute la[2];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = 1;
    la[1].id = cudaLaunchAttributeClusterDimension;             // local cluster mode: a tile's chunks
    la[1].val.clusterDim.x = (unsigned)(p.clu ? p.clu : 1);
    la[1].val.clusterDim.y = 1;
    la[1].val.clusterDim.z = 1;
    cfg.attrs = la;
    cfg.numAttrs = p.clu ? 2 : 1;
    // the local-mode code lives in its own instantiation: the streaming kernel's code (and
    // I-cache footprint) is the same as without it
    if constexpr (NPAD <= kTcMaxN)
        if (p.local) return cudaLaunchKernelEx(&cfg, bitgemm_tc_kernel<NPAD, true>, g, p, pmap, smap);
    return cudaLaunchKernelEx(&cfg, bitgemm_tc_kernel<NPAD, false>, g, p, pmap, smap);
}

}  // namespace

cudaError_t tc_weight_maps(const GemmArgs& g, CUtensorMap* pmap, CUtensorMap* smap)
{
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    return weight_maps_cached(g, dev, pmap, smap);
}

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
        case 64: return launch_t<64>(g, s);
        case kTcWideN: return launch_t<kTcWideN>(g, s);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace pb
