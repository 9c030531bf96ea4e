// pb_lstm_tc.cu -- the LSTM recurrence as ONE persistent tensor-engine kernel (SURVEY §8(f)
// f1): every timestep's 4-gate matvec W_hh h_t ("replace each linear layer
// ... LSTM" with the bitlayer product) plus the cell, with a grid barrier per timestep
// instead of a launch.
//
// The input projection W_ih x_t + b of all T timesteps is one batched call before this
// kernel (pb_lstm_seq); here gx[t] is added to the recurrent pre-activations.  Per timestep
// (Alg. 2 on h_t):
//   a1-a2  every CTA reads h_t (B x H floats, L2): max|h_t[b,:]| -> f_b (reading G8),
//          sum_c x_q over all H, and the activation digits of its own K-chunk straight into
//          the MMA's B operand in SMEM (ballot transpose, pb_common.cuh);
//   a3-a4  tcgen05.mma kind::mxf4 (two weight bitlayers per nibble, as pb_gemm_tc.cu) over
//          the CTA's unit = 128 gate rows x 1024 columns, accumulated exactly in TMEM;
//   a5     the unit's exact int64 row sums; a tile split over several CTAs (K > 1024) is
//          summed exactly (red.add) and finished by the contributor that completes it:
//          dequant (G13) + gx[t] -> the four gates of 32 hidden units (gate-interleaved rows,
//          lanes 4j..4j+3) -> c' = s(f) c + s(i) tanh(g), h' = s(o) tanh(c') (reading G15);
//   then one grid barrier (monotonic counter, pb_tc_device.cuh) publishes h_{t+1}.
// The weights do not depend on h: warp 0 streams the unit's weight tiles through the TMA ring
// and the converters build the A operand in TMEM for the next timestep while this one waits
// on its barrier, so a timestep costs the barrier, the h read and the MMAs -- not a launch.
//
// One CTA per unit (tiles x chunks <= #SMs, all co-resident): 128 CTAs for H = 2048.
// Warp roles (480 threads): 0 TMA producer, 1 TMEM allocator + MMA issuer, 2 idle after setup,
// 3..10 converters (two h-sets of 4), 11..14 per-step prologue + epilogue.
#include <cuda.h>
#include <cstdint>
#include <cuda_runtime.h>
#include <cstdlib>
#include <mutex>

#include "pb_common.cuh"
#include "pb_internal.h"
#include "pb_tc_device.cuh"

namespace pb {
namespace {

constexpr int kConvWarps = 8;
constexpr int kConv0 = 3;
constexpr int kEpi0 = kConv0 + kConvWarps;
constexpr int kEpiWarps = 4;
constexpr int kThreads = 32 * (kEpi0 + kEpiWarps);
constexpr int kMaxSlots = 4;                  // A slots in TMEM
constexpr int kMaxSPass = 2;                  // resident passes whose A lives in SMEM (SS MMAs)
constexpr int kMaxWStages = 16;
constexpr uint32_t kHdrBytes = 4096;

struct LBars {
    uint64_t a_full[kMaxSlots + kMaxSPass], a_empty[kMaxSlots];
    uint64_t w_full[kMaxWStages], w_empty[kMaxWStages];
    uint64_t b_full, d_full, d_empty, h_full, h_empty;
    uint64_t red_full;                         // cluster leader: the other chunks' partial sums are in
    uint64_t gx_full[2];                       // step t's gx rows of the tile are in SMEM (by t & 1: warp 2
                                               // runs one step ahead, a single barrier would overrun)
    unsigned long long epoch0;                 // barrier instance of this call's step 0
    uint32_t tmem_base;
    int fin;                                   // this step: the CTA completed its tile (1) or not
    float red[kEpiWarps][kLstmMaxB];           // per-warp partial max|h[b,:]|
    float pmax[2][kEpiWarps];                  // B = 1 producer: per-warp max|h_{t+1}| (by t & 1)
    int f[2][kLstmMaxB];                       // f_b of step t at [t & 1]
    double sc[2][kLstmMaxB];                   // s_w 2^-f_b
    float scl[2][kLstmMaxB];                   // 2^f_b as fp32 (the cast's fast path)
};
static_assert(sizeof(LBars) <= kHdrBytes, "LBars must fit the SMEM header");

// Cluster (DSMEM) helpers: the CTAs of one cluster are the K-chunks of one row tile.
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_u64(uint32_t addr, unsigned long long v) {
    asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAITC_%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAITC_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

struct LPlan {
    int tiles, chunks;
    int slots, sf_col, d_col, wstages;
    int passes, Gp, regions;
    int resident;              // the unit's A (all passes) stays on chip for every timestep
    int spass;                 // resident: the last spass passes keep A in SMEM (64 KiB each, carved
                               // from the weight ring, idle after step 0; SS MMAs), the rest in TMEM
    int helpers;               // resident, B = 1, even a <= 16: the converter warps build the
                               // digits of steps t >= 1 (with their A converted once, they idle)
};

template <int NPAD>
__global__ void __launch_bounds__(kThreads, 1)
lstm_persist_kernel(const LstmArgs g, const LPlan p, const __grid_constant__ CUtensorMap pmap,
                    const __grid_constant__ CUtensorMap smap)
{
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte aligned as an offset into smem_raw (not through an integer cast), so the compiler
    // keeps the shared window: every access through `bars` is LDS/STS, not a generic LD/ST
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    LBars& bars = *reinterpret_cast<LBars*>(smem);
    constexpr uint32_t kBTile = NPAD * 32;
    constexpr uint32_t kBStage = (kChunkWords / 2) * kBTile;
    constexpr bool kWide = NPAD > kTcMaxN;
    uint8_t* wtile0 = smem + kHdrBytes;
    uint8_t* sa = wtile0 + p.wstages * kWTileBytes;            // [spass][16 MMAs][4 KiB] SMEM A
    uint8_t* bstage = sa + (size_t)p.spass * 16 * 4096;
    const uint32_t s_tot_s = smem_u32(bstage + kBStage);       // [b][128] u64 (B > 1)
    uint8_t* hbuf = bstage + kBStage + (size_t)g.B * kTcRows * 8;  // [b][1024] fp32: the K-chunk of h_t
    const uint32_t redbuf_s = smem_u32(hbuf + (size_t)g.B * kChunkWords * 32 * 4);   // [chunks-1][b][128] u64
    float* gxbuf = reinterpret_cast<float*>(hbuf + (size_t)g.B * kChunkWords * 32 * 4 +
                                            (size_t)(p.chunks - 1) * g.B * kTcRows * 8);   // [2][b][128] fp32
    float* cst = gxbuf + 2 * g.B * kTcRows;                     // [b][32] the leader's cell state
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rt = blockIdx.x / p.chunks, kc = blockIdx.x - rt * p.chunks;
    const int T = g.T;

    if (threadIdx.x == 0) {
        for (int s = 0; s < p.slots; ++s) {
            mbar_init(&bars.a_full[s], 4);
            mbar_init(&bars.a_empty[s], 1);
        }
        for (int s = p.slots; s < p.slots + p.spass; ++s) mbar_init(&bars.a_full[s], 4);
        for (int s = 0; s < p.wstages; ++s) {
            mbar_init(&bars.w_full[s], 1);
            mbar_init(&bars.w_empty[s], 4);
        }
        mbar_init(&bars.b_full, 1);
        mbar_init(&bars.d_full, 1);
        mbar_init(&bars.d_empty, kEpiWarps);
        mbar_init(&bars.h_full, 2);                // the copies (expect_tx) + f_b of the step
        mbar_init(&bars.h_empty, 1);
        mbar_init(&bars.red_full, 1);              // the leader's expect_tx; the others' st.async bytes
        mbar_init(&bars.gx_full[0], 1);
        mbar_init(&bars.gx_full[1], 1);
        fence_mbar_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(&pmap) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&smap) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            smem_u32(&bars.tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync();                                // barrier inits visible to the cluster's CTAs
    tc_fence_after();
    const uint32_t tmem = bars.tmem_base;
    if (warp >= kConv0 && warp < kConv0 + 4) {
        store_scale_factors(tmem, warp, p.sf_col);
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_trigger();

    if (warp == 0) {
        // ---------------------------------------------- weight tiles of this CTA's unit, every
        // timestep (L2-resident after the first), as far ahead as the ring allows
        int tc = 0;
        for (int t = 0; t < (p.resident ? 1 : T); ++t)
            for (int ps = 0; ps < p.passes; ++ps) {
                const bool stored_pair = 2 * ps + 1 < g.L;
                for (int h = 0; h < (stored_pair ? 2 : 1); ++h, ++tc) {
                    const int st = tc % p.wstages;
                    mbar_wait(&bars.w_empty[st], (uint32_t)(((tc / p.wstages) & 1) ^ 1));
                    if (elect_one()) {
                        mbar_arrive_expect_tx(&bars.w_full[st], kWTileBytes);
                        if (stored_pair)
                            tma_load_3d(wtile0 + st * kWTileBytes, &pmap, kc * 2 * kChunkWords + h * kChunkWords,
                                        rt * kTcRows, ps, &bars.w_full[st]);
                        else
                            tma_load_3d(wtile0 + st * kWTileBytes, &smap, kc * kChunkWords, rt * kTcRows, 0,
                                        &bars.w_full[st]);
                    }
                    __syncwarp();
                }
            }
    } else if (warp == 1) {
        // ---------------------------------------------- MMA issuer
        const uint32_t idesc = mxf4_idesc(NPAD);
        const uint32_t sfa = tmem + p.sf_col;
        const uint64_t bdesc0 = b_desc(smem_u32(bstage));
        uint32_t slot = 0, phase = 0;
        for (int t = 0; t < T; ++t) {
            mbar_wait(&bars.b_full, (uint32_t)(t & 1));                 // h_t's digits are in SMEM
            if (t > 0) mbar_wait(&bars.d_empty, (uint32_t)((t - 1) & 1));   // D(t-1) drained
            tc_fence_after();
            for (int ps = 0; ps < p.passes; ++ps) {
                int region, sexp;
                bool first;
                pass_region_g(p.Gp, p.passes, g.k_used, ps, region, sexp, first);
                const uint32_t dcol = tmem + (uint32_t)(p.d_col + region * NPAD);
                const uint32_t sfb = tmem + (uint32_t)(p.sf_col + 4 * (1 + sexp));
                if (p.resident) slot = (uint32_t)ps;
                if (!p.resident || t == 0) mbar_wait(&bars.a_full[slot], p.resident ? 0u : phase);
                tc_fence_after();
                if (elect_one()) {
                    if (p.resident && ps >= p.slots) {
                        // A in SMEM (SS): 16 tiles of 128 rows x 32 B, 4 KiB apart
                        const uint64_t ad0 = b_desc(smem_u32(sa) + (uint32_t)(ps - p.slots) * 16u * 4096u);
#pragma unroll
                        for (int uu = 0; uu < 16; ++uu)
                            tc_mma_ss(dcol, ad0 + (uint64_t)(uu * (4096 / 16)), bdesc0 + uu * (kBTile / 16), idesc,
                                      (uu == 0 && first) ? 0u : 1u, sfa, sfb);
                    } else {
                        const uint32_t a0 = tmem + slot * 128;
#pragma unroll
                        for (int uu = 0; uu < 16; ++uu)
                            tc_mma(dcol, a0 + 8 * uu, bdesc0 + uu * (kBTile / 16), idesc, (uu == 0 && first) ? 0u : 1u,
                                   sfa, sfb);
                    }
                    if (!p.resident) tc_commit(&bars.a_empty[slot]);
                }
                __syncwarp();
                if (++slot == (uint32_t)p.slots) {
                    slot = 0;
                    phase ^= 1;
                }
            }
            if (elect_one()) tc_commit(&bars.d_full);
            __syncwarp();
        }
    } else if (warp >= kConv0 && warp < kEpi0) {
        // ---------------------------------------------- converters (as pb_gemm_tc.cu): pass pc of
        // the whole run goes to h-set pc & 1 and A slot pc % slots
        const int cw = warp - kConv0;
        const int h = cw >> 2;
        const int q = warp & 3;
        const int m = q * 32 + lane;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const uint32_t wtile_s = smem_u32(wtile0) + (uint32_t)m * 128;
        const uint32_t swz = (uint32_t)(m & 7);
        int tc = 0, pc = 0;
        int slot = h % p.slots, sphase = (h / p.slots) & 1;
        int pend_slot = -1;
        auto publish = [&]() {
            if (pend_slot >= 0) {
                tmem_st_wait();
                if (pend_slot >= p.slots) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // SMEM A
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars.a_full[pend_slot]);
                pend_slot = -1;
            }
        };
        for (int t = 0; t < (p.resident ? 1 : T); ++t)
            for (int ps = 0; ps < p.passes; ++ps, ++pc) {
                const bool stored_pair = 2 * ps + 1 < g.L;
                const bool use_lo = 2 * ps + 1 < g.k_used;
                const int ntile = stored_pair ? 2 : 1;
                if ((pc & 1) != h) {
                    tc += ntile;
                    continue;
                }
                const int st0 = tc % p.wstages, st1 = (tc + ntile - 1) % p.wstages;
                mbar_wait(&bars.w_full[st0], (uint32_t)((tc / p.wstages) & 1));
                if (stored_pair) mbar_wait(&bars.w_full[st1], (uint32_t)(((tc + 1) / p.wstages) & 1));
                publish();
                if (p.resident) slot = ps;                    // slots fresh: nothing to wait for
                else mbar_wait(&bars.a_empty[slot], (uint32_t)(sphase ^ 1));
                tc_fence_after();
                const int kind = stored_pair ? (use_lo ? 0 : 1) : 2;
                const int sgn = ps == 0 ? (g.offset ? 2 : 1) : 0;   // the sign layer's pass: signed nibbles
                const uint32_t t0 = wtile_s + (uint32_t)st0 * kWTileBytes;
                const uint32_t t1 = wtile_s + (uint32_t)st1 * kWTileBytes;
                const uint32_t dst = tmem + lane_off + (uint32_t)(slot * 128);
                if (p.resident && ps >= p.slots) {
                    // A of this pass in SMEM: the row's line of the core matrices
                    const uint32_t sdst = smem_u32(sa) + (uint32_t)(ps - p.slots) * 16u * 4096u +
                                          (uint32_t)((m >> 3) * 256 + (m & 7) * 16);
                    if (kind == 0)
                        convert_pass<0, true>(t0, t1, swz, sdst, 0u, sgn, 0, &bars.w_empty[st0], &bars.w_empty[st1], lane);
                    else if (kind == 1)
                        convert_pass<1, true>(t0, t1, swz, sdst, 0u, sgn, 0, &bars.w_empty[st0], &bars.w_empty[st1], lane);
                    else
                        convert_pass<2, true>(t0, t1, swz, sdst, 0u, sgn, 0, &bars.w_empty[st0], &bars.w_empty[st1], lane);
                } else if (kind == 0)
                    convert_pass<0>(t0, t1, swz, dst, 0u, sgn, 0, &bars.w_empty[st0], &bars.w_empty[st1], lane);
                else if (kind == 1)
                    convert_pass<1>(t0, t1, swz, dst, 0u, sgn, 0, &bars.w_empty[st0], &bars.w_empty[st1], lane);
                else
                    convert_pass<2>(t0, t1, swz, dst, 0u, sgn, 0, &bars.w_empty[st0], &bars.w_empty[st1], lane);
                tc += ntile;
                pend_slot = slot;
                slot += 2;
                while (slot >= p.slots) {
                    slot -= p.slots;
                    sphase ^= 1;
                }
            }
        publish();
        if (p.helpers && T > 1) {
            // ---- steps t >= 1: this warp's 4 words (cw + 8k) of the CTA's K-chunk of h_t, polled
            //      as tagged values (the epilogue warps poll the max slots meanwhile), then cast
            //      with f_b (named barrier 2) and transposed into the B operand (barrier 3)
            pdl_wait();
            const unsigned long long sbase = ld_acquire_gpu_u64(g.stepctr);
            const int H = (int)g.H, a = g.a, nd = act_digits(a);
            const int cbase = kc * kChunkWords * 32, cvalid = H - cbase;
            const uint32_t bstage_s = smem_u32(bstage);
            const uint32_t amask = (1u << a) - 1u;
            const float lim = (float)(1 << (a - 1));
            for (int t = 1; t < T; ++t) {
                const int par = t & 1;
                const uint32_t tag = (uint32_t)(sbase + (unsigned long long)t);
                const unsigned long long* hx = g.hx + (int64_t)par * H + cbase;
                unsigned long long hv[4];
                bool ok;
                do {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int cl = (cw + 8 * k) * 32 + lane;
                        hv[k] = cl < cvalid ? ld_relaxed_gpu_u64(hx + cl) : (unsigned long long)tag << 32;
                    }
                    ok = true;
#pragma unroll
                    for (int k = 0; k < 4; ++k) ok = ok && (uint32_t)(hv[k] >> 32) == tag;
                } while (!ok);
                asm volatile("barrier.sync 2, 384;" ::: "memory");   // f_b of step t in bars (non-aligned: two code sites)
                uint32_t u[4], reg[4];
                if (bars.scl[par][0] != 0.f) {
                    const float sc = bars.scl[par][0];
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        u[k] = (uint32_t)__float2int_rz(fminf(fmaxf(__uint_as_float((uint32_t)hv[k]) * sc, -lim), lim - 1.0f));
                } else {
                    const int f = bars.f[par][0];
#pragma unroll
                    for (int k = 0; k < 4; ++k) u[k] = (uint32_t)act_cast(__uint_as_float((uint32_t)hv[k]), f, a);
                }
                int dk = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) reg[k] = digit_regs_shfl(u[k] & amask, a, lane, dk);
                if (dk < nd) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        asm volatile("st.shared.u32 [%0], %1;" ::"r"(bstage_s + b_operand_offset(NPAD, cw + 8 * k, dk, lane & 3)),
                                     "r"(reg[k]) : "memory");
                }
                if (nd < NPAD) {
#pragma unroll 1
                    for (int k = 0; k < 4; ++k)
                        for (int n = nd + lane; n < NPAD; n += 32)
                            put_b_operand_smem(bstage_s, NPAD, cw + 8 * k, n, make_uint4(0, 0, 0, 0));
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic SMEM writes -> MMA
                asm volatile("barrier.sync 3, 384;" ::: "memory");          // B of step t complete
            }
        }
    } else if (warp == 2) {
        // ---------------------------------------------- step gate: the tile's gx[t] rows (leader),
        // and for B > 1: once h_t is complete on every CTA (grid barrier of step t-1), this CTA's
        // K-chunk of h_t (B rows of <= 1024 floats) into SMEM (1-D bulk copies on h_full) and
        // f_b from the epoch-tagged atomicMax slots.  (B = 1 exchanges h through tagged values,
        // read by the epilogue warps themselves.)
        pdl_wait();
        asm volatile("fence.proxy.async.global;" ::: "memory");   // gx / h0 (earlier kernels) -> bulk reads
        unsigned long long gbase = 0;
        if (lane == 0) gbase = grid_base(g.gbar);
        const int H = (int)g.H;
        const int c0 = kc * kChunkWords * 32;
        const int ncol = H - c0 < kChunkWords * 32 ? H - c0 : kChunkWords * 32;
        const int64_t r0 = (int64_t)rt * kTcRows;
        const int nrow = g.R - r0 < kTcRows ? (int)(g.R - r0) : kTcRows;
        const bool tagx = g.B == 1;
        for (int t = 0; t < T; ++t) {
            if (t > 0) mbar_wait(&bars.h_empty, (uint32_t)((t - 1) & 1));   // the prologue of step t-1 is done
            if (lane == 0 && kc == 0) {
                // the tile's rows of gx[t] (no dependence on h): in flight while the step waits
                mbar_arrive_expect_tx(&bars.gx_full[t & 1], (uint32_t)(g.B * nrow * 4));
                for (int b = 0; b < g.B; ++b)
                    bulk_g2s(gxbuf + ((t & 1) * g.B + b) * kTcRows, g.gx + ((int64_t)t * g.B + b) * g.R + r0,
                             (uint32_t)(nrow * 4), &bars.gx_full[t & 1]);
            }
            if (tagx) continue;
            if (lane == 0) {
                if (t > 0) {
                    const unsigned long long* c = reinterpret_cast<const unsigned long long*>(g.gbar);
                    while (ld_acquire_gpu_u64(c) < gbase + (unsigned long long)t * kGridStride) {
                    }
                    asm volatile("fence.proxy.async.global;" ::: "memory");   // generic h stores -> bulk reads
                }
                const float* x = t == 0 ? g.h0 : g.h_seq + (int64_t)(t - 1) * g.B * H;
                mbar_arrive_expect_tx(&bars.h_full, (uint32_t)(g.B * ncol * 4));
                for (int b = 0; b < g.B; ++b)
                    bulk_g2s(hbuf + (size_t)b * kChunkWords * 32 * 4, x + (int64_t)b * H + c0, (uint32_t)(ncol * 4),
                             &bars.h_full);
            }
            __syncwarp();
            if (t > 0 && lane < g.B) {
                const unsigned long long v = __ldcg(g.maxslot + ((t & 1) * kLstmMaxB + lane));
                const int f = act_frac_of(__uint_as_float((uint32_t)v), g.a);
                bars.f[t & 1][lane] = f;
                bars.sc[t & 1][lane] = col_scale(g.scale, f);
                bars.scl[t & 1][lane] = (f >= -126 && f <= 127) ? __int_as_float((127 + f) << 23) : 0.f;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars.h_full);
        }
    } else if (warp >= kEpi0) {
        // ---------------------------------------------- per-step prologue + epilogue (128 threads)
        const int pt = threadIdx.x - kEpi0 * 32, ew = pt >> 5;
        const int q = warp & 3;
        const int m = q * 32 + lane;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const int B = g.B, H = (int)g.H, a = g.a;
        const int nd = act_digits(a);
        const int64_t R = g.R;
        const int64_t row = (int64_t)rt * kTcRows + m;
        const uint32_t bstage_s = smem_u32(bstage);
        const uint32_t hbuf_s = smem_u32(hbuf);
        const bool tagx = B == 1;                     // h exchanged as tagged values (below)
        const int cbase = kc * kChunkWords * 32;      // first column of this CTA's K-chunk
        const int cvalid = H - cbase;                 // valid columns of the chunk (may exceed 1024)
        const bool finish = kc == 0;                  // the tile's leader finishes it (the cell)
        pdl_wait();                                   // h0 / c0 / gx come from earlier kernels
        if (pt == 0) bars.epoch0 = grid_base(g.gbar) / kGridStride;
        // tag base of this call: h_t (t >= 1) carries (uint32)(sbase + t); CTA 0 advances the
        // counter by T at its end (after every CTA read it: step 1 needs every tile's step 0)
        const unsigned long long sbase = ld_acquire_gpu_u64(g.stepctr);
        // diagnostics: 3 records per step at indices reserved once (no atomic inside the steps)
        long long* tlb = nullptr;
        if (g.tl && pt == 0) {
            const unsigned long long i0 = atomicAdd(reinterpret_cast<unsigned long long*>(g.tl), 4ull * T);
            if (i0 + 4ull * T <= (unsigned long long)kTlRecords) tlb = g.tl + 10 + 10 * (long long)i0;
        }
        // the cell state of the leader's 32 hidden units stays in SMEM across timesteps
        if (finish && (lane & 3) == 0 && row < R)
            for (int b = 0; b < B; ++b) cst[b * 32 + (m >> 2)] = g.c0[(int64_t)b * H + (row >> 2)];
        for (int t = 0; t < T; ++t) {
            const int par = t & 1;
            if (finish && p.chunks > 1 && pt == 0)                 // this step's partial sums from the others
                mbar_arrive_expect_tx(&bars.red_full, (uint32_t)((p.chunks - 1) * B * kTcRows * 8));
            long long tm[6] = {0, 0, 0, 0, 0, 0};
            long long ck[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
            long long cgx = 0, cfin[3] = {0, 0, 0};
            if (g.tl) tm[0] = gtimer();
            // ---- a1: f_b from max|h_t[b,:]| (reading G8).  Step 0 reads all of h0.  For t > 0 the
            //      CTAs that produced h_t published its maxima: B = 1 per-tile tagged slots, read
            //      together with the chunk's tagged h values (one L2 round trip, no barrier);
            //      B > 1 epoch-tagged atomicMax slots behind the grid barrier (warp 2)
            float hv0[8];                              // B = 1: this thread's 8 values of h_t
            if (t == 0) {
                for (int b = 0; b < B; ++b) {
                    const float4* x4 = reinterpret_cast<const float4*>(g.h0 + (int64_t)b * H);
                    float mx = 0.f;
                    for (int c = pt; c < H / 4; c += 128) {
                        const float4 v = __ldcg(x4 + c);
                        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
                    }
#pragma unroll
                    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                    if (lane == 0) bars.red[ew][b] = mx;
                }
                if (tagx) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const int cl = (ew + kEpiWarps * k) * 32 + lane;
                        hv0[k] = cl < cvalid ? __ldcg(g.h0 + cbase + cl) : 0.f;
                    }
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (pt < B) {
                    float mx = bars.red[0][pt];
#pragma unroll
                    for (int w = 1; w < kEpiWarps; ++w) mx = fmaxf(mx, bars.red[w][pt]);
                    bars.f[0][pt] = act_frac_of(mx, a);
                    bars.sc[0][pt] = col_scale(g.scale, bars.f[0][pt]);
                    const int f = bars.f[0][pt];
                    bars.scl[0][pt] = (f >= -126 && f <= 127) ? __int_as_float((127 + f) << 23) : 0.f;
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
            } else if (p.helpers) {
                // the converter warps poll h_t and build the digits; here: the tiles' max slots
                const uint32_t tag = (uint32_t)(sbase + (unsigned long long)t);
                const unsigned long long* sl = g.mxs + ((int64_t)par * gridDim.x + blockIdx.x) * kLstmMaxTiles;
                unsigned long long sv = (unsigned long long)tag << 32;
                if (pt < p.tiles) {
                    sv = ld_relaxed_gpu_u64(sl + pt);
                    while ((uint32_t)(sv >> 32) != tag) sv = ld_relaxed_gpu_u64(sl + pt);
                }
                const float mx = __uint_as_float(__reduce_max_sync(0xffffffffu, (uint32_t)sv));
                if (lane == 0) bars.red[ew][0] = mx;
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (pt == 0) {
                    const float m4 = fmaxf(fmaxf(bars.red[0][0], bars.red[1][0]), fmaxf(bars.red[2][0], bars.red[3][0]));
                    const int f = act_frac_of(m4, a);
                    bars.f[par][0] = f;
                    bars.sc[par][0] = col_scale(g.scale, f);
                    bars.scl[par][0] = (f >= -126 && f <= 127) ? __int_as_float((127 + f) << 23) : 0.f;
                }
                if (g.tl) {
                    tm[4] = gtimer();
                    tm[5] = 1;
                }
                asm volatile("barrier.sync 2, 384;" ::: "memory");   // f_b to the converter warps (non-aligned)
            } else if (tagx) {
                const uint32_t tag = (uint32_t)(sbase + (unsigned long long)t);
                const unsigned long long* hx = g.hx + (int64_t)par * H + cbase;
                // this CTA's mailbox: one tagged max|h_t| per tile, written by the tiles' leaders
                const unsigned long long* sl = g.mxs + ((int64_t)par * gridDim.x + blockIdx.x) * kLstmMaxTiles;
                // warp 0 polls the tiles' slots (2 per lane); then every thread loads its 8 values
                // once (written before the slots; re-polled only if a tag is still old)
                unsigned long long hv[8], sv = (unsigned long long)tag << 32;
                int rounds = 0;
                if (ew == 0) {
                    unsigned long long s0, s1;
                    bool ok;
                    do {
                        ++rounds;
                        s0 = lane < p.tiles ? ld_relaxed_gpu_u64(sl + lane) : (unsigned long long)tag << 32;
                        s1 = lane + 32 < p.tiles ? ld_relaxed_gpu_u64(sl + lane + 32) : (unsigned long long)tag << 32;
                        ok = (uint32_t)(s0 >> 32) == tag && (uint32_t)(s1 >> 32) == tag;
                    } while (!__all_sync(0xffffffffu, ok));
                    sv = __uint_as_float((uint32_t)s0) > __uint_as_float((uint32_t)s1) ? s0 : s1;
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int cl = (ew + kEpiWarps * k) * 32 + lane;
                    hv[k] = cl < cvalid ? ld_relaxed_gpu_u64(hx + cl) : (unsigned long long)tag << 32;
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int cl = (ew + kEpiWarps * k) * 32 + lane;
                    while ((uint32_t)(hv[k] >> 32) != tag) hv[k] = ld_relaxed_gpu_u64(hx + cl);
                }
                if (g.tl) {
                    tm[4] = gtimer();
                    tm[5] = rounds;
                }
                float mx = __uint_as_float((uint32_t)sv);
#pragma unroll
                for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                if (lane == 0) bars.red[ew][0] = mx;
#pragma unroll
                for (int k = 0; k < 8; ++k) hv0[k] = __uint_as_float((uint32_t)hv[k]);
                asm volatile("bar.sync 1, 128;" ::: "memory");
                mx = fmaxf(fmaxf(bars.red[0][0], bars.red[1][0]), fmaxf(bars.red[2][0], bars.red[3][0]));
                const int f = act_frac_of(mx, a);
                if (pt == 0) {
                    bars.f[par][0] = f;
                    bars.sc[par][0] = col_scale(g.scale, f);
                    bars.scl[par][0] = (f >= -126 && f <= 127) ? __int_as_float((127 + f) << 23) : 0.f;
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
            }
            if (!tagx) mbar_wait(&bars.h_full, (uint32_t)(t & 1));
            if (g.tl) tm[1] = gtimer();
            if (g.tl) ck[0] = clock64();
            // ---- a1-a2: the digits of this CTA's chunk into the B operand.  One round = the 32
            //      words of batch column b (warp ew takes words ew, ew + 4, ...): 8 independent
            //      casts and transposes per warp, no branches inside the round
            // the exact fp32 cast of act_cast (pb_common.cuh) when every f_b of the step is in range
            bool fast = a <= 24;
            for (int b = 0; b < B && fast; ++b) fast = bars.scl[par][b] != 0.f;
            const float lim = (float)(1 << ((a <= 24 ? a : 24) - 1));
            const bool shfl_digits = !(a & 1) && a <= 16;
            const uint32_t amask = a >= 32 ? ~0u : ((1u << a) - 1u);
            static_assert(kEpiWarps * 8 == kChunkWords, "a round covers one batch column");
            const bool helped = p.helpers && t > 0;       // the converter warps built the digits
#pragma unroll 1
            for (int b = 0; b < (helped ? 0 : B); ++b) {
                uint32_t u[8];
                float v[8];
                if (tagx) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) v[k] = hv0[k];
                } else {
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const int cl = (ew + kEpiWarps * k) * 32 + lane;
                        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[k]) : "r"(hbuf_s + (uint32_t)((b * kChunkWords * 32 + cl) * 4)));
                        v[k] = cl < cvalid ? v[k] : 0.f;      // stale SMEM past the copied columns
                    }
                }
                if (fast) {
                    const float sc = bars.scl[par][b];
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        u[k] = (uint32_t)__float2int_rz(fminf(fmaxf(v[k] * sc, -lim), lim - 1.0f));
                } else {
                    const int f = bars.f[par][b];
#pragma unroll   // (indexed registers: no local-memory array)
                    for (int k = 0; k < 8; ++k) u[k] = (uint32_t)act_cast(v[k], f, a);
                }
                if (g.tl && b == 0) {
                    uint32_t z = 0;
#pragma unroll
                    for (int k = 0; k < 8; ++k) z |= u[k];
                    asm volatile("" ::"r"(z));
                    ck[8] = clock64();
                }
                if (shfl_digits) {
                    // even a <= 16: per-lane digit nibbles + a nibble transpose (no ballots)
                    uint32_t reg[8];
                    int dk = 0;
#pragma unroll
                    for (int k = 0; k < 8; ++k) reg[k] = digit_regs_shfl(u[k] & amask, a, lane, dk);
                    if (dk < nd) {
#pragma unroll
                        for (int k = 0; k < 8; ++k)
                            asm volatile("st.shared.u32 [%0], %1;" ::"r"(bstage_s + b_operand_offset(NPAD, ew + kEpiWarps * k, b * nd + dk, lane & 3)),
                                         "r"(reg[k]) : "memory");
                    }
                } else {
                    uint32_t mm[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) mm[k] = 0;
#pragma unroll 1
                    for (int j = 0; j < a; ++j) {
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const uint32_t w = __ballot_sync(0xffffffffu, (u[k] >> (a - 1 - j)) & 1u);
                            if (lane == j) mm[k] = w;
                        }
                    }
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        uint4 dv;
                        if (digit_of_lane(mm[k], lane, a, dv))
                            put_b_operand_smem(bstage_s, NPAD, ew + kEpiWarps * k, b * nd + (lane >> 1), dv);
                    }
                }
            }
            if (B * nd < NPAD && !helped) {                    // zero digit rows past the batch
#pragma unroll 1
                for (int k = 0; k < 8; ++k)
                    for (int n = B * nd + lane; n < NPAD; n += 32)
                        put_b_operand_smem(bstage_s, NPAD, ew + kEpiWarps * k, n, make_uint4(0, 0, 0, 0));
            }
            if (g.tl) ck[1] = clock64();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic SMEM writes -> MMA
            if (helped)
                asm volatile("barrier.sync 3, 384;" ::: "memory");           // the converter warps' digits
            else
                asm volatile("bar.sync 1, 128;" ::: "memory");
            if (g.tl) ck[2] = clock64();
            if (pt == 0) {
                mbar_arrive(&bars.b_full);
                mbar_arrive(&bars.h_empty);
            }
            if (g.tl) tm[2] = gtimer();
            // ---- a3-a4 done: drain D into exact per-row sums per batch column (s_tot)
            mbar_wait(&bars.d_full, (uint32_t)(t & 1));
            tc_fence_after();
            if (g.tl) tm[3] = gtimer();
            if (g.tl) ck[3] = clock64();
            unsigned long long tot1 = 0;
            for (int r = 0; r < p.regions; ++r) {
                int last = (r + 1) * p.Gp - 1;
                if (last > p.passes - 1) last = p.passes - 1;
                const unsigned long long wr = layer_mag(g.L, g.offset, pass_lo(g.k_used, last));
                const uint32_t dreg = tmem + lane_off + (uint32_t)(p.d_col + r * NPAD);
                if (!kWide && B == 1) {
                    uint32_t dv[NPAD];
                    ld_tmem_cols<NPAD>(dreg, dv);
                    tmem_ld_wait();
                    unsigned long long hh = d2i(dv[0]);
#pragma unroll
                    for (int e = 1; e < NPAD; ++e) {
                        const int sh = (e == nd - 1 && (a & 1)) ? 1 : 2;
                        hh = (e < nd) ? (hh << sh) + d2i(dv[e]) : hh;
                    }
                    tot1 += hh * wr;
                } else if (!plane_sums_dispatch<NPAD>(a, dreg, B, m, s_tot_s, wr, r == 0)) {
                    // any other a: serial digit Horner per batch column
                    constexpr int kCG = NPAD < 32 ? NPAD : 32;
                    unsigned long long hh = 0;
                    int j = 0, bc = 0;
                    for (int c0 = 0; c0 < NPAD && bc < B; c0 += kCG) {
                        uint32_t dv[kCG];
                        ld_tmem_cols<kCG>(dreg + (uint32_t)c0, dv);
                        tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < kCG; ++e)
                            if (bc < B) {
                                const int sh = (j == nd - 1 && (a & 1)) ? 1 : 2;
                                hh = j == 0 ? d2i(dv[e]) : (hh << sh) + d2i(dv[e]);
                                if (++j == nd) {
                                    const uint32_t sa = s_tot_s + (uint32_t)(bc * kTcRows + m) * 8u;
                                    st_shared_u64(sa, r == 0 ? hh * wr : hh * wr + ld_shared_u64(sa));
                                    j = 0;
                                    ++bc;
                                }
                            }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars.d_empty);
            if (g.tl) ck[4] = clock64();
            auto tot_of = [&](int b) -> unsigned long long {
                return (!kWide && B == 1) ? tot1 : ld_shared_u64(s_tot_s + (uint32_t)(b * kTcRows + m) * 8u);
            };
            // ---- a5: a tile's K-chunks are the CTAs of one cluster: the others put their exact
            //      partial sums into the leader's SMEM (DSMEM) and the leader finishes the tile
            if (!finish) {
                // every thread's sums go with their byte count to the leader's barrier (st.async)
                const uint32_t rb = mapa_shared(redbuf_s + (uint32_t)(((kc - 1) * B * kTcRows + m) * 8), 0);
                const uint32_t rbar = mapa_shared(smem_u32(&bars.red_full), 0);
                for (int b = 0; b < B; ++b)
                    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(
                                     rb + (uint32_t)(b * kTcRows * 8)),
                                 "l"(tot_of(b)), "r"(rbar)
                                 : "memory");
            } else if (p.chunks > 1) {
                mbar_wait_cluster(&bars.red_full, (uint32_t)(t & 1));
            }
            if (g.tl) ck[5] = clock64();
            if (finish) {
                float* h_out = g.h_seq + (int64_t)t * B * H;
                const uint32_t tag1 = (uint32_t)(sbase + (unsigned long long)t + 1);   // tag of h_{t+1}
                unsigned long long* hx1 = g.hx + (int64_t)((t + 1) & 1) * H;
                mbar_wait(&bars.gx_full[t & 1], (uint32_t)((t >> 1) & 1));
                if (g.tl) ck[6] = clock64();
                if (g.tl) cgx = ck[6];
                long long cf[3] = {0, 0, 0};
                for (int b = 0; b < B; ++b) {
                    unsigned long long tt = tot_of(b);
                    for (int r = 1; r < p.chunks; ++r)
                        tt += ld_shared_u64(redbuf_s + (uint32_t)((((r - 1) * B + b) * kTcRows + m) * 8));
                    const float v = row < R ? dequant_sc((long long)tt, bars.sc[par][b]) + gxbuf[(par * B + b) * kTcRows + m] : 0.f;
                    if (g.tl && b == 0) {
                        asm volatile("" ::"f"(v));
                        cf[0] = clock64();
                    }
                    // each gate lane applies its own nonlinearity (tanh for g, sigmoid else), then
                    // the unit's lane gathers the four activations
                    const float act = (lane & 3) == 2 ? tanhf(v) : sigmoidf_(v);
                    const int q0 = lane & ~3;
                    const float si = __shfl_sync(0xffffffffu, act, q0), sf = __shfl_sync(0xffffffffu, act, q0 + 1);
                    const float tg = __shfl_sync(0xffffffffu, act, q0 + 2), so = __shfl_sync(0xffffffffu, act, q0 + 3);
                    float hn = 0.f;
                    if ((lane & 3) == 0 && row < R) {
                        const int64_t i = (int64_t)b * H + (row >> 2);
                        float cn;
                        lstm_cell_act(si, sf, tg, so, cst[b * 32 + (m >> 2)], hn, cn);
                        cst[b * 32 + (m >> 2)] = cn;
                        if (tagx && t + 1 < T)
                            st_relaxed_gpu_u64(hx1 + (row >> 2), ((unsigned long long)tag1 << 32) | __float_as_uint(hn));
                        h_out[i] = hn;
                        if (g.c_seq) g.c_seq[(int64_t)t * B * H + i] = cn;
                        if (t == T - 1) g.c_last[i] = cn;
                    }
                    if (g.tl && b == 0) {
                        asm volatile("" ::"f"(hn));
                        cf[1] = clock64();
                    }
                    // max|h_{t+1}[b,:]| over this warp's 8 hidden units -> step t+1's f_b (non-negative
                    // floats order as their bit patterns: one redux)
                    const float mh = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(fabsf(hn))));
                    if (g.tl && b == 0) {
                        asm volatile("" ::"f"(mh));
                        cf[2] = clock64();
                        cfin[0] = cf[0];
                        cfin[1] = cf[1];
                        cfin[2] = cf[2];
                    }
                    if (lane == 0 && t + 1 < T) {
                        if (tagx)
                            bars.pmax[par][ew] = mh;
                        else
                            atomicMax(g.maxslot + (((t + 1) & 1) * kLstmMaxB + b),
                                      ((bars.epoch0 + (unsigned long long)t + 1) << 32) | __float_as_uint(mh));
                    }
                }
            }
            // ---- publish h_{t+1}.  B = 1: the tile's max|h| slot after the 4 warps' maxima; B > 1:
            //      every CTA arrives at the grid barrier (the 128 threads' stores are ordered before
            //      thread 0's release by bar.sync)
            if (g.tl) ck[7] = clock64();
            if (!tagx || finish) asm volatile("bar.sync 1, 128;" ::: "memory");
            if (!tagx) {
                if (pt == 0) grid_arrive(g.gbar);
            } else if (finish && t + 1 < T) {
                // every CTA's mailbox slot of this tile (distinct lines per reader: no polled hot spot)
                const float mh = fmaxf(fmaxf(bars.pmax[par][0], bars.pmax[par][1]), fmaxf(bars.pmax[par][2], bars.pmax[par][3]));
                const unsigned long long sv = ((unsigned long long)(uint32_t)(sbase + (unsigned long long)t + 1) << 32) | __float_as_uint(mh);
                for (int i = pt; i < (int)gridDim.x; i += 128)
                    st_relaxed_gpu_u64(g.mxs + ((int64_t)((t + 1) & 1) * gridDim.x + i) * kLstmMaxTiles + rt, sv);
                if (g.tl && pt == 0) ck[6] = gtimer();
            }
            if (tlb) {
                long long* rr = tlb + 40 * t;
                const long long rec[40] = {7, blockIdx.x, t, tm[0], tm[1], tm[2], tm[3], finish ? 1 : 0, gtimer(), 0,
                                           8, blockIdx.x, t, ck[1] - ck[0], ck[2] - ck[0], ck[3] - ck[0], ck[4] - ck[0],
                                           ck[5] - ck[0], ck[8] - ck[0], ck[7] - ck[0],
                                           9, blockIdx.x, t, tm[4], tm[5], finish ? ck[6] : 0, 0, 0, 0, 0,
                                           10, blockIdx.x, t, cgx - ck[0], cfin[0] - ck[0], cfin[1] - ck[0], cfin[2] - ck[0], 0, 0, 0};
#pragma unroll
                for (int k = 0; k < 40; ++k) rr[k] = rec[k];
            }
        }
        // the next call's tags start past this call's: CTA 0 advances the step counter
        if (blockIdx.x == 0 && pt == 0) asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(g.stepctr), "l"((unsigned long long)T) : "memory");
    }
    tc_fence_before();
    cluster_sync();                                // no CTA leaves while its SMEM may be written
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// SMEM besides the weight ring: header, B stage, per-row sums, the K-chunk of h_t, and the
// leader's buffer for the other chunks' partial sums.
uint32_t lstm_fixed_smem(int B, int npad, int chunks) {
    return 1024 + kHdrBytes + (uint32_t)(kChunkWords / 2) * npad * 32 + (uint32_t)B * kTcRows * 8 +
           (uint32_t)B * kChunkWords * 32 * 4 + (uint32_t)(chunks - 1) * B * kTcRows * 8 + 2u * B * kTcRows * 4 +
           (uint32_t)B * 32 * 4;
}

// Comparison knob: NAME=0 disables a default-on mode.
bool getenv_flag_off(const char* name) {
    const char* ev = getenv(name);
    return ev && ev[0] == '0';
}

bool make_lplan(const LstmArgs& g, int npad, int sms, LPlan& p)
{
    if (g.B < 1 || g.B > kLstmMaxB || g.T < 1 || g.L < 1 || g.L > 16 || g.H % 4 || g.R != 4 * g.H) return false;
    if ((int64_t)g.B * act_digits(g.a) > npad) return false;
    p.tiles = (int)((g.R + kTcRows - 1) / kTcRows);
    p.chunks = (int)((g.kwords + kChunkWords - 1) / kChunkWords);
    if ((int64_t)p.tiles * p.chunks > sms) return false;       // one unit per CTA, all co-resident
    if (p.tiles > kLstmMaxTiles || p.tiles * p.chunks > kLstmMaxCtas) return false;   // mailbox slots
    if (p.chunks > 8) return false;                             // a tile's chunks form one (portable) cluster
    p.Gp = tc_group_passes(g.kwords);
    if (p.Gp < 1) return false;
    p.passes = (g.k_used + 1) / 2;
    p.regions = (p.passes + p.Gp - 1) / p.Gp;
    p.d_col = 512 - (p.regions * npad + 31) / 32 * 32;          // one accumulator set
    p.sf_col = p.d_col - 64;
    p.slots = p.sf_col / 128;
    if (p.slots > kMaxSlots) p.slots = kMaxSlots;
    if (p.slots < 2) return false;
    // A of every pass resident (converted once, at step 0) when it fits the A ring
    p.resident = (p.passes <= p.slots && !getenv_flag_off("PB_LSTM_RESIDENT")) ? 1 : 0;
    p.spass = 0;
    if (!p.resident && p.passes - p.slots <= kMaxSPass && !getenv_flag_off("PB_LSTM_RESIDENT") &&
        !getenv_flag_off("PB_LSTM_SMEM_A")) {
        p.resident = 1;                                         // the last passes' A in SMEM
        p.spass = p.passes - p.slots;
    }
    if (p.resident && !p.spass) p.slots = p.passes;
    p.helpers = (p.resident && g.B == 1 && !(g.a & 1) && g.a <= 16 && !getenv_flag_off("PB_LSTM_HELPERS")) ? 1 : 0;
    p.wstages = (int)((kSmemMax - lstm_fixed_smem(g.B, npad, p.chunks)) / kWTileBytes) - 4 * p.spass;
    if (p.wstages > kMaxWStages) p.wstages = kMaxWStages;
    // >= 4: the two converter h-sets wait on the tiles of consecutive passes (2 tiles each); with
    // fewer stages a parity wait could see a barrier two phases behind it
    return p.wstages >= 4;
}

std::mutex g_lmu;
bool g_lattr[64][5];

template <int NPAD>
cudaError_t launch_lt(const LstmArgs& g, cudaStream_t s)
{
    int dev = 0, sms = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    LPlan p;
    if (!make_lplan(g, NPAD, sms, p)) return cudaErrorNotSupported;
    constexpr int ai = NPAD == 8 ? 0 : (NPAD == 16 ? 1 : (NPAD == 32 ? 2 : (NPAD == 64 ? 3 : 4)));
    if (dev >= 0 && dev < 64 && !g_lattr[dev][ai]) {
        std::lock_guard<std::mutex> lk(g_lmu);
        e = cudaFuncSetAttribute(lstm_persist_kernel<NPAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax);
        if (e != cudaSuccess) return e;
        g_lattr[dev][ai] = true;
    }
    GemmArgs ga{};
    ga.bits = g.bits;
    ga.R = g.R;
    ga.kwords = g.kwords;
    ga.L = g.L;
    CUtensorMap pmap, smap;
    if ((e = tc_weight_maps(ga, &pmap, &smap)) != cudaSuccess) return e;
    const uint32_t smem = lstm_fixed_smem(g.B, NPAD, p.chunks) + (uint32_t)(p.wstages + 4 * p.spass) * kWTileBytes;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(p.tiles * p.chunks), 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute la[2];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = 1;
    la[1].id = cudaLaunchAttributeClusterDimension;             // a tile's K-chunks: one cluster
    la[1].val.clusterDim.x = (unsigned)p.chunks;
    la[1].val.clusterDim.y = 1;
    la[1].val.clusterDim.z = 1;
    cfg.attrs = la;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, lstm_persist_kernel<NPAD>, g, p, pmap, smap);
}

}  // namespace

int lstm_persist_npad(int64_t batch, int32_t a) {
    const int64_t n = batch * act_digits(a);
    if (batch < 1 || batch > kLstmMaxB || a < 1 || a > 32 || n > kTcWideN) return 0;
    return n <= 8 ? 8 : (n <= 16 ? 16 : (n <= 32 ? 32 : (n <= 64 ? 64 : kTcWideN)));
}

bool lstm_persist_supported(const LstmArgs& g)
{
    const int npad = lstm_persist_npad(g.B, g.a);
    if (!npad) return false;
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return false;
    LPlan p;
    return make_lplan(g, npad, sms, p);
}

cudaError_t launch_lstm_persist(const LstmArgs& g, cudaStream_t s)
{
    switch (lstm_persist_npad(g.B, g.a)) {
        case 8: return launch_lt<8>(g, s);
        case 16: return launch_lt<16>(g, s);
        case 32: return launch_lt<32>(g, s);
        case 64: return launch_lt<64>(g, s);
        case kTcWideN: return launch_lt<kTcWideN>(g, s);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace pb
