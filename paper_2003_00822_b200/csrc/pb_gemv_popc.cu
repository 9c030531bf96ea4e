// pb_gemv_popc.cu -- steps a3 + a4 + a5 on CUDA cores (engine PB_ENGINE_POPC).
//
//   a3  C_ij[r,b] = popc(W_i[r,:] AND X_j[b,:])        (P:120-124, P:205-206:
//       "instead of the xnor operation we use the and operation")
//   a4  acc = sum_{i<k_used} S_i sum_j T_j C_ij + o * sum_c x_q
//   a5  y   = (float) ldexp((double)acc * s_w, -f_b)             (G13)
//
// One warp per output row (grid-stride).  Lanes stream the row's packed
// weight words with coalesced 128-bit non-allocating loads (a stored layer
// pair: 64 columns of both layers per load, de-interleaved into the two layer
// words with 4 logic ops, pb.h) and AND/POPC them against the activation planes,
// which one thread stages into shared memory per CTA with a 1-D TMA bulk
// copy (cp.async.bulk -> UBLKCP) completing on an mbarrier.  Planes are laid
// out [a][kwords] so a lane's LDS.128 hits 4 consecutive banks: conflict-free.
// Per-plane counts stay int32 in registers for one layer, are folded with
// the plane scales T_j into a wrapping 64-bit sum, then weighted by S_i;
// the per-lane partials are reduced with 64-bit warp shuffles.
#include <cstdint>
#include <mutex>
#include <cuda_runtime.h>

#include "pb_common.cuh"
#include "pb_internal.h"

namespace pb {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxDevices = 64;               // per-device launch state
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kMaxSmemPlanes = 160 * 1024;

template <int APAD>
__device__ __forceinline__ void and_popc(const uint4 w, const uint4* __restrict__ P, int64_t kw4,
                                         int64_t v, int a, uint32_t (&cnt)[APAD])
{
#pragma unroll
    for (int j = 0; j < APAD; ++j) {
        if (j < a) {
            const uint4 p = P[j * kw4 + v];
            cnt[j] += __popc(w.x & p.x) + __popc(w.y & p.y) + __popc(w.z & p.z) + __popc(w.w & p.w);
        }
    }
}

template <int APAD, bool use_smem>
__global__ void __launch_bounds__(kThreads)
bitgemv_popc_kernel(const GemmArgs g)
{
    extern __shared__ __align__(16) uint32_t s_planes[];
    __shared__ __align__(8) uint64_t bar;
    const int b = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int a = g.a;
    const int64_t kw4 = g.kwords / 4;
    const uint32_t plane_bytes = (uint32_t)(a * g.kwords * 4);

    if constexpr (use_smem) if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    pdl_wait();          // planes come from the activation kernel
    pdl_trigger();
    if constexpr (use_smem) asm volatile("fence.proxy.async.global;" ::: "memory");   // generic writes -> bulk copy

    const uint32_t* gp = g.planes + (int64_t)b * a * g.kwords;
    if constexpr (use_smem) {
        if (threadIdx.x == 0) {
            mbar_arrive_expect_tx(&bar, plane_bytes);
            constexpr uint32_t kChunk = 32 * 1024;
            for (uint32_t off = 0; off < plane_bytes; off += kChunk) {
                const uint32_t n = plane_bytes - off < kChunk ? plane_bytes - off : kChunk;
                bulk_g2s(reinterpret_cast<char*>(s_planes) + off,
                         reinterpret_cast<const char*>(gp) + off, n, &bar);
            }
        }
        mbar_wait(&bar, 0);
    }
    const uint4* P = reinterpret_cast<const uint4*>(use_smem ? s_planes : gp);
    if constexpr (use_smem) __builtin_assume(__isShared(P));

    for (int64_t r = (int64_t)blockIdx.x * kWarps + warp; r < g.R; r += (int64_t)gridDim.x * kWarps) {
        unsigned long long tot = 0;
        for (int i = 0; i < g.k_used;) {
            if (i + 1 < g.L) {
                // stored pair (i, i+1) (pb.h): one 128-bit load = blocks 2v, 2v+1 of both
                // layers; de-interleave the (lower, upper) bit pairs back into layer words
                const bool use_lo = i + 1 < g.k_used;
                const uint4* prow = reinterpret_cast<const uint4*>(g.bits + ((int64_t)i * g.R + 2 * r) * g.kwords);
                const uint2* P2 = reinterpret_cast<const uint2*>(P);
                const int64_t kw2 = g.kwords / 2;
                uint32_t ch[APAD], cl[APAD];
#pragma unroll
                for (int j = 0; j < APAD; ++j) ch[j] = cl[j] = 0;
                for (int64_t v = lane; v < kw2; v += 32) {
                    const uint4 q = ld_stream_u4(prow + v);
                    const uint32_t lo0 = (q.x & 0x55555555u) | ((q.y << 1) & 0xAAAAAAAAu);
                    const uint32_t hi0 = ((q.x >> 1) & 0x55555555u) | (q.y & 0xAAAAAAAAu);
                    const uint32_t lo1 = (q.z & 0x55555555u) | ((q.w << 1) & 0xAAAAAAAAu);
                    const uint32_t hi1 = ((q.z >> 1) & 0x55555555u) | (q.w & 0xAAAAAAAAu);
#pragma unroll
                    for (int j = 0; j < APAD; ++j) {
                        if (j < a) {
                            const uint2 x = P2[j * kw2 + v];
                            ch[j] += __popc(hi0 & x.x) + __popc(hi1 & x.y);
                            if (use_lo) cl[j] += __popc(lo0 & x.x) + __popc(lo1 & x.y);
                        }
                    }
                }
                unsigned long long sh = 0, sl = 0;
#pragma unroll
                for (int j = 0; j < APAD; ++j)
                    if (j < a) {
                        sh += plane_scale(a, j) * (unsigned long long)ch[j];
                        sl += plane_scale(a, j) * (unsigned long long)cl[j];
                    }
                tot += layer_scale(g.L, g.offset, i) * sh;
                if (use_lo) tot += layer_scale(g.L, g.offset, i + 1) * sl;
                i += 2;
            } else {
                // the canonical last layer of an odd L
                const uint4* wrow = reinterpret_cast<const uint4*>(g.bits + ((int64_t)i * g.R + r) * g.kwords);
                uint32_t cnt[APAD];
#pragma unroll
                for (int j = 0; j < APAD; ++j) cnt[j] = 0;
                int64_t v = lane;
                for (; v + 32 < kw4; v += 64) {
                    const uint4 w0 = ld_stream_u4(wrow + v);
                    const uint4 w1 = ld_stream_u4(wrow + v + 32);
                    and_popc<APAD>(w0, P, kw4, v, a, cnt);
                    and_popc<APAD>(w1, P, kw4, v + 32, a, cnt);
                }
                for (; v < kw4; v += 32) and_popc<APAD>(ld_stream_u4(wrow + v), P, kw4, v, a, cnt);
                unsigned long long s = 0;
#pragma unroll
                for (int j = 0; j < APAD; ++j)
                    if (j < a) s += plane_scale(a, j) * (unsigned long long)cnt[j];
                tot += layer_scale(g.L, g.offset, i) * s;
                i += 1;
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        if (lane == 0) {
            if (g.offset || g.mid) {           // binary offset and / or the midpoint offset
                unsigned long long sx = 0;
                for (int p = 0; p < g.nsplit; ++p) sx += (unsigned long long)g.xsum[(int64_t)b * kXsumStride + p];
                tot += ((unsigned long long)g.offset + g.mid) * sx;
            }
            const long long accv = (long long)tot;
            const int64_t o = (int64_t)b * g.R + r;
            if (g.acc) g.acc[o] = accv;
            float yv = dequant(accv, g.scale, g.f[b]);
            if (g.bias) yv += g.bias[r];
            if (g.accumulate) yv += g.y[o];
            g.y[o] = apply_fn(yv, g.fn);
        }
    }
}

template <int APAD, bool use_smem>
cudaError_t launch_t2(const GemmArgs& g, cudaStream_t s)
{
    const uint32_t plane_bytes = (uint32_t)(g.a * g.kwords * 4);
    const size_t smem = use_smem ? plane_bytes : 0;
    // per-device launch state (the function attribute and the SM count are per device/context;
    // occupancy depends only on the dynamic smem size: the last query is cached)
    struct State {
        bool attr_set = false;
        int sms = 0, occ = 1;
        size_t last_smem = ~size_t(0);
    };
    static State st[kMaxDevices];
    static std::mutex mu;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(mu);
    State& d = st[dev];
    if (!d.attr_set) {
        e = cudaFuncSetAttribute(bitgemv_popc_kernel<APAD, use_smem>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmemPlanes);
        if (e != cudaSuccess) return e;
        if ((e = cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
        d.attr_set = true;
    }
    if (smem != d.last_smem) {
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.occ, bitgemv_popc_kernel<APAD, use_smem>, kThreads, smem);
        if (e != cudaSuccess) return e;
        if (d.occ < 1) d.occ = 1;
        d.last_smem = smem;
    }
    const int sms = d.sms, occ = d.occ;
    int64_t want = (g.R + kWarps - 1) / kWarps;
    int64_t cap = (int64_t)sms * occ / (g.B > 0 ? g.B : 1);
    if (cap < 1) cap = 1;
    const int64_t gx = want < cap ? want : cap;

    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)gx, (unsigned)g.B, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, bitgemv_popc_kernel<APAD, use_smem>, g);
}

template <int APAD>
cudaError_t launch_t(const GemmArgs& g, cudaStream_t s)
{
    const uint32_t plane_bytes = (uint32_t)(g.a * g.kwords * 4);
    return plane_bytes <= kMaxSmemPlanes ? launch_t2<APAD, true>(g, s) : launch_t2<APAD, false>(g, s);
}

}  // namespace

cudaError_t launch_gemv_popc(const GemmArgs& g, cudaStream_t s)
{
    if (g.R == 0 || g.B == 0) return cudaSuccess;
    if (g.a <= 1) return launch_t<1>(g, s);
    if (g.a <= 2) return launch_t<2>(g, s);
    if (g.a <= 4) return launch_t<4>(g, s);
    if (g.a <= 8) return launch_t<8>(g, s);
    if (g.a <= 16) return launch_t<16>(g, s);
    return launch_t<32>(g, s);
}

}  // namespace pb
