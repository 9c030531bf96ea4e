// pb_act.cu -- steps a1 + a2 of the hot path on sm_100a:
//   a1 activation fixed-point cast  x_q = trunc(x * 2^f_b)   (Alg. 2 line 1, P:195;
//      P:154 "a multiplication and a cast"; f_b per reading G8)
//   a2 bitwise transpose of x_q into activation bitplanes
// One warp turns 32 consecutive columns into `a` plane words with `a`
// __ballot_sync votes (VOTE.ANY), sign plane first.  Σ_c x_q (needed only for
// the binary-mode offset term) is produced as per-CTA partial sums.
// When the tensor engine is used (a*B <= 32) the kernel also emits the MMA
// B operand (tcgen05 kind::mxf4, packed e2m1, K-major no-swizzle canonical
// layout): per 2 words (64 columns) one N_pad x 32-byte tile.  The 16 bytes
// of word w in plane row n are 4 uint32 (r = 0..3) whose nibble e holds
// X_n bit (4e + r) as the e2m1 code 2.0 (0b0100); against a weight nibble
// 1.0 * hi_bit + 0.5 * lo_bit (pb_gemm_tc.cu) the product is exactly
// (2 hi + lo) * x_bit.  Words in [kwords, roundup(kwords, 32)) -- the K tail
// of the last 32-word chunk -- get zero B so that the chunk tail contributes
// nothing whatever the weight operand holds there.
//
// Grid: (nsplit, B) CTAs of 512 threads.  Every CTA recomputes max|x[b,:]|
// (an L2-resident re-read of K floats) so no second launch or grid sync is
// needed; it then transposes its own slice of words.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "pb_common.cuh"
#include "pb_internal.h"

namespace pb {
namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kActAuto = -1024;   // == PB_ACT_AUTO

__global__ void __launch_bounds__(kThreads)
act_quant_transpose_kernel(const float* __restrict__ x, int64_t K, int64_t kwords, int a,
                           int act_frac, int words_per_cta, int32_t* __restrict__ f_out,
                           long long* __restrict__ xsum_part, uint32_t* __restrict__ planes,
                           uint8_t* __restrict__ bexp, int npad, int bs, size_t slice_bytes, long long* tl)
{
    long long t_launch = 0, t_go = 0;
    if (tl) t_launch = gtimer();
    pdl_wait();          // x may be the previous kernel's output
    if (tl) t_go = gtimer();
    pdl_trigger();       // let the dependent GEMV start its prologue

    const int b = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float* xb = x + (int64_t)b * K;

    // ---- a1 (part 1): column max |x| (order-independent, exact) ----
    float m = 0.f;
    if ((K & 3) == 0 && ((reinterpret_cast<uintptr_t>(xb) & 15) == 0)) {
        // issue 8 independent 128-bit loads per thread before using any
        const float4* x4 = reinterpret_cast<const float4*>(xb);
        const int64_t n4 = K / 4;
        for (int64_t c0 = tid; c0 < n4; c0 += 8 * kThreads) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t c = c0 + (int64_t)u * kThreads;
                v[u] = c < n4 ? __ldg(x4 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
                m = fmaxf(m, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
        }
    } else {
        for (int64_t c = tid; c < K; c += kThreads) m = fmaxf(m, fabsf(__ldg(xb + c)));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ float s_max[kWarps];
    __shared__ long long s_sum[kWarps];
    if (lane == 0) s_max[warp] = m;
    __syncthreads();
    m = s_max[0];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) m = fmaxf(m, s_max[w]);

    const int f = (act_frac == kActAuto) ? act_frac_of(m, a) : act_frac;
    if (blockIdx.x == 0 && tid == 0) f_out[b] = f;

    // ---- a1 (part 2) + a2: cast, saturate, ballot-transpose ----
    int64_t w0 = (int64_t)blockIdx.x * words_per_cta;
    int64_t w1 = w0 + words_per_cta;
    if (w1 > kwords) w1 = kwords;
    if (npad && blockIdx.x == gridDim.x - 1) {
        // zero B for the chunk tail [kwords, roundup(kwords, 32)); with a capped split the
        // last CTA's own range may start beyond kwords, so it starts at min(w0, kwords)
        if (w0 > kwords) w0 = kwords;
        w1 = (kwords + 31) / 32 * 32;
    }
    uint32_t* pb = planes + (int64_t)b * a * kwords;
    long long xs = 0;
    for (int64_t w = w0 + warp; w < w1; w += kWarps) {
        const int64_t c = 32 * w + lane;
        const float v = c < K ? __ldg(xb + c) : 0.f;
        const long long q = act_cast(v, f, a);
        xs += q;
        uint32_t mine = 0;
        for (int j = 0; j < a; ++j) {
            const uint32_t word = __ballot_sync(0xffffffffu, (unsigned)((q >> (a - 1 - j)) & 1));
            if (lane == j) mine = word;
        }
        if (lane < a && w < kwords) pb[(int64_t)lane * kwords + w] = mine;
        if (npad) {
            // lane 2k < a writes digit row n = b_local*nd + k of the column's slice (wide mode:
            // slices of bs columns, slice-major; narrow: one slice); the slice's last column
            // zeroes its padding rows [nd*nb, npad)
            const int nd = act_digits(a);
            const int sl = b / bs, bl = b - sl * bs;
            const int nb = (int)gridDim.y - sl * bs < bs ? (int)gridDim.y - sl * bs : bs;
            uint8_t* bx = bexp + (size_t)sl * slice_bytes;
            uint4 dv;
            if (digit_of_lane(mine, lane, a, dv)) put_b_operand(bx, npad, w, bl * nd + (lane >> 1), dv);
            if (bl == nb - 1)
                for (int n = nb * nd + lane; n < npad; n += 32) put_b_operand(bx, npad, w, n, make_uint4(0, 0, 0, 0));
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) xs += __shfl_xor_sync(0xffffffffu, xs, o);
    if (lane == 0) s_sum[warp] = xs;
    __syncthreads();
    if (tid == 0) {
        long long t = 0;
        for (int w = 0; w < kWarps; ++w) t += s_sum[w];
        xsum_part[(int64_t)b * kXsumStride + blockIdx.x] = t;
        if (tl) {
            long long* r = tl_record(tl);
            if (r) {
                unsigned smid;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                const long long rec[10] = {0, blockIdx.x + (long long)blockIdx.y * gridDim.x, smid, 0, t_launch, t_go,
                                           gtimer(), 0, 0, 0};
                for (int k = 0; k < 10; ++k) r[k] = rec[k];
            }
        }
    }
}

}  // namespace

// Diagnostics timeline buffer (pb_debug_timeline): allocated at the first
// launch when PB_TC_DEBUG=6, else null.
long long* debug_tl() {
    static int state = 0;          // 0 = unknown, 1 = off, 2 = on
    static long long* buf = nullptr;
    if (state == 0) {
        const char* ev = getenv("PB_TC_DEBUG");
        state = 1;
        if (ev && atoi(ev) >= 6 &&
            cudaMalloc(&buf, sizeof(long long) * (size_t)(10 + 10 * kTlRecords)) == cudaSuccess &&
            cudaMemset(buf, 0, sizeof(long long) * 10) == cudaSuccess)
            state = 2;
    }
    return state == 2 ? buf : nullptr;
}

cudaError_t launch_act_quant(const float* x, int64_t B, int64_t K, int64_t kwords, int a,
                             int act_frac, void* ws, const WsLayout& l, cudaStream_t s)
{
    if (B == 0 || kwords == 0) return cudaSuccess;
    static bool carveout[64] = {};                // per device (a function attribute is per context)
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && dev >= 0 && dev < 64 && !carveout[dev]) {
        // keep the SM in its max-shared-memory configuration between this kernel and
        // the tensor-engine GEMM (which needs 162 KiB): no L1/SMEM repartition per launch
        cudaFuncSetAttribute(act_quant_transpose_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                             (int)cudaSharedmemCarveoutMaxShared);
        carveout[dev] = true;
    }
    char* base = static_cast<char*>(ws);
    const int nsplit = act_nsplit(kwords);
    const int wpc = (int)((kwords + nsplit - 1) / nsplit);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nsplit, (unsigned)B, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // tensor-engine operand tiles: the narrow layout when the whole batch is one launch's
    // slice, else the wide slice-major layout, else none (POPC engine planes only)
    int npad = 0, bs = (int)B;
    size_t slice_bytes = 0;
    if (l.npad && tc_npad(B, a) == l.npad) {
        npad = l.npad;
    } else if (l.wbs) {
        npad = kTcWideN;
        bs = l.wbs;
        slice_bytes = l.wslice_bytes;
    }
    return cudaLaunchKernelEx(&cfg, act_quant_transpose_kernel, x, K, kwords, a, act_frac, wpc,
                              reinterpret_cast<int32_t*>(base + l.off_f),
                              reinterpret_cast<long long*>(base + l.off_xsum),
                              reinterpret_cast<uint32_t*>(base + l.off_planes),
                              reinterpret_cast<uint8_t*>(base + l.off_bexp), npad, bs, slice_bytes, debug_tl());
}

}  // namespace pb
