// pb_pack.cu -- step a0 on the GPU: the PB_Q_GRID quantiser and the
// bitlayer packer of pb_api.cpp for a weight matrix already in device memory, so a
// 16384 x 16384 layer packs in milliseconds instead of seconds on the host.
//
// Same arithmetic as the host packer (and the oracle): Q(W) grid step
// d = (max - min) / 2^(L-1) from the exact float extrema (clipping is
// monotonic, so min/max of clip(W) = clip(min/max of W)); code
// m = clamp(rint(clip(W)/d)) in double (IEEE division and rint, ties to even,
// reading G4); layer i = bit L-1-i of the L-bit two's complement (P:137,
// P:175-177, reading G2); paired storage as in include/pb.h.
#include <cstdint>
#include <cuda_runtime.h>

#include "pb_common.cuh"
#include "pb_internal.h"

namespace pb {
namespace {

// per-block float extrema -> out[2*block], out[2*block+1]
__global__ void minmax_kernel(const float* __restrict__ W, int64_t n, float* __restrict__ out)
{
    float mn = INFINITY, mx = -INFINITY;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const float w = W[e];
        mn = fminf(mn, w);
        mx = fmaxf(mx, w);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    __shared__ float smn[32], smx[32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        smn[warp] = mn;
        smx[warp] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            mn = fminf(mn, smn[w]);
            mx = fmaxf(mx, smx[w]);
        }
        out[2 * blockIdx.x] = mn;
        out[2 * blockIdx.x + 1] = mx;
    }
}

__device__ __forceinline__ double clipv(double w, double clip) {
    if (clip > 0) {
        if (w > clip) w = clip;
        if (w < -clip) w = -clip;
    }
    return w;
}

// one thread per (row r, 32-column word c < kw): 32 codes -> L canonical words ->
// paired storage (layers 2p, 2p+1 as (lower, upper) bit pairs of even / odd columns)
__global__ void pack_grid_kernel(const float* __restrict__ W, int64_t R, int64_t K, int64_t kw, int L, double d,
                                 double clip, int all_zero, uint32_t* __restrict__ dst)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= R * kw) return;
    const int64_t r = t / kw, c = t - r * kw;
    const double lo = -ldexp(1.0, L - 1), hi = ldexp(1.0, L - 1) - 1.0;
    uint32_t lay[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) lay[i] = 0u;
    const float* wr = W + r * K;
    for (int j = 0; j < 32; ++j) {
        const int64_t col = 32 * c + j;
        if (col >= K) break;
        double m = rint(clipv((double)wr[col], clip) / d);
        m = m < lo ? lo : (m > hi ? hi : m);
        const uint32_t u = all_zero ? 0u : (uint32_t)(int32_t)m;
#pragma unroll
        for (int i = 0; i < 16; ++i)
            if (i < L) lay[i] |= ((u >> (L - 1 - i)) & 1u) << j;
    }
#pragma unroll
    for (int p = 0; p < 8; ++p) {
        if (2 * p + 1 < L) {
            const uint32_t up = lay[2 * p], low = lay[2 * p + 1];
            uint32_t* row = dst + (int64_t)(2 * p) * R * kw + r * 2 * kw;
            row[2 * c] = (low & 0x55555555u) | ((up & 0x55555555u) << 1);
            row[2 * c + 1] = ((low >> 1) & 0x55555555u) | (up & 0xAAAAAAAAu);
        }
    }
    if (L & 1) {
        uint32_t last = 0u;
#pragma unroll
        for (int i = 0; i < 16; ++i)
            if (i == L - 1) last = lay[i];
        dst[((int64_t)(L - 1) * R + r) * kw + c] = last;
    }
}

}  // namespace

cudaError_t launch_minmax(const float* W, int64_t n, float* partial, int blocks, cudaStream_t s)
{
    minmax_kernel<<<blocks, 256, 0, s>>>(W, n, partial);
    return cudaGetLastError();
}

cudaError_t launch_pack_grid(const float* W, int64_t R, int64_t K, int64_t kw, int L, double d, double clip,
                             int all_zero, uint32_t* dst, cudaStream_t s)
{
    const int64_t n = R * kw;
    if (n == 0) return cudaSuccess;
    pack_grid_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(W, R, K, kw, L, d, clip, all_zero, dst);
    return cudaGetLastError();
}

}  // namespace pb
