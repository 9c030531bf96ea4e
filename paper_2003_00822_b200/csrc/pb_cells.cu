// pb_cells.cu -- elementwise tails of the layer helpers and the row-shard
// permute.  fp32, CUDA cores, coalesced.
//   LSTM (reading G15, PyTorch nn.LSTM gate order i, f, g, o):
//     c' = sigmoid(f) * c + sigmoid(i) * tanh(g);  h' = sigmoid(o) * tanh(c')
//   RNN:  h' = tanh(gates)
#include <cstdint>
#include <cuda_runtime.h>

#include "pb_common.cuh"
#include "pb_internal.h"

namespace pb {
namespace {


__global__ void lstm_cell_kernel(const float* __restrict__ gates, const float* __restrict__ c,
                                 int64_t B, int64_t H, float* __restrict__ h_out,
                                 float* __restrict__ c_out)
{
    pdl_wait();
    const int64_t n = B * H;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t / H, k = t - b * H;
        const float* g = gates + b * 4 * H;
        float hn, cn;
        lstm_cell(g[k], g[H + k], g[2 * H + k], g[3 * H + k], c[t], hn, cn);
        c_out[t] = cn;
        h_out[t] = hn;
    }
}

// Gate-interleaved pre-activations (pb_lstm_seq: row 4k + gate), [B][H][4].
__global__ void lstm_cell_ilv_kernel(const float* __restrict__ gates, const float* __restrict__ c,
                                     int64_t B, int64_t H, float* __restrict__ h_out,
                                     float* __restrict__ c_out)
{
    pdl_wait();
    const int64_t n = B * H;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const float4 g = reinterpret_cast<const float4*>(gates)[t];
        float hn, cn;
        lstm_cell(g.x, g.y, g.z, g.w, c[t], hn, cn);
        c_out[t] = cn;
        h_out[t] = hn;
    }
}

__global__ void rnn_cell_kernel(const float* __restrict__ gates, int64_t n, float* __restrict__ h_out)
{
    pdl_wait();
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x)
        h_out[t] = tanhf(gates[t]);
}

// gathered [N][B][Rs] -> y [B][R], dropping the padding rows of the last shards.
__global__ void permute_shards_kernel(const float* __restrict__ gathered, int64_t B, int64_t Rs,
                                      int nranks, int64_t R, float* __restrict__ y)
{
    const int64_t n = B * R;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t / R, r = t - b * R;
        const int64_t g = r / Rs, rr = r - g * Rs;
        y[t] = gathered[(g * B + b) * Rs + rr];
    }
}

unsigned grid_for(int64_t n, int threads) {
    int64_t g = (n + threads - 1) / threads;
    if (g > 148 * 16) g = 148 * 16;
    if (g < 1) g = 1;
    return (unsigned)g;
}

}  // namespace

cudaError_t launch_lstm_cell(const float* gates, const float* c, int64_t B, int64_t H,
                             float* h_out, float* c_out, cudaStream_t s)
{
    if (B * H == 0) return cudaSuccess;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid_for(B * H, 256));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, lstm_cell_kernel, gates, c, B, H, h_out, c_out);
}

cudaError_t launch_lstm_cell_ilv(const float* gates, const float* c, int64_t B, int64_t H,
                                 float* h_out, float* c_out, cudaStream_t s)
{
    if (B * H == 0) return cudaSuccess;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid_for(B * H, 256));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, lstm_cell_ilv_kernel, gates, c, B, H, h_out, c_out);
}

cudaError_t launch_rnn_cell(const float* gates, int64_t B, int64_t H, float* h_out, cudaStream_t s)
{
    if (B * H == 0) return cudaSuccess;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid_for(B * H, 256));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, rnn_cell_kernel, gates, B * H, h_out);
}

cudaError_t launch_permute_shards(const float* gathered, int64_t B, int64_t rows_per_rank,
                                  int nranks, int64_t R, float* y, cudaStream_t s)
{
    if (B * R == 0) return cudaSuccess;
    permute_shards_kernel<<<grid_for(B * R, 256), 256, 0, s>>>(gathered, B, rows_per_rank, nranks, R, y);
    return cudaGetLastError();
}

}  // namespace pb
