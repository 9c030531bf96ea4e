// pb_internal.h -- launchers shared between the host API (pb_api.cpp) and the
// sm_100a kernels (pb_act.cu, pb_gemv_popc.cu, pb_gemm_mma.cu, pb_cells.cu).
// Product code only; nothing here is shared with oracle/.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace pb {

constexpr int kMaxSplit = 64;        // activation kernel CTAs per batch column (max)
constexpr size_t kAlign = 256;

inline size_t align_up(size_t v, size_t a = kAlign) { return (v + a - 1) / a * a; }

// Workspace carve-up (documented in pb.h, pb_workspace_bytes).
struct WsLayout {
    size_t off_f, off_xsum, off_planes, total;
};
inline WsLayout ws_layout(int64_t batch, int64_t kwords, int32_t act_bits) {
    WsLayout l;
    l.off_f = 0;
    l.off_xsum = align_up(sizeof(int32_t) * (size_t)batch);
    l.off_planes = align_up(l.off_xsum + sizeof(long long) * (size_t)batch * kMaxSplit);
    l.total = align_up(l.off_planes + sizeof(uint32_t) * (size_t)batch * act_bits * kwords);
    return l;
}

inline int act_nsplit(int64_t kwords) {
    int64_t n = (kwords + 31) / 32;
    if (n < 1) n = 1;
    if (n > kMaxSplit) n = kMaxSplit;
    return (int)n;
}

struct GemmArgs {
    const uint32_t* bits;   // [L][R][kwords]
    int64_t R, kwords;
    int L, offset, k_used, a;
    double scale;
    const uint32_t* planes; // [B][a][kwords]
    const int32_t* f;       // [B]
    const long long* xsum;  // [B][nsplit]
    int nsplit;
    int64_t B;
    float* y;               // [B][R]
    long long* acc;         // [B][R] or null
    const float* bias;      // [R] or null
    int fn;
    int accumulate;
};

cudaError_t launch_act_quant(const float* x, int64_t B, int64_t K, int64_t kwords, int a,
                             int act_frac, void* ws, cudaStream_t s);
cudaError_t launch_gemv_popc(const GemmArgs& g, cudaStream_t s);
cudaError_t launch_gemm_mma(const GemmArgs& g, cudaStream_t s);
bool mma_supported(const GemmArgs& g);
cudaError_t launch_lstm_cell(const float* gates, const float* c, int64_t B, int64_t H,
                             float* h_out, float* c_out, cudaStream_t s);
cudaError_t launch_rnn_cell(const float* gates, int64_t B, int64_t H, float* h_out,
                            cudaStream_t s);
cudaError_t launch_permute_shards(const float* gathered, int64_t B, int64_t rows_per_rank,
                                  int nranks, int64_t R, float* y, cudaStream_t s);

}  // namespace pb
