// pb_internal.h -- launchers shared between the host API (pb_api.cpp) and the
// sm_100a kernels (pb_act.cu, pb_gemv_popc.cu, pb_gemm_tc.cu, pb_cells.cu).
// Product code only; nothing here is shared with oracle/.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace pb {

constexpr int kMaxSplit = 64;        // activation kernel CTAs per batch column (max)
constexpr size_t kAlign = 256;
constexpr int kTcRows = 128;         // tensor engine row tile (MMA M)
constexpr int kTcMaxN = 64;          // tensor engine narrow mode: ceil(a/2) * batch <= 64 digit columns per
                                     // launch (MMA N padded to 8/16/32/64)
constexpr int kTcMaxB = 32;          // tensor engine: batch columns per launch
constexpr int kTcWideN = 128;        // wide mode: MMA N = 128 plane columns per slice, every slice
                                     // of the batch in one launch (single-buffered accumulator)
constexpr int kMaxRanks = 8;         // pb_matmul_rowshard_p2p: ranks of one node

inline size_t align_up(size_t v, size_t a = kAlign) { return (v + a - 1) / a * a; }

// Activation digits per batch column: the a planes stacked in pairs (pb_common.cuh).
inline int digits_of(int32_t a) { return (a + 1) / 2; }
// MMA N (digit columns batch * ceil(a/2) padded to a legal tcgen05 kind::mxf4 N for M = 128),
// 0 when the tensor engine's narrow operand tiles are not produced for this shape.
inline int tc_npad(int64_t batch, int32_t a) {
    const int64_t n = batch * digits_of(a);
    if (a <= 0 || n <= 0 || n > kTcMaxN || batch > kTcMaxB) return 0;
    return n <= 8 ? 8 : (n <= 16 ? 16 : (n <= 32 ? 32 : 64));
}
// Batch columns per narrow tensor-engine launch: the whole batch when it fits, else slices of
// min(32, 64 / ceil(a/2)) columns (pb_matmul / pb_linear run one fused launch per slice).
inline int64_t tc_slice(int64_t batch, int32_t a) {
    if (tc_npad(batch, a) > 0 || a <= 0) return batch;
    int64_t s = kTcMaxN / digits_of(a);
    if (s > kTcMaxB) s = kTcMaxB;
    return s < 1 ? 1 : s;
}
// Wide mode (digit columns > 64): batch columns per 128-column slice (at most kTcWideB: the
// per-slice epilogue sums, 1 KiB each, share SMEM with >= 4 weight stages), else 0.
constexpr int kTcWideB = 16;
inline int tc_wide_bs(int64_t batch, int32_t a) {
    if (a < 1 || a > 32 || tc_npad(batch, a) > 0 || batch <= 0) return 0;
    const int bs = kTcWideN / digits_of(a);
    return bs < kTcWideB ? bs : kTcWideB;
}

// Workspace carve-up (documented in pb.h, pb_workspace_bytes):
//   [tile counters int32 x kMaxTiles]   stream-K arrival counters; zero on
//                                       entry, every call leaves them zero
//   [grid barrier uint64]               fused tensor-engine path: monotonic
//                                       arrival counter (+2^20 per call)
//   [work counters int32 x 2]           tensor engine: item claims, finished
//                                       CTAs (left zero)
//   [end barrier uint64]                tensor engine (dynamic schedule):
//                                       monotonic arrival counter
//   [tile sums int64 x kAccTiles x B x 128]   tensor engine: partial-tile
//                                       accumulators (left zero)
//   [f_b int32 x B][Σx_q partials int64 x B x kXsumStride][bit planes [B][a][kwords]]
//   [tensor-engine B operand tiles: one N_pad x 32-byte e2m1 tile per 2 words
//    (64 columns), kwords rounded up to 32 words]
// Every region except the counters is fully rewritten by each call, so one
// zero-filled workspace can serve calls of any shape (not concurrently).
constexpr int kMaxTiles = 8192;      // tensor engine: rows <= 8192 * 128
constexpr int kMaxCtas = 160;        // tensor engine grid cap (B200: 148 SMs)
constexpr int kXsumStride = kMaxCtas;   // Σx_q partials per batch column (act CTAs or fused GEMM CTAs)
constexpr int kAccTiles = 2048;      // tensor engine: rows <= 2048 * 128 (partial-tile accumulators)
struct WsLayout {
    size_t off_count, off_slots, off_f, off_xsum, off_planes, off_bexp, total;
    int npad;                 // narrow: MMA N of one launch's slice (0: no narrow operand tiles)
    int wbs;                  // wide mode: batch columns per slice (0: off); operand tiles are
    int64_t wslices;          //   slice-major, [slice][chunk][16 words-pairs][128 x 32 B]
    size_t wslice_bytes;
};
inline WsLayout ws_layout(int64_t batch, int64_t kwords, int32_t act_bits) {
    WsLayout l;
    const int64_t bs = tc_slice(batch, act_bits);          // tensor-engine operands per slice
    l.npad = tc_npad(bs, act_bits);
    l.off_count = 0;
    l.off_slots = align_up(sizeof(int32_t) * (kMaxTiles + 6));
    // partial-tile sums sized for the largest slice this act_bits can launch (not this batch's),
    // so calls of different batch sizes with the same act_bits can share one workspace: the
    // region every call expects zero on entry is the same for all of them
    int64_t bs_max = act_bits > 0 ? kTcMaxN / digits_of(act_bits) : 1;
    if (bs_max > kTcMaxB) bs_max = kTcMaxB;
    if (bs_max < 1) bs_max = 1;
    if (bs_max < bs) bs_max = bs;
    l.wbs = tc_wide_bs(batch, act_bits);
    l.wslices = l.wbs ? (batch + l.wbs - 1) / l.wbs : 0;
    l.wslice_bytes = (size_t)((kwords + 31) / 32 * 32) * 16 * kTcWideN;
    // wide mode indexes its shared-tile sums by the CTA boundary inside the tile
    // (<= kMaxCtas + 1 slots of wbs x 128), which always fits the narrow region
    const size_t slots = (l.npad || l.wbs) ? sizeof(long long) * kAccTiles * (size_t)bs_max * kTcRows : 0;
    l.off_f = align_up(l.off_slots + slots);
    l.off_xsum = align_up(l.off_f + sizeof(int32_t) * (size_t)batch);
    l.off_planes = align_up(l.off_xsum + sizeof(long long) * (size_t)batch * kXsumStride);
    l.off_bexp = align_up(l.off_planes + sizeof(uint32_t) * (size_t)batch * act_bits * kwords);
    size_t bexp = (size_t)((kwords + 31) / 32 * 32) * 16 * (size_t)l.npad;
    if (l.wbs && (size_t)l.wslices * l.wslice_bytes > bexp) bexp = (size_t)l.wslices * l.wslice_bytes;
    l.total = align_up(l.off_bexp + bexp);
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
    int32_t* f;             // [B]
    long long* xsum;        // [B][kXsumStride], nsplit used
    int nsplit;
    int64_t B;
    int bs;                 // batch columns per slice: B (narrow, one slice) or kTcWideN / a (wide)
    float* y;               // [B][R]
    long long* acc;         // [B][R] or null
    const float* bias;      // [R] or null
    int fn;
    int accumulate;
    unsigned long long mid;       // midpoint offset 2^(L-k_used-1) (pb_matmul_ex PB_MM_MIDPOINT), else 0
    // tensor engine operands (valid when npad > 0)
    int npad;
    uint8_t* bexp;                // [kwords][npad x 32 canonical tile]
    unsigned long long* accbuf;   // [kAccTiles][B][128] partial tile sums, zero between calls
    int* counters;                // [kMaxTiles]
    long long* tl;                // diagnostics timeline (pb_debug_timeline) or null
    // fused activation path (tensor engine, pb_matmul / pb_linear): when x is set the
    // GEMM kernel itself runs steps a1-a2 (writing f, xsum, bexp) before the MMAs
    const float* x;               // [B][K] or null
    int64_t K;
    int act_frac;
    int* gbar;                    // grid barrier: monotonic uint64 arrival counter (+2^20 per call)
    int* work;                    // tensor engine {item claim counter, finished CTAs}, zero between calls
    int* ebar;                    // end-of-work grid barrier (dynamic schedule), monotonic uint64
    // fused LSTM cell (pb_lstm_seq, tensor engine): rows are gate-interleaved (row 4k + gate,
    // gates i, f, g, o); the finalisation applies the cell to the four pre-activations of
    // hidden unit k (dequant + bias + y when accumulate) and writes h, c instead of y
    int cell;                     // 0 = none, 1 = LSTM
    int64_t H;                    // hidden units (R / 4)
    const float* cell_c;          // [B][H] c_t
    float* cell_h;                // [B][H] h_{t+1}
    float* cell_c_out;            // [B][H] c_{t+1}
    // fused row-shard all-gather over peer memory (pb_matmul_rowshard_p2p):
    // the finalisation stores this shard's y rows straight into every rank's y_full
    // [B][R_total] (IPC / NVLink P2P mappings); then every CTA adds to every rank's arrival
    // counter (red.release.sys) and waits on its own: one cross-rank barrier, no NCCL
    int nranks;                   // 0 = off
    int64_t R_total, row0;        // global rows, this shard's first global row
    float* peer_y[kMaxRanks];     // rank p's y_full (this slice's batch offset applied)
    unsigned long long* peer_ctr[kMaxRanks];
    unsigned long long* local_ctr;
};

// Persistent LSTM recurrence (pb_lstm_tc.cu): all T timesteps of
// h_{t+1}, c_{t+1} = cell(gx[t] + W_hh h_t, c_t) in one launch, one CTA per (row tile,
// K-chunk) unit of W_hh, a grid barrier per timestep.
constexpr int kLstmMaxTiles = 64;   // persistent LSTM: 128-row tiles of W_hh (H <= 2048)
constexpr int kLstmMaxCtas = 160;   // persistent LSTM grid (tiles x chunks <= #SMs)
constexpr int kLstmMaxB = 32;        // batch columns (digit columns B * ceil(a/2) <= 128)
struct LstmArgs {
    const uint32_t* bits;   // W_hh [L][4H][kwords], gate-interleaved rows (row 4k + gate)
    int64_t R, kwords, H;   // R = 4H
    int L, offset, k_used, a;
    double scale;
    int B, T;
    const float* h0;        // [B][H]
    const float* c0;        // [B][H]
    const float* gx;        // [T][B][4H]: W_ih x_t + bias (hoisted), gate-interleaved
    float* h_seq;           // [T][B][H]
    float* c_seq;           // [T][B][H] or null
    float* c_last;          // [B][H]
    float* cbuf0;           // [B][H] x 2 ping-pong c_t when c_seq is null
    float* cbuf1;
    unsigned long long* accbuf;   // [tiles][B][128] exact split-tile sums, zero between calls
    int* counters;                // [tiles], zero between calls
    int* gbar;                    // monotonic grid-barrier counter (+2^20 per timestep)
    unsigned long long* maxslot;  // [2][kLstmMaxB] epoch-tagged max|h| (zero-filled once, never reset)
    // B = 1 exchange without a grid barrier: h_t and the per-tile max|h_t| as self-validating
    // 64-bit values (tag << 32) | float bits, tag = (uint32)(step counter at call start + t)
    unsigned long long* hx;       // [2][H] tagged h_t (by t & 1)
    unsigned long long* mxs;      // [2][CTAs][kLstmMaxTiles] mailboxes: tagged per-tile max|h_t|
    unsigned long long* stepctr;  // + T per call (workspace-resident, zero-filled once)
    long long* tl;                // diagnostics timeline (PB_TC_DEBUG=6) or null
};
int lstm_persist_npad(int64_t batch, int32_t a);
// Workspace of the B = 1 tagged exchange: step counter, per-tile slots, h_t by parity.
inline size_t lstm_xchg_bytes(int64_t H) {
    return align_up(256 + sizeof(unsigned long long) * (2 * (size_t)kLstmMaxCtas * kLstmMaxTiles + 2 * (size_t)H));
}
bool lstm_persist_supported(const LstmArgs& g);
cudaError_t launch_lstm_persist(const LstmArgs& g, cudaStream_t s);

// Diagnostics timeline (PB_TC_DEBUG=6): device log, [0] = record counter,
// records of 10 int64 from index 10; null when off.
constexpr long long kTlRecords = 1 << 16;
long long* debug_tl();


cudaError_t launch_act_quant(const float* x, int64_t B, int64_t K, int64_t kwords, int a,
                             int act_frac, void* ws, const WsLayout& l, cudaStream_t s);
cudaError_t launch_gemv_popc(const GemmArgs& g, cudaStream_t s);
cudaError_t launch_gemm_tc(const GemmArgs& g, cudaStream_t s);
bool tc_supported(const GemmArgs& g);
cudaError_t launch_lstm_cell(const float* gates, const float* c, int64_t B, int64_t H,
                             float* h_out, float* c_out, cudaStream_t s);
cudaError_t launch_lstm_cell_ilv(const float* gates, const float* c, int64_t B, int64_t H,
                                 float* h_out, float* c_out, cudaStream_t s);
cudaError_t launch_minmax(const float* W, int64_t n, float* partial, int blocks, cudaStream_t s);
cudaError_t launch_pack_grid(const float* W, int64_t R, int64_t K, int64_t kw, int L, double d, double clip,
                             int all_zero, uint32_t* dst, cudaStream_t s);
constexpr int kPackBlocks = 1024;    // pb_quantize_pack_weights_device: min/max partial blocks
cudaError_t launch_rnn_cell(const float* gates, int64_t B, int64_t H, float* h_out,
                            cudaStream_t s);
cudaError_t launch_permute_shards(const float* gathered, int64_t B, int64_t rows_per_rank,
                                  int nranks, int64_t R, float* y, cudaStream_t s);

}  // namespace pb
