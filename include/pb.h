/*
 * pb.h -- C ABI of libpb, the B200 (sm_100a) PrecisionBatching bitlayer
 * matvec / skinny-matmul library.
 *
 * Paper: "PrecisionBatching", arXiv 2003.00822 (/root/reference/PAPER.md,
 * cited "P:<line>").  The library implements the inference stage (Alg. 2,
 * P:183-202) on the GPU and the preprocessing stage (Alg. 1) on
 * the host.  Numerical readings of the paper (tie rules, activation scaling,
 * layouts, ...) are the G1..G16 entries of DESIGN.md "Readings".
 *
 * Conventions for every entry point
 *   - Plain C types only.  Device pointers are raw CUDA device addresses;
 *     `pb_stream` is a cudaStream_t passed as an opaque pointer (NULL = the
 *     legacy default stream).
 *   - Ownership: the caller allocates every buffer (packed weights,
 *     workspace, x, y, acc).  Nothing in pb_matmul* allocates or frees device
 *     memory and nothing synchronises the host; calls are stream-ordered and
 *     CUDA-graph capturable.  The only library-owned object is pb_comm.
 *   - Errors: arguments are validated before any launch.  A non-OK status
 *     leaves outputs untouched and sets a thread-local message readable with
 *     pb_last_error().  Launch failures map to PB_ECUDA; device faults
 *     surface at the caller's next synchronisation.  No exceptions cross the
 *     ABI; the library never prints or exits.
 *   - There is no CPU fallback: every compute entry point runs CUDA kernels
 *     and fails with PB_ECUDA when no device is usable.
 */
#ifndef PB_H_
#define PB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PB_OK = 0,
    PB_EINVAL = 1,      /* bad argument: null/misaligned pointer, out-of-range size or knob */
    PB_ERANGE = 2,      /* int64 accumulator bound (reading G11) or a code out of range     */
    PB_EDEGENERATE = 3, /* informational: max(W) == min(W); a valid pack was still written  */
    PB_ECUDA = 4,       /* CUDA runtime error (no device, launch failure, ...)              */
    PB_ENCCL = 5        /* NCCL unavailable or failed                                       */
} pb_status;

typedef void* pb_stream;

/* Weight quantisation modes for pb_quantize_pack_weights (Alg. 1). */
enum {
    PB_Q_GRID = 0,    /* default: code = clamp(rint(W/d)), d = (max-min)/2^(L-1), s_w = d (G1, G3) */
    PB_Q_ALG1 = 1,    /* literal Alg. 1: W_q = trunc(Q(W)*2^16), max_bit window, floor (G2, G3)  */
    PB_Q_BINARY = 2   /* 1-bit +-v code, v = mean|W| (G7); requires layers == 1          */
};

/* act_frac value selecting the per-column power-of-two fixed point (G8). */
#define PB_ACT_AUTO (-1024)

/* Epilogue functions for pb_linear (applied in fp32 after the bias). */
enum { PB_FN_NONE = 0, PB_FN_RELU = 1, PB_FN_TANH = 2, PB_FN_SIGMOID = 3 };

/* Kernel engine for the binary product (step a3).  AUTO picks per shape. */
enum { PB_ENGINE_AUTO = 0, PB_ENGINE_POPC = 1, PB_ENGINE_MMA = 2 };

/*
 * Packed weight bitlayers (D1).  Plain descriptor; `bits` is
 * caller-owned memory (host or device) of L * rows * kwords uint32 words.
 * Bitlayer W_i: layer 0 = the sign layer, layer i holds bit
 * (L-1-i) of the L-bit two's-complement code; padding columns are zero
 * (AND-neutral).  kwords = 4*ceil(cols/128).  Its canonical word for
 * 32-column block c of row r is  Wc_i[r][c] = sum_j W_i[r, 32c + j] << j.
 * Storage ("paired bitlayers", the stacking of P:206): layers (2p, 2p+1)
 * share the span of layer slots 2p and 2p+1, as rows of 2*kwords words
 *     pair[p][row][2c + e],  e = 0 (even columns), 1 (odd columns),
 *     bit 2k   of pair[p][r][2c + e] = W_{2p+1}[r, 32c + 2k + e]   (lower)
 *     bit 2k+1 of pair[p][r][2c + e] = W_{2p}  [r, 32c + 2k + e]   (upper)
 * so each 2-bit field is one column's (upper, lower) bit pair.  With L odd
 * the last layer W_{L-1} is stored canonically in slot L-1:
 *     bits[(L-1)*rows*kwords + r*kwords + c] = Wc_{L-1}[r][c].
 * Represented weight: W ~= scale * (sum_i S_i * W_i + offset) with
 * S_0 = -2^(L-1) (or -2 when offset = 1, binary mode) and S_i = 2^(L-1-i).
 */
typedef struct {
    uint32_t* bits;
    int64_t rows, cols, kwords;
    int32_t layers;   /* L, 1..16 */
    int32_t offset;   /* o: 0, or 1 for the binary +-v code (L = 1)    */
    double scale;     /* s_w: value of one code LSB                    */
} pb_weights;

/* Thread-local description of the last non-OK status ("" if none). */
const char* pb_last_error(void);
const char* pb_version(void);

/* kwords = 4*ceil(cols/128) (16-byte row pitch). */
int64_t pb_kwords(int64_t cols);

/* Bytes of a packed [layers][rows][kwords] buffer (P:124 memory model:
 * layers*rows*cols/8 algorithmic, plus row padding). */
size_t pb_packed_bytes(int64_t rows, int64_t cols, int32_t layers);

/*
 * Offline preprocessing, Alg. 1 and §3.3.  Host code,
 * double precision, no GPU needed when dst_is_device == 0.
 *   W_host      [rows][cols] float32, row-major, host memory.
 *   layers      L = stored bitlayers (1..16); PB_Q_GRID/ALG1 need L >= 2,
 *               PB_Q_BINARY needs L == 1 (reading G1).
 *   clip        > 0: clamp W to [-clip, clip] first; <= 0: none.
 *   dst         pb_packed_bytes(rows, cols, layers) bytes, 16-byte aligned;
 *               device memory if dst_is_device (copied on stream s, which
 *               is synchronised before return: this call is offline).
 *   out         filled descriptor (bits = dst).
 * Returns PB_EDEGENERATE (with a valid zero/+-1 pack) when max(W) == min(W).
 */
pb_status pb_quantize_pack_weights(const float* W_host, int64_t rows, int64_t cols,
                                   int32_t layers, int32_t quant_mode, float clip,
                                   void* dst, int32_t dst_is_device, pb_stream s,
                                   pb_weights* out);

/* PB_Q_GRID with a caller-provided grid step d (> 0): code =
 * clamp(rint(W/d)), scale = d.  Used to pack the row shards of one layer on
 * several ranks with the layer's global d = (max(W) - min(W)) / 2^(L-1), so
 * every shard carries exactly the codes of the unsharded layer (§8(e)). */
pb_status pb_quantize_pack_weights_step(const float* W_host, int64_t rows, int64_t cols,
                                        int32_t layers, double step, void* dst,
                                        int32_t dst_is_device, pb_stream s, pb_weights* out);

/* The Q(W) grid step of P:149, d = (w_max - w_min) / 2^(L-1) for L = layers stored
 * bitlayers (reading G1), from given extrema -- e.g. the min/max all-reduced over the
 * row shards of one layer, so every rank packs with the unsharded layer's grid.
 * Degenerate extrema (w_max == w_min, reading G5): *step = |w_max|, or 1 when both are 0,
 * and PB_EDEGENERATE is returned (the step is still written).  PB_EINVAL for a NULL
 * step, layers outside [2,16], non-finite extrema or w_min > w_max.  Host only. */
pb_status pb_grid_step(double w_min, double w_max, int32_t layers, double* step);

/* Step a0 on the GPU, for a float32 W [rows][cols] already
 * in device memory: the PB_Q_GRID quantiser (readings G4, G5) and
 * the bitlayer packer, producing exactly the bytes and scale of
 * pb_quantize_pack_weights(PB_Q_GRID) / _step.  step == 0: grid from the
 * extrema (clip > 0 clips first; ws = pb_pack_device_workspace_bytes() of
 * device scratch for the min/max partials); step > 0: that grid step (row
 * shards, as pb_quantize_pack_weights_step; clip and ws unused).
 * dst: device, pb_packed_bytes(rows, cols, layers), 16-byte aligned.  Offline:
 * synchronises the stream.  PB_EINVAL for layers outside [2,16] (binary and
 * literal Alg. 1 packing stay on the host), PB_EDEGENERATE as the host packer. */
size_t pb_pack_device_workspace_bytes(void);
pb_status pb_quantize_pack_weights_device(const float* W_dev, int64_t rows, int64_t cols,
                                          int32_t layers, float clip, double step, void* dst,
                                          void* ws, size_t ws_bytes, pb_stream s,
                                          pb_weights* out);

/* Pack caller-supplied integer codes [rows][cols] (L-bit two's complement;
 * for offset = 1, L must be 1 and codes are +-1 meaning 1 - 2*bit).  Used by
 * tests and by callers with their own quantiser.  PB_ERANGE if a code does
 * not fit. */
pb_status pb_pack_codes(const int32_t* codes_host, int64_t rows, int64_t cols,
                        int32_t layers, int32_t offset, double scale,
                        void* dst, int32_t dst_is_device, pb_stream s, pb_weights* out);

/* Clip-threshold search (reading G6: 64 candidates (k/64)*max|W|,
 * objective mean |s_w*code - W|, ties -> larger).  Host only, offline. */
pb_status pb_search_clip(const float* W_host, int64_t rows, int64_t cols, int32_t layers,
                         float* clip_out);

/*
 * Workspace of one call (batch columns of a layer with `cols` inputs):
 *   [stream-K tile counters int32 x 8192]     zero on entry, left zero on exit
 *   [grid barrier uint64]                     monotonic arrival counter (any
 *                                             value on entry; grows by 2^20 per call)
 *   [work counters int32 x 2]                 zero on entry, left zero
 *   [end barrier uint64]                      monotonic arrival counter
 *   [tensor-engine partial-tile sums int64 x 2048 x S x 128, S = the largest
 *    batch slice of one narrow launch for this act_bits, min(32, 64 / ceil(act_bits/2))]
 *                                             zero on entry, left zero
 *   [f_b int32 x batch][x_q partial sums int64 x batch x 160]
 *   [planes uint32 x batch x act_bits x kwords]
 *   [tensor-engine B operand tiles (activation planes stacked in pairs: ceil(a/2)
 *    digit rows per batch column): narrow, roundup(kwords, 32) x N_pad x 16 bytes,
 *    N_pad = ceil(a/2) * slice padded to 8/16/32/64, slice = batch when
 *    ceil(a/2)*batch <= 64 and batch <= 32, else min(32, 64/ceil(a/2)) columns;
 *    wide mode (larger batches): slice-major 128-row tiles, one slice per
 *    128/ceil(a/2) batch columns, every slice of the batch]
 * each region 256-byte aligned.  The workspace must be zero-filled before its
 * first use (the counters); every other region is rewritten by each call, so
 * one workspace serves calls of any shape with the same act_bits (the
 * partial-tile sums sit at the same place for all of them), but not two
 * calls concurrently.
 */
size_t pb_workspace_bytes(int64_t batch, int64_t cols, int32_t act_bits);

/*
 * Steps a1+a2: per batch column b, quantise x[b,:] to
 * x_q = trunc(x * 2^f_b) (f_b per reading G8, or act_frac literal with
 * saturation) and bit-transpose into act_bits planes (sign plane first) in
 * the workspace.  x: device [batch][cols] float32.
 */
pb_status pb_act_quantize(const float* x, int64_t batch, int64_t cols, int32_t act_bits,
                          int32_t act_frac, void* ws, size_t ws_bytes, pb_stream s);

/*
 * Steps a3-a5: for every output row r and
 * batch column b, C_ij = popc(W_i[r,:] AND X_j[b,:]) for i < k_used, j < a,
 *   acc = sum_i S_i sum_j T_j C_ij + offset * sum_c x_q[b,c]   (exact int64)
 *   y   = fn( (float)ldexp((double)acc * scale, -f_b) + bias[r] (+ y_old) )
 * reading the planes that pb_act_quantize left in ws.
 *   y         device [batch][rows] float32 (required);
 *   acc       device [batch][rows] int64 or NULL;
 *   bias      device [rows] float32 or NULL;  fn: PB_FN_*;
 *   accumulate  nonzero: add the previous contents of y before fn.
 * k_used: weight bitlayers accumulated, 1..L, always the sign layer plus
 * the most significant ones (reading G12).
 */
pb_status pb_bitgemm(const void* ws, size_t ws_bytes, int64_t batch, const pb_weights* w,
                     int32_t k_used,
                     int32_t act_bits, float* y, int64_t* acc, const float* bias,
                     int32_t fn, int32_t accumulate, pb_stream s);

/* The whole hot path, Alg. 2: pb_act_quantize + pb_bitgemm (PB_FN_NONE,
 * no bias).  y = W x in the paper's statement L_i(x) = Wx. */
pb_status pb_matmul(const float* x, int64_t batch, const pb_weights* w, int32_t k_used,
                    int32_t act_bits, int32_t act_frac, float* y, int64_t* acc,
                    void* ws, size_t ws_bytes, pb_stream s);

/* pb_matmul with options.  flags:
 *   PB_MM_MIDPOINT  with k_used < L, represent each truncated code by the centre of
 *                   its dropped range, m_trunc + 2^(L-k_used-1) (reading G12 gives the
 *                   floor-truncated m_trunc; the midpoint is not in the paper): acc
 *                   gains exactly 2^(L-k_used-1) * sum_c x_q[b,c].  No effect when
 *                   k_used = L or for binary weights. */
enum { PB_MM_MIDPOINT = 1 };
pb_status pb_matmul_ex(const float* x, int64_t batch, const pb_weights* w, int32_t k_used,
                       int32_t act_bits, int32_t act_frac, int32_t flags, float* y,
                       int64_t* acc, void* ws, size_t ws_bytes, pb_stream s);

/* FC layer helper: y = fn(W x + bias) (P:256 MNIST FC layers). */
pb_status pb_linear(const float* x, int64_t batch, const pb_weights* w, int32_t k_used,
                    int32_t act_bits, int32_t act_frac, const float* bias, int32_t fn,
                    float* y, void* ws, size_t ws_bytes, pb_stream s);

/* Workspace for pb_rnn_step / pb_lstm_step: activation workspace for
 * max(E, H) columns plus a [batch][gate_rows] float32 gate buffer. */
size_t pb_cell_workspace_bytes(int64_t batch, int64_t in_cols, int64_t hidden,
                               int32_t act_bits, int32_t gates);

/* Elman RNN step (reading G15): h' = tanh(W_ih x + b_ih + W_hh h + b_hh).
 * W_ih [H][E], W_hh [H][H]; x [batch][E], h, h_out [batch][H] (device). */
pb_status pb_rnn_step(const float* x_t, const float* h, const pb_weights* w_ih,
                      const pb_weights* w_hh, const float* b_ih, const float* b_hh,
                      int32_t k_used_ih, int32_t k_used_hh, int32_t act_bits, int64_t batch,
                      float* h_out, void* ws, size_t ws_bytes, pb_stream s);

/* LSTM step (gate order i,f,g,o as PyTorch nn.LSTM, G15):
 * gates = W_ih x + b_ih + W_hh h + b_hh, [batch][4H];
 * c' = sigmoid(f) c + sigmoid(i) tanh(g);  h' = sigmoid(o) tanh(c').
 * W_ih [4H][E], W_hh [4H][H] (device). */
pb_status pb_lstm_step(const float* x_t, const float* h, const float* c,
                       const pb_weights* w_ih, const pb_weights* w_hh,
                       const float* b_ih, const float* b_hh, int32_t k_used_ih,
                       int32_t k_used_hh, int32_t act_bits, int64_t batch,
                       float* h_out, float* c_out, void* ws, size_t ws_bytes, pb_stream s);

/* LSTM over a sequence (P:258-260 LSTM LM, P:317 NLI encoders;
 * reading G15).  Rows of W_ih [4H][E], W_hh [4H][H] and bias [4H] are
 * GATE-INTERLEAVED: row 4k + q is gate q (i, f, g, o) of hidden unit k, i.e.
 * PyTorch's gate-major rows permuted (paper_2003_00822_b200.interleave_gates);
 * Q(W) is permutation-invariant, so the codes are those of the gate-major
 * matrix.  Steps:
 *   1. gx[t][b] = W_ih x[t][b] + bias for all steps*batch columns in one
 *      batched call (the input projection hoisted out of the recurrence);
 *   2. per t: pre = W_hh h_t + gx[t]; c_{t+1} = sigmoid(f) c_t + sigmoid(i) tanh(g),
 *      h_{t+1} = sigmoid(o) tanh(c_{t+1}).  When W_hh's (128-row tile, 1024-column
 *      chunk) units fit the SMs at once (H <= 2048, batch <= 32), ALL steps run in
 *      ONE persistent tensor-engine launch (a1-a5 + the cell per step; h exchanged
 *      between CTAs through the workspace, tagged by a workspace step counter that
 *      grows by `steps` per call); else one fused launch per step (the cell in the
 *      finalisation, which holds the 4 gate rows of a unit in adjacent lanes), or
 *      planes + GEMM + a cell kernel.  The workspace must be zero-filled before its
 *      first use and is not shared by concurrent calls.
 *   x      device [steps][batch][E];  h0, c0 device [batch][H];
 *   bias   device [4H] (b_ih + b_hh, interleaved) or NULL;
 *   h_seq  device [steps][batch][H]: h_1 .. h_steps (required);
 *   c_seq  device [steps][batch][H] or NULL: c_1 .. c_steps;
 *   c_last device [batch][H]: c_steps (required).
 * Stream-ordered, graph-capturable, no allocation.  PB_EINVAL: shapes, NULLs,
 * k_used outside [1, L] of either matrix, steps*batch > 65535 (the hoisted
 * projection is one batched call), workspace < pb_lstm_seq_workspace_bytes;
 * PB_ERANGE: the reading-G11 accumulator bound of either matrix.  Every check
 * runs before the first launch. */
size_t pb_lstm_seq_workspace_bytes(int64_t steps, int64_t batch, int64_t in_cols,
                                   int64_t hidden, int32_t act_bits);
pb_status pb_lstm_seq(const float* x, int64_t steps, int64_t batch, const float* h0,
                      const float* c0, const pb_weights* w_ih, const pb_weights* w_hh,
                      const float* bias, int32_t k_used_ih, int32_t k_used_hh,
                      int32_t act_bits, float* h_seq, float* c_seq, float* c_last,
                      void* ws, size_t ws_bytes, pb_stream s);

/* Select the binary-product engine (process-wide; default AUTO). */
pb_status pb_set_engine(int32_t engine);
int32_t pb_get_engine(void);

/* Diagnostics: per-CTA kernel timeline (globaltimer ns), kept only when the
 * environment variable PB_TC_DEBUG=6 is set at the library's first launch.
 * Copies up to max_records records of 10 int64 each into host memory dst:
 *   {kind, cta, sm, units, t0, t1, t2, t3, t4, t5}
 *   kind 0 = activation cast/transpose CTA: t0 launch, t1 PDL wait done, t2 end;
 *   kind 1 = tensor-engine GEMM CTA: t0 start, t1 B operand ready (PDL wait
 *            done), t2 first MMA issue, t3 last MMA issue, t4 epilogue done,
 *            t5 exit.
 * Synchronises the device, clears the log and returns the number of records
 * copied; -1 when no log is kept. */
int64_t pb_debug_timeline(int64_t* dst, int64_t max_records);

/* ---------------- multi-GPU row sharding ----------------
 * Rank g of N holds rows [row0, row0 + nrows) of every bitlayer, packed as
 * its own pb_weights with rows = pb_shard_rows(...).  Balanced split:
 * rows_per_rank = ceil(R/N); the last ranks may hold fewer (or zero) rows. */
pb_status pb_shard_rows(int64_t rows_total, int32_t nranks, int32_t rank,
                        int64_t* row0, int64_t* nrows);

typedef struct pb_comm pb_comm;
/* NCCL unique id (128 bytes) to broadcast from rank 0 (e.g. via
 * torch.distributed).  NCCL is loaded at run time (libnccl.so.2). */
pb_status pb_comm_unique_id(void* id128);
pb_status pb_comm_init(pb_comm** comm, const void* id128, int32_t nranks, int32_t rank);
pb_status pb_comm_destroy(pb_comm* comm);

/* Fused row-shard all-gather over peer memory (a6 without NCCL).
 * One process per GPU, ranks 1, 2, 4 or 8 of one node.  pb_p2p_create
 * allocates this rank's library-owned buffer [256 B arrival counter][y_full
 * batch x rows_total float32] and writes its CUDA IPC handle
 * (pb_p2p_handle_bytes()); the caller all-gathers the handles in rank order
 * (e.g. torch.distributed) and calls pb_p2p_open.  pb_matmul_rowshard_p2p runs
 * a1-a5 on this rank's shard (w_shard rows = ceil(R/N), padded) in ONE fused
 * tensor-engine launch whose finalisation stores each y row straight into
 * every rank's y_full over NVLink (IPC mappings; the same buffer layout on
 * every rank) and then joins a cross-rank barrier on the arrival counters
 * (red.release.sys / ld.acquire.sys), so when the kernel completes on any rank
 * its y_full holds all R rows -- bit-identical to pb_matmul on the whole layer.
 * Stream-ordered; the same call sequence on every rank.  PB_EINVAL when the
 * shape is outside the tensor engine's fused path (use pb_matmul_rowshard). */
typedef struct pb_p2p pb_p2p;
size_t pb_p2p_handle_bytes(void);
pb_status pb_p2p_create(pb_p2p** p2p, int32_t nranks, int32_t rank, int64_t batch,
                        int64_t rows_total, void* handle_out);
pb_status pb_p2p_open(pb_p2p* p2p, const void* handles /* nranks x pb_p2p_handle_bytes() */);
/* In-process alternative to pb_p2p_open (one process driving several GPUs with
 * peer access enabled, or several ranks on one GPU): all[q] is rank q's object. */
pb_status pb_p2p_open_peers(pb_p2p* p2p, pb_p2p* const* all);
float* pb_p2p_y(pb_p2p* p2p);               /* device [batch][rows_total] */
pb_status pb_p2p_destroy(pb_p2p* p2p);
pb_status pb_matmul_rowshard_p2p(const float* x, int64_t batch, const pb_weights* w_shard,
                                 int64_t rows_total, int32_t k_used, int32_t act_bits,
                                 int32_t act_frac, pb_p2p* p2p, void* ws, size_t ws_bytes,
                                 pb_stream s);

/* Extra workspace for pb_matmul_rowshard: gather buffer [N][batch][ceil(R/N)]. */
size_t pb_rowshard_workspace_bytes(int64_t batch, int64_t cols, int32_t act_bits,
                                   int64_t rows_total, int32_t nranks);

/* Row-sharded y = W x: local pb_matmul on this rank's shard, then an NCCL
 * all-gather of the y shards over NVLink on stream s, then (batch > 1 or
 * uneven split) a permute into y_full [batch][rows_total].  x is replicated;
 * every rank computes the same f_b and planes, so y_full is bit-identical to
 * the single-GPU result. */
pb_status pb_matmul_rowshard(const float* x, int64_t batch, const pb_weights* w_shard,
                             int64_t rows_total, int32_t k_used, int32_t act_bits,
                             int32_t act_frac, float* y_full, pb_comm* comm,
                             void* ws, size_t ws_bytes, pb_stream s);

#ifdef __cplusplus
}
#endif
#endif /* PB_H_ */
