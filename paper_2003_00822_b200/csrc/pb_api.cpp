// pb_api.cpp -- host side of libpb: the C ABI declared in include/pb.h.
//   * argument validation (before any launch), thread-local error text;
//   * the offline packer: Q(W) / Alg. 1 / binary
//     +-v in double precision, then the L-bitlayer decomposition
//      packed 32 columns per uint32 word;
//   * kernel launches for the hot path (Alg. 2) and the layer
//     helpers, all stream-ordered, no host sync, no allocation;
//   * the row-shard all-gather over NCCL (loaded at run time).
// Product code: shares nothing with oracle/.
#include <dlfcn.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>

#include "pb.h"
#include "pb_internal.h"

namespace {

thread_local char g_err[512] = "";
int g_engine = PB_ENGINE_AUTO;

pb_status fail(pb_status st, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return st;
}

pb_status cuda_fail(cudaError_t e, const char* what) {
    cudaGetLastError();   // clear the sticky-free error state
    return fail(PB_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

int ceil_log2(int64_t v) {
    int k = 0;
    while (((int64_t)1 << k) < v) ++k;
    return k;
}

// ------------------------------------------------------------------ packer
// Quantisers: double precision, FMA-free operation sequences (reading G13's
// rule applied offline): grid  d = (max-min)/2^(L-1), code = clamp(rint(w/d)).
struct QuantOut {
    std::vector<int32_t> codes;
    double scale = 1.0;
    int offset = 0;
    bool degenerate = false;
};

inline double clipv(double w, double clip) {
    if (clip > 0) {
        if (w > clip) w = clip;
        if (w < -clip) w = -clip;
    }
    return w;
}

void minmax(const float* W, int64_t n, double clip, double& mn, double& mx) {
    mx = -INFINITY;
    mn = INFINITY;
    for (int64_t e = 0; e < n; ++e) {
        const double w = clipv((double)W[e], clip);
        mx = w > mx ? w : mx;
        mn = w < mn ? w : mn;
    }
}

// Q(W) step d with the degenerate rule of reading G5.
double grid_step(double mn, double mx, int n, bool& degenerate) {
    double d = (mx - mn) / std::ldexp(1.0, n);
    degenerate = false;
    if (d == 0.0) {
        degenerate = true;
        d = std::fabs(mx);
        if (d == 0.0) d = 1.0;
    }
    return d;
}

pb_status quantize_grid(const float* W, int64_t n, int L, double clip, QuantOut& q) {
    double mn, mx;
    minmax(W, n, clip, mn, mx);
    bool deg;
    const double d = grid_step(mn, mx, L - 1, deg);
    const double lo = -std::ldexp(1.0, L - 1), hi = std::ldexp(1.0, L - 1) - 1.0;
    q.codes.resize((size_t)n);
    q.scale = d;
    q.offset = 0;
    q.degenerate = deg;
    bool all_zero = deg && mx == 0.0 && mn == 0.0;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < n; ++e) {
        double m = std::rint(clipv((double)W[e], clip) / d);
        m = m < lo ? lo : (m > hi ? hi : m);
        q.codes[(size_t)e] = all_zero ? 0 : (int32_t)m;
    }
    if (all_zero) q.scale = 1.0;
    return PB_OK;
}

pb_status quantize_alg1(const float* W, int64_t n, int L, double clip, QuantOut& q) {
    // Alg. 1: W_q = Int(Q(W) * 2^16); max_bit = floor(log2 max|W_q|);
    // keep bit positions max_bit+1 (sign) .. max_bit-n+1 (reading G2).
    const int nb = L - 1;
    double mn, mx;
    minmax(W, n, clip, mn, mx);
    bool deg;
    const double d = grid_step(mn, mx, nb, deg);
    std::vector<int64_t> wq((size_t)n);
    int64_t maxabs = 0;
    for (int64_t e = 0; e < n; ++e) {
        const double Q = d * std::rint(clipv((double)W[e], clip) / d);
        const double t = std::trunc(Q * 65536.0);
        if (std::fabs(t) >= 9.0e18) return fail(PB_ERANGE, "Alg. 1: W_q overflows int64");
        wq[(size_t)e] = (int64_t)t;
        const int64_t a = wq[(size_t)e] < 0 ? -wq[(size_t)e] : wq[(size_t)e];
        maxabs = a > maxabs ? a : maxabs;
    }
    q.codes.assign((size_t)n, 0);
    q.offset = 0;
    q.degenerate = deg;
    if (maxabs == 0) {
        q.scale = 1.0;
        q.degenerate = true;
        return PB_OK;
    }
    int max_bit = 63 - __builtin_clzll((unsigned long long)maxabs);
    const int lo = max_bit - nb + 1;
    for (int64_t e = 0; e < n; ++e) {
        const int64_t v = wq[(size_t)e];
        q.codes[(size_t)e] = (int32_t)(lo >= 0 ? (v >> lo) : (v * ((int64_t)1 << (-lo))));
    }
    q.scale = std::ldexp(1.0, lo - 16);
    return PB_OK;
}

pb_status quantize_binary(const float* W, int64_t n, double clip, QuantOut& q) {
    // P:152 1-bit +-v; v = mean|W| (reading G7); bit = [W < 0]; code 1 - 2*bit.
    double s = 0.0;
    q.codes.resize((size_t)n);
    for (int64_t e = 0; e < n; ++e) {
        const double w = clipv((double)W[e], clip);
        s += std::fabs(w);
        q.codes[(size_t)e] = w < 0.0 ? -1 : 1;
    }
    q.scale = s / (double)n;
    q.offset = 1;
    q.degenerate = false;
    if (q.scale == 0.0) {
        q.scale = 1.0;
        q.degenerate = true;
    }
    return PB_OK;
}

// Decompose + pack: layer i = bit (L-1-i) of the L-bit two's-complement code
// (binary mode: the single layer is [code == -1]).
pb_status pack(const int32_t* codes, int64_t R, int64_t K, int L, int offset, std::vector<uint32_t>& out) {
    const int64_t kw = pb_kwords(K);
    out.assign((size_t)L * (size_t)R * (size_t)kw, 0u);
    const int64_t lo = offset ? -1 : -((int64_t)1 << (L - 1));
    const int64_t hi = offset ? 1 : ((int64_t)1 << (L - 1)) - 1;
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int64_t r = 0; r < R; ++r) {
        for (int64_t c = 0; c < K; ++c) {
            const int32_t m = codes[r * K + c];
            if (m < lo || m > hi || (offset && m == 0)) {
                bad = 1;
                continue;
            }
            const uint32_t u = offset ? (m == -1 ? 1u : 0u) : (uint32_t)m;
            const uint32_t bit = 1u << (c & 31);
            for (int i = 0; i < L; ++i)
                if ((u >> (L - 1 - i)) & 1u) out[((size_t)i * R + r) * kw + (c >> 5)] |= bit;
        }
    }
    if (bad) return fail(PB_ERANGE, "a code does not fit %d-bit two's complement%s", L,
                         offset ? " (binary mode needs codes +-1)" : "");
    // paired storage (pb.h): layers (2p, 2p+1) -> rows of 2*kw words, even/odd columns
    // interleaved as (lower, upper) bit pairs; an odd last layer stays canonical
    if (L >= 2) {
        const std::vector<uint32_t> canon(out.begin(), out.begin() + (size_t)(L / 2) * 2 * R * kw);
        for (int p = 0; 2 * p + 1 < L; ++p) {
#pragma omp parallel for schedule(static)
            for (int64_t r = 0; r < R; ++r) {
                const uint32_t* hi = &canon[((size_t)(2 * p) * R + r) * kw];
                const uint32_t* lo = &canon[((size_t)(2 * p + 1) * R + r) * kw];
                uint32_t* dst = &out[(size_t)(2 * p) * R * kw + (size_t)r * 2 * kw];
                for (int64_t c = 0; c < kw; ++c) {
                    uint32_t e0 = 0, e1 = 0;
                    for (int k = 0; k < 16; ++k) {
                        e0 |= ((lo[c] >> (2 * k)) & 1u) << (2 * k) | ((hi[c] >> (2 * k)) & 1u) << (2 * k + 1);
                        e1 |= ((lo[c] >> (2 * k + 1)) & 1u) << (2 * k) | ((hi[c] >> (2 * k + 1)) & 1u) << (2 * k + 1);
                    }
                    dst[2 * c] = e0;
                    dst[2 * c + 1] = e1;
                }
            }
        }
    }
    return PB_OK;
}

pb_status store(const std::vector<uint32_t>& host, int64_t R, int64_t K, int L, int offset, double scale,
                void* dst, int dst_is_device, pb_stream s, pb_weights* out) {
    const size_t bytes = host.size() * sizeof(uint32_t);
    if (dst_is_device) {
        cudaStream_t st = static_cast<cudaStream_t>(s);
        cudaError_t e = cudaMemcpyAsync(dst, host.data(), bytes, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return cuda_fail(e, "pack: copy to device");
    } else if (bytes) {
        std::memcpy(dst, host.data(), bytes);
    }
    out->bits = static_cast<uint32_t*>(dst);
    out->rows = R;
    out->cols = K;
    out->kwords = pb_kwords(K);
    out->layers = L;
    out->offset = offset;
    out->scale = scale;
    return PB_OK;
}

// ------------------------------------------------------------------ launch
pb_status check_weights(const pb_weights* w) {
    if (!w) return fail(PB_EINVAL, "weights descriptor is NULL");
    if (w->layers < 1 || w->layers > 16) return fail(PB_EINVAL, "layers=%d not in [1,16]", w->layers);
    if (w->offset != 0 && !(w->offset == 1 && w->layers == 1))
        return fail(PB_EINVAL, "offset=%d requires layers == 1 (binary mode)", w->offset);
    if (w->rows < 0 || w->cols < 0) return fail(PB_EINVAL, "negative rows/cols");
    if (w->kwords != pb_kwords(w->cols)) return fail(PB_EINVAL, "kwords=%lld != 4*ceil(cols/128)", (long long)w->kwords);
    if (w->rows > 0 && w->kwords > 0 && (!w->bits || !aligned(w->bits, 16)))
        return fail(PB_EINVAL, "bits must be a non-NULL 16-byte aligned device pointer");
    return PB_OK;
}

pb_status check_act(int64_t batch, int64_t cols, int32_t a, int32_t act_frac) {
    if (batch < 0 || batch > 65535) return fail(PB_EINVAL, "batch=%lld not in [0,65535]", (long long)batch);
    if (cols < 0) return fail(PB_EINVAL, "cols < 0");
    if (a < 1 || a > 32) return fail(PB_EINVAL, "act_bits=%d not in [1,32]", a);
    if (act_frac != PB_ACT_AUTO && (act_frac < -126 || act_frac > 126))
        return fail(PB_EINVAL, "act_frac=%d not PB_ACT_AUTO or in [-126,126]", act_frac);
    return PB_OK;
}

pb_status check_ws(const void* ws, size_t ws_bytes, int64_t batch, int64_t cols, int32_t a) {
    const size_t need = pb_workspace_bytes(batch, cols, a);
    if (!ws || !aligned(ws, 16)) return fail(PB_EINVAL, "workspace must be non-NULL and 16-byte aligned");
    if (ws_bytes < need) return fail(PB_EINVAL, "workspace %zu bytes < required %zu", ws_bytes, need);
    return PB_OK;
}

}  // namespace

extern "C" {

const char* pb_last_error(void) { return g_err; }
const char* pb_version(void) { return "pbatch-b200 0.1 (sm_100a)"; }

int64_t pb_kwords(int64_t cols) { return cols <= 0 ? 0 : 4 * ((cols + 127) / 128); }

size_t pb_packed_bytes(int64_t rows, int64_t cols, int32_t layers) {
    if (rows < 0 || cols < 0 || layers < 1) return 0;
    return (size_t)layers * (size_t)rows * (size_t)pb_kwords(cols) * sizeof(uint32_t);
}

pb_status pb_quantize_pack_weights(const float* W_host, int64_t rows, int64_t cols, int32_t layers,
                                   int32_t quant_mode, float clip, void* dst, int32_t dst_is_device,
                                   pb_stream s, pb_weights* out) {
    g_err[0] = 0;
    if (!out) return fail(PB_EINVAL, "out is NULL");
    if (rows < 0 || cols < 0) return fail(PB_EINVAL, "negative rows/cols");
    if (rows * cols > 0 && !W_host) return fail(PB_EINVAL, "W_host is NULL");
    if (pb_packed_bytes(rows, cols, layers) > 0 && (!dst || !aligned(dst, 16)))
        return fail(PB_EINVAL, "dst must be non-NULL and 16-byte aligned");
    if (quant_mode == PB_Q_BINARY) {
        if (layers != 1) return fail(PB_EINVAL, "PB_Q_BINARY needs layers == 1");
    } else if (quant_mode == PB_Q_GRID || quant_mode == PB_Q_ALG1) {
        if (layers < 2 || layers > 16) return fail(PB_EINVAL, "layers=%d not in [2,16]", layers);
    } else {
        return fail(PB_EINVAL, "unknown quant_mode %d", quant_mode);
    }
    const int64_t n = rows * cols;
    QuantOut q;
    pb_status st = PB_OK;
    if (n == 0) {
        q.scale = 1.0;
        q.offset = quant_mode == PB_Q_BINARY ? 1 : 0;
        q.degenerate = true;
    } else if (quant_mode == PB_Q_GRID) {
        st = quantize_grid(W_host, n, layers, clip, q);
    } else if (quant_mode == PB_Q_ALG1) {
        st = quantize_alg1(W_host, n, layers, clip, q);
    } else {
        st = quantize_binary(W_host, n, clip, q);
    }
    if (st != PB_OK) return st;
    std::vector<uint32_t> host;
    if (n == 0) {
        host.assign(pb_packed_bytes(rows, cols, layers) / 4, 0u);
    } else if ((st = pack(q.codes.data(), rows, cols, layers, q.offset, host)) != PB_OK) {
        return st;
    }
    st = store(host, rows, cols, layers, q.offset, q.scale, dst, dst_is_device, s, out);
    if (st != PB_OK) return st;
    if (q.degenerate) {
        fail(PB_EDEGENERATE, "max(W) == min(W): degenerate grid (reading G5)");
        return PB_EDEGENERATE;
    }
    return PB_OK;
}

size_t pb_pack_device_workspace_bytes(void) { return pb::align_up(sizeof(float) * 2 * pb::kPackBlocks); }

pb_status pb_quantize_pack_weights_device(const float* W_dev, int64_t rows, int64_t cols, int32_t layers,
                                          float clip, double step, void* dst, void* ws, size_t ws_bytes,
                                          pb_stream s, pb_weights* out) {
    g_err[0] = 0;
    if (!out) return fail(PB_EINVAL, "out is NULL");
    if (rows < 0 || cols < 0) return fail(PB_EINVAL, "negative rows/cols");
    if (layers < 2 || layers > 16) return fail(PB_EINVAL, "layers=%d not in [2,16] (PB_Q_GRID)", layers);
    if (step < 0.0 || !std::isfinite(step)) return fail(PB_EINVAL, "step must be 0 (from the extrema) or > 0");
    const int64_t n = rows * cols;
    if (n > 0 && !W_dev) return fail(PB_EINVAL, "W_dev is NULL");
    if (pb_packed_bytes(rows, cols, layers) > 0 && (!dst || !aligned(dst, 16)))
        return fail(PB_EINVAL, "dst must be non-NULL and 16-byte aligned");
    if (step == 0.0 && n > 0 && (!ws || !aligned(ws, 16) || ws_bytes < pb_pack_device_workspace_bytes()))
        return fail(PB_EINVAL, "workspace < pb_pack_device_workspace_bytes()");
    const cudaStream_t cs = static_cast<cudaStream_t>(s);
    double d = step;
    bool deg = false, all_zero = false;
    if (n == 0) {
        d = 1.0;
        deg = true;
    } else if (step == 0.0) {
        // Q(W) grid from the exact float extrema (clip is monotonic: applied after)
        int blocks = (int)((n + 256 * 64 - 1) / (256 * 64));
        blocks = blocks < 1 ? 1 : (blocks > pb::kPackBlocks ? pb::kPackBlocks : blocks);
        float* part = static_cast<float*>(ws);
        cudaError_t e = pb::launch_minmax(W_dev, n, part, blocks, cs);
        std::vector<float> h((size_t)2 * blocks);
        if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), part, sizeof(float) * h.size(), cudaMemcpyDeviceToHost, cs);
        if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
        if (e != cudaSuccess) return cuda_fail(e, "pack: min/max");
        float fmn = INFINITY, fmx = -INFINITY;
        for (int b = 0; b < blocks; ++b) {
            fmn = std::fmin(fmn, h[2 * b]);
            fmx = std::fmax(fmx, h[2 * b + 1]);
        }
        const double mn = clipv((double)fmn, clip), mx = clipv((double)fmx, clip);
        d = grid_step(mn, mx, layers - 1, deg);
        all_zero = deg && mx == 0.0 && mn == 0.0;
    }
    if (n > 0) {
        cudaError_t e = pb::launch_pack_grid(W_dev, rows, cols, pb_kwords(cols), layers, d,
                                             step == 0.0 ? (double)clip : 0.0, all_zero ? 1 : 0,
                                             static_cast<uint32_t*>(dst), cs);
        if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
        if (e != cudaSuccess) return cuda_fail(e, "pack: bitlayers");
    } else if (pb_packed_bytes(rows, cols, layers) > 0) {
        cudaError_t e = cudaMemsetAsync(dst, 0, pb_packed_bytes(rows, cols, layers), cs);
        if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
        if (e != cudaSuccess) return cuda_fail(e, "pack: zero fill");
    }
    out->bits = static_cast<uint32_t*>(dst);
    out->rows = rows;
    out->cols = cols;
    out->kwords = pb_kwords(cols);
    out->layers = layers;
    out->offset = 0;
    out->scale = all_zero ? 1.0 : d;
    if (deg && step == 0.0) {
        fail(PB_EDEGENERATE, "max(W) == min(W): degenerate grid (reading G5)");
        return PB_EDEGENERATE;
    }
    return PB_OK;
}

pb_status pb_grid_step(double w_min, double w_max, int32_t layers, double* step) {
    g_err[0] = 0;
    if (!step) return fail(PB_EINVAL, "step is NULL");
    if (layers < 2 || layers > 16) return fail(PB_EINVAL, "layers=%d not in [2,16]", layers);
    if (!std::isfinite(w_min) || !std::isfinite(w_max) || w_min > w_max)
        return fail(PB_EINVAL, "extrema must be finite with min <= max");
    bool deg = false;
    *step = grid_step(w_min, w_max, layers - 1, deg);
    if (deg) {
        fail(PB_EDEGENERATE, "max(W) == min(W): degenerate grid (reading G5)");
        return PB_EDEGENERATE;
    }
    return PB_OK;
}

pb_status pb_quantize_pack_weights_step(const float* W_host, int64_t rows, int64_t cols, int32_t layers,
                                        double step, void* dst, int32_t dst_is_device, pb_stream s,
                                        pb_weights* out) {
    g_err[0] = 0;
    if (!out) return fail(PB_EINVAL, "out is NULL");
    if (rows < 0 || cols < 0) return fail(PB_EINVAL, "negative rows/cols");
    if (rows * cols > 0 && !W_host) return fail(PB_EINVAL, "W_host is NULL");
    if (layers < 2 || layers > 16) return fail(PB_EINVAL, "layers=%d not in [2,16]", layers);
    if (!(step > 0.0) || !std::isfinite(step)) return fail(PB_EINVAL, "step must be finite and > 0");
    if (pb_packed_bytes(rows, cols, layers) > 0 && (!dst || !aligned(dst, 16)))
        return fail(PB_EINVAL, "dst must be non-NULL and 16-byte aligned");
    const int64_t n = rows * cols;
    const double lo = -std::ldexp(1.0, layers - 1), hi = std::ldexp(1.0, layers - 1) - 1.0;
    std::vector<int32_t> codes((size_t)n);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < n; ++e) {
        double m = std::rint((double)W_host[e] / step);
        m = m < lo ? lo : (m > hi ? hi : m);
        codes[(size_t)e] = (int32_t)m;
    }
    std::vector<uint32_t> host;
    pb_status st = pack(codes.data(), rows, cols, layers, 0, host);
    if (st != PB_OK) return st;
    return store(host, rows, cols, layers, 0, step, dst, dst_is_device, s, out);
}

pb_status pb_pack_codes(const int32_t* codes_host, int64_t rows, int64_t cols, int32_t layers,
                        int32_t offset, double scale, void* dst, int32_t dst_is_device, pb_stream s,
                        pb_weights* out) {
    g_err[0] = 0;
    if (!out) return fail(PB_EINVAL, "out is NULL");
    if (layers < 1 || layers > 16) return fail(PB_EINVAL, "layers=%d not in [1,16]", layers);
    if (offset != 0 && !(offset == 1 && layers == 1)) return fail(PB_EINVAL, "offset needs layers == 1");
    if (rows < 0 || cols < 0) return fail(PB_EINVAL, "negative rows/cols");
    if (rows * cols > 0 && !codes_host) return fail(PB_EINVAL, "codes_host is NULL");
    if (pb_packed_bytes(rows, cols, layers) > 0 && (!dst || !aligned(dst, 16)))
        return fail(PB_EINVAL, "dst must be non-NULL and 16-byte aligned");
    std::vector<uint32_t> host;
    pb_status st = pack(codes_host, rows, cols, layers, offset, host);
    if (st != PB_OK) return st;
    return store(host, rows, cols, layers, offset, scale, dst, dst_is_device, s, out);
}

pb_status pb_search_clip(const float* W_host, int64_t rows, int64_t cols, int32_t layers, float* clip_out) {
    g_err[0] = 0;
    if (!W_host || !clip_out || rows * cols <= 0) return fail(PB_EINVAL, "bad arguments");
    if (layers < 2 || layers > 16) return fail(PB_EINVAL, "layers=%d not in [2,16]", layers);
    const int64_t n = rows * cols;
    double mx = 0.0;
    for (int64_t e = 0; e < n; ++e) mx = std::fabs((double)W_host[e]) > mx ? std::fabs((double)W_host[e]) : mx;
    if (mx == 0.0) {
        *clip_out = 0.f;
        return fail(PB_EDEGENERATE, "all-zero W");
    }
    constexpr int kCand = 64;
    double best = INFINITY;
    float best_t = (float)mx;
    QuantOut q;
    for (int k = 1; k <= kCand; ++k) {
        const float t = (float)((double)k / (double)kCand * mx);
        quantize_grid(W_host, n, layers, (double)t, q);
        double err = 0.0;
        for (int64_t e = 0; e < n; ++e) err += std::fabs(q.scale * (double)q.codes[(size_t)e] - (double)W_host[e]);
        err /= (double)n;
        if (err <= best) {
            best = err;
            best_t = t;
        }
    }
    *clip_out = best_t;
    return PB_OK;
}

size_t pb_workspace_bytes(int64_t batch, int64_t cols, int32_t act_bits) {
    if (batch < 0 || cols < 0 || act_bits < 1 || act_bits > 32) return 0;
    return pb::ws_layout(batch, pb_kwords(cols), act_bits).total;
}

pb_status pb_act_quantize(const float* x, int64_t batch, int64_t cols, int32_t act_bits, int32_t act_frac,
                          void* ws, size_t ws_bytes, pb_stream s) {
    g_err[0] = 0;
    pb_status st = check_act(batch, cols, act_bits, act_frac);
    if (st != PB_OK) return st;
    if ((st = check_ws(ws, ws_bytes, batch, cols, act_bits)) != PB_OK) return st;
    if (batch * cols > 0 && (!x || !aligned(x, 4))) return fail(PB_EINVAL, "x must be a non-NULL device pointer");
    const pb::WsLayout l = pb::ws_layout(batch, pb_kwords(cols), act_bits);
    cudaError_t e = pb::launch_act_quant(x, batch, cols, pb_kwords(cols), act_bits, act_frac, ws, l,
                                         static_cast<cudaStream_t>(s));
    if (e != cudaSuccess) return cuda_fail(e, "act_quant_transpose launch");
    return PB_OK;
}

// One matvec's knobs: the descriptor, k_used in [1, L] (reading G12) and the int64
// accumulator bound of reading G11, |acc| <= K 2^(L-1) 2^(a-1) (+ K 2^(a-1) for the offset)
// < 2^63.  Checked before any launch by every entry point that runs the matvec.
static pb_status check_matvec(const pb_weights* w, int32_t k_used, int32_t act_bits, const char* what) {
    pb_status st = check_weights(w);
    if (st != PB_OK) return st;
    if (k_used < 1 || k_used > w->layers)
        return fail(PB_EINVAL, "%s: k_used=%d not in [1,%d]", what, k_used, w->layers);
    if (act_bits < 1 || act_bits > 32) return fail(PB_EINVAL, "act_bits=%d not in [1,32]", act_bits);
    const int bound = ceil_log2(w->cols > 1 ? w->cols : 1) + w->layers + act_bits - 2 + (w->offset ? 1 : 0);
    if (bound > 62) return fail(PB_ERANGE, "%s: accumulator bound 2^%d exceeds int64 (reading G11)", what, bound + 1);
    return PB_OK;
}

static pb_status validate_gemm(const void* ws, size_t ws_bytes, int64_t batch, const pb_weights* w,
                               int32_t k_used, int32_t act_bits, const float* y, const int64_t* acc,
                               int32_t fn) {
    pb_status st = check_weights(w);
    if (st != PB_OK) return st;
    if ((st = check_act(batch, w->cols, act_bits, PB_ACT_AUTO)) != PB_OK) return st;
    if ((st = check_ws(ws, ws_bytes, batch, w->cols, act_bits)) != PB_OK) return st;
    if ((st = check_matvec(w, k_used, act_bits, "W")) != PB_OK) return st;
    if (fn < PB_FN_NONE || fn > PB_FN_SIGMOID) return fail(PB_EINVAL, "fn=%d unknown", fn);
    if (batch * w->rows > 0 && (!y || !aligned(y, 4))) return fail(PB_EINVAL, "y must be a non-NULL device pointer");
    if (acc && !aligned(acc, 8)) return fail(PB_EINVAL, "acc must be 8-byte aligned");
    return PB_OK;
}

// Steps a3-a5 (and, when x is given and the tensor engine takes the shape, a1-a2
// fused into the same kernel).  Returns PB_EINVAL with *fused_done = false when x
// is given but the fused path does not apply (the caller then runs a1-a2 first).
// Fused LSTM cell operands of one pb_lstm_seq step (GemmArgs cell mode), or null.
struct CellOut {
    int64_t H;
    const float* c;     // [B][H]
    float* h_out;       // [B][H]
    float* c_out;       // [B][H]
};

// Fused all-gather operands of pb_matmul_rowshard_p2p (GemmArgs nranks > 0), or null.
struct P2POut {
    int nranks;
    int64_t R_total, row0;
    float* peer_y[pb::kMaxRanks];
    unsigned long long* peer_ctr[pb::kMaxRanks];
    unsigned long long* local_ctr;
};

static pb_status run_gemm(const void* ws, int64_t batch, const pb_weights* w, int32_t k_used, int32_t act_bits,
                          float* y, int64_t* acc, const float* bias, int32_t fn, int32_t accumulate, pb_stream s,
                          const float* x, int32_t act_frac, bool* fused_done, const CellOut* cell = nullptr,
                          const P2POut* p2p = nullptr, bool midpoint = false) {
    if (fused_done) *fused_done = false;

    const pb::WsLayout l = pb::ws_layout(batch, w->kwords, act_bits);
    char* base = static_cast<char*>(const_cast<void*>(ws));
    pb::GemmArgs g;
    g.bits = w->bits;
    g.R = w->rows;
    g.kwords = w->kwords;
    g.L = w->layers;
    g.offset = w->offset;
    g.k_used = k_used;
    g.a = act_bits;
    g.scale = w->scale;
    g.planes = reinterpret_cast<const uint32_t*>(base + l.off_planes);
    g.f = reinterpret_cast<int32_t*>(base + l.off_f);
    g.xsum = reinterpret_cast<long long*>(base + l.off_xsum);
    g.nsplit = pb::act_nsplit(w->kwords);
    g.B = batch;
    g.bs = (int)batch;
    g.y = y;
    g.acc = reinterpret_cast<long long*>(acc);
    g.bias = bias;
    g.fn = fn;
    g.accumulate = accumulate ? 1 : 0;
    g.mid = (midpoint && k_used < w->layers && !w->offset) ? (1ull << (w->layers - k_used - 1)) : 0ull;
    g.npad = pb::tc_npad(batch, act_bits);     // whole batch in one tensor-engine launch (else 0)
    if (!g.npad && l.wbs && !x) {              // wide mode: every 128-column slice in one launch
        g.npad = pb::kTcWideN;
        g.bs = l.wbs;
    }
    g.bexp = reinterpret_cast<uint8_t*>(base + l.off_bexp);
    g.accbuf = reinterpret_cast<unsigned long long*>(base + l.off_slots);
    g.counters = reinterpret_cast<int*>(base + l.off_count);
    g.tl = pb::debug_tl();
    g.x = nullptr;
    g.K = w->cols;
    g.act_frac = act_frac;
    g.gbar = g.counters + pb::kMaxTiles;
    g.work = g.counters + pb::kMaxTiles + 2;
    g.ebar = g.counters + pb::kMaxTiles + 4;
    g.cell = 0;
    g.H = 0;
    g.cell_c = nullptr;
    g.cell_h = nullptr;
    g.cell_c_out = nullptr;
    g.nranks = 0;
    g.R_total = 0;
    g.row0 = 0;
    for (int q = 0; q < pb::kMaxRanks; ++q) {
        g.peer_y[q] = nullptr;
        g.peer_ctr[q] = nullptr;
    }
    g.local_ctr = nullptr;

    cudaError_t e;
    const cudaStream_t cs = static_cast<cudaStream_t>(s);
    if (x) {
        // fused a1-a5, one launch per batch slice of <= 64 plane columns (pb::tc_slice); every
        // slice must fit the tensor engine, else the caller runs the split path
        if (g_engine == PB_ENGINE_POPC) return PB_EINVAL;
        // the widest slice whose launches all fit the engine (more accumulator groups leave
        // fewer TMEM columns for the A ring, so a wide N may need a narrower slice)
        pb::GemmArgs gs = g;
        auto slices_fit = [&](int64_t bs) {
            for (int64_t b0 = 0; b0 < batch; b0 += bs) {
                gs.B = batch - b0 < bs ? batch - b0 : bs;
                gs.bs = (int)gs.B;
                gs.npad = pb::tc_npad(gs.B, act_bits);
                if (!pb::tc_supported(gs)) return false;
            }
            return true;
        };
        int64_t bs = pb::tc_slice(batch, act_bits);
        while (bs > 1 && !slices_fit(bs)) bs = (bs + 1) / 2;
        if (!slices_fit(bs)) return PB_EINVAL;
        for (int64_t b0 = 0; b0 < batch; b0 += bs) {
            gs.B = batch - b0 < bs ? batch - b0 : bs;
            gs.bs = (int)gs.B;
            gs.npad = pb::tc_npad(gs.B, act_bits);
            gs.x = x + b0 * w->cols;
            gs.y = y + b0 * w->rows;
            gs.acc = acc ? reinterpret_cast<long long*>(acc) + b0 * w->rows : nullptr;
            gs.f = g.f + b0;
            gs.xsum = g.xsum + b0 * pb::kXsumStride;
            if (p2p) {
                gs.nranks = p2p->nranks;
                gs.R_total = p2p->R_total;
                gs.row0 = p2p->row0;
                for (int q = 0; q < p2p->nranks; ++q) {
                    gs.peer_y[q] = p2p->peer_y[q] + b0 * p2p->R_total;
                    gs.peer_ctr[q] = p2p->peer_ctr[q];
                }
                gs.local_ctr = p2p->local_ctr;
            }
            if (cell) {
                gs.cell = 1;
                gs.H = cell->H;
                gs.cell_c = cell->c + b0 * cell->H;
                gs.cell_h = cell->h_out + b0 * cell->H;
                gs.cell_c_out = cell->c_out + b0 * cell->H;
            }
            e = pb::launch_gemm_tc(gs, cs);
            if (e != cudaSuccess) return cuda_fail(e, "fused bitgemm launch");
        }
        *fused_done = true;
        return PB_OK;
    }
    if (p2p) return PB_EINVAL;                   // peer all-gather: the tensor engine's fused path only
    if (cell) {                                  // the cell needs the tensor engine's finalisation
        if (g_engine == PB_ENGINE_POPC || !pb::tc_supported(g)) return PB_EINVAL;
        g.cell = 1;
        g.H = cell->H;
        g.cell_c = cell->c;
        g.cell_h = cell->h_out;
        g.cell_c_out = cell->c_out;
        e = pb::launch_gemm_tc(g, cs);
        if (e != cudaSuccess) return cuda_fail(e, "bitgemm (cell) launch");
        return PB_OK;
    }
    if (g_engine == PB_ENGINE_MMA) {
        if (!pb::tc_supported(g))
            return fail(PB_EINVAL, "PB_ENGINE_MMA on the split path needs act_bits*batch <= 64, batch <= 32 "
                                   "and rows <= 262144");
        e = pb::launch_gemm_tc(g, cs);
    } else if (g_engine == PB_ENGINE_AUTO && pb::tc_supported(g)) {
        e = pb::launch_gemm_tc(g, cs);
    } else {
        e = pb::launch_gemv_popc(g, cs);
    }
    if (e != cudaSuccess) return cuda_fail(e, "bitgemm launch");
    return PB_OK;
}

pb_status pb_bitgemm(const void* ws, size_t ws_bytes, int64_t batch, const pb_weights* w, int32_t k_used,
                     int32_t act_bits, float* y, int64_t* acc, const float* bias, int32_t fn,
                     int32_t accumulate, pb_stream s) {
    g_err[0] = 0;
    pb_status st = validate_gemm(ws, ws_bytes, batch, w, k_used, act_bits, y, acc, fn);
    if (st != PB_OK) return st;
    if (batch == 0 || w->rows == 0) return PB_OK;
    return run_gemm(ws, batch, w, k_used, act_bits, y, acc, bias, fn, accumulate, s, nullptr, 0, nullptr);
}

// a1-a5: one fused tensor-engine kernel when it takes the shape, else the
// activation kernel followed by pb_bitgemm's engine.
// Whether a launch of nb batch columns fits the tensor engine (pb_gemm_tc.cu make_plan).
static bool tc_fits(const pb_weights* w, int64_t nb, int32_t k_used, int32_t act_bits) {
    pb::GemmArgs g{};
    g.R = w->rows;
    g.kwords = w->kwords;
    g.L = w->layers;
    g.k_used = k_used;
    g.a = act_bits;
    g.B = nb;
    g.bs = (int)nb;
    g.npad = pb::tc_npad(nb, act_bits);
    return g.npad > 0 && pb::tc_supported(g);
}

// Whether a batch of nb columns runs in wide mode (one launch, 128-column slices).
static bool tc_fits_wide(const pb_weights* w, int64_t nb, int32_t k_used, int32_t act_bits) {
    pb::GemmArgs g{};
    g.R = w->rows;
    g.kwords = w->kwords;
    g.L = w->layers;
    g.k_used = k_used;
    g.a = act_bits;
    g.B = nb;
    g.bs = pb::tc_wide_bs(nb, act_bits);
    g.npad = pb::kTcWideN;
    return g.bs > 0 && pb::tc_supported(g);
}

static pb_status act_and_gemm(const float* x, int64_t batch, const pb_weights* w, int32_t k_used, int32_t act_bits,
                              int32_t act_frac, const float* bias, int32_t fn, float* y, int64_t* acc, void* ws,
                              size_t ws_bytes, pb_stream s, bool midpoint = false) {
    pb_status st = validate_gemm(ws, ws_bytes, batch, w, k_used, act_bits, y, acc, fn);
    if (st != PB_OK) return st;
    if ((st = check_act(batch, w->cols, act_bits, act_frac)) != PB_OK) return st;
    if (batch == 0 || w->rows == 0) return PB_OK;
    if (!x || !aligned(x, 4)) return fail(PB_EINVAL, "x must be a non-NULL device pointer");
    // Batches wider than one tensor-engine launch: one planes launch + one GEMM launch per
    // slice (measured 11-13% faster than fused slices, whose prologues redo the per-column
    // work on every CTA); PB_SLICE_SPLIT=0 keeps the fused slices
    static int slice_split = -1;
    if (slice_split < 0) {
        const char* ev = getenv("PB_SLICE_SPLIT");
        slice_split = ev ? atoi(ev) : 1;
    }
    if (g_engine != PB_ENGINE_POPC && pb::tc_npad(batch, act_bits) == 0 && tc_fits_wide(w, batch, k_used, act_bits)) {
        // wide mode: planes + operand tiles of every column in one launch, then one
        // tensor-engine launch over all 128-column slices
        if ((st = pb_act_quantize(x, batch, w->cols, act_bits, act_frac, ws, ws_bytes, s)) != PB_OK) return st;
        return run_gemm(ws, batch, w, k_used, act_bits, y, acc, bias, fn, 0, s, nullptr, 0, nullptr, nullptr, nullptr,
                        midpoint);
    }
    if (slice_split && batch > 1 && g_engine != PB_ENGINE_POPC && tc_fits(w, batch, k_used, act_bits)) {
        // a batch that fits one narrow launch: planes kernel + one GEMM launch (the fused
        // prologue's per-column work on every CTA is the longer path once batch > 1)
        if ((st = pb_act_quantize(x, batch, w->cols, act_bits, act_frac, ws, ws_bytes, s)) != PB_OK) return st;
        return run_gemm(ws, batch, w, k_used, act_bits, y, acc, bias, fn, 0, s, nullptr, 0, nullptr, nullptr, nullptr,
                        midpoint);
    }
    int64_t bs = pb::tc_slice(batch, act_bits);
    while (bs > 1 && !tc_fits(w, bs, k_used, act_bits)) bs = (bs + 1) / 2;   // as the fused path narrows
    if (slice_split && bs < batch && g_engine != PB_ENGINE_POPC && tc_fits(w, bs, k_used, act_bits) &&
        tc_fits(w, batch % bs ? batch % bs : bs, k_used, act_bits)) {
        // one planes launch + one tensor-engine launch per slice of bs columns
        for (int64_t b0 = 0; b0 < batch; b0 += bs) {
            const int64_t nb = batch - b0 < bs ? batch - b0 : bs;
            if ((st = pb_act_quantize(x + b0 * w->cols, nb, w->cols, act_bits, act_frac, ws, ws_bytes, s)) != PB_OK)
                return st;
            st = run_gemm(ws, nb, w, k_used, act_bits, y + b0 * w->rows, acc ? acc + b0 * w->rows : nullptr,
                          bias, fn, 0, s, nullptr, 0, nullptr, nullptr, nullptr, midpoint);
            if (st != PB_OK) return st;
        }
        return PB_OK;
    }
    bool fused = false;
    st = run_gemm(ws, batch, w, k_used, act_bits, y, acc, bias, fn, 0, s, x, act_frac, &fused, nullptr, nullptr,
                  midpoint);
    if (fused || (st != PB_OK && st != PB_EINVAL)) return st;
    if ((st = pb_act_quantize(x, batch, w->cols, act_bits, act_frac, ws, ws_bytes, s)) != PB_OK) return st;
    return run_gemm(ws, batch, w, k_used, act_bits, y, acc, bias, fn, 0, s, nullptr, 0, nullptr, nullptr, nullptr,
                    midpoint);
}

pb_status pb_matmul(const float* x, int64_t batch, const pb_weights* w, int32_t k_used, int32_t act_bits,
                    int32_t act_frac, float* y, int64_t* acc, void* ws, size_t ws_bytes, pb_stream s) {
    g_err[0] = 0;
    return act_and_gemm(x, batch, w, k_used, act_bits, act_frac, nullptr, PB_FN_NONE, y, acc, ws, ws_bytes, s);
}

pb_status pb_matmul_ex(const float* x, int64_t batch, const pb_weights* w, int32_t k_used, int32_t act_bits,
                       int32_t act_frac, int32_t flags, float* y, int64_t* acc, void* ws, size_t ws_bytes,
                       pb_stream s) {
    g_err[0] = 0;
    if (flags & ~PB_MM_MIDPOINT) return fail(PB_EINVAL, "unknown flags 0x%x", flags);
    return act_and_gemm(x, batch, w, k_used, act_bits, act_frac, nullptr, PB_FN_NONE, y, acc, ws, ws_bytes, s,
                        (flags & PB_MM_MIDPOINT) != 0);
}

pb_status pb_linear(const float* x, int64_t batch, const pb_weights* w, int32_t k_used, int32_t act_bits,
                    int32_t act_frac, const float* bias, int32_t fn, float* y, void* ws, size_t ws_bytes,
                    pb_stream s) {
    g_err[0] = 0;
    return act_and_gemm(x, batch, w, k_used, act_bits, act_frac, bias, fn, y, nullptr, ws, ws_bytes, s);
}

size_t pb_cell_workspace_bytes(int64_t batch, int64_t in_cols, int64_t hidden, int32_t act_bits, int32_t gates) {
    const int64_t k = in_cols > hidden ? in_cols : hidden;
    const size_t a = pb_workspace_bytes(batch, k, act_bits);
    return pb::align_up(a) + pb::align_up(sizeof(float) * (size_t)batch * (size_t)gates * (size_t)hidden);
}

static pb_status cell_common(const float* x_t, const float* h, const pb_weights* w_ih, const pb_weights* w_hh,
                             const float* b_ih, const float* b_hh, int32_t k_ih, int32_t k_hh, int32_t a,
                             int64_t batch, int gates, void* ws, size_t ws_bytes, pb_stream s, float** gbuf,
                             bool outs_ok) {
    pb_status st;
    if ((st = check_matvec(w_ih, k_ih, a, "W_ih")) != PB_OK) return st;
    if ((st = check_matvec(w_hh, k_hh, a, "W_hh")) != PB_OK) return st;
    const int64_t H = w_hh->cols;
    if (w_ih->rows != gates * H || w_hh->rows != gates * H)
        return fail(PB_EINVAL, "W_ih/W_hh must have %d*H rows (H = W_hh cols = %lld)", gates, (long long)H);
    if ((st = check_act(batch, w_ih->cols > H ? w_ih->cols : H, a, PB_ACT_AUTO)) != PB_OK) return st;
    const size_t need = pb_cell_workspace_bytes(batch, w_ih->cols, H, a, gates);
    if (!ws || !aligned(ws, 16) || ws_bytes < need) return fail(PB_EINVAL, "cell workspace %zu < %zu", ws_bytes, need);
    if (!outs_ok) return fail(PB_EINVAL, "x/h and the outputs (h_out, and c/c_out for the LSTM) must be non-NULL");
    const int64_t k = w_ih->cols > H ? w_ih->cols : H;
    const size_t act_ws = pb::align_up(pb_workspace_bytes(batch, k, a));
    *gbuf = reinterpret_cast<float*>(static_cast<char*>(ws) + act_ws);
    // gates = (W_ih x + b_ih), then gates = (W_hh h + b_hh) + gates
    if ((st = pb_act_quantize(x_t, batch, w_ih->cols, a, PB_ACT_AUTO, ws, act_ws, s)) != PB_OK) return st;
    if ((st = pb_bitgemm(ws, act_ws, batch, w_ih, k_ih, a, *gbuf, nullptr, b_ih, PB_FN_NONE, 0, s)) != PB_OK) return st;
    if ((st = pb_act_quantize(h, batch, H, a, PB_ACT_AUTO, ws, act_ws, s)) != PB_OK) return st;
    return pb_bitgemm(ws, act_ws, batch, w_hh, k_hh, a, *gbuf, nullptr, b_hh, PB_FN_NONE, 1, s);
}

pb_status pb_rnn_step(const float* x_t, const float* h, const pb_weights* w_ih, const pb_weights* w_hh,
                      const float* b_ih, const float* b_hh, int32_t k_used_ih, int32_t k_used_hh, int32_t act_bits,
                      int64_t batch, float* h_out, void* ws, size_t ws_bytes, pb_stream s) {
    g_err[0] = 0;
    float* gates = nullptr;
    const bool outs = batch == 0 || (x_t && h && h_out);
    pb_status st = cell_common(x_t, h, w_ih, w_hh, b_ih, b_hh, k_used_ih, k_used_hh, act_bits, batch, 1, ws,
                               ws_bytes, s, &gates, outs);
    if (st != PB_OK) return st;
    cudaError_t e = pb::launch_rnn_cell(gates, batch, w_hh->cols, h_out, static_cast<cudaStream_t>(s));
    if (e != cudaSuccess) return cuda_fail(e, "rnn_cell launch");
    return PB_OK;
}

pb_status pb_lstm_step(const float* x_t, const float* h, const float* c, const pb_weights* w_ih,
                       const pb_weights* w_hh, const float* b_ih, const float* b_hh, int32_t k_used_ih,
                       int32_t k_used_hh, int32_t act_bits, int64_t batch, float* h_out, float* c_out, void* ws,
                       size_t ws_bytes, pb_stream s) {
    g_err[0] = 0;
    float* gates = nullptr;
    const bool outs = batch == 0 || (x_t && h && c && h_out && c_out);
    pb_status st = cell_common(x_t, h, w_ih, w_hh, b_ih, b_hh, k_used_ih, k_used_hh, act_bits, batch, 4, ws,
                               ws_bytes, s, &gates, outs);
    if (st != PB_OK) return st;
    cudaError_t e = pb::launch_lstm_cell(gates, c, batch, w_hh->cols, h_out, c_out, static_cast<cudaStream_t>(s));
    if (e != cudaSuccess) return cuda_fail(e, "lstm_cell launch");
    return PB_OK;
}

// ------------------------------------------------------------ LSTM sequence
size_t pb_lstm_seq_workspace_bytes(int64_t steps, int64_t batch, int64_t in_cols, int64_t hidden, int32_t act_bits) {
    if (steps < 0 || batch < 0 || in_cols < 0 || hidden < 0) return 0;
    const int64_t k = in_cols > hidden ? in_cols : hidden;
    const int64_t cols = steps * batch > batch ? steps * batch : batch;
    return pb::align_up(pb_workspace_bytes(cols, k, act_bits)) +
           pb::align_up(sizeof(float) * (size_t)cols * 4 * (size_t)hidden) +
           2 * pb::align_up(sizeof(float) * (size_t)batch * (size_t)hidden) +
           pb::align_up(sizeof(unsigned long long) * 2 * pb::kLstmMaxB) +   // persistent kernel: max|h| slots
           pb::lstm_xchg_bytes(hidden);                                     // B = 1 tagged h exchange
}

pb_status pb_lstm_seq(const float* x, int64_t steps, int64_t batch, const float* h0, const float* c0,
                      const pb_weights* w_ih, const pb_weights* w_hh, const float* bias, int32_t k_used_ih,
                      int32_t k_used_hh, int32_t act_bits, float* h_seq, float* c_seq, float* c_last, void* ws,
                      size_t ws_bytes, pb_stream s) {
    g_err[0] = 0;
    pb_status st;
    if ((st = check_matvec(w_ih, k_used_ih, act_bits, "W_ih")) != PB_OK) return st;
    if ((st = check_matvec(w_hh, k_used_hh, act_bits, "W_hh")) != PB_OK) return st;
    const int64_t H = w_hh->cols, E = w_ih->cols;
    if (w_ih->rows != 4 * H || w_hh->rows != 4 * H)
        return fail(PB_EINVAL, "W_ih/W_hh must have 4*H rows (H = W_hh cols = %lld)", (long long)H);
    if (steps < 0 || batch < 0) return fail(PB_EINVAL, "steps/batch < 0");
    if (steps * batch > 65535)
        return fail(PB_EINVAL, "steps*batch=%lld > 65535 (the hoisted input projection is one batched call)",
                    (long long)(steps * batch));
    if (steps == 0 || batch == 0 || H == 0) return PB_OK;
    if (!x || !h0 || !c0 || !h_seq || !c_last) return fail(PB_EINVAL, "x/h0/c0/h_seq/c_last is NULL");
    const size_t need = pb_lstm_seq_workspace_bytes(steps, batch, E, H, act_bits);
    if (!ws || !aligned(ws, 16) || ws_bytes < need) return fail(PB_EINVAL, "lstm_seq workspace %zu < %zu", ws_bytes, need);
    const int64_t k = E > H ? E : H;
    const int64_t cols = steps * batch;
    const size_t act_ws = pb::align_up(pb_workspace_bytes(cols, k, act_bits));
    char* base = static_cast<char*>(ws);
    float* gx = reinterpret_cast<float*>(base + act_ws);
    float* cb[2];
    cb[0] = reinterpret_cast<float*>(base + act_ws + pb::align_up(sizeof(float) * (size_t)cols * 4 * (size_t)H));
    cb[1] = cb[0] + pb::align_up(sizeof(float) * (size_t)batch * (size_t)H) / sizeof(float);
    // 1. the input projection of every timestep in one batched call (GEMM regime):
    //    gx[t][b] = W_ih x[t][b] + bias (gate-interleaved rows)
    if ((st = act_and_gemm(x, cols, w_ih, k_used_ih, act_bits, PB_ACT_AUTO, bias, PB_FN_NONE, gx, nullptr, ws,
                           act_ws, s)) != PB_OK)
        return st;
    // 2. the recurrence: all T timesteps in ONE persistent tensor-engine launch (a grid barrier
    //    per timestep, pb_lstm_tc.cu) when W_hh's units fit the SMs at once; PB_LSTM_PERSIST=0
    //    selects the per-timestep launches below
    const char* pev = getenv("PB_LSTM_PERSIST");      // comparison knob, read per call
    const int persist_env = pev ? atoi(pev) : 1;
    if (persist_env && g_engine != PB_ENGINE_POPC) {
        pb::LstmArgs la{};
        la.bits = w_hh->bits;
        la.R = w_hh->rows;
        la.kwords = w_hh->kwords;
        la.H = H;
        la.L = w_hh->layers;
        la.offset = w_hh->offset;
        la.k_used = k_used_hh;
        la.a = act_bits;
        la.scale = w_hh->scale;
        la.B = (int)batch;
        la.T = (int)steps;
        la.h0 = h0;
        la.c0 = c0;
        la.gx = gx;
        la.h_seq = h_seq;
        la.c_seq = c_seq;
        la.c_last = c_last;
        la.cbuf0 = cb[0];
        la.cbuf1 = cb[1];
        const pb::WsLayout lw = pb::ws_layout(cols, k > 0 ? pb_kwords(k) : 0, act_bits);
        la.counters = reinterpret_cast<int*>(base + lw.off_count);
        la.gbar = la.counters + pb::kMaxTiles;
        la.accbuf = reinterpret_cast<unsigned long long*>(base + lw.off_slots);
        la.tl = pb::debug_tl();
        la.maxslot = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(cb[1]) +
                                                           pb::align_up(sizeof(float) * (size_t)batch * (size_t)H));
        // [stepctr][pad to 256][mxs 2 x kLstmMaxTiles][hx 2 x H]
        char* xg = reinterpret_cast<char*>(la.maxslot) + pb::align_up(sizeof(unsigned long long) * 2 * pb::kLstmMaxB);
        la.stepctr = reinterpret_cast<unsigned long long*>(xg);
        la.mxs = reinterpret_cast<unsigned long long*>(xg + 256);
        la.hx = la.mxs + 2 * pb::kLstmMaxCtas * pb::kLstmMaxTiles;
        const bool room = (lw.npad || lw.wbs) &&
                          (size_t)((la.R + pb::kTcRows - 1) / pb::kTcRows) * (size_t)batch * pb::kTcRows * 8 <=
                              lw.off_f - lw.off_slots;
        if (room && H % 4 == 0 && batch <= pb::kLstmMaxB && pb::lstm_persist_supported(la)) {
            cudaError_t e = pb::launch_lstm_persist(la, static_cast<cudaStream_t>(s));
            if (e != cudaSuccess) return cuda_fail(e, "persistent lstm launch");
            return PB_OK;
        }
    }
    // 2. per timestep: W_hh h_t + gx[t], then the cell -- fused into the tensor engine's
    //    finalisation when the shape allows (one launch for batch 1; planes kernel + GEMM when
    //    a batch > 1 fits one tensor-engine launch: measured faster than the fused prologue's
    //    per-column work), else planes + GEMM + cell kernel
    static int split_env = -2;
    if (split_env == -2) {
        const char* ev = getenv("PB_LSTM_SPLIT");   // comparison knob: 0 = always fused, 1 = always split
        split_env = ev ? atoi(ev) : -1;
    }
    const bool split_first = split_env >= 0 ? split_env > 0
                                            : (batch > 1 && (pb::tc_npad(batch, act_bits) > 0 ||
                                                             tc_fits_wide(w_hh, batch, k_used_hh, act_bits)));
    for (int64_t t = 0; t < steps; ++t) {
        const float* h_in = t == 0 ? h0 : h_seq + (t - 1) * batch * H;
        const float* c_in = t == 0 ? c0 : (c_seq ? c_seq + (t - 1) * batch * H : cb[(t - 1) & 1]);
        float* h_out = h_seq + t * batch * H;
        float* c_out = c_seq ? c_seq + t * batch * H : (t == steps - 1 ? c_last : cb[t & 1]);
        float* gt = gx + t * batch * 4 * H;
        const CellOut co{H, c_in, h_out, c_out};
        bool fused = false;
        if (!split_first) {
            st = run_gemm(ws, batch, w_hh, k_used_hh, act_bits, gt, nullptr, nullptr, PB_FN_NONE, 1, s, h_in,
                          PB_ACT_AUTO, &fused, &co);
            if (st != PB_OK && st != PB_EINVAL) return st;
        }
        if (!fused) {
            // planes by the activation kernel, then the tensor engine with the cell in its
            // finalisation (batched h: the fused prologue's per-column work is the longer path)
            g_err[0] = 0;
            if ((st = pb_act_quantize(h_in, batch, H, act_bits, PB_ACT_AUTO, ws, act_ws, s)) != PB_OK) return st;
            st = run_gemm(ws, batch, w_hh, k_used_hh, act_bits, gt, nullptr, nullptr, PB_FN_NONE, 1, s, nullptr, 0,
                          nullptr, &co);
            if (st != PB_OK && st != PB_EINVAL) return st;
            fused = st == PB_OK;
        }
        if (!fused) {
            g_err[0] = 0;                        // planes are in ws already: GEMM, then the cell kernel
            if ((st = run_gemm(ws, batch, w_hh, k_used_hh, act_bits, gt, nullptr, nullptr, PB_FN_NONE, 1, s, nullptr,
                               0, nullptr)) != PB_OK)
                return st;
            cudaError_t e = pb::launch_lstm_cell_ilv(gt, c_in, batch, H, h_out, c_out, static_cast<cudaStream_t>(s));
            if (e != cudaSuccess) return cuda_fail(e, "lstm_cell_ilv launch");
        }
        if (c_seq && t == steps - 1) {
            cudaError_t e = cudaMemcpyAsync(c_last, c_out, sizeof(float) * (size_t)batch * (size_t)H,
                                            cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(s));
            if (e != cudaSuccess) return cuda_fail(e, "c_last copy");
        }
    }
    return PB_OK;
}

pb_status pb_set_engine(int32_t engine) {
    if (engine < PB_ENGINE_AUTO || engine > PB_ENGINE_MMA) return fail(PB_EINVAL, "engine=%d unknown", engine);
    g_engine = engine;
    return PB_OK;
}
int32_t pb_get_engine(void) { return g_engine; }

// ------------------------------------------------------------ diagnostics timeline

int64_t pb_debug_timeline(int64_t* dst, int64_t max_records) {
    long long* tl = pb::debug_tl();
    if (!tl) return -1;
    if (cudaDeviceSynchronize() != cudaSuccess) return -1;
    long long n = 0;
    if (cudaMemcpy(&n, tl, sizeof n, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    if (n > pb::kTlRecords) n = pb::kTlRecords;
    if (n > max_records) n = max_records;
    if (n > 0 && dst &&
        cudaMemcpy(dst, tl + 10, sizeof(long long) * 10 * (size_t)n, cudaMemcpyDeviceToHost) != cudaSuccess)
        return -1;
    cudaMemset(tl, 0, sizeof(long long));
    cudaDeviceSynchronize();
    return n;
}

// ------------------------------------------------------------ row sharding
pb_status pb_shard_rows(int64_t rows_total, int32_t nranks, int32_t rank, int64_t* row0, int64_t* nrows) {
    if (rows_total < 0 || nranks < 1 || rank < 0 || rank >= nranks || !row0 || !nrows)
        return fail(PB_EINVAL, "bad shard arguments");
    const int64_t rs = (rows_total + nranks - 1) / nranks;
    int64_t r0 = rs * rank;
    if (r0 > rows_total) r0 = rows_total;
    int64_t n = rows_total - r0;
    if (n > rs) n = rs;
    *row0 = r0;
    *nrows = n;
    return PB_OK;
}

}  // extern "C"

// NCCL is resolved at run time so that libpb loads (and the CPU tests run)
// without it; when torch has already loaded libnccl.so.2 we reuse that copy.
struct pb_comm {
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0;
};

namespace {
struct Nccl {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        n.AllGather = reinterpret_cast<decltype(n.AllGather)>(dlsym(h, "ncclAllGather"));
        n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
        n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.AllGather && n.GetErrorString;
    });
    return n;
}
pb_status nccl_fail(ncclResult_t r, const char* what) {
    return fail(PB_ENCCL, "%s: %s", what, nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error");
}
}  // namespace

extern "C" {

pb_status pb_comm_unique_id(void* id128) {
    g_err[0] = 0;
    if (!id128) return fail(PB_EINVAL, "id128 is NULL");
    if (!nccl().ok) return fail(PB_ENCCL, "libnccl.so.2 not loadable");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    ncclResult_t r = nccl().GetUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    std::memcpy(id128, &id, 128);
    return PB_OK;
}

pb_status pb_comm_init(pb_comm** comm, const void* id128, int32_t nranks, int32_t rank) {
    g_err[0] = 0;
    if (!comm || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return fail(PB_EINVAL, "bad comm arguments");
    if (!nccl().ok) return fail(PB_ENCCL, "libnccl.so.2 not loadable");
    ncclUniqueId id;
    std::memcpy(&id, id128, 128);
    pb_comm* c = new pb_comm;
    ncclResult_t r = nccl().CommInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_fail(r, "ncclCommInitRank");
    }
    c->nranks = nranks;
    c->rank = rank;
    *comm = c;
    return PB_OK;
}

pb_status pb_comm_destroy(pb_comm* comm) {
    if (!comm) return PB_OK;
    if (comm->comm && nccl().ok) nccl().CommDestroy(comm->comm);
    delete comm;
    return PB_OK;
}

size_t pb_rowshard_workspace_bytes(int64_t batch, int64_t cols, int32_t act_bits, int64_t rows_total,
                                   int32_t nranks) {
    if (nranks < 1) return 0;
    const int64_t rs = (rows_total + nranks - 1) / nranks;
    return pb::align_up(pb_workspace_bytes(batch, cols, act_bits)) +
           pb::align_up(sizeof(float) * (size_t)batch * (size_t)rs) +
           pb::align_up(sizeof(float) * (size_t)batch * (size_t)rs * (size_t)nranks);
}

pb_status pb_matmul_rowshard(const float* x, int64_t batch, const pb_weights* w_shard, int64_t rows_total,
                             int32_t k_used, int32_t act_bits, int32_t act_frac, float* y_full, pb_comm* comm,
                             void* ws, size_t ws_bytes, pb_stream s) {
    g_err[0] = 0;
    if (!comm) return fail(PB_EINVAL, "comm is NULL");
    pb_status st = check_weights(w_shard);
    if (st != PB_OK) return st;
    const int N = comm->nranks;
    const int64_t rs = (rows_total + N - 1) / N;
    if (w_shard->rows != rs)
        return fail(PB_EINVAL, "shard rows %lld != ceil(R/N) = %lld (pad the last shards with zero rows)",
                    (long long)w_shard->rows, (long long)rs);
    const size_t need = pb_rowshard_workspace_bytes(batch, w_shard->cols, act_bits, rows_total, N);
    if (!ws || !aligned(ws, 16) || ws_bytes < need) return fail(PB_EINVAL, "rowshard workspace %zu < %zu", ws_bytes, need);
    if (batch * rows_total > 0 && !y_full) return fail(PB_EINVAL, "y_full is NULL");
    const size_t act_ws = pb::align_up(pb_workspace_bytes(batch, w_shard->cols, act_bits));
    char* base = static_cast<char*>(ws);
    const cudaStream_t cs = static_cast<cudaStream_t>(s);
    if (batch == 1 && rs * N == rows_total) {
        // y_full is [R]: compute this rank's rows in place, all-gather in place.
        float* mine = y_full + (int64_t)comm->rank * rs;
        if ((st = pb_matmul(x, batch, w_shard, k_used, act_bits, act_frac, mine, nullptr, ws, act_ws, s)) != PB_OK)
            return st;
        ncclResult_t r = nccl().AllGather(mine, y_full, (size_t)rs, ncclFloat32, comm->comm, cs);
        if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
        return PB_OK;
    }
    float* ylocal = reinterpret_cast<float*>(base + act_ws);
    float* gathered = reinterpret_cast<float*>(base + act_ws + pb::align_up(sizeof(float) * (size_t)batch * rs));
    if ((st = pb_matmul(x, batch, w_shard, k_used, act_bits, act_frac, ylocal, nullptr, ws, act_ws, s)) != PB_OK)
        return st;
    ncclResult_t r = nccl().AllGather(ylocal, gathered, (size_t)(batch * rs), ncclFloat32, comm->comm, cs);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
    cudaError_t e = pb::launch_permute_shards(gathered, batch, rs, N, rows_total, y_full, cs);
    if (e != cudaSuccess) return cuda_fail(e, "permute launch");
    return PB_OK;
}

// ------------------------------------------------------------ fused peer all-gather (f2)
struct pb_p2p {
    int nranks = 0, rank = 0;
    int64_t batch = 0, rows_total = 0;
    char* local = nullptr;                  // [counter: 256 B][y_full: batch x rows_total float32]
    char* peer[pb::kMaxRanks] = {};         // opened IPC mappings (own rank: local)
    bool opened = false;
    bool borrowed = false;                  // peers opened in-process (pb_p2p_open_peers): nothing to close
};

static size_t p2p_bytes(int64_t batch, int64_t rows_total) {
    return 256 + pb::align_up(sizeof(float) * (size_t)batch * (size_t)rows_total);
}

pb_status pb_p2p_create(pb_p2p** out, int32_t nranks, int32_t rank, int64_t batch, int64_t rows_total,
                        void* handle_out) {
    g_err[0] = 0;
    if (!out || !handle_out) return fail(PB_EINVAL, "out/handle_out is NULL");
    if (nranks < 1 || nranks > pb::kMaxRanks || (nranks & (nranks - 1)))
        return fail(PB_EINVAL, "nranks=%d: 1, 2, 4 or 8 ranks of one node", nranks);
    if (rank < 0 || rank >= nranks) return fail(PB_EINVAL, "rank=%d not in [0,%d)", rank, nranks);
    if (batch < 1 || rows_total < 1) return fail(PB_EINVAL, "batch and rows_total must be >= 1");
    pb_p2p* p = new pb_p2p;
    p->nranks = nranks;
    p->rank = rank;
    p->batch = batch;
    p->rows_total = rows_total;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&p->local), p2p_bytes(batch, rows_total));
    if (e == cudaSuccess) e = cudaMemset(p->local, 0, p2p_bytes(batch, rows_total));
    cudaIpcMemHandle_t h;
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p->local);
    if (e != cudaSuccess) {
        if (p->local) cudaFree(p->local);
        delete p;
        return cuda_fail(e, "p2p buffer / IPC handle");
    }
    std::memcpy(handle_out, &h, sizeof h);
    *out = p;
    return PB_OK;
}

size_t pb_p2p_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

pb_status pb_p2p_open(pb_p2p* p, const void* handles) {
    g_err[0] = 0;
    if (!p || !handles) return fail(PB_EINVAL, "p2p/handles is NULL");
    if (p->opened) return PB_OK;
    for (int q = 0; q < p->nranks; ++q) {
        if (q == p->rank) {
            p->peer[q] = p->local;
            continue;
        }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const char*>(handles) + (size_t)q * sizeof h, sizeof h);
        void* ptr = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
        p->peer[q] = static_cast<char*>(ptr);
    }
    p->opened = true;
    return PB_OK;
}

pb_status pb_p2p_open_peers(pb_p2p* p, pb_p2p* const* all) {
    g_err[0] = 0;
    if (!p || !all) return fail(PB_EINVAL, "p2p/all is NULL");
    if (p->opened) return PB_OK;
    for (int q = 0; q < p->nranks; ++q) {
        if (!all[q] || all[q]->nranks != p->nranks || all[q]->rank != q || all[q]->batch != p->batch ||
            all[q]->rows_total != p->rows_total)
            return fail(PB_EINVAL, "peer %d does not match (nranks, rank, batch, rows_total)", q);
        p->peer[q] = all[q]->local;
    }
    p->opened = true;
    p->borrowed = true;
    return PB_OK;
}

float* pb_p2p_y(pb_p2p* p) { return p ? reinterpret_cast<float*>(p->local + 256) : nullptr; }

pb_status pb_p2p_destroy(pb_p2p* p) {
    if (!p) return PB_OK;
    cudaDeviceSynchronize();
    for (int q = 0; q < p->nranks; ++q)
        if (p->peer[q] && q != p->rank && !p->borrowed) cudaIpcCloseMemHandle(p->peer[q]);
    if (p->local) cudaFree(p->local);
    delete p;
    return PB_OK;
}

pb_status pb_matmul_rowshard_p2p(const float* x, int64_t batch, const pb_weights* w_shard, int64_t rows_total,
                                 int32_t k_used, int32_t act_bits, int32_t act_frac, pb_p2p* p, void* ws,
                                 size_t ws_bytes, pb_stream s) {
    g_err[0] = 0;
    if (!p || !p->opened) return fail(PB_EINVAL, "p2p is NULL or not opened (pb_p2p_open)");
    if (batch != p->batch || rows_total != p->rows_total)
        return fail(PB_EINVAL, "batch/rows_total differ from the p2p buffer's");
    pb_status st = validate_gemm(ws, ws_bytes, batch, w_shard, k_used, act_bits, pb_p2p_y(p), nullptr, PB_FN_NONE);
    if (st != PB_OK) return st;
    if ((st = check_act(batch, w_shard->cols, act_bits, act_frac)) != PB_OK) return st;
    const int N = p->nranks;
    const int64_t rs = (rows_total + N - 1) / N;
    if (w_shard->rows != rs)
        return fail(PB_EINVAL, "shard rows %lld != ceil(R/N) = %lld (pad the last shards with zero rows)",
                    (long long)w_shard->rows, (long long)rs);
    if (!x || !aligned(x, 4)) return fail(PB_EINVAL, "x must be a non-NULL device pointer");
    P2POut po;
    po.nranks = N;
    po.R_total = rows_total;
    po.row0 = rs * p->rank;
    for (int q = 0; q < N; ++q) {
        po.peer_y[q] = reinterpret_cast<float*>(p->peer[q] + 256);
        po.peer_ctr[q] = reinterpret_cast<unsigned long long*>(p->peer[q]);
    }
    po.local_ctr = reinterpret_cast<unsigned long long*>(p->local);
    bool fused = false;
    st = run_gemm(ws, batch, w_shard, k_used, act_bits, nullptr, nullptr, nullptr, PB_FN_NONE, 0, s, x, act_frac,
                  &fused, nullptr, &po);
    if (st == PB_OK && !fused) st = PB_EINVAL;
    if (st == PB_EINVAL && !g_err[0])
        return fail(PB_EINVAL, "the fused peer all-gather needs the tensor engine's fused path for this shape");
    return st;
}

}  // extern "C"
