/*
 * pb_oracle.c -- the CPU ORACLE for the PrecisionBatching bitlayer matvec.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (libpb.so, paper_2003_00822_b200/) never imports, links
 * or executes anything under oracle/, and this file shares no code, header,
 * table or constant generator with it.
 *
 * What it is: a plain, slow, literal CPU implementation of what the paper
 * (arXiv 2003.00822, "PrecisionBatching", /root/reference/PAPER.md = "P:n")
 * computes, in the paper's order:
 *   Alg. 1  weight quantisation Q(W) and bitlayer
 *                       decomposition with a negated sign layer;
 *   Alg. 2  activation fixed-point cast, bitwise
 *                       transpose into bitplanes, the
 *                       per-(weight bitlayer, activation bitplane) 0/1
 *                       products, the shift-weighted
 *                       reduction with [-2^(a-1) ... 2^0] and the
 *                       final rescale.
 * Every bit is stored in its own byte and every product is a plain loop.
 * Integers are accumulated in __int128 and checked to fit int64; floating
 * point is IEEE double (compile with -ffp-contract=off).
 *
 * Readings of the paper that this file takes are the SURVEY.md §8(c) ledger
 * entries G1..G16 and are listed in DESIGN.md ("Readings").  Each function
 * names the passage it follows.
 *
 * Parity pins (tests/test_oracle_pins.py): the Supplement §1 worked example
 * (P:386-467), exhaustive two's-complement identity, brute-force
 * integer matmul of the quantised values, the binary special case, k_used
 * truncation, Q(W) closed forms, the activation cast, convergence to float,
 * or_lstm_cell against PyTorch's nn.LSTMCell in float64 (reading G15).
 * parity unpinned: or_search_clip (G6: the paper fixes no candidate set; it
 * is checked only for the property "never worse than no clip").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_EINVAL 1
#define OR_ERANGE 2
#define OR_EDEGENERATE 3

/* ------------------------------------------------------------------------ */
/* Alg. 1 line 1 / §3.3: Q(W) = d * round(W / d),  d = (max(W)-min(W)) / 2^n
 * (P:148-150).  round = rint, ties to even (reading G4).  Optional clip t>0
 * clamps W to [-t, t] first ("optimize over a clipping threshold").
 * Writes Q (double) and d.  Returns OR_EDEGENERATE when max == min.        */
int or_quantize_round(const float* W, int64_t n_el, int n, double clip,
                      double* Q, double* d_out)
{
    if (!W || n_el <= 0 || n < 0 || n > 62) return OR_EINVAL;
    double mx = -INFINITY, mn = INFINITY;
    for (int64_t e = 0; e < n_el; ++e) {
        double w = (double)W[e];
        if (clip > 0) { if (w > clip) w = clip; if (w < -clip) w = -clip; }
        if (w > mx) mx = w;
        if (w < mn) mn = w;
    }
    double d = (mx - mn) / ldexp(1.0, n);
    int status = OR_OK;
    if (d == 0.0) {                       /* reading G5 */
        d = fabs(mx);
        status = OR_EDEGENERATE;
        if (d == 0.0) d = 1.0;
    }
    for (int64_t e = 0; e < n_el; ++e) {
        double w = (double)W[e];
        if (clip > 0) { if (w > clip) w = clip; if (w < -clip) w = -clip; }
        if (Q) Q[e] = d * rint(w / d);
    }
    if (d_out) *d_out = d;
    return status;
}

/* Integer codes of Q(W) on the L-bit two's-complement range (reading G1:
 * L = n+1 stored bitlayers, n = L-1; "[-2^n, 2^n - 1]").
 * code = clamp(rint(W/d)), scale s_w = d, so W ~= s_w * code.               */
int or_quantize_grid(const float* W, int64_t n_el, int L, double clip,
                     int32_t* codes, double* scale)
{
    if (!W || !codes || L < 2 || L > 16) return OR_EINVAL;
    double d;
    int status = or_quantize_round(W, n_el, L - 1, clip, NULL, &d);
    if (status == OR_EINVAL) return status;
    double lo = -ldexp(1.0, L - 1), hi = ldexp(1.0, L - 1) - 1.0;
    double mx = 0.0;
    for (int64_t e = 0; e < n_el; ++e) {
        double w = (double)W[e];
        if (clip > 0) { if (w > clip) w = clip; if (w < -clip) w = -clip; }
        if (fabs(w) > mx) mx = fabs(w);
        double m = rint(w / d);
        if (m < lo) m = lo;
        if (m > hi) m = hi;
        codes[e] = (int32_t)m;
    }
    if (status == OR_EDEGENERATE && mx == 0.0) {   /* all-zero W: zero codes, s_w = 1 */
        for (int64_t e = 0; e < n_el; ++e) codes[e] = 0;
        d = 1.0;
    }
    *scale = d;
    return status;
}

/* Alg. 1, literally, reading G2 for the index range:
 *   W_q     <- Int(QuantizeRound(W, n) * 2^16)            (Int = trunc, G4)
 *   max_bit <- max(log2(|W_q|))                            (floor)
 *   bitlayers at positions max_bit+1 (sign, scale negated), max_bit, ...,
 *   max_bit-n+1; so the stored code is floor(W_q / 2^lo), lo = max_bit-n+1,
 *   with scale s_w = 2^(lo-16).                                             */
int or_quantize_alg1(const float* W, int64_t n_el, int L, double clip,
                     int32_t* codes, double* scale)
{
    if (!W || !codes || L < 2 || L > 16) return OR_EINVAL;
    int n = L - 1;
    double* Q = (double*)malloc(sizeof(double) * (size_t)n_el);
    if (!Q) return OR_EINVAL;
    double d;
    int status = or_quantize_round(W, n_el, n, clip, Q, &d);
    int64_t maxabs = 0;
    int64_t* Wq = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_el);
    if (!Wq) { free(Q); return OR_EINVAL; }
    for (int64_t e = 0; e < n_el; ++e) {
        double t = trunc(Q[e] * 65536.0);
        if (fabs(t) >= 9.0e18) { free(Q); free(Wq); return OR_ERANGE; }
        Wq[e] = (int64_t)t;
        int64_t a = Wq[e] < 0 ? -Wq[e] : Wq[e];
        if (a > maxabs) maxabs = a;
    }
    free(Q);
    if (maxabs == 0) {
        for (int64_t e = 0; e < n_el; ++e) codes[e] = 0;
        *scale = 1.0;
        free(Wq);
        return OR_EDEGENERATE;
    }
    int max_bit = 0;
    while ((maxabs >> (max_bit + 1)) != 0) ++max_bit;   /* floor(log2 max|W_q|) */
    int lo = max_bit - n + 1;
    for (int64_t e = 0; e < n_el; ++e) {
        int64_t m;
        if (lo >= 0) {
            /* floor division by 2^lo: drop the bits below position lo */
            int64_t p = (int64_t)1 << lo;
            m = Wq[e] / p;
            if ((Wq[e] % p) != 0 && Wq[e] < 0) m -= 1;
        } else {
            m = Wq[e] * ((int64_t)1 << (-lo));
        }
        codes[e] = (int32_t)m;
    }
    free(Wq);
    *scale = ldexp(1.0, lo - 16);
    return status;   /* OR_EDEGENERATE when max(W) == min(W) (reading G5) */
}

/* §3.3 1-bit case: "exclude representing 0 and instead opt to
 * represent a positive and negative value".  Reading G7: v = mean|W|;
 * stored bitlayer = [W < 0] (sign(0) = +1), represented code 1 - 2*bit
 * (sign layer scale -2 plus offset +1, reading G1).                        */
int or_quantize_binary(const float* W, int64_t n_el, double clip,
                       uint8_t* bits, double* v_out)
{
    if (!W || !bits || n_el <= 0) return OR_EINVAL;
    double s = 0.0;
    for (int64_t e = 0; e < n_el; ++e) {
        double w = (double)W[e];
        if (clip > 0) { if (w > clip) w = clip; if (w < -clip) w = -clip; }
        s += fabs(w);
        bits[e] = (uint8_t)(w < 0.0 ? 1 : 0);
    }
    double v = s / (double)n_el;
    int status = OR_OK;
    if (v == 0.0) { v = 1.0; status = OR_EDEGENERATE; }
    *v_out = v;
    return status;
}

/* Scale of stored weight bitlayer i:
 * S_0 = -2^(L-1) (negated sign layer), S_i = 2^(L-1-i).  Binary mode
 * (L = 1 with offset 1): S_0 = -2 (reading G1).                             */
int64_t or_weight_layer_scale(int L, int offset, int i)
{
    if (i == 0) return offset ? -2 : -((int64_t)1 << (L - 1));
    return (int64_t)1 << (L - 1 - i);
}

/* Scale of activation bitplane j ("[-2^31 2^30 .. 2^0]"):
 * T_0 = -2^(a-1), T_j = 2^(a-1-j).                                          */
int64_t or_plane_scale(int a, int j)
{
    if (j == 0) return -((int64_t)1 << (a - 1));
    return (int64_t)1 << (a - 1 - j);
}

/* Decomposition into bitlayers: layer i holds bit
 * (L-1-i) of the L-bit two's-complement pattern of the code, sign first.
 * layers is [L][n_el], one byte per bit.                                    */
int or_decompose(const int32_t* codes, int64_t n_el, int L, uint8_t* layers)
{
    if (!codes || !layers || L < 1 || L > 16) return OR_EINVAL;
    int64_t lo = -((int64_t)1 << (L - 1)), hi = ((int64_t)1 << (L - 1)) - 1;
    for (int64_t e = 0; e < n_el; ++e)
        if (codes[e] < lo || codes[e] > hi) return OR_ERANGE;
    for (int i = 0; i < L; ++i)
        for (int64_t e = 0; e < n_el; ++e)
            layers[(int64_t)i * n_el + e] =
                (uint8_t)((((uint32_t)codes[e]) >> (L - 1 - i)) & 1u);
    return OR_OK;
}

/* Activation fixed-point cast (Alg. 2 line 1: x_q <- Int(x * 2^16);
 * P:154 "a multiplication and a cast"; "The fixed point may be changed
 * depending on the scale").  Reading G8:
 *   act_frac == OR_ACT_AUTO: per column b, e_b = frexp exponent of
 *     max_c |x[b,c]| (so max < 2^e_b), f_b = (a-1) - e_b, all-zero -> f_b = 0;
 *   otherwise f_b = act_frac (the literal Alg. 2 uses 16), with saturation
 *     to [-2^(a-1), 2^(a-1)-1].
 *   x_q = trunc(x * 2^f_b).                                                 */
#define OR_ACT_AUTO (-1024)
int or_quantize_activation(const float* x, int64_t B, int64_t K, int a,
                           int act_frac, int64_t* xq, int32_t* f_out)
{
    if (!x || !xq || !f_out || a < 1 || a > 32 || B < 0 || K < 0) return OR_EINVAL;
    double lo = -ldexp(1.0, a - 1), hi = ldexp(1.0, a - 1) - 1.0;
    for (int64_t b = 0; b < B; ++b) {
        int f;
        if (act_frac == OR_ACT_AUTO) {
            double mx = 0.0;
            for (int64_t c = 0; c < K; ++c) {
                double v = fabs((double)x[b * K + c]);
                if (v > mx) mx = v;
            }
            if (mx == 0.0) f = 0;
            else { int e; (void)frexp(mx, &e); f = (a - 1) - e; }
        } else {
            f = act_frac;
        }
        f_out[b] = f;
        for (int64_t c = 0; c < K; ++c) {
            double v = trunc(ldexp((double)x[b * K + c], f));
            if (v < lo) v = lo;
            if (v > hi) v = hi;
            xq[b * K + c] = (int64_t)v;
        }
    }
    return OR_OK;
}

/* Bitwise transpose into activation bitplanes: plane j of
 * column b holds bit (a-1-j) of the a-bit two's-complement pattern of x_q,
 * sign plane first.  planes is [B][a][K], one byte per bit.                 */
int or_transpose(const int64_t* xq, int64_t B, int64_t K, int a, uint8_t* planes)
{
    if (!xq || !planes || a < 1 || a > 32) return OR_EINVAL;
    for (int64_t b = 0; b < B; ++b)
        for (int j = 0; j < a; ++j)
            for (int64_t c = 0; c < K; ++c)
                planes[(b * a + j) * K + c] =
                    (uint8_t)((((uint64_t)xq[b * K + c]) >> (a - 1 - j)) & 1u);
    return OR_OK;
}

/* The bit-serial product and reduction of Alg. 2:
 *   C_ij[r,b] = sum_c W_i[r,c] AND X_j[b,c]          (0/1 products)
 *   acc[r,b]  = sum_{i<k_used} S_i sum_j T_j C_ij + o * sum_c x_q[b,c]
 *   y[b,r]    = (float) ldexp((double)acc * s_w, -f_b)     (reading G13)
 * layers [L][R][K], planes [B][a][K], xq [B][K] (for the offset term),
 * acc [B][R] (nullable), y [B][R] (nullable).  nthreads > 1 splits rows
 * (used only to time the oracle; integer results are order-independent).   */
/* midpoint (an option the paper does not have): with k_used < L the
 * kept layers represent the floor-truncated code m_trunc (reading G12); the midpoint
 * option represents m_trunc + 2^(L - k_used - 1), the centre of the dropped range, so
 * the product gains 2^(L - k_used - 1) * sum_c x_q[b, c].                             */
int or_bitserial_mid(const uint8_t* layers, int64_t R, int64_t K, int L, int offset,
                     int k_used, double scale, const uint8_t* planes,
                     const int64_t* xq, const int32_t* f, int64_t B, int a,
                     int64_t* acc, float* y, int nthreads, int midpoint)
{
    if (!layers || !planes || !f || k_used < 1 || k_used > L || a < 1 || a > 32)
        return OR_EINVAL;
    const int64_t mid = (midpoint && k_used < L && !offset) ? ((int64_t)1 << (L - k_used - 1)) : 0;
    if ((offset || mid) && !xq) return OR_EINVAL;
    int bad = 0;
    if (nthreads < 1) nthreads = 1;
#ifdef _OPENMP
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 1) reduction(|:bad)
#endif
    for (int64_t r = 0; r < R; ++r) {
        for (int64_t b = 0; b < B; ++b) {
            __int128 total = 0;
            for (int i = 0; i < k_used; ++i) {
                const uint8_t* Wi = layers + ((int64_t)i * R + r) * K;
                __int128 s = 0;
                for (int j = 0; j < a; ++j) {
                    const uint8_t* Xj = planes + (b * a + j) * K;
                    int64_t C = 0;
                    for (int64_t c = 0; c < K; ++c) C += (Wi[c] & Xj[c]);
                    s += (__int128)or_plane_scale(a, j) * C;
                }
                total += (__int128)or_weight_layer_scale(L, offset, i) * s;
            }
            if (offset) {
                __int128 sx = 0;
                for (int64_t c = 0; c < K; ++c) sx += xq[b * K + c];
                total += (__int128)offset * sx;
            }
            if (mid) {
                __int128 sx = 0;
                for (int64_t c = 0; c < K; ++c) sx += xq[b * K + c];
                total += (__int128)mid * sx;
            }
            if (total > (__int128)INT64_MAX || total < (__int128)INT64_MIN) { bad = 1; continue; }
            int64_t v = (int64_t)total;
            if (acc) acc[b * R + r] = v;
            if (y) {
                double t = (double)v * scale;
                t = ldexp(t, -f[b]);
                y[b * R + r] = (float)t;
            }
        }
    }
    return bad ? OR_ERANGE : OR_OK;
}

int or_bitserial(const uint8_t* layers, int64_t R, int64_t K, int L, int offset,
                 int k_used, double scale, const uint8_t* planes,
                 const int64_t* xq, const int32_t* f, int64_t B, int a,
                 int64_t* acc, float* y, int nthreads)
{
    return or_bitserial_mid(layers, R, K, L, offset, k_used, scale, planes, xq, f, B, a, acc, y,
                            nthreads, 0);
}

/* Whole Alg. 2 from integer codes: decompose -> cast -> transpose ->
 * bit-serial product -> reduce -> dequant.  Convenience composition of the
 * functions above, each step in the paper's order.                          */
int or_pbatch_mid(const int32_t* codes, int64_t R, int64_t K, int L, int offset,
                  double scale, int k_used, const float* x, int64_t B, int a,
                  int act_frac, int64_t* acc, float* y, int32_t* f_out, int nthreads,
                  int midpoint)
{
    if (!codes || !x || R < 0 || K < 0 || B < 0) return OR_EINVAL;
    if (L < 1 || L > 16 || (offset && L != 1)) return OR_EINVAL;
    /* binary mode (L == 1, offset 1): codes carry 1 - 2*bit */
    uint8_t* layers = (uint8_t*)malloc((size_t)L * (size_t)(R * K) + 1);
    int64_t* xq = (int64_t*)malloc(sizeof(int64_t) * (size_t)(B * K) + 8);
    uint8_t* planes = (uint8_t*)malloc((size_t)(B * a * K) + 1);
    int32_t* f = (int32_t*)malloc(sizeof(int32_t) * (size_t)B + 4);
    int st = OR_EINVAL;
    if (!layers || !xq || !planes || !f) goto done;
    if (L == 1 && offset) {
        /* code = 1 - 2*bit  ->  bit = (1 - code) / 2 */
        for (int64_t e = 0; e < R * K; ++e) {
            if (codes[e] != 1 && codes[e] != -1) { st = OR_ERANGE; goto done; }
            layers[e] = (uint8_t)(codes[e] == -1 ? 1 : 0);
        }
    } else {
        st = or_decompose(codes, R * K, L, layers);
        if (st != OR_OK) goto done;
    }
    st = or_quantize_activation(x, B, K, a, act_frac, xq, f);
    if (st != OR_OK) goto done;
    st = or_transpose(xq, B, K, a, planes);
    if (st != OR_OK) goto done;
    st = or_bitserial_mid(layers, R, K, L, offset, k_used, scale, planes, xq, f, B, a,
                          acc, y, nthreads, midpoint);
    if (f_out) for (int64_t b = 0; b < B; ++b) f_out[b] = f[b];
done:
    free(layers); free(xq); free(planes); free(f);
    return st;
}

int or_pbatch(const int32_t* codes, int64_t R, int64_t K, int L, int offset,
              double scale, int k_used, const float* x, int64_t B, int a,
              int act_frac, int64_t* acc, float* y, int32_t* f_out, int nthreads)
{
    return or_pbatch_mid(codes, R, K, L, offset, scale, k_used, x, B, a, act_frac, acc, y,
                         f_out, nthreads, 0);
}

/* Clip-threshold search ("optimize over a clipping threshold to find a
 * quantized matrix with the smallest mean error").  Reading G6: candidates
 * t_k = (k/64) max|W|, k = 1..64, objective mean |Q(clip(W)) - W| using the
 * codes the packer would store (clamped grid); ties go to the larger t.
 * parity unpinned (any candidate set is a valid reading).                   */
int or_search_clip(const float* W, int64_t n_el, int L, int ncand, float* clip_out)
{
    if (!W || n_el <= 0 || L < 2 || L > 16 || ncand < 1) return OR_EINVAL;
    double mx = 0.0;
    for (int64_t e = 0; e < n_el; ++e) if (fabs((double)W[e]) > mx) mx = fabs((double)W[e]);
    if (mx == 0.0) { *clip_out = 0.0f; return OR_EDEGENERATE; }
    int32_t* codes = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_el);
    if (!codes) return OR_EINVAL;
    double best = INFINITY; float best_t = (float)mx;
    for (int k = 1; k <= ncand; ++k) {
        float t = (float)((double)k / (double)ncand * mx);
        double s;
        if (or_quantize_grid(W, n_el, L, (double)t, codes, &s) == OR_EINVAL) continue;
        double err = 0.0;
        for (int64_t e = 0; e < n_el; ++e) err += fabs(s * (double)codes[e] - (double)W[e]);
        err /= (double)n_el;
        if (err <= best) { best = err; best_t = t; }
    }
    free(codes);
    *clip_out = best_t;
    return OR_OK;
}

/* Elementwise LSTM / RNN cells in double (reading G15: PyTorch nn.LSTM gate
 * order i, f, g, o; RNN cell = tanh).  gates [B][4H] (pre-activation, the
 * sum of the two quantised matvecs plus biases).  Pinned to torch.nn.LSTMCell
 * (tests/test_oracle_pins.py::test_lstm_cell_matches_torch_lstmcell).       */
static double or_sigmoid(double v) { return 1.0 / (1.0 + exp(-v)); }

int or_lstm_cell(const double* gates, const float* c, int64_t B, int64_t H,
                 double* h_out, double* c_out)
{
    for (int64_t b = 0; b < B; ++b)
        for (int64_t k = 0; k < H; ++k) {
            const double* g = gates + b * 4 * H;
            double ig = or_sigmoid(g[k]);
            double fg = or_sigmoid(g[H + k]);
            double gg = tanh(g[2 * H + k]);
            double og = or_sigmoid(g[3 * H + k]);
            double cn = fg * (double)c[b * H + k] + ig * gg;
            c_out[b * H + k] = cn;
            h_out[b * H + k] = og * tanh(cn);
        }
    return OR_OK;
}

int or_num_threads_available(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
