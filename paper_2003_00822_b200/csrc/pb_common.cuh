// pb_common.cuh -- small device helpers for the sm_100a kernels (product code).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "pb_internal.h"

namespace pb {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 128-bit streaming load of packed weights: read once, do not pollute L1.
__device__ __forceinline__ uint4 ld_stream_u4(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// ---- mbarrier + 1-D TMA bulk copy (cp.async.bulk -> UBLKCP) ----
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
#ifdef PB_WAIT_HINT
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
#else
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
#endif
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
#ifdef PB_WAIT_HINT
        , "r"((uint32_t)PB_WAIT_HINT)
#endif
        : "memory");
}
// global -> shared bulk copy, completion counted on `bar` (bytes % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Shift-weighted reduction scales: T_j and S_i as wrapping
// 64-bit integers.  All accumulation is done modulo 2^64, which is exact as
// long as the final value fits int64 (the G11 guard checked on the host).
// Step a1 (Alg. 2 line 1; readings G7/G8): x_q = Int(x * 2^f) with
// the power-of-two scaling exact in double, saturation to the a-bit two's
// complement range (only reachable with a literal act_frac) and truncation
// toward zero.
__device__ __forceinline__ double pow2d(int e) {   // 2^e, e in [-1022, 1023]
    return __hiloint2double((1023 + e) << 20, 0);
}
static __device__ __noinline__ long long act_cast_f64(float v, int f, int a) {
    const double lim = (double)(1ll << (a - 1));
    double t = (f >= -1000 && f <= 1000) ? (double)v * pow2d(f) : ldexp((double)v, f);
    t = fmin(fmax(t, -lim), lim - 1.0);
    return __double2ll_rz(t);
}
__device__ __forceinline__ long long act_cast(float v, int f, int a) {
    if (a <= 24 && f >= -126 && f <= 127) {
        // fp32 is exact here: v * 2^f is exact whenever |v * 2^f| >= 2^-126, smaller
        // magnitudes truncate to 0 either way, and the clamp bounds +-2^(a-1), 2^(a-1)-1
        // are representable for a <= 24 -- the same integer as the double form below
        const float lim = (float)(1 << (a - 1));
        float t = v * __int_as_float((127 + f) << 23);
        t = fminf(fmaxf(t, -lim), lim - 1.0f);
        return (long long)__float2int_rz(t);
    }
    return act_cast_f64(v, f, a);                       // a > 24 or an extreme literal act_frac
}
// f_b from max|x[b,:]| (reading G8): the largest f with max|x| * 2^f < 2^(a-1).
__device__ __forceinline__ int act_frac_of(float m, int a) {
    if (m == 0.f) return 0;
    int e;
    frexpf(m, &e);           // m = frac * 2^e, frac in [0.5, 1): m < 2^e
    return (a - 1) - e;
}
// Tensor-engine B operand (pb_gemm_tc.cu): the activation planes stacked in pairs (the
// "multiple bitlayers may be stacked together" of P:206, applied to the activation side as
// it is to the weights): digit k of a column is d_k = 2 X_2k + X_2k+1 with weight
// U_k = 2^(a-2-2k), the sign pair carries its negative plane weight, d_0 = -2 X_0 + X_1,
// and an odd a leaves the last plane alone, d = X_(a-1) with U = 1 (a = 1: d_0 = -X_0).
// Then sum_k U_k d_k = sum_j T_j X_j = x_q exactly (T_0 = -2^(a-1), T_j = 2^(a-1-j)).
// Each digit is stored as the e2m1 value 2 d in {-4, -2, 0, 2, 4, 6} (exact), so against a
// weight nibble 1.0 hi + 0.5 lo the product is the integer (2 hi + lo) d.
__host__ __device__ constexpr int act_digits(int a) { return (a + 1) / 2; }
// 4 registers of e2m1 nibbles (register r, nibble e <-> column 4e + r of the 32-column word)
// from the digit's plane words hi (X_2k) and lo (X_2k+1); branch-free over the kinds with
// ms = sign digit, ml = lone plane (all-ones masks): bit 3 = sign, bit 2 = any,
// bit 1 = 2d >= 4 or the sign pair's -4, bit 0 = 2d = 6.
__device__ __forceinline__ uint4 digit_regs(uint32_t hi, uint32_t lo, uint32_t ms, uint32_t ml) {
    uint32_t v[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const uint32_t H = (hi >> r) & 0x11111111u, Lo = (lo >> r) & 0x11111111u & ~ml;
        const uint32_t b3 = H & ms, b2 = H | Lo, b1 = H & ~ml & (~ms | ~Lo), b0 = H & Lo & ~ms;
        v[r] = (b3 << 3) | (b2 << 2) | (b1 << 1) | b0;
    }
    return make_uint4(v[0], v[1], v[2], v[3]);
}
// Digit row n of word w into the K-major no-swizzle canonical layout of the N_pad x 32-byte
// tile of words (w & ~1, w | 1).
__device__ __forceinline__ void put_b_operand(uint8_t* bexp, int npad, int64_t w, int n, uint4 v) {
    uint8_t* tile = bexp + (w >> 1) * npad * 32 + (w & 1) * 128;
    *reinterpret_cast<uint4*>(tile + (n >> 3) * 256 + (n & 7) * 16) = v;
}
// The same into a shared-memory tile (explicit st.shared: a generic store would resolve its
// address space at run time).
__device__ __forceinline__ void put_b_operand_smem(uint32_t tile_s, int npad, int64_t w, int n, uint4 v) {
    const uint32_t a = tile_s + (uint32_t)((w >> 1) * npad * 32 + (w & 1) * 128 + (n >> 3) * 256 + (n & 7) * 16);
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
// After a ballot transpose (lane j < a holds plane word j of a 32-column word): the lanes
// 2k < a hold digit k's registers (the pair partner's plane comes from lane 2k + 1).
// Warp-collective; returns whether this lane writes digit lane / 2.
__device__ __forceinline__ bool digit_of_lane(uint32_t mine, int lane, int a, uint4& v) {
    const uint32_t partner = __shfl_down_sync(0xffffffffu, mine, 1);
    v = digit_regs(mine, partner, lane == 0 ? ~0u : 0u, lane == a - 1 ? ~0u : 0u);   // branch-free
    return !(lane & 1) && lane < a;
}

// The same digit rows without a ballot transpose, for an even a <= 16 (warp-collective):
// every lane holds x_q of its column 32w + lane as the a-bit pattern u.  A lane first forms
// its 8 digit nibbles (digit k in nibble 7 - k; digits >= ceil(a/2) are 0): the pairs of the
// top-aligned pattern spread to 4-bit slots, then the e2m1 code of 2 d (as digit_regs, the
// sign digit 0 in nibble 7).  The 8 lanes sharing r = lane & 3 then transpose their 8 x 8
// nibble matrix in 3 butterfly stages (shfl_xor 16, 8, 4), after which lane 4e + r holds
// register r of digit k = 7 - e: nibble j = the digit of column 4j + r.  Returns that
// register; *k receives the digit (the caller stores it when k < ceil(a/2)).
__device__ __forceinline__ uint32_t digit_regs_shfl(uint32_t u, int a, int lane, int& k) {
    const uint32_t p = (u << (32 - a)) >> 16;        // pair j (bits 2j, 2j+1) = digit 7 - j
    uint32_t x = (p | (p << 8)) & 0x00FF00FFu;
    x = (x | (x << 4)) & 0x0F0F0F0Fu;
    x = (x | (x << 2)) & 0x33333333u;                // pair j in nibble j: bit 0 = lo, bit 1 = hi
    const uint32_t L = x & 0x11111111u, H = (x >> 1) & 0x11111111u;
    const uint32_t gen = ((H | L) << 2) | (H << 1) | (H & L);             // 0, 2, 4, 6
    const uint32_t sgn = (H << 3) | ((H | L) << 2) | ((H & ~L) << 1);     // 0, 2, -4, -2
    x = (gen & 0x0FFFFFFFu) | (sgn & 0xF0000000u);
    const int e = lane >> 2;
    uint32_t t = __shfl_xor_sync(0xffffffffu, x, 16);
    x = (e & 4) ? ((x & 0xFFFF0000u) | (t >> 16)) : ((x & 0x0000FFFFu) | (t << 16));
    t = __shfl_xor_sync(0xffffffffu, x, 8);
    x = (e & 2) ? ((x & 0xFF00FF00u) | ((t >> 8) & 0x00FF00FFu)) : ((x & 0x00FF00FFu) | ((t & 0x00FF00FFu) << 8));
    t = __shfl_xor_sync(0xffffffffu, x, 4);
    x = (e & 1) ? ((x & 0xF0F0F0F0u) | ((t >> 4) & 0x0F0F0F0Fu)) : ((x & 0x0F0F0F0Fu) | ((t & 0x0F0F0F0Fu) << 4));
    k = 7 - e;
    return x;
}
// Byte offset of register r of digit row n, word w in a tile set of N_pad rows (the layout of
// put_b_operand).
__device__ __forceinline__ uint32_t b_operand_offset(int npad, int64_t w, int n, int r) {
    return (uint32_t)((w >> 1) * npad * 32 + (w & 1) * 128 + (n >> 3) * 256 + (n & 7) * 16 + r * 4);
}

// Next diagnostics-timeline record (pb_internal.h, pb_debug_timeline) or null when full.
__device__ __forceinline__ long long* tl_record(long long* tl) {
    const unsigned long long i = atomicAdd(reinterpret_cast<unsigned long long*>(tl), 1ull);
    return i < (unsigned long long)kTlRecords ? tl + 10 + 10 * (long long)i : nullptr;
}
__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned long long plane_scale(int a, int j) {
    const unsigned long long p = 1ull << (a - 1 - j);
    return j == 0 ? (0ull - p) : p;
}
__device__ __forceinline__ unsigned long long layer_scale(int L, int offset, int i) {
    if (i == 0) return offset ? (0ull - 2ull) : (0ull - (1ull << (L - 1)));
    return 1ull << (L - 1 - i);
}

// Dequant epilogue (reading G13): y = (float) ldexp((double)acc * s_w, -f_b),
// then bias / accumulate / fn in fp32.
__device__ __forceinline__ float dequant(long long acc, double scale, int f) {
    double t = __dmul_rn(__ll2double_rn(acc), scale);
    t = ldexp(t, -f);
    return __double2float_rn(t);
}
// The same with the column's scale folded: y = (float)((double)acc * (s_w 2^-f_b)).  Scaling
// by an exact power of two commutes with round-to-nearest while nothing under- or overflows
// (here |acc| < 2^63, s_w >= 2^-170 and f_b in [-130, 180] keep every value normal), so this
// is bit-identical to dequant() with one FP64 multiply fewer (col_scale is exact).
__device__ __forceinline__ double col_scale(double scale, int f) { return ldexp(scale, -f); }
__device__ __forceinline__ float dequant_sc(long long acc, double sc) {
    return __double2float_rn(__dmul_rn(__ll2double_rn(acc), sc));
}
// LSTM cell (reading G15: PyTorch nn.LSTM gates i, f, g, o; fp32 as P:128 keeps the
// nonlinearities in full precision): c' = sigmoid(f) c + sigmoid(i) tanh(g),
// h' = sigmoid(o) tanh(c').
__device__ __forceinline__ float sigmoidf_(float v) { return 1.f / (1.f + expf(-v)); }
__device__ __forceinline__ void lstm_cell(float gi, float gf, float gg, float go, float c, float& h_out,
                                          float& c_out) {
    const float cn = sigmoidf_(gf) * c + sigmoidf_(gi) * tanhf(gg);
    c_out = cn;
    h_out = sigmoidf_(go) * tanhf(cn);
}
// The same from the gates' activations (sigmoid(i), sigmoid(f), tanh(g), sigmoid(o)), each
// computed by the lane that holds its gate.
__device__ __forceinline__ void lstm_cell_act(float si, float sf, float tg, float so, float c, float& h_out,
                                              float& c_out) {
    const float cn = sf * c + si * tg;
    c_out = cn;
    h_out = so * tanhf(cn);
}
__device__ __forceinline__ float apply_fn(float v, int fn) {
    switch (fn) {
        case 1: return v > 0.f ? v : 0.f;
        case 2: return tanhf(v);
        case 3: return 1.f / (1.f + expf(-v));
        default: return v;
    }
}

}  // namespace pb
