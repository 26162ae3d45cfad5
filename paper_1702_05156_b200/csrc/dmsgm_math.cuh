// dmsgm_math.cuh -- small __host__ __device__ helpers of the DMSGM kernel.
//
// Kept host-compilable so the byte-SWAR and cut-point logic can be checked
// exhaustively on the CPU (tests/test_host_math.py builds a tiny host shim).
// All fp32 arithmetic here is written with explicit round-to-nearest
// operations so that nvcc never contracts it into FMAs (the kernel is also
// built with -fmad=false); on the host the shim is built with -ffp-contract=off.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define DM_HD __host__ __device__ __forceinline__
#else
#define DM_HD static inline
#endif

namespace dmsgm {

#if defined(__CUDA_ARCH__)
DM_HD float f_add(float a, float b) { return __fadd_rn(a, b); }
DM_HD float f_sub(float a, float b) { return __fsub_rn(a, b); }
DM_HD float f_mul(float a, float b) { return __fmul_rn(a, b); }
DM_HD float f_div(float a, float b) { return __fdiv_rn(a, b); }
DM_HD uint32_t byte_sign_spread(uint32_t m) {
    // PRMT generic mode: selector nibble 8+i replicates the msb of byte i.
    uint32_t r;
    asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(r) : "r"(m));
    return r;
}
#else
DM_HD float f_add(float a, float b) { volatile float r = a + b; return r; }
DM_HD float f_sub(float a, float b) { volatile float r = a - b; return r; }
DM_HD float f_mul(float a, float b) { volatile float r = a * b; return r; }
DM_HD float f_div(float a, float b) { volatile float r = a / b; return r; }
DM_HD uint32_t byte_sign_spread(uint32_t m) {
    uint32_t r = 0;
    for (int i = 0; i < 4; ++i)
        if (m & (0x80u << (8 * i))) r |= 0xFFu << (8 * i);
    return r;
}
#endif

// Per-byte (x - y) mod 256, no borrow across bytes (SWAR subtraction).
DM_HD uint32_t sub_bytes(uint32_t x, uint32_t y) {
    return ((x | 0x80808080u) - (y & 0x7F7F7F7Fu)) ^ ((x ^ ~y) & 0x80808080u);
}

// Per-byte unsigned v > w  ->  0xFF / 0x00.  v > w  <=>  v + (255 - w) carries out of bit 7.
DM_HD uint32_t gt_bytes(uint32_t v, uint32_t w) {
    const uint32_t k = ~w;
    const uint32_t s = (v & 0x7F7F7F7Fu) + (k & 0x7F7F7F7Fu);   // bit 7 = carry into bit 7
    const uint32_t maj = (v & k) | ((v | k) & s);                // carry out of bit 7 (in bit 7)
    return byte_sign_spread(maj);
}

// Mask of four pixels against per-byte background intervals [a, a+w] (w >= 0),
// with per-byte "all foreground" override f (0xFF bytes): 255 = foreground.
DM_HD uint32_t mask_bytes(uint32_t px, uint32_t a, uint32_t w, uint32_t f) {
    return gt_bytes(sub_bytes(px, a), w) | f;
}

// Literal per-pixel classification predicate of App. E P:657 with reading R14:
// foreground iff fl(fl(I - mu)^2) > T.
DM_HD bool fg_pred(float I, float mu, float T) {
    const float d = f_sub(I, mu);
    return f_mul(d, d) > T;
}

// Background interval of the classification for integer intensities.
// {I in Z : !fg_pred(I, mu, T)} is an interval [a, b] (fl(I-mu) is monotone in I and
// fl(x*x) is monotone in |x|).  Returns it clamped to [0,255] as (a, w = b - a) and
// `empty` when no intensity in [0,255] is background.  The estimate floor(mu +/- r),
// r ~ sqrt(T), is refined by testing the literal predicate at est-1, est, est+1.
struct Interval {
    int a;
    int w;
    bool empty;
};

DM_HD Interval bg_interval(float mu, float T, float r) {
    // r: any estimate of sqrt(T) with relative error << 1/512 (caller supplies it).
    float hi_f = f_add(mu, r);
    float lo_f = f_sub(mu, r);
    hi_f = hi_f < -2.0f ? -2.0f : (hi_f > 257.0f ? 257.0f : hi_f);
    lo_f = lo_f < -2.0f ? -2.0f : (lo_f > 257.0f ? 257.0f : lo_f);
#if defined(__CUDA_ARCH__)
    const int hi = __float2int_rd(hi_f);
    const int lo = __float2int_ru(lo_f);
#else
    const int hi = (int)__builtin_floorf(hi_f);
    const int lo = (int)__builtin_ceilf(lo_f);
#endif
    // upper end: the largest k in {hi+1, hi, hi-1} that is background
    const bool p_h1 = fg_pred((float)(hi + 1), mu, T);
    const bool p_h0 = fg_pred((float)hi, mu, T);
    const bool p_hm = fg_pred((float)(hi - 1), mu, T);
    // lower end: the smallest k in {lo-1, lo, lo+1} that is background
    const bool p_lm = fg_pred((float)(lo - 1), mu, T);
    const bool p_l0 = fg_pred((float)lo, mu, T);
    const bool p_l1 = fg_pred((float)(lo + 1), mu, T);
    const bool none_hi = p_h1 && p_h0 && p_hm;
    const bool none_lo = p_lm && p_l0 && p_l1;
    int b = !p_h1 ? hi + 1 : (!p_h0 ? hi : hi - 1);
    int a = !p_lm ? lo - 1 : (!p_l0 ? lo : lo + 1);
    a = a < 0 ? 0 : a;
    b = b > 255 ? 255 : b;
    Interval iv;
    iv.empty = none_hi || none_lo || a > b;
    iv.a = iv.empty ? 0 : a;
    iv.w = iv.empty ? 0 : b - a;
    return iv;
}

}  // namespace dmsgm
