// dmsgm_math.cuh -- small __host__ __device__ helpers of the DMSGM kernel.
//
// Kept host-compilable so the packed-pixel mask and cut-point logic can be checked
// exhaustively on the CPU (tests/test_host_math.py builds a tiny host shim).
// fp32 arithmetic here is written with explicit round-to-nearest operations so
// that nvcc never contracts it into FMAs (the kernel is also built with
// -fmad=false); on the host the shim is built with -ffp-contract=off.
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
DM_HD float f_fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
// PRMT generic mode: result byte i = byte sel_i of {a, b}; selector nibble bit 3
// replicates the sign (msb) of the selected byte.
DM_HD uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}
#else
#include <math.h>
DM_HD float f_add(float a, float b) { volatile float r = a + b; return r; }
DM_HD float f_sub(float a, float b) { volatile float r = a - b; return r; }
DM_HD float f_mul(float a, float b) { volatile float r = a * b; return r; }
DM_HD float f_div(float a, float b) { volatile float r = a / b; return r; }
DM_HD float f_fma(float a, float b, float c) { return fmaf(a, b, c); }
DM_HD uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    const uint64_t x = ((uint64_t)b << 32) | a;
    uint32_t r = 0;
    for (int i = 0; i < 4; ++i) {
        const uint32_t s = (sel >> (4 * i)) & 0xF;
        uint32_t byte = (uint32_t)(x >> (8 * (s & 7))) & 0xFF;
        if (s & 8) byte = (byte & 0x80) ? 0xFF : 0x00;
        r |= byte << (8 * i);
    }
    return r;
}
#endif

// Bytes {0,1} / {2,3} of a pixel word as two 16-bit lanes (zero-extended).
DM_HD uint32_t lanes_lo(uint32_t w) { return prmt(w, 0, 0x4140); }
DM_HD uint32_t lanes_hi(uint32_t w) { return prmt(w, 0, 0x4342); }

// Literal per-pixel classification predicate of App. E P:657 with reading R14:
// foreground iff fl(fl(I - mu)^2) > T.
DM_HD bool fg_pred(float I, float mu, float T) {
    const float d = f_sub(I, mu);
    return f_mul(d, d) > T;
}

// Background interval of the classification for integer intensities.
// {I in Z : !fg_pred(I, mu, T)} is an interval [a, b] (fl(I-mu) is monotone in I and
// fl(x*x) is monotone in |x|).  Returned clamped to [0,255]; a = 256 when no intensity
// in [0,255] is background.  The estimate floor(mu +/- r), r ~ sqrt(T), is refined by
// testing the literal predicate at est-1, est, est+1 (SURVEY pin P13, host-tested).
struct Interval {
    int a;
    int b;
};

DM_HD Interval bg_interval(float mu, float T, float r, bool may_be_empty = true) {
    // r: any estimate of sqrt(T) with relative error << 1/512 (caller supplies it).
    // may_be_empty = false is allowed when T >= 0.25 is guaranteed: the integer nearest
    // to mu then has fl(d*d) <= 0.25 <= T, so the interval is never empty.
    float hi_f = f_add(mu, r);
    float lo_f = f_sub(mu, r);
    hi_f = hi_f < -2.0f ? -2.0f : (hi_f > 257.0f ? 257.0f : hi_f);
    lo_f = lo_f < -2.0f ? -2.0f : (lo_f > 257.0f ? 257.0f : lo_f);
    const float hf = floorf(hi_f);          // candidates are small integers: exact in fp32
    const float lf = ceilf(lo_f);
    // upper end: the largest k in {hi+1, hi, hi-1} that is background
    const bool p_h1 = fg_pred(f_add(hf, 1.0f), mu, T);
    const bool p_h0 = fg_pred(hf, mu, T);
    // lower end: the smallest k in {lo-1, lo, lo+1} that is background
    const bool p_lm = fg_pred(f_sub(lf, 1.0f), mu, T);
    const bool p_l0 = fg_pred(lf, mu, T);
    bool none = false;
    if (may_be_empty) {
        const bool p_hm = fg_pred(f_sub(hf, 1.0f), mu, T);
        const bool p_l1 = fg_pred(f_add(lf, 1.0f), mu, T);
        none = (p_h1 && p_h0 && p_hm) || (p_lm && p_l0 && p_l1);
    }
    const int hi = (int)hf, lo = (int)lf;
    int b = !p_h1 ? hi + 1 : (!p_h0 ? hi : hi - 1);
    int a = !p_lm ? lo - 1 : (!p_l0 ? lo : lo + 1);
    a = a < 0 ? 0 : a;
    b = b > 255 ? 255 : b;
    Interval iv;
    iv.a = (none || a > b) ? 256 : a;
    iv.b = b < 0 ? 0 : b;
    return iv;
}

// Fast form of bg_interval.  With r within 1.5e-4 of sqrt(T) (rsqrt estimate) and T <= 3e5,
// |fl(mu +/- r) - (mu +/- sqrt(T))| < 2e-4, and the literal predicate can only differ from
// exact arithmetic within ~5e-5 of k = mu +/- sqrt(T).  So when mu +/- r lies more than
// 1e-3 away from an integer, floor(mu + r) / ceil(mu - r) ARE the interval ends; otherwise
// (about 0.2% of blocks) the predicate-tested form decides.  Host-tested against the
// literal predicate (tests/test_host_math.py).
DM_HD bool interval_is_clear(float x) {
    const float f = f_sub(x, floorf(x));
    return f > 1e-3f && f < 0.999f;
}

DM_HD Interval bg_interval_fast(float mu, float T, float r, bool may_be_empty, bool* slow) {
    const float hi_f = f_add(mu, r);
    const float lo_f = f_sub(mu, r);
    const bool clear = interval_is_clear(hi_f) && interval_is_clear(lo_f) && T <= 3.0e5f &&
                       hi_f > -1.0f && lo_f < 256.0f;
    *slow = !clear;
    Interval iv;
    int b = (int)floorf(hi_f);
    int a = (int)ceilf(lo_f);
    a = a < 0 ? 0 : a;
    b = b > 255 ? 255 : b;
    iv.a = a > b ? 256 : a;     // (may_be_empty only matters on the slow path: an empty
    iv.b = b < 0 ? 0 : b;       //  interval has no integer in (lo_f, hi_f) -> a > b here)
    (void)may_be_empty;
    return iv;
}

// Per-16-bit-lane keys of an interval: x = lane + (0x8000 - a) has bit 15 set iff
// lane >= a; y = (0x8000 + b) - lane has bit 15 set iff lane <= b (lanes <= 255, so no
// carry/borrow crosses a lane).  a = 256 makes x's bit 15 always clear (all foreground).
DM_HD uint32_t key_a(int a) { return (uint32_t)(0x8000 - a); }
DM_HD uint32_t key_b(int b) { return (uint32_t)(0x8000 + b); }

// Mask of four pixels given as two 16-bit-lane words (lanes_lo / lanes_hi) and the
// packed keys of each lane's block: 0xFF = foreground (outside [a, b]).
DM_HD uint32_t mask_word(uint32_t lo, uint32_t hi, uint32_t ka_lo, uint32_t kb_lo, uint32_t ka_hi,
                         uint32_t kb_hi) {
    const uint32_t fl = ~((lo + ka_lo) & (kb_lo - lo));   // bit 15 / 31: pixel 0 / 1 foreground
    const uint32_t fh = ~((hi + ka_hi) & (kb_hi - hi));   // bit 15 / 31: pixel 2 / 3 foreground
    return prmt(fl, fh, 0xFDB9);                          // sign-spread bytes 1,3 of fl, fh
}

}  // namespace dmsgm
