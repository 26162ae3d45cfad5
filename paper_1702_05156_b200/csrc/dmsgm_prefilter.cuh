// dmsgm_prefilter.cuh -- the optional frame preprocessing of the step:
// separable Gaussian then 3x3 median (§2.1, §3.3.1, App. C/D;
// readings R30-R34 of DESIGN.md §2).
//
// One streaming kernel (see dmsgm_prefilter_kernel below): a warp walks a 120-column strip
// of a frame down kPfBand rows, with the row pass, the column pass (a register ring of
// partial sums) and the median in registers -- no shared memory, no CTA barriers.
// HBM traffic: 1 B/px read (+ the strips' 1-column and band halos, L2) + 1 B/px written;
// the step kernel then reads the output.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dmsgm_math.cuh"
#include "dmsgm_pair.cuh"

namespace dmsgm {

constexpr int kPfMaxG = 3;        // Gaussian radius <= 3 (size <= 7)

struct PrefilterArgs {
    const uint8_t* in;
    long long in_stride;          // bytes between streams
    int in_pitch;
    uint8_t* out;
    long long out_stride;
    int out_pitch;
    int W, H;
    int g;                        // Gaussian radius (0 = off)
    int m;                        // median radius (0 or 1)
    float taps[2 * kPfMaxG + 1];
};

// Median of the 3x3 windows of 4 adjacent output pixels (R33).  Pixels are handled as
// 16-bit lanes (two per register) with the native 2- and 3-input u16x2 min/max: every
// window column is sorted once across the 3 rows (lo, mid, hi), and
//   median9 = med3(max3(lo_a, lo_b, lo_c), med3(mid_a, mid_b, mid_c), min3(hi_a, hi_b, hi_c))
// for the window's three sorted columns a, b, c (the classic sorted-columns identity).
__device__ __forceinline__ uint32_t med3_u16x2(uint32_t a, uint32_t b, uint32_t c) {
    return __vmaxu2(__vminu2(a, b), __vminu2(__vmaxu2(a, b), c));
}
__device__ __forceinline__ uint32_t median3x3x4(const uint32_t (&w0)[3], const uint32_t (&w1)[3]) {
    // w0[dy] = columns x-1 .. x+2 of row dy, w1[dy] = columns x+3 .. x+6 (bytes, little-endian)
    uint32_t lo[3][3], mi[3][3], hi[3][3];   // [column pair: (x-1,x) (x+1,x+2) (x+3,x+4)][sorted]
    {
        uint32_t c[3][3];
#pragma unroll
        for (int dy = 0; dy < 3; ++dy) {
            c[0][dy] = __byte_perm(w0[dy], 0u, 0x4140);   // (x-1, x)
            c[1][dy] = __byte_perm(w0[dy], 0u, 0x4342);   // (x+1, x+2)
            c[2][dy] = __byte_perm(w1[dy], 0u, 0x4140);   // (x+3, x+4)
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            lo[k][0] = __vimin3_u16x2(c[k][0], c[k][1], c[k][2]);
            hi[k][0] = __vimax3_u16x2(c[k][0], c[k][1], c[k][2]);
            // the middle one is the sum minus the extremes (lanes <= 3 * 255: no carry or
            // borrow crosses the 16-bit lanes)
            mi[k][0] = c[k][0] + c[k][1] + c[k][2] - lo[k][0] - hi[k][0];
        }
    }
    // windows of outputs (x, x+1): column pairs (x-1,x) (x,x+1) (x+1,x+2);
    // of outputs (x+2, x+3): (x+1,x+2) (x+2,x+3) (x+3,x+4)
    const auto shift = [](uint32_t a, uint32_t b) { return __byte_perm(a, b, 0x5432); };   // (a.hi, b.lo)
    const uint32_t l01 = shift(lo[0][0], lo[1][0]), m01 = shift(mi[0][0], mi[1][0]), h01 = shift(hi[0][0], hi[1][0]);
    const uint32_t l23 = shift(lo[1][0], lo[2][0]), m23 = shift(mi[1][0], mi[2][0]), h23 = shift(hi[1][0], hi[2][0]);
    const uint32_t p01 = med3_u16x2(__vimax3_u16x2(lo[0][0], l01, lo[1][0]), med3_u16x2(mi[0][0], m01, mi[1][0]),
                                    __vimin3_u16x2(hi[0][0], h01, hi[1][0]));
    const uint32_t p23 = med3_u16x2(__vimax3_u16x2(lo[1][0], l23, lo[2][0]), med3_u16x2(mi[1][0], m23, mi[2][0]),
                                    __vimin3_u16x2(hi[1][0], h23, hi[2][0]));
    return __byte_perm(p01, p23, 0x6420);      // (x, x+1, x+2, x+3) as bytes
}

// 0x4B000000 | byte k of the 12-byte string w0 w1 w2 (k a compile-time constant): one PRMT
__device__ __forceinline__ uint32_t byte_magic(uint32_t w0, uint32_t w1, uint32_t w2, int k) {
    const uint32_t w = k < 4 ? w0 : (k < 8 ? w1 : w2);
    return __byte_perm(w, 0x4B000000u, 0x7540u | (uint32_t)(k & 3));
}

// ---------------------------------------------------------------------------
// Streaming kernel: no shared memory, no CTA barriers.  A warp owns a vertical strip of
// 120 output columns x kPfBand rows of one frame; lane L holds the 4 columns
// gx = xw - 4 + 4L .. gx + 3 (lanes 0 and 31 are the strip's 1-column halo; lanes 1-30
// produce output) and walks down the strip:
//   input row r (clamped, R32): one 32-bit load per lane, prefetched kPfRing rows ahead;
//     the neighbours' words by two shuffles give bytes gx-4 .. gx+7;
//   row pass (R31): 4 outputs as 2 pairs ((0, 2), (1, 3)), fma(p, tap_t, acc) ascending
//     t, bytes made exact floats by a PRMT into 0x4B000000 and one paired subtraction;
//   column pass: input row r contributes tap t to Gaussian row r + G - t, so 2G+1
//     partial accumulators rotate through a register ring (the row loop is unrolled by
//     the ring size, so every ring index is a compile-time constant); row r - G is
//     complete at tap 2G: rounded to nearest-even (acc + 2^23, low byte);
//   median (R33): the last 3 Gaussian rows as (x-1 .. x+2, x+3 .. x+6) word pairs (two
//     shuffles + PRMT per Gaussian row), median3x3x4, one 32-bit store.
// Borders: input rows / columns are clamped (the passes stay exact); Gaussian values
// outside the image take their clamped value for the median (R32): Gaussian row -1 / H
// is row 0 / H-1 again, column -1 / W is column 0 / W-1 again.
// ---------------------------------------------------------------------------
constexpr int kPfOutW = 120;      // output columns per warp (lanes 1..30)
#ifndef DMSGM_PF_BAND
#define DMSGM_PF_BAND 40
#endif
constexpr int kPfBand = DMSGM_PF_BAND;   // output rows per warp (A/B at C4: 32/40/48/64 rows -> 117.6/115.1/119.0/121.2 us)
#ifndef DMSGM_PF_WARPS
#define DMSGM_PF_WARPS 8
#endif
#ifndef DMSGM_PF_MINB
#define DMSGM_PF_MINB 1
#endif
constexpr int kPfWarps = DMSGM_PF_WARPS;   // warps per CTA (independent strips)

template <int G, int M>
__global__ void __launch_bounds__(32 * kPfWarps, DMSGM_PF_MINB) dmsgm_prefilter_kernel(const PrefilterArgs a) {
    constexpr int NR = 2 * G + 1;                   // column-pass ring (rows in flight)
    const int lane = threadIdx.x & 31;
    const int strip = blockIdx.x * kPfWarps + (threadIdx.x >> 5);
    const int xw = strip * kPfOutW;
    if (xw >= a.W) return;                          // warp-uniform
    const int s = blockIdx.z;
    const int ys = blockIdx.y * kPfBand;
    const int ye = min(ys + kPfBand, a.H);          // output rows [ys, ye)
    const uint8_t* in = a.in + (long long)s * a.in_stride;
    uint8_t* out = a.out + (long long)s * a.out_stride;
    const int gx = xw - 4 + 4 * lane;               // this lane's 4 columns
    const int x = gx;                               // output columns (lanes 1..30)
    const bool writer = lane >= 1 && lane <= 30 && x < a.W;
    // Gaussian rows [g0, g1] feed the output rows (clamped to the image)
    const int g0 = M ? max(ys - 1, 0) : ys, g1 = M ? min(ye, a.H - 1) : ye - 1;

    auto load_word = [&](int r) -> uint32_t {       // clamped row r, columns gx .. gx+3 (clamped)
        const uint8_t* row = in + (long long)min(max(r, 0), a.H - 1) * a.in_pitch;
        if (gx >= 0 && gx + 4 <= a.W) return __ldg(reinterpret_cast<const unsigned int*>(row + gx));
        return 0x01010101u * (uint32_t)__ldg(row + (gx < 0 ? 0 : a.W - 1));
    };
    // median window: (x-1 .. x+2, x+3 .. x+6) of the last 3 Gaussian rows.  The rows pushed
    // are E(ys-1), E(ys), ..., E(ye) with E(y) = Gaussian row clamp(y) (R32): row 0 is pushed
    // twice at the top of the image, row H-1 twice at the bottom; after push i >= 2 the
    // window is centred on output row ys + i - 2.
    uint32_t mw0[3] = {0, 0, 0}, mw1[3] = {0, 0, 0};
    int pushed = 0;
    auto emit_gauss = [&](int gy, uint32_t gw) {    // Gaussian row gy (bytes of columns gx .. gx+3)
        if constexpr (M == 0) {
            if (writer) *reinterpret_cast<uint32_t*>(out + (long long)gy * a.out_pitch + x) = gw;
        } else {
            const uint32_t left = __shfl_up_sync(0xffffffffu, gw, 1), right = __shfl_down_sync(0xffffffffu, gw, 1);
            uint32_t w0 = __byte_perm(left, gw, 0x6543), w1 = __byte_perm(gw, right, 0x6543);
            if (x == 0) w0 = __byte_perm(w0, 0u, 0x3211);          // column -1 := column 0
            if (x + 4 == a.W) w1 = __byte_perm(w1, 0u, 0x3200);    // column W := column W-1
            const int reps = (gy == 0 ? 2 : 1) + (gy == a.H - 1 && ye == a.H ? 1 : 0);
            for (int k = 0; k < reps; ++k) {
                mw0[0] = mw0[1]; mw0[1] = mw0[2]; mw0[2] = w0;
                mw1[0] = mw1[1]; mw1[1] = mw1[2]; mw1[2] = w1;
                if (++pushed >= 3) {
                    const int y = ys + pushed - 3;
                    const uint32_t m = median3x3x4(mw0, mw1);
                    if (writer) *reinterpret_cast<uint32_t*>(out + (long long)y * a.out_pitch + x) = m;
                }
            }
        }
    };

    if constexpr (G == 0) {
        for (int gy = g0; gy <= g1; ++gy) emit_gauss(gy, load_word(gy));
    } else {
        float2 acc[NR][2];
        uint32_t q[NR];                              // prefetched input words (ring, NR rows ahead)
        const int r0 = g0 - G, r1 = g1 + G;          // input rows in streaming order
#pragma unroll
        for (int j = 0; j < NR; ++j) q[j] = load_word(r0 + j);
#pragma unroll
        for (int j = 0; j < NR; ++j) acc[j][0] = acc[j][1] = f2_bc(0.0f);
        float tap[NR];
#pragma unroll
        for (int t = 0; t < NR; ++t) tap[t] = a.taps[t];
        for (int rb = r0; rb <= r1; rb += NR) {
#pragma unroll
            for (int ph = 0; ph < NR; ++ph) {
                const int r = rb + ph;
                if (r > r1) break;                   // warp-uniform
                const uint32_t w = q[ph];
                q[ph] = load_word(r + NR);
                // row pass of input row r
                const uint32_t wl = __shfl_up_sync(0xffffffffu, w, 1), wr = __shfl_down_sync(0xffffffffu, w, 1);
                // outputs paired (0, 2) and (1, 3): the operand pairs (p[k], p[k+2]),
                // k = 0 .. 2G+1, are built directly by PRMT (no register moves)
                float2 pp[2 * G + 2];
#pragma unroll
                for (int k = 0; k < 2 * G + 2; ++k)
                    pp[k] = f2_sub(make_float2(__uint_as_float(byte_magic(wl, w, wr, k + 4 - G)),
                                               __uint_as_float(byte_magic(wl, w, wr, k + 6 - G))),
                                   f2_bc(8388608.0f));
                float2 h01 = f2_bc(0.0f), h23 = f2_bc(0.0f);     // (h0, h2), (h1, h3)
#pragma unroll
                for (int t = 0; t < NR; ++t) {
                    h01 = f2_fma(pp[t], f2_bc(tap[t]), h01);
                    h23 = f2_fma(pp[t + 1], f2_bc(tap[t]), h23);
                }
                // column pass: row r is tap t of Gaussian row r + G - t, whose accumulator
                // sits in ring slot (ph + G - t) mod NR (rb is a multiple of NR from r0)
#pragma unroll
                for (int t = 0; t < NR; ++t) {
                    const int slot = (ph + G - t + 2 * NR) % NR;
                    if (t == 0) {
                        acc[slot][0] = f2_fma(h01, f2_bc(tap[0]), f2_bc(0.0f));
                        acc[slot][1] = f2_fma(h23, f2_bc(tap[0]), f2_bc(0.0f));
                    } else {
                        acc[slot][0] = f2_fma(h01, f2_bc(tap[t]), acc[slot][0]);
                        acc[slot][1] = f2_fma(h23, f2_bc(tap[t]), acc[slot][1]);
                    }
                }
                // Gaussian row r - G is complete (tap 2G just added): round and emit
                const int gy = r - G;
                if (gy >= g0) {
                    const int slot = (ph + G - 2 * G + 2 * NR) % NR;
                    const float2 u01 = f2_add(acc[slot][0], f2_bc(8388608.0f));
                    const float2 u23 = f2_add(acc[slot][1], f2_bc(8388608.0f));
                    // u01 = (g0, g2), u23 = (g1, g3)
                    const uint32_t gw = __byte_perm(__byte_perm(__float_as_uint(u01.x), __float_as_uint(u23.x), 0x0040),
                                                    __byte_perm(__float_as_uint(u01.y), __float_as_uint(u23.y), 0x0040),
                                                    0x5410);
                    emit_gauss(gy, gw);
                }
            }
        }
    }
}

}  // namespace dmsgm
