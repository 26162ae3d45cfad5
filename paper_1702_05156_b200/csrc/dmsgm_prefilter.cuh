// dmsgm_prefilter.cuh -- the optional frame preprocessing of the step:
// separable Gaussian then 3x3 median (§2.1, §3.3.1, App. A/B;
// readings R30-R34 of DESIGN.md §2).
//
// One kernel, one 124 x 32 output tile per CTA (256 threads), everything in shared memory:
//   1. the input tile with a halo of R = g + m pixels (g = Gaussian radius, m = median
//      radius) is loaded with CLAMPED coordinates (R32) -- which makes both Gaussian
//      passes exact without further clamping (a row pass depends only on its image row);
//   2. row pass (fp32, fma chain in ascending tap order, R31) -> float tile;
//   3. column pass -> rounded to nearest-even, clamped to [0, 255] -> u8 tile;
//      positions outside the image are then overwritten by their clamped source (the
//      median's border rule, R32, R33);
//   4. 3x3 median of 4 pixels per thread (sorted columns, native u16x2 min/max),
//      written as 32-bit words.
// HBM traffic: 1 B/px read + 1 B/px written; the step kernel then reads the output.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dmsgm_math.cuh"
#include "dmsgm_pair.cuh"

namespace dmsgm {

constexpr int kPfTileX = 124;     // output columns per CTA (+ the median halo = 32 groups of 4)
constexpr int kPfTileY = 32;      // output rows per CTA
constexpr int kPfThreads = 256;
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
            mi[k][0] = med3_u16x2(c[k][0], c[k][1], c[k][2]);
            hi[k][0] = __vimax3_u16x2(c[k][0], c[k][1], c[k][2]);
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

// G = Gaussian radius, M = median radius (compile-time: the tile geometry depends on them)
template <int G, int M>
struct PfTile {
    static constexpr int R = G + M;                       // input halo (<= 4)
    static constexpr int IN_H = kPfTileY + 2 * R;         // input tile rows
    // input tile columns: x0 - 4 .. x0 + 128 + 4 (+ slack), so the tile's first column x0
    // sits on a 4-byte boundary: smem column j <-> image column x0 - 4 + j
    static constexpr int IN_PITCH = 160;                  // 10 chunks of 16 bytes (see the load)
    static constexpr int V_W = kPfTileX + 2 * M;          // Gaussian output columns (median halo)
    static constexpr int V_H = kPfTileY + 2 * M;
    static constexpr int H_PITCH = 128;                   // floats per row-pass row: 32 groups of 4
                                                          // (one per lane; V_W <= 126 are used)
    static constexpr int V_PITCH = 144;                   // bytes per Gaussian-output row
    static_assert(R <= 4, "halo of at most 4 pixels");
};

__device__ __forceinline__ uint32_t byte_at(uint32_t w0, uint32_t w1, uint32_t w2, int k) {
    // byte k (0..11) of the 12-byte little-endian string w0 w1 w2 (k is a compile-time constant)
    const uint32_t w = k < 4 ? w0 : (k < 8 ? w1 : w2);
    return (w >> (8 * (k & 3))) & 0xFFu;
}

// 0x4B000000 | byte k of the 12-byte string w0 w1 w2 (k a compile-time constant): one PRMT
__device__ __forceinline__ uint32_t byte_magic(uint32_t w0, uint32_t w1, uint32_t w2, int k) {
    const uint32_t w = k < 4 ? w0 : (k < 8 ? w1 : w2);
    return __byte_perm(w, 0x4B000000u, 0x7540u | (uint32_t)(k & 3));
}

template <int G, int M>
__global__ void __launch_bounds__(kPfThreads) dmsgm_prefilter_kernel(const PrefilterArgs a) {
    using T = PfTile<G, M>;
    constexpr int R = T::R;
    __shared__ __align__(16) uint8_t in_s[T::IN_H * T::IN_PITCH];
    __shared__ __align__(16) float h_s[G > 0 ? T::IN_H * T::H_PITCH : 4];
    __shared__ __align__(16) uint8_t v_s[T::V_H * T::V_PITCH];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int x0 = blockIdx.x * kPfTileX, y0 = blockIdx.y * kPfTileY, s = blockIdx.z;
    const uint8_t* in = a.in + (long long)s * a.in_stride;

    // 1. input rows y0-R .. y0+32+R, columns x0-4 .. x0+131, clamped (R32).  Smem column
    //    j of row r holds image column xs + j, xs = (x0 - 4) rounded down to 16 bytes; the
    //    tile starts at column o = x0 - 4 - xs (a multiple of 4).  Interior tiles (the 160
    //    bytes of every row inside the image rows and the row pitch): asynchronous 16-byte
    //    copies.  Border tiles: clamped 4-pixel words (W % 4 == 0, so a word is wholly inside
    //    or wholly outside the image; an outside word repeats the nearest border pixel).
    const int xs = (x0 - 4) & ~15, o = (x0 - 4) - xs;
    const bool interior = (((uintptr_t)in | (uintptr_t)a.in_pitch) & 15) == 0 && xs >= 0 &&
                          xs + T::IN_PITCH <= a.in_pitch && x0 + kPfTileX + R <= a.W && y0 - R >= 0 &&
                          y0 - R + T::IN_H <= a.H;
    if (interior) {
        const uint32_t dst0 = (uint32_t)__cvta_generic_to_shared(in_s);
        const uint8_t* src0 = in + (long long)(y0 - R) * a.in_pitch + xs;
        for (int i = threadIdx.x; i < T::IN_H * (T::IN_PITCH / 16); i += kPfThreads) {
            const int r = i / (T::IN_PITCH / 16), c = i - r * (T::IN_PITCH / 16);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst0 + r * T::IN_PITCH + 16 * c),
                         "l"(src0 + (long long)r * a.in_pitch + 16 * c) : "memory");
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    } else {
        constexpr int WORDS = 34;
        for (int i = threadIdx.x; i < T::IN_H * WORDS; i += kPfThreads) {
            const int r = i / WORDS, wc = i - r * WORDS;
            const int y = min(max(y0 - R + r, 0), a.H - 1);
            const uint8_t* row = in + (long long)y * a.in_pitch;
            const int x = x0 - 4 + 4 * wc;
            uint32_t w;
            if (x >= 0 && x < a.W) w = __ldg(reinterpret_cast<const unsigned int*>(row + x));
            else w = 0x01010101u * row[x < 0 ? 0 : a.W - 1];
            *reinterpret_cast<uint32_t*>(in_s + r * T::IN_PITCH + o + 4 * wc) = w;
        }
    }
    __syncthreads();

    // Gaussian output v_s: image rows y0-M .. y0+32+M, columns x0-M .. x0+128+M
    // (v column c <-> image column x0 - M + c)
    if constexpr (G > 0) {
        // 2. row pass, fp32 fma chain in ascending tap order (R31): every input row, 32
        //    groups of 4 output columns (lane l: group l)
        for (int r = warp; r < T::IN_H; r += kPfThreads / 32) {
            {
                const int g = lane;
                // inputs of v columns 4g .. 4g+3: smem columns 4g + (4 - R) + k, k = 0 .. 3 + 2G
                const uint32_t* src = reinterpret_cast<const uint32_t*>(in_s + r * T::IN_PITCH + o + 4 * g);
                const uint32_t w0 = src[0], w1 = src[1], w2 = src[2];
                // bytes as exact floats without conversion instructions: (0x4B000000 | b) is
                // 2^23 + b, minus 2^23 (pairs of FADD2)
                float p[4 + 2 * G + 1];
#pragma unroll
                for (int k = 0; k < 4 + 2 * G; k += 2) {
                    const float2 m = make_float2(__uint_as_float(byte_magic(w0, w1, w2, k + 4 - R)),
                                                 __uint_as_float(byte_magic(w0, w1, w2, k + 5 - R)));
                    const float2 v = f2_sub(m, f2_bc(8388608.0f));
                    p[k] = v.x;
                    p[k + 1] = v.y;
                }
                // outputs (0, 1) and (2, 3) as pairs: blur_q = fma(p[q + t], tap_t, blur_q),
                // t ascending from 0 (R31), lane by lane
                float2 o01 = f2_bc(0.0f), o23 = f2_bc(0.0f);
#pragma unroll
                for (int t = 0; t <= 2 * G; ++t) {
                    o01 = f2_fma(make_float2(p[t], p[t + 1]), f2_bc(a.taps[t]), o01);
                    o23 = f2_fma(make_float2(p[t + 2], p[t + 3]), f2_bc(a.taps[t]), o23);
                }
                *reinterpret_cast<float4*>(h_s + r * T::H_PITCH + 4 * g) = make_float4(o01.x, o01.y, o23.x, o23.y);
            }
        }
        __syncthreads();
        // 3. column pass at the V_H rows, rounded once to u8 (R31).  No clamp is needed:
        //    the taps are positive and sum to 1 within 1e-6, so 0 <= acc < 255.5
        for (int r = warp; r < T::V_H; r += kPfThreads / 32) {
            {
                const int g = lane;
                float2 acc01 = f2_bc(0.0f), acc23 = f2_bc(0.0f);
#pragma unroll
                for (int t = 0; t <= 2 * G; ++t) {
                    const float4 h = *reinterpret_cast<const float4*>(h_s + (r + t) * T::H_PITCH + 4 * g);
                    acc01 = f2_fma(make_float2(h.x, h.y), f2_bc(a.taps[t]), acc01);
                    acc23 = f2_fma(make_float2(h.z, h.w), f2_bc(a.taps[t]), acc23);
                }
                // nearest, ties to even: acc in [0, 255.5), so acc + 2^23 rounds to 2^23 + rint(acc)
                // and its low byte is the result
                const float2 u01 = f2_add(acc01, f2_bc(8388608.0f)), u23 = f2_add(acc23, f2_bc(8388608.0f));
                const uint32_t w = __byte_perm(__byte_perm(__float_as_uint(u01.x), __float_as_uint(u01.y), 0x0040),
                                               __byte_perm(__float_as_uint(u23.x), __float_as_uint(u23.y), 0x0040), 0x5410);
                *reinterpret_cast<uint32_t*>(v_s + r * T::V_PITCH + 4 * g) = w;
            }
        }
    } else {
        // no Gaussian: v = the input (v column c <-> smem column c + 4 - M)
        for (int r = warp; r < T::V_H; r += kPfThreads / 32)
            for (int c = lane; c < T::V_W; c += 32) v_s[r * T::V_PITCH + c] = in_s[r * T::IN_PITCH + o + c + 4 - M];
    }
    __syncthreads();

    if constexpr (M > 0) {
        // positions of v outside the image take their clamped value (the median clamps,
        // R32); the sources are inside the image and never written here: no race
        // (M = 1: at most the first / last row and the first / last columns of v; rows
        // first, then columns, so a corner takes the clamped corner value)
        const int last_r = min(T::V_H - 1, a.H - 1 - (y0 - M)), last_c = min(T::V_W - 1, a.W - 1 - (x0 - M));
        if (y0 == 0 || last_r < T::V_H - 1) {
            for (int c = threadIdx.x; c < T::V_W; c += kPfThreads) {
                if (y0 == 0) v_s[c] = v_s[T::V_PITCH + c];
                for (int r = last_r + 1; r < T::V_H; ++r) v_s[r * T::V_PITCH + c] = v_s[last_r * T::V_PITCH + c];
            }
            __syncthreads();
        }
        if (x0 == 0 || last_c < T::V_W - 1) {
            for (int r = threadIdx.x; r < T::V_H; r += kPfThreads) {
                uint8_t* row = v_s + r * T::V_PITCH;
                if (x0 == 0) row[0] = row[1];
                for (int c = last_c + 1; c < T::V_W; ++c) row[c] = row[last_c];
            }
            __syncthreads();
        }
    }

    // 4. median (or the Gaussian output itself): a warp per output row, 4 pixels per lane
    uint8_t* out = a.out + (long long)s * a.out_stride;
    for (int r = warp; r < kPfTileY; r += kPfThreads / 32) {
        const int y = y0 + r, x = x0 + 4 * lane;
        if (lane >= kPfTileX / 4 || y >= a.H || x >= a.W) continue;
        uint32_t w;
        if constexpr (M > 0) {
            uint32_t w0[3], w1[3];
#pragma unroll
            for (int dy = 0; dy < 3; ++dy) {
                const uint8_t* row = v_s + (r + dy) * T::V_PITCH + 4 * lane;
                w0[dy] = *reinterpret_cast<const uint32_t*>(row);       // columns x-1 .. x+2
                w1[dy] = *reinterpret_cast<const uint32_t*>(row + 4);   // x+3 .. x+6
            }
            w = median3x3x4(w0, w1);
        } else {
            w = *reinterpret_cast<const uint32_t*>(v_s + r * T::V_PITCH + 4 * lane);
        }
        *reinterpret_cast<uint32_t*>(out + (long long)y * a.out_pitch + x) = w;
    }
}

}  // namespace dmsgm
