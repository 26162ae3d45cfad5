// dmsgm_prefilter.cuh -- the optional frame preprocessing of the step:
// separable Gaussian then 3x3 median (§2.1, §3.3.1, App. C/D;
// readings R30-R34 of DESIGN.md §2).
//
// One streaming kernel (dmsgm_prefilter_kernel below): a warp walks a 240-column strip of
// a frame down kPfBand rows; the row pass, the column pass (a register ring of partial
// sums) and the median all stay in registers -- no shared memory, no CTA barriers.
// HBM traffic: 1 B/px read (+ the strips' column and band halos, L2-served) + 1 B/px
// written; the step kernel then reads the output.  The kernel is issue-bound, so the
// design minimises instructions per pixel.
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
    uint32_t one;                 // 1 (a runtime operand: see pf_sort3)
};

// Exact fp32 value 2^23 + byte k of w ("magic" float: its low byte is the byte, bytes 1-2
// are zero, byte 3 is 0x4B) -- one PRMT.
__device__ __forceinline__ uint32_t pf_magic(uint32_t w, int k) { return __byte_perm(w, 0x4B000000u, 0x7540u | (uint32_t)k); }

// 3x3 median building blocks on 16-bit lanes (two columns per register), with the native
// 2- and 3-input u16x2 min / max.
__device__ __forceinline__ uint32_t pf_med3(uint32_t a, uint32_t b, uint32_t c) {
    return __vmaxu2(__vminu2(a, b), __vminu2(__vmaxu2(a, b), c));
}
struct PfSorted {
    uint32_t lo, mi, hi;
};
// a column triple sorted per lane; the middle one is the sum minus the extremes (lanes <=
// 3 * 255: no carry or borrow crosses the 16-bit lanes)
#ifndef DMSGM_PF_IMAD_MED
#define DMSGM_PF_IMAD_MED 0
#endif
#ifndef DMSGM_PF_IMAD_SORT
#define DMSGM_PF_IMAD_SORT 1
#endif
__device__ __forceinline__ PfSorted pf_sort3(uint32_t a, uint32_t b, uint32_t c, uint32_t one) {
    PfSorted s;
    s.lo = __vimin3_u16x2(a, b, c);
    s.hi = __vimax3_u16x2(a, b, c);
#if DMSGM_PF_IMAD_SORT
    // the sum on the FMA pipe (IMAD x * one + y with `one` = 1 from the kernel parameters,
    // which ptxas cannot fold into an IADD3): the kernel is bound by the ALU pipe, where the
    // min / max / PRMT work runs
    uint32_t t;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(a), "r"(one), "r"(b));
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(c), "r"(one), "r"(t));
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(s.lo), "r"(0u - one), "r"(t));
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(s.mi) : "r"(s.hi), "r"(0u - one), "r"(t));
#else
    (void)one;
    s.mi = a + b + c - s.lo - s.hi;
#endif
    return s;
}
// Medians of the 3x3 windows of the C output columns x .. x+C-1 (R33).  ra / rb / rc = rows
// y-1 / y / y+1, each as C/2+1 words of column pairs: word k = (x-1+2k, x+2k) (16-bit
// lanes).  Window columns sorted once per row triple; median9 = med3(max3 of the lows, med3
// of the middles, min3 of the highs) over the window's three sorted columns (the
// sorted-columns identity).  Output pair j = columns (x+2j, x+2j+1) reads sorted words j,
// j+1 and their middle pair (x+2j, x+2j+1) = (hi half of word j, lo half of word j+1).
template <int C>
__device__ __forceinline__ void pf_median(const uint32_t (&ra)[C / 2 + 1], const uint32_t (&rb)[C / 2 + 1],
                                          const uint32_t (&rc)[C / 2 + 1], uint32_t (&o)[C / 4], uint32_t one) {
    constexpr int NW = C / 2 + 1;
    PfSorted s[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) s[k] = pf_sort3(ra[k], rb[k], rc[k], one);
    uint32_t p[C / 2];
#pragma unroll
    for (int j = 0; j < C / 2; ++j) {
        const uint32_t lo_m = __byte_perm(s[j].lo, s[j + 1].lo, 0x5432);
        const uint32_t mi_m = __byte_perm(s[j].mi, s[j + 1].mi, 0x5432);
        const uint32_t hi_m = __byte_perm(s[j].hi, s[j + 1].hi, 0x5432);
        // med3 of the middles: min / max on the ALU pipe, or (DMSGM_PF_IMAD_MED pairs of the C/2)
        // the sum minus the extremes with the sums on the FMA pipe (pf_sort3)
        const uint32_t mm = j < DMSGM_PF_IMAD_MED ? pf_sort3(s[j].mi, mi_m, s[j + 1].mi, one).mi
                                                  : pf_med3(s[j].mi, mi_m, s[j + 1].mi);
        p[j] = pf_med3(__vimax3_u16x2(s[j].lo, lo_m, s[j + 1].lo), mm, __vimin3_u16x2(s[j].hi, hi_m, s[j + 1].hi));
    }
#pragma unroll
    for (int q = 0; q < C / 4; ++q) o[q] = __byte_perm(p[2 * q], p[2 * q + 1], 0x6420);   // 4 columns as bytes
}

// ---------------------------------------------------------------------------
// Streaming kernel.  A warp owns a vertical strip of 30 C output columns x kPfBand rows of
// one frame.  Lane L holds the C columns x = xw - C + C L .. x + C - 1 as C/4 words (lanes
// 0 and 31 are the strip's column halo; lanes 1-30 write) and walks down the strip:
//   input row r (clamped, R32): C/4 4-byte cp.async per lane into a shared ring, U-1 rows
//     ahead (no register waits on a load in flight);
//   row pass (R31): the C outputs as C/2 pairs (x+j, x+j+C/2), fma(p, tap_t, acc) in
//     ascending t; an operand pair (p[x+k], p[x+k+C/2]) is two PRMTs into 2^23 + byte and
//     one paired subtraction -- 2G+C/2 pairs per row; bytes beyond the lane's own come from
//     the neighbours' words by two shuffles;
//   column pass: input row r contributes tap t to Gaussian row r + G - t, so 2G+1 partial
//     accumulators rotate through a register ring; the row loop is unrolled by the ring
//     size U, so every ring slot is a compile-time register.  Gaussian row r - G is
//     complete at tap 2G: acc + 2^23 holds its nearest-even rounding in the low byte;
//   median (R33): from those magic floats, the C/2+1 column-pair words of the Gaussian row
//     (one PRMT each; columns x-1 and x+C by one shuffle per side) enter a ring of U rows;
//     output row gy-1 is the median of Gaussian rows gy-2 .. gy (pf_median), C/4 stores.
// Borders (R32), all exact: input rows / columns are clamped when staged (edge words
// replicate the edge byte); Gaussian column -1 / W is column 0 / W-1 again (selects on the
// pair words), Gaussian row -1 is row 0 again (its words are copied into row -1's ring
// slot) and output row H-1 takes rows H-2, H-1, H-1.
// The steady-state rows of a band run without any of those checks (pf_row's CHECK /
// EDGE template flags); instructions per pixel are what bounds the kernel.
// ---------------------------------------------------------------------------
#ifndef DMSGM_PF_EDGE_SPLIT
#define DMSGM_PF_EDGE_SPLIT 0      // 1: a third copy of the row code without column clamping
#endif
#ifndef DMSGM_PF_COLS
#define DMSGM_PF_COLS 8
#endif
constexpr int kPfLaneCols = DMSGM_PF_COLS;   // columns per lane (4 or 8)
constexpr int kPfOutW = 30 * kPfLaneCols;    // output columns per warp (lanes 1..30)
#ifndef DMSGM_PF_BAND
#define DMSGM_PF_BAND 120
#endif
constexpr int kPfBand = DMSGM_PF_BAND;       // output rows per warp
#ifndef DMSGM_PF_WARPS
#define DMSGM_PF_WARPS 8
#endif
#ifndef DMSGM_PF_MINB
#define DMSGM_PF_MINB 2
#endif
constexpr int kPfWarps = DMSGM_PF_WARPS;     // warps per CTA (independent strips)

template <int G>
struct PfGeom {
    static constexpr int C = kPfLaneCols;
    static constexpr int WPL = C / 4;         // words per lane
    static constexpr int D = C / 2;           // pair distance: output pairs (x+j, x+j+D)
    static constexpr int NR = 2 * G + 1;      // column-pass ring
    static constexpr int U = G == 0 ? 3 : NR; // unroll = staging ring = median ring (>= 3)
    static constexpr int NW = C / 2 + 1;      // median column-pair words per row
    static constexpr int SLOT = 32 * C;       // bytes per staging ring slot (one row of the warp)
};

// Per-lane constants of a strip (see the kernel).
struct PfLane {
    uint32_t ring;                // shared address of this lane's word in ring slot 0
    const uint8_t* src[2];        // row-0 address of the lane's input words (clamped columns)
    uint8_t* dst;                 // row-0 address of the lane's output columns
    uint32_t sel[2];              // column clamping selectors (0x3210 = keep)
    int pitch_in, pitch_out, W, H, x;
    int ys, g0, r1;
    bool writer, clamp_l, clamp_m, clamp_r, bottom;
};

// One input row r at ring phase PH (compile-time: every ring slot is a fixed register).
// CHECK = false for the steady state, where the caller guarantees: r <= r1, the staged row
// r + U - 1 lies in [0, H-1] and <= r1, gy = r - G >= max(g0, ys + 1, 1) and gy < H - 1
// (no warm-up row, border row or band end).  EDGE = false when no lane of the warp
// touches a frame border (no column clamping).  Returns false when r is past the band.
template <int G, int M, int PH, bool CHECK, bool EDGE>
__device__ __forceinline__ bool pf_row(const PrefilterArgs& a, const PfLane& L, int r,
                                       float2 (&acc)[G > 0 ? 2 * G + 1 : 1][kPfLaneCols / 2],
                                       uint32_t (&mw)[M ? PfGeom<G>::U : 1][kPfLaneCols / 2 + 1]) {
    using Q = PfGeom<G>;
    constexpr int C = Q::C, D = Q::D, NR = Q::NR, U = Q::U, NW = Q::NW;
    if (CHECK && r > L.r1) return false;                     // warp-uniform
    // row r is in slot PH once at most U-2 younger groups are pending; then row r+U-1 goes
    // into slot PH-1 (row r-1's, consumed in the previous phase)
    asm volatile("cp.async.wait_group %0;" ::"n"(U - 2) : "memory");
    uint32_t w[Q::WPL];
    if constexpr (Q::WPL == 2)
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w[0]), "=r"(w[1]) : "r"(L.ring + PH * Q::SLOT) : "memory");
    else
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w[0]) : "r"(L.ring + PH * Q::SLOT) : "memory");
    if (EDGE) {
#pragma unroll
        for (int c = 0; c < Q::WPL; ++c) w[c] = __byte_perm(w[c], 0u, L.sel[c]);
    }
    {
        const int rs = r + U - 1;
        if (!CHECK || rs <= L.r1) {
            const long long ro = (long long)(CHECK ? min(max(rs, 0), L.H - 1) : rs) * L.pitch_in;
            const uint32_t d = L.ring + ((PH + U - 1) % U) * Q::SLOT;
#pragma unroll
            for (int c = 0; c < Q::WPL; ++c)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d + 4 * c), "l"(L.src[c] + ro) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    const int gy = r - G;                                    // the Gaussian row completed by row r
    uint32_t u[D][2];                                        // its C values as magic floats: (x+j, x+j+D)
    if constexpr (G > 0) {
        // row pass of input row r: bytes x-4 .. x+C+3 from the neighbours' words
        const uint32_t wl = __shfl_up_sync(0xffffffffu, w[Q::WPL - 1], 1), wr = __shfl_down_sync(0xffffffffu, w[0], 1);
        auto src = [&](int i) -> uint32_t {                  // magic float of byte x+i, i in [-G, C-1+G]
            return i < 0 ? pf_magic(wl, 4 + i) : (i < C ? pf_magic(w[i / 4], i % 4) : pf_magic(wr, i - C));
        };
        float2 pq[2 * G + D];                                // pq[k] = (p[x+k-G], p[x+k-G+D])
#pragma unroll
        for (int k = 0; k < 2 * G + D; ++k)
            pq[k] = f2_sub(make_float2(__uint_as_float(src(k - G)), __uint_as_float(src(k - G + D))), f2_bc(8388608.0f));
        float2 h[D];
#pragma unroll
        for (int j = 0; j < D; ++j) {
            h[j] = f2_mul(pq[j], f2_bc(a.taps[0]));          // fma(p, w0, 0.f)
#pragma unroll
            for (int t = 1; t < NR; ++t) h[j] = f2_fma(pq[j + t], f2_bc(a.taps[t]), h[j]);
        }
        // column pass: row r is tap t of Gaussian row r + G - t, ring slot (PH + 2G - t) mod NR
#pragma unroll
        for (int t = 0; t < NR; ++t) {
            const int slot = (PH + 2 * G - t) % NR;
#pragma unroll
            for (int j = 0; j < D; ++j)
                acc[slot][j] = t == 0 ? f2_mul(h[j], f2_bc(a.taps[0])) : f2_fma(h[j], f2_bc(a.taps[t]), acc[slot][j]);
        }
        if (CHECK && gy < L.g0) return true;                 // warm-up rows of the band
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const float2 v = f2_add(acc[PH % NR][j], f2_bc(8388608.0f));   // round to nearest even
            u[j][0] = __float_as_uint(v.x);
            u[j][1] = __float_as_uint(v.y);
        }
    } else {
#pragma unroll
        for (int j = 0; j < D; ++j) {
            u[j][0] = pf_magic(w[j / 4], j % 4);
            u[j][1] = pf_magic(w[(j + D) / 4], (j + D) % 4);
        }
    }
    auto mag = [&](int c) -> uint32_t { return c < D ? u[c][0] : u[c - D][1]; };   // column x+c, c in [0, C)
    if constexpr (M == 0) {
        // the Gaussian row is the output (g0 = ys .. g1 = ye - 1)
        if (L.writer) {
            uint8_t* o = L.dst + (long long)gy * L.pitch_out;
#pragma unroll
            for (int q = 0; q < Q::WPL; ++q)
                if (q == 0 || L.x + 4 * q < L.W)
                    *reinterpret_cast<uint32_t*>(o + 4 * q) =
                        __byte_perm(__byte_perm(mag(4 * q), mag(4 * q + 1), 0x0040),
                                    __byte_perm(mag(4 * q + 2), mag(4 * q + 3), 0x0040), 0x5410);
        }
    } else {
        // column-pair words (x-1+2k, x+2k) of Gaussian row gy, into ring slot PH
        uint32_t lm = __shfl_up_sync(0xffffffffu, mag(C - 1), 1);   // column x-1 (left lane's x+C-1)
        uint32_t rm = __shfl_down_sync(0xffffffffu, mag(0), 1);     // column x+C (right lane's x)
        uint32_t m4 = C == 8 ? mag(4) : 0u;                          // column x+4 (C = 8)
        if (EDGE) {                                                  // Gaussian column -1 := 0, W := W-1
            lm = L.clamp_l ? mag(0) : lm;
            rm = L.clamp_r ? mag(C - 1) : rm;
            if (C == 8) m4 = L.clamp_m ? mag(3) : m4;
        }
        auto colm = [&](int c) -> uint32_t { return c < 0 ? lm : (c >= C ? rm : (C == 8 && c == 4 ? m4 : mag(c))); };
        constexpr int P1 = (PH + U - 1) % U, P2 = (PH + U - 2) % U;
#pragma unroll
        for (int k = 0; k < NW; ++k) mw[PH][k] = __byte_perm(colm(2 * k - 1), colm(2 * k), 0x5410);
        if (CHECK && gy == 0) {                              // Gaussian row -1 := row 0 (R32)
#pragma unroll
            for (int k = 0; k < NW; ++k) mw[P1][k] = mw[PH][k];
        }
        auto emit = [&](int y, const uint32_t (&ra)[NW], const uint32_t (&rb)[NW], const uint32_t (&rc)[NW]) {
            uint32_t o[Q::WPL];
            pf_median<C>(ra, rb, rc, o, a.one);
            if (L.writer) {
                uint8_t* op = L.dst + (long long)y * L.pitch_out;
#pragma unroll
                for (int q = 0; q < Q::WPL; ++q)
                    if (q == 0 || L.x + 4 * q < L.W) *reinterpret_cast<uint32_t*>(op + 4 * q) = o[q];
            }
        };
        if (!CHECK || gy >= L.ys + 1) emit(gy - 1, mw[P2], mw[P1], mw[PH]);   // rows gy-2 .. gy
        if (CHECK && L.bottom && gy == L.H - 1) emit(gy, mw[P1], mw[PH], mw[PH]);   // row H-1: H-2, H-1, H-1
    }
    return true;
}

// U consecutive input rows rb .. rb + U - 1 (rb at ring phase 0)
template <int G, int M, bool CHECK, bool EDGE, int PH = 0>
__device__ __forceinline__ bool pf_block(const PrefilterArgs& a, const PfLane& L, int rb,
                                         float2 (&acc)[G > 0 ? 2 * G + 1 : 1][kPfLaneCols / 2],
                                         uint32_t (&mw)[M ? PfGeom<G>::U : 1][kPfLaneCols / 2 + 1]) {
    if constexpr (PH < PfGeom<G>::U) {
        if (!pf_row<G, M, PH, CHECK, EDGE>(a, L, rb + PH, acc, mw)) return false;
        return pf_block<G, M, CHECK, EDGE, PH + 1>(a, L, rb, acc, mw);
    } else {
        return true;
    }
}

template <int G, int M>
__global__ void __launch_bounds__(32 * kPfWarps, G >= 3 ? 1 : DMSGM_PF_MINB) dmsgm_prefilter_kernel(const PrefilterArgs a) {
    using Q = PfGeom<G>;
    constexpr int C = Q::C, U = Q::U;
    const int lane = threadIdx.x & 31;
    const int strip = blockIdx.x * kPfWarps + (threadIdx.x >> 5);
    const int xw = strip * kPfOutW;
    if (xw >= a.W) return;                          // warp-uniform
    const int s = blockIdx.z;
    const int ys = blockIdx.y * kPfBand;
    const int ye = min(ys + kPfBand, a.H);          // output rows [ys, ye)
    PfLane L;
    L.x = xw - C + C * lane;                        // this lane's first column
    L.W = a.W;
    L.H = a.H;
    L.pitch_in = a.in_pitch;
    L.pitch_out = a.out_pitch;
    L.writer = lane >= 1 && lane <= 30 && L.x < a.W;
    L.ys = ys;
    // Gaussian rows [g0, g1] feed the output rows (clamped to the image); input rows [r0, r1]
    L.g0 = M ? max(ys - 1, 0) : ys;
    const int g1 = M ? min(ye, a.H - 1) : ye - 1;
    const int r0 = L.g0 - G;
    L.r1 = g1 + G;
    L.bottom = ye == a.H;
    // Input rows are staged by cp.async into a per-warp shared-memory ring of U rows (C bytes
    // per lane), U-1 rows ahead of their use: no register ever waits on a load in flight
    // (a register ring of loads makes ptxas copy in-flight registers at the loop back edge).
    // Column clamping (R32) is folded into the staging: word c of the lane stages the aligned
    // word at column off and keeps it (selector 0x3210) or replicates its byte 0 / 3 (column
    // 0 / W-1) when the row is consumed.
    __shared__ __align__(16) uint32_t ring_all[kPfWarps * U * 32 * Q::WPL];
    L.ring = (uint32_t)__cvta_generic_to_shared(ring_all + ((threadIdx.x >> 5) * U * 32 + lane) * Q::WPL);
    const uint8_t* in = a.in + (long long)s * a.in_stride;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const int col = L.x + 4 * c;
        L.src[c] = in + (col < 0 ? 0 : (col + 4 > a.W ? a.W - 4 : col));
        L.sel[c] = col < 0 ? 0x0000u : (col + 4 > a.W ? 0x3333u : 0x3210u);
    }
    L.dst = a.out + (long long)s * a.out_stride + L.x;
    // Gaussian column clamping for the median: column -1 := 0, column W := W-1
    L.clamp_l = L.x == 0;
    L.clamp_m = C == 8 && L.x + 4 == a.W;
    L.clamp_r = L.x + C == a.W;
    const bool edge = xw - C < 0 || xw + kPfOutW + C > a.W;   // warp-uniform

#pragma unroll
    for (int j = 0; j < U - 1; ++j) {
        const uint32_t d = L.ring + j * Q::SLOT;
        const long long ro = (long long)min(max(r0 + j, 0), a.H - 1) * a.in_pitch;
#pragma unroll
        for (int c = 0; c < Q::WPL; ++c)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d + 4 * c), "l"(L.src[c] + ro) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    float2 acc[G > 0 ? Q::NR : 1][Q::D];
    uint32_t mw[M ? U : 1][Q::NW];                  // median ring: column-pair words per Gaussian row

    // blocks of U rows from r0: checked ones (band start, band end, frame borders) around a
    // steady state of unchecked blocks rb in [lo_u, hi_u] (pf_row's CHECK = false contract)
    const int lo_u = max(r0 + 2 * G, max(ys + 1 + G, 1 + G));
    const int hi_u = min(L.r1 - 2 * U + 2, min(a.H - 2 * U + 1, a.H - 1 + G - U));
    int rb = r0;
    for (; rb <= L.r1 && (rb < lo_u || rb > hi_u); rb += U)
        if (!pf_block<G, M, true, true>(a, L, rb, acc, mw)) return;      // the band ended inside the block
#if DMSGM_PF_EDGE_SPLIT
    if (edge) {
        for (; rb <= hi_u; rb += U) pf_block<G, M, false, true>(a, L, rb, acc, mw);
    } else {
        for (; rb <= hi_u; rb += U) pf_block<G, M, false, false>(a, L, rb, acc, mw);
    }
#else
    (void)edge;
    for (; rb <= hi_u; rb += U) pf_block<G, M, false, true>(a, L, rb, acc, mw);
#endif
    for (; rb <= L.r1; rb += U)
        if (!pf_block<G, M, true, true>(a, L, rb, acc, mw)) return;
}

}  // namespace dmsgm
