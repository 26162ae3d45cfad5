// dmsgm_klt.cuh -- sm_100a kernels of the motion estimation that feeds the DMSGM step its
// homographies (App. F: goodFeaturesToTrack ->
// calcOpticalFlowPyrLK(Size(20,20), 5) -> findHomography(CV_RANSAC)).  Readings R38-R42
// (include/dmsgm_klt.h).  One launch of each kernel covers every stream of
// the batch:
//   klt_score_kernel    exact Sobel/structure tensor, fp64 lambda_min, 3x3 local maxima
//                       appended as 64-bit keys (score bits | ~raster index), per-stream
//                       max score (R38)
//   klt_select_kernel   one CTA per stream: exact top-2048 of the qualifying keys by an
//                       8-pass radix select, bitonic sort in shared memory, greedy
//                       min-distance selection by one warp over a cell grid (R38)
//   klt_pyramid_kernel  all box-pyramid levels of prev and next in one pass, 16-byte rows (R39)
//   klt_lk_kernel       one warp per corner, pyramidal Lucas-Kanade in fp32 (R40)
//   klt_compact_kernel  tracked pairs -> RANSAC matches (f64), one warp per stream
//   klt_ransac_kernel   one warp per (stream, 4 iterations): SplitMix64 sample, 8x8 fp64
//                       solve row-parallel on 8 lanes, inlier count (R42)
//   klt_refit_kernel    one warp per stream: best model, its inliers, normalized DLT by
//                       the smallest eigenvector of A^T A (inverse iteration, fp64) (R41)
#pragma once
#include <cuda_runtime.h>
#include <limits.h>
#include <stdint.h>

#include "dmsgm_pair.cuh"     // paired fp32 (FFMA2 / FMUL2 / FADD2)

namespace dmsgm_klt {

using dmsgm::f2_add;
using dmsgm::f2_bc;
using dmsgm::f2_fma;
using dmsgm::f2_mul;
using dmsgm::f2_sub;

constexpr int kMaxLevels = 6;        // levels 0..5
constexpr int kMaxCorners = 1024;
constexpr int kBatch = 2048;         // keys per greedy batch (radix-selected, then sorted)
constexpr int kSelThreads = 1024;
constexpr int kTX = 32, kTY = 8;     // score tile

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// ---------------------------------------------------------------------------------------
// K1: Shi-Tomasi score (R38) + 3x3 local maxima -> candidate keys, per-stream max score
// ---------------------------------------------------------------------------------------
struct ScoreArgs {
    const uint8_t* frames;
    long long fstride;
    int pitch, W, H;
    unsigned long long* cand;   // [S][cap]
    int cap;
    unsigned* count;            // [S]
    unsigned* maxbits;          // [S] float bits of the max score (scores are >= +0)
};

__global__ void __launch_bounds__(256) klt_score_kernel(const ScoreArgs a) {
    const int s = blockIdx.z;
    const uint8_t* f = a.frames + (long long)s * a.fstride;
    const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
    const int W = a.W, H = a.H, pitch = a.pitch;
    // gradients at (clamp(x0-2+i), clamp(y0-2+j)): the replicated-border gradient products
    // of the structure-tensor window (the oracle pads the products, not the pixels)
    __shared__ int gxs[kTY + 4][kTX + 4];
    __shared__ int gys[kTY + 4][kTX + 4];
    __shared__ float sc[kTY + 2][kTX + 2];
    __shared__ float wmax[8];
    const int tid = threadIdx.x;
    for (int k = tid; k < (kTY + 4) * (kTX + 4); k += 256) {
        const int j = k / (kTX + 4), i = k - j * (kTX + 4);
        const int X = clampi(x0 - 2 + i, 0, W - 1), Y = clampi(y0 - 2 + j, 0, H - 1);
        const int xm = X > 0 ? X - 1 : 0, xp = X < W - 1 ? X + 1 : W - 1;
        const int ym = Y > 0 ? Y - 1 : 0, yp = Y < H - 1 ? Y + 1 : H - 1;
        const uint8_t* rm = f + (long long)ym * pitch;
        const uint8_t* r0 = f + (long long)Y * pitch;
        const uint8_t* rp = f + (long long)yp * pitch;
        const int mm = __ldg(rm + xm), m0 = __ldg(rm + X), mp = __ldg(rm + xp);
        const int zm = __ldg(r0 + xm), zp = __ldg(r0 + xp);
        const int pm = __ldg(rp + xm), p0 = __ldg(rp + X), pp = __ldg(rp + xp);
        gxs[j][i] = (mp + 2 * zp + pp) - (mm + 2 * zm + pm);
        gys[j][i] = (pm + 2 * p0 + pp) - (mm + 2 * m0 + mp);
    }
    __syncthreads();
    for (int k = tid; k < (kTY + 2) * (kTX + 2); k += 256) {
        const int j = k / (kTX + 2), i = k - j * (kTX + 2);
        const int X = x0 - 1 + i, Y = y0 - 1 + j;
        float v = -1.0f;                              // outside the frame: never compared
        if (X >= 0 && X < W && Y >= 0 && Y < H) {
            int sa = 0, sb = 0, scc = 0;
#pragma unroll
            for (int dy = 0; dy < 3; ++dy)
#pragma unroll
                for (int dx = 0; dx < 3; ++dx) {
                    const int gx = gxs[j + dy][i + dx], gy = gys[j + dy][i + dx];
                    sa += gx * gx;
                    sb += gx * gy;
                    scc += gy * gy;
                }
            const long long d = (long long)(sa - scc) * (long long)(sa - scc) + 4LL * (long long)sb * (long long)sb;
            const double lam = __dmul_rn(__dsub_rn((double)(sa + scc), __dsqrt_rn((double)d)), 0.5);
            v = __double2float_rn(lam);
        }
        sc[j][i] = v;
    }
    __syncthreads();
    const int tx = tid & 31, ty = tid >> 5;
    const int x = x0 + tx, y = y0 + ty;
    const bool in = x < W && y < H;
    const float v = in ? sc[ty + 1][tx + 1] : 0.0f;
    bool cand = in && x >= 1 && x < W - 1 && y >= 1 && y < H - 1 && v > 0.0f;
    if (cand) {
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
            for (int dx = 0; dx < 3; ++dx) cand &= v >= sc[ty + dy][tx + dx];
    }
    // block max of the score over every pixel of the frame (the oracle's score.max())
    float m = v;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (tx == 0) wmax[ty] = m;
    // candidates: warp-aggregated append
    const unsigned bal = __ballot_sync(0xffffffffu, cand);
    if (bal) {
        unsigned base = 0;
        if (tx == 0) base = atomicAdd(a.count + s, (unsigned)__popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (cand) {
            const unsigned pos = base + __popc(bal & ((1u << tx) - 1u));
            const unsigned idx = (unsigned)(y * W + x);
            if (pos < (unsigned)a.cap)
                a.cand[(long long)s * a.cap + pos] =
                    ((unsigned long long)__float_as_uint(v) << 32) | (unsigned long long)(0xFFFFFFFFu - idx);
        }
    }
    __syncthreads();
    if (tid == 0) {
        float bm = wmax[0];
        for (int w = 1; w < 8; ++w) bm = fmaxf(bm, wmax[w]);
        atomicMax(a.maxbits + s, __float_as_uint(bm));    // scores >= +0: bits order like values
    }
}

// Streaming form of K1 for 4-byte aligned frames (W % 4 = 0): a warp walks a vertical strip
// of 120 columns down kScoreBand rows; lane L holds columns x = xw - 4 + 4L .. x + 3 (lanes 0
// and 31 are the strip's halo, lanes 1-30 produce).  Per input row r (clamped: the Sobel of
// replicated pixels, R38): the horizontal Sobel parts dX = p(c+1) - p(c-1) and
// sX = p(c-1) + 2 p(c) + p(c+1) into a 3-row ring; gradient row g = r - 1, its products
// Ix^2, IxIy, Iy^2 and their horizontal 3-sums (neighbour columns by shuffles, columns -1 / W
// replicated) into a 3-row ring (product row -1 / H is row 0 / H-1 again: the oracle pads the
// products, not the pixels); score row t = r - 2 from the vertical 3-sums (exact integers,
// fp64 lambda_min, identical to K1); 3x3 local-maximum test of row m = r - 3 against the score
// ring.  Candidates and the per-stream maximum exactly as K1.  ~8x fewer instructions than K1,
// whose 32x8 tiles recompute 1.7x the gradients and 1.3x the scores with byte loads.
constexpr int kScoreBand = 120;
#ifndef DMSGM_SCORE_PREFETCH
#define DMSGM_SCORE_PREFETCH 8
#endif
constexpr int kScorePrefetch = DMSGM_SCORE_PREFETCH;
constexpr int kCbuf = 384;          // per-warp candidate buffer (keys): flushed above kCbuf - 128
constexpr int kScoreWarps = 8;

struct ScoreLane {
    float sl, s0[4], sr;      // a score row: left neighbour column, own 4, right neighbour column
};

__device__ __forceinline__ float klt_lambda_min(int a, int b, int c) {
    const double t = (double)(a - c), tb = (double)b;
    const double d = __fma_rn(t, t, __dmul_rn(4.0 * tb, tb));        // exact: < 2^51
    return __double2float_rn(__dmul_rn(__dsub_rn((double)(a + c), __dsqrt_rn(d)), 0.5));
}

__global__ void __launch_bounds__(32 * kScoreWarps) klt_score_stream_kernel(const ScoreArgs a) {
    const int lane = threadIdx.x & 31;
    const int strip = blockIdx.x * kScoreWarps + (threadIdx.x >> 5);
    const int xw = strip * 120;
    const int W = a.W, H = a.H;
    if (xw >= W) return;                                   // warp-uniform
    const int s = blockIdx.z;
    const int ys = blockIdx.y * kScoreBand, ye = min(ys + kScoreBand, H);
    const uint8_t* f = a.frames + (long long)s * a.fstride;
    const int x = xw - 4 + 4 * lane;
    const bool mine = lane >= 1 && lane <= 30 && x < W;    // this lane's columns are produced here
    // clamped word load (columns -4..-1 replicate column 0, columns >= W replicate W-1)
    const int off = x < 0 ? 0 : (x >= W ? W - 4 : x);
    const uint32_t sel = x < 0 ? 0x0000u : (x >= W ? 0x3333u : 0x3210u);
    const bool cl = x == 0, cr = x + 4 == W;               // product columns -1 / W replicated
    int dX[3][4], sX[3][4];                                // horizontal Sobel parts, rows r mod 3
    int hxx[3][4], hxy[3][4], hyy[3][4];                   // horizontal 3-sums of the products
    ScoreLane sc[3];                                       // score rows
    float smax = 0.0f;
    // candidate keys of this warp, flushed to the stream's list in blocks
    __shared__ unsigned long long cbuf_all[kScoreWarps][kCbuf];
    unsigned long long* cbuf = cbuf_all[threadIdx.x >> 5];
    int nbuf = 0;                                          // (warp-uniform)
    auto flush = [&]() {
        __syncwarp();
        if (nbuf == 0) return;
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(a.count + s, (unsigned)nbuf);
        base = __shfl_sync(0xffffffffu, base, 0);
        for (int i = lane; i < nbuf; i += 32)
            if (base + i < (unsigned)a.cap) a.cand[(long long)s * a.cap + base + i] = cbuf[i];
        __syncwarp();
        nbuf = 0;
    };
    const int r0 = ys - 3, r1 = ye + 2;
    // the input word of the NEXT row is loaded one row ahead (its L1 / L2 latency hides
    // behind this row's arithmetic)
    uint32_t wnext = __ldg(reinterpret_cast<const unsigned int*>(f + (long long)clampi(r0, 0, H - 1) * a.pitch + off));
    for (int rb = r0; rb <= r1; rb += 3) {
#pragma unroll
        for (int ph = 0; ph < 3; ++ph) {
            const int r = rb + ph;
            if (r > r1) break;                             // warp-uniform
            // --- input row r: dX, sX of columns x .. x+3 ---
            {
                // the row kScorePrefetch ahead into L1: the one-ahead load then waits ~L1, not HBM
                asm volatile("prefetch.global.L1 [%0];" ::"l"(f + (long long)clampi(r + kScorePrefetch, 0, H - 1) * a.pitch + off));
                const uint32_t w = __byte_perm(wnext, 0u, sel);
                wnext = __ldg(reinterpret_cast<const unsigned int*>(f + (long long)clampi(r + 1, 0, H - 1) * a.pitch + off));
                const uint32_t wl = __shfl_up_sync(0xffffffffu, w, 1), wr = __shfl_down_sync(0xffffffffu, w, 1);
                int p[6];
                p[0] = (int)(wl >> 24);
#pragma unroll
                for (int k = 0; k < 4; ++k) p[k + 1] = (int)((w >> (8 * k)) & 0xFFu);
                p[5] = (int)(wr & 0xFFu);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    dX[ph][c] = p[c + 2] - p[c];
                    sX[ph][c] = p[c] + 2 * p[c + 1] + p[c + 2];
                }
            }
            // --- gradient row g = r - 1 (dX / sX rows g-1, g, g+1 = ring slots ph-2, ph-1, ph) ---
            const int g = r - 1;
            const int pm1 = (ph + 2) % 3, pm2 = (ph + 1) % 3;
            if (g >= 0 && g >= ys - 2 && g <= H) {
                if (g < H) {
                    int Pxx[4], Pxy[4], Pyy[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int ix = dX[pm2][c] + 2 * dX[pm1][c] + dX[ph][c];
                        const int iy = sX[ph][c] - sX[pm2][c];
                        Pxx[c] = ix * ix;
                        Pxy[c] = ix * iy;
                        Pyy[c] = iy * iy;
                    }
                    int lxx = __shfl_up_sync(0xffffffffu, Pxx[3], 1), rxx = __shfl_down_sync(0xffffffffu, Pxx[0], 1);
                    int lxy = __shfl_up_sync(0xffffffffu, Pxy[3], 1), rxy = __shfl_down_sync(0xffffffffu, Pxy[0], 1);
                    int lyy = __shfl_up_sync(0xffffffffu, Pyy[3], 1), ryy = __shfl_down_sync(0xffffffffu, Pyy[0], 1);
                    if (cl) { lxx = Pxx[0]; lxy = Pxy[0]; lyy = Pyy[0]; }
                    if (cr) { rxx = Pxx[3]; rxy = Pxy[3]; ryy = Pyy[3]; }
                    // slot of hs row g: the ring is indexed by the row of the NEXT stage, g -> (ph + 2) % 3
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        hxx[pm1][c] = (c == 0 ? lxx : Pxx[c - 1]) + Pxx[c] + (c == 3 ? rxx : Pxx[c + 1]);
                        hxy[pm1][c] = (c == 0 ? lxy : Pxy[c - 1]) + Pxy[c] + (c == 3 ? rxy : Pxy[c + 1]);
                        hyy[pm1][c] = (c == 0 ? lyy : Pyy[c - 1]) + Pyy[c] + (c == 3 ? ryy : Pyy[c + 1]);
                    }
                    if (g == 0) {                          // product row -1 := row 0
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            hxx[pm2][c] = hxx[pm1][c]; hxy[pm2][c] = hxy[pm1][c]; hyy[pm2][c] = hyy[pm1][c];
                        }
                    }
                } else {                                   // g == H: product row H := row H-1
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        hxx[pm1][c] = hxx[pm2][c]; hxy[pm1][c] = hxy[pm2][c]; hyy[pm1][c] = hyy[pm2][c];
                    }
                }
            }
            // --- score row t = r - 2 (hs rows t-1, t, t+1 = slots ph, ph+1, ph+2 of the hs ring:
            //     hs row q sits in slot (q + 1 - r0) mod 3 ... i.e. rows t-1 / t / t+1 in pm2 / ph / pm1) ---
            const int t = r - 2;
            if (t >= max(ys - 1, 0) && t <= min(ye, H - 1)) {
                ScoreLane& S = sc[ph];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int sa = hxx[pm2][c] + hxx[ph][c] + hxx[pm1][c];
                    const int sb = hxy[pm2][c] + hxy[ph][c] + hxy[pm1][c];
                    const int scc = hyy[pm2][c] + hyy[ph][c] + hyy[pm1][c];
                    S.s0[c] = klt_lambda_min(sa, sb, scc);
                    if (mine && t >= ys && t < ye && x + c < W) smax = fmaxf(smax, S.s0[c]);
                }
                S.sl = __shfl_up_sync(0xffffffffu, S.s0[3], 1);
                S.sr = __shfl_down_sync(0xffffffffu, S.s0[0], 1);
            }
            // --- local maxima of row m = r - 3 (score rows m-1, m, m+1 = slots ph-2, ph-1, ph) ---
            const int m = r - 3;
            if (m >= max(ys, 1) && m <= min(ye - 1, H - 2)) {
                const ScoreLane& U = sc[pm2];
                const ScoreLane& C = sc[pm1];
                const ScoreLane& D = sc[ph];
                bool cand[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const float v = C.s0[c];
                    const float ul = c == 0 ? U.sl : U.s0[c - 1], ur = c == 3 ? U.sr : U.s0[c + 1];
                    const float cl_ = c == 0 ? C.sl : C.s0[c - 1], cr_ = c == 3 ? C.sr : C.s0[c + 1];
                    const float dl = c == 0 ? D.sl : D.s0[c - 1], dr = c == 3 ? D.sr : D.s0[c + 1];
                    const float nb = fmaxf(fmaxf(fmaxf(ul, U.s0[c]), fmaxf(ur, cl_)), fmaxf(fmaxf(cr_, dl), fmaxf(D.s0[c], dr)));
                    const int xc = x + c;
                    cand[c] = mine && xc >= 1 && xc < W - 1 && v > 0.0f && v >= nb;
                }
                // append to the warp's shared-memory buffer (every lane takes part: cand is
                // false where not mine); the buffer goes to the stream's list by one atomic
                // per flush (an atomic per ballot left the warp waiting on its round trip)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const unsigned bal = __ballot_sync(0xffffffffu, cand[c]);
                    if (cand[c]) {
                        const unsigned idx = (unsigned)(m * W + x + c);
                        cbuf[nbuf + __popc(bal & ((1u << lane) - 1u))] =
                            ((unsigned long long)__float_as_uint(C.s0[c]) << 32) | (unsigned long long)(0xFFFFFFFFu - idx);
                    }
                    nbuf += __popc(bal);
                }
                if (nbuf > kCbuf - 128) flush();
            }
        }
    }
    flush();
    // per-stream max over every pixel (scores >= +0: bits order like values)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) smax = fmaxf(smax, __shfl_xor_sync(0xffffffffu, smax, o));
    if (lane == 0) atomicMax(a.maxbits + s, __float_as_uint(smax));
}

// ---------------------------------------------------------------------------------------
// K2: quality threshold, exact top-kBatch radix select, bitonic sort, greedy min-distance
// ---------------------------------------------------------------------------------------
struct SelectArgs {
    const unsigned long long* cand;
    int cap;
    const unsigned* count;
    const unsigned* maxbits;
    double quality, min_dist2;
    int W, max_corners;
    int cell, gw, gh;            // greedy cell grid: cell side (px), columns, rows
    uint16_t* grid_global;       // [S][gh][gw] when the grid does not fit shared memory (else null)
    int* corners_out;            // [S][max_corners][2]
    int* counts_out;             // [S]
    unsigned* overflow;          // set to 1 if a stream had more candidates than cap
};

__device__ __forceinline__ bool qualifies(unsigned long long k, double thr) {
    return (double)__uint_as_float((unsigned)(k >> 32)) >= thr;
}

__global__ void __launch_bounds__(kSelThreads) klt_select_kernel(const SelectArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    unsigned long long* batch = reinterpret_cast<unsigned long long*>(sm);      // [kBatch]
    unsigned* hist = reinterpret_cast<unsigned*>(batch + kBatch);               // [256]
    int* kept = reinterpret_cast<int*>(hist + 256);                             // [kMaxCorners][2]
    uint32_t* pxy = reinterpret_cast<uint32_t*>(kept + 2 * kMaxCorners);        // [kBatch] x | y << 16
    uint32_t* pcell = pxy + kBatch;                                              // [kBatch] cx | cy << 16
    uint16_t* grid_s = reinterpret_cast<uint16_t*>(pcell + kBatch);
    __shared__ unsigned long long s_prefix, s_mask;
    __shared__ unsigned s_rem, s_total, s_m;
    __shared__ int s_nkept, s_done, s_exact;
    const int s = blockIdx.x, tid = threadIdx.x;
    const unsigned cnt = a.count[s];
    if (tid == 0 && cnt > (unsigned)a.cap) *a.overflow = 1u;
    const int n = cnt < (unsigned)a.cap ? (int)cnt : a.cap;
    const unsigned long long* cand = a.cand + (long long)s * a.cap;
    const float mx = __uint_as_float(a.maxbits[s]);
    const double thr = a.quality * (double)mx;
    uint16_t* grid = a.grid_global ? a.grid_global + (long long)s * a.gw * a.gh : grid_s;
    const int ncell = a.gw * a.gh;
    for (int i = tid; i < ncell; i += kSelThreads) grid[i] = 0;
    if (tid == 0) { s_nkept = 0; s_done = !(mx > 0.0f) || a.max_corners == 0; }
    __syncthreads();
    unsigned long long upper = ~0ull;             // this batch: keys below `upper`
    while (!s_done) {
        // ---- exact radix select of the kBatch-th largest qualifying key below `upper` ----
        if (tid == 0) { s_prefix = 0; s_mask = 0; s_rem = kBatch; s_exact = 0; }
        unsigned long long cut = 0;
        bool all = false;
        for (int pass = 0; pass < 8; ++pass) {
            const int shift = 56 - 8 * pass;
            if (tid < 256) hist[tid] = 0;
            __syncthreads();
            const unsigned long long pre = s_prefix, msk = s_mask;
            // 8 keys per thread in flight (one load at a time left the pass latency-bound)
            for (int i0 = tid; i0 < n; i0 += 8 * kSelThreads) {
                unsigned long long kk[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int i = i0 + u * kSelThreads;
                    kk[u] = i < n ? cand[i] : ~0ull;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const unsigned long long k = kk[u];
                    if (i0 + u * kSelThreads < n && k < upper && (k & msk) == pre && qualifies(k, thr))
                        atomicAdd(&hist[(k >> shift) & 255u], 1u);
                }
            }
            __syncthreads();
            if (tid == 0) {
                if (pass == 0) {
                    unsigned t = 0;
                    for (int d = 0; d < 256; ++d) t += hist[d];
                    s_total = t;
                }
                if (pass > 0 || s_total > (unsigned)kBatch) {
                    unsigned cum = 0, rem = s_rem;
                    int d = 255;
                    for (; d > 0; --d) {
                        if (cum + hist[d] >= rem) break;
                        cum += hist[d];
                    }
                    s_rem = rem - cum;
                    s_prefix |= (unsigned long long)d << shift;
                    s_mask |= 0xFFull << shift;
                    // the whole bucket d is needed: keys >= prefix | d << shift (low bits 0)
                    // are exactly the kBatch largest -- the remaining passes would only find
                    // the smallest of them
                    s_exact = hist[d] == rem - cum;
                }
            }
            __syncthreads();
            if (s_total <= (unsigned)kBatch) { all = true; break; }
            if (s_exact) break;
        }
        if (!all) cut = s_prefix;                 // the kBatch-th largest key (keys are unique)
        // ---- gather the batch: qualifying keys in [cut, upper) ----
        if (tid == 0) s_m = 0;
        __syncthreads();
        for (int i0 = tid & ~31; i0 < n; i0 += 4 * kSelThreads) {       // warp-aggregated append
            unsigned long long kk[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * kSelThreads + (tid & 31);
                kk[u] = i < n ? cand[i] : 0ull;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * kSelThreads + (tid & 31);
                const unsigned long long k = kk[u];
                const bool in = i < n && k < upper && k >= cut && qualifies(k, thr);
                const unsigned bal = __ballot_sync(0xffffffffu, in);
                unsigned b0 = 0;
                if ((tid & 31) == 0 && bal) b0 = atomicAdd(&s_m, (unsigned)__popc(bal));
                b0 = __shfl_sync(0xffffffffu, b0, 0);
                if (in) batch[b0 + __popc(bal & ((1u << (tid & 31)) - 1u))] = k;
            }
        }
        __syncthreads();
        const int m = (int)s_m;
        int P = 1;
        while (P < m) P <<= 1;
        for (int i = m + tid; i < P; i += kSelThreads) batch[i] = 0ull;
        __syncthreads();
        // ---- bitonic sort, descending ----
        for (int size = 2; size <= P; size <<= 1)
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int i = tid; i < P; i += kSelThreads) {
                    const int j = i ^ stride;
                    if (j > i) {
                        const unsigned long long u = batch[i], w = batch[j];
                        const bool desc = (i & size) == 0;
                        if (desc ? (u < w) : (u > w)) { batch[i] = w; batch[j] = u; }
                    }
                }
                __syncthreads();
            }
        // ---- decode the batch in parallel: pixel and greedy cell of every key ----
        for (int j = tid; j < m; j += kSelThreads) {
            const unsigned idx = 0xFFFFFFFFu - (unsigned)batch[j];
            const int y = (int)(idx / (unsigned)a.W), x = (int)(idx - (unsigned)y * (unsigned)a.W);
            pxy[j] = (uint32_t)x | ((uint32_t)y << 16);
            pcell[j] = (uint32_t)(x / a.cell) | ((uint32_t)(y / a.cell) << 16);
        }
        __syncthreads();
        // ---- greedy selection by warp 0, 32 keys at a time (a cell holds at most one kept
        //      corner; cells of side ceil(d / sqrt 2), so a conflict lies within +-2 cells):
        //      (1) each lane tests its key against the corners kept so far (grid);
        //      (2) each lane collects which EARLIER surviving keys of the chunk lie within d;
        //      (3) a 32-step scan in rank order keeps a survivor iff none of its earlier
        //          conflicting survivors was kept -- exactly the sequential greedy's decisions;
        //      (4) the kept ones are appended in rank order (up to max_corners). ----
        if (tid < 32) {
            const int lane = tid;
            int nk = s_nkept;
            for (int base = 0; base < m && nk < a.max_corners; base += 32) {
                const int j = base + lane;
                const bool valid = j < m;
                const uint32_t xy = valid ? pxy[j] : 0u, ce = valid ? pcell[j] : 0u;
                const int x = (int)(xy & 0xFFFFu), y = (int)(xy >> 16);
                const int cx = (int)(ce & 0xFFFFu), cy = (int)(ce >> 16);
                bool conflict = false;
                if (valid) {
                    for (int gy = max(cy - 2, 0); gy <= min(cy + 2, a.gh - 1) && !conflict; ++gy)
                        for (int gx = max(cx - 2, 0); gx <= min(cx + 2, a.gw - 1); ++gx) {
                            const int e = grid[gy * a.gw + gx];
                            if (e) {
                                const int ddx = x - kept[2 * (e - 1)], ddy = y - kept[2 * (e - 1) + 1];
                                if ((double)(ddx * ddx + ddy * ddy) < a.min_dist2) { conflict = true; break; }
                            }
                        }
                }
                const unsigned surv = __ballot_sync(0xffffffffu, valid && !conflict);
                unsigned earlier = 0;                   // earlier survivors of the chunk within d
                for (int k = 0; k < 32; ++k) {
                    const int xk = __shfl_sync(0xffffffffu, x, k), yk = __shfl_sync(0xffffffffu, y, k);
                    const int ddx = x - xk, ddy = y - yk;
                    if (k < lane && ((surv >> k) & 1u) && (double)(ddx * ddx + ddy * ddy) < a.min_dist2)
                        earlier |= 1u << k;
                }
                unsigned keep = 0;
                int room = a.max_corners - nk;
                for (int k = 0; k < 32 && room > 0; ++k) {
                    const unsigned ek = __shfl_sync(0xffffffffu, earlier, k);
                    if (((surv >> k) & 1u) && !(ek & keep)) { keep |= 1u << k; --room; }
                }
                if ((keep >> lane) & 1u) {
                    const int idx = nk + __popc(keep & ((1u << lane) - 1u));
                    kept[2 * idx] = x;
                    kept[2 * idx + 1] = y;
                    grid[cy * a.gw + cx] = (uint16_t)(idx + 1);
                    a.corners_out[((long long)s * a.max_corners + idx) * 2] = x;
                    a.corners_out[((long long)s * a.max_corners + idx) * 2 + 1] = y;
                }
                nk += __popc(keep);
                __syncwarp();
            }
            if (lane == 0) {
                s_nkept = nk;
                s_done = nk >= a.max_corners || all;
            }
        }
        __syncthreads();
        upper = cut;
    }
    if (tid == 0) a.counts_out[s] = s_nkept;
}

// ---------------------------------------------------------------------------------------
// K3: box pyramid levels 1..nlev-1 of one or two images per stream (R39), all levels in one
// pass.  A CTA owns a 32 x 64 tile of level 1 (64 x 128 pixels of level 0; 16 x 32 of level
// 2, ... 2 x 4 of level 5).  Level 1: a thread averages 8 consecutive level-1 pixels from two
// 16-byte level-0 row loads on 16-bit lanes (exact: the 2x2 sum + 2 <= 1022 fits a lane), one
// 8-byte store; levels >= 2 from the previous level's tile in shared memory.  Partial chunks
// (frame edges, unaligned frames) take the per-pixel path -- the same integers.
// ---------------------------------------------------------------------------------------
struct PyrArgs {
    const uint8_t* img0[2];
    long long stride0[2];
    int pitch0[2];
    int dset[2];                   // destination set of image i (level L >= 1: [2][S][h_L][w_L])
    int vec[2];                    // level-0 rows 16-byte aligned (base and pitch)
    uint8_t* lev[kMaxLevels];
    int w[kMaxLevels], h[kMaxLevels];
    int nlev, S;
};

constexpr int kPyrTX = 64, kPyrTY = 32;   // level-1 tile

__device__ __forceinline__ uint32_t pyr_avg2(uint32_t a, uint32_t b) {
    // bytes (a0 a1 a2 a3) of row 2y, (b0 b1 b2 b3) of row 2y+1 -> level-1 pixels
    // (a0+a1+b0+b1+2)>>2 in byte 0 and (a2+a3+b2+b3+2)>>2 in byte 2
    const uint32_t e = (a & 0x00FF00FFu) + ((a >> 8) & 0x00FF00FFu) + (b & 0x00FF00FFu) + ((b >> 8) & 0x00FF00FFu) +
                       0x00020002u;
    return (e >> 2) & 0x00FF00FFu;
}

__global__ void __launch_bounds__(256) klt_pyramid_kernel(const PyrArgs a) {
    __shared__ __align__(16) uint8_t t1[kPyrTY][kPyrTX];
    __shared__ uint8_t t2[kPyrTY / 2][kPyrTX / 2];
    const int z = blockIdx.z, set = z / a.S, s = z - set * a.S;
    const long long zd = (long long)a.dset[set] * a.S + s;        // destination image index
    const uint8_t* src = a.img0[set] + (long long)s * a.stride0[set];
    const int p0 = a.pitch0[set];
    const int tid = threadIdx.x;
    {
        // level 1: thread = 8 consecutive pixels of one row of the tile
        const int ty = tid >> 3, tx = (tid & 7) * 8;
        const int y = blockIdx.y * kPyrTY + ty, x = blockIdx.x * kPyrTX + tx;
        const int w1 = a.w[1], h1 = a.h[1];
        uint32_t lo = 0, hi = 0;
        if (y < h1) {
            const uint8_t* r0 = src + (long long)(2 * y) * p0 + 2 * x;
            uint8_t* o = a.lev[1] + (zd * h1 + y) * w1 + x;
            if (a.vec[set] && x + 8 <= w1) {
                const uint4 u = __ldg(reinterpret_cast<const uint4*>(r0));
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(r0 + p0));
                lo = __byte_perm(pyr_avg2(u.x, v.x), pyr_avg2(u.y, v.y), 0x6420);
                hi = __byte_perm(pyr_avg2(u.z, v.z), pyr_avg2(u.w, v.w), 0x6420);
                if ((w1 & 7) == 0) {
                    *reinterpret_cast<uint2*>(o) = make_uint2(lo, hi);
                } else {
#pragma unroll
                    for (int k = 0; k < 8; ++k) o[k] = (uint8_t)((k < 4 ? lo : hi) >> (8 * (k & 3)));
                }
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (x + k < w1) {
                        const uint8_t* q = r0 + 2 * k;
                        const uint32_t v = ((uint32_t)q[0] + q[1] + q[p0] + q[p0 + 1] + 2u) >> 2;
                        o[k] = (uint8_t)v;
                        if (k < 4) lo |= v << (8 * k); else hi |= v << (8 * (k - 4));
                    }
                }
            }
        }
        *reinterpret_cast<uint2*>(&t1[ty][tx]) = make_uint2(lo, hi);
    }
    // levels >= 2 from the previous level's tile
    for (int L = 2; L < a.nlev; ++L) {
        __syncthreads();
        const int tw = kPyrTX >> (L - 1), th = kPyrTY >> (L - 1);
        const int wL = a.w[L], hL = a.h[L];
        for (int k = tid; k < tw * th; k += 256) {
            const int ty = k / tw, tx = k - ty * tw;
            uint32_t v;
            if (L & 1) {   // L = 3, 5: from t2 (level L-1)
                v = ((uint32_t)t2[2 * ty][2 * tx] + t2[2 * ty][2 * tx + 1] + t2[2 * ty + 1][2 * tx] +
                     t2[2 * ty + 1][2 * tx + 1] + 2u) >> 2;
            } else {       // L = 2, 4: from t1
                v = ((uint32_t)t1[2 * ty][2 * tx] + t1[2 * ty][2 * tx + 1] + t1[2 * ty + 1][2 * tx] +
                     t1[2 * ty + 1][2 * tx + 1] + 2u) >> 2;
            }
            const int x = blockIdx.x * tw + tx, y = blockIdx.y * th + ty;
            if (x < wL && y < hL) a.lev[L][(zd * hL + y) * wL + x] = (uint8_t)v;
            if (L & 1) t1[ty][tx] = (uint8_t)v;
            else t2[ty][tx] = (uint8_t)v;
        }
    }
}

// ---------------------------------------------------------------------------------------
// K4: pyramidal Lucas-Kanade, one warp per corner (R40)
// ---------------------------------------------------------------------------------------
struct Img {
    const uint8_t* p;
    long long stride;   // bytes between streams
    int pitch, w, h;
};

struct LkArgs {
    Img prev[kMaxLevels], next[kMaxLevels];
    int nlev, win, max_iters, max_corners;
    float eps2, min_eig;
    const int* corners;     // [S][max_corners][2]
    const int* counts;      // [S]
    float* tracked;         // [S][max_corners][2]
    uint8_t* status;        // [S][max_corners]
};

// bilinear value at continuous coordinates (pixel centres at +0.5), border pixels repeated
__device__ __forceinline__ float bil(const uint8_t* img, int pitch, int w, int h, float cx, float cy) {
    const float ux = __fsub_rn(cx, 0.5f), uy = __fsub_rn(cy, 0.5f);
    const float xf = floorf(ux), yf = floorf(uy);
    const float fx = __fsub_rn(ux, xf), fy = __fsub_rn(uy, yf);
    const int x0 = (int)xf, y0 = (int)yf;
    const int xa = clampi(x0, 0, w - 1), xb = clampi(x0 + 1, 0, w - 1);
    const int ya = clampi(y0, 0, h - 1), yb = clampi(y0 + 1, 0, h - 1);
    const uint8_t* ra = img + (long long)ya * pitch;
    const uint8_t* rb = img + (long long)yb * pitch;
    const float gx = __fsub_rn(1.0f, fx);
    const float top = __fadd_rn(__fmul_rn((float)__ldg(ra + xa), gx), __fmul_rn((float)__ldg(ra + xb), fx));
    const float bot = __fadd_rn(__fmul_rn((float)__ldg(rb + xa), gx), __fmul_rn((float)__ldg(rb + xb), fx));
    return __fadd_rn(__fmul_rn(top, __fsub_rn(1.0f, fy)), __fmul_rn(bot, fy));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Pixel (x, y) of a level image as a float, border pixels repeated (R40's bilinear rule).
__device__ __forceinline__ float pix_clamped(const uint8_t* img, int pitch, int w, int h, int x, int y) {
    return (float)__ldg(img + (long long)clampi(y, 0, h - 1) * pitch + clampi(x, 0, w - 1));
}

// One warp per corner (R40).  The window's samples s = p_L + (i - half, j - half) all share
// the fractional part of p_L (p_L = c / 2^L and the offsets are exact in fp32), so on
// prev the bilinear values of the (win+2)^2 integer-offset grid around the window are
// computed once per level into shared memory with common weights -- bitwise the values
// bil() gives at every sample and at its +-1 neighbours -- and I, Ix, Iy are read from it.
// On next, each iteration's samples s + g + v likewise share one fractional offset (the
// guess is added to the window's base point once), so a sample is 4 byte loads and the
// blend with common weights; windows wholly inside the level image skip the clamps.
constexpr int kLkWarps = 4;       // warps (corners) per CTA
constexpr int kLkMaxWin = 32;

#ifndef DMSGM_LK_MINB
#define DMSGM_LK_MINB 4
#endif
#ifndef DMSGM_LK_PAIRED
#define DMSGM_LK_PAIRED 1
#endif
constexpr int kLkMargin = 4;     // next-image region: the window +- this many pixels of flow per level
#ifndef DMSGM_LK_BATCH
#define DMSGM_LK_BATCH 8
#endif
constexpr int kLkBatch = DMSGM_LK_BATCH;   // staging rows per batch of loads

// NS = samples per lane: ceil(win^2 / 32); WIN = the window as a compile-time constant (the
// paper's Size(20,20): the window-geometry terms fold) or 0 (a.win at run time).  The staged
// next-image region holds (pixel, right neighbour) pairs, so a sample's 4 taps are two
// 8-byte shared loads.
template <int NS, int WIN = 0>
__global__ void __launch_bounds__(32 * kLkWarps, NS <= 13 ? DMSGM_LK_MINB : 1) klt_lk_kernel(const LkArgs a) {
    constexpr int MW = NS <= 8 ? 16 : (NS <= 13 ? 20 : kLkMaxWin);   // largest window of this variant
    constexpr bool STAGE = NS <= 13;       // (win > 20: the regions would exceed 48 KB; global reads)
    constexpr int MR = STAGE ? MW + 1 + 2 * kLkMargin : 1;             // next-region side
    __shared__ float patch_all[kLkWarps][(MW + 2) * (MW + 2)];
    __shared__ float2 region_all[kLkWarps][MR * MR];   // (v[y][x], v[y][x+1])
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * kLkWarps + (threadIdx.x >> 5);
    const int s = blockIdx.y;
    if (i >= a.max_corners) return;
    const long long o = (long long)s * a.max_corners + i;
    if (i >= a.counts[s]) {
        if (lane == 0) {
            a.status[o] = 0;
            a.tracked[2 * o] = __int_as_float(0x7fc00000);
            a.tracked[2 * o + 1] = __int_as_float(0x7fc00000);
        }
        return;
    }
    float* patch = patch_all[threadIdx.x >> 5];
    float2* region = region_all[threadIdx.x >> 5];
    const float cx = (float)a.corners[2 * o] + 0.5f, cy = (float)a.corners[2 * o + 1] + 0.5f;
    const int win = WIN ? WIN : a.win, nsamp = win * win, pw = win + 2, rs = win + 1 + 2 * kLkMargin;
    const float half = 0.5f * (float)(win - 1);
    // sample q = lane + 32 k of the window, (ii, jj) = (q % win, q / win): its offset in the
    // next-image region
    int roff[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        const int q = lane + 32 * k, jj = q / win;
        roff[k] = q < nsamp ? jj * rs + (q - jj * win) : 0;
    }
    float gx = 0.0f, gy = 0.0f;
    bool ok = true;
    for (int L = a.nlev - 1; L >= 0 && ok; --L) {
        const Img P = a.prev[L], Q = a.next[L];
        const uint8_t* pp = P.p + (long long)s * P.stride;
        const uint8_t* qp = Q.p + (long long)s * Q.stride;
        const float sc = __int_as_float((127 - L) << 23);        // 2^-L
        const float plx = __fmul_rn(cx, sc), ply = __fmul_rn(cy, sc);
        // window sample (ii, jj) sits at u = p_L - half - 0.5 + ii (+ the guess on next):
        // floor / fraction of the base point once (exact: p_L and the offsets are short)
        {
            const float ux = __fsub_rn(__fadd_rn(plx, __fsub_rn(0.0f, half)), 0.5f);
            const float uy = __fsub_rn(__fadd_rn(ply, __fsub_rn(0.0f, half)), 0.5f);
            const float xf = floorf(ux), yf = floorf(uy);
            const float fx = __fsub_rn(ux, xf), fy = __fsub_rn(uy, yf);
            const float gxw = __fsub_rn(1.0f, fx), gyw = __fsub_rn(1.0f, fy);
            const int X0 = (int)xf, Y0 = (int)yf;
            // patch[(jj + 1) * pw + (ii + 1)] = bil(prev, sample (ii, jj)), ii, jj in [-1, win]:
            // row by row, lane = column (pw <= 34 columns: lanes 0-31, then a second pass)
            __syncwarp();
            for (int c0 = 0; c0 < pw; c0 += 32) {
                const int ci = c0 + lane;                   // patch column
                if (ci < pw) {
                    const int x = X0 + ci - 1;
                    const int xa = clampi(x, 0, P.w - 1), xb = clampi(x + 1, 0, P.w - 1);
                    // row y's horizontal blend is row y+1's top: computed once per image row
                    const uint8_t* r0 = pp + (long long)clampi(Y0 - 1, 0, P.h - 1) * P.pitch;
                    float top = __fadd_rn(__fmul_rn((float)__ldg(r0 + xa), gxw), __fmul_rn((float)__ldg(r0 + xb), fx));
                    // rows in batches of kLkBatch: the batch's byte loads are all in flight before
                    // the first blend (one load round trip per batch, not per row)
                    for (int rj0 = 0; rj0 < pw; rj0 += kLkBatch) {
                        uint32_t va[kLkBatch], vb[kLkBatch];
#pragma unroll
                        for (int u = 0; u < kLkBatch; ++u) {
                            const uint8_t* rb = pp + (long long)clampi(Y0 + rj0 + u, 0, P.h - 1) * P.pitch;
                            va[u] = __ldg(rb + xa);
                            vb[u] = __ldg(rb + xb);
                        }
#pragma unroll
                        for (int u = 0; u < kLkBatch; ++u) {
                            if (rj0 + u < pw) {
                                const float bot = __fadd_rn(__fmul_rn((float)va[u], gxw), __fmul_rn((float)vb[u], fx));
                                patch[(rj0 + u) * pw + ci] = __fadd_rn(__fmul_rn(top, gyw), __fmul_rn(bot, fy));
                                top = bot;
                            }
                        }
                    }
                }
            }
            __syncwarp();
        }
        // the next-image region of this level: the window at the level's initial guess,
        // +- kLkMargin pixels, as floats in shared memory (clamped, R40's border rule); the
        // iterations read it while their window stays inside
        int RX0, RY0;
        {
            const float ux = __fsub_rn(__fadd_rn(__fadd_rn(plx, gx), __fsub_rn(0.0f, half)), 0.5f);
            const float uy = __fsub_rn(__fadd_rn(__fadd_rn(ply, gy), __fsub_rn(0.0f, half)), 0.5f);
            RX0 = STAGE ? (int)floorf(ux) - kLkMargin : INT_MIN / 2;      // INT_MIN / 2: never inside
            RY0 = (int)floorf(uy) - kLkMargin;
            __syncwarp();
            if (STAGE) {
                for (int c0 = 0; c0 < rs; c0 += 32) {
                    const int ci = c0 + lane;
                    if (ci < rs) {
                        const int xa = clampi(RX0 + ci, 0, Q.w - 1), xb = clampi(RX0 + ci + 1, 0, Q.w - 1);
                        for (int rj0 = 0; rj0 < rs; rj0 += kLkBatch) {
                            uint32_t v[kLkBatch], w[kLkBatch];
#pragma unroll
                            for (int u = 0; u < kLkBatch; ++u) {
                                const uint8_t* row = qp + (long long)clampi(RY0 + rj0 + u, 0, Q.h - 1) * Q.pitch;
                                v[u] = __ldg(row + xa);
                                w[u] = __ldg(row + xb);
                            }
#pragma unroll
                            for (int u = 0; u < kLkBatch; ++u)
                                if (rj0 + u < rs) region[(rj0 + u) * rs + ci] = make_float2((float)v[u], (float)w[u]);
                        }
                    }
                }
            }
            __syncwarp();
        }
        float I[NS], Ix[NS], Iy[NS];
        float gxx = 0.0f, gxy = 0.0f, gyy = 0.0f;
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            I[k] = Ix[k] = Iy[k] = 0.0f;
            if (lane + 32 * k < nsamp) {
                const int q = lane + 32 * k, jj = q / win;
                const float* c0 = patch + (jj + 1) * pw + (q - jj * win) + 1;
                I[k] = c0[0];
                Ix[k] = __fmul_rn(__fsub_rn(c0[1], c0[-1]), 0.5f);
                Iy[k] = __fmul_rn(__fsub_rn(c0[pw], c0[-pw]), 0.5f);
                gxx = __fadd_rn(gxx, __fmul_rn(Ix[k], Ix[k]));
                gxy = __fadd_rn(gxy, __fmul_rn(Ix[k], Iy[k]));
                gyy = __fadd_rn(gyy, __fmul_rn(Iy[k], Iy[k]));
            }
        }
        gxx = warp_sum(gxx);
        gxy = warp_sum(gxy);
        gyy = warp_sum(gyy);
        const float dd = __fsub_rn(gxx, gyy);
        const float lam = __fmul_rn(__fsub_rn(__fadd_rn(gxx, gyy),
                                              __fsqrt_rn(__fadd_rn(__fmul_rn(dd, dd), __fmul_rn(4.0f, __fmul_rn(gxy, gxy))))),
                                    0.5f);
        const float det = __fsub_rn(__fmul_rn(gxx, gyy), __fmul_rn(gxy, gxy));
        float vx = 0.0f, vy = 0.0f;
        const float rdet = __frcp_rn(det);
        if (__fdiv_rn(lam, (float)nsamp) < a.min_eig || !(det > 0.0f)) {
            if (L == 0) { ok = false; break; }
            gx = __fmul_rn(2.0f, gx);                    // a coarse level without texture: skipped
            gy = __fmul_rn(2.0f, gy);
            continue;
        }
        for (int it = 0; it < a.max_iters; ++it) {
            float bx = 0.0f, by = 0.0f;
            const float ox = __fadd_rn(gx, vx), oy = __fadd_rn(gy, vy);
            // the iteration's window on next: base point, its floor and common fraction
            const float ux = __fsub_rn(__fadd_rn(__fadd_rn(plx, ox), __fsub_rn(0.0f, half)), 0.5f);
            const float uy = __fsub_rn(__fadd_rn(__fadd_rn(ply, oy), __fsub_rn(0.0f, half)), 0.5f);
            const float xf = floorf(ux), yf = floorf(uy);
            const float fx = __fsub_rn(ux, xf), fy = __fsub_rn(uy, yf);
            const float gxw = __fsub_rn(1.0f, fx), gyw = __fsub_rn(1.0f, fy);
            const int X0 = (int)xf, Y0 = (int)yf;
            const int dxr = X0 - RX0, dyr = Y0 - RY0;
            if ((unsigned)dxr <= 2u * kLkMargin && (unsigned)dyr <= 2u * kLkMargin) {
                // the window (and its +1 neighbours) inside the staged region; branch-free: a
                // lane's padding samples (q >= win^2) read offset 0 and have I = Ix = Iy = 0, so
                // they add exactly +0 to both sums
                const float2* base = region + dyr * rs + dxr;
#if DMSGM_LK_PAIRED
                // two samples per paired instruction (FFMA2 / FMUL2 / FADD2), the blend and
                // the sums as fmas: ~4.5 FP instructions per sample instead of 12 (LK is
                // compared with the oracle within a tolerance, not bitwise)
                const float2 GXW = f2_bc(gxw), FX = f2_bc(fx), GYW = f2_bc(gyw), FY = f2_bc(fy);
                float2 bx2 = f2_bc(0.0f), by2 = f2_bc(0.0f);
#pragma unroll
                for (int k = 0; k + 1 < NS; k += 2) {
                    const float2* ra = base + roff[k];
                    const float2* rb = base + roff[k + 1];
                    const float2 ta = ra[0], tb = rb[0], ua = ra[rs], ub = rb[rs];   // (left, right) taps
                    const float2 p00 = make_float2(ta.x, tb.x), p10 = make_float2(ta.y, tb.y);
                    const float2 p01 = make_float2(ua.x, ub.x), p11 = make_float2(ua.y, ub.y);
                    const float2 top = f2_fma(p00, GXW, f2_mul(p10, FX));
                    const float2 bot = f2_fma(p01, GXW, f2_mul(p11, FX));
                    const float2 e = f2_sub(make_float2(I[k], I[k + 1]), f2_fma(top, GYW, f2_mul(bot, FY)));
                    bx2 = f2_fma(e, make_float2(Ix[k], Ix[k + 1]), bx2);
                    by2 = f2_fma(e, make_float2(Iy[k], Iy[k + 1]), by2);
                }
                bx = __fadd_rn(bx2.x, bx2.y);
                by = __fadd_rn(by2.x, by2.y);
                if constexpr (NS & 1) {
                    const float2* r0 = base + roff[NS - 1];
                    const float2 t0 = r0[0], u0 = r0[rs];
                    const float top = __fmaf_rn(t0.x, gxw, __fmul_rn(t0.y, fx));
                    const float bot = __fmaf_rn(u0.x, gxw, __fmul_rn(u0.y, fx));
                    const float e = __fsub_rn(I[NS - 1], __fmaf_rn(top, gyw, __fmul_rn(bot, fy)));
                    bx = __fmaf_rn(e, Ix[NS - 1], bx);
                    by = __fmaf_rn(e, Iy[NS - 1], by);
                }
#else
#pragma unroll
                for (int k = 0; k < NS; ++k) {
                    const float2* r0 = base + roff[k];
                    const float p00 = r0[0].x, p10 = r0[0].y, p01 = r0[rs].x, p11 = r0[rs].y;
                    const float top = __fadd_rn(__fmul_rn(p00, gxw), __fmul_rn(p10, fx));
                    const float bot = __fadd_rn(__fmul_rn(p01, gxw), __fmul_rn(p11, fx));
                    const float e = __fsub_rn(I[k], __fadd_rn(__fmul_rn(top, gyw), __fmul_rn(bot, fy)));
                    bx = __fadd_rn(bx, __fmul_rn(e, Ix[k]));
                    by = __fadd_rn(by, __fmul_rn(e, Iy[k]));
                }
#endif
            } else {
#pragma unroll
                for (int k = 0; k < NS; ++k) {
                    if (lane + 32 * k < nsamp) {
                        const int q = lane + 32 * k, jj = q / win;
                        const int x = X0 + (q - jj * win), y = Y0 + jj;
                        const float top = __fadd_rn(__fmul_rn(pix_clamped(qp, Q.pitch, Q.w, Q.h, x, y), gxw),
                                                    __fmul_rn(pix_clamped(qp, Q.pitch, Q.w, Q.h, x + 1, y), fx));
                        const float bot = __fadd_rn(__fmul_rn(pix_clamped(qp, Q.pitch, Q.w, Q.h, x, y + 1), gxw),
                                                    __fmul_rn(pix_clamped(qp, Q.pitch, Q.w, Q.h, x + 1, y + 1), fx));
                        const float e = __fsub_rn(I[k], __fadd_rn(__fmul_rn(top, gyw), __fmul_rn(bot, fy)));
                        bx = __fadd_rn(bx, __fmul_rn(e, Ix[k]));
                        by = __fadd_rn(by, __fmul_rn(e, Iy[k]));
                    }
                }
            }
            bx = warp_sum(bx);
            by = warp_sum(by);
            // G^-1 b with the level's 1/det (one correctly rounded reciprocal per level instead
            // of two IEEE divisions per iteration; LK is compared within a tolerance, R40)
            const float dx = __fmul_rn(__fsub_rn(__fmul_rn(gyy, bx), __fmul_rn(gxy, by)), rdet);
            const float dy = __fmul_rn(__fsub_rn(__fmul_rn(gxx, by), __fmul_rn(gxy, bx)), rdet);
            vx = __fadd_rn(vx, dx);
            vy = __fadd_rn(vy, dy);
            if (L == 0) {
                const float qx = __fadd_rn(plx, __fadd_rn(gx, vx)), qy = __fadd_rn(ply, __fadd_rn(gy, vy));
                if (!(qx >= 0.0f && qx < (float)P.w && qy >= 0.0f && qy < (float)P.h)) { ok = false; break; }
            }
            if (__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)) < a.eps2) break;
        }
        if (!ok) break;
        if (L > 0) {
            gx = __fmul_rn(2.0f, __fadd_rn(gx, vx));
            gy = __fmul_rn(2.0f, __fadd_rn(gy, vy));
        } else {
            gx = __fadd_rn(gx, vx);
            gy = __fadd_rn(gy, vy);
        }
    }
    if (lane == 0) {
        a.status[o] = ok ? 1 : 0;
        a.tracked[2 * o] = ok ? __fadd_rn(cx, gx) : __int_as_float(0x7fc00000);
        a.tracked[2 * o + 1] = ok ? __fadd_rn(cy, gy) : __int_as_float(0x7fc00000);
    }
}

// ---------------------------------------------------------------------------------------
// K5: tracked pairs -> matches (src = frame-t point, dst = frame-(t-1) corner centre)
// ---------------------------------------------------------------------------------------
struct CompactArgs {
    const int* corners;
    const int* counts;
    const float* tracked;
    const uint8_t* status;
    int max_corners, S;
    double* src;    // [S][max_corners][2]
    double* dst;
    int* mcount;    // [S]
};

__global__ void klt_compact_kernel(const CompactArgs a) {
    const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (s >= a.S) return;
    const int cnt = a.counts[s];
    int n = 0;
    for (int b = 0; b < cnt; b += 32) {
        const int i = b + lane;
        const long long o = (long long)s * a.max_corners + i;
        const bool st = i < cnt && a.status[o];
        const unsigned bal = __ballot_sync(0xffffffffu, st);
        if (st) {
            const long long w = (long long)s * a.max_corners + n + __popc(bal & ((1u << lane) - 1u));
            a.src[2 * w] = (double)a.tracked[2 * o];
            a.src[2 * w + 1] = (double)a.tracked[2 * o + 1];
            a.dst[2 * w] = (double)a.corners[2 * o] + 0.5;
            a.dst[2 * w + 1] = (double)a.corners[2 * o + 1] + 0.5;
        }
        n += __popc(bal);
    }
    if (lane == 0) a.mcount[s] = n;
}

// ---------------------------------------------------------------------------------------
// K6: RANSAC hypotheses (R42), one warp per (stream, 4 iterations)
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ bool ransac_sample(unsigned long long seed, int it, int n, int (&idx)[4]) {
    int got = 0;
    for (int k = 0; k < 64 && got < 4; ++k) {
        const unsigned long long z = splitmix64((seed << 32) + (unsigned long long)it * 64ull + (unsigned long long)k);
        const int i = (int)(((z >> 32) * (unsigned long long)n) >> 32);
        bool dup = false;
        for (int j = 0; j < got; ++j) dup |= idx[j] == i;
        if (!dup) idx[got++] = i;
    }
    return got == 4;
}

__device__ __forceinline__ bool collinear4(const double (&px)[4], const double (&py)[4]) {
    double xmin = px[0], xmax = px[0], ymin = py[0], ymax = py[0];
    for (int k = 1; k < 4; ++k) {
        xmin = fmin(xmin, px[k]); xmax = fmax(xmax, px[k]);
        ymin = fmin(ymin, py[k]); ymax = fmax(ymax, py[k]);
    }
    const double ext = fmax(fmax(__dsub_rn(xmax, xmin), __dsub_rn(ymax, ymin)), 1e-12);
    const double lim = __dmul_rn(__dmul_rn(1e-6, ext), ext);
    for (int p = 0; p < 4; ++p)
        for (int q = p + 1; q < 4; ++q)
            for (int r = q + 1; r < 4; ++r) {
                const double ux = __dsub_rn(px[q], px[p]), uy = __dsub_rn(py[q], py[p]);
                const double vx = __dsub_rn(px[r], px[p]), vy = __dsub_rn(py[r], py[p]);
                if (fabs(__dsub_rn(__dmul_rn(ux, vy), __dmul_rn(uy, vx))) <= lim) return true;
            }
    return false;
}

// The homography (h8 = 1) through 4 correspondences: 8x8 system, Gaussian elimination with
// partial pivoting in fp64.  false for a degenerate sample.
__device__ bool minimal_h(const double (&x)[4], const double (&y)[4], const double (&u)[4], const double (&v)[4],
                          double (&h)[9]) {
    if (collinear4(x, y) || collinear4(u, v)) return false;
    double A[8][9];
    for (int i = 0; i < 4; ++i) {
        double* r0 = A[2 * i];
        double* r1 = A[2 * i + 1];
        r0[0] = x[i]; r0[1] = y[i]; r0[2] = 1.0; r0[3] = 0.0; r0[4] = 0.0; r0[5] = 0.0;
        r0[6] = -__dmul_rn(u[i], x[i]); r0[7] = -__dmul_rn(u[i], y[i]); r0[8] = u[i];
        r1[0] = 0.0; r1[1] = 0.0; r1[2] = 0.0; r1[3] = x[i]; r1[4] = y[i]; r1[5] = 1.0;
        r1[6] = -__dmul_rn(v[i], x[i]); r1[7] = -__dmul_rn(v[i], y[i]); r1[8] = v[i];
    }
    for (int c = 0; c < 8; ++c) {
        int piv = c;
        double best = fabs(A[c][c]);
        for (int r = c + 1; r < 8; ++r)
            if (fabs(A[r][c]) > best) { best = fabs(A[r][c]); piv = r; }
        if (!(best > 0.0)) return false;
        if (piv != c)
            for (int k = 0; k < 9; ++k) { const double t = A[c][k]; A[c][k] = A[piv][k]; A[piv][k] = t; }
        for (int r = c + 1; r < 8; ++r) {
            const double f = __ddiv_rn(A[r][c], A[c][c]);
            for (int k = c + 1; k < 9; ++k) A[r][k] = __dsub_rn(A[r][k], __dmul_rn(f, A[c][k]));
        }
    }
    for (int r = 7; r >= 0; --r) {
        double acc = A[r][8];
        for (int k = r + 1; k < 8; ++k) acc = __dsub_rn(acc, __dmul_rn(A[r][k], h[k]));
        h[r] = __ddiv_rn(acc, A[r][r]);
    }
    h[8] = 1.0;
    return true;
}

__device__ __forceinline__ double reproj_err2(const double (&h)[9], double x, double y, double u, double v) {
    const double w = __dadd_rn(__dadd_rn(__dmul_rn(h[6], x), __dmul_rn(h[7], y)), h[8]);
    const double px = __ddiv_rn(__dadd_rn(__dadd_rn(__dmul_rn(h[0], x), __dmul_rn(h[1], y)), h[2]), w);
    const double py = __ddiv_rn(__dadd_rn(__dadd_rn(__dmul_rn(h[3], x), __dmul_rn(h[4], y)), h[5]), w);
    const double ex = __dsub_rn(px, u), ey = __dsub_rn(py, v);
    return __dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey));
}

struct RansacArgs {
    const double* src;    // [S][max_corners][2]
    const double* dst;
    const int* mcount;    // [S]
    int max_corners, iters;
    unsigned long long seed;
    double thresh2;
    int* iter_counts;     // [S][iters]
};

// One warp per 4 iterations: lanes 8g .. 8g+7 hold the 8 rows of iteration 4w+g's 8x8
// system (row r: its 9 coefficients), so the elimination runs row-parallel -- per column the
// pivot by a 3-step (value, lower row) max within the 8 lanes, the row swap and the pivot
// row by shuffles, each row's f = A[r][c] / A[c][c] and update on its own lane -- with
// exactly minimal_h's operations on every entry (the same pivots, quotients, products and
// differences in the same order: the same h, bit for bit).  Then each group counts its
// hypothesis' inliers over the matches (8 lanes).  Replaces one warp per iteration in which
// all 32 lanes repeated one serial solve (~70 % of its instructions).
constexpr int kRansacWarps = 4;
constexpr int kRansacPerWarp = 4;

__device__ __forceinline__ double shfl_d(double v, int src) {
    return __hiloint2double(__shfl_sync(0xffffffffu, __double2hiint(v), src),
                            __shfl_sync(0xffffffffu, __double2loint(v), src));
}
__device__ __forceinline__ double shfl_xor_d(double v, int m) {
    return __hiloint2double(__shfl_xor_sync(0xffffffffu, __double2hiint(v), m),
                            __shfl_xor_sync(0xffffffffu, __double2loint(v), m));
}

__global__ void __launch_bounds__(32 * kRansacWarps) klt_ransac_kernel(const RansacArgs a) {
    const int w = blockIdx.x * kRansacWarps + (threadIdx.x >> 5), lane = threadIdx.x & 31, s = blockIdx.y;
    if (w * kRansacPerWarp >= a.iters) return;                     // warp-uniform
    const int g = lane >> 3, r = lane & 7, base = lane & ~7;       // group (iteration) and row
    const int it = w * kRansacPerWarp + g;
    const int n = a.mcount[s];
    const double* src = a.src + (long long)s * a.max_corners * 2;
    const double* dst = a.dst + (long long)s * a.max_corners * 2;
    int idx[4];
    bool ok = it < a.iters && n >= 4 && ransac_sample(a.seed, it, n, idx);
    double xs = 0.0, ys = 0.0, us = 0.0, vs = 0.0;                  // this row's correspondence
    if (ok) {
        double x[4], y[4], u[4], v[4];
        for (int k = 0; k < 4; ++k) {
            x[k] = src[2 * idx[k]]; y[k] = src[2 * idx[k] + 1];
            u[k] = dst[2 * idx[k]]; v[k] = dst[2 * idx[k] + 1];
        }
        ok = !collinear4(x, y) && !collinear4(u, v);
        const int i = r >> 1;
        xs = i == 0 ? x[0] : i == 1 ? x[1] : i == 2 ? x[2] : x[3];
        ys = i == 0 ? y[0] : i == 1 ? y[1] : i == 2 ? y[2] : y[3];
        us = i == 0 ? u[0] : i == 1 ? u[1] : i == 2 ? u[2] : u[3];
        vs = i == 0 ? v[0] : i == 1 ? v[1] : i == 2 ? v[2] : v[3];
    }
    // row r of minimal_h's system: even r = 2i: (x, y, 1, 0, 0, 0, -u x, -u y, u);
    // odd r = 2i+1: (0, 0, 0, x, y, 1, -v x, -v y, v)
    const bool odd = r & 1;
    const double t = odd ? vs : us;
    double A[9];
    A[0] = odd ? 0.0 : xs; A[1] = odd ? 0.0 : ys; A[2] = odd ? 0.0 : 1.0;
    A[3] = odd ? xs : 0.0; A[4] = odd ? ys : 0.0; A[5] = odd ? 1.0 : 0.0;
    A[6] = -__dmul_rn(t, xs); A[7] = -__dmul_rn(t, ys); A[8] = t;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        // pivot: the first row >= c of the largest |A[r][c]| (minimal_h's strict '>' scan from
        // row c: a NaN row below c never wins; a NaN at row c fails the sample)
        const double av = fabs(A[c]);
        const bool nan_c = __shfl_sync(0xffffffffu, (int)(av != av), base + c) != 0;
        double kv = r < c ? -2.0 : (r == c ? av : (av != av ? -1.0 : av));
        int kr = r;
#pragma unroll
        for (int m = 1; m < 8; m <<= 1) {
            const double ov = shfl_xor_d(kv, m);
            const int orow = __shfl_xor_sync(0xffffffffu, kr, m);
            if (ov > kv || (ov == kv && orow < kr)) { kv = ov; kr = orow; }
        }
        ok = ok && !nan_c && kv > 0.0;
        const int piv = kr;
        // swap rows c and piv (columns c .. 8; the columns left of c are never read again)
        const int from = r == c ? piv : (r == piv ? c : r);
#pragma unroll
        for (int k = c; k < 9; ++k) A[k] = shfl_d(A[k], base + from);
        // eliminate below the pivot row
        double P[9];
#pragma unroll
        for (int k = c; k < 9; ++k) P[k] = shfl_d(A[k], base + c);
        if (r > c) {
            const double f = __ddiv_rn(A[c], P[c]);
#pragma unroll
            for (int k = c + 1; k < 9; ++k) A[k] = __dsub_rn(A[k], __dmul_rn(f, P[k]));
        }
    }
    // back substitution, h[8] = 1: row r on lane r, h broadcast as it is found
    double h[9];
    h[8] = 1.0;
#pragma unroll
    for (int rr = 7; rr >= 0; --rr) {
        double acc = A[8];
#pragma unroll
        for (int k = rr + 1; k < 8; ++k) acc = __dsub_rn(acc, __dmul_rn(A[k], h[k]));
        h[rr] = shfl_d(__ddiv_rn(acc, A[rr]), base + rr);
    }
    // inliers of this group's hypothesis over the matches, 8 lanes
    int cnt = 0;
    if (ok)
        for (int j = r; j < n; j += 8)
            cnt += reproj_err2(h, src[2 * j], src[2 * j + 1], dst[2 * j], dst[2 * j + 1]) < a.thresh2;
#pragma unroll
    for (int m = 4; m > 0; m >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, m);
    if (r == 0 && it < a.iters) a.iter_counts[(long long)s * a.iters + it] = ok ? cnt : -1;
}

// ---------------------------------------------------------------------------------------
// K7: best model -> inliers -> normalized DLT (R41), one warp per stream
// ---------------------------------------------------------------------------------------
struct RefitArgs {
    const double* src;
    const double* dst;
    const int* mcount;
    const int* iter_counts;
    int max_corners, iters, S;
    unsigned long long seed;
    double thresh2;
    double* H_out;          // [S][9]
    uint8_t* inliers;       // [S][max_corners] (may be null)
    int* ok_out;            // [S] (may be null)
};

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Smallest-eigenvalue eigenvector of the symmetric positive semi-definite 9x9 A^T A (the
// right singular vector of A's smallest singular value, R41) by inverse iteration in fp64
// on A^T A + delta I, delta = 1e-10 trace (positive definite whatever the roundoff; the
// eigenvectors are A^T A's): Cholesky factor L, then 6 iterations x <- (L L^T)^-1 x / |.|
// from the all-ones vector.  Per iteration the error shrinks by (l1 + delta) / (l2 + delta),
// ~1e-3 or less for a normalised DLT with noise: 6 iterations reach fp64 roundoff.  One
// lane, L in shared memory: ~5 k cycles, where Jacobi rotations (a dependent chain of
// divisions and square roots per rotation) took ~40 us of the kernel's 93 us.
__device__ void min_eigvec9_inv(const double* m, double* L, double* out) {
    double tr = 0.0;
#pragma unroll
    for (int i = 0; i < 9; ++i) tr += m[i * 9 + i];
    const double delta = 1e-10 * tr;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        double d = m[j * 9 + j] + delta;
#pragma unroll
        for (int k = 0; k < j; ++k) d -= L[j * 9 + k] * L[j * 9 + k];
        d = sqrt(d > 0.0 ? d : delta);
        L[j * 9 + j] = d;
        const double rd = 1.0 / d;
#pragma unroll
        for (int i = j + 1; i < 9; ++i) {
            double t = m[i * 9 + j];
#pragma unroll
            for (int k = 0; k < j; ++k) t -= L[i * 9 + k] * L[j * 9 + k];
            L[i * 9 + j] = t * rd;
        }
    }
    double rdiag[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) rdiag[i] = 1.0 / L[i * 9 + i];
    double x[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) x[i] = 1.0;
    for (int it = 0; it < 6; ++it) {
        double y[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) {                // L y = x
            double t = x[i];
#pragma unroll
            for (int k = 0; k < i; ++k) t -= L[i * 9 + k] * y[k];
            y[i] = t * rdiag[i];
        }
#pragma unroll
        for (int i = 8; i >= 0; --i) {               // L^T x = y
            double t = y[i];
#pragma unroll
            for (int k = i + 1; k < 9; ++k) t -= L[k * 9 + i] * x[k];
            x[i] = t * rdiag[i];
        }
        double n2 = 0.0;
#pragma unroll
        for (int i = 0; i < 9; ++i) n2 += x[i] * x[i];
        const double rn = 1.0 / sqrt(n2);
#pragma unroll
        for (int i = 0; i < 9; ++i) x[i] *= rn;
    }
#pragma unroll
    for (int i = 0; i < 9; ++i) out[i] = x[i];
}

__global__ void klt_refit_kernel(const RefitArgs a) {
    __shared__ double sm_m[4][81], sm_l[4][81], sm_e[4][9];
    const int w = threadIdx.x >> 5;
    const int s = blockIdx.x * (blockDim.x >> 5) + w, lane = threadIdx.x & 31;
    if (s >= a.S) return;
    const int n = a.mcount[s];
    const double* src = a.src + (long long)s * a.max_corners * 2;
    const double* dst = a.dst + (long long)s * a.max_corners * 2;
    double* Ho = a.H_out + 9 * (long long)s;
    // best iteration: most inliers, ties to the earliest
    int best = -1, bit = -1;
    for (int j = lane; j < a.iters; j += 32) {
        const int c = a.iter_counts[(long long)s * a.iters + j];
        if (c > best) { best = c; bit = j; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const int ob = __shfl_xor_sync(0xffffffffu, best, o), oi = __shfl_xor_sync(0xffffffffu, bit, o);
        if (ob > best || (ob == best && oi < bit && oi >= 0)) { best = ob; bit = oi; }
    }
    bool okm = best >= 4 && n >= 4;
    double h[9];
    if (okm) {
        int idx[4];
        double x[4], y[4], u[4], v[4];
        ransac_sample(a.seed, bit, n, idx);
        for (int k = 0; k < 4; ++k) {
            x[k] = src[2 * idx[k]]; y[k] = src[2 * idx[k] + 1];
            u[k] = dst[2 * idx[k]]; v[k] = dst[2 * idx[k] + 1];
        }
        okm = minimal_h(x, y, u, v, h);
    }
    if (!okm) {
        if (lane < 9) Ho[lane] = (lane % 4 == 0) ? 1.0 : 0.0;
        for (int j = lane; j < n && a.inliers; j += 32) a.inliers[(long long)s * a.max_corners + j] = 0;
        if (lane == 0 && a.ok_out) a.ok_out[s] = 0;
        return;
    }
    // inliers of the best model; Hartley normalisation of both sets over them
    // (the inlier test once: bit k of inm is match lane + 32 k; n <= kMaxCorners = 1024)
    double sx = 0, sy = 0, su = 0, sv = 0, cnt = 0;
    uint32_t inm = 0;
    for (int j = lane, k = 0; j < n; j += 32, ++k) {
        const bool in = reproj_err2(h, src[2 * j], src[2 * j + 1], dst[2 * j], dst[2 * j + 1]) < a.thresh2;
        if (a.inliers) a.inliers[(long long)s * a.max_corners + j] = in;
        inm |= (uint32_t)in << k;
        if (in) { sx += src[2 * j]; sy += src[2 * j + 1]; su += dst[2 * j]; sv += dst[2 * j + 1]; cnt += 1.0; }
    }
    cnt = warp_sum_d(cnt);
    const double mx = warp_sum_d(sx) / cnt, my = warp_sum_d(sy) / cnt;
    const double mu = warp_sum_d(su) / cnt, mv = warp_sum_d(sv) / cnt;
    double ds = 0, dd = 0;
    for (int j = lane, k = 0; j < n; j += 32, ++k) {
        if (inm >> k & 1u) {
            ds += sqrt((src[2 * j] - mx) * (src[2 * j] - mx) + (src[2 * j + 1] - my) * (src[2 * j + 1] - my));
            dd += sqrt((dst[2 * j] - mu) * (dst[2 * j] - mu) + (dst[2 * j + 1] - mv) * (dst[2 * j + 1] - mv));
        }
    }
    ds = warp_sum_d(ds) / cnt;
    dd = warp_sum_d(dd) / cnt;
    const double ks = ds > 0 ? sqrt(2.0) / ds : 1.0, kd = dd > 0 ? sqrt(2.0) / dd : 1.0;
    // A^T A of the normalized system, 45 distinct entries per lane, then the warp sum
    double M[45];
#pragma unroll
    for (int k = 0; k < 45; ++k) M[k] = 0.0;
    for (int j = lane, kb = 0; j < n; j += 32, ++kb) {
        if (!(inm >> kb & 1u)) continue;
        const double X = ks * (src[2 * j] - mx), Y = ks * (src[2 * j + 1] - my);
        const double U = kd * (dst[2 * j] - mu), Vv = kd * (dst[2 * j + 1] - mv);
        const double r1[9] = {0, 0, 0, -X, -Y, -1, Vv * X, Vv * Y, Vv};
        const double r2[9] = {X, Y, 1, 0, 0, 0, -U * X, -U * Y, -U};
        int k = 0;
#pragma unroll
        for (int p = 0; p < 9; ++p)
#pragma unroll
            for (int q = p; q < 9; ++q) M[k++] += r1[p] * r1[q] + r2[p] * r2[q];
    }
#pragma unroll
    for (int k = 0; k < 45; ++k) M[k] = warp_sum_d(M[k]);
    double* m = sm_m[w];
    if (lane == 0) {
        int k = 0;
        for (int p = 0; p < 9; ++p)
            for (int q = p; q < 9; ++q) { m[p * 9 + q] = M[k]; m[q * 9 + p] = M[k]; ++k; }
    }
    __syncwarp();
    if (lane == 0) min_eigvec9_inv(m, sm_l[w], sm_e[w]);
    __syncwarp();
    if (lane == 0) {
        const double* e = sm_e[w];
        // H = Td^-1 Hn Ts, Ts = [[ks,0,-ks mx],[0,ks,-ks my],[0,0,1]], Td^-1 = [[1/kd,0,mu],[0,1/kd,mv],[0,0,1]]
        double T[9];   // Hn Ts
        for (int r = 0; r < 3; ++r) {
            T[3 * r + 0] = e[3 * r + 0] * ks;
            T[3 * r + 1] = e[3 * r + 1] * ks;
            T[3 * r + 2] = -e[3 * r + 0] * ks * mx - e[3 * r + 1] * ks * my + e[3 * r + 2];
        }
        double R[9];
        for (int c = 0; c < 3; ++c) {
            R[0 + c] = T[0 + c] / kd + mu * T[6 + c];
            R[3 + c] = T[3 + c] / kd + mv * T[6 + c];
            R[6 + c] = T[6 + c];
        }
        const double z = R[8];
        for (int q = 0; q < 9; ++q) Ho[q] = R[q] / z;
        if (a.ok_out) a.ok_out[s] = (int)cnt;
    }
}

}  // namespace dmsgm_klt
