/*
 * warp_oracle.c -- TEST INFRASTRUCTURE ONLY (part of the oracle library).
 *
 * Frame-warp motion compensation, the paper's own MC variant:
 * App. F P:691-692 estimates H from the previous to the current frame and calls
 * warpPerspective(next, n, H, size, INTER_LINEAR | WARP_INVERSE_MAP), i.e. every pixel
 * of the output (previous frame's coordinates) samples the current frame at H p;
 * §3.1.3 "we transform the current frame to match the previous frame".  The models are
 * then updated without warping (readings R35-R37):
 *
 *   R35 direction: our homography H_t maps frame-t coordinates to frame-(t-1) ones (R3),
 *       so App. F's H is H_t^-1: out(x, y) samples frame t at H_t^-1 (x + 1/2, y + 1/2)
 *       (pixel centres, R2).  H_t^-1 is the adjugate of H_t (the projective scale
 *       cancels), normalised so its last entry is 1 (fp64).
 *   R36 arithmetic: like R17, the displacement form in fp32 with g = A - I rounded once:
 *       X = x + 1/2, Y = y + 1/2, e = fma(g6, X, fma(g7, Y, g8)), w = 1 + e,
 *       px = fma(-X, e, fma(g0, X, fma(g1, Y, g2))), py = fma(-Y, e, fma(g3, X, fma(g4, Y, g5))),
 *       r = 1/w, sx = x + px r, sy = y + py r (the sample position in pixel-index space).
 *       A degenerate map (w <= 0, a displacement of 2^20 pixels or more, NaN, or a zero
 *       normalising entry) leaves the pixel unchanged.
 *   R37 sampling: bilinear with the nearest border pixel outside the frame:
 *       x0 = floor(sx), fx = sx - x0 (exact), taps at clamp(x0), clamp(x0 + 1) (same for
 *       y); top = fma(fx, p10 - p00, p00), bottom = fma(fx, p11 - p01, p01),
 *       v = fma(fy, bottom - top, top) in fp32, rounded to nearest (ties to even).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "dmsgm_oracle.h"

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* R35: A = adj(H) / adj(H)[8]; returns 0 when the normalising entry is zero. */
static int inverse_normalised(const double* h, double* a) {
    a[0] = h[4] * h[8] - h[5] * h[7];
    a[1] = h[2] * h[7] - h[1] * h[8];
    a[2] = h[1] * h[5] - h[2] * h[4];
    a[3] = h[5] * h[6] - h[3] * h[8];
    a[4] = h[0] * h[8] - h[2] * h[6];
    a[5] = h[2] * h[3] - h[0] * h[5];
    a[6] = h[3] * h[7] - h[4] * h[6];
    a[7] = h[1] * h[6] - h[0] * h[7];
    a[8] = h[0] * h[4] - h[1] * h[3];
    if (!(a[8] != 0.0) || !isfinite(a[8])) return 0;
    for (int i = 0; i < 9; ++i) a[i] /= a[8];
    return 1;
}

int dmsgm_oracle_warp_frame(int width, int height, const uint8_t* in, size_t in_pitch, const double* h,
                            uint8_t* out, size_t out_pitch) {
    if (!in || !out || !h || width < 1 || height < 1 || in_pitch < (size_t)width || out_pitch < (size_t)width)
        return -1;
    double a[9];
    const int ok = inverse_normalised(h, a);
    float g[9];
    for (int i = 0; i < 9; ++i) g[i] = (float)((i == 0 || i == 4 || i == 8) ? a[i] - 1.0 : a[i]);
    for (int y = 0; y < height; ++y)
        for (int x = 0; x < width; ++x) {
            const uint8_t self = in[(size_t)y * in_pitch + x];
            if (!ok) {
                out[(size_t)y * out_pitch + x] = self;
                continue;
            }
            /* R36 */
            const float X = (float)x + 0.5f, Y = (float)y + 0.5f;
            const float e = fmaf(g[6], X, fmaf(g[7], Y, g[8]));
            const float w = 1.0f + e;
            const float px = fmaf(-X, e, fmaf(g[0], X, fmaf(g[1], Y, g[2])));
            const float py = fmaf(-Y, e, fmaf(g[3], X, fmaf(g[4], Y, g[5])));
            const float r = 1.0f / w;
            const float dx = px * r, dy = py * r;
            if (!(w > 0.0f) || !(fabsf(dx) < 1048576.0f && fabsf(dy) < 1048576.0f)) {
                out[(size_t)y * out_pitch + x] = self;
                continue;
            }
            const float sx = (float)x + dx, sy = (float)y + dy;
            /* R37 */
            const float flx = floorf(sx), fly = floorf(sy);
            const float fx = sx - flx, fy = sy - fly;
            const int ix = (int)flx, iy = (int)fly;
            const int x0 = clampi(ix, 0, width - 1), x1 = clampi(ix + 1, 0, width - 1);
            const int y0 = clampi(iy, 0, height - 1), y1 = clampi(iy + 1, 0, height - 1);
            const float p00 = (float)in[(size_t)y0 * in_pitch + x0], p10 = (float)in[(size_t)y0 * in_pitch + x1];
            const float p01 = (float)in[(size_t)y1 * in_pitch + x0], p11 = (float)in[(size_t)y1 * in_pitch + x1];
            const float top = fmaf(fx, p10 - p00, p00);
            const float bottom = fmaf(fx, p11 - p01, p01);
            const float v = fmaf(fy, bottom - top, top);
            float q = rintf(v);
            q = q < 0.0f ? 0.0f : (q > 255.0f ? 255.0f : q);
            out[(size_t)y * out_pitch + x] = (uint8_t)q;
        }
    return 0;
}
