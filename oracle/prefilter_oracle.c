/*
 * prefilter_oracle.c -- TEST INFRASTRUCTURE ONLY (part of the oracle library).
 *
 * The frame preprocessing of PAPER.md §2.1 as the paper implements it on the
 * GPU (§3.3.1, App. C P:545-567 Gaussian, App. D P:569-589 median), written
 * out step by step; the readings R30-R34 of DESIGN.md §2 fix what the paper leaves open:
 *
 *   R30 taps: w_i = exp(-(i-c)^2 / (2 sigma^2)), c = (k-1)/2, i = 0..k-1 (Eq. 1; its
 *       1/(sigma sqrt(2 pi)) factor cancels in the normalisation), computed and
 *       normalised to sum 1 in double, then rounded to float.
 *   R31 separable (§3.3.1 "convolve first the rows and then the columns"): each pass
 *       is App. C's loop over the 1-D window, blur = 0.f; blur += pixel * weight in
 *       ascending tap order, evaluated as fmaf(pixel, weight, blur) (the contraction
 *       nvcc applies to the paper's CUDA code).  The row pass's result stays float
 *       (real arithmetic between the passes); the column pass's sum is rounded to the
 *       nearest integer (ties to even) and clamped to [0, 255] -- ONE quantization to the
 *       u8 frame the model consumes.  (App. C's static_cast<unsigned char> truncation,
 *       applied after each pass, would darken a constant frame by up to 2 grey levels
 *       whenever the float taps sum below 1; DESIGN.md records the choice.)
 *   R32 borders: App. C/D "Clamp filter to the image border", to the last valid index.
 *   R33 median: the 3x3 window ("the surrounding 8 pixels ... as well as the current
 *       pixel", §3.1.1), clamped, its middle order statistic (App. D sorts the
 *       window and takes window[len/2]).
 *   R34 order: Gaussian, then median, on the raw frame; the result replaces the frame
 *       for the whole DMSGM step (S4 and S8).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "dmsgm_oracle.h"

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* R30 */
int dmsgm_oracle_gauss_taps(int size, float sigma, float* taps) {
    if (!taps || size < 1 || size % 2 == 0 || size > 15 || !(sigma > 0.0f)) return -1;
    const int c = (size - 1) / 2;
    double t[15], sum = 0.0;
    for (int i = 0; i < size; ++i) {
        const double x = (double)(i - c);
        t[i] = exp(-(x * x) / (2.0 * (double)sigma * (double)sigma));
        sum += t[i];
    }
    for (int i = 0; i < size; ++i) taps[i] = (float)(t[i] / sum);
    return 0;
}

/* R31 + R32: the row pass (u8 frame -> float image). */
static void gauss_rows(int width, int height, const uint8_t* in, size_t in_pitch, float* out, const float* taps,
                       int size) {
    const int half = (size - 1) / 2;
    for (int r = 0; r < height; ++r)
        for (int col = 0; col < width; ++col) {
            float blur = 0.0f;
            for (int i = -half; i <= half; ++i) {
                const float pixel = (float)in[(size_t)r * in_pitch + clampi(col + i, 0, width - 1)];
                blur = fmaf(pixel, taps[i + half], blur);
            }
            out[(size_t)r * width + col] = blur;
        }
}

/* R31 + R32: the column pass (float image -> u8 frame, one rounding). */
static void gauss_cols(int width, int height, const float* in, uint8_t* out, size_t out_pitch, const float* taps,
                       int size) {
    const int half = (size - 1) / 2;
    for (int r = 0; r < height; ++r)
        for (int col = 0; col < width; ++col) {
            float blur = 0.0f;
            for (int i = -half; i <= half; ++i)
                blur = fmaf(in[(size_t)clampi(r + i, 0, height - 1) * width + col], taps[i + half], blur);
            float q = rintf(blur);                          /* nearest, ties to even */
            q = q < 0.0f ? 0.0f : (q > 255.0f ? 255.0f : q);
            out[(size_t)r * out_pitch + col] = (uint8_t)q;
        }
}

/* R33: insertion sort of the clamped (2 radius + 1)^2 window, middle element (App. D). */
static void median_filter(int width, int height, const uint8_t* in, size_t in_pitch, uint8_t* out,
                          size_t out_pitch, int radius) {
    uint8_t window[81];
    for (int r = 0; r < height; ++r)
        for (int col = 0; col < width; ++col) {
            int n = 0;
            for (int i = -radius; i <= radius; ++i)
                for (int j = -radius; j <= radius; ++j)
                    window[n++] = in[(size_t)clampi(r + i, 0, height - 1) * in_pitch + clampi(col + j, 0, width - 1)];
            for (int a = 1; a < n; ++a) {           /* insertionSort(window, window_len) */
                const uint8_t v = window[a];
                int b = a - 1;
                while (b >= 0 && window[b] > v) {
                    window[b + 1] = window[b];
                    --b;
                }
                window[b + 1] = v;
            }
            out[(size_t)r * out_pitch + col] = window[n / 2];
        }
}

/* R34: Gaussian (gauss_size 1 = off) then median (median_radius 0 = off). */
int dmsgm_oracle_prefilter(int width, int height, const uint8_t* in, size_t in_pitch, uint8_t* out,
                           size_t out_pitch, int gauss_size, float gauss_sigma, int median_radius) {
    if (!in || !out || width < 1 || height < 1 || in_pitch < (size_t)width || out_pitch < (size_t)width) return -1;
    if (median_radius < 0 || median_radius > 4) return -1;
    float taps[15];
    if (dmsgm_oracle_gauss_taps(gauss_size, gauss_sigma, taps)) return -1;
    const size_t n = (size_t)width * height;
    uint8_t* a = (uint8_t*)malloc(n);
    uint8_t* b = (uint8_t*)malloc(n);
    float* f = (float*)malloc(n * sizeof(float));
    if (!a || !b || !f) {
        free(a);
        free(b);
        free(f);
        return -2;
    }
    for (int r = 0; r < height; ++r) memcpy(a + (size_t)r * width, in + (size_t)r * in_pitch, width);
    if (gauss_size > 1) {
        gauss_rows(width, height, a, width, f, taps, gauss_size);
        gauss_cols(width, height, f, a, width, taps, gauss_size);
    }
    if (median_radius > 0) {
        median_filter(width, height, a, width, b, width, median_radius);
        memcpy(a, b, n);
    }
    for (int r = 0; r < height; ++r) memcpy(out + (size_t)r * out_pitch, a + (size_t)r * width, width);
    free(a);
    free(b);
    free(f);
    return 0;
}
